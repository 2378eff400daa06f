# the paper's MSE tables with the final round-2 kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3000 python tools/mse_table.py > gpurun_out/g36_mse_table.md 2> gpurun_out/g36_mse.err; echo "rc=$?" >> gpurun_out/g36_mse.err
