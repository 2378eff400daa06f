cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg3 --no-cpu-baseline > gpurun_out/g39_cfg3.log 2>&1
timeout 1500 python bench.py --config cfg5 --M 16384 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g39_cfg5_M16384.log 2>&1
timeout 900 python bench.py --config cfg2 --no-cpu-baseline --no-cfg5 > gpurun_out/g39_cfg2.log 2>&1
