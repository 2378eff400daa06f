cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
free -g > gpurun_out/g17_free.txt
timeout 1800 python tools/largest.py 22 3200 > gpurun_out/g17_largest.log 2>&1; echo "rc=$?" >> gpurun_out/g17_largest.log
