cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/shard_efficiency.py cfg4 > gpurun_out/g31_shard4.log 2>&1
timeout 1500 python tools/shard_efficiency.py cfg5 > gpurun_out/g31_shard5.log 2>&1
