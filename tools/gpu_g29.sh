cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q -rf > gpurun_out/g29_fuzz.log 2>&1; echo "rc=$?" >> gpurun_out/g29_fuzz.log
