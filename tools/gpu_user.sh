# GPU check of the NVRTC / user-problem path + the static parity suite + cfg4 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_user.py -q -rf --timeout 600 > gpurun_out/pytest_user.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_user.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 600 -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_quick.log
