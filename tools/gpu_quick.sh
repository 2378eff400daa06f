# quick GPU check: parity subset + cfg4 bench (no cpu baseline)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 600 -x -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_quick.log
if [ -n "$PROFILE" ]; then
  timeout 300 python tools/profile_step.py cfg4 > gpurun_out/profile_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 14 -c 1 -f -o gpurun_out/step_cfg4_$PROFILE python tools/profile_step.py cfg4 > gpurun_out/ncu_full.log 2>&1
fi
