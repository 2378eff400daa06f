cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 900 -k "d19 or d12 or cfg5 or lp0" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_A5.log 2>&1
for so in $ALTS; do
  SRMDP_LIB=$so timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench5_$(basename $so .so).log 2>&1
done
