# A/B of builds on cfg4 and cfg5 (+ parity subset on each alternative)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_A.log 2>&1
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_A5.log 2>&1
for so in $ALTS; do
  b=$(basename $so .so)
  SRMDP_LIB=$so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "solve_parity or full_size" > gpurun_out/pytest_$b.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$b.log
  SRMDP_LIB=$so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$b.log 2>&1
  SRMDP_LIB=$so timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench5_$b.log 2>&1
done
