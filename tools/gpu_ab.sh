# A/B: bench the default build and the alternative builds given in $ALTS (space-separated .so paths)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 600 -k "not full_size" --deselect tests/test_gpu_parity.py::test_errors > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_A.log 2>&1
for so in $ALTS; do
  SRMDP_LIB=$so timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$(basename $so .so).log 2>&1
done
