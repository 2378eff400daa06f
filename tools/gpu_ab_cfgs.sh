# A/B of builds on cfg3, cfg4 (and cfg5 if CFG5=1) + parity subset of the default build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 600 -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
for so in default $ALTS; do
  b=$(basename $so .so)
  lib=""; [ "$so" != default ] && lib="SRMDP_LIB=$so"
  env $lib timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b3_$b.log 2>&1
  env $lib timeout 600 python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b4_$b.log 2>&1
  [ -n "$CFG5" ] && env $lib timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b5_$b.log 2>&1
done
