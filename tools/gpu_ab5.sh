# A/B of builds on cfg5 only
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for so in default $ALTS; do
  b=$(basename $so .so)
  lib=""; [ "$so" != default ] && lib="SRMDP_LIB=$so"
  env $lib timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b5_$b.log 2>&1
done
