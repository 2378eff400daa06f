# one ncu --set full capture of the cfg4 step kernel at i=15 (after a plain run exits 0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/profile_step.py ${CFG:-cfg4} > gpurun_out/profile_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s ${SKIP:-14} -c 1 -f -o gpurun_out/step_${CFG:-cfg4}_$TAG python tools/profile_step.py ${CFG:-cfg4} > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full.log
