# ncu evidence for the current kernels: full captures (cfg4 i=15, cfg5 i=3), executed FP64 flops over every launch, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --query-metrics 2>/dev/null | grep -iE "dmma|pipe_fp64|sass_thread_inst_executed_op_d" > gpurun_out/g4_metrics.txt
timeout 300 python tools/profile_step.py cfg4 > gpurun_out/g4_plain4.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 14 -c 1 -f -o gpurun_out/r02_cfg4_i15 python tools/profile_step.py cfg4 > gpurun_out/g4_ncu4.log 2>&1
timeout 300 python tools/profile_step.py cfg5 > gpurun_out/g4_plain5.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -f -o gpurun_out/r02_cfg5_i3 python tools/profile_step.py cfg5 > gpurun_out/g4_ncu5.log 2>&1
M="smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"
DM=$(grep -oE "^ *[a-z_]+__[a-z_]*dmma[a-z_]*" gpurun_out/g4_metrics.txt | head -1 | tr -d ' ')
echo "dmma metric: $DM" > gpurun_out/g4_dmma.txt
for c in cfg4 cfg5; do
  timeout 1200 ncu --metrics $M${DM:+,$DM.sum} --clock-control none -k regex:step_kernel --csv --log-file gpurun_out/g4_exec_$c.csv python tools/profile_step.py $c > gpurun_out/g4_exec_$c.log 2>&1
done
timeout 900 python bench.py --no-cfg5 --no-cpu-baseline > gpurun_out/g4_bench_plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g4_launches.csv python bench.py --no-cfg5 --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/g4_ncu_launches.log 2>&1
