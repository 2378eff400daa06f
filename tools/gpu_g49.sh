# d = 22 largest benchmark and cfg5 executed-flop counts with the 128-thread d > 8 kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python tools/largest.py 22 3200 > gpurun_out/g49_largest.log 2>&1; echo "rc=$?" >> gpurun_out/g49_largest.log
timeout 1200 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__inst_executed_pipe_fp64_op_dmma.sum \
  --clock-control none -k regex:step_kernel --csv --log-file gpurun_out/g49_exec5.csv python tools/profile_step.py cfg5 > gpurun_out/g49_exec5.log 2>&1; echo "rc=$?" >> gpurun_out/g49_exec5.log
