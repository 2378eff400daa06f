# evidence for the current kernels: tests, smoke, bench, launch list, ncu full captures, executed flops
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/g18_all.log 2>&1; echo "rc=$?" >> gpurun_out/g18_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g18_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/g18_smoke.log
timeout 900 python bench.py > gpurun_out/g18_bench.log 2>&1; echo "rc=$?" >> gpurun_out/g18_bench.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/g18_bench_ref.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g18_launches.csv python bench.py --no-cfg5 --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/g18_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 14 -c 1 -f -o gpurun_out/r02b_cfg4_i15 python tools/profile_step.py cfg4 > gpurun_out/g18_ncu4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -f -o gpurun_out/r02b_cfg5_i3 python tools/profile_step.py cfg5 > gpurun_out/g18_ncu5.log 2>&1
M="smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum"
for c in cfg4 cfg5; do
  timeout 1200 ncu --metrics $M --clock-control none -k regex:step_kernel --csv --log-file gpurun_out/g18_exec_$c.csv python tools/profile_step.py $c > gpurun_out/g18_exec_$c.log 2>&1
done
