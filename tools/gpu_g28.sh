# final round-2 evidence: tests (product and bounds-checked builds), smoke, bench, reference arm, launch list, ncu captures, executed flops
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfs --timeout 1200 > gpurun_out/g28_all.log 2>&1; echo "rc=$?" >> gpurun_out/g28_all.log
SRMDP_LIB=ablibs/bounds.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_user.py -q -rfs --timeout 1200 > gpurun_out/g28_bounds.log 2>&1; echo "rc=$?" >> gpurun_out/g28_bounds.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g28_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/g28_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/g28_bench.log 2>&1; echo "rc=$?" >> gpurun_out/g28_bench.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/g28_bench_ref.log 2>&1
timeout 600 python tools/step_profile.py cfg4 > gpurun_out/g28_stepprof4.log 2>&1
timeout 600 python tools/step_profile.py cfg5 > gpurun_out/g28_stepprof5.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g28_launches.csv python bench.py --no-cfg5 --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/g28_ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 14 -c 1 -f -o gpurun_out/r02d_cfg4_i15 python tools/profile_step.py cfg4 > gpurun_out/g28_ncu4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -f -o gpurun_out/r02d_cfg5_i3 python tools/profile_step.py cfg5 > gpurun_out/g28_ncu5.log 2>&1
