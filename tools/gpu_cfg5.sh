cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1
SRMDP_LIB=paper_2407_21085_b200/libsrmdp_b200_lb3hd.so timeout 900 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg5_lb3hd.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 600 -k "d19 or cfg5" > gpurun_out/pytest_d19.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_d19.log
timeout 300 python tools/profile_step.py cfg5 > gpurun_out/profile_plain5.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -f -o gpurun_out/step_cfg5 python tools/profile_step.py cfg5 > gpurun_out/ncu_full5.log 2>&1
