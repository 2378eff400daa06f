# Full round measurement on one B200: tests, smoke, bench (+clocks), launch list, top-kernel ncu capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
(nproc; lscpu | grep "Model name") > gpurun_out/host.txt
timeout 120 ./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_plain_for_ncu.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py > gpurun_out/ncu_launches.log 2>&1
timeout 300 python tools/profile_step.py cfg4 > gpurun_out/profile_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 14 -c 1 -f -o gpurun_out/step_cfg4_$TAG python tools/profile_step.py cfg4 > gpurun_out/ncu_full.log 2>&1
