# Final round-2 evidence after the 128-thread d > 8 kernel: smoke, bench (cfg4 + cfg5), reference arm, cfg5 ncu capture, d = 22 largest
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g48_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g48_smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/g48_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/g48_bench.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/g48_bench_ref.log 2>&1
timeout 1500 python bench.py --config cfg5 --M 16384 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g48_cfg5_M16384.log 2>&1
timeout 300 python tools/profile_step.py cfg5 > gpurun_out/g48_plain5.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -f -o gpurun_out/r02h_cfg5_i3 python tools/profile_step.py cfg5 > gpurun_out/g48_ncu5.log 2>&1
