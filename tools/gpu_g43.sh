# Final round-2 evidence from the committed tree (streamed record scratch at d > 8).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "from paper_2407_21085_b200 import build as b; b.build()" > gpurun_out/g43_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rfs --timeout 900 > gpurun_out/g43_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/g43_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g43_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g43_smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/g43_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/g43_bench.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/g43_bench_ref.log 2>&1
timeout 300 python tools/profile_step.py cfg5 > gpurun_out/g43_plain5.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -f -o gpurun_out/r02g_cfg5_i3 python tools/profile_step.py cfg5 > gpurun_out/g43_ncu5.log 2>&1
