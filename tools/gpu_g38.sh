# sanity run of the committed tree: GPU tests, smoke, bench (driver invocation)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfs --timeout 1200 > gpurun_out/g38_all.log 2>&1; echo "rc=$?" >> gpurun_out/g38_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g38_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/g38_smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/g38_bench.log 2>&1; echo "rc=$?" >> gpurun_out/g38_bench.log
