cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/g0_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g0_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/g0_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/g0_bench.log
