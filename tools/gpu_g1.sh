# Parity-gap tests (round 2) + full GPU suite + a bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 1200 -k "trunc or full_sweep or cells_bit_exact or dump_unsupported or 1e-10 or L1e or full_size" > gpurun_out/g1_new.log 2>&1; echo "rc=$?" >> gpurun_out/g1_new.log
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/g1_all.log 2>&1; echo "rc=$?" >> gpurun_out/g1_all.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/g1_bench.log 2>&1; echo "rc=$?" >> gpurun_out/g1_bench.log
