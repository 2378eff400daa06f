# A/B: two DMMA accumulator chains, warp triangular solves (d > 8)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/ab.py --rounds 2 --config cfg5 paper_2407_21085_b200/libsrmdp_b200.so ablibs/acc1.so ablibs/ws0.so > gpurun_out/g6_ab_cfg5.log 2>&1
timeout 900 python tools/ab.py --rounds 3 paper_2407_21085_b200/libsrmdp_b200.so ablibs/acc1.so > gpurun_out/g6_ab_cfg4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "d19 or d12 or d11 or 1e-10 or trunc" > gpurun_out/g6_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g6_parity.log
