# full GPU suite, the bounds-checked build over the parity suites, A/B (counters, MMA split), bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/g3_all.log 2>&1; echo "rc=$?" >> gpurun_out/g3_all.log
SRMDP_LIB=ablibs/bounds.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_user.py -q -rf --timeout 1200 > gpurun_out/g3_bounds.log 2>&1; echo "rc=$?" >> gpurun_out/g3_bounds.log
timeout 900 python tools/ab.py --rounds 4 paper_2407_21085_b200/libsrmdp_b200.so ablibs/cnt0.so ablibs/cnt1.so ablibs/kbal0.so ablibs/r1.so > gpurun_out/g3_ab_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 2 --config cfg5 paper_2407_21085_b200/libsrmdp_b200.so ablibs/cnt0.so ablibs/kbal0.so ablibs/r1.so > gpurun_out/g3_ab_cfg5.log 2>&1
timeout 900 python bench.py > gpurun_out/g3_bench.log 2>&1; echo "rc=$?" >> gpurun_out/g3_bench.log
