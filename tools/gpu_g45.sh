# 128-thread CTAs at d > 8: full GPU suite, bounds-checked parity, A/B cfg5 / cfg4 against the committed kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rfs --timeout 900 > gpurun_out/g45_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/g45_pytest_gpu.log
SRMDP_LIB=ablibs/bounds.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_user.py -q -rfs --timeout 1200 > gpurun_out/g45_bounds.log 2>&1; echo "rc=$?" >> gpurun_out/g45_bounds.log
timeout 1500 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/new.so > gpurun_out/g45_cfg5.log 2>&1
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/new.so > gpurun_out/g45_cfg4.log 2>&1
