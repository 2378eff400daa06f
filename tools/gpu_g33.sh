cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SRMDP_LIB=ablibs/band.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_user.py -q -x -rfs > gpurun_out/g33_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g33_parity.log
timeout 1500 python tools/ab.py --rounds 2 --config cfg5 ablibs/cur.so ablibs/band.so > gpurun_out/g33_cfg5.log 2>&1
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/band.so > gpurun_out/g33_cfg4.log 2>&1
