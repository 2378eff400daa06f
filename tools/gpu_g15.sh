cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/sc2.so ablibs/sc3.so ablibs/sc5.so > gpurun_out/g15_ab_cfg5.log 2>&1
SRMDP_LIB=ablibs/sc3.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "d19 or d12 or d11" > gpurun_out/g15_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g15_parity.log
