cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/t192.so > gpurun_out/g51_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 3 --config cfg3 ablibs/cur.so ablibs/t192.so > gpurun_out/g51_cfg3.log 2>&1
SRMDP_LIB=ablibs/t192.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -rfs > gpurun_out/g51_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g51_parity.log
