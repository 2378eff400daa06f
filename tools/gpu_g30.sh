cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SRMDP_LIB=ablibs/ahead.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_exact or cells or solve_parity" > gpurun_out/g30_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g30_parity.log
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/ahead.so > gpurun_out/g30_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 3 --config cfg3 ablibs/cur.so ablibs/ahead.so > gpurun_out/g30_cfg3.log 2>&1
