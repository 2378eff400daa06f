cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "reciprocal or sqrt" > gpurun_out/g22_rcp.log 2>&1; echo "rc=$?" >> gpurun_out/g22_rcp.log
SRMDP_LIB=ablibs/sfast.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_exact or solve_parity or trunc or full_sweep" > gpurun_out/g22_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g22_parity.log
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/sfast.so > gpurun_out/g22_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 3 --N 2 ablibs/cur.so ablibs/sfast.so > gpurun_out/g22_cfg4N2.log 2>&1
timeout 900 python tools/ab.py --rounds 3 --config cfg3 ablibs/cur.so ablibs/sfast.so > gpurun_out/g22_cfg3.log 2>&1
timeout 1500 python tools/ab.py --rounds 2 --config cfg5 ablibs/cur.so ablibs/sfast.so > gpurun_out/g22_cfg5.log 2>&1
