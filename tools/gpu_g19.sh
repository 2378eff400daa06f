cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SRMDP_LIB=ablibs/reuse.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "solve_parity or trunc or full_sweep or lp0 or equi" > gpurun_out/g19_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g19_parity.log
timeout 2400 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/reuse.so > gpurun_out/g19_ab_cfg5.log 2>&1
timeout 1200 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/reuse.so > gpurun_out/g19_ab_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 3 --config cfg3 ablibs/cur.so ablibs/reuse.so > gpurun_out/g19_ab_cfg3.log 2>&1
