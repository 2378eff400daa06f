cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/cen2.so ablibs/mag.so ablibs/cen2mag.so > gpurun_out/g14_ab_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 3 --config cfg3 ablibs/cur.so ablibs/cen2.so ablibs/mag.so ablibs/cen2mag.so > gpurun_out/g14_ab_cfg3.log 2>&1
timeout 2400 python tools/ab.py --rounds 2 --config cfg5 ablibs/cur.so ablibs/cen2.so ablibs/mag.so ablibs/cen2mag.so > gpurun_out/g14_ab_cfg5.log 2>&1
SRMDP_LIB=ablibs/cen2mag.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_exact or trunc or bookkeeping or cfg1 or cfg2" > gpurun_out/g14_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g14_parity.log
