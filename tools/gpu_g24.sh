cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SRMDP_LIB=ablibs/kdbits.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_exact or cells" > gpurun_out/g24_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g24_parity.log
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/kdbits.so > gpurun_out/g24_cfg4.log 2>&1
timeout 1500 python tools/ab.py --rounds 2 --config cfg5 ablibs/cur.so ablibs/kdbits.so > gpurun_out/g24_cfg5.log 2>&1
