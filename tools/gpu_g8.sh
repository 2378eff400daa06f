cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/ab.py --rounds 3 --config cfg5 ablibs/bm.so ablibs/ws0.so ablibs/r1.so > gpurun_out/g8_ab_cfg5.log 2>&1
timeout 900 python tools/ab.py --rounds 3 ablibs/bm.so ablibs/ws0.so ablibs/r1.so > gpurun_out/g8_ab_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 3 --config cfg3 ablibs/bm.so ablibs/ws0.so ablibs/r1.so > gpurun_out/g8_ab_cfg3.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/g8_all.log 2>&1; echo "rc=$?" >> gpurun_out/g8_all.log
