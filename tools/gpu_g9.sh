cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python tools/ab.py --rounds 3 --config cfg5 ablibs/bm.so ablibs/p2u0.so ablibs/p2u2.so ablibs/kbal0.so ablibs/hdju2.so ablibs/hdbu4.so ablibs/r1.so > gpurun_out/g9_ab_cfg5.log 2>&1
timeout 900 python tools/ab.py --rounds 3 ablibs/bm.so ablibs/p2u0.so ablibs/p2u2.so ablibs/kbal0.so > gpurun_out/g9_ab_cfg4.log 2>&1
