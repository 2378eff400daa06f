cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python tools/ab.py --rounds 3 --config cfg5 ablibs/su0.so ablibs/bm.so ablibs/cnt2.so ablibs/cnt0.so ablibs/r1.so > gpurun_out/g10_ab_cfg5.log 2>&1
timeout 1200 python tools/ab.py --rounds 3 ablibs/su0.so ablibs/ju1.so ablibs/c4.so ablibs/cnt0.so > gpurun_out/g10_ab_cfg4.log 2>&1
