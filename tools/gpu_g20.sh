cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/c4.so ablibs/c4ju1.so ablibs/ju1.so > gpurun_out/g20_ab_cfg4.log 2>&1
timeout 1200 python tools/ab.py --rounds 3 --config cfg3 ablibs/cur.so ablibs/c4.so ablibs/c4ju1.so ablibs/ju1.so > gpurun_out/g20_ab_cfg3.log 2>&1
