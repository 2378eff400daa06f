cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/WARP_SOLVE.so ablibs/MMA_REUSE.so ablibs/MMA_ACC2.so > gpurun_out/g47_cfg5.log 2>&1
