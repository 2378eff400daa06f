cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python tools/ab.py --rounds 3 --config cfg5 ablibs/sc5.so ablibs/sc10.so ablibs/cur.so > gpurun_out/g16_ab_cfg5.log 2>&1
