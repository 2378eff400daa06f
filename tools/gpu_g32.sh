cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/ab.py --rounds 2 --config cfg5 ablibs/cur.so ablibs/xstart.so > gpurun_out/g32_cfg5.log 2>&1
