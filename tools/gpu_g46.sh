cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/t64.so > gpurun_out/g46_cfg5.log 2>&1
