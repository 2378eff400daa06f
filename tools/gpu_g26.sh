cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/bu0.so ablibs/bu5.so > gpurun_out/g26_cfg5.log 2>&1
