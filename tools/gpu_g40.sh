cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/cs.so > gpurun_out/g40_cfg5.log 2>&1
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/cs.so > gpurun_out/g40_cfg4.log 2>&1
