cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/ch3.so ablibs/ch10.so ablibs/ju2.so > gpurun_out/g50_cfg5.log 2>&1
