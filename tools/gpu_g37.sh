cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/tc2.so ablibs/nocarve.so > gpurun_out/g37_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 3 --config cfg3 ablibs/cur.so ablibs/tc2.so ablibs/nocarve.so > gpurun_out/g37_cfg3.log 2>&1
