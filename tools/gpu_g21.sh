# timing-only decomposition of the per-path-start cost (wrong-result builds; N = 2 sweeps weigh the fixed part)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/ab.py --rounds 3 --N 2 ablibs/cur.so ablibs/xp2.so ablibs/xfold.so ablibs/xstart.so > gpurun_out/g21_cfg4_N2.log 2>&1
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/xp2.so ablibs/xfold.so ablibs/xstart.so > gpurun_out/g21_cfg4.log 2>&1
timeout 1200 python tools/ab.py --rounds 2 --config cfg5 ablibs/cur.so ablibs/xp2.so ablibs/xfold.so ablibs/xstart.so > gpurun_out/g21_cfg5.log 2>&1
