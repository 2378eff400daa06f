cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 1200 > gpurun_out/g11_all.log 2>&1; echo "rc=$?" >> gpurun_out/g11_all.log
timeout 1500 python tools/ab.py --rounds 2 --config cfg5 ablibs/cur.so ablibs/r1.so > gpurun_out/g11_ab_cfg5.log 2>&1
timeout 900 python bench.py > gpurun_out/g11_bench.log 2>&1; echo "rc=$?" >> gpurun_out/g11_bench.log
timeout 600 python tools/step_profile.py cfg4 > gpurun_out/g11_stepprof4.log 2>&1
timeout 600 python tools/step_profile.py cfg5 > gpurun_out/g11_stepprof5.log 2>&1
