cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/cs2.so > gpurun_out/g41_cfg5.log 2>&1
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/cs2.so > gpurun_out/g41_cfg4.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -rfs > gpurun_out/g41_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g41_parity.log
