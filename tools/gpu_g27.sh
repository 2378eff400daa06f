cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -rfs -x > gpurun_out/g27_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g27_parity.log
timeout 1800 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/fastonly.so > gpurun_out/g27_cfg5.log 2>&1
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/fastonly.so > gpurun_out/g27_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 3 --config cfg3 ablibs/cur.so ablibs/fastonly.so > gpurun_out/g27_cfg3.log 2>&1
