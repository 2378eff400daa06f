cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/ab.py --rounds 3 --config cfg5 ablibs/cur.so ablibs/ws0.so ablibs/r1.so > gpurun_out/g7_ab_cfg5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "d19 or d12 or d11 or trunc" > gpurun_out/g7_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g7_parity.log
