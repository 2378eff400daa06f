# sqrt check, parity subset, A/B of r1 vs current vs current-without-fast-math
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sqrt_check tools/sqrt_check.cu && timeout 300 /tmp/sqrt_check > gpurun_out/g2_sqrt.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf --timeout 600 -x -k "not full_sweep and not full_size" > gpurun_out/g2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/g2_parity.log
timeout 900 python tools/ab.py --rounds 4 paper_2407_21085_b200/libsrmdp_b200.so ablibs/r1.so ablibs/nofast.so > gpurun_out/g2_ab_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 2 --config cfg5 paper_2407_21085_b200/libsrmdp_b200.so ablibs/r1.so ablibs/nofast.so > gpurun_out/g2_ab_cfg5.log 2>&1
