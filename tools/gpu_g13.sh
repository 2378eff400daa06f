cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mc_probe tools/mc_probe.cu -lcuda > gpurun_out/g13_mc_build.log 2>&1 && timeout 120 /tmp/mc_probe > gpurun_out/g13_mc_probe.log 2>&1; echo "rc=$?" >> gpurun_out/g13_mc_probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rs -x -k "nvls or p2p or nccl" > gpurun_out/g13_nvls.log 2>&1; echo "rc=$?" >> gpurun_out/g13_nvls.log
