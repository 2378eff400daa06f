cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mc_probe tools/mc_probe.cu -lcuda > gpurun_out/g12_mc_build.log 2>&1 && timeout 120 /tmp/mc_probe > gpurun_out/g12_mc_probe.log 2>&1; echo "rc=$?" >> gpurun_out/g12_mc_probe.log
nvidia-smi topo -m > gpurun_out/g12_topo.txt 2>&1; nvidia-smi -q | grep -iA3 "fabric\|nvlink" | head -40 >> gpurun_out/g12_topo.txt 2>&1
SRMDP_LIB=ablibs/bounds.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_user.py -q -rf --timeout 1200 > gpurun_out/g12_bounds.log 2>&1; echo "rc=$?" >> gpurun_out/g12_bounds.log
