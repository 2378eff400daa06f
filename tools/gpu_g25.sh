cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rfs -x -k "p2p or nccl or nvls or checkpoint" > gpurun_out/g25_xw.log 2>&1; echo "rc=$?" >> gpurun_out/g25_xw.log
timeout 900 python tools/ab.py --rounds 3 ablibs/cur.so ablibs/xw.so > gpurun_out/g25_cfg4.log 2>&1
timeout 600 python - > gpurun_out/g25_p2p_time.log 2>&1 <<'PY'
# one GPU: the plain solve vs the fused exchange with separate flag kernels vs in-kernel flags (cfg4)
import sys, time; sys.path.insert(0, '.')
import workloads
from paper_2407_21085_b200 import srmdp
w = workloads.cfg4()
for name, fl in (("plain", 0), ("p2p_separate", srmdp.FLAG_P2P_EXCHANGE), ("p2p_inkernel", srmdp.FLAG_P2P_EXCHANGE | srmdp.FLAG_INKERNEL_FLAGS)):
    with srmdp.Solver(w, flags=srmdp.FLAG_TIME_KERNELS | fl) as s:
        s.solve()
        t = []
        for _ in range(3):
            t0 = time.perf_counter(); s.solve(); t.append(time.perf_counter() - t0)
        st = s.stats()
        print(name, "solve_s", min(t), "kernel_ms", st["kernel_ms"], "gather_ms", st["gather_ms"])
PY
