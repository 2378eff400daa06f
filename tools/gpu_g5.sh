# A/B: 128-thread CTAs (7 / 6 per SM), d > 8 start-point unroll
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/ab.py --rounds 3 paper_2407_21085_b200/libsrmdp_b200.so ablibs/t128c7.so ablibs/t128c6.so > gpurun_out/g5_ab_cfg4.log 2>&1
timeout 900 python tools/ab.py --rounds 3 --config cfg3 paper_2407_21085_b200/libsrmdp_b200.so ablibs/t128c7.so ablibs/t128c6.so > gpurun_out/g5_ab_cfg3.log 2>&1
timeout 1200 python tools/ab.py --rounds 2 --config cfg5 paper_2407_21085_b200/libsrmdp_b200.so ablibs/su1.so ablibs/su2.so ablibs/t128c7.so ablibs/t128c6.so > gpurun_out/g5_ab_cfg5.log 2>&1
