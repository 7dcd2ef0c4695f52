# correctness of the WS variant (small, bounded) then A/B
export RQMC_B200_LIB=$PWD/paper_1408_5526_b200/librqmc_b200_ws.so
timeout 300 python -m pytest tests -m gpu -q -x -k "theta_vs_reference or x1_theta or xhash_theta_bit_exact and d20 or c2_theta" > gpurun_out/ws_tests.log 2>&1; echo wstests=$?; tail -3 gpurun_out/ws_tests.log
unset RQMC_B200_LIB
LIBS="cur ws" ROUNDS=2 bash tools/gpu_ab2.sh "--reps 1024" "--reps 512 --generator philox" "--workload c3 --reps 64" "--workload c5 --reps 128"
