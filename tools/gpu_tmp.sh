LIBS="cur ws1 ws1m2 ws1m4" ROUNDS=2 bash tools/gpu_ab2.sh "--reps 1024" 
export RQMC_B200_LIB=$PWD/paper_1408_5526_b200/librqmc_b200_ws1.so
TAG=ws1 bash tools/gpu_prof_sass.sh > /dev/null 2>&1
unset RQMC_B200_LIB
