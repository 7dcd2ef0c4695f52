mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bigdim.py -q -x > gpurun_out/bigdim.log 2>&1; echo bigdim=$?; tail -15 gpurun_out/bigdim.log
LIBS="old new" ROUNDS=2 bash tools/gpu_ab2.sh "--workload c2" "--workload c3 --reps 64" "--workload c4" "--workload c5 --reps 128"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
