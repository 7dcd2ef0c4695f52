# Round check: GPU parity suite, then the full measurement sweep (tools/gpu_sweep.sh).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
P=${P:-gpurun_out/r01g} bash tools/gpu_sweep.sh > gpurun_out/sweep_table.txt 2>&1
tail -40 gpurun_out/sweep_table.txt
