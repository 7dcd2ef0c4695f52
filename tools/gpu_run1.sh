set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
cat gpurun_out/bench_c2.json
for g in philox sobol-gray sfc64 rasrap-counter; do timeout 300 python bench.py --generator $g --no-cpu-baseline --steps 3 >> gpurun_out/bench_c2_gens.json 2>>gpurun_out/bench_err.log; done
timeout 600 python bench.py --workload c3 --reps 64 --steps 3 >> gpurun_out/bench_c3.json 2>>gpurun_out/bench_err.log
timeout 600 python bench.py --workload c5 --reps 64 --steps 3 >> gpurun_out/bench_c5.json 2>>gpurun_out/bench_err.log
for g in philox sfc64 rasrap-recursive sobol-gray; do timeout 300 python bench.py --workload c4 --generator $g --steps 3 >> gpurun_out/bench_c4.json 2>>gpurun_out/bench_err.log; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>>gpurun_out/bench_err.log
cat gpurun_out/*.json | cut -c1-400
