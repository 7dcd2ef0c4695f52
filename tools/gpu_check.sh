# Full GPU test suite + smoke + the main bench lines (short).
mkdir -p gpurun_out; rm -f gpurun_out/quick.json
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for wl in "c2" "c2 --generator philox" "c2 --generator sobol-gray" "c3 --reps 64" "c5 --reps 128" "c4" "c4 --generator philox"; do
  timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 3 >> gpurun_out/quick.json 2>>gpurun_out/quick.err
done
python tools/bench_table.py gpurun_out/quick.json
