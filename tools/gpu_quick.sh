# quick GPU check: parity tests + short benches of the main workloads
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/quick.json
for w in c2 c3 c5; do timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 3 $([ $w != c2 ] && echo --reps 64) >> gpurun_out/quick.json 2>>gpurun_out/quick.err; done
timeout 300 python bench.py --generator philox --no-cpu-baseline --steps 3 >> gpurun_out/quick.json 2>>gpurun_out/quick.err
for g in philox rasrap-recursive; do timeout 300 python bench.py --workload c4 --generator $g --steps 3 >> gpurun_out/quick.json 2>>gpurun_out/quick.err; done
python tools/bench_table.py gpurun_out/quick.json
