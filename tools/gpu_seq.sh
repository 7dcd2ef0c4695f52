timeout 900 python -m pytest tests/test_gpu_seq.py -x -q > gpurun_out/pytest_seq.log 2>&1; echo seq=$?; tail -30 gpurun_out/pytest_seq.log
rm -f gpurun_out/seq.json
for g in twister xorwow kakutani; do timeout 300 python bench.py --generator $g --no-cpu-baseline --steps 3 >> gpurun_out/seq.json 2>>gpurun_out/seq.err; timeout 300 python bench.py --workload c3 --reps 64 --generator $g --no-cpu-baseline --steps 3 >> gpurun_out/seq.json 2>>gpurun_out/seq.err; done
python tools/bench_table.py gpurun_out/seq.json; tail -5 gpurun_out/seq.err
