# Full measurement sweep: default bench line (C2 rasrap, with CPU baseline),
# every generator on C2, C3/C5 samples with CPU baseline, C4 streams, reference arm.
rm -f gpurun_out/sweep.json
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
cat gpurun_out/bench_default.json >> gpurun_out/sweep.json
for g in rasrap-counter philox sobol-gray sobol-counter sfc64 twister xorwow kakutani; do
  timeout 300 python bench.py --generator $g --no-cpu-baseline --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err
done
timeout 600 python bench.py --workload c1 --steps 5 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err
timeout 900 python bench.py --workload c3 --reps 64 --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err
timeout 900 python bench.py --workload c5 --reps 64 --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err
for g in philox xorwow; do timeout 600 python bench.py --workload c3 --reps 64 --generator $g --no-cpu-baseline --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err; done
for g in philox sfc64 rasrap-recursive sobol-gray; do timeout 300 python bench.py --workload c4 --generator $g --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>>gpurun_out/sweep.err
cat gpurun_out/bench_reference.json >> gpurun_out/sweep.json
python tools/bench_table.py gpurun_out/sweep.json
python -c "import __graft_entry__ as g; g.smoke()"
