# Full measurement sweep: default bench line (C2 rasrap, with CPU baseline),
# every generator on C2, C3/C5 samples with CPU baseline, C4 streams, reference arm.
rm -f gpurun_out/sweep.json
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
cat gpurun_out/bench_default.json >> gpurun_out/sweep.json
for g in rasrap-counter philox sobol-gray sobol-counter sfc64 twister xorwow kakutani; do
  timeout 300 python bench.py --generator $g --no-cpu-baseline --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err
done
timeout 600 python bench.py --workload c1 --steps 5 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err
timeout 900 python bench.py --workload c3 --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err
timeout 900 python bench.py --workload c5 --reps 256 --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err
for g in philox sobol-gray; do timeout 600 python bench.py --workload c5 --reps 128 --generator $g --no-cpu-baseline --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err; done
for g in philox xorwow; do timeout 600 python bench.py --workload c3 --reps 64 --generator $g --no-cpu-baseline --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err; done
for g in philox sfc64 rasrap-recursive sobol-gray; do timeout 300 python bench.py --workload c4 --generator $g --steps 3 >> gpurun_out/sweep.json 2>>gpurun_out/sweep.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>>gpurun_out/sweep.err
cat gpurun_out/bench_reference.json >> gpurun_out/sweep.json
python tools/bench_table.py gpurun_out/sweep.json
python -c "import __graft_entry__ as g; g.smoke()"
# ncu evidence for the headline kernels (one capture each) + launch list of the default bench
P=${P:-gpurun_out/prof8}; mkdir -p $P
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c2_rasrap -f python tools/profile_step.py --workload c2 --reps 16 > $P/c2.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c3_mbs -f python tools/profile_step.py --workload c3 --reps 4 --n 262144 > $P/c3.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c5_libor80 -f python tools/profile_step.py --workload c5 --reps 2 --n 262144 > $P/c5.log 2>&1
timeout 600 $NCU -k regex:k_stream -s 1 -c 1 -o $P/c4_philox -f python bench.py --workload c4 --generator philox --steps 1 --warmup 1 --reps 2000000 > $P/c4.log 2>&1
for r in $P/*.ncu-rep; do python tools/ncu_summary.py $r x 40 > ${r%.ncu-rep}_summary.txt 2>&1; mv $r /tmp/; done  # reports stay on the box (64 MiB copy-back limit)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $P/launch_bench.log 2>&1
