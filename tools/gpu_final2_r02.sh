# Re-measure the configs changed after r02f (C5: 24 rates in shared memory;
# C4 Rasrap: 6 CTAs/SM) + ncu of both + the GPU tests.
P=${P:-gpurun_out/r02h}; mkdir -p $P; rm -f $P/sweep.json
timeout 1200 python bench.py --workload c5 --steps 1 --warmup 3 >> $P/sweep.json 2>>$P/sweep.err
for g in philox sobol-gray; do timeout 600 python bench.py --workload c5 --reps 1024 --generator $g --no-cpu-baseline --steps 3 >> $P/sweep.json 2>>$P/sweep.err; done
for g in philox sfc64 rasrap-recursive sobol-gray rasrap-counter; do timeout 300 python bench.py --workload c4 --generator $g --steps 50 --warmup 5 >> $P/sweep.json 2>>$P/sweep.err; done
timeout 900 python bench.py --steps 20 --warmup 5 > $P/bench_default.json 2>>$P/sweep.err; cat $P/bench_default.json >> $P/sweep.json
python tools/bench_table.py $P/sweep.json
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c5_libor80 -f python tools/profile_step.py --workload c5 --reps 2 --n 262144 > $P/ncu_c5.log 2>&1
timeout 600 $NCU -k regex:k_stream -s 1 -c 1 -o $P/c4_rasrap -f python bench.py --workload c4 --generator rasrap-recursive --steps 1 --warmup 1 --reps 2000000 > $P/ncu_c4r.log 2>&1
for r in $P/*.ncu-rep; do python tools/ncu_summary.py $r x 40 > ${r%.ncu-rep}_summary.txt 2>&1; rm -f $r; done
grep -h "fp64_cycles\|registers_per" $P/*_summary.txt
timeout 1500 python -m pytest tests -m gpu -q -x > $P/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 $P/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; tail -1 $P/smoke.log
