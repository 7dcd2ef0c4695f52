# Round-2 measurement sweep (one B200): default bench line (C2 Rasrap with CPU
# baseline + parity), every C2 generator, C1, C3 and C5 at full M with CPU
# baseline + parity, C4 streams (enough steps for clock samples), reference
# arm, ncu summaries of the headline kernels + launch list.  P=prefix dir.
P=${P:-gpurun_out/r02}; mkdir -p $P
rm -f $P/sweep.json
timeout 900 python bench.py --steps 20 --warmup 5 > $P/bench_default.json 2> $P/bench_default.err
cat $P/bench_default.json >> $P/sweep.json
for g in rasrap-counter philox sobol-gray sobol-counter sfc64 twister xorwow kakutani; do
  timeout 300 python bench.py --generator $g --no-cpu-baseline --steps 5 >> $P/sweep.json 2>>$P/sweep.err
done
timeout 600 python bench.py --workload c1 --steps 5000 --warmup 50 >> $P/sweep.json 2>>$P/sweep.err
timeout 900 python bench.py --workload c3 --steps 5 >> $P/sweep.json 2>>$P/sweep.err
for g in philox sobol-gray xorwow; do timeout 600 python bench.py --workload c3 --generator $g --no-cpu-baseline --steps 3 >> $P/sweep.json 2>>$P/sweep.err; done
timeout 1200 python bench.py --workload c5 --steps 1 --warmup 3 >> $P/sweep.json 2>>$P/sweep.err
for g in philox sobol-gray; do timeout 600 python bench.py --workload c5 --reps 1024 --generator $g --no-cpu-baseline --steps 3 >> $P/sweep.json 2>>$P/sweep.err; done
for g in philox sfc64 rasrap-recursive sobol-gray; do timeout 300 python bench.py --workload c4 --generator $g --steps 50 --warmup 5 >> $P/sweep.json 2>>$P/sweep.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 2 > $P/bench_reference.json 2>>$P/sweep.err
cat $P/bench_reference.json >> $P/sweep.json
python tools/bench_table.py $P/sweep.json
python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; tail -1 $P/smoke.log
# ncu (one capture each) -> summaries, then the launch list of the default bench
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c2_rasrap -f python tools/profile_step.py --workload c2 --reps 16 > $P/ncu_c2.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c2_philox -f python tools/profile_step.py --workload c2 --generator philox --reps 16 > $P/ncu_c2p.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c2_sobol -f python tools/profile_step.py --workload c2 --generator sobol-gray --reps 16 > $P/ncu_c2s.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c3_mbs -f python tools/profile_step.py --workload c3 --reps 4 --n 262144 > $P/ncu_c3.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c5_libor80 -f python tools/profile_step.py --workload c5 --reps 2 --n 262144 > $P/ncu_c5.log 2>&1
timeout 600 $NCU -k regex:k_stream -s 1 -c 1 -o $P/c4_rasrap -f python bench.py --workload c4 --generator rasrap-recursive --steps 1 --warmup 1 --reps 2000000 > $P/ncu_c4r.log 2>&1
timeout 600 $NCU -k regex:k_stream -s 1 -c 1 -o $P/c4_philox -f python bench.py --workload c4 --generator philox --steps 1 --warmup 1 --reps 2000000 > $P/ncu_c4p.log 2>&1
for r in $P/*.ncu-rep; do python tools/ncu_summary.py $r x 40 > ${r%.ncu-rep}_summary.txt 2>&1; rm -f $r; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $P/launch_bench.log 2>&1
ls $P
