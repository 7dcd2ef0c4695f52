P=gpurun_out/prof6; mkdir -p $P
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o /tmp/c2_rasrap -f python tools/profile_step.py --workload c2 --reps 16 > $P/c2.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o /tmp/c2_sobol -f python tools/profile_step.py --workload c2 --generator sobol-gray --reps 16 > $P/c2s.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o /tmp/c3_mbs -f python tools/profile_step.py --workload c3 --reps 4 --n 262144 > $P/c3.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o /tmp/c5_libor80 -f python tools/profile_step.py --workload c5 --reps 2 --n 262144 > $P/c5.log 2>&1
for r in c2_rasrap c2_sobol c3_mbs c5_libor80; do python tools/ncu_summary.py /tmp/$r.ncu-rep x 40 > $P/${r}_summary.txt 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $P/launch_bench.log 2>&1
ls -la $P
