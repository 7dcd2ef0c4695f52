# ncu captures of the fused path kernels (one GPU, serial), summaries into gpurun_out/
set -x
P=gpurun_out/prof
mkdir -p $P
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c2_rasrap -f python tools/profile_step.py --workload c2 --reps 16 > $P/c2_rasrap.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c2_philox -f python tools/profile_step.py --workload c2 --generator philox --reps 16 > $P/c2_philox.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c3_mbs -f python tools/profile_step.py --workload c3 --reps 4 --n 262144 > $P/c3_mbs.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c5_libor80 -f python tools/profile_step.py --workload c5 --reps 2 --n 262144 > $P/c5.log 2>&1
timeout 600 $NCU -k regex:k_stream -s 1 -c 1 -o $P/c4_philox -f python bench.py --workload c4 --generator philox --steps 1 --warmup 1 --reps 2000000 > $P/c4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $P/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $P/launch_bench.log 2>&1
for r in $P/*.ncu-rep; do python tools/ncu_summary.py $r x 40 > ${r%.ncu-rep}_summary.txt 2>&1; done
ls -la $P
