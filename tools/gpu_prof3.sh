P=gpurun_out/prof3
mkdir -p $P
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:k_stream -s 1 -c 1 -o $P/c4_philox -f python bench.py --workload c4 --generator philox --steps 1 --warmup 1 --reps 2000000 > $P/c4.log 2>&1
timeout 600 $NCU -k regex:k_paths_seq -s 1 -c 1 -o $P/c2_kakutani -f python tools/profile_step.py --workload c2 --generator kakutani --reps 8 > $P/kak.log 2>&1
for r in $P/*.ncu-rep; do python tools/ncu_summary.py $r x 40 > ${r%.ncu-rep}_summary.txt 2>&1; done
timeout 300 python bench.py --generator kakutani --no-cpu-baseline --steps 3 | python tools/bench_table.py /dev/stdin
