set -x
P=gpurun_out/prof2
mkdir -p $P
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c2_rasrap -f python tools/profile_step.py --workload c2 --reps 16 > $P/c2_rasrap.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c2_philox -f python tools/profile_step.py --workload c2 --generator philox --reps 16 > $P/c2_philox.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c3_mbs -f python tools/profile_step.py --workload c3 --reps 4 --n 262144 > $P/c3_mbs.log 2>&1
timeout 600 $NCU -k regex:k_paths_seq -s 1 -c 1 -o $P/c2_xorwow -f python tools/profile_step.py --workload c2 --generator xorwow --reps 16 > $P/c2_xorwow.log 2>&1
for r in $P/*.ncu-rep; do python tools/ncu_summary.py $r x 60 > ${r%.ncu-rep}_summary.txt 2>&1; done
ls -la $P
