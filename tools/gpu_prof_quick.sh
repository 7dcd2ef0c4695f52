# ncu --set full of the C2 path kernel (rasrap + philox) and C3 MBS; summaries only
P=${P:-gpurun_out/profq}; mkdir -p $P
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o /tmp/q_c2_rasrap -f python tools/profile_step.py --workload c2 --reps 16 > $P/c2.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o /tmp/q_c2_philox -f python tools/profile_step.py --workload c2 --generator philox --reps 16 > $P/c2p.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o /tmp/q_c3_mbs -f python tools/profile_step.py --workload c3 --reps 4 --n 262144 > $P/c3.log 2>&1
for r in c2_rasrap c2_philox c3_mbs; do python tools/ncu_summary.py /tmp/q_$r.ncu-rep x 40 > $P/${r}_summary.txt 2>&1; done
ls $P
