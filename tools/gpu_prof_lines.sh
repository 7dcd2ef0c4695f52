# ncu --set full of the C2 path kernel (rasrap, sobol-gray, philox) with long per-line tables
P=${P:-gpurun_out/profl}; mkdir -p $P
NCU="ncu --set full --clock-control none --import-source on"
for g in rasrap-recursive sobol-gray philox; do
  timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o /tmp/l_$g -f python tools/profile_step.py --workload c2 --generator $g --reps 16 > $P/c2_$g.log 2>&1
  python tools/ncu_summary.py /tmp/l_$g.ncu-rep x 200 > $P/c2_${g}_summary.txt 2>&1
done
ls $P
