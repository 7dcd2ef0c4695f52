# ncu captures of the path kernels (one GPU, serial): reports into gpurun_out/prof_${TAG}
set -x
TAG=${TAG:-r02}
P=gpurun_out/prof_$TAG
mkdir -p $P
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c2_rasrap -f python tools/profile_step.py --workload c2 --reps 16 > $P/c2_rasrap.log 2>&1
if [ -z "$ONLY_C2" ]; then
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c3_mbs -f python tools/profile_step.py --workload c3 --reps 4 --n 262144 > $P/c3_mbs.log 2>&1
timeout 600 $NCU -k regex:k_paths -s 1 -c 1 -o $P/c5_libor80 -f python tools/profile_step.py --workload c5 --reps 2 --n 262144 > $P/c5.log 2>&1
timeout 600 $NCU -k regex:k_stream -s 1 -c 1 -o $P/c4_rasrap -f python bench.py --workload c4 --generator rasrap-recursive --steps 1 --warmup 1 --reps 2000000 > $P/c4r.log 2>&1
fi
for r in $P/*.ncu-rep; do
  python tools/ncu_summary.py $r x 60 > ${r%.ncu-rep}_summary.txt 2>&1
  ncu -i $r --page source --csv --print-source=cuda > ${r%.ncu-rep}_src.csv 2>/dev/null
  ncu -i $r --page raw --csv > ${r%.ncu-rep}_raw.csv 2>/dev/null
  gzip -f ${r%.ncu-rep}_src.csv ${r%.ncu-rep}_raw.csv
  [ -n "$KEEP_REP" ] || rm -f $r
done
ls -la $P
