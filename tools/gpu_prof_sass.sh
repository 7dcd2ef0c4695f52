# One ncu capture of the C2 path kernel; per-SASS-instruction metrics CSV (gzip) into gpurun_out/
TAG=${TAG:-r02}
P=gpurun_out/sass_$TAG
mkdir -p $P
WL=${WL:-c2}; GEN=${GEN:-rasrap-recursive}; REPS=${REPS:-16}; NN=${NN:-0}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_paths -s 1 -c 1 -o $P/k -f python tools/profile_step.py --workload $WL --generator $GEN --reps $REPS --n $NN > $P/k.log 2>&1
python tools/ncu_summary.py $P/k.ncu-rep x 80 > $P/summary.txt 2>&1
ncu -i $P/k.ncu-rep --page source --csv --print-source=sass > $P/sass.csv 2>/dev/null
gzip -f $P/sass.csv
rm -f $P/k.ncu-rep
ls -la $P
