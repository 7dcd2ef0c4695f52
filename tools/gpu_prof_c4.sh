# One ncu capture of the config-4 Rasrap stream kernel; per-SASS CSV (gzip) into gpurun_out/sass_c4
P=gpurun_out/sass_c4; mkdir -p $P
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream_chunks -s 2 -c 1 -o $P/k -f python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > $P/k.log 2>&1
python tools/ncu_summary.py $P/k.ncu-rep x 80 > $P/summary.txt 2>&1
ncu -i $P/k.ncu-rep --page source --csv --print-source=sass > $P/sass.csv 2>/dev/null
gzip -f $P/sass.csv; rm -f $P/k.ncu-rep; ls -la $P
