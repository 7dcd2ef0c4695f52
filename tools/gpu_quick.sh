# Quick check after a kernel change: Rasrap parity subset + short bench lines.
mkdir -p gpurun_out
rm -f gpurun_out/quick.json
timeout 900 python -m pytest tests -m gpu -q -x -k "${TESTK:-rasrap or xhash or c2_ or c3_ or c5_}" > gpurun_out/quick_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/quick_tests.log
for wl in ${WLS:-"c2" "c3 --reps 64" "c5 --reps 128" "c4"}; do
  timeout 300 python bench.py --workload $wl --generator ${GEN:-rasrap-recursive} --no-cpu-baseline --steps 3 >> gpurun_out/quick.json 2>>gpurun_out/quick.err
done
python tools/bench_table.py gpurun_out/quick.json
