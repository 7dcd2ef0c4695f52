# compute-sanitizer evidence over tools/sanitize_smoke.py: memcheck (+ leak check),
# racecheck (shared-memory hazards, warp-level included), synccheck
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check full --error-exitcode 7 python tools/sanitize_smoke.py > gpurun_out/sanitize/memcheck.log 2>&1; echo memcheck=$?
timeout 1500 $CS --tool racecheck --racecheck-report all --print-limit 5000 --error-exitcode 7 python tools/sanitize_smoke.py > gpurun_out/sanitize/racecheck.log 2>&1; echo racecheck=$?
timeout 1500 $CS --tool synccheck --error-exitcode 7 python tools/sanitize_smoke.py > gpurun_out/sanitize/synccheck.log 2>&1; echo synccheck=$?
for f in gpurun_out/sanitize/*.log; do echo "== $f"; grep -E "SUMMARY|smoke ok" $f; done
grep "Read Thread\|Write Thread" gpurun_out/sanitize/racecheck.log | sed -E 's/Thread \([0-9,]+\)//; s/\+0x[0-9a-f]+//' | sort | uniq -c | sort -rn | head -20
gzip -f gpurun_out/sanitize/racecheck.log
