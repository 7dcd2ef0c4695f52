rm -f gpurun_out/occ.json
for b in 3 4 5; do for g in rasrap-recursive philox; do
RQ_BLOCKS_PER_SM=$b timeout 300 python bench.py --generator $g --no-cpu-baseline --steps 3 --reps 512 | sed "s|^{|{\"bps\": $b, |" >> gpurun_out/occ.json
done; done
python - <<'PY'
import json
for l in open("gpurun_out/occ.json"):
    d=json.loads(l); print(d["bps"], d["config"]["generator"], "%.4e"%d["value"])
PY
