# A/B over several library builds: LIBS="a.so b.so ..." bash tools/gpu_abn.sh "<bench args>" ...
rm -f gpurun_out/ab.json
for lib in paper_1408_5526_b200/librqmc_b200.so $LIBS; do
  for args in "$@"; do
    RQMC_B200_LIB=$PWD/$lib timeout 300 python bench.py $args --no-cpu-baseline --steps 3 | sed "s|^{|{\"lib\": \"$lib\", |" >> gpurun_out/ab.json 2>>gpurun_out/ab.err
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/ab.json"):
    if l.startswith("{"):
        d=json.loads(l); c=d["config"]
        print(d["lib"].split("/")[-1][:28], c.get("workload","")[:24], c.get("generator"), "%.4e"%d["value"], "frac %.3f"%d["roofline"]["frac"])
PY
