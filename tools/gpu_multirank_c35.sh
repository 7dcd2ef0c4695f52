# Strong-scaling path of configs 3 and 5 with 1 and 2 ranks sharing the one
# B200: the theta hash must not depend on the rank count.
P=gpurun_out/r02k; mkdir -p $P; rm -f $P/multirank.jsonl
for wl in "c3 --reps 16" "c5 --reps 32"; do
  timeout 600 python bench.py --workload $wl --steps 2 --warmup 3 --no-cpu-baseline >> $P/multirank.jsonl 2>>$P/multirank.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --workload $wl --steps 2 --warmup 3 --no-cpu-baseline 2>>$P/multirank.err | grep '^{' >> $P/multirank.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/r02k/multirank.jsonl"):
    j = json.loads(l)
    print(j["config"]["workload"][:24], "n_gpus", j["n_gpus"], "M/rank", j.get("M_per_rank"), "sha", j.get("theta_sha16"), "%.3e" % j["value"])
PY
