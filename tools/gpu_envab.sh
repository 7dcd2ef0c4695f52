for r in 1 2; do
for b in 134217728 268435456 536870912; do
  echo -n "batch=$b "; RQ_BATCH_PATHS=$b timeout 300 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().split('\n')[-1]); print('%.4e'%j['value'])"
  echo -n "c3 batch=$b "; RQ_BATCH_PATHS=$b timeout 300 python bench.py --workload c3 --reps 64 --no-cpu-baseline --steps 3 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read().strip().split('\n')[-1]); print('%.4e'%j['value'])"
done; done
