# Multi-rank check of bench.py on a one-GPU box: torchrun with 2 and 4 ranks
# sharing the device (gloo gather), plus the reference arm under torchrun.
# Each run must print exactly one JSON line (rank 0).
mkdir -p gpurun_out
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus $n --steps 3 --warmup 3 --reps 64 > gpurun_out/mr_$n.json 2> gpurun_out/mr_$n.err
  echo "n=$n rc=$? lines=$(grep -c '^{' gpurun_out/mr_$n.json)"; cut -c1-300 gpurun_out/mr_$n.json
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err
echo "ref rc=$? lines=$(grep -c '^{' gpurun_out/mr_ref.json)"; cut -c1-300 gpurun_out/mr_ref.json
timeout 300 python bench.py --reps 64 --steps 3 --no-cpu-baseline | cut -c1-300
