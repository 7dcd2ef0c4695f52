# Final round-2 evidence: the full sweep, then the strong-scaling path with 2
# ranks sharing the one B200 (same theta hash as one rank), then the GPU tests.
P=${P:-gpurun_out/r02f}
P=$P bash tools/gpu_sweep_r02.sh
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $P/bench_2rank_shared_gpu.json 2> $P/bench_2rank.err
tail -1 $P/bench_2rank_shared_gpu.json | cut -c1-400
for f in $P/*.ncu-rep; do rm -f $f; done
timeout 1500 python -m pytest tests -m gpu -q -x > $P/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $P/pytest_gpu.log
