# MBS rescale parity + new bench line (strong scaling, parity) + 2-rank shared-GPU bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_benchsize.py -q -k "mbs" > gpurun_out/mbs_edge.log 2>&1; echo mbs=$?; tail -5 gpurun_out/mbs_edge.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
tail -c 3000 gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo bench2=$?
tail -c 1500 gpurun_out/bench_2rank.json; tail -5 gpurun_out/bench_2rank.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo ref=$?; cat gpurun_out/bench_ref.json | tail -c 1500
