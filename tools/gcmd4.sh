mkdir -p gpurun_out/r01c
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 4 --params 10211381248 --S 80 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r01c/bench_n4_10b.json.log 2> gpurun_out/r01c/bench_n4_10b.err; echo "10b rc=$?"
tail -c 600 gpurun_out/r01c/bench_n4_10b.json.log
