mkdir -p gpurun_out/r01c
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29553 bench.py --gpus 4 --tensors intellect1 --S 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r01c/bench_n4_cfg5.json.log 2> gpurun_out/r01c/bench_n4_cfg5.err; echo "cfg5 rc=$?"
tail -c 700 gpurun_out/r01c/bench_n4_cfg5.json.log
