mkdir -p gpurun_out/r01b
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tests/nccl_parity_worker.py 2>&1 | grep -E "MISMATCH|asked|parity|Error" | head -20
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 tools/nccl_timeline.py 1e9 0 16 > gpurun_out/r01b/timeline_n4.txt 2>&1
for N in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29550 + N)) bench.py --gpus $N > gpurun_out/r01b/bench_n$N.json.log 2> gpurun_out/r01b/bench_n$N.err; echo "bench N=$N rc=$?"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29560 bench.py --gpus 4 --transport nccl --no-e2e > gpurun_out/r01b/bench_n4_nccl.json.log 2>&1; echo "nccl rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/r01b/bench_ref_n4.json.log 2>&1; echo "ref rc=$?"
