mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for t in nccl p2p; do
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29561 tests/retry_worker.py $t > gpurun_out/retry_$t.log 2>&1; echo "retry $t rc=$?"
  grep -E "retry|Error|error" gpurun_out/retry_$t.log | tail -8
done
timeout 600 python -m pytest tests/test_gpu_nccl.py -x -q 2>&1 | tail -5
