# Where a small-message round's time goes (peer transport, 2 GPUs)
mkdir -p gpurun_out/small
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/small/build.log 2>&1 || exit 1
for n in 262144 4194304; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/nccl_timeline.py $n 0 4 2>&1 | grep -vE "^W|warn" | head -20
done
