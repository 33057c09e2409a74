mkdir -p gpurun_out/rp
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rp/build.log 2>&1 || exit 1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29534 tests/retry_worker.py p2p > gpurun_out/rp/out.txt 2> gpurun_out/rp/err.txt; echo "p2p4 rc=$?"
grep -v "^\s*$" gpurun_out/rp/out.txt | tail -12; grep -iE "error|timeout|Traceback|File|line" gpurun_out/rp/err.txt | head -30
