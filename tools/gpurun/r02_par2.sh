mkdir -p gpurun_out/r02par
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=${NG:-2} --master-addr 127.0.0.1 --master-port 29751 tests/nccl_parity_worker.py > gpurun_out/r02par/out.txt 2> gpurun_out/r02par/err.txt; echo "rc=$?"
tail -5 gpurun_out/r02par/out.txt; grep -E "Error|error" gpurun_out/r02par/err.txt | grep -v elastic | head -10
