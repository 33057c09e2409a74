# 4 GPUs: one decode launch per round (peer transport): sweep, bench, multi-GPU tests
mkdir -p gpurun_out/r02n4i
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29741 tools/sweep_msg.py 268435456 10 > gpurun_out/r02n4i/sweep_n4.jsonl 2> gpurun_out/r02n4i/sweep_n4.err; echo "sweep rc=$?"
python -c "
import json
for l in open('gpurun_out/r02n4i/sweep_n4.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['fp32_MB'], round(d['ours_int8_ms'],4), round(d['ours_fp32_ms'],4), round(d['nccl_fp32_ms'],4))"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29742 bench.py --gpus 4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02n4i/p2p.json 2> gpurun_out/r02n4i/p2p.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02n4i/p2p.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'], d['parity']['theta_mismatches'])"
timeout 900 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_ring.py -q --timeout 600 > gpurun_out/r02n4i/tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02n4i/tests.txt
