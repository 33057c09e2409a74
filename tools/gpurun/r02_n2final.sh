# 2 GPUs: multi-GPU suite + bench (the driver's N=2 scaling point)
mkdir -p gpurun_out/r02n2f
timeout 1200 python -m pytest tests/test_gpu_nccl.py -v --timeout 600 > gpurun_out/r02n2f/mg_tests.txt 2>&1; echo "mg tests rc=$?"
grep -E "PASS|FAIL|passed|failed" gpurun_out/r02n2f/mg_tests.txt | head -8
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29791 bench.py --gpus 2 > gpurun_out/r02n2f/bench_n2.json 2> gpurun_out/r02n2f/bench_n2.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02n2f/bench_n2.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'], d['parity']['theta_mismatches'], d['e2e']['value'], d['nvlink']['avg_GBps_per_direction'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29792 bench.py --gpus 2 --impl reference > gpurun_out/r02n2f/ref_n2.json 2> gpurun_out/r02n2f/ref_n2.err; echo "ref rc=$?"; tail -1 gpurun_out/r02n2f/ref_n2.json | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29793 tools/sweep_msg.py 1073741824 10 > gpurun_out/r02n2f/sweep_n2.jsonl 2> gpurun_out/r02n2f/sweep_n2.err; echo "sweep rc=$?"
python -c "
import json
for l in open('gpurun_out/r02n2f/sweep_n2.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['fp32_MB'], round(d['ours_int8_ms'],4), round(d['ours_fp32_ms'],4), round(d['nccl_fp32_ms'],4))"
