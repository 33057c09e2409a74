# 4 GPUs: multi-GPU tests twice (culprit attribution past k=2), benches (P2P, NCCL, 10.2B S=80), sweep
mkdir -p gpurun_out/r02n4f
for i in 1 2; do
timeout 900 python -m pytest tests/test_gpu_nccl.py -v --timeout 600 > gpurun_out/r02n4f/mg_tests_$i.txt 2>&1; echo "mg tests $i rc=$?"
grep -E "PASS|FAIL|passed|failed" gpurun_out/r02n4f/mg_tests_$i.txt | head -8
done
B() { name=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29701 \
    bench.py --gpus 4 "$@" > gpurun_out/r02n4f/$name.json 2> gpurun_out/r02n4f/$name.err
  echo "$name rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/r02n4f/$name.json').read().strip().splitlines()[-1]);print(round(d['ms_per_step'],3), d['value'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity'], (d.get('e2e') or {}).get('value'))" 2>&1 | tail -1)"; }
B p2p --steps 20 --warmup 3
B nccl --steps 10 --warmup 3 --transport nccl --no-e2e
B p2p_10b_S80 --steps 5 --warmup 3 --params 10.211381248e9 --S 80 --no-e2e
B p2p_cfg5 --steps 5 --warmup 3 --params 10.211381248e9 --S 4 --tensors intellect1 --no-e2e
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29702 tools/sweep_msg.py 1073741824 10 > gpurun_out/r02n4f/sweep_n4.jsonl 2> gpurun_out/r02n4f/sweep_n4.err; echo "sweep rc=$?"
python -c "
import json
for l in open('gpurun_out/r02n4f/sweep_n4.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['fp32_MB'], round(d['ours_int8_ms'],4), round(d['ours_fp32_ms'],4), round(d['nccl_fp32_ms'],4))"
