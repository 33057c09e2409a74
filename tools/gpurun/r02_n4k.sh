# 4 GPUs: shorter spin back-off caps (flag polls) vs the previous build: sweep (<= 256 MB) + bench
mkdir -p gpurun_out/r02n4k
for v in cur new cur new; do
  L=""; [ $v != new ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29771 tools/sweep_msg.py 67108864 20 > gpurun_out/r02n4k/sweep_$v.jsonl 2> gpurun_out/r02n4k/sweep_$v.err
  echo "$v $(python -c "
import json
print([ (d['fp32_MB'], round(d['ours_int8_ms'],4)) for d in (json.loads(l) for l in open('gpurun_out/r02n4k/sweep_$v.jsonl') if l.startswith('{'))])")"
done
for v in cur new; do
  L=""; [ $v != new ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29772 bench.py --gpus 4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-parity > gpurun_out/r02n4k/bench_$v.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/r02n4k/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3))"
done
