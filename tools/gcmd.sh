B() { timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$TAG', '$*', d['ms_per_step'], [round(k[x]['ms_per_step'],2) for x in k])"; }
timeout 600 python -m pytest tests/test_gpu_ring.py tests/test_gpu_codec.py -q -x --timeout=300 2>&1 | tail -2
TAG=mix B; TAG=mix B --S 64
EMESH_QUANT_MIX=0 TAG=nomix B
for L in 1 2 3; do EMESH_QUANT_LAG=$L TAG=mixlag$L B; done
timeout 120 python tools/trace_quant.py 1e9 16 2>&1 | tail -4
