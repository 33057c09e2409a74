timeout 600 python -m pytest tests -m gpu -q -x --timeout=200 2>&1 | tail -5
for L in 1 2; do echo "LAG $L"; EMESH_QUANT_LAG=$L timeout 120 python tools/trace_quant.py 1e9 16 2>&1 | tail -10; done
for L in 1 1.5 2 3; do EMESH_QUANT_LAG=$L timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LAG $L S16', d['ms_per_step'], d['kernels'])"; done
for L in 1 2 3; do EMESH_QUANT_LAG=$L timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --S 64 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LAG $L S64', d['ms_per_step'])"; done
