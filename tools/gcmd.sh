B() { timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$TAG', '$*', d['ms_per_step'], [round(k[x]['ms_per_step'],2) for x in k])"; }
timeout 600 python -m pytest tests -m gpu -q -x --timeout=200 2>&1 | tail -3
TAG=u4 B; TAG=u4 B --S 64
