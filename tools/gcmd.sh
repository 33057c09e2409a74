B() { timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$TAG', '$*', d['ms_per_step'], [round(k[x]['ms_per_step'],2) for x in k])"; }
EMESH_LIB=build_var/libemesh_u4b4.so timeout 600 python -m pytest tests/test_gpu_ring.py -q -x --timeout=200 2>&1 | tail -2
EMESH_LIB=build_var/libemesh_u4b4.so TAG=u4b4 B; EMESH_LIB=build_var/libemesh_u4b4.so TAG=u4b4 B --S 64
EMESH_LIB=build_var/libemesh_u4b2.so TAG=u4b2 B; EMESH_LIB=build_var/libemesh_u4b2.so TAG=u4b2 B --S 64
