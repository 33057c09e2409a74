B() { timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$TAG', '$*', d['ms_per_step'], [round(k[x]['ms_per_step'],2) for x in k])"; }
TAG=base B
for v in s2b3 s2b4; do EMESH_LIB=build_var/libemesh_$v.so TAG=$v B; EMESH_LIB=build_var/libemesh_$v.so TAG=$v B --S 64; done
EMESH_LIB=build_var/libemesh_s2b4.so EMESH_QUANT_LAG=1.5 TAG=s2b4lag15 B
