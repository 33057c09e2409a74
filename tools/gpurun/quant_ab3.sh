# A/B on the default build: STATS prefetches its next half-unit of theta into L1 (spf)
mkdir -p gpurun_out/ab3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab3/build.log 2>&1 || exit 1
run() {
  name=$1; shift
  env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab3/$name.json 2> gpurun_out/ab3/$name.err
  python -c "
import json
d = json.loads(open('gpurun_out/ab3/$name.json').read().strip().splitlines()[-1])
k = d['kernels']
print('$name', round(d['ms_per_step'], 3), round(sum(v['ms_per_step'] for n, v in k.items() if n.startswith('quant')), 3))" || tail -3 gpurun_out/ab3/$name.err
}
for r in 1 2 3; do
run base$r
run spf$r EMESH_LIB=build_var/libemesh_spf.so
done
