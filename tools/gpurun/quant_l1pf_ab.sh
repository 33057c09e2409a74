# A/B: BIN scratch prefetch into L1 (EMESH_BIN_L1PF) x smem carveout, one GPU, config 2
mkdir -p gpurun_out/pf
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pf/build.log 2>&1 || { tail -20 gpurun_out/pf/build.log; exit 1; }
run() {
  name=$1; shift
  env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pf/$name.json 2> gpurun_out/pf/$name.err
  python -c "
import json
d = json.loads(open('gpurun_out/pf/$name.json').read().strip().splitlines()[-1])
k = d['kernels']
print('$name', round(d['ms_per_step'], 3), d['roofline']['achieved'], {n: round(v['ms_per_step'], 3) for n, v in k.items()})" || tail -3 gpurun_out/pf/$name.err
}
run base
run pf64 EMESH_LIB=build_var/libemesh_pf64.so
run pfna EMESH_LIB=build_var/libemesh_pfna.so
run na EMESH_LIB=build_var/libemesh_na.so
run base2
run pfna2 EMESH_LIB=build_var/libemesh_pfna.so
run na2 EMESH_LIB=build_var/libemesh_na.so
