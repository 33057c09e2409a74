# A/B: scratch x L2 residency (evict_last stores) x BIN lag, one GPU, config 2
mkdir -p gpurun_out/l2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/l2/build.log 2>&1 || { tail -20 gpurun_out/l2/build.log; exit 1; }
run() {  # name, env...
  name=$1; shift
  env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/l2/$name.json 2> gpurun_out/l2/$name.err
  python - "$name" <<'PY'
import json, sys
name = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/l2/{name}.json").read().strip().splitlines()[-1])
    r = d.get("roofline", {})
    print(f"{name:22s} ms/step {d['ms_per_step']:.3f}  quant {r.get('achieved')} {r.get('unit')} frac {r.get('frac')}  kernels {d.get('kernels', '')}")
except Exception as e:
    print(name, "FAILED", e, open(f"gpurun_out/l2/{name}.err").read()[-500:])
PY
}
run base
run evl EMESH_LIB=build_var/libemesh_evl.so
run base_lag075 EMESH_QUANT_LAG=0.75
run evl_lag075 EMESH_LIB=build_var/libemesh_evl.so EMESH_QUANT_LAG=0.75
run base_lag3 EMESH_QUANT_LAG=3
run evl_fwd EMESH_LIB=build_var/libemesh_evl.so EMESH_BIN_REVERSE=0
run base2
for v in base evl; do
  lib=paper_2412_01152_b200/libemesh_b200.so; [ $v = evl ] && lib=build_var/libemesh_evl.so
  EMESH_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_quant --launch-skip 21 --launch-count 3 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/l2/ncu_$v.csv 2>&1; echo "ncu $v rc=$?"
  grep -E "dram__bytes|gpu__time|hit_rate" gpurun_out/l2/ncu_$v.csv | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}' | head -12
done
