# 1 GPU: warp-aggregated bucket-limb atomics (match_any + redux) vs per-lane atomics; parity under the variant
mkdir -p gpurun_out/r02ab5
for v in new wagg new wagg; do
  L=""; [ $v != new ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02ab5/bench_$v.json 2> gpurun_out/r02ab5/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02ab5/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3),d['roofline']['avg_launch_ms'],d['roofline']['frac'],{k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'], d['parity']['cb_mismatches'])"
done
EMESH_LIB=build_var/libwagg.so timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_ring.py tests/test_gpu_scale.py -q -x > gpurun_out/r02ab5/tests_wagg.txt 2>&1; echo "tests wagg rc=$?"; tail -2 gpurun_out/r02ab5/tests_wagg.txt
