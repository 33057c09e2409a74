# 1 GPU: larger quantizer tiles for big batches (6 / 7 warp units per tile; limb split 6/25)
mkdir -p gpurun_out/r02ab11
for v in cur u6 u7 cur u6 u7; do
  env EMESH_LIB=build_var/lib$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02ab11/bench_$v.json 2> gpurun_out/r02ab11/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02ab11/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), d['roofline']['avg_launch_ms'], {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()}, d['parity']['code_mismatches'], d['parity']['cb_mismatches'])"
done
for v in u6 u7; do EMESH_LIB=build_var/lib$v.so timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_ring.py tests/test_gpu_scale.py -q -x > gpurun_out/r02ab11/tests_$v.txt 2>&1; echo "tests $v rc=$?"; tail -1 gpurun_out/r02ab11/tests_$v.txt; done
