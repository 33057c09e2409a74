mkdir -p gpurun_out/r02f
timeout 900 python -m pytest tests/test_gpu_scale.py -v -x --timeout 400 --durations=0 > gpurun_out/r02f/scale.txt 2>&1; echo "scale rc=$?"
grep -E "passed|failed|PASS|FAIL|Error|assert" gpurun_out/r02f/scale.txt | head -20
timeout 900 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/r02f/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02f/gpu_tests.txt
for v in default nopf; do
  L=""; [ $v = nopf ] && L="EMESH_LIB=build_var/libnopf.so"
  env $L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02f/bench_$v.json 2> gpurun_out/r02f/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02f/bench_$v.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d['roofline']['frac'],d['roofline']['avg_launch_ms'],{k:v['ms_per_step'] for k,v in d['kernels'].items()}, d.get('parity'))"
done
