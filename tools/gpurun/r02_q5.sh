mkdir -p gpurun_out/r02l
timeout 900 python -m pytest tests -m gpu -x -q --timeout 200 > gpurun_out/r02l/gpu_tests.txt 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r02l/gpu_tests.txt
EMESH_LIB=build_var/libw8.so timeout 300 python -m pytest tests/test_cpp_shim.py tests/test_gpu_codec.py tests/test_gpu_ring.py -x -q --timeout 200 > gpurun_out/r02l/gpu_tests_w8.txt 2>&1; echo "tests w8 rc=$?"
tail -2 gpurun_out/r02l/gpu_tests_w8.txt
for v in default w8 nobin nomom nobinmom; do
  L=""; [ $v != default ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r02l/bench_$v.json 2> gpurun_out/r02l/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02l/bench_$v.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['avg_launch_ms'],{k:round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
