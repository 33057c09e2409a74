# final HEAD: GPU suite, smoke, short bench
mkdir -p gpurun_out/r02last
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/r02last/gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02last/gpu_tests.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke OK')" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02last/bench.json 2> gpurun_out/r02last/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r02last/bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['parity']['code_mismatches'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
