# What the driver runs at round end: build, GPU suite, smoke(), default bench
mkdir -p gpurun_out/rend
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/rend/build.log 2>&1 || { tail -20 gpurun_out/rend/build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/rend/bench.json 2> gpurun_out/rend/bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/rend/bench.json
