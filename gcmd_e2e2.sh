mkdir -p gpurun_out/e2e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e2e/build.log 2>&1 || { tail -20 gpurun_out/e2e/build.log; exit 1; }
timeout 600 python tools/e2e_probe.py 2>&1 | tail -5
EMESH_HOST_SERIAL=1 timeout 600 python tools/e2e_probe.py 2>&1 | tail -5 | head -3
