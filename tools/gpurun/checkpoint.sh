mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_checkpoint.py -x -q 2>&1 | tail -15
nproc; free -g | head -2
timeout 600 python tools/ckpt_speed.py 2e8 2>&1 | tee gpurun_out/ckpt_speed.txt
