mkdir -p gpurun_out/fp
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fp/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -x -q -m gpu -k "nccl or p2p or multi or retry" > gpurun_out/fp/default.txt 2>&1; echo "default rc=$?"
grep -E "^FAILED|Error|assert" gpurun_out/fp/default.txt | head -20
EMESH_TILE_UNITS=4 timeout 900 python -m pytest tests -x -q -m gpu -k "nccl or p2p or multi or retry" > gpurun_out/fp/t4.txt 2>&1; echo "t4 rc=$?"
tail -3 gpurun_out/fp/t4.txt
