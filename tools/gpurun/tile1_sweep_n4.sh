# 1-unit tiles (EMESH_TILE_UNITS=1) vs the size-based default on small messages, k=2 and k=4; parity with 1-unit tiles
mkdir -p gpurun_out/t1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t1/build.log 2>&1 || { tail -20 gpurun_out/t1/build.log; exit 1; }
EMESH_TILE_UNITS=1 timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_codec.py -x -q 2>&1 | tail -2
for v in 0 1; do
EMESH_TILE_UNITS=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2966$v tools/sweep_msg.py 268435456 5 > gpurun_out/t1/sweep_n4_t$v.jsonl 2> gpurun_out/t1/sweep4_$v.err; echo "sweep4 t$v rc=$?"
CUDA_VISIBLE_DEVICES=0,1 EMESH_TILE_UNITS=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2967$v tools/sweep_msg.py 16777216 5 > gpurun_out/t1/sweep_n2_t$v.jsonl 2> gpurun_out/t1/sweep2_$v.err; echo "sweep2 t$v rc=$?"
done
for f in gpurun_out/t1/*.jsonl; do echo $f; python -c "
import json
for l in open('$f'):
    if l.startswith('{'): r=json.loads(l); print(r['fp32_MB'], round(r['ours_int8_ms'],3), round(r['ours_fp32_ms'],3), round(r['nccl_fp32_ms'],3))"; done
