# (1) ncu evidence for the final round-1 build (launch list + k_quant<3> / k_apply<1> full captures, GPU 0)
# (2) A/B: 2 warp units per tile (build_var/libemesh_u2.so, -DEMESH_UNITS_PER_WARP=2): parity, config 2, small messages
mkdir -p gpurun_out/fin gpurun_out/u2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin/build.log 2>&1 || { tail -20 gpurun_out/fin/build.log; exit 1; }
EMESH_LIB=build_var/libemesh_u2.so timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_codec.py -x -q 2>&1 | tail -2
for rep in 1 2; do
for v in base u2; do
if [ $v = u2 ]; then L=build_var/libemesh_u2.so; else L=; fi
CUDA_VISIBLE_DEVICES=0 EMESH_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/u2/$v$rep.json 2> gpurun_out/u2/$v.err
python -c "import json;d=json.loads(open('gpurun_out/u2/$v$rep.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3), d['roofline']['frac'], d['clocks']['sm_mhz'])"
done; done
for v in base u2; do
if [ $v = u2 ]; then L=build_var/libemesh_u2.so; else L=; fi
CUDA_VISIBLE_DEVICES=0,1 EMESH_LIB=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2964${#v} tools/sweep_msg.py 268435456 5 > gpurun_out/u2/sweep_$v.jsonl 2> gpurun_out/u2/sweep_$v.err; echo "sweep $v rc=$?"
cut -c1-200 gpurun_out/u2/sweep_$v.jsonl | head -12
done
export CUDA_VISIBLE_DEVICES=0
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/bench.json 2>&1; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/fin/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_quant --launch-skip 21 --launch-count 1 -o gpurun_out/fin/kq -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/ncu_kq.log 2>&1; echo kq rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply --launch-skip 20 --launch-count 1 -o gpurun_out/fin/ka -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin/ncu_ka.log 2>&1; echo ka rc=$?
