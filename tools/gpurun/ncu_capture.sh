# ncu evidence for the current build (one GPU): launch list + one full capture of k_quant<3> and k_apply<1>
mkdir -p gpurun_out/ncu2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu2/build.log 2>&1 || exit 1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2/bench.json 2>&1; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/ncu2/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_quant --launch-skip 21 --launch-count 1 -o gpurun_out/ncu2/kq -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2/ncu_kq.log 2>&1; echo kq rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply --launch-skip 20 --launch-count 1 -o gpurun_out/ncu2/ka -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2/ncu_ka.log 2>&1; echo ka rc=$?
