# quantizer A/B (lane-replicated lookup tables vs round-1 kernel), tests, ncu of both
mkdir -p gpurun_out/r02x
for v in base new base new; do
  L=""; [ $v != new ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r02x/bench_$v.json 2> gpurun_out/r02x/bench_$v.err; echo "bench $v rc=$?"
  python -c "
import json;d=json.loads(open('gpurun_out/r02x/bench_$v.json').read().strip().splitlines()[-1]);print('$v', round(d['ms_per_step'],3),d['roofline']['avg_launch_ms'],d['roofline']['frac'],{k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})"
done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02x/gpu_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02x/gpu_tests.txt
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct
for v in base new; do
  L=""; [ $v != new ] && L="EMESH_LIB=build_var/lib$v.so"
  env $L timeout 600 ncu --metrics $M --clock-control none -k regex:k_quant -c 16 --csv --log-file gpurun_out/r02x/ncu_$v.csv python bench.py --profile-only > gpurun_out/r02x/ncu_$v.log 2>&1; echo "ncu $v rc=$?"
done
