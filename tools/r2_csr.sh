#!/bin/bash
# round 2: staged CSR sweep parity + bench A/B, config-4 ncu evidence
python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -k "csr or golden" -x -q -s 2>&1 | tail -12 > gpurun_out/t_csr.log
python -m pytest tests/test_gpu_fullsize.py -k "2-4" -x -q 2>&1 | tail -3 >> gpurun_out/t_csr.log
for o in 1 0; do
  python bench.py --workload 2 --tsteps 20 --steps 3 --warmup 1 --no-e2e --no-cpu --opt csr_stage=$o > gpurun_out/bench_c2_stage$o.json 2> gpurun_out/bench_c2_stage$o.err
done
CMD="python bench.py --workload 4 --tsteps 1 --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/plain4.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_config4.csv $CMD > gpurun_out/ncu_l4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rb_sweep2 -s 40 -c 1 -o gpurun_out/r2_sweep2_config4 $CMD > gpurun_out/ncu_f4.log 2>&1
CMD2="python bench.py --workload 2 --tsteps 1 --steps 1 --warmup 1 --no-e2e --no-cpu"
ncu --set full --clock-control none --import-source on -k regex:k_csr_sweep -s 40 -c 1 -o gpurun_out/r2_csr_staged_config2 $CMD2 > gpurun_out/ncu_f2.log 2>&1
cat gpurun_out/t_csr.log; tail -n 3 gpurun_out/ncu_*.log
for o in 1 0; do python tools/summ.py < gpurun_out/bench_c2_stage$o.json; tail -2 gpurun_out/bench_c2_stage$o.err; done
