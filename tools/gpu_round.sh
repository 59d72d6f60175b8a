#!/bin/bash
# Round evidence: default bench line, other configs, launch list, ncu full capture.
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json; echo
for w in 2 3; do python bench.py --workload $w --tsteps 60 --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_w$w.json 2> gpurun_out/bench_w$w.err; python tools/summ.py < gpurun_out/bench_w$w.json; done
python bench.py --workload 4 --tsteps 20 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_w4.json 2> gpurun_out/bench_w4.err; python tools/summ.py < gpurun_out/bench_w4.json
python bench.py --workload 0 --no-e2e > gpurun_out/bench_w0.json 2> gpurun_out/bench_w0.err; python tools/summ.py < gpurun_out/bench_w0.json
CMD="python bench.py --tsteps 3 --steps 1 --warmup 3 --no-e2e --no-cpu --omega 1.9639"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_rb_sweep2 -s 20 -c 1 -o gpurun_out/sweep2_full $CMD > gpurun_out/ncu_full.log 2>&1
tail -n 2 gpurun_out/ncu_launches.log gpurun_out/ncu_full.log
