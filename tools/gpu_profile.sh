#!/bin/bash
# Round profile: default bench line, launch list of a short bench run, full ncu
# capture of the sweep kernel.  Outputs under gpurun_out/.
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 2500 gpurun_out/bench.json
CMD="python bench.py --tsteps 3 --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_rb_sweep_fused -s 20 -c 1 -o gpurun_out/fused_full $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_launches.log gpurun_out/ncu_full.log
