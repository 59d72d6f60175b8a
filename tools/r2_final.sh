#!/bin/bash
# round 2 closing evidence on the final build (one gpurun call)
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_final_pytest_gpu.log 2>&1
tail -n 2 gpurun_out/r2_final_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final_smoke.log 2>&1; tail -n 3 gpurun_out/r2_final_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_final_bench_config4.json 2> gpurun_out/r2_final_bench_config4.err
python tools/summ.py < gpurun_out/r2_final_bench_config4.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_final_reference_arm.json 2> gpurun_out/r2_final_reference_arm.err
tail -c 300 gpurun_out/r2_final_reference_arm.json; echo
CMD="python bench.py --tsteps 1 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/r2_final_plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_final_launches_config4.csv $CMD > gpurun_out/r2_final_ncu.log 2>&1
tail -n 2 gpurun_out/r2_final_ncu.log
