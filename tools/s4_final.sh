#!/bin/bash
# session 4 closing evidence on HEAD (one gpurun call): GPU suite, smoke,
# config-4 headline, reference arm, ncu launch list of the bench command
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/s4_pytest_gpu.log 2>&1
tail -n 2 $O/s4_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/s4_smoke.log 2>&1; tail -n 3 $O/s4_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/s4_bench_config4.json 2> $O/s4_bench_config4.err
python tools/summ.py < $O/s4_bench_config4.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/s4_reference_arm.json 2> $O/s4_reference_arm.err
tail -c 300 $O/s4_reference_arm.json; echo
for w in 1 2 3; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu > $O/s4_bench_config$w.json 2> $O/s4_bench_config$w.err
  python tools/summ.py < $O/s4_bench_config$w.json
done
CMD="python bench.py --tsteps 1 --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > $O/s4_plain.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/s4_launches_config4.csv $CMD > $O/s4_ncu.log 2>&1
tail -n 2 $O/s4_ncu.log
