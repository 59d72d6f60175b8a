#!/bin/bash
# round 2, final build: bench lines of configs 0-3 (config 4 is the default bench line)
run() { name=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/$name.json 2> gpurun_out/$name.err; python tools/summ.py < gpurun_out/$name.json; python -c "import json,sys; d=json.loads(open('gpurun_out/$name.json').read().strip().splitlines()[-1]); print('   e2e', (d.get('e2e') or {}).get('value'))" 2>/dev/null; }
run r2_final_bench_config0 --workload 0 --steps 3 --warmup 3 --no-cpu
run r2_final_bench_config1 --workload 1 --steps 3 --warmup 3 --no-cpu
run r2_final_bench_config2 --workload 2 --steps 3 --warmup 3 --no-cpu
run r2_final_bench_config3 --workload 3 --tsteps 100 --steps 3 --warmup 3 --no-cpu
