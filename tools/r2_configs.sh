#!/bin/bash
# round 2: bench lines of the other configs and the 8-slab emulation of config 4
run() { name=$1; shift; python bench.py "$@" > gpurun_out/$name.json 2> gpurun_out/$name.err; python tools/summ.py < gpurun_out/$name.json; tail -n 2 gpurun_out/$name.err; }
run b_c1 --workload 1 --steps 3 --warmup 1 --no-cpu
run b_c3 --workload 3 --tsteps 100 --steps 3 --warmup 1 --no-cpu
run b_c0 --workload 0 --steps 3 --warmup 1 --no-cpu --no-e2e
run b_c4_slab8_copy --workload 4 --tsteps 2 --steps 2 --warmup 1 --slabs 8 --no-e2e --no-cpu
run b_c4_slab8_p2p --workload 4 --tsteps 2 --steps 2 --warmup 1 --slabs 8 --transport p2p --no-e2e --no-cpu
run b_c4_slab1 --workload 4 --tsteps 2 --steps 2 --warmup 1 --no-e2e --no-cpu
