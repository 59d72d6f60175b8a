#!/bin/bash
# config 4 split into n row slabs advanced on ONE GPU (slab launches serialised on one stream): protocol
# overhead of the exchange transports against the single grid (not a scaling measurement)
run() { echo "== $1"; shift; timeout 900 python bench.py --workload 4 --tsteps 2 --steps 2 --warmup 1 --no-e2e --no-cpu "$@" 2>/dev/null | python tools/summ.py; }
run "single grid"
for n in 2 4 8; do
  run "slabs=$n copy" --slabs $n --transport copy
  run "slabs=$n p2p" --slabs $n --transport p2p
done
run "single grid (again)"
