#!/bin/bash
# programmatic dependent launch on / off, interleaved, same box
for rep in 1 2; do
for w in 1 4; do
  for o in "" "--opt pdl=0"; do
    if [ $w = 4 ]; then T="--tsteps 8 --steps 6 --warmup 2"; else T="--steps 2 --warmup 1"; fi
    echo -n "w$w [$o] rep $rep: "; timeout 600 python bench.py --workload $w $T --no-e2e --no-cpu $o 2>/dev/null | python tools/summ.py
  done
done
done
