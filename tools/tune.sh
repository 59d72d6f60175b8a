#!/bin/bash
# quick sweep-kernel tuning on config 1 (first 60 time steps); one summary line
# per variant.  Variants: one per line of $VARIANTS_FILE (space-separated
# key=value library options), default tools/variants.txt.
out=${1:-gpurun_out/tune.txt}
vf=${VARIANTS_FILE:-tools/variants.txt}
extra=${EXTRA:-}
: > $out
while IFS= read -r o; do
  [ -z "$o" ] && continue
  args=""
  for kv in $o; do args="$args --opt $kv"; done
  echo "== $o $extra" >> $out
  timeout 300 python bench.py --tsteps 60 --steps 2 --warmup 1 --no-e2e --no-cpu $extra $args 2>&1 | python tools/summ.py >> $out
done < "$vf"
cat $out
