#!/bin/bash
# A/B of two builds of the library on the same box, interleaved:
#   bash tools/ab_lib.sh "<bench args>" reps libA libB ...
ARGS="$1"; REPS="$2"; shift 2
for r in $(seq 1 $REPS); do
  for lib in "$@"; do
    echo -n "$(basename $lib) rep $r: "
    PGB200_LIB=$PWD/paper_1409_7166_b200/lib/$lib python bench.py $ARGS --no-e2e --no-cpu 2>/dev/null | python tools/summ.py
  done
done
