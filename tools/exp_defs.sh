set -e
for defs in "-DPG_L2_AHEAD=0" "-DPG_L2_AHEAD=2" "-DPG_L2_AHEAD=4" "-DPG_L2_AHEAD=8"; do
  PG_EXTRA_DEFS="$defs" python -m paper_1409_7166_b200.build --force --prof > /dev/null 2>&1
  echo "=== defs: $defs"
  PGB200_LIB=paper_1409_7166_b200/lib/libpgb200_prof.so timeout 200 python tools/phase_prof.py fuse=2 fuse=2,width=32
done
