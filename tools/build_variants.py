"""Build experiment libraries lib/libpgb200_<name>.so with extra -D flags:
    python tools/build_variants.py name=DEF1,DEF2 name2=DEF3 ..."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1409_7166_b200 import build as B  # noqa: E402

for spec in sys.argv[1:]:
    name, _, defs = spec.partition("=")
    print(B.build(variant=name, defs=tuple(d for d in defs.split(",") if d)))
