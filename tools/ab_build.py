"""Build A/B variants of libvinp.so into build_variants/ (dev only).
usage: python tools/ab_build.py NAME=DEF1,DEF2 [NAME2=...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1503_05528_b200.build import build, ROOT  # noqa: E402

for spec in sys.argv[1:]:
    name, defs = spec.split("=", 1)
    out = os.path.join(ROOT, "build_variants", f"{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    build(force=True, defines=[d for d in defs.split(",") if d], out=out)
    print(out)
