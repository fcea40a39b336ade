"""Quality (mean d^2 vs exact brute force) of jump-flood schedules at level 1, first outer iteration."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_quality import _quality  # noqa: E402

SCHEDULES = [((8, 4, 2, 1), 0), ((8, 4, 2, 1), 1), ((16, 8, 4, 2, 1), 0), ((4, 2, 1), 1),
             ((16, 8, 4, 2, 1), 1), ((2, 1), 1), ((1,), 1)]
for name in sys.argv[1:] or ["c1", "c2"]:
    for steps, pol in SCHEDULES:
        print(json.dumps(_quality(name, steps=steps, sign_policy=pol)), flush=True)
