"""Quality (mean d^2 vs exact brute force) of jump-flood schedules at level 1, first outer iteration."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_quality import _quality  # noqa: E402

SCHEDULES = [((8, 4, 2, 1), 0), ((8, 4, 2, 1), 1), ((16, 8, 4, 2, 1), 1), ((32, 16, 8, 4, 2, 1), 1),
             ((64, 32, 16, 8, 4, 2, 1), 1), ((8, 4, 2, 1, 8, 4, 2, 1), 1), ((16, 8, 4, 2, 1, 2, 1), 1)]
if os.environ.get("QS_SCHEDULES"):
    SCHEDULES = json.loads(os.environ["QS_SCHEDULES"])
for name in sys.argv[1:] or ["c1", "c2"]:
    for steps, pol in SCHEDULES:
        import time
        import torch
        t = time.perf_counter()
        q = _quality(name, steps=tuple(steps), sign_policy=pol)
        torch.cuda.synchronize()
        q["wall_s"] = round(time.perf_counter() - t, 2)
        print(json.dumps(q), flush=True)
