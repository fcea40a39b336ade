"""Reproduce App. B Table 2 on the GPU: direct Monte-Carlo of the paper's simulation
(vinp_patch_ambiguity), next to the exact value (oracle integral) and the paper's printed value.
Multi-GPU: run under torch.distributed.run; trial ranges are split across ranks, hits all-reduced.
  python tools/table2.py [--budget 20] [--out profiles/r01_table2.json]"""
import argparse
import json
import math
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1503_05528_b200 import vinp as V  # noqa: E402
import oracle.oracle as orc  # noqa: E402  (exact reference value only)

SIZES = [("3x3", 9, 8e-2), ("5x5", 25, 1e-2), ("3x3x3", 27, 6e-3), ("7x7", 49, 4.1e-4),
         ("9x9", 81, 5.5e-6), ("11x11", 121, 3e-7), ("5x5x5", 125, 2e-7)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=float, default=20.0, help="seconds per patch size (all ranks)")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world > 1:
        dist.init_process_group("nccl")
    rows = []
    for name, N, paper in SIZES:
        exact = orc.ambiguity_exact(N)
        # calibrate the trial rate on this GPU
        cal = 2_000_000
        V.patch_ambiguity(N, cal, 5.0, 99)
        torch.cuda.synchronize()
        t = time.perf_counter()
        V.patch_ambiguity(N, cal, 5.0, 98)
        torch.cuda.synchronize()
        rate = cal / (time.perf_counter() - t) * world
        want = int(2000 / exact)  # ~2000 expected hits
        trials = int(min(want, rate * args.budget))
        per = -(-trials // world)
        hits = torch.zeros(1, dtype=torch.int64, device="cuda")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        V.patch_ambiguity(N, per, 5.0, 1, trial0=rank * per, hits=hits)
        b.record()
        torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(hits)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        h = int(hits.item())
        n = per * world
        p = h / n
        se = math.sqrt(max(p * (1 - p), 1e-300) / n)
        rows.append(dict(patch=name, N=N, trials=n, hits=h, estimate=p, std_err=se, exact=exact,
                         z=(p - exact) / math.sqrt(exact * (1 - exact) / n), paper=paper,
                         paper_over_exact=paper / exact, seconds=float(ms.item()) / 1000,
                         trials_per_s=n / (float(ms.item()) / 1000)))
        if rank == 0:
            print(json.dumps(rows[-1]), flush=True)
    if rank == 0 and args.out:
        with open(args.out, "w") as f:
            json.dump(dict(n_gpus=world, sigma2=25, rows=rows), f, indent=1)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
