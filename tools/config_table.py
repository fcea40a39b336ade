"""BASELINE.md §3 results table on one GPU: for each config, a full Alg. 4 run (after one warm-up)
with per-level CUDA-event times, outer iterations, patch-updates, patch-updates/s and the
algorithmic-byte model fraction of the measured HBM bandwidth."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from gen.synth import CONFIGS, generate  # noqa: E402
from paper_1503_05528_b200 import Config, Inpainter  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def main():
    rows = []
    for name in sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]:
        c = CONFIGS[name]
        v, m, _ = generate(name, device="cuda")
        cfg = Config(levels=c.levels, pm_iters=c.pm_iters, fixed_outer=c.fixed_outer, max_outer=c.max_outer,
                     lam=c.lam, seed=c.seed, graphs=os.environ.get("VINP_NO_GRAPHS") is None)
        ip = Inpainter(c.W, c.H, c.T, cfg, "cuda")
        ip.load(v, m)
        ip.run()  # warm-up
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ip.load(v, m)
        st = ip.run(timing=True)
        b.record()
        torch.cuda.synchronize()
        total = a.elapsed_time(b) / 1000
        pu = st.total_patch_updates
        row = dict(config=name, dims=[c.W, c.H, c.T], levels=c.levels, step_s=total,
                   patch_updates=pu, stale_skipped=st.total_stale_skipped, patch_updates_per_s=pu / total,
                   graphs=cfg.graphs,
                   model_frac_of_hbm=(625 * pu / total / 1e9) / HBM,
                   levels_detail=[dict(level=l["level"], outer=l["outer"], s=l["ms"] / 1000) for l in st.levels],
                   onion_s=st.onion_ms / 1000, onion_layers=st.onion_layers,
                   targets_l1=ip.levels[0].n_targets, holes_l1=ip.levels[0].n_holes)
        print(json.dumps(row), flush=True)
        rows.append(row)
        del ip
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(rows, open(os.path.join(ROOT, "gpurun_out", "config_table.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
