"""Whole-pipeline parity at BASELINE.json's full sizes (VERDICT r01 "Next round" 2).

* c4 (1280x720x120, L = 4, K = 10, stopping rule): the entire Alg. 4 on the GPU in the
  bench's launch configuration against `or_inpaint` on the host cores: per-level outer-iteration
  counts, per-level patch-update counts, the stopping statistic of every outer iteration, and the
  output video, bit for bit.  (c5 the same with VINP_E2E_C5=1: ~10 min of oracle time.)
* c5 level 1, one complete outer iteration, every target slot: the GPU state is brought to the
  first outer iteration of level 1 exactly as Alg. 4 does; then for each of the 51 passes of the
  ANN search (evaluate, 10 x (4 propagations + random search)) the oracle recomputes the pass over
  ALL 18.0 M target slots from the GPU's input state of that pass, and the weighted reconstruction
  over all 16.6 M holes: NNF words bit-exact, patch-update counts equal, fp32 values within 1e-3
  and the committed u8 working copy equal.
"""
import os

import numpy as np
import pytest
import torch

from gen.synth import CONFIGS, generate
import oracle_ops as OO

pytestmark = pytest.mark.gpu


def _cfg(c):
    from paper_1503_05528_b200 import Config
    return Config(levels=c.levels, pm_iters=c.pm_iters, fixed_outer=c.fixed_outer, max_outer=c.max_outer,
                  lam=c.lam, seed=c.seed)


@pytest.mark.parametrize("name", ["c4"] + (["c5"] if os.environ.get("VINP_E2E_C5") else []))
def test_whole_pipeline_full_size(orc, name):
    from paper_1503_05528_b200 import inpaint
    c = CONFIGS[name]
    v, m, _ = generate(name)
    out, stats, _ = inpaint(v, m, _cfg(c), device="cuda")
    g = out.cpu().numpy()
    ref, st = orc.inpaint(v.numpy(), m.numpy(), c.levels, pm_iters=c.pm_iters, fixed_outer=c.fixed_outer,
                          max_outer=c.max_outer, lam=c.lam, seed=c.seed)
    report = dict(outer_gpu=[l["outer"] for l in stats.levels], outer_orc=st["outer_iters"],
                  pu_gpu=[l["patch_updates"] for l in stats.levels], pu_orc=st["patch_updates"],
                  stale_gpu=[l["stale_skipped"] for l in stats.levels], stale_orc=st["stale"],
                  diff_voxels=int((g != ref).any(-1).sum()))
    print(name, report)
    for l in range(c.levels):
        assert stats.levels[l]["change_fixed"] == st["change_fixed"][l], ("stopping statistic", l + 1)
    assert report["outer_gpu"] == report["outer_orc"]
    # R41: evaluated + skipped stale = the oracle's count, and the skipped sets agree
    assert report["stale_gpu"] == report["stale_orc"]
    assert [a + b for a, b in zip(report["pu_gpu"], report["stale_gpu"])] == report["pu_orc"]
    assert report["diff_voxels"] == 0


def _level1_state(name):
    """Alg. 4 down to the first outer iteration of level 1 (onion peel, one outer iteration per
    coarser level... exactly as many as Alg. 4 runs there, upsample, unweighted reconstruction)."""
    from paper_1503_05528_b200 import Inpainter, vinp as V
    from paper_1503_05528_b200.driver import stop_now
    c = CONFIGS[name]
    v, m, _ = generate(name, device="cuda")
    ip = Inpainter(c.W, c.H, c.T, _cfg(c), "cuda")
    ip.load(v, m)
    ip.onion_peel()
    for l in range(c.levels, 1, -1):
        s_, f_ = ip.states[l - 1], ip.states[l - 2]
        k = 0
        while True:
            s_.prev_rgb.copy_(s_.cur_rgb)
            ip.ann_search(s_, k)
            ip.reconstruct(s_, V.WEIGHTED)
            ip.change.zero_()
            V.change_l1(s_.cur_rgb[:s_.lv.n_holes], s_.prev_rgb[:s_.lv.n_holes], ip.change)
            k += 1
            if stop_now(int(ip.change.item()), s_.lv.n_holes, k, c.max_outer):
                break
        V.nnf_upsample(s_.lv, s_.a, f_.lv, f_.a, ip.prm)
        ip.reconstruct(f_, V.UNWEIGHTED)
    torch.cuda.synchronize()
    return ip


def test_c5_level1_one_outer_iteration_every_slot(orc):
    from paper_1503_05528_b200 import vinp as V
    ip = _level1_state("c5")
    st = ip.states[0]
    lv = st.lv
    prm = ip.prm
    nt, nh = lv.n_targets, lv.n_holes
    host = V.Level(lv.W, lv.H, lv.T, 1, torch.device("cpu"))
    for name in ("vox", "flags", "slot", "targets", "holes", "sources"):
        setattr(host, name, getattr(lv, name).cpu())
    host.n_targets, host.n_holes, host.n_sources = nt, nh, lv.n_sources
    ol = OO._OLevel(host)
    cnt = torch.zeros(2, dtype=torch.int64, device="cuda")  # evaluated, stale skipped (R41)
    assert st.a.stamp is not None and st.b.stamp is not None

    def gpu(x):
        return OO._to_orc(host, V.NNF(x.e.cpu(), x.n.cpu()))

    def equal(f, g, what):
        for arr in ("dx", "dy", "dt", "D", "n"):
            a, b = getattr(f, arr)[:nt], getattr(g, arr)[:nt]
            if not np.array_equal(a, b):
                bad = np.flatnonzero(a != b)
                raise AssertionError(f"{what}: {arr} differs at {bad.size} slots, first {bad[:5]}")

    # evaluate
    f_in = gpu(st.a)
    cnt.zero_()
    V.nnf_evaluate(lv, st.a, prm, counter=cnt)
    f_ref = f_in.copy()
    c_ref = orc.evaluate(ol, f_ref, prm.lam)
    equal(gpu(st.a), f_ref, "evaluate")
    assert int(cnt[0]) == c_ref
    passes = 1
    total = c_ref
    skipped = 0
    clk = V.PassClock()
    snaps = {}
    for k in range(1, ip.cfg.pm_iters + 1):
        sign = 1 if k % 2 == 1 else -1
        for s in ip.cfg.steps:
            f_in = gpu(st.a)
            cnt.zero_()
            V.propagate(lv, st.a, st.b, prm, s, sign, counter=cnt, pass_id=clk.pass_id,
                        since=clk.since(s, sign))
            clk.tick(s, sign)
            f_ref = f_in.copy()
            stale = np.zeros(1, np.int64)
            c_ref = orc.propagate(ol, f_in, f_ref, prm.lam, s, sign, prev=snaps.get((s, sign)), stale=stale)
            snaps[(s, sign)] = f_in
            equal(gpu(st.b), f_ref, f"propagate k={k} s={s}")
            assert int(cnt[1]) == int(stale[0]), ("stale count", k, s)
            assert int(cnt[0]) + int(cnt[1]) == c_ref, ("propagate count", k, s)
            st.a, st.b = st.b, st.a
            passes += 1
            total += c_ref
            skipped += int(stale[0])
        f_in = gpu(st.a)
        cnt.zero_()
        V.random_search(lv, st.a, st.b, prm, 0, k, counter=cnt, pass_id=clk.pass_id)
        clk.tick()
        f_ref = f_in.copy()
        c_ref = orc.random_search(ol, f_in, f_ref, prm.lam, prm.seed, prm.rho, ol.rmax, 1, 0, k)
        equal(gpu(st.b), f_ref, f"random search k={k}")
        assert int(cnt[0]) == c_ref, ("random search count", k)
        st.a, st.b = st.b, st.a
        passes += 1
        total += c_ref
    assert passes == 51
    # weighted reconstruction of every hole, then the committed working copy
    f_a = gpu(st.a)
    V.reconstruct(lv, st.a, V.WEIGHTED, st.cur_rgb, st.cur_tex, commit=True)
    g_rgb = st.cur_rgb[:nh].cpu().numpy()
    g_tex = st.cur_tex[:nh].cpu().numpy()
    o_rgb = np.zeros((nh, 3), np.float32)
    o_tex = np.zeros((nh, 2), np.float32)
    orc.reconstruct(ol, f_a, orc.WEIGHTED, -1, 0, nh, o_rgb, o_tex)
    err = max(np.abs(o_rgb - g_rgb).max(), np.abs(o_tex - g_tex).max())
    exact = float(np.mean(o_rgb == g_rgb))
    print(f"c5 l1 outer iteration: {total} candidates ({skipped} stale, skipped on the GPU), "
          f"reconstruct max |err| {err:.2e}, exact {exact:.6f}")
    assert skipped > 0
    assert err <= 1e-3
    orc.commit(ol, o_rgb, o_tex, 0, nh)
    vb = lv.vox.view(torch.uint8).view(lv.N, 8).cpu().numpy()
    holes = host.holes.numpy()[:nh]
    assert np.array_equal(vb[holes, :3], ol.rgb[holes]) and np.array_equal(vb[holes, 4:6], ol.tex[holes])
