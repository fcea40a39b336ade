"""Mutation check of the oracle's pins (VERDICT r01 "Next round" 1).

Each mutation is a plausible one-token mistake in oracle.c.  For each, a mutated copy of oracle.c
is built in a temp dir (oracle.py builds `$VINP_ORACLE_SRC` instead of oracle/oracle.c) and the
CPU pins are run against it; the mutation is "caught" when at least one pin fails.
usage: python tools/mutation_check.py [--json out.json]
"""
import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")

# (name, passage, old, new, occurrence index of `old` to replace (0-based), or None if unique)
MUTATIONS = [
    ("eq13_layer_lt_to_le", "Eq. 13 P:829-832 (N'_p = layer(q) < j)",
     "!(lv->layer[q] < layer_j)", "!(lv->layer[q] <= layer_j)", None),
    ("propagate_strict_to_le", "R25 P:379 (strictly smaller)",
     "if (D < bestD) {", "if (D <= bestD) {", 0),
    ("random_search_strict_to_le", "R25 P:438 ('<')",
     "if (D < bestD) {", "if (D <= bestD) {", 1),
    ("stop_threshold_0.1_to_1.0", "P:933-934 (e <= 0.1)",
     "return 10 * (__int128)e_fixed <= 3", "return 1 * (__int128)e_fixed <= 3", None),
    ("stop_cap_ge_to_gt", "P:935-936 (at most 20 iterations)",
     "if (k >= max_outer) return 1;", "if (k > max_outer) return 1;", None),
    ("r20_unweighted_skips_n0", "R20 P:921-922 / P:499 (s = 1 after upsampling)",
     "if (mode != OR_UNWEIGHTED && nnf->n[s] == 0) continue;", "if (nnf->n[s] == 0) continue;", None),
    ("onion_writes_later_layers", "S:400 / S:417 (layer j written once, earlier frozen)",
     "if (layer_j >= 0 && lv->layer[p] != layer_j) continue;",
     "if (layer_j >= 0 && lv->layer[p] < layer_j) continue;", None),
    ("onion_commit_ge_j", "S:400 (each hole voxel committed once)",
     "if (lv->layer[lv->holes[hh]] == j) {", "if (lv->layer[lv->holes[hh]] >= j) {", None),
    ("propagate_dup_not_skipped", "R33 (duplicates are not evaluated or counted)",
     "      if (dup) continue;\n", "      (void)dup;\n", 0),
    ("random_search_dup_not_skipped", "R33 (duplicates are not evaluated or counted)",
     "      if (dup) continue;\n", "      (void)dup;\n", 1),
    ("percentile_rank_floor", "R10 P:495-496 (nearest rank ceil(0.75 m))",
     "int r = (3 * m + 3) / 4;", "int r = (3 * m) / 4 + (m < 4);", None),
    ("stale_own_entry", "R41 (stale: the neighbour's entry, not the target's)",
     "if (prev && prev->dx[rs] == vx && prev->dy[rs] == vy && prev->dt[rs] == vt) nst += 1;",
     "if (prev && prev->dx[s] == vx && prev->dy[s] == vy && prev->dt[s] == vt) nst += 1;", None),
    ("stale_before_dedup", "R41 (stale counted among evaluated candidates, after R33)",
     "      if (dup) continue;\n      seen[nseen][0] = vx; seen[nseen][1] = vy; seen[nseen][2] = vt; ++nseen;\n      /* R41",
     "      if (prev && prev->dx[rs] == vx && prev->dy[rs] == vy && prev->dt[rs] == vt) nst += 1;\n"
     "      if (dup) continue;\n      seen[nseen][0] = vx; seen[nseen][1] = vy; seen[nseen][2] = vt; ++nseen;\n      /* R41",
     None),
    ("best_patch_tie_last", "R13 / S:324 (ties -> smallest q)",
     "if (key_less(nnf->D[cs[i]], nnf->n[cs[i]], nnf->D[cs[best]], nnf->n[cs[best]])) best = i;",
     "if (!key_less(nnf->D[cs[best]], nnf->n[cs[best]], nnf->D[cs[i]], nnf->n[cs[i]])) best = i;", None),
]

PINS = ["tests/test_oracle_pins.py", "tests/test_oracle_rules.py"]


def apply(src, old, new, occ):
    if occ is None:
        assert src.count(old) == 1, (old, src.count(old))
        return src.replace(old, new)
    i = -1
    for _ in range(occ + 1):
        i = src.index(old, i + 1)
    return src[:i] + new + src[i + len(old):]


def main():
    base = open(SRC).read()
    rows = []
    for name, passage, old, new, occ in MUTATIONS:
        d = tempfile.mkdtemp(prefix="mut_")
        try:
            path = os.path.join(d, "oracle.c")
            with open(path, "w") as f:
                f.write(apply(base, old, new, occ))
            env = dict(os.environ, VINP_ORACLE_SRC=path)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x",
                                "-m", "not gpu", *PINS], cwd=ROOT, env=env, capture_output=True, text=True)
            failed = [l.split(" ")[1] for l in r.stdout.splitlines() if l.startswith("FAILED")]
            rows.append(dict(mutation=name, passage=passage, caught=r.returncode != 0,
                             first_failing_pin=failed[0] if failed else None))
            print(json.dumps(rows[-1]), flush=True)
        finally:
            shutil.rmtree(d, ignore_errors=True)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(rows, f, indent=1)
    return 0 if all(r["caught"] for r in rows) else 1


if __name__ == "__main__":
    sys.exit(main())
