"""The oracle under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY §5 aux item): whole Alg. 4
(or_inpaint, 2 levels with the onion peel and the stopping rule) and the realignment chain on a
small volume, built from oracle/oracle.c with `-fsanitize=address,undefined` into a standalone
driver (tests/native/oracle_asan_main.c).  Any sanitizer report or a leak fails the test; the
output must equal the normal oracle build's."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _build(tmp_path):
    exe = str(tmp_path / "oracle_asan")
    cmd = ["gcc", "-O1", "-g", "-std=c11", "-ffp-contract=off", "-fopenmp", "-fno-omit-frame-pointer",
           "-fsanitize=address,undefined", "-fno-sanitize-recover=all", "-I", os.path.join(ROOT, "oracle"),
           os.path.join(ROOT, "tests", "native", "oracle_asan_main.c"), os.path.join(ROOT, "oracle", "oracle.c"),
           "-lm", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0 and "sanitize" in r.stderr and "cannot find" in r.stderr:
        pytest.skip("sanitizer runtime not installed")
    assert r.returncode == 0, r.stderr[-3000:]
    return exe


def test_oracle_pipeline_under_asan_ubsan(tmp_path, orc):
    from gen.synth import random_volume
    exe = _build(tmp_path)
    v, m, _ = random_volume(36, 28, 10, seed=5, hole_frac=0.06)
    v, m = v.numpy(), m.numpy()
    T, H, W, _ = v.shape
    fi, fm, fo = (str(tmp_path / n) for n in ("rgb.u8", "mask.u8", "out.u8"))
    v.tofile(fi)
    m.tofile(fm)
    env = dict(os.environ, OMP_NUM_THREADS="2",
               ASAN_OPTIONS="detect_leaks=1:abort_on_error=0:halt_on_error=1",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1")
    r = subprocess.run([exe, str(W), str(H), str(T), "2", "2", "0", fi, fm, fo], capture_output=True,
                       text=True, env=env, timeout=600)
    assert r.returncode == 0 and "runtime error" not in r.stderr and "ERROR: " not in r.stderr, \
        (r.returncode, r.stderr[-4000:])
    out = np.fromfile(fo, dtype=np.uint8).reshape(v.shape)
    ref, _ = orc.inpaint(v, m, 2, pm_iters=2)
    assert np.array_equal(out, ref)
