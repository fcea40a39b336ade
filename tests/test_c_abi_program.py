"""The C ABI on its own: examples/c_pipeline.c drives Alg. 4 (one level, c1 configuration) through
include/vinp.h with cudaMalloc'd buffers and no Python/torch in the loop.  CPU: it compiles with
-Wall -Werror against the header and links against libvinp.so (every declaration it uses resolves).
GPU: its output video and patch-update count equal the oracle's, bit for bit."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1503_05528_b200")
CUDA = "/usr/local/cuda"


def _compile(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "libvinp.so")):
        pytest.skip("libvinp.so not built")
    exe = str(tmp_path / "c_pipeline")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I",
           f"{CUDA}/include", os.path.join(ROOT, "examples", "c_pipeline.c"), "-L", LIBDIR, "-lvinp",
           "-L", f"{CUDA}/lib64", "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_compiles_and_links(tmp_path):
    _compile(tmp_path)


@pytest.mark.gpu
def test_c_program_equals_oracle(tmp_path, orc):
    from gen.synth import generate
    exe = _compile(tmp_path)
    v, m, _ = generate("c1")
    v, m = v.numpy(), m.numpy()
    T, H, W, _ = v.shape
    fi, fm, fo = (str(tmp_path / n) for n in ("rgb.u8", "mask.u8", "out.u8"))
    v.tofile(fi)
    m.tofile(fm)
    r = subprocess.run([exe, str(W), str(H), str(T), "4", "3", fi, fm, fo], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    out = np.fromfile(fo, dtype=np.uint8).reshape(v.shape)
    ref, st = orc.inpaint(v, m, 1, pm_iters=4, fixed_outer=3)
    assert np.array_equal(out, ref)
    pu = int(r.stdout.split("patch-updates")[1].split()[0])
    stale = int(r.stdout.split("stale-skipped")[1].split()[0])
    assert stale == sum(st["stale"])  # R41
    assert pu + stale == sum(st["patch_updates"])
