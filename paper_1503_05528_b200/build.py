"""Builds libvinp.so (sm_100a) in-tree with nvcc.  `python -m paper_1503_05528_b200.build`."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libvinp.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr"]

# align.cu: fp64 expressions evaluated as written (no FMA contraction), like the oracle (R38)
PER_FILE = {"align.cu": ["-fmad=false"]}


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(os.path.join(HERE, "csrc", "*.inc")) + [os.path.join(ROOT, "include", "vinp.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out=None) -> str:
    """defines/out: variant builds for A/B timing (tools/); the product uses the defaults."""
    lib = out or LIB
    if not force and not defines and not _stale():
        return LIB
    objs = []
    log = []
    for src in sources():
        tag = "" if not defines else "_" + os.path.basename(lib)[:-3]
        obj = os.path.join(HERE, "csrc", os.path.basename(src)[:-3] + tag + ".o")
        extra = PER_FILE.get(os.path.basename(src), [])
        cmd = [NVCC, *ARCH, *FLAGS, *extra, *["-D" + d for d in defines], "-I", os.path.join(ROOT, "include"),
               "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append(r.stderr)
        if r.returncode != 0:
            errs = [l for l in r.stderr.splitlines() if "error" in l.lower()]
            raise RuntimeError(f"nvcc failed on {src}:\n" + "\n".join(errs[:20] or [r.stderr[-4000:]]))
        objs.append(obj)
    cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    with open(os.path.join(HERE, "csrc", "ptxas.log" if not defines else f"ptxas{tag}.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
