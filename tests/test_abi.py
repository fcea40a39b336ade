"""CPU-only: the C-ABI library loads and exports every symbol include/vinp.h declares."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "vinp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vinp_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    from paper_1503_05528_b200 import build, vinp
    names = _declared()
    assert len(names) >= 24
    nm = subprocess.run(["nm", "-D", "--defined-only", vinp.LIB_PATH], capture_output=True, text=True,
                        check=True).stdout
    exported = set(re.findall(r"\b(vinp_[a-z0-9_]+)\b", nm))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert sorted(vinp.EXPORTED) == names  # the binding wraps every declared call


def test_library_is_sm100a():
    from paper_1503_05528_b200 import vinp
    out = subprocess.run(["cuobjdump", "--list-elf", vinp.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_argument_errors_are_synchronous():
    """Bad arguments fail before any device work (no GPU needed)."""
    import pytest
    from paper_1503_05528_b200 import vinp
    lv = vinp.Level(W=0, H=0, T=0, level=1, device=None)
    with pytest.raises(vinp.VinpError):
        vinp.build_pyramid(None, None, [lv]) if False else vinp._check(
            vinp._lib.vinp_build_pyramid(None, None, None, 1, None), "vinp_build_pyramid")
    rc = vinp._lib.vinp_change_l1(None, None, 1, None, None)
    assert rc == 1 and b"bad args" in vinp._lib.vinp_last_error()


def test_level_dims_host_only():
    """vinp_level_dims is host-only (no GPU): ceil halving of W and H, T unchanged."""
    from paper_1503_05528_b200 import vinp
    assert vinp.level_dims(1920, 1080, 100, 4) == [(1920, 1080, 100), (960, 540, 100), (480, 270, 100),
                                                   (240, 135, 100)]
    assert vinp.level_dims(854, 480, 7, 3) == [(854, 480, 7), (427, 240, 7), (214, 120, 7)]
    with pytest.raises(vinp.VinpError):
        vinp.level_dims(4096, 4096, 200, 1)  # >= 2^31 voxels
    with pytest.raises(vinp.VinpError):
        vinp.level_dims(10, 10, 10, 0)
