"""CPU-only: the C-ABI library loads and exports every symbol include/vinp.h declares."""
import os
import re
import subprocess

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
