"""CPU checks of the C ABI library: it loads and exports every symbol that
include/rc.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rc_[a-z_]+)\s*\(", src)))


def test_build_and_exports():
    from paper_1809_01334_b200 import build
    so = build.build()
    lib = ctypes.CDLL(so)
    names = declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), f"librc.so does not export {n}"
    lib.rc_version.restype = ctypes.c_int32
    assert lib.rc_version() == 4


def test_binding_covers_header():
    from paper_1809_01334_b200 import rc
    assert set(declared_symbols()) <= set(rc.EXPORTS)


def test_no_oracle_in_product():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_1809_01334_b200")
    for dp, _, fns in os.walk(pkg):
        for fn in fns:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, fn), errors="ignore").read()
                assert "import oracle" not in txt and "liboracle" not in txt and "oracle.h" not in txt, fn
