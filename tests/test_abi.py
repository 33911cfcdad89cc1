"""CPU checks of the boundary: libfk.so loads and exports every symbol include/fk.h declares
(no compute calls without a GPU), and the Python binding carries the same names."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_five_calls():
    names = _declared()
    for f in ("fk_moments_type1", "fk_rhs_type1", "fk_additive_cross_moments", "fk_solve", "fk_predict_type2"):
        assert f in names
    assert "fk_workspace_bytes" in names and "fk_last_error" in names


def test_library_exports_every_declared_symbol():
    from paper_2509_02649_b200 import build

    path = build.build()
    lib = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(lib, name), name
    lib.fk_version.restype = ctypes.c_char_p
    assert lib.fk_version().startswith(b"fk ")


def test_binding_has_the_c_names():
    from paper_2509_02649_b200 import fk

    for name in _declared():
        if name in ("fk_last_error", "fk_version"):
            continue
        assert callable(getattr(fk, name)), name


def test_no_oracle_in_product_path():
    """The product package never imports the oracle (the two share no code)."""
    pkg = os.path.join(ROOT, "paper_2509_02649_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle/" not in txt, f
