"""CPU checks of the C-ABI boundary: libm3e.so loads without a GPU and exports
every entry point include/m3e.h declares; the binding's record layouts match the
header's struct sizes; the product path refuses to run without its library."""
import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "m3e.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*|uint64_t)\s+(m3e_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2206_11535_b200 import m3e
    L = ctypes.CDLL(m3e.LIB_PATH)
    names = _declared()
    assert len(names) >= 11
    for n in names:
        assert hasattr(L, n), n
    assert sorted(m3e.EXPORTED) == names
    L.m3e_version.restype = ctypes.c_char_p
    assert b"sm_100a" in L.m3e_version()


def test_record_layouts_match_header():
    from paper_2206_11535_b200 import m3e
    src = open(os.path.join(ROOT, "include", "m3e.h")).read()
    for name, dt in [("m3e_frame_out", m3e.FRAME_DTYPE), ("m3e_track", m3e.TRACK_DTYPE),
                     ("m3e_vertex", m3e.VERTEX_DTYPE), ("m3e_fit_record", m3e.FIT_DTYPE)]:
        m = re.search(r"\((\d+) B\)[^*]*\*/\s*typedef struct %s\b" % name, src)
        assert m, name
        assert int(m.group(1)) == dt.itemsize, name


def test_no_gpu_means_error_not_fallback():
    """Without a CUDA device m3e_create fails loudly (there is no CPU path)."""
    import torch
    if torch.cuda.is_available():
        return
    from paper_2206_11535_b200 import m3e
    try:
        m3e.Context(0)
    except RuntimeError as e:
        assert "libm3e error" in str(e)
    else:
        raise AssertionError("m3e_create succeeded without a GPU")


def test_product_package_does_not_import_oracle():
    import subprocess
    import sys
    code = ("import sys; import paper_2206_11535_b200, paper_2206_11535_b200.m3e; "
            "assert 'oracle' not in sys.modules, 'product imported the oracle'")
    subprocess.check_call([sys.executable, "-c", code], cwd=ROOT)
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2206_11535_b200")):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in txt and "m3e_oracle" not in txt and "or_params" not in txt, fn


def test_library_has_no_unresolved_internal_symbols():
    """Every C++ symbol of the library is defined in it (a shared library links
    with undefined symbols; this catches a missing kernel launcher on CPU)."""
    import subprocess
    from paper_2206_11535_b200 import m3e
    out = subprocess.run(["nm", "-D", "--undefined-only", m3e.LIB_PATH], capture_output=True, text=True).stdout
    bad = [l for l in out.split("\n") if "m3e" in l]
    assert not bad, bad
    ctypes.CDLL(m3e.LIB_PATH, mode=os.RTLD_NOW)
