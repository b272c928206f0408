"""C-ABI surface checks that need no GPU: every function declared in
include/fairsched_b200.h is exported by libfsb200.so and bound in _lib.py, and
without a device the library fails loudly (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fairsched_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_functions():
    fns = header_functions()
    assert "fs_worker_fill" in fns and "fs_dispatch" in fns and "fs_trie_match" in fns
    assert len(fns) >= 40


def test_library_exports_every_header_symbol():
    from paper_2501_14312_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_ctypes_bindings_cover_header():
    from paper_2501_14312_b200 import _lib
    assert set(_lib.SIGNATURES) == set(header_functions())
    _lib.load()


def test_fill_result_struct_layout():
    # fs_fill_result / fs_records field order must match the header
    from paper_2501_14312_b200 import _lib
    text = open(HEADER).read()
    body = text[text.index("typedef struct {\n    int64_t cap_adm;"):]
    body = body[: body.index("} fs_fill_result;")]
    names = re.findall(r"\*?\s*([a-z_]+);", body)
    names = [n for n in names if n not in ("fs_records",)]
    assert [f for f, _ in _lib.FsFillResult._fields_] == ["cap_adm", "adm_req", "adm_mlen", "adm_unpinned",
                                                           "adm_pinned_before", "adm_path_node", "adm_rec_end",
                                                           "recs", "n_adm", "n_queued", "used", "pinned",
                                                           "device_ms"]
    assert names[:7] == ["cap_adm", "adm_req", "adm_mlen", "adm_unpinned", "adm_pinned_before",
                         "adm_path_node", "adm_rec_end"]


def _has_gpu():
    from paper_2501_14312_b200 import _lib
    n = ctypes.c_int(0)
    return _lib.load().fs_device_count(ctypes.byref(n)) == 0 and n.value > 0


def test_no_cpu_fallback_without_device():
    if _has_gpu():
        pytest.skip("a GPU is present")
    from paper_2501_14312_b200 import FsError
    from paper_2501_14312_b200.device import Context
    with pytest.raises(FsError) as ei:
        Context(0)
    assert ei.value.code == 2 and "no CPU fallback" in str(ei.value)


def test_policies_refuse_non_device_worker():
    from types import SimpleNamespace

    from paper_2501_14312_b200.policies import GpuDlpm
    pol = GpuDlpm(10)
    pol.attach(SimpleNamespace(queue=[], batch={}, tree=object()))
    with pytest.raises(TypeError):
        pol.fill()
