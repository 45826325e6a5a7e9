"""CPU: the C-ABI library builds for sm_100a, loads, and exports every function include/subspec.h
declares; the ctypes binding covers exactly that surface.  No compute calls (no GPU here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    h = open(os.path.join(ROOT, "include", "subspec.h")).read()
    h = re.sub(r"/\*.*?\*/", "", h, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z_0-9]+)\s*\(", h)))


def test_header_declares_the_method_calls():
    d = _declared()
    for name in ("ss_load_weights", "ss_build_substitutes", "ss_draft_tree", "ss_verify_tree",
                 "ss_accept_and_commit", "ss_create", "ss_destroy", "ss_prefill", "ss_last_error"):
        assert name in d


def test_library_builds_loads_and_exports_all():
    from paper_2509_18344_b200.build import build
    lib_path = build()
    lib = ctypes.CDLL(lib_path)
    for name in _declared():
        assert hasattr(lib, name), name


def test_binding_covers_header():
    from paper_2509_18344_b200 import binding
    assert sorted(binding.EXPORTED) == _declared()


def test_sass_uses_tensor_cores_and_tma():
    """The dequant-GEMV is compiled for sm_100a with HMMA (tensor cores) and UBLKCP (TMA bulk copy)."""
    import subprocess
    from paper_2509_18344_b200.build import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    assert "HMMA" in out and "UBLKCP" in out
