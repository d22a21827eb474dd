"""The drop-in boundary: C ABI exports, no oracle/CPU fallback in the product.

* libolsb.so loads on a CPU-only machine and exports every symbol declared
  in include/olsb.h (no compute calls without a GPU);
* the product package never imports the oracle or the reference;
* the engine fails loudly when there is no CUDA device.
"""

import ctypes
import os
import re

import pytest

from conftest import ROOT, has_gpu

PKG = os.path.join(ROOT, "paper_1910_01972_b200")
HEADER = os.path.join(ROOT, "include", "olsb.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(olsb_\w+)\s*\(", text,
                                 flags=re.M)))


def test_header_declares_the_plugin_seam():
    syms = header_symbols()
    for must in ("olsb_fused_c2c", "olsb_filter_spectra_c2c",
                 "olsb_dif_fwd_batch", "olsb_dit_inv_batch",
                 "olsb_spectra_perm_to_dev", "olsb_error_string"):
        assert must in syms


def test_library_builds_and_exports_every_header_symbol():
    from paper_1910_01972_b200 import _lib
    from paper_1910_01972_b200 import build as B
    path = B.build()
    lib = ctypes.CDLL(path)
    for sym in header_symbols():
        assert hasattr(lib, sym), sym
    # the ctypes binding covers the header exactly
    assert set(_lib.SIGNATURES) == set(header_symbols())
    # argument validation needs no GPU
    _lib.load()
    L = _lib.load()
    assert L.olsb_version() >= 100
    assert L.olsb_spectra_dev_len(2048) == 2048
    assert L.olsb_spectra_dev_len(3000) == -1
    assert L.olsb_dif_fwd_batch(None, None, 1, 100, 0, None) == -1
    assert L.olsb_dif_fwd_batch(None, None, 1, 64, 0, None) == -2
    assert L.olsb_dif_fwd_batch(None, None, 0, 64, 7, None) == 0
    assert L.olsb_fused_c2c(None, 0, 10, None, 1, 64, 5, 0, 60, 4, -4, 0, 1,
                            2, 1.0, None, 10, 0, 0, None) == -4
    assert b"power of two" in L.olsb_error_string(-1)


def test_library_is_sm100a_code():
    import subprocess
    from paper_1910_01972_b200 import build as B
    res = subprocess.run(["cuobjdump", "--list-elf", B.build()],
                         capture_output=True, text=True)
    assert "sm_100a" in res.stdout


def test_product_never_imports_oracle_or_reference():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if not f.endswith((".py", ".cu", ".cuh", ".h")):
                continue
            src = open(os.path.join(dirpath, f)).read()
            assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
            assert not re.search(r"^\s*(import|from)\s+olsconv\b", src,
                                 re.M), f
            assert "/root/reference" not in src, f


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure mode")
def test_engine_fails_loudly_without_gpu():
    import paper_1910_01972_b200 as oc
    with pytest.raises(RuntimeError):
        oc.make_signal([1 + 1j, 2], "complex")
