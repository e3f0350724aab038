"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/kronphi_b200.h declares (no compute without a
GPU), and the Python binding knows all of them."""
import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "kronphi_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(kp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2304_02327_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header():
    from paper_2304_02327_b200 import _lib
    _lib.load()
    bound = set(_lib.EXPORTS) | {n for n, _, _ in _lib._EXTRA_SIGS}
    missing = [s for s in declared_symbols() if s not in bound]
    assert not missing, missing


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2304_02327_b200 as kp
    with pytest.raises(kp.KronphiError):
        kp.Context(0)


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS (no PTX JIT, no other arch)."""
    import subprocess
    from paper_2304_02327_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)
