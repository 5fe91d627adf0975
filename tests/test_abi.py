"""The C-ABI library loads, exports every symbol declared in include/tnc.h and
agrees with the ctypes struct layouts (no GPU needed)."""

import re
from pathlib import Path

from paper_2011_02621_b200 import _native as NV

ROOT = Path(__file__).resolve().parents[1]


def test_header_declares_exactly_the_bound_symbols():
    hdr = (ROOT / "include" / "tnc.h").read_text()
    declared = set(re.findall(r"\b(tnc_[a-z_]+)\s*\(", hdr))
    assert declared == set(NV.EXPORTS)


def test_library_exports_all_symbols():
    L = NV.lib()
    for name in NV.EXPORTS:
        assert hasattr(L, name), name
    assert L.tnc_version() >= 100


def test_struct_layouts_match():
    import ctypes as C

    L = NV.lib()
    for i, cls in enumerate((NV.Site, NV.StepDesc, NV.ProjectDesc, NV.SliceSumDesc, NV.PathDesc)):
        assert L.tnc_struct_size(i) == C.sizeof(cls), cls.__name__


def test_device_check_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        return
    L = NV.lib()
    assert L.tnc_device_check() != 0
    assert L.tnc_last_error()
