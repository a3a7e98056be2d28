"""CPU-side checks of the boundary (-m "not gpu"): the C-ABI library builds, loads and exports
every symbol include/tsw.h declares; argument structs match the header; no CPU fallback."""
import ctypes
import os
import re

import pytest

from paper_2005_11931_b200 import build, tsw

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "tsw.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tsw_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    path = build.build()
    lib = ctypes.CDLL(path)
    declared = _declared()
    assert len(declared) >= 19
    for name in declared:
        assert hasattr(lib, name), f"libtsw.so does not export {name}"
    assert sorted(tsw.EXPORTS) == declared


def test_struct_layout_matches_header():
    assert ctypes.sizeof(tsw.tsw_grid_desc) == 4 + 4 + 8 + 8 + 8 + 8 + 4 * 6 + 8
    assert tsw.tsw_grid_desc.nx.offset == 8
    assert tsw.tsw_grid_desc.stream.offset == 64
    assert ctypes.sizeof(tsw.tsw_coeff_desc) == 4 + 4 + 8 * 4 + 8 + 8


def test_sm100a_code_in_library():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", build.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_no_cpu_fallback():
    assert "sm_100a" in tsw.tsw_version()
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    with pytest.raises(tsw.TswError) as e:
        tsw.tsw_create(2, 64, 64, 0.1, 0.1)
    assert e.value.status == tsw.TSW_ERR_CUDA
    assert "no CPU fallback" in str(e.value)


def test_argument_validation_before_device_work():
    # invalid grids are rejected before any CUDA call (status ARG, not CUDA)
    for args in ((3, 64, 64, 0.1, 0.1), (2, 2, 64, 0.1, 0.1), (2, 64, 64, -0.1, 0.1), (1, 64, 5, 0.1, 0.1)):
        with pytest.raises(tsw.TswError) as e:
            tsw.tsw_create(*args)
        assert e.value.status == tsw.TSW_ERR_ARG
    with pytest.raises(tsw.TswError) as e:
        tsw.tsw_create(2, 64, 64, 0.1, 0.1, rank=2, nranks=2)
    assert e.value.status == tsw.TSW_ERR_ARG
