"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
entry point include/ectgpu.h declares, and fails loudly (no CPU fallback) when
no B200 is present."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "ectgpu.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ect_[a-z0-9_]+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("ect_ctx_create", "ect_mesh_create", "ect_matrix_create", "ect_matrix_assemble",
                 "ect_matrix_export_csc", "ect_rhs_coil", "ect_spmv", "ect_solve",
                 "ect_delta_impedance", "ect_session_create", "ect_session_solve_positions"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_1602_03207_b200 import ect
    lib = ect.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_struct_layouts_match_header():
    from paper_1602_03207_b200 import ect
    # ect_materials: 17 doubles + 2 int32 + complex z_surface (materials.hpp:21-48 order)
    assert ctypes.sizeof(ect.Materials) == 17 * 8 + 8 + 16
    assert ctypes.sizeof(ect.Physics) == ctypes.sizeof(__import__("oracle.ref").ref.Physics)
    assert ctypes.sizeof(ect.SignalPoint) == 8 * 13 + 4 * 5 + 4  # padded to 8
    from oracle import ref
    assert ctypes.sizeof(ref.Materials) == ctypes.sizeof(ect.Materials)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1602_03207_b200 import ect
    with pytest.raises(ect.CudaError):
        ect.Context(0)


def test_built_for_sm100a():
    import subprocess
    lib = ROOT / "paper_1602_03207_b200" / "lib" / "libectgpu.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
