"""CPU-side checks of the drop-in boundary: the C-ABI library exists, loads,
and exports every symbol include/fastfca_b200.h declares (no compute calls —
there is no GPU here), and the Python host logic behaves without a device.
"""

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1805_06572_b200 import _backend, _lib
from paper_1805_06572_b200.errors import BackendUnavailableError

REPO = Path(__file__).resolve().parents[1]
HEADER = REPO / "include" / "fastfca_b200.h"


def header_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ffca_[A-Za-z0-9_]+)\s*\(", text)))


def test_header_declares_the_contract():
    syms = header_symbols()
    # the 11 kernel-module functions of the reference plugin + run level
    for name in ("fast_transform", "fast_e_step", "fast_v_update", "S_update",
                 "fast_log_likelihood", "fast_iteration", "fca_e_step", "fca_v_update",
                 "fca_log_likelihood", "fca_iteration", "fastfca_run", "fca_run", "gevd_hpd"):
        assert f"ffca_{name}" in syms


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.ffca_version().decode().startswith("fastfca_b200")
    assert lib.ffca_device_arch() == 100


def test_ctypes_signatures_cover_the_header():
    declared = set(header_symbols())
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert declared == bound


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_run_args_layout_matches_c():
    # 3 int64 + 4 int32 + 10 pointers + size_t + pointer + int64 + 2 pointers
    # + int bin_parts (padded to 8)
    assert ctypes.sizeof(_lib.RunArgs) == 24 + 16 + 8 * 10 + 8 + 8 + 8 + 8 + 8 + 8
    assert _lib.RunArgs.bin_parts.offset == 160


def test_workspace_size_query_needs_no_device():
    lib = _lib.load()
    n = lib.ffca_fastfca_workspace_size(1, 500, 257, 2, 10, 7, 0)
    assert n > 0
    assert lib.ffca_fastfca_workspace_size(1, 500, 257, 9, 10, 7, 0) == 0  # I > 8 rejected
    assert lib.ffca_fca_workspace_size(256, 1250, 257, 4, 20, 1, 0) > 0


def test_backend_selector_is_cuda_only(monkeypatch):
    assert _backend.select_backend("cuda") == "cuda"
    assert _backend.select_backend("auto") == "cuda"
    with pytest.raises(ValueError):
        _backend.select_backend("numpy")
    monkeypatch.setenv("FASTFCA_BACKEND", "numba")
    with pytest.raises(ValueError):
        _backend.select_backend(None)
    monkeypatch.setenv("FASTFCA_BACKEND", "cuda")
    assert _backend.select_backend(None) == "cuda"


def test_product_path_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1805_06572_b200 import fastfca_run, init_random

    y = np.ones((4, 3, 2), dtype=complex)
    with pytest.raises(BackendUnavailableError):
        init_random(y, 0)
    with pytest.raises(BackendUnavailableError):
        from paper_1805_06572_b200.types import SpatialModel

        fastfca_run(y, SpatialModel(np.ones((2, 4, 3)), np.stack([np.eye(2)] * 3)[None].repeat(
            2, 0), np.ones(3) * 1e-9), 1)


def test_package_never_imports_the_oracle():
    pkg = REPO / "paper_1805_06572_b200"
    for p in pkg.rglob("*.py"):
        assert not re.search(r"^\s*(from|import)\s+oracle", p.read_text(), re.M), p


def test_missing_library_raises(tmp_path):
    with pytest.raises(BackendUnavailableError):
        _lib.load(tmp_path / "nope.so")


def test_run_args_offsets_match_the_header(tmp_path):
    """Every ctypes field of RunArgs sits at the offset gcc gives the C struct."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    names = [f[0] for f in _lib.RunArgs._fields_]
    src = tmp_path / "layout.c"
    src.write_text(
        "#include <stddef.h>\n#include <stdio.h>\n#include \"fastfca_b200.h\"\n"
        "int main(void) {\n  printf(\"%zu\\n\", sizeof(ffca_run_args));\n"
        + "".join(f"  printf(\"%zu\\n\", offsetof(ffca_run_args, {n}));\n" for n in names)
        + "  return 0;\n}\n")
    exe = tmp_path / "layout"
    inc = Path(__file__).resolve().parents[1] / "include"
    subprocess.run(["gcc", f"-I{inc}", "-I/usr/local/cuda/include", str(src), "-o", str(exe)],
                   check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    assert got[0] == ctypes.sizeof(_lib.RunArgs)
    assert got[1:] == [getattr(_lib.RunArgs, n).offset for n in names]


def test_status_codes_match_the_header():
    """Every FFCA_* integer constant the header defines has the same value in
    the ctypes layer (status codes, dtypes, flags)."""
    import re

    from paper_1805_06572_b200 import _lib

    text = (REPO / "include" / "fastfca_b200.h").read_text()
    found = 0
    for name, val in re.findall(r"#define\s+(FFCA_\w+)\s+\(?(0x[0-9a-fA-F]+|\d+)u?\)?", text):
        py = getattr(_lib, name, None)
        if py is None:
            py = getattr(_lib, name.replace("FFCA_", "", 1), None)
        assert py is not None, f"{name} missing from _lib"
        assert py == int(val, 0), (name, py, val)
        found += 1
    assert found >= 10
