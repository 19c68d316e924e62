"""The C-ABI library loads on CPU, exports exactly what include/svb200.h declares, and
rejects bad arguments before touching CUDA (no compute calls here)."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "svb200.h"


@pytest.fixture(scope="module")
def lib():
    from paper_1601_07195_b200 import _lib
    from paper_1601_07195_b200.build import build

    build()
    return _lib.load()


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|uint64_t|const char \*)\s*(sv_\w+)\s*\(", text, re.M)))


def test_header_declares_abi_and_binding_matches():
    from paper_1601_07195_b200 import _lib

    names = declared()
    assert len(names) >= 14
    assert sorted(_lib.EXPORTS) == names


def test_library_exports_every_declared_symbol(lib):
    from paper_1601_07195_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (sv_\w+)$", out, re.M))
    for name in declared():
        assert name in exported, name
        assert hasattr(lib, name)


def test_constants_match_header(lib):
    from paper_1601_07195_b200 import _lib

    text = HEADER.read_text()
    for name in ("SV_FUSED_MAX_TILE", "SV_FUSED_MAX_GATES", "SV_NORM_SCRATCH", "SV_TILE_GATHER"):
        assert int(re.search(rf"#define {name} (\d+)", text).group(1)) == getattr(_lib, name)
    assert lib.sv_version() == _lib.ABI_VERSION
    assert ctypes.sizeof(_lib.SvGate) == 72


def test_argument_validation_without_gpu(lib):
    from paper_1601_07195_b200 import _lib

    q = (ctypes.c_double * 8)(*[1, 0, 0, 0, 0, 0, 1, 0])
    fake = 1 << 20  # aligned, never dereferenced: validation fails first
    assert lib.sv_apply_single(None, 4, 0, q, None) == _lib.SV_EINVAL
    assert lib.sv_apply_single(fake + 8, 4, 0, q, None) == _lib.SV_EINVAL  # misaligned
    assert lib.sv_apply_single(fake, 4, 4, q, None) == _lib.SV_EINVAL
    assert b"not in [0, 4)" in lib.sv_last_error()
    assert lib.sv_apply_single(fake, 4, -1, q, None) == _lib.SV_EINVAL
    assert lib.sv_apply_controlled(fake, 4, 2, 2, q, None) == _lib.SV_EINVAL
    assert b"must differ" in lib.sv_last_error()
    assert lib.sv_apply_controlled(fake, 4, 0, 4, q, None) == _lib.SV_EINVAL
    g = (_lib.SvGate * 1)()
    g[0].target, g[0].control = 5, -1
    assert lib.sv_apply_fused(fake, 10, 5, g, 1, None) == _lib.SV_EINVAL  # target >= l
    assert lib.sv_apply_fused(fake, 10, 14, g, 1, None) == _lib.SV_EINVAL  # l > tile / m
    assert lib.sv_apply_fused(fake, 10, 6, g, 0, None) == _lib.SV_EINVAL
    assert lib.sv_apply_fused(fake, 10, 6, g, _lib.SV_FUSED_MAX_GATES + 1, None) == _lib.SV_EINVAL
    assert lib.sv_exchange(fake, fake, 8, 1, -1, q, None) == _lib.SV_EINVAL  # aliasing
    assert lib.sv_exchange(fake, fake + 4096, 8, 1, 8, q, None) == _lib.SV_EINVAL  # control not local
    assert lib.sv_norm_sq(fake, 8, 8, None, None) == _lib.SV_EINVAL
    assert lib.sv_init_basis(fake, 3, 8, None) == _lib.SV_EINVAL
    with pytest.raises(ValueError):
        _lib.check(lib.sv_apply_single(None, 4, 0, q, None))


def test_host_tensors_are_refused():
    """No CPU path: a host tensor raises instead of being computed on the CPU."""
    import torch

    import paper_1601_07195_b200 as sv

    with pytest.raises(TypeError):
        sv.apply_single_raw(torch.zeros(8, dtype=torch.complex128), 0, sv.hadamard())
    with pytest.raises(TypeError):
        sv.LocalState(sv.Layout(3), torch.zeros(8, dtype=torch.complex128))


def test_product_package_never_imports_the_oracle():
    pkg = ROOT / "paper_1601_07195_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")):
        src = f.read_text()
        assert "from oracle" not in src and "import oracle" not in src, f
        assert "sv_oracle" not in src and "libsv_oracle" not in src, f
