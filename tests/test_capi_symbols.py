"""The C-ABI libraries load on a CPU-only host and export every entry point
their headers declare (no compute calls here)."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2203_11733_b200" / "lib"


def declared(header: Path):
    text = re.sub(r"/\*.*?\*/", "", header.read_text(), flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(gbem_\w+)\s*\(", text, flags=re.M)))


@pytest.mark.parametrize("header,lib", [("gbem_gpu.h", "libgbem_gpu.so"), ("gbem_host.h", "libgbem_host.so")])
def test_library_exports_every_declared_symbol(header, lib):
    names = declared(ROOT / "include" / header)
    assert len(names) >= 10
    so = C.CDLL(str(LIB / lib))
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_python_bindings_cover_the_header():
    from paper_2203_11733_b200 import _native, api
    gpu = {n for n, _, _ in _native.GPU_SYMBOLS}
    assert set(declared(ROOT / "include" / "gbem_gpu.h")) == gpu
    assert set(declared(ROOT / "include" / "gbem_host.h")) == set(api.HOST_SYMBOLS)


def test_context_creation_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2203_11733_b200._native import Context, GbemError
    with pytest.raises(GbemError) as e:
        Context(0)
    assert e.value.code == 3
