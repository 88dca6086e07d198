"""The factorisation's trailing update staged by bulk copies (k_syrk_bulk, gbem_dmma_gemm.cuh) is
bit-identical to the cp.async kernel it replaced (k_syrk_gen) on ragged and odd shapes, repeatedly
(the stage-release race of the first version showed up as 8 x 32 blocks of differing entries in one
run out of three).  The checker is tools/bulk_check.cu, compiled on the box."""
import pathlib
import shutil
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]


@pytest.mark.gpu
def test_bulk_update_bit_identical_to_cp_async_update(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "bulk_check"
    subprocess.run([nvcc, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(exe),
                    str(ROOT / "tools" / "bulk_check.cu")], check=True, cwd=ROOT, timeout=600)
    out = subprocess.run([str(exe), "quick"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAILS 0" in out.stdout, out.stdout
