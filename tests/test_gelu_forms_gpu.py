"""The GELU / GELU' epilogues evaluate the same fit in a scalar form (ragged
edges) and an FP32x2 pair form (full chunks). Tiles land on either path
depending on shapes and layouts (e.g. the expert-parallel exchange path vs the
local path), so the two forms must agree bit-for-bit: checked over every bf16
GELU' operand and 2^27 hashed fp32 GELU operands (scripts/micro/gelu_pair_check.cu)."""
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gelu_scalar_and_pair_forms_bit_identical(cuda, tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path / "gelu_pair_check")
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           "-I" + os.path.join(ROOT, "paper_2110_03888_b200/csrc"), "-I" + os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "scripts/micro/gelu_pair_check.cu"), "-o", exe])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120).stdout
    assert "gelu' (all bf16): 0 mismatches" in out, out
    assert "gelu (2^27 fp32): 0 mismatches" in out, out
