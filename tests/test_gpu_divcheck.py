"""The branch-free correctly rounded reciprocal, quotient and square root of the replay and sweep kernels
(agft_internal.cuh xrcp_nb / xdiv_nb / xsqrt_nb) against the IEEE operations, bit for bit, on random
operands over the ranges the kernels use (tools/div_check.cu: ~2.4e9 comparisons).  The parity suite
checks the same property end to end (every sum bit-exact against the oracle)."""
import json
import os
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_branch_free_division_and_sqrt_bit_exact(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    if not (os.path.exists(nvcc) or shutil.which("nvcc")):
        pytest.skip("nvcc not available")
    exe = str(tmp_path / "div_check")
    subprocess.check_call([nvcc if os.path.exists(nvcc) else "nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-o", exe, os.path.join(ROOT, "tools", "div_check.cu")])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["err"] == "no error", res
    assert res["compared"] > 1e9
    assert res["mismatches"] == 0, res
