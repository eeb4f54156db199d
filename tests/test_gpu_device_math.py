"""Device helpers of the hot path checked on the B200 against the CUDA library: daba::log1p_pos (the Cauchy loss's
log1p for q >= 0, device_math.cuh) within 4 ulp of the library log1p over q in [1e-300, 1e300]
(tools/log1p_check.cu: 2^24 log-uniform samples per band, including the branch point sqrt(2) - 1)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_log1p_pos_within_4_ulp(tmp_path):
    exe = str(tmp_path / "log1p_check")
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-I", os.path.join(ROOT, "include"),
                           "-o", exe, os.path.join(ROOT, "tools", "log1p_check.cu")])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "max ulp over all bands" in out.stdout and "no error" in out.stdout, out.stdout
