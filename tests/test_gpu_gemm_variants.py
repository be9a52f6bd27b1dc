"""GEMM variants selected by the library's experiment switches (one fresh process each:
switches are read once per process) vs fp64 numpy: C = A B (Eq. 5's dense transform,
P:161), both tensor-core kernels (single CTA and CTA pair) and ragged shapes.  Bar: the
3xTF32 path's 3e-5 relative (test_gpu_parity.test_gemm_parity)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROC = r"""
import sys, numpy as np, torch
from paper_2206_00057_b200 import capi as D
M, N, K, bt, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
torch.cuda.set_device(0)
g = torch.Generator().manual_seed(M + 7 * N + 13 * K)
A = torch.rand(M, K, generator=g) * 2 - 1
B = (torch.rand(N, K, generator=g) if bt else torch.rand(K, N, generator=g)) * 2 - 1
C = torch.empty(M, N, device="cuda")
D.digest_gemm(A.cuda(), B.cuda(), C, bt=bool(bt))
torch.cuda.synchronize()
np.savez(out, A=A.numpy(), B=B.numpy(), C=C.cpu().numpy())
"""

SHAPES = [(3000, 256, 100, 0), (3000, 256, 256, 0), (3000, 48, 256, 0), (3000, 256, 48, 0),
          (200, 256, 100, 0), (777, 36, 52, 0), (1000, 256, 48, 1)]
CASES = [(s, {"DIGEST_GEMM_RAWHI": v}) for s in SHAPES for v in ("0", "1")]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("shape,env", CASES, ids=[f"{m}x{n}x{k}{'bt' if b else ''}-" +
                                                  "-".join(f"{k_[-5:]}{v}" for k_, v in e.items())
                                                  for (m, n, k, b), e in CASES])
def test_gemm_variant(shape, env, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    M, N, K, bt = shape
    out = str(tmp_path / "c.npz")
    r = subprocess.run([sys.executable, "-c", PROC, str(M), str(N), str(K), str(bt), out],
                       env={**os.environ, **env, "DIGEST_KNOBS": "1", "PYTHONPATH": ROOT},
                       capture_output=True, text=True, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    d = np.load(out)
    Bm = d["B"].astype(np.float64)
    ref = d["A"].astype(np.float64) @ (Bm.T if bt else Bm)
    err = np.abs(d["C"] - ref).max() / np.abs(ref).max()
    assert err <= 3e-5, err


def _run(shape, env, path):
    M, N, K, bt = shape
    r = subprocess.run([sys.executable, "-c", PROC, str(M), str(N), str(K), str(bt), path],
                       env={**os.environ, **env, "DIGEST_KNOBS": "1", "PYTHONPATH": ROOT},
                       capture_output=True, text=True, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)["C"]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("shape", SHAPES, ids=[f"{m}x{n}x{k}{'bt' if b else ''}" for m, n, k, b in SHAPES])
def test_gemm_raw_hi_is_bit_identical(shape, tmp_path):
    """The default feeds the raw fp32 A tile as A_hi (kind::tf32 reads the upper 19 bits);
    it must equal the explicit truncation split bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c_raw = _run(shape, {"DIGEST_GEMM_RAWHI": "1"}, str(tmp_path / "a.npz"))
    c_split = _run(shape, {"DIGEST_GEMM_RAWHI": "0"}, str(tmp_path / "b.npz"))
    assert np.array_equal(c_raw.view(np.uint32), c_split.view(np.uint32))
