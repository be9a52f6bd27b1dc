"""Every SpMM kernel variant the library can select (environment switches, one fresh
process each) vs the oracle's fp64 P_m X_ext (Eq. 5) on a graph with rows of
0..~200 nonzeros (several 32-pair chunks and ragged tails), a random 3-way partition
(halo columns through the second source pointer) and widths that exercise every lane
layout.  Bar: 1e-4 relative (north_star)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
from oracle.gcn import layer_forward

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# round-1 kernels for narrow widths (DIGEST_SPMM_N=0 turns the lean kernel off)
CASES = [(48, {"DIGEST_SPMM_V12": str(v), "DIGEST_SPMM_N": "0"}) for v in range(8)]
CASES += [(48, {"DIGEST_SPMM_PFH": "1", "DIGEST_SPMM_N": "0"}),
          (48, {"DIGEST_SPMM_GRID": "1", "DIGEST_SPMM_N": "0"})]
# the lean narrow kernel: every variant, ragged widths, all three products
CASES += [(w, {"DIGEST_SPMM_N": str(n), "MODE": m}) for w in (48, 64, 100, 128) for n in (1, 2, 3, 4, 5, 6, 7, 8, 9)
          for m in ("0", "1", "2")]
CASES += [(w, {"DIGEST_SPMM_N": n, "MODE": m}) for n in ("1", "5") for w in (20, 32, 36, 52, 48, 100)
          for m in ("0", "1", "2")]
# w=196..256: the grouped kernel (default, 2 rows per warp) and the row-per-warp kernel (V=7),
# all three products; w=200: the ragged last float4 of a lane (RAG)
CASES += [(w, {"DIGEST_SPMM_V": v, "MODE": m}) for v in ("0", "7") for w in (256, 200)
          for m in ("0", "1", "2")]
CASES += [(256, {"DIGEST_SPMM_V": "17", "DIGEST_HOT_ROWS": "600", "MODE": m}) for m in ("0", "1", "2")]
# several 4096-row windows of the partition's length-grouped row order (grouped kernel)
CASES += [(w, {"DIGEST_SPMM_N": n, "MODE": m, "NODES": "40000"}) for n in ("1", "5")
          for w in (48, 100) for m in ("0", "1", "2")]
CASES += [(256, {"MODE": m, "NODES": "40000"}) for m in ("0", "1", "2")]
# the grouped kernel with per-lane (col, val) loads (N=11; the default loads them cooperatively)
CASES += [(w, {"DIGEST_SPMM_N": n, "MODE": m}) for n in ("11", "13") for w in (48, 100)
          for m in ("0", "1", "2")]
CASES += [(w, {"DIGEST_SPMM_N": "13", "MODE": m, "NODES": "40000"}) for w in (48, 100)
          for m in ("0", "1", "2")]
CASES += [(256, {"DIGEST_SPMM_V": "18", "MODE": m}) for m in ("0", "1", "2")]
# column slabs of the lean kernel (balanced, <= SMAX floats)
CASES += [(w, {"DIGEST_SPMM_SMAX": sm, "MODE": m}) for w, sm in ((100, "64"), (100, "48"),
                                                                  (256, "64"), (256, "32"),
                                                                  (128, "64"), (1024, "64"))
          for m in ("0", "1", "2")]
CASES += [(100, {"DIGEST_SPMM_V25": str(v)}) for v in range(6)]
CASES += [(256, {"DIGEST_SPMM_V": str(v)}) for v in range(7)]
CASES += [(256, {"DIGEST_SPMM_SLAB": "64"}), (256, {"DIGEST_SPMM_HINTS": "0"}),
          (256, {"DIGEST_SPMM_GRID": "0"}), (100, {"DIGEST_SPMM_SLAB": "32"})]
CASES += [(w, {}) for w in (4, 8, 16, 32, 64, 128, 384, 512, 1024)]
CASES += [(128, {"DIGEST_SPMM_V32": "1"})]
# TMA row-gather kernel (single-source products): P_in (mode 1) and P_out^T (mode 2)
CASES += [(w, {"DIGEST_SPMM_TMA": "1", "DIGEST_SPMM_N": "0", "MODE": m})
          for w in (4, 16, 48, 100, 128, 256) for m in ("1", "2")]
CASES += [(w, {"DIGEST_SPMM_MB": mb, "DIGEST_SPMM_N": "0"}) for w in (48, 100, 256)
          for mb in ("1", "4")]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("width,env", CASES, ids=[f"w{w}-" + "-".join(f"{k[-4:]}{v}" for k, v in e.items())
                                                  for w, e in CASES])
def test_spmm_variant(width, env, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = str(tmp_path / "y.npz")
    env = dict(env)
    mode = int(env.pop("MODE", "0"))
    nodes = env.pop("NODES", "3000")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "spmm_variant_proc.py"), out,
                        str(width), "5", str(mode), nodes], env={**os.environ, **env, "DIGEST_KNOBS": "1", "PYTHONPATH": ROOT},
                       capture_output=True, text=True, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    d = np.load(out)
    op = oracle.oracle_partition(d["ip"], d["ix"], d["part"], 3, 1)
    if mode == 0:
        ref = layer_forward(op, d["xl"], d["xh"], np.eye(width), relu=False)["A"]
    else:
        from oracle.gcn import prop_matrix
        P = prop_matrix(op)
        P_in, P_out = P[:, :op.n_local], P[:, op.n_local:]
        ref = (P_in @ d["xl"]) if mode == 1 else (P_out.T @ d["xl"])
    err = np.abs(d["y"] - ref).max() / np.abs(ref).max()
    assert err <= 1e-4, err
