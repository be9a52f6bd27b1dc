"""Time digest_propagate (the SpMM) alone on a BASELINE-shaped partition.

    python tools/spmm_bench.py [--config products] [--parts 1] [--rank 0] [--width 256]
                               [--iters 5] [--mode 0]
Prints per-launch ms, GTEPS and edge-gather GB/s (the SURVEY §8.d.4 byte model).
Variants are selected through the library's experiment switches (DIGEST_KNOBS=1 plus
DIGEST_SPMM_SLAB, ...).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2206_00057_b200 import capi as D  # noqa: E402
from paper_2206_00057_b200.engine import Partition  # noqa: E402
from synth import get_config, make_graph, make_block_parts  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--parts", type=int, default=1)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--widths", default="256,100,48")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--mode", type=int, default=0)
    ap.add_argument("--scale", type=float, default=1.0,
                    help="nodes and edges of the config scaled by this factor (e.g. an "
                         "L2-resident footprint)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    cfg = get_config(a.config)
    if a.scale != 1.0:
        from synth.configs import scaled
        cfg = scaled(cfg, a.scale)
    ip, ix = make_graph(cfg)
    part_of = make_block_parts(cfg, a.parts)
    p = Partition(torch.as_tensor(ip).cuda(), torch.as_tensor(ix).cuda(),
                  torch.as_tensor(part_of).cuda(), a.parts, a.rank)
    info = p.info
    nnz = info.nnz if a.mode == 0 else (info.nnz_in if a.mode == 1 else info.rh_nnz)
    rows = info.n_local if a.mode != 2 else info.n_halo
    for w in [int(x) for x in a.widths.split(",")]:
        xl = torch.rand(info.n_local, w, device="cuda")
        xh = torch.rand(max(info.n_halo, 1), w, device="cuda")
        y = torch.empty(max(rows, 1), w, device="cuda")
        n0 = D.digest_launch_count()
        D.digest_propagate(p.handle, a.mode, xl, xh, w, w, y)
        torch.cuda.synchronize()
        lpp = D.digest_launch_count() - n0
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(max(a.iters, 0)):
            D.digest_propagate(p.handle, a.mode, xl, xh, w, w, y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / max(a.iters, 1)
        alg = nnz * (8 + 4 * w) + rows * (4 * w + 8)
        print(json.dumps({"config": a.config, "scale": a.scale, "parts": a.parts, "mode": a.mode, "width": w,
                          "ms": round(ms, 3), "gteps": round(nnz / ms / 1e6, 2),
                          "edge_gather_gbs": round(alg / ms / 1e6, 1),
                          "launches_per_product": lpp, "nnz": nnz, "rows": rows,
                          "src_rows": info.n_local + (info.n_halo if a.mode == 0 else 0),
                          "alg_bytes": alg,
                          "knobs": {k: v for k, v in os.environ.items()
                                    if k.startswith("DIGEST_")}}), flush=True)


if __name__ == "__main__":
    main()
