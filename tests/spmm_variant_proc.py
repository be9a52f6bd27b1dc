"""Subprocess body of tests/test_gpu_spmm_variants.py: the SpMM variant is chosen by the
library's environment switches (read once per process), so each variant runs in a fresh
process.  Computes Y through digest_propagate (mode 0: P_m X_ext, the full row, Eq. 5's
P_in X + P_out X~ as one product; 1: P_in X_local; 2: P_out^T X_local) and writes Y and
the inputs to an npz."""
import sys

import numpy as np
import torch


def main(out, width, seed, mode=0, nodes=3000):
    torch.cuda.set_device(0)
    from paper_2206_00057_b200.engine import Partition
    from synth import small_config, make_graph, make_random_parts
    cfg = small_config(num_nodes=nodes, nnz=30 * nodes, d0=8, hidden=(8,), seed=seed)
    ip, ix = make_graph(cfg)
    part = make_random_parts(cfg.num_nodes, 3, seed)
    p = Partition(torch.as_tensor(ip).cuda(), torch.as_tensor(ix).cuda(),
                  torch.as_tensor(part).cuda(), 3, 1)
    from paper_2206_00057_b200 import capi as D
    g = torch.Generator().manual_seed(seed)
    xl = torch.rand(p.n_local, width, generator=g) * 2 - 1
    xh = torch.rand(p.n_halo, width, generator=g) * 2 - 1
    rows = p.n_halo if mode == 2 else p.n_local
    y = torch.empty(max(rows, 1), width, device="cuda")
    D.digest_propagate(p.handle, mode, xl.cuda(), xh.cuda(), width, width, y)
    torch.cuda.synchronize()
    np.savez(out, y=y.cpu().numpy(), xl=xl.numpy(), xh=xh.numpy(), ip=ip, ix=ix, part=part)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]),
         int(sys.argv[4]) if len(sys.argv) > 4 else 0, int(sys.argv[5]) if len(sys.argv) > 5 else 3000)
