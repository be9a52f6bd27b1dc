"""Time the dense kernels alone on bench-sized shapes (CUDA events).

    python tools/gemm_bench.py [--rows 2449029] [--iters 5]

* forward GEMM  Z = A W        (digest_gemm, 3xTF32 tcgen05)      for (K, N) in SHAPES
* weight grad   G_W = A^T D    (digest_layer_bwd on an edgeless partition, P = I, so the
                                only heavy work is the bf16x6 split-K kernel)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2206_00057_b200 import capi as D  # noqa: E402
from paper_2206_00057_b200.engine import Partition  # noqa: E402

SHAPES = [(100, 256), (256, 256), (256, 48)]


def timeit(fn, iters):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=2449029)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--shapes", default="", help="e.g. 256x48,100x256 (K x N); default all")
    a = ap.parse_args()
    shapes = [tuple(int(v) for v in s.split("x")) for s in a.shapes.split(",")] if a.shapes else SHAPES
    torch.cuda.set_device(0)
    n = a.rows
    ip = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    ix = torch.zeros(0, dtype=torch.int32, device="cuda")
    po = torch.zeros(n, dtype=torch.int32, device="cuda")
    p = Partition(ip, ix, po, 1, 0)
    for K, N in shapes:
        A = torch.rand(n, K, device="cuda") - 0.5
        W = torch.rand(K, N, device="cuda") - 0.5
        Z = torch.empty(n, N, device="cuda")
        ms = timeit(lambda: D.digest_gemm(A, W, Z), a.iters)
        fl = 2.0 * n * K * N
        print(json.dumps({"kernel": "gemm_fwd", "K": K, "N": N, "ms": round(ms, 3),
                          "tflops_alg": round(fl / ms / 1e9, 1)}), flush=True)
        sv, sc = D.digest_layer_workspace(p.handle, K, N, D.ORDER_AGG_FIRST)
        saved = torch.empty(max(sv, 256), dtype=torch.uint8, device="cuda")
        scratch = torch.empty(max(sc, 256), dtype=torch.uint8, device="cuda")
        G = torch.rand(n, N, device="cuda") - 0.5
        GW = torch.empty(K, N, device="cuda")
        D.digest_layer_fwd(p.handle, A, None, 0, W, K, N, 0, D.ORDER_AGG_FIRST, Z, saved, scratch)
        ms = timeit(lambda: D.digest_layer_bwd(p.handle, A, None, 0, W, K, N, 0, D.ORDER_AGG_FIRST,
                                               saved, None, G, GW, None, scratch), a.iters)
        print(json.dumps({"kernel": "wgrad", "K": K, "N": N, "ms": round(ms, 3),
                          "tflops_alg": round(fl / ms / 1e9, 1)}), flush=True)
        # input gradient with the ReLU mask fused in the epilogue: G_in = (G W^T) * [H > 0]
        # (transform-first order: there the mask is applied in the GEMM epilogue)
        GI = torch.empty(n, K, device="cuda")
        Hm = torch.rand(n, K, device="cuda") - 0.5
        del saved, scratch
        sv, sc = D.digest_layer_workspace(p.handle, K, N, D.ORDER_XFORM_FIRST)
        saved = torch.empty(max(sv, 256), dtype=torch.uint8, device="cuda")
        scratch = torch.empty(max(sc, 256), dtype=torch.uint8, device="cuda")
        D.digest_layer_fwd(p.handle, A, None, 0, W, K, N, 0, D.ORDER_XFORM_FIRST, Z, saved, scratch)
        ldw = -(-((K + 31) // 32) // 4) * 4
        Hb = torch.randint(-2 ** 31, 2 ** 31 - 1, (n, ldw), dtype=torch.int32, device="cuda")
        for kind, gm in (("float", Hm), ("bits", (Hb.data_ptr(), ldw))):
            bwd = lambda: D.digest_layer_bwd(p.handle, A, None, 0, W, K, N, 0,  # noqa
                                             D.ORDER_XFORM_FIRST, saved, None, G, GW, GI,
                                             scratch, gin_mask=gm)
            bwd()
            torch.cuda.synchronize()
            D.digest_prof_enable(True)
            for _ in range(a.iters):
                bwd()
            torch.cuda.synchronize()
            det = D.digest_prof_read_detail()
            D.digest_prof_enable(False)
            for d in det:
                if d["cls"] == "gemm" and d["launches"]:
                    print(json.dumps({"kernel": "bwd_detail", "mask": kind, "K": K, "N": N,
                                      "tag": d["tag"], "ms": round(d["ms"] / a.iters, 3)}),
                          flush=True)
        del A, W, Z, G, saved, scratch, GI, Hm, Hb


if __name__ == "__main__":
    main()
