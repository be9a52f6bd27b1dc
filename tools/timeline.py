"""Per-phase device timeline of DIGEST epochs (no nsys in this image): CUDA events are
recorded on the launching stream around every phase of every part -- pull, layer l
forward, push of level l, loss, layer l backward, halo-gradient return, AGG, update --
and written as a Chrome trace (chrome://tracing, Perfetto) plus a per-phase summary.

    python tools/timeline.py [--config products] [--parts 8] [--epochs 3] [--sync-interval 1]
                             [--out profiles/r2_timeline_products_loopback8.json]

The parts run in one process on one GPU (LoopbackGroup, linked stores): the trace
shows where an M-GPU epoch spends its time per part and what the exchange costs
("the cost of pull/push operations is hidden by the layer forward").
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--parts", type=int, default=8)
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--sync-interval", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    from paper_2206_00057_b200 import engine as E
    from synth import get_config, make_inputs, make_block_parts
    cfg = get_config(a.config)
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, a.parts)
    tc = E.TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=a.sync_interval,
                       lr=0.01, optimizer="adam")
    ws = E.build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                         part, a.parts, tc)
    grp = E.LoopbackGroup(ws)
    marks = []   # (label, part, start event, end event)
    part_of = {id(w): m for m, w in enumerate(ws)}

    def wrap(cls, name, label):
        orig = getattr(cls, name)

        def f(self, *args, **kw):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = orig(self, *args, **kw)
            e1.record()
            lab = label(args) if callable(label) else label
            marks.append((lab, part_of.get(id(self), -1), e0, e1))
            return out
        setattr(cls, name, f)

    W = E.DigestWorker
    wrap(W, "pull", "pull")
    wrap(W, "forward_layer", lambda args: f"fwd L{args[0]}")
    wrap(W, "push", lambda args: f"push l{args[0]}")
    wrap(W, "compute_loss", "loss")
    wrap(W, "backward_layer", lambda args: f"bwd L{args[0]}")
    wrap(W, "return_halo_grad", lambda args: f"return l{args[0] - 1}")
    wrap(W, "update", "update")
    # AGG of the loopback group: one call for all parts
    from paper_2206_00057_b200 import capi as D
    orig_ar = D.digest_grad_allreduce_local

    def ar(*args, **kw):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        orig_ar(*args, **kw)
        e1.record()
        marks.append(("AGG", -1, e0, e1))
    E.D.digest_grad_allreduce_local = ar

    grp.epoch(1)                                  # warm-up, not traced
    torch.cuda.synchronize()
    marks.clear()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for r in range(2, 2 + a.epochs):
        grp.epoch(r)
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record()
    torch.cuda.synchronize()
    total = t0.elapsed_time(t1)
    events, summary = [], {}
    for lab, m, e0, e1 in marks:
        ts, dur = t0.elapsed_time(e0), e0.elapsed_time(e1)
        events.append({"name": lab, "ph": "X", "ts": ts * 1e3, "dur": dur * 1e3, "pid": 0,
                       "tid": f"part {m}" if m >= 0 else "group"})
        key = lab.split()[0] if lab.startswith(("push", "return")) else lab
        summary[key] = summary.get(key, 0.0) + dur
    out = a.out or os.path.join(ROOT, "profiles",
                                f"r2_timeline_{a.config}_loopback{a.parts}.json")
    res = {"config": a.config, "parts": a.parts, "epochs": a.epochs,
           "sync_interval": a.sync_interval, "ms_per_epoch": total / a.epochs,
           "phase_ms_per_epoch": {k: round(v / a.epochs, 4) for k, v in
                                  sorted(summary.items(), key=lambda kv: -kv[1])},
           "exchange_share": (summary.get("push", 0) + summary.get("pull", 0)) / max(total, 1e-9)}
    with open(out, "w") as f:
        json.dump({"traceEvents": events, "otherData": res}, f)
    print(json.dumps(res), flush=True)
    grp.close()


if __name__ == "__main__":
    main()
