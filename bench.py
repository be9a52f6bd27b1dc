#!/usr/bin/env python
"""DIGEST epoch benchmark on B200 (one partition per GPU).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config products]
                    [--mode async|sync] [--impl ours|reference]

A step is one full DIGEST training epoch (Alg. 1) of the products-shaped
workload (BASELINE.json configs[4]) partitioned into M = N parts, one per GPU:
pull (every N_sync epochs), L layer forwards with the boundary push, loss,
backward, gradient allreduce and the optimizer step, all in libdigest.so.
Prints ONE JSON line on rank 0.

--impl reference times the CPU oracle (the base contract's reference arm for this
tier) on the host cores, on a bounded sample of the same workload.
"""
import argparse
import csv
import json
import os
import resource
import socket
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "epoch time (s) and SpMM GTEPS + HBM GB/s % of peak at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="products")
    ap.add_argument("--mode", default="async", choices=["async", "sync"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sample-frac", type=float, default=0.0,
                    help="oracle sample: fraction of nodes/edges of the workload (0 = auto: "
                         "0.1, shrunk so the --impl reference run of K+W oracle epochs stays "
                         "within a few minutes)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sync-interval", type=int, default=0,
                    help="override the config's N_sync (the Fig. 6 sweep, SURVEY f1)")
    ap.add_argument("--fresh", action="store_true",
                    help="zero-staleness exchange every level and epoch (SURVEY f1)")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N>1 exchange: library kernels over CUDA-IPC peer windows (default) "
                         "or NCCL send/recv + allreduce")
    ap.add_argument("--share-gpu", action="store_true",
                    help="testing only: every rank on cuda:0, gloo process group (timings are "
                         "time-sliced, not a scaling number)")
    ap.add_argument("--loopback", type=int, default=0,
                    help="N=1 only: train M partitions in one process on one GPU (linked stores, "
                         "the sync-interval / exchange-cost sweep); the step covers all M parts")
    ap.add_argument("--graph", action="store_true",
                    help="N=1, M=1: capture one epoch in a CUDA graph and replay it (Adam step "
                         "count on the device); kernel times then come from an eager pass")
    ap.add_argument("--store-bf16", action="store_true",
                    help="bf16 stale store and transfers (SURVEY f3 (ii)); off by default")
    ap.add_argument("--cache-l1", action="store_true",
                    help="aggregate the static layer-1 inputs once (SURVEY f3 (i)); off by default")
    ap.add_argument("--no-ncu", action="store_true",
                    help="skip the ncu DRAM-traffic probe of the dominant kernel")
    ap.add_argument("--no-parts-variant", action="store_true",
                    help="N=1: skip the variant that trains the config's paper partition count "
                         "(products: 8) on this GPU, the stale-halo exchange included")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p.get("bf16_tflops"), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------- clocks during the timed region
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.proc, self.lines = gpu, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- oracle (reference arm / cpu_baseline)
def oracle_sample_epoch_seconds(cfg_name, M, frac, steps, warmup):
    """Time oracle epochs on a products-shaped graph scaled to `frac` of the nodes and edges;
    returns per-step seconds extrapolated to the full workload (time / frac)."""
    from synth import get_config, make_inputs, make_block_parts
    from synth.configs import scaled
    import oracle
    cfg = scaled(get_config(cfg_name), frac)
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, M)
    parts = [oracle.oracle_partition(inp.indptr, inp.indices, part, M, m) for m in range(M)]
    times, cpu = [], 0.0
    for i in range(warmup + steps):
        r0 = resource.getrusage(resource.RUSAGE_SELF)
        t0 = time.perf_counter()
        oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                            cfg.num_classes, part, M, sync_interval=get_config(cfg_name).sync_interval,
                            epochs=1, parts=parts)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
            r1 = resource.getrusage(resource.RUSAGE_SELF)
            cpu += (r1.ru_utime - r0.ru_utime) + (r1.ru_stime - r0.ru_stime)
    sample = (f"{steps} oracle epoch(s) of a {cfg_name}-shaped graph scaled to {frac:g} of the "
              f"nodes/edges ({cfg.num_nodes} nodes, {cfg.nnz} nnz, dims {list(cfg.dims)}, M={M}); "
              f"time x {1 / frac:g}")
    # threads actually used: CPU seconds / wall seconds of the timed oracle epochs (SciPy's
    # sparse products run on one thread, the dense products on the BLAS pool)
    eff = cpu / max(sum(times), 1e-9)
    return [t / frac for t in times], sample, round(eff, 2)


def full_size_oracle(cfg_name):
    """The committed timing of ONE unsampled oracle epoch of this workload on a GPU box's
    host cores (tools/oracle_full_epoch.py), beside the sampled value: it shows how far the
    linear extrapolation of the sample is off (context, not re-measured in this run)."""
    p = os.path.join(ROOT, "profiles", "r2_oracle_full_epoch.jsonl")
    try:
        for ln in open(p):
            d = json.loads(ln)
            if d.get("config") == cfg_name and d.get("frac") == 1.0 and d.get("parts", 1) == 1:
                return {"epoch_s": d["epoch_s"], "cores_effective": d.get("cores_effective"),
                        "source": "profiles/r2_oracle_full_epoch.jsonl"}
    except Exception:   # noqa: BLE001
        pass
    return None


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def reference_frac(a):
    """Oracle sample size: 10% of the workload per epoch (~12-18 s on 8-16 host cores for
    products), scaled down so K + W epochs take about 8 such epochs in total."""
    if a.sample_frac > 0:
        return a.sample_frac
    return max(0.01, min(0.1, 0.1 * 8.0 / max(1, a.steps + a.warmup)))


def run_reference(a, rank, world):
    if rank != 0:
        return
    M = max(world, a.gpus)
    per, sample, eff = oracle_sample_epoch_seconds(a.config, M, reference_frac(a), a.steps,
                                                   a.warmup)
    v = float(np.mean(per))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": a.config, "parts": M},
            "cpu_baseline": {"value": v, "unit": "s", "cores": eff, "cores_available": cores(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def run_ours(a, rank, world, local):
    import torch
    import torch.distributed as dist
    if a.share_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if a.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    coll_dev = "cpu" if a.share_gpu else "cuda"
    from paper_2206_00057_b200 import capi as D
    from paper_2206_00057_b200.engine import TrainConfig, build_workers
    from synth import get_config, make_inputs, make_block_parts

    cfg = get_config(a.config)
    M = world
    loop = a.loopback > 1 and world == 1
    if loop:
        M = a.loopback
        a.no_e2e = True
    t0 = time.time()
    inp = make_inputs(cfg)
    part_of = make_block_parts(cfg, M)
    t_gen = time.time() - t0

    comm_grad = comm_halo = None
    if world > 1 and a.transport == "peer":
        # every rank must map every peer's window; if CUDA IPC is unavailable anywhere (e.g.
        # a container without IPC permissions) all ranks agree to use NCCL instead
        from paper_2206_00057_b200.dist import connect_peer_comm, grad_count
        err = None
        try:
            comm_grad = comm_halo = connect_peer_comm(world, rank, grad_count(cfg.dims))
        except Exception as ex:   # noqa: BLE001  (reported, then agreed on below)
            err = ex
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device=coll_dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            if rank == 0:
                print(f"warning: peer transport unavailable ({err}); using NCCL", file=sys.stderr)
            if comm_grad is not None:
                D.digest_comm_destroy(comm_grad)
            comm_grad = comm_halo = None
            a.transport = "nccl"
    if world > 1 and a.transport == "nccl":
        from paper_2206_00057_b200.dist import broadcast_ids
        ids = broadcast_ids(D.digest_comm_unique_id, 2, rank, device=coll_dev)
        comm_grad = D.digest_comm_init(ids[0], world, rank)
        comm_halo = D.digest_comm_init(ids[1], world, rank)
    try:
        uuid = str(torch.cuda.get_device_properties(torch.cuda.current_device()).uuid)
    except Exception:   # noqa: BLE001
        uuid = None
    rank_info = {"rank": rank, "device": torch.cuda.current_device(), "uuid": uuid,
                 "transport": a.transport if world > 1 else None,
                 "exchange_init": "ok" if world == 1 or comm_grad is not None else "failed"}
    print(f"bench rank {rank}/{world}: cuda:{rank_info['device']} {uuid} transport="
          f"{rank_info['transport']} init={rank_info['exchange_init']}", file=sys.stderr,
          flush=True)

    n_sync = a.sync_interval or cfg.sync_interval
    tc = TrainConfig(dims=cfg.dims, num_classes=cfg.num_classes, sync_interval=n_sync,
                     lr=0.01, optimizer="adam", async_push=(a.mode == "async"),
                     cache_l1=a.cache_l1, fresh=a.fresh, transport=a.transport,
                     store_bf16=a.store_bf16, device_step=a.graph)
    t1 = time.time()
    if loop:
        from paper_2206_00057_b200.engine import LoopbackGroup
        ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                           part_of, M, tc)
        grp = LoopbackGroup(ws)
        w = ws[0]
    else:
        (w,) = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                             part_of, M, tc, ranks=[rank], comm_grad=comm_grad, comm_halo=comm_halo)
        grp = w
    torch.cuda.synchronize()
    t_part = time.time() - t1
    info = w.part.info
    if world > 1:   # refuse to start if the per-peer boundary counts disagree (NCCL would hang)
        from paper_2206_00057_b200.dist import check_exchange_plan
        check_exchange_plan(info.send_count, info.recv_count, world, device=coll_dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    r = 0
    for _ in range(a.warmup):
        r += 1
        grp.epoch(r)
    barrier()

    # ---- optional CUDA graph of one epoch (M=1: every epoch launches the same kernels with
    # the same arguments once the Adam step count lives on the device)
    graph, graph_launches = None, 0
    if a.graph:
        if world > 1 or loop:
            raise SystemExit("--graph needs N=1 and one partition")

        def capture():
            nonlocal r
            r += 1                  # the captured epoch's host bookkeeping (versions) runs once
            g = torch.cuda.CUDAGraph()
            nl0 = D.digest_launch_count()
            with torch.cuda.graph(g):
                w.epoch(r)          # M=1: pull/push launch nothing
            return g, D.digest_launch_count() - nl0

        torch.cuda.synchronize()
        graph, graph_launches = capture()
        torch.cuda.synchronize()

    def step():
        if graph is not None:
            graph.replay()
        else:
            grp.epoch(r)

    # ---- timed region (device time, CUDA events on the launching stream)
    clk = ClockSampler(local)
    clk.start()
    D.digest_prof_enable(True)
    n0 = D.digest_launch_count()
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    e0, e1 = ev[0], ev[-1]
    e0.record(stream)
    sched = []
    for i in range(a.steps):
        r += 1
        sched.append((r - 1) % n_sync == 0)   # Alg. 1: the epochs that push
        step()
        ev[i + 1].record(stream)
    barrier()
    launches = D.digest_launch_count() - n0 + graph_launches * (a.steps if graph else 0)
    ms = e0.elapsed_time(e1)
    clocks = clk.stop()
    if graph is not None:   # graph replays record no per-kernel events: profile an eager pass
        D.digest_prof_read()
        for _ in range(a.steps):
            r += 1
            grp.epoch(r)
        torch.cuda.synchronize()
    prof = D.digest_prof_read()
    detail = D.digest_prof_detail()
    D.digest_prof_enable(False)
    ms_max = max_over_ranks(ms)
    step_s = ms_max / 1e3 / a.steps
    # push and non-push epochs reported separately (rank-local, this rank)
    per_ep = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.steps)]
    split = {}
    for name, want in (("push_epochs", True), ("other_epochs", False)):
        xs = [t for t, p in zip(per_ep, sched) if p == want]
        split[name] = {"n": len(xs), "mean_ms": float(np.mean(xs)) if xs else None}

    # ---- e2e: same epochs through the public API, every step's inputs copied from pinned
    # host memory inside the timed region.  Input pipeline as a data loader would run it:
    # step i+1's inputs are copied on a copy stream into the second of two device buffers
    # while step i computes (events order the buffer reuse); the loss is read back to the
    # host after every step.
    e2e = None
    if not a.no_e2e:
        keys = [k for k in ("x_local", "x_halo", "labels", "train_mask") if getattr(w, k) is not None]
        host = {k: getattr(w, k).cpu().pin_memory() for k in keys}
        dev = [{k: getattr(w, k) for k in keys}, {k: torch.empty_like(getattr(w, k)) for k in keys}]
        loss_h = torch.zeros(1, dtype=torch.float64).pin_memory()
        h2d = sum(t.numel() * t.element_size() for t in host.values())
        cs = torch.cuda.Stream()
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        consumed = [torch.cuda.Event(), torch.cuda.Event()]

        def load(i):
            b = i % 2
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(consumed[b])
                for k, t in host.items():
                    dev[b][k].copy_(t, non_blocking=True)
                copied[b].record(cs)

        graphs = []
        if graph is not None:   # one graph per input buffer, captured before the timed region
            for b in range(2):
                for k in keys:
                    setattr(w, k, dev[b][k])
                torch.cuda.synchronize()
                graphs.append(capture()[0])
            torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        cs.wait_event(f0)
        load(0)
        for i in range(a.steps):
            r += 1
            b = i % 2
            stream.wait_event(copied[b])
            for k in keys:
                setattr(w, k, dev[b][k])
            if i + 1 < a.steps:
                load(i + 1)
            if graphs:
                graphs[b].replay()
            else:
                w.epoch(r)
            consumed[b].record(stream)
            loss_h.copy_(w.loss, non_blocking=True)
        f1.record(stream)
        barrier()
        e2e_s = max_over_ranks(f0.elapsed_time(f1)) / 1e3 / a.steps
        e2e = {"value": e2e_s, "unit": "s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": 8, "input_pipeline": "double-buffered, copy stream"}

    # ---- variant (same run, same workers): the exact layer-1 aggregation cache (SURVEY f3
    # (i)).  Not the headline: it skips recomputing P_m X^(0) after the first epoch (valid
    # only while the features are static; the paper recomputes layer 1 every epoch).
    variants = {}
    if (not a.cache_l1 and not a.graph and graph is None
            and (cfg.dims[0] <= cfg.dims[1] or tc.order == D.ORDER_AGG_FIRST)):
        for x in getattr(grp, "workers", [w]):
            x.cfg.cache_l1, x._a1_ready = True, False
        r += 1
        grp.epoch(r)                       # aggregates A1 once
        barrier()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        v0.record(stream)
        for _ in range(a.steps):
            r += 1
            grp.epoch(r)
        v1.record(stream)
        barrier()
        variants["cache_l1"] = {"ms_per_step": max_over_ranks(v0.elapsed_time(v1)) / a.steps,
                                "note": "layer-1 aggregation A1 = P_m X^(0) computed once "
                                        "(static features), exact"}
        for x in getattr(grp, "workers", [w]):
            x.cfg.cache_l1, x._a1_ready = False, False

    # ---- roofline of the dominant kernel: the SpMM product (all its column-slab launches)
    # of the width with the largest time.  HBM roof on the DRAM bytes ncu counts for one
    # such product of this build (dram_probe, run below after the timed regions), the
    # edge-gather model beside it, and the L2->SM gather roof measured on
    # this B200 by tools/gather_roof.cu (profiles/r2_gather_roof.jsonl).
    hbm, bf16, src = peaks()
    dom = max((d for d in detail if d["cls"] == "spmm"), key=lambda d: d["ms"], default=None)
    roof = None
    probe = None
    if dom and dom["ms"] > 0 and rank == 0 and world == 1 and not loop and not a.no_ncu:
        probe = dram_probe(a.config, M, rank, int(dom["tag"]))
    if dom and dom["ms"] > 0:
        W_ = int(dom["tag"])
        rate_alg = dom["bytes"] / (dom["ms"] / 1e3)              # edge-gather B/s (all launches)
        n_rows, n_src, nnz_ = info.n_local, info.n_local + info.n_halo, info.nnz
        alg_prod = nnz_ * (8.0 + 4 * W_) + n_rows * (4.0 * W_ + 8)
        compulsory = 8.0 * nnz_ + 4.0 * W_ * n_src + 4.0 * W_ * n_rows
        n_prod = max(1, int(round(dom["bytes"] / alg_prod)))
        avg_s = dom["ms"] / 1e3 / n_prod
        roof = {"bound": "hbm", "unit": "GB/s", "peak": hbm, "peak_source": src,
                "kernel": f"SpMM product width {W_} ({dom['launches'] // n_prod} launch(es) each)",
                "products": n_prod, "avg_ms": avg_s * 1e3,
                "alg_bytes_per_launch": alg_prod, "compulsory_bytes": compulsory}
        if probe and probe.get("traffic"):
            t = probe["traffic"]
            roof.update({"achieved": t / avg_s / 1e9, "frac": t / avg_s / 1e9 / hbm,
                         "traffic": t, "traffic_over_compulsory": t / compulsory,
                         "achieved_basis": "ncu DRAM bytes (read+write) of one product in this "
                                           "run / live mean product time (CUDA events)",
                         "traffic_probe": probe})
        else:
            roof.update({"achieved": rate_alg / 1e9, "frac": rate_alg / 1e9 / hbm, "traffic": None,
                         "achieved_basis": "edge-gather model (DRAM traffic unavailable: "
                                           f"{(probe or {}).get('error', 'probe not run')})"})
        roof["effective"] = {"achieved": rate_alg / 1e9, "frac": rate_alg / 1e9 / hbm,
                             "model": "edge-gather bytes 8+4w per nonzero + 4w+8 per row "
                                      "(SURVEY 8.d.4), every gathered row counted"}
        l2 = gather_roof(W_)
        if l2:
            roof["l2_fabric"] = {"peak": l2["gbs"], "achieved": rate_alg / 1e9,
                                 "frac": rate_alg / 1e9 / l2["gbs"],
                                 "basis": f"L2-resident random row gathers, width {l2['width']} "
                                          f"({l2['variant']}), profiles/r2_gather_roof.jsonl"}
    spmm = prof["spmm"]
    nnz_per_s = None
    gteps = None
    if spmm["ms"] > 0:
        # nonzeros traversed = flops / (2 * width), summed per launch in the detail table
        nz = sum(d["flops"] / (2.0 * d["tag"]) for d in detail if d["cls"] == "spmm" and d["tag"])
        gteps = nz / (spmm["ms"] / 1e3) / 1e9
    # per-rank evidence for N > 1: devices, exchange init, halo size, exchange time
    ranks = [rank_info]
    exch = None
    if world > 1:
        ri = dict(rank_info, n_halo=info.n_halo,
                  pack_ms_per_step=prof["pack"]["ms"] / a.steps)
        ranks = [None] * world
        dist.all_gather_object(ranks, ri)
        exch = {"n_halo_max": max(r["n_halo"] for r in ranks),
                "push_pull_ms_per_step_max": max(r["pack_ms_per_step"] for r in ranks),
                "distinct_devices": len({r["uuid"] for r in ranks})}
    cpu = None
    if rank == 0 and world == 1 and not loop:   # the oracle baseline is timed at N=1 only
        per, sample, eff = oracle_sample_epoch_seconds(a.config, M, a.sample_frac or 0.1, 1, 1)
        cpu = {"value": float(np.mean(per)), "unit": "s", "cores": eff,
               "cores_available": cores(), "kind": "oracle", "sample": sample,
               "full_size_check": full_size_oracle(a.config)}
    # ---- variant: DIGEST's own mechanism at N=1.  With one partition per GPU, N=1 has no
    # halo and no exchange; here the config's paper partition count (products: 8) is
    # trained on this GPU in one process -- every part's stale-halo SpMM, the pushes into
    # the linked stores every N_sync epochs, the pulls and the 8-way gradient sum (Alg. 1).
    # The step covers all parts' work, so ms_per_step / parts is the per-GPU share an 8-GPU
    # run would have if the parts ran concurrently.
    vparts = VARIANT_PARTS.get(a.config, 0)
    if (world == 1 and not loop and not a.graph and not a.no_parts_variant and vparts > 1
            and not a.cache_l1):
        grp.close()
        w.part.close()
        del w, grp
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        variants[f"parts{vparts}_on_one_gpu"] = parts_variant(a, cfg, inp, tc, vparts)
        grp = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": step_s, "unit": "s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": a.config, "num_nodes": cfg.num_nodes, "nnz": cfg.nnz,
                       "parts": M, "dims": list(cfg.dims), "sync_interval": n_sync,
                       "fresh": a.fresh, "transport": a.transport if world > 1 else None,
                       "loopback_parts_on_one_gpu": M if loop else None,
                       "mode": a.mode, "cache_l1": a.cache_l1, "store_bf16": a.store_bf16,
                       "cuda_graph": a.graph,
                       "n_local": info.n_local, "n_halo": info.n_halo,
                       "nnz_local": info.nnz, "l2": "inputs larger than L2 (no flush needed)"},
            "roofline": roof,
            "variants": variants,
            "ranks": ranks,
            "exchange": exch,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "spmm_gteps_rank0": gteps,
            "epoch_ms_by_schedule_rank0": split,
            "kernel_ms_per_step": {k: v["ms"] / a.steps for k, v in prof.items()},
            # algorithmic flops (2 M N K per GEMM, 2 w per SpMM nonzero, counted once)
            "kernel_gflop_per_step": {k: v["flops"] / a.steps / 1e9 for k, v in prof.items()},
            # per (class, tag): spmm:<width>, gemm:1KKKKNNN forward-type, 2MMMMNNN weight grad,
            # 3KKKKNNN CTA-pair forward-type
            "kernel_detail_ms_per_step": {f"{d['cls']}:{d['tag']}": round(d["ms"] / a.steps, 3)
                                          for d in detail},
            "setup_s": {"generate": t_gen, "partition_and_setup": t_part},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()      # no rank unmaps a buffer a peer may still read
    if grp is not None:
        grp.close()
    if world > 1:
        D.digest_comm_destroy(comm_grad)
        if comm_halo != comm_grad:
            D.digest_comm_destroy(comm_halo)
        dist.destroy_process_group()


NCU = "/usr/local/cuda/bin/ncu"

# the partition count each BASELINE.json config is quoted on (its largest)
VARIANT_PARTS = {"products": 8, "reddit": 8, "arxiv": 8, "flickr": 4, "cora": 2}


def parts_variant(a, cfg, inp, tc, M):
    """All M partitions of the workload trained on this GPU in one process (linked stores):
    W warm-up epochs, then K epochs timed with CUDA events on the launching stream."""
    import torch
    from paper_2206_00057_b200 import capi as D
    from paper_2206_00057_b200.engine import build_workers, LoopbackGroup
    from synth import make_block_parts
    part_of = make_block_parts(cfg, M)
    ws = build_workers(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                       part_of, M, tc)
    grp = LoopbackGroup(ws)
    stream = torch.cuda.current_stream()
    n_sync = tc.sync_interval
    r = 0
    for _ in range(a.warmup):
        r += 1
        grp.epoch(r)
    torch.cuda.synchronize()
    D.digest_prof_read()
    D.digest_prof_enable(True)
    n0 = D.digest_launch_count()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    ev[0].record(stream)
    sched = []
    for i in range(a.steps):
        r += 1
        sched.append((r - 1) % n_sync == 0)
        grp.epoch(r)
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    launches = D.digest_launch_count() - n0
    prof = D.digest_prof_read()
    D.digest_prof_enable(False)
    ms = ev[0].elapsed_time(ev[-1]) / a.steps
    per_ep = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.steps)]
    split = {}
    for name, want in (("push_epochs", True), ("other_epochs", False)):
        xs = [t for t, p in zip(per_ep, sched) if p == want]
        split[name] = {"n": len(xs), "mean_ms": float(np.mean(xs)) if xs else None}
    infos = [x.part.info for x in ws]
    out = {"parts": M, "ms_per_step": ms, "ms_per_part": ms / M,
           "n_halo_total": int(sum(i.n_halo for i in infos)),
           "n_local_total": int(sum(i.n_local for i in infos)),
           "halo_over_local": float(sum(i.n_halo for i in infos) / sum(i.n_local for i in infos)),
           "nnz_total": int(sum(i.nnz for i in infos)),
           "epoch_ms_by_schedule": split,
           "kernel_ms_per_step": {k: v["ms"] / a.steps for k, v in prof.items()},
           "gpu_launches": int(launches),
           "note": "all M parts of the workload on this GPU in one process (linked stale "
                   "stores: pull/push of every part's halo rows every N_sync epochs, M-way "
                   "gradient sum); the step covers all M parts"}
    grp.close()
    for x in ws:
        x.part.close()
    del ws, grp
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def dram_probe(config, parts, rank, width, timeout=300):
    """DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of ONE SpMM product of
    width `width` on this build, this partition and this GPU: ncu profiles
    tools/spmm_bench.py (a warm-up product, then the counted one; every column-slab launch
    of the product summed).  Counters only -- no time from the profiled run is reported."""
    if not os.path.exists(NCU):
        return {"error": "ncu not found"}
    with tempfile.TemporaryDirectory() as td:
        log = os.path.join(td, "ncu.csv")
        cmd = [NCU, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum",
               "--kernel-name", "regex:k_spmm", "--print-units", "base", "--csv",
               "--log-file", log, sys.executable, os.path.join(ROOT, "tools", "spmm_bench.py"),
               "--config", config, "--parts", str(parts), "--rank", str(rank), "--widths",
               str(width), "--iters", "1"]
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        except Exception as ex:   # noqa: BLE001
            return {"error": f"ncu run failed: {ex}"}
        info = None
        for ln in r.stdout.splitlines():
            if ln.startswith("{"):
                info = json.loads(ln)
        if r.returncode != 0 or info is None or not os.path.exists(log):
            return {"error": f"ncu rc={r.returncode}: {r.stderr[-300:]}"}
        with open(log) as f:
            lines = [ln for ln in f if ln.startswith('"')]
        per, names = {}, {}
        for row in csv.DictReader(lines):
            try:
                i = int(row["ID"])
                per[i] = per.get(i, 0.0) + float(row["Metric Value"].replace(",", ""))
                names[i] = row["Kernel Name"]
            except (KeyError, ValueError):
                continue
        lpp = int(info["launches_per_product"])
        ids = sorted(per)[-lpp:]
        if len(ids) < lpp:
            return {"error": f"ncu captured {len(per)} launches, expected >= {lpp}"}
        return {"traffic": sum(per[i] for i in ids), "launches": lpp,
                "kernels": sorted({names[i].split("(")[0] for i in ids}),
                "alg_bytes": info["alg_bytes"], "how": "ncu --metrics dram__bytes_read.sum,"
                "dram__bytes_write.sum on tools/spmm_bench.py (same build, same partition)"}


def gather_roof(width):
    """Best L2-resident (footprint <= 48 MB) random row-gather rate of the nearest measured
    width from profiles/r2_gather_roof.jsonl (tools/gather_roof.cu on this pool's B200)."""
    p = os.path.join(ROOT, "profiles", "r2_gather_roof.jsonl")
    try:
        rows = [json.loads(x) for x in open(p) if x.startswith("{")]
    except Exception:
        return None
    rows = [r for r in rows if r.get("kind") == "gather" and r["footprint_mb"] <= 48]
    if not rows:
        return None
    w = min({r["width"] for r in rows}, key=lambda x: abs(x - width))
    return max((r for r in rows if r["width"] == w), key=lambda r: r["gbs"])


def free_port():
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    return port


def main():
    a = parse()
    rank, world, local = dist_env()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ and a.impl == "ours":
        # one process per GPU: start the N ranks ourselves (same launch as the driver's)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        print(f"bench: --gpus {a.gpus} without WORLD_SIZE: launching {a.gpus} ranks: "
              + " ".join(cmd[1:6]), file=sys.stderr, flush=True)
        os.execv(sys.executable, cmd)
    if a.gpus != world and world > 1:
        print(f"warning: --gpus {a.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if a.impl == "reference":
        run_reference(a, rank, world)
    else:
        run_ours(a, rank, world, local)


if __name__ == "__main__":
    main()
