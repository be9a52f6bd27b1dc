"""Time ONE full-size oracle epoch (no sampling) to validate bench.py's extrapolated
cpu_baseline (a 10% sample x 10).  CPU only; prints one JSON line.

    python tools/oracle_full_epoch.py [--config products] [--parts 1] [--frac 1.0]
                                      [--epochs 1] [--threads 0]

--threads T pins the BLAS/OpenMP pools to T threads (0 = leave them at the default, i.e.
all host cores); SURVEY 8.d.6 asks for Cora at 200 epochs single- and all-thread.
"""
import argparse
import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="products")
    ap.add_argument("--parts", type=int, default=1)
    ap.add_argument("--frac", type=float, default=1.0)
    ap.add_argument("--epochs", type=int, default=1)
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    if a.threads > 0:   # before numpy/scipy load their thread pools
        for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[k] = str(a.threads)
    import oracle
    from synth import get_config, make_inputs, make_block_parts
    from synth.configs import scaled
    cfg = get_config(a.config) if a.frac >= 1.0 else scaled(get_config(a.config), a.frac)
    t0 = time.perf_counter()
    inp = make_inputs(cfg)
    part = make_block_parts(cfg, a.parts)
    parts = [oracle.oracle_partition(inp.indptr, inp.indices, part, a.parts, m)
             for m in range(a.parts)]
    t_setup = time.perf_counter() - t0
    r0 = resource.getrusage(resource.RUSAGE_SELF)
    t0 = time.perf_counter()
    oracle.oracle_train(inp.indptr, inp.indices, inp.x, inp.y, inp.train_mask, inp.weights,
                        cfg.num_classes, part, a.parts, sync_interval=cfg.sync_interval, epochs=a.epochs,
                        parts=parts)
    wall = time.perf_counter() - t0
    r1 = resource.getrusage(resource.RUSAGE_SELF)
    cpu = (r1.ru_utime - r0.ru_utime) + (r1.ru_stime - r0.ru_stime)
    print(json.dumps({"config": a.config, "frac": a.frac, "parts": a.parts,
                      "num_nodes": cfg.num_nodes, "nnz": cfg.nnz, "epochs": a.epochs,
                      "epoch_s": wall / a.epochs, "threads_requested": a.threads or None,
                      "cores_effective": round(cpu / wall, 2),
                      "cores_available": len(os.sched_getaffinity(0)),
                      "max_rss_gb": r1.ru_maxrss / 1e6, "setup_s": t_setup}), flush=True)


if __name__ == "__main__":
    main()
