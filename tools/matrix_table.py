"""Render BASELINE.md section 5 (the results table) from the committed measurements.

    python tools/matrix_table.py > /tmp/table.md

Inputs (all under profiles/): the products M=1 bench line (r2_bench_products_M1.json), the
measurement matrix (r2_matrix.jsonl: `bench.py --config X [--loopback M] --mode Y`), the
ncu DRAM counters of one part's SpMM products (r2_matrix_ncu_*.csv) and the oracle epochs on
the GPU box's host cores (r2_oracle_full_epoch.jsonl, r2_oracle_configs.jsonl).
"""
import csv
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6554.2



def ncu_dram(name):
    """{width: (bytes, ns, l2hit)} of the first product of each width in a matrix ncu csv."""
    f = os.path.join(P, f"r2_matrix_ncu_{name}.csv")
    if not os.path.exists(f):
        return {}
    per = {}
    for row in csv.DictReader([ln for ln in open(f) if ln.startswith('"')]):
        d = per.setdefault(int(row["ID"]), {"k": row["Kernel Name"]})
        d[row["Metric Name"]] = float(row["Metric Value"].replace(",", ""))
    out = {}
    for i in sorted(per):
        d = per[i]
        key = d["k"].split("(")[0]
        if key in out:
            continue
        out[key] = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
                    d["gpu__time_duration.sum"], d["lts__t_sector_hit_rate.pct"])
    return out


def oracle_rows():
    rows = {}
    for fn in ("r2_oracle_full_epoch.jsonl", "r2_oracle_configs.jsonl"):
        f = os.path.join(P, fn)
        if not os.path.exists(f):
            continue
        for ln in open(f):
            d = json.loads(ln)
            if d.get("frac", 1.0) != 1.0:
                continue
            key = (d["config"], d.get("parts", 1))
            th = d.get("threads_requested")
            rows.setdefault(key, []).append(
                f"{d['epoch_s']:.3g} ({'1 thread' if th == 1 else '%.1f of %d cores' % (d['cores_effective'], d['cores_available'])})")
    return rows


def main():
    lines = []
    b = os.path.join(P, "r2_bench_products_M1.json")
    if os.path.exists(b):
        lines.append(json.load(open(b)))
    lines += [json.loads(x) for x in open(os.path.join(P, "r2_matrix.jsonl"))]
    orc = oracle_rows()
    ncu = {("products", 8): ncu_dram("products8"), ("reddit", 8): ncu_dram("reddit8"),
           ("reddit", 1): ncu_dram("reddit1")}
    print("| Config | M | mode | epoch time per GPU (s) | SpMM GTEPS (on the B200) | "
          "SpMM HBM GB/s (ncu, dominant product) | %% of %.0f | effective GB/s (edge-gather) | "
          "GEMM TFLOP/s (algorithmic) | oracle s/epoch (threads) | SM MHz |" % PEAK)
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for d in lines:
        c = d["config"]
        M = c["parts"]
        loop = c.get("loopback_parts_on_one_gpu")
        step = d["ms_per_step"] / 1e3
        per_gpu = step / M if loop else step
        eg = (d.get("roofline") or {}).get("effective", {}).get("achieved")
        gemm_ms = d["kernel_ms_per_step"]["gemm"]
        gflop = d.get("kernel_gflop_per_step", {}).get("gemm")
        roof = d.get("roofline") or {}
        hbm = pct = "—"
        if roof.get("traffic") and roof.get("avg_ms"):
            hbm = "%.0f (w=%s)" % (roof["traffic"] / (roof["avg_ms"] / 1e3) / 1e9,
                                   roof["kernel"].split()[3])
            pct = "%.0f%%" % (100 * roof["frac"])
        nc = ncu.get((c["workload"], M))
        if nc and (hbm == "—" or loop):
            k, (by, ns, hit) = max(nc.items(), key=lambda kv: kv[1][1])
            hbm = "%.0f (part 0, L2 hit %.0f%%)" % (by / ns, hit)
            pct = "%.0f%%" % (100 * by / ns / PEAK)
        gteps = d.get("spmm_gteps_rank0")
        o = orc.get((c["workload"], M)) or ([] if M != 1 else orc.get((c["workload"], 1), []))
        clk = d.get("clocks") or {}
        print(f"| {c['workload']} | {M}{' (loopback)' if loop else ''} | {c['mode']} | "
              f"{per_gpu:.4g}{' = step/%d' % M if loop else ''} | "
              f"{gteps:.1f} | {hbm} | {pct} | {eg:.0f} | "
              f"{'%.0f' % (gflop / gemm_ms) if gflop else '—'} | {'; '.join(o) if o else '—'} | "
              f"{clk.get('sm_mhz') or '—'} |")


if __name__ == "__main__":
    main()
