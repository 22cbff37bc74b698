"""Summarise one gpu_profile.sh round (gpurun_out/<tag>/) into profiles/:
  * <tag>_ncu_summary.md  -- launch-list shares and, per `--set full` capture, time, DRAM bytes,
                             achieved GB/s or TFLOP/s, tensor-pipe / issue utilisation
  * ncu_traffic.json       -- dram read+write bytes per launch of the roofline kernels (bench.py reads it)
Usage: python tools/summarize_profiles.py r01h [profiles-prefix]"""
import collections
import csv
import json
import os
import sys

ROOT = __file__.rsplit("/tools/", 1)[0]
FP64_PEAK = 37.1
HBM_PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6462.7) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6462.7


def short(name):
    return name.split("(")[0].replace("void ", "").replace("lrc::", "").replace("<unnamed>::", "") \
        .replace("unnamed>::", "")


def read_csv_block(path):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    return list(csv.reader(lines[start:]))


def launch_shares(path):
    rows = read_csv_block(path)
    ix = {h: i for i, h in enumerate(rows[0])}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = short(r[ix["Kernel Name"]])
        tot[k] += float(r[ix["Metric Value"]].replace(",", ""))
        cnt[k] += 1
    T = sum(tot.values())
    return [(k, cnt[k], v / 1e6, v / T) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])]


def full_rows(path):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[0], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def g(d, k):
        try:
            return float(d[ix[k]].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")
    out = []
    for d in data:
        unit_t = rows[1][ix["gpu__time_duration.sum"]]
        t = g(d, "gpu__time_duration.sum")
        t_ms = t / 1e6 if unit_t == "ns" else (t / 1e3 if unit_t in ("us", "usecond") else t)
        rd, wr = g(d, "dram__bytes_read.sum"), g(d, "dram__bytes_write.sum")
        ur, uw = rows[1][ix["dram__bytes_read.sum"]], rows[1][ix["dram__bytes_write.sum"]]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(ur, 1)
        wr *= scale.get(uw, 1)
        out.append({"kernel": short(d[ix["Kernel Name"]]), "ms": t_ms, "dram_bytes": rd + wr,
                    "tensor_pct": g(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                    "issue_pct": g(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    "dram_pct": g(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                    "regs": g(d, "launch__registers_per_thread"), "grid": g(d, "launch__grid_size")})
    return out


def main():
    tag = sys.argv[1]
    prefix = sys.argv[2] if len(sys.argv) > 2 else tag
    src = os.path.join(ROOT, "gpurun_out", tag)
    md = [f"# ncu summary, round {tag}", "",
          "Captured by `tools/gpu_profile.sh` (ncu `--clock-control none`; cold-cache, serialised launches:",
          "compare shares and utilisations, not absolute times, with the bench's CUDA-event numbers).", ""]
    bench = os.path.join(src, "bench.json")
    if os.path.exists(bench):
        b = json.load(open(bench))
        md += ["## Bench line (no profiler)", "",
               f"* value {b['value']:.2f} it/s, e2e {b['e2e']['value']:.2f} it/s",
               f"* roofline ({b['roofline']['kernel']}): {b['roofline']['achieved']:.2f} "
               f"{b['roofline']['unit']} = {b['roofline']['frac']:.3f} of {b['roofline']['peak']}; "
               f"CUDA-event share {b['roofline']['share']:.3f}",
               f"* SpMM: {b['roofline_spmm']['avg_ms']:.3f} ms, {b['roofline_spmm']['achieved']:.0f} GB/s = "
               f"{b['roofline_spmm']['frac']:.3f} of HBM"]
        if b.get("config5_dense_spmm"):
            d = b["config5_dense_spmm"]
            md.append(f"* config 5 dense: {d['avg_ms']:.3f} ms, {d['tflops']:.2f} TFLOP/s, {d['achieved']:.0f} GB/s")
        if b.get("iteration_roofline"):
            it = b["iteration_roofline"]
            md.append(f"* iteration roofline {it['roofline_ms']:.2f} ms vs measured {it['measured_ms_per_iteration']:.2f} "
                      f"ms/iteration: frac {it['frac']:.3f}")
        md.append("")
    lpath = os.path.join(src, "launches.csv")
    if os.path.exists(lpath):
        md += ["## Launch list (`--metrics gpu__time_duration.sum`, bench command, one stream)", "",
               "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
        md += [f"| `{k}` | {c} | {t:.2f} | {s:.3f} |" for k, c, t, s in launch_shares(lpath)]
        md.append("")
    traffic = {}
    for cap in ("spmm_full", "ts_full", "dense_full"):
        p = os.path.join(src, cap + "_raw.csv")
        if not os.path.exists(p):
            continue
        md += [f"## `--set full`: {cap}", "",
               "| kernel | ms | DRAM bytes | GB/s | tensor pipe % | issue % | DRAM % | regs | grid |",
               "|---|---:|---:|---:|---:|---:|---:|---:|---:|"]
        for r in full_rows(p):
            md.append(f"| `{r['kernel']}` | {r['ms']:.3f} | {r['dram_bytes'] / 1e9:.3f} G | "
                      f"{r['dram_bytes'] / r['ms'] / 1e6:.0f} | {r['tensor_pct']:.1f} | {r['issue_pct']:.1f} | "
                      f"{r['dram_pct']:.1f} | {r['regs']:.0f} | {r['grid']:.0f} |")
            k = r["kernel"]
            if k.startswith(("spmm_u_kernel", "spmm_tma_kernel")):
                traffic["spmm"] = r["dram_bytes"]
            elif k.startswith("ts_kernel") and k.endswith("0>"):
                # captures run pass 1 (over Ucat) before pass 2 (over Y) within an iteration
                traffic["ts_gram2" if "ts_gram" in traffic else "ts_gram"] = r["dram_bytes"]
            elif k.startswith("ts_kernel") and k.endswith("1>"):
                traffic["ts_store"] = r["dram_bytes"]
            elif k.startswith("spmm_dense_kernel"):
                traffic["dense"] = r["dram_bytes"]
        md.append("")
    out = os.path.join(ROOT, "profiles", f"{prefix}_ncu_summary.md")
    open(out, "w").write("\n".join(md) + "\n")
    if traffic:
        json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print(out, traffic)


if __name__ == "__main__":
    main()
