"""Summarise an ncu --set full report: per kernel duration, DRAM bytes, pipe utilisation, stall mix,
and the source lines with the most stall samples.  Usage: python tools/ncu_summary.py REPORT [top]"""
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.per_cycle_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def source(rep, idx):
    out = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--kernel-id", f"::regex:.*:{idx}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    lines = [(r[0], r[1], int(r[4])) for r in rows[3:] if len(r) > 4 and r[0] != "" and r[4].isdigit()]
    return lines


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    for i, d in enumerate(raw(rep)):
        print(f"== [{i + 1}] {d.get('Kernel Name', '')[:90]}")
        for k in KEYS:
            if k in d:
                print(f"   {k} = {d[k]}")
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(v) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v.isdigit()}
        tot = sum(st.values()) or 1
        print("   stalls: " + ", ".join(f"{k}={v / tot:.2f}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
        lines = source(rep, i + 1)
        tl = sum(v for _, _, v in lines) or 1
        for ln, src, v in sorted(lines, key=lambda x: -x[2])[:top]:
            print(f"   {100 * v / tl:5.1f}% L{ln:>5} {src.strip()[:100]}")


if __name__ == "__main__":
    main()
