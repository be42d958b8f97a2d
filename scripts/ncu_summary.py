"""Summarise an ncu report: key SOL metrics, DRAM bytes, stall reasons by instruction.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--top 40]
"""

import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uma.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg",
    "smsp__cycles_active.avg", "lts__t_bytes.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    rows = ncu_csv(rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2:]
    res = []
    for v in vals:
        d = {}
        for h, u, x in zip(hdr, units, v):
            d[h] = (x, u)
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--all", action="store_true")
    a = ap.parse_args()
    for i, d in enumerate(raw_metrics(a.rep)):
        print(f"== launch {i}: {d.get('Kernel Name', ('?',))[0][:100]}")
        keys = list(d) if a.all else KEYS
        for k in keys:
            if k in d:
                print(f"   {k:75s} {d[k][0]:>18s} {d[k][1]}")
    rows = ncu_csv(a.rep, "--page", "source", "--print-source", "sass")
    hdr = rows[1]
    isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = collections.Counter()
    per = []
    for r in rows[2:]:
        try:
            ex, st = int(r[iex]), int(r[ist])
        except (ValueError, IndexError):
            continue
        reasons = {hdr[i]: int(r[i]) for i in stall_cols if r[i] not in ("", "0")}
        for k, v in reasons.items():
            tot[k] += v
        per.append((st, ex, r[isrc].strip(), reasons))
    total = sum(p[0] for p in per)
    print(f"== stall samples {total}; executed warp-instructions {sum(p[1] for p in per)}")
    for k, v in tot.most_common(12):
        print(f"   {k:28s} {v:7d} {100.0 * v / max(total, 1):5.1f}%")
    print(f"== top {a.top} instructions by samples")
    for st, ex, src, reasons in sorted(per, key=lambda p: -p[0])[:a.top]:
        rs = ",".join(f"{k[6:]}={v}" for k, v in sorted(reasons.items(), key=lambda x: -x[1])[:3])
        print(f"   {st:6d} {ex:9d}  {src[:60]:60s} {rs}")


if __name__ == "__main__":
    main()
