"""Turn the gpurun ncu outputs into tracked summaries under profiles/ (round tag as argv[1]).

  profiles/<tag>_traffic.csv        per (M,N,K): duration, DRAM read/write, algorithmic bytes
  profiles/ncu_traffic.json         per-launch DRAM bytes keyed "MxNxK" (read by bench.py)
  profiles/<tag>_launches.md        launch list of the bench command: per kernel count / avg / share
  profiles/<tag>_ncu_full_*.txt     ncu --set full summary of the dominant kernel
"""

import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def read_ncu_csv(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr = r
            return hdr, rows[i + 1:]
    raise ValueError(path)


def alg_bytes(M, N, K, g=128):
    return K * N // 2 + 4 * (K // g) * N + 2 * M * K + 2 * M * N


def traffic(tag):
    hdr, rows = read_ncu_csv(os.path.join(OUT, f"traffic_{tag}.csv"))
    order = json.load(open(os.path.join(OUT, "traffic_order.json")))
    iid, iname, imet, ival = (hdr.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    per = collections.OrderedDict()
    for r in rows:
        if "w4a16" not in r[iname]:
            continue
        per.setdefault(r[iid], {})[r[imet]] = float(r[ival])
    launches = list(per.values())
    assert len(launches) == len(order), (len(launches), len(order))
    res, lines = {}, ["M,N,K,duration_us,dram_read_MB,dram_write_MB,traffic_MB,algorithmic_MB,traffic/algorithmic,GBps_alg"]
    for key, m in zip(order, launches):
        M, N, K = (int(x) for x in key.split("x"))
        tr = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        ab = alg_bytes(M, N, K)
        dur = m["gpu__time_duration.sum"] * 1e-9 if m["gpu__time_duration.sum"] > 1e3 else m["gpu__time_duration.sum"] * 1e-6
        res[key] = tr
        lines.append(f"{M},{N},{K},{dur*1e6:.2f},{m['dram__bytes_read.sum']/1e6:.3f},{m['dram__bytes_write.sum']/1e6:.3f},"
                     f"{tr/1e6:.3f},{ab/1e6:.3f},{tr/ab:.4f},{ab/dur/1e9:.1f}")
    open(os.path.join(PROF, f"{tag}_traffic.csv"), "w").write("\n".join(lines) + "\n")
    json.dump(res, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)


def launches(tag):
    hdr, rows = read_ncu_csv(os.path.join(OUT, f"launches_{tag}.csv"))
    iname, ival, iunit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows:
        nm = r[iname].split("(")[0]
        v = float(r[ival]) * (1e-3 if r[iunit] == "ns" else 1.0)
        agg.setdefault(nm, []).append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list ({tag}): `ncu --metrics gpu__time_duration.sum --clock-control none -k regex:w4a16 "
             f"python bench.py --steps 2 --warmup 3` (cold-cache, serialised: compare shares, not absolutes)", "",
             "| kernel | launches | avg us | total us | share |", "|---|---|---|---|---|"]
    for nm, v in agg.items():
        lines.append(f"| `{nm}` | {len(v)} | {sum(v)/len(v):.2f} | {sum(v):.1f} | {100*sum(v)/tot:.1f}% |")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")
    os.replace(os.path.join(OUT, f"launches_{tag}.csv"), os.path.join(PROF, f"{tag}_launches.csv"))


def full(tag, rep, name):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep, "--top", "40"],
                         capture_output=True, text=True).stdout
    open(os.path.join(PROF, f"{tag}_ncu_full_{name}.txt"), "w").write(out)


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    if os.path.exists(os.path.join(OUT, f"traffic_{tag}.csv")):
        traffic(tag)
    if os.path.exists(os.path.join(OUT, f"launches_{tag}.csv")):
        launches(tag)
    for f in sys.argv[2:]:
        full(tag, os.path.join(OUT, f), os.path.splitext(os.path.basename(f))[0])
