"""Summarise the parity ratios a `pytest -m gpu` run logs (gpurun_out/parity_ratios.jsonl, one line
per checked GEMM: tag, relFro, max_ratio, max_ratio_strict; reading R12) into a Markdown table by
tag family (the first tag field).   python scripts/parity_summary.py LOG "header line" > OUT.md"""
import ast
import collections
import json
import math
import sys

log, header = sys.argv[1], sys.argv[2]
rows = collections.defaultdict(list)
for line in open(log):
    rec = json.loads(line)
    try:
        tag = ast.literal_eval(rec["tag"])
        fam = str(tag[0]) if isinstance(tag, tuple) and tag else str(tag)
    except (ValueError, SyntaxError):
        fam = rec["tag"] or "(untagged)"
    rows[fam].append(rec)


def mx(vals):
    vals = [v for v in vals if v is not None and not (isinstance(v, float) and math.isnan(v))]
    return max(vals) if vals else float("nan")


n = sum(len(v) for v in rows.values())
print(header + "\n")
print("Reading R12 (DESIGN.md §4, `oracle/compare.py`): `max_ratio` = max |err| / (B + ½ ulp_out), "
      "`max_ratio_strict` = max |err| / B. Pass = relFro ≤ 5e-3 and max_ratio ≤ 1. "
      f"Source: `gpurun_out/parity_ratios.jsonl` of that run ({n} logged checks).\n")
print("| family (first tag field) | checks | max relFro | max max_ratio | max max_ratio_strict |")
print("|---|---|---|---|---|")
for fam, recs in sorted(rows.items(), key=lambda kv: -len(kv[1])):
    print(f"| {fam} | {len(recs)} | {mx([r['relfro'] for r in recs]):.2e} | {mx([r['max_ratio'] for r in recs]):.3f} | "
          f"{mx([r['max_ratio_strict'] for r in recs]):.3f} |")
