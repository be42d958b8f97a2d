"""g=128 vs g=64 on cluster-mode decode shapes, graph-timed, after a warm-up and then again
after a burst of prefill GEMMs (power state)."""
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from graph_perf import time_graph  # noqa: E402
from paper_2508_15601_b200 import api, synth  # noqa: E402


def clk():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                          capture_output=True, text=True).stdout.strip()


def run(tag):
    for N, K in ((4096, 14336), (14336, 4096), (6144, 4096)):
        row = []
        for g in (128, 64):
            sets = []
            for i in range(4):
                d = synth.awq_like_torch(1, N, K, group=g, seed=200 + i)
                sets.append((api.pack_w4(d["q"], d["s"], d["z"], g), d["s"], d["z"]))
            A = torch.randn(16, K, device="cuda").to(torch.bfloat16)
            C = torch.empty(16, N, device="cuda", dtype=torch.bfloat16)
            calls = [(lambda p=p, s=s, z=z: api.gemm_w4a16(A, p, s, z, out=C)) for (p, s, z) in sets] * 6
            row.append(f"g{g}:{time_graph(calls) / len(calls):.1f}")
        print(tag, N, K, " ".join(row), clk(), flush=True)


run("cold")
d = synth.awq_like_torch(1, 28672, 4096, seed=9)
p = api.pack_w4(d["q"], d["s"], d["z"], 128)
A = torch.randn(8192, 4096, device="cuda").to(torch.bfloat16)
for _ in range(40):
    api.gemm_w4a16(A, p, d["s"], d["z"])
torch.cuda.synchronize()
print("after prefill burst", clk())
run("hot")
