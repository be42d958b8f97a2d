"""Per-shape decode timing through CUDA-graph replay (no host launch overhead in the timed
region; development aid, bench.py is the contract).  Weight sets rotate so the weights of
one replay exceed L2.

    python scripts/graph_perf.py [--ms 1,16] [--shapes qkv,o,gate_up,down] [--mix]
"""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}


def bytes_alg(M, N, K, g=128):
    return K * N // 2 + 4 * (K // g) * N + 2 * M * K + 2 * M * N


def make_sets(N, K, n):
    out = []
    for i in range(n):
        d = synth.awq_like_torch(1, N, K, seed=100 + i)
        out.append((api.pack_w4(d["q"], d["s"], d["z"], 128), d["s"], d["z"]))
    return out


def time_graph(calls, reps=10):
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())  # inputs were made on the default stream
    with torch.cuda.stream(stream):
        for c in calls:
            c()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for c in calls:
            c()
    with torch.cuda.stream(stream):
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps  # us per replay


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1,16")
    ap.add_argument("--shapes", default="qkv,o,gate_up,down")
    ap.add_argument("--mix", action="store_true", help="also the bench-like mixed sequence")
    a = ap.parse_args()
    ms = [int(x) for x in a.ms.split(",")]
    names = a.shapes.split(",")
    sets = {}
    for name in names:
        N, K = SHAPES[name]
        sets[name] = make_sets(N, K, max(2, min(8, int(3 * 126e6 // (K * N // 2)) + 1)))
    acts = {M: torch.randn(M, 14336, device="cuda").to(torch.bfloat16) for M in ms}
    for name in names:
        N, K = SHAPES[name]
        for M in ms:
            A = acts[M][:, :K].contiguous()
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            ss = sets[name]
            calls = [(lambda p=p, s=s, z=z: api.gemm_w4a16(A, p, s, z, out=C)) for (p, s, z) in ss] * max(1, 24 // len(ss))
            t = time_graph(calls) / len(calls)
            print(f"   {name:8s} M={M:3d} {t:7.2f} us {bytes_alg(M, N, K) / t / 1e3:7.0f} GB/s  cfg {api.query_gemm_config(M, N, K)}",
                  flush=True)
    if a.mix:
        calls, tot = [], 0
        for layer in range(2):
            for M in ms:
                for name in names:
                    N, K = SHAPES[name]
                    p, s, z = sets[name][layer % len(sets[name])]
                    A = acts[M][:, :K].contiguous()
                    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                    calls.append(lambda A=A, p=p, s=s, z=z, C=C: api.gemm_w4a16(A, p, s, z, out=C))
                    tot += bytes_alg(M, N, K)
        t = time_graph(calls)
        print(f"   mix of {len(calls)} launches: {t:.1f} us, {tot / t / 1e3:.0f} GB/s ({t / len(calls):.2f} us/launch)")
