"""CFG#4 / CFG#3 sweep (BASELINE.json configs[3], configs[4]): group size x M x layer shapes of
Llama-3-8B, Llama-3-70B, Qwen2-72B and a Mixtral expert, graph-timed, each point against its own
roofline min(TC_peak, HBM_peak * AI(M)).  Prints a markdown table (profiles/r01_sweep_cfg4.md).

    python scripts/sweep_cfg4.py [--ms 1,16,64,256,1024,4096,8192] [--quick]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from graph_perf import time_graph  # noqa: E402
from paper_2508_15601_b200 import api, synth  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [
    ("llama3-8b", "qkv", 6144, 4096), ("llama3-8b", "o", 4096, 4096), ("llama3-8b", "gate_up", 28672, 4096),
    ("llama3-8b", "down", 4096, 14336),
    ("llama3-70b", "qkv", 10240, 8192), ("llama3-70b", "o", 8192, 8192), ("llama3-70b", "gate_up", 57344, 8192),
    ("llama3-70b", "down", 8192, 28672),
    ("qwen2-72b", "qkv", 10240, 8192), ("qwen2-72b", "o", 8192, 8192), ("qwen2-72b", "gate_up", 59136, 8192),
    ("qwen2-72b", "down", 8192, 29568),
    ("mixtral", "expert w1", 14336, 4096),
]


def alg_bytes(M, N, K, g):
    return K * N // 2 + 4 * (K // g) * N + 2 * M * K + 2 * M * N


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1,16,64,256,1024,4096,8192")
    ap.add_argument("--quick", action="store_true", help="8B shapes only")
    a = ap.parse_args()
    ms = [int(x) for x in a.ms.split(",")]
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm, tc = float(pk["hbm_gbs"]) * 1e9, float(pk["bf16_tflops"]) * 1e12
    print(f"peaks: HBM {hbm / 1e9:.0f} GB/s, bf16 {tc / 1e12:.0f} TFLOP/s (MEASURED_PEAKS.json); "
          f"roofline(M) = min(TC, HBM * flops/bytes)\n")
    print("| model | layer | N | K | g | M | us | GB/s | TFLOP/s | bound | frac of roofline | config |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    shapes = SHAPES[:4] if a.quick else SHAPES
    for model, layer, N, K in shapes:
        groups = (128, 64) if model in ("llama3-8b", "mixtral") else (128,)
        for g in groups:
            wbytes = K * N // 2
            nsets = max(1, min(4, int(3 * 126e6 // wbytes) + 1))
            sets = []
            for i in range(nsets):
                d = synth.awq_like_torch(1, N, K, group=g, seed=200 + i)
                sets.append((api.pack_w4(d["q"], d["s"], d["z"], g), d["s"], d["z"]))
                del d
            for M in ms:
                A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
                C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                reps = max(1, min(24, int(2e12 // max(1, 2 * M * N * K)) + 1))
                calls = [(lambda p=p, s=s, z=z: api.gemm_w4a16(A, p, s, z, out=C)) for (p, s, z) in sets]
                calls = (calls * ((reps + len(calls) - 1) // len(calls)))[:max(reps, len(calls))]
                t = time_graph(calls, reps=3) / len(calls) * 1e-6
                fl = 2 * M * N * K
                by = alg_bytes(M, N, K, g)
                roof_t = max(fl / tc, by / hbm)
                bound = "tensor" if fl / tc > by / hbm else "hbm"
                cfg = api.query_gemm_config(M, N, K)
                print(f"| {model} | {layer} | {N} | {K} | {g} | {M} | {t * 1e6:.1f} | {by / t / 1e9:.0f} | "
                      f"{fl / t / 1e12:.1f} | {bound} | {roof_t / t:.3f} | t{cfg['tile_m']} s{cfg['split_k']} k{cfg['kind']} |",
                      flush=True)
                del A, C
            del sets
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
