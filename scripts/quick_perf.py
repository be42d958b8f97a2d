"""Quick per-shape timing of tm_gemm_w4a16 (development aid; bench.py is the contract).

Rotates over enough distinct weight sets to exceed L2, times with CUDA events."""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_15601_b200 import api, synth  # noqa: E402

SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}


def bytes_alg(M, N, K, g=128):
    return K * N // 2 + 4 * (K // g) * N + 2 * M * K + 2 * M * N


def run(M, N, K, reps=50, tile=0, split=0):
    api.set_gemm_override(tile, split)
    wbytes = K * N // 2
    nsets = max(1, min(16, int(3 * 126e6 // wbytes) + 1))
    sets = []
    for i in range(nsets):
        d = synth.awq_like_torch(1, N, K, seed=i)
        p = api.pack_w4(d["q"], d["s"], d["z"], 128)
        sets.append((p, d["s"], d["z"]))
        del d
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for i in range(5):
        p, s, z = sets[i % nsets]
        api.gemm_w4a16(A, p, s, z, out=C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        p, s, z = sets[i % nsets]
        api.gemm_w4a16(A, p, s, z, out=C)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    cfg = api.query_gemm_config(M, N, K)
    api.set_gemm_override(0, 0)
    return dict(M=M, N=N, K=K, us=t * 1e6, GBps=bytes_alg(M, N, K) / t / 1e9, TFLOPs=2 * M * N * K / t / 1e12, **cfg)


def torch_ref(M, N, K, reps=20):
    W = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        torch.matmul(A, W)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        torch.matmul(A, W)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e-3
    return dict(us=t * 1e6, TFLOPs=2 * M * N * K / t / 1e12)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="1,16,64,2048,8192")
    ap.add_argument("--shapes", default="qkv,o,gate_up,down")
    ap.add_argument("--sweep", action="store_true")
    a = ap.parse_args()
    for name in a.shapes.split(","):
        N, K = SHAPES[name]
        for M in [int(x) for x in a.ms.split(",")]:
            r = run(M, N, K)
            r["shape"] = name
            if M >= 1024:
                r["torch_bf16_TFLOPs"] = torch_ref(M, N, K)["TFLOPs"]
            print(json.dumps(r), flush=True)
            if a.sweep and M <= 64:
                for tile in ([16] if M <= 16 else [32, 64]):
                    for split in (1, 2, 3, 4, 6, 8):
                        try:
                            rr = run(M, N, K, tile=tile, split=split)
                            print("  sweep", json.dumps(rr), flush=True)
                        except Exception as e:  # noqa: BLE001
                            print("  sweep fail", tile, split, e)
