#!/usr/bin/env python
"""bench.py -- W4A16 GEMM throughput on B200 (driver contract).

Workload (BASELINE.json configs[1], the config the metric is quoted on): Llama-3-8B decode
GEMMs -- qkv (N=6144, K=4096), o (4096, 4096), gate_up (28672, 4096), down (4096, 14336) -- at
M = 1, 8, 16 tokens, group 128, bf16 activations, over L distinct synthetic layers (default 4,
436 MB of packed weights, > 3x the 126 MB L2, so every step streams weights from HBM).
One step = every (M, layer, shape) GEMM once (48 launches at L = 4).

value  = algorithmic bytes of the step (packed codes + fp16 s/z + A + C) / time,
         device-timed with CUDA events around a CUDA-graph replay of K steps, inputs resident.
e2e    = same through the public API with each GEMM's A copied from pinned host memory and
         C copied back to pinned host memory inside the timed region.
N > 1  : tensor parallel (torchrun, one process per GPU, NCCL): qkv and gate_up column-parallel,
         o and down row-parallel with an fp32 all-reduce + finalize; strong scaling of the same
         workload; time = max over ranks.
--impl reference: the CPU oracle (oracle/gemm.py, fp64) on a bounded sample of the workload.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SHAPES = [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]
ROW_PARALLEL = {"o", "down"}
METRIC = "W4A16 GEMM TFLOP/s + HBM GB/s vs B200 roofline, Llama-3 shapes, M=1-8192"
WORKLOAD = "Llama-3-8B decode GEMMs (qkv/o/gate_up/down), M in {1,8,16}, group 128, bf16"


def alg_bytes(M, N, K, g=128):
    return K * N // 2 + 4 * (K // g) * N + 2 * M * K + 2 * M * N


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=float(d["hbm_gbs"]), tc=float(d["bf16_tflops"]), src="measured")
    return dict(hbm=6650.0, tc=1590.0, src="fallback")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                power.append(float(parts[6]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        sm.sort()
        return dict(sm_mhz=sm[len(sm) // 2], sm_max_mhz=max(mx), reasons=sorted(reasons), samples=len(sm),
                    power_w_max=max(power) if power else None)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------------- our arm
def build_layers(L, world, rank, device):
    import torch
    from paper_2508_15601_b200 import api, synth
    from paper_2508_15601_b200.tp import shard_bounds
    layers = []
    for li in range(L):
        lay = {}
        for name, N, K in SHAPES:
            d = synth.awq_like_torch(1, N, K, group=128, seed=7000 + 17 * li + N + K, device=device)
            q, s, z = d["q"], d["s"], d["z"]
            if world > 1 and name in ROW_PARALLEL:
                lo, hi = shard_bounds(K, world, rank, 128)
                q, s, z = q[lo:hi].contiguous(), s[lo // 128:hi // 128].contiguous(), z[lo // 128:hi // 128].contiguous()
                kind = "row"
            elif world > 1:
                lo, hi = shard_bounds(N, world, rank, 128)
                q, s, z = q[:, lo:hi].contiguous(), s[:, lo:hi].contiguous(), z[:, lo:hi].contiguous()
                kind = "col"
            else:
                lo, hi, kind = 0, N, "full"
            p = api.pack_w4(q, s, z, 128)
            lay[name] = dict(packed=p, s=s, z=z, N=N, K=K, kind=kind, lo=lo, hi=hi)
            del d, q
        layers.append(lay)
        torch.cuda.synchronize()
    return layers


def make_io(layers, ms, device, world):
    import torch
    io = {}
    g = torch.Generator(device=device)
    g.manual_seed(1234)
    for M in ms:
        for name, N, K in SHAPES:
            w = layers[0][name]
            Kl = (w["hi"] - w["lo"]) if w["kind"] == "row" else K
            Nl = (w["hi"] - w["lo"]) if w["kind"] == "col" else N
            A = torch.randn(M, Kl, device=device, generator=g).to(torch.bfloat16)
            C = torch.empty(M, Nl, device=device, dtype=torch.bfloat16)
            P = torch.empty(M, N, device=device, dtype=torch.float32) if w["kind"] == "row" else None
            io[(M, name)] = dict(A=A, C=C, P=P)
    return io


def run_step(layers, io, ms, e2e=None):
    """One step: every (M, layer, shape) GEMM.  e2e: dict of pinned host buffers -> copies in."""
    from paper_2508_15601_b200 import api
    from paper_2508_15601_b200.tp import allreduce_sum_fp32
    n = 0
    for M in ms:
        for lay in layers:
            for name, N, K in SHAPES:
                w, b = lay[name], io[(M, name)]
                if e2e is not None:
                    b["A"].copy_(e2e[(M, name)]["A"], non_blocking=True)
                if w["kind"] == "row":
                    api.gemm_w4a16_partial_f32(b["A"], w["packed"], w["s"], w["z"], out=b["P"])
                    allreduce_sum_fp32(b["P"])
                    api.tp_finalize(b["P"], out=b["C"])
                    n += 2
                else:
                    api.gemm_w4a16(b["A"], w["packed"], w["s"], w["z"], out=b["C"])
                    n += 1
                if e2e is not None:
                    e2e[(M, name)]["C"].copy_(b["C"], non_blocking=True)
    return n


def step_bytes(ms, L):
    tot, flops = 0, 0
    for M in ms:
        for _ in range(L):
            for _, N, K in SHAPES:
                tot += alg_bytes(M, N, K)
                flops += 2 * M * N * K
    return tot, flops


def time_graph(graph, steps, stream):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def per_shape_detail(layers, io, ms, reps=20, stream=None):
    """Per-(M, shape) timing outside the timed region (context): CUDA-graph replay of `reps`
    launches of one shape rotating over the L layers, like the main leg."""
    import torch
    from paper_2508_15601_b200 import api
    out = []
    for M in ms:
        for name, N, K in SHAPES:
            b = io[(M, name)]
            if layers[0][name]["kind"] == "row":
                continue
            calls = [(lambda w=layers[r % len(layers)][name]: api.gemm_w4a16(b["A"], w["packed"], w["s"], w["z"],
                                                                              out=b["C"])) for r in range(reps)]
            with torch.cuda.stream(stream):
                for c in calls:
                    c()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for c in calls:
                        c()
                g.replay()
                torch.cuda.synchronize()
                t = time_graph(g, 3, stream) / 3 / reps
            out.append(dict(M=M, shape=name, us=round(t * 1e6, 2), GBps=round(alg_bytes(M, N, K) / t / 1e9, 1),
                            cfg=api.query_gemm_config(M, N if layers[0][name]["kind"] == "full" else
                                                      layers[0][name]["hi"] - layers[0][name]["lo"], K),
                            timing="CUDA-graph replay, %d launches rotating over the layers" % reps))
    return out


def prefill_leg(stream, steps=5, M=8192):
    """Secondary (tensor-bound) leg: the four Llama-3-8B layer GEMMs at M = 8192 tokens (BASELINE
    configs[2]), one synthetic layer, graph-timed like the main leg; reported against the dense
    bf16 tensor peak.  Not part of `value`."""
    import torch
    from paper_2508_15601_b200 import api, synth
    calls, flops = [], 0
    keep = []
    for name, N, K in SHAPES:
        d = synth.awq_like_torch(1, N, K, seed=7)
        p = api.pack_w4(d["q"], d["s"], d["z"], 128)
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        keep.append((p, d["s"], d["z"], A, C))
        calls.append(lambda p=p, s=d["s"], z=d["z"], A=A, C=C: api.gemm_w4a16(A, p, s, z, out=C))
        flops += 2 * M * N * K
    with torch.cuda.stream(stream):
        for _ in range(3):
            for c in calls:
                c()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for c in calls:
                c()
        g.replay()
        torch.cuda.synchronize()
        t = time_graph(g, steps, stream) / steps
    del keep, g
    torch.cuda.empty_cache()
    return t, flops


def ncu_traffic(ms, L):
    """Per-launch DRAM traffic of the GEMM kernel from the committed ncu capture, if present."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    vals = []
    for M in ms:
        for _, N, K in SHAPES:
            key = f"{M}x{N}x{K}"
            if key not in d:
                return None
            vals.append(d[key])
    return float(sum(vals) / len(vals))


def cpu_baseline(seconds_budget=20.0):
    """Oracle (oracle/gemm.py fp64) on a bounded sample: one layer's four GEMMs at M=16."""
    import numpy as np
    from threadpoolctl import threadpool_info
    from oracle.gemm import gemm_f64
    from paper_2508_15601_b200 import synth
    t_total, b_total, done = 0.0, 0, []
    for name, N, K in SHAPES:
        d = synth.awq_like(16, N, K, group=128, seed=42)
        t0 = time.perf_counter()
        gemm_f64(d["A"], d["q"], d["s"], d["z"], 128)
        t_total += time.perf_counter() - t0
        b_total += alg_bytes(16, N, K)
        done.append(name)
        if t_total > seconds_budget:
            break
    threads = max([x.get("num_threads", 1) for x in threadpool_info()] + [1])
    return dict(value=round(b_total / t_total / 1e9, 3), unit="GB/s", cores=threads, kind="oracle",
                sample=f"oracle fp64 GEMM (dequant + numpy matmul) of one layer's {'/'.join(done)} at M=16; "
                       f"{t_total:.1f} s on host; os.cpu_count()={os.cpu_count()}")


def bench_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2508_15601_b200 import api
    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    ms = [int(x) for x in args.ms.split(",")]
    L = args.layers
    layers = build_layers(L, world, rank, device)
    io = make_io(layers, ms, device, world)
    # pinned host buffers for the e2e leg
    host = {k: dict(A=v["A"].cpu().pin_memory(), C=torch.empty(v["C"].shape, dtype=v["C"].dtype).pin_memory())
            for k, v in io.items()}
    stream = torch.cuda.Stream(device)
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            n_launch = run_step(layers, io, ms)
        torch.cuda.synchronize()
        use_graph = world == 1
        if use_graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                run_step(layers, io, ms)
            ge = torch.cuda.CUDAGraph()
            with torch.cuda.graph(ge, stream=stream):
                run_step(layers, io, ms, e2e=host)
            for _ in range(2):
                g.replay()
                ge.replay()
            torch.cuda.synchronize()
    nbytes, nflops = step_bytes(ms, L)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        with torch.cuda.stream(stream):
            if use_graph:
                t = time_graph(g, args.steps, stream)
            else:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(args.steps):
                    run_step(layers, io, ms)
                e1.record(stream)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) * 1e-3
    torch.cuda.synchronize()
    # e2e (host copies in the timed region)
    with torch.cuda.stream(stream):
        if use_graph:
            te = time_graph(ge, args.steps, stream)
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                run_step(layers, io, ms, e2e=host)
            e1.record(stream)
            torch.cuda.synchronize()
            te = e0.elapsed_time(e1) * 1e-3
    if world > 1:
        tt = torch.tensor([t, te], device=device, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t, te = float(tt[0]), float(tt[1])
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    per_step = t / args.steps
    value = nbytes / per_step / 1e9
    e2e_value = nbytes / (te / args.steps) / 1e9
    peaks = load_peaks()
    h2d = sum(io[(M, n)]["A"].numel() * 2 for M in ms for n, _, _ in SHAPES) * L
    d2h = sum(io[(M, n)]["C"].numel() * 2 for M in ms for n, _, _ in SHAPES) * L
    if world == 1:
        detail = per_shape_detail(layers, io, ms, stream=stream)  # same stream: its stream-K workspace
    else:
        detail = None
    traffic = ncu_traffic(ms, L)
    gemm_launches = len(ms) * L * len(SHAPES)
    res = dict(
        metric=METRIC, value=round(value, 1), unit="GB/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
        ms_per_step=round(per_step * 1e3, 4), higher_is_better=True, scaling="strong" if world > 1 else "weak",
        vs_baseline=None, dtype="bf16 act x u4 weights (fp32 accumulate)", data="synthetic",
        config=dict(workload=WORKLOAD, layers=L, ms=ms, group=128, shapes={n: [N, K] for n, N, K in SHAPES},
                    parallelism=f"tp{world}" if world > 1 else "single-GPU",
                    weights_bytes_per_step=int(sum(K * N // 2 for _, N, K in SHAPES) * L * len(ms)),
                    l2_policy="inputs larger than L2: %d MB of packed weights per pass (> 3 x 126 MB L2)" %
                              (sum(K * N // 2 for _, N, K in SHAPES) * L // 2 ** 20),
                    timing="CUDA-graph replay of K steps, CUDA events on the launch stream"),
        tflops=round(nflops / per_step / 1e12, 2),
        roofline=dict(bound="hbm", achieved=round(value, 1), peak=peaks["hbm"], unit="GB/s",
                      frac=round(value / peaks["hbm"], 4), traffic=traffic,
                      peak_source=f"MEASURED_PEAKS.json hbm_gbs ({peaks['src']}); achieved = algorithmic bytes per "
                                  f"launch / average launch duration over the timed region (launches back to back)"),
        e2e=dict(value=round(e2e_value, 1), unit="GB/s", h2d_bytes_per_step=int(h2d), d2h_bytes_per_step=int(d2h)),
        gpu_launches=int((n_launch if world > 1 else gemm_launches) * args.steps),
        detail=detail,
    )
    clk = clk.summary()
    res["clocks"] = clk
    if world == 1 and not args.no_prefill:
        tp, fl = prefill_leg(stream)
        achieved = fl / tp / 1e12
        res["prefill"] = dict(
            workload="Llama-3-8B prefill GEMMs (qkv/o/gate_up/down) at M=8192, group 128, bf16 (BASELINE configs[2])",
            us_per_step=round(tp * 1e6, 1), tflops=round(achieved, 1),
            roofline=dict(bound="tensor", achieved=round(achieved, 1), peak=peaks["tc"], unit="TFLOP/s",
                          frac=round(achieved / peaks["tc"], 4),
                          peak_source=f"MEASURED_PEAKS.json bf16_tflops ({peaks['src']}, burst: cuBLAS bf16 8192^3)"))
    if world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline()
    print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------------- reference arm
def bench_reference(args):
    """The CPU oracle as it stands, each step a bounded sample (one (M, shape) GEMM restricted
    to a 512-column slice, cycling through the workload's 12 (M, shape) pairs)."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    from threadpoolctl import threadpool_info
    from oracle.gemm import gemm_f64
    from paper_2508_15601_b200 import synth
    ms = [int(x) for x in args.ms.split(",")]
    pairs = [(M, name, N, K) for M in ms for name, N, K in SHAPES]
    cols = 512
    data = {}
    for M, name, N, K in pairs:
        if (name, K) not in data:
            data[(name, K)] = synth.awq_like(max(ms), cols, K, group=128, seed=5)
    for w in range(args.warmup):
        M, name, N, K = pairs[w % len(pairs)]
        d = data[(name, K)]
        gemm_f64(d["A"][:M], d["q"], d["s"], d["z"], 128)
    nbytes = 0
    t0 = time.perf_counter()
    for st in range(args.steps):
        M, name, N, K = pairs[st % len(pairs)]
        d = data[(name, K)]
        gemm_f64(d["A"][:M], d["q"], d["s"], d["z"], 128)
        nbytes += alg_bytes(M, cols, K)
    t = time.perf_counter() - t0
    value = nbytes / t / 1e9
    threads = max([x.get("num_threads", 1) for x in threadpool_info()] + [1])
    res = dict(
        impl="reference", metric=METRIC, value=round(value, 4), unit="GB/s", n_gpus=world, steps=args.steps,
        warmup=args.warmup, ms_per_step=round(t / args.steps * 1e3, 3), higher_is_better=True,
        scaling="strong" if world > 1 else "weak", vs_baseline=None, dtype="f64", data="synthetic",
        config=dict(workload=WORKLOAD, sample=f"{cols}-column slice per step", ms=ms, group=128),
        cpu_baseline=dict(value=round(value, 4), unit="GB/s", cores=threads, kind="oracle",
                          sample=f"each step: oracle fp64 GEMM of one (M, shape) pair on a {cols}-column slice"),
        e2e=dict(value=round(value, 4), unit="GB/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
    )
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--ms", default="1,8,16")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prefill", action="store_true", help="skip the secondary M=8192 tensor-bound leg")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
