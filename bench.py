#!/usr/bin/env python
"""bench.py -- W4A16 GEMM throughput on B200 (driver contract).

Workload (BASELINE.json configs[1], the config the metric is quoted on): Llama-3-8B decode
GEMMs -- qkv (N=6144, K=4096), o (4096, 4096), gate_up (28672, 4096), down (4096, 14336) -- at
M = 1, 8, 16 tokens, group 128, bf16 activations, over L distinct synthetic layers (default 4,
436 MB of packed weights, > 3x the 126 MB L2, so every step streams weights from HBM).
One step = every (M, layer, shape) GEMM once (48 launches at L = 4).

value  = algorithmic bytes of the step (packed codes + fp16 s/z + A + C) / time,
         device-timed with CUDA events around a CUDA-graph replay of K steps, inputs resident.
e2e    = same through the public API with the step's activations copied from pinned host memory
         (one copy) and its outputs copied back (one copy) inside the timed region, on two copy
         streams double-buffered against the compute graph.
N > 1  : tensor parallel (torchrun, one process per GPU, NCCL; `--gpus N` alone self-launches
         the N ranks): qkv and gate_up column-parallel, o and down row-parallel with an fp32
         all-reduce + finalize (paper_2508_15601_b200/tp.py classes); the step, all-reduces
         included, is one CUDA graph; strong scaling of the same workload; time = max over
         ranks; GEMM and all-reduce times are reported separately under "tp".
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
    """L synthetic Llama-3-8B layers as the product's tensor-parallel layer classes
    (paper_2508_15601_b200/tp.py): qkv/gate_up ColumnParallelW4, o/down RowParallelW4 at
    world > 1; every layer ColumnParallelW4 over the whole N (one shard) at world = 1."""
    import torch
    from paper_2508_15601_b200 import synth
    from paper_2508_15601_b200.tp import ColumnParallelW4, RowParallelW4
    layers = []
    for li in range(L):
        lay = {}
        for name, N, K in SHAPES:
            d = synth.awq_like_torch(1, N, K, group=128, seed=7000 + 17 * li + N + K, device=device)
            if world > 1 and name in ROW_PARALLEL:
                lay[name] = RowParallelW4(d["q"], d["s"], d["z"], 128, world, rank)
            else:
                lay[name] = ColumnParallelW4(d["q"], d["s"], d["z"], 128, world if world > 1 else 1,
                                             rank if world > 1 else 0)
            del d
        layers.append(lay)
        torch.cuda.synchronize()
    return layers


def make_io(layers, ms, device, nsets=2):
    """Per buffer set: every (M, shape)'s A and C as views into one contiguous device buffer
    (so the end-to-end leg moves a step's inputs and outputs with one copy each way)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(1234)
    shapes = []
    for M in ms:
        for name, N, K in SHAPES:
            w = layers[0][name]
            row = hasattr(w, "local_partial")
            Kl = (w.hi - w.lo) if row else K
            Nl = N if row else (w.hi - w.lo)
            shapes.append((M, name, Kl, Nl, row, N))
    a_elems = sum(M * Kl for M, _, Kl, _, _, _ in shapes)
    c_elems = sum(M * Nl for M, _, _, Nl, _, _ in shapes)
    src = torch.randn(a_elems, device=device, generator=g).to(torch.bfloat16)
    sets = []
    for _ in range(nsets):
        A_all = src.clone()
        C_all = torch.empty(c_elems, device=device, dtype=torch.bfloat16)
        io, ao, co = {}, 0, 0
        for M, name, Kl, Nl, row, N in shapes:
            A = A_all[ao:ao + M * Kl].view(M, Kl)
            C = C_all[co:co + M * Nl].view(M, Nl)
            P = torch.empty(M, N, device=device, dtype=torch.float32) if row else None
            io[(M, name)] = dict(A=A, C=C, P=P)
            ao += M * Kl
            co += M * Nl
        sets.append(dict(io=io, A_all=A_all, C_all=C_all))
    return sets


def run_step(layers, io, ms, part="all", reducer=None):
    """One step: every (M, layer, shape) GEMM.  part: "all"; "gemm" (the local GEMMs and the
    finalize of row-parallel layers, no collective); "comm" (only the all-reduces).
    reducer (--tp-reduce symm): row-parallel layers use the fused NEXT-1 epilogue (partial
    into symmetric memory + tm_tp_allreduce_finalize) instead of NCCL + tm_tp_finalize."""
    from paper_2508_15601_b200 import api
    from paper_2508_15601_b200.tp import allreduce_sum_fp32
    n = 0
    for M in ms:
        for lay in layers:
            for name, N, K in SHAPES:
                w, b = lay[name], io[(M, name)]
                if hasattr(w, "local_partial") and reducer is not None:
                    if part != "comm":
                        w.local_partial(b["A"], out=reducer.partial(M, N))
                        n += 1
                    if part != "gemm":
                        reducer.finalize(M, N, b["C"])
                        n += 1
                elif hasattr(w, "local_partial"):  # row-parallel: fp32 partial, all-reduce, finalize
                    if part != "comm":
                        w.local_partial(b["A"], out=b["P"])
                        n += 1
                    if part != "gemm":
                        allreduce_sum_fp32(b["P"])
                    if part != "comm":
                        api.tp_finalize(b["P"], out=b["C"])
                        n += 1
                elif part != "comm":
                    w(b["A"], out=b["C"])
                    n += 1
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
    """Seconds for `steps` replays, CUDA events on `stream` (the replays are issued on it)."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(steps):
            graph.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def capture(fn, stream):
    import torch
    torch.cuda.synchronize()  # inputs made on the default stream are complete before `stream` reads them
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            fn()
        g.replay()
    torch.cuda.synchronize()
    return g


def per_shape_detail(layers, io, ms, reps=20, stream=None):
    """Per-(M, shape) timing outside the timed region (context): CUDA-graph replay of `reps`
    launches of one shape rotating over the L layers, like the main leg."""
    from paper_2508_15601_b200 import api
    out = []
    for M in ms:
        for name, N, K in SHAPES:
            b = io[(M, name)]
            if hasattr(layers[0][name], "local_partial"):
                continue
            calls = [(lambda w=layers[r % len(layers)][name]: w(b["A"], out=b["C"])) for r in range(reps)]
            g = capture(lambda: [c() for c in calls], stream)
            t = time_graph(g, 3, stream) / 3 / reps
            Nl = layers[0][name].hi - layers[0][name].lo
            out.append(dict(M=M, shape=name, us=round(t * 1e6, 2), GBps=round(alg_bytes(M, Nl, K) / t / 1e9, 1),
                            cfg=api.query_gemm_config(M, Nl, K),
                            timing="CUDA-graph replay, %d launches rotating over the layers" % reps))
    return out


def prefill_leg(stream, min_seconds=1.0, M=8192):
    """Secondary (tensor-bound) leg: the four Llama-3-8B layer GEMMs at M = 8192 tokens (BASELINE
    configs[2]), one synthetic layer, graph-timed like the main leg with the clocks sampled over
    a timed region of >= min_seconds; reported against the dense bf16 tensor peak.  Not part
    of `value`.  torch.matmul bf16 on the same shapes (the paper's E2 comparison)
    is timed beside it."""
    import torch
    from paper_2508_15601_b200 import api, synth
    calls, dense, flops = [], [], 0
    keep = []
    for name, N, K in SHAPES:
        d = synth.awq_like_torch(1, N, K, seed=7)
        p = api.pack_w4(d["q"], d["s"], d["z"], 128)
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        Wd = torch.randn(K, N, device="cuda").to(torch.bfloat16)
        keep.append((p, d["s"], d["z"], A, C, Wd))
        calls.append(lambda p=p, s=d["s"], z=d["z"], A=A, C=C: api.gemm_w4a16(A, p, s, z, out=C))
        dense.append(lambda A=A, Wd=Wd, C=C: torch.matmul(A, Wd, out=C))
        flops += 2 * M * N * K
    with torch.cuda.stream(stream):
        for _ in range(3):
            for c in calls + dense:
                c()
    torch.cuda.synchronize()
    g = capture(lambda: [c() for c in calls], stream)
    gd = capture(lambda: [c() for c in dense], stream)
    t1 = time_graph(g, 2, stream) / 2
    steps = min(2000, max(5, int(min_seconds / t1) + 1))
    with ClockSampler(torch.cuda.current_device()) as clk:
        t = time_graph(g, steps, stream) / steps
    nd = min(1000, max(5, int(min_seconds / 2 / t1) + 1))
    td = time_graph(gd, nd, stream) / nd
    del keep, g, gd
    torch.cuda.empty_cache()
    return t, flops, steps, clk.summary(), td


def moe_leg(stream, reps=20):
    """Context leg (§8(f) NEXT-3, CFG#4 Mixtral expert shape N = 14336, K = 4096): decode of 8
    experts with 4 routed tokens each (16 tokens, top-2) as ONE grouped launch vs one launch per
    expert; 3 weight sets rotate (750 MB > L2).  GB/s = bytes of the experts read / time."""
    import torch
    from paper_2508_15601_b200 import api, synth
    N, K, E, g, m = 14336, 4096, 8, 128, [4] * 8
    sets = []
    for rep in range(3):
        ds = [synth.awq_like_torch(1, N, K, group=g, seed=900 + 10 * rep + e) for e in range(E)]
        s_ = torch.stack([d["s"] for d in ds])
        z_ = torch.stack([d["z"] for d in ds])
        sets.append((api.pack_experts([d["q"] for d in ds], s_, z_, g), s_, z_,
                     [api.pack_w4(d["q"], d["s"], d["z"], g) for d in ds], ds))
    A = torch.randn(sum(m), K, device="cuda").to(torch.bfloat16)
    C = torch.empty(sum(m), N, device="cuda", dtype=torch.bfloat16)
    nbytes = E * (K * N // 2 + 4 * (K // g) * N) + 2 * sum(m) * (K + N)

    def grouped(i):
        pe, s_, z_, _, _ = sets[i % 3]
        api.gemm_w4a16_grouped(A, pe, s_, z_, m, out=C)

    def separate(i):
        _, _, _, singles, ds = sets[i % 3]
        for e in range(E):
            api.gemm_w4a16(A[4 * e:4 * e + 4], singles[e], ds[e]["s"], ds[e]["z"], out=C[4 * e:4 * e + 4])

    gg = capture(lambda: [grouped(i) for i in range(reps)], stream)
    gs = capture(lambda: [separate(i) for i in range(reps)], stream)
    tg = time_graph(gg, 3, stream) / 3 / reps
    ts = time_graph(gs, 3, stream) / 3 / reps
    del sets
    torch.cuda.empty_cache()
    return dict(workload="Mixtral-8x7B expert w1 (N=14336, K=4096, g=128), 8 experts x 4 tokens, bf16",
                grouped_us=round(tg * 1e6, 2), grouped_GBps=round(nbytes / tg / 1e9, 1),
                per_expert_launches_us=round(ts * 1e6, 2), per_expert_GBps=round(nbytes / ts / 1e9, 1),
                grouped_frac_of_hbm=round(nbytes / tg / 1e9 / load_peaks()["hbm"], 4))


def attention_leg(stream, reps=20, B=32, L=8192):
    """Context leg (§8(f) NEXT-2): one decode step of 8-bit-KV attention with Llama-3-8B heads
    (Hq 32, Hkv 8, D 128), B sequences of L cached tokens, two caches rotating (1.1 GB > L2).
    GB/s = KV codes + (scale, zero) words + Q + O bytes / time."""
    import torch
    from paper_2508_15601_b200 import api
    Hq, Hkv, D = 32, 8, 128
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    sets = []
    for _ in range(2):
        kc = torch.randint(0, 256, (B, Hkv, L, D), dtype=torch.uint8, device="cuda", generator=g)
        vc = torch.randint(0, 256, (B, Hkv, L, D), dtype=torch.uint8, device="cuda", generator=g)
        sc = (torch.rand(B, Hkv, L, device="cuda", generator=g) * 0.02 + 0.01).half()
        zz = torch.full((B, Hkv, L), 128.0, device="cuda").half()
        sets.append((kc, vc, api.pack_kv_sz(sc, zz), api.pack_kv_sz(sc, zz)))
    Q = torch.randn(B, Hq, D, device="cuda", generator=g).to(torch.bfloat16)
    sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
    ws = api.attn_workspace(B, Hq, Hkv, L)
    O = torch.empty_like(Q)
    gr = capture(lambda: [api.attn_decode_kv8(Q, *sets[i % 2][:2], *sets[i % 2][2:], sl, workspace=ws, out=O)
                          for i in range(reps)], stream)
    t = time_graph(gr, 3, stream) / 3 / reps
    nbytes = B * Hkv * L * (2 * D + 8) + 2 * B * Hq * D * 2
    del sets
    torch.cuda.empty_cache()
    return dict(workload=f"decode attention, 8-bit KV cache, Hq=32 Hkv=8 D=128, B={B} L={L}, bf16 Q/O",
                us=round(t * 1e6, 2), GBps=round(nbytes / t / 1e9, 1),
                frac_of_hbm=round(nbytes / t / 1e9 / load_peaks()["hbm"], 4))


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
                cpu_model=cpu_model(),
                sample=f"oracle fp64 GEMM (dequant + numpy matmul) of one layer's {'/'.join(done)} at M=16; "
                       f"{t_total:.1f} s on host; os.cpu_count()={os.cpu_count()}")


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def time_e2e(graphs, sets, host_A, host_C, steps, comp):
    """End to end through the public API: every step copies its inputs host -> device (one
    pinned-memory copy of all the step's activations) and its outputs device -> host (one copy of
    all the step's C), on two copy streams, double-buffered so step i's copies overlap step
    i +- 1's GEMMs.  Timed with CUDA events from before the first input copy to after the last
    output copy."""
    import torch
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(comp)
    h2d.wait_event(e0)
    for i in range(steps):
        b = i % 2
        if i >= 2:
            h2d.wait_event(ev_comp[b])  # step i - 2 finished reading this input buffer
        with torch.cuda.stream(h2d):
            sets[b]["A_all"].copy_(host_A, non_blocking=True)
        ev_in[b].record(h2d)
        comp.wait_event(ev_in[b])
        if i >= 2:
            comp.wait_event(ev_out[b])  # step i - 2's outputs have left this buffer
        with torch.cuda.stream(comp):
            graphs[b].replay()
        ev_comp[b].record(comp)
        d2h.wait_event(ev_comp[b])
        with torch.cuda.stream(d2h):
            host_C.copy_(sets[b]["C_all"], non_blocking=True)
        ev_out[b].record(d2h)
    comp.wait_stream(d2h)
    e1.record(comp)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def bench_ours(args):
    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    ms = [int(x) for x in args.ms.split(",")]
    L = args.layers
    layers = build_layers(L, world, rank, device)
    reducer = None
    if world > 1 and args.tp_reduce == "symm":
        from paper_2508_15601_b200.tp import SymmReducer
        reducer = SymmReducer(max(ms) * max(N for _, N, _ in SHAPES), device=device)
    sets = make_io(layers, ms, device)
    io = sets[0]["io"]
    host_A = sets[0]["A_all"].cpu().pin_memory()
    host_C = torch.empty(sets[0]["C_all"].numel(), dtype=torch.bfloat16).pin_memory()
    stream = torch.cuda.Stream(device)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            n_launch = run_step(layers, io, ms, reducer=reducer)
    torch.cuda.synchronize()
    # the whole step -- GEMMs and, under TP, the NCCL all-reduces -- is one CUDA graph
    graphs = [capture(lambda st=st: run_step(layers, st["io"], ms, reducer=reducer), stream) for st in sets]
    g = graphs[0]
    time_graph(g, 2, stream)
    nbytes, nflops = step_bytes(ms, L)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t = time_graph(g, args.steps, stream)
    torch.cuda.synchronize()
    te = time_e2e(graphs, sets, host_A, host_C, args.steps, stream)
    tp_detail = None
    if world > 1:
        gg = capture(lambda: run_step(layers, io, ms, part="gemm", reducer=reducer), stream)
        gc = capture(lambda: run_step(layers, io, ms, part="comm", reducer=reducer), stream)
        dist.barrier()
        t_gemm = time_graph(gg, args.steps, stream)
        dist.barrier()
        t_comm = time_graph(gc, args.steps, stream)
        tt = torch.tensor([t, te, t_gemm, t_comm], device=device, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t, te, t_gemm, t_comm = (float(x) for x in tt)
        ar_bytes = sum(M * N * 4 for M in ms for n, N, K in SHAPES if n in ROW_PARALLEL) * L
        tp_detail = dict(
            gemm_ms_per_step=round(t_gemm / args.steps * 1e3, 4), allreduce_ms_per_step=round(t_comm / args.steps * 1e3, 4),
            allreduce_bytes_per_step=int(ar_bytes), allreduces_per_step=len(ms) * L * len(ROW_PARALLEL),
            reduce=args.tp_reduce,
            note="max over ranks of CUDA-graph replays of (a) only the local GEMMs (+ finalize for nccl) and (b) only "
                 "the reductions (fp32 NCCL all-reduces, or the fused symmetric-memory all-reduce + finalize kernel "
                 "for symm); the step graph (value) runs both in order")
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    per_step = t / args.steps
    value = nbytes / per_step / 1e9
    e2e_value = nbytes / (te / args.steps) / 1e9
    peaks = load_peaks()
    h2d = host_A.numel() * 2
    d2h = host_C.numel() * 2
    detail = per_shape_detail(layers, io, ms, stream=stream) if world == 1 else None
    traffic = ncu_traffic(ms, L)
    res = dict(
        metric=METRIC, value=round(value, 1), unit="GB/s", n_gpus=world, steps=args.steps, warmup=args.warmup,
        ms_per_step=round(per_step * 1e3, 4), higher_is_better=True, scaling="strong" if world > 1 else "weak",
        vs_baseline=None, dtype="bf16 act x u4 weights (fp32 accumulate)", data="synthetic",
        config=dict(workload=WORKLOAD, layers=L, ms=ms, group=128, shapes={n: [N, K] for n, N, K in SHAPES},
                    parallelism=f"tp{world}" if world > 1 else "single-GPU",
                    weights_bytes_per_step=int(sum(K * N // 2 for _, N, K in SHAPES) * L * len(ms)),
                    l2_policy="inputs larger than L2: %d MB of packed weights per pass (> 3 x 126 MB L2)" %
                              (sum(K * N // 2 for _, N, K in SHAPES) * L // 2 ** 20),
                    timing="CUDA-graph replay of K steps, CUDA events on the launch stream" +
                           ("; max over ranks" if world > 1 else "")),
        tflops=round(nflops / per_step / 1e12, 2),
        roofline=dict(bound="hbm", achieved=round(value, 1), peak=peaks["hbm"], unit="GB/s",
                      frac=round(value / peaks["hbm"], 4), traffic=traffic,
                      peak_source=f"MEASURED_PEAKS.json hbm_gbs ({peaks['src']}); achieved = algorithmic bytes per "
                                  f"launch / average launch duration over the timed region (launches back to back)"),
        e2e=dict(value=round(e2e_value, 1), unit="GB/s", h2d_bytes_per_step=int(h2d), d2h_bytes_per_step=int(d2h),
                 copies_per_step="1 H2D (all activations) + 1 D2H (all outputs), pinned host memory, two copy "
                                 "streams, double-buffered against the compute graph"),
        gpu_launches=int(n_launch * args.steps),
        detail=detail,
    )
    if tp_detail:
        res["tp"] = tp_detail
    res["clocks"] = clk.summary()
    if world == 1 and not args.no_prefill:
        tp_, fl, nsteps, pclk, td = prefill_leg(stream)
        achieved = fl / tp_ / 1e12
        res["prefill"] = dict(
            workload="Llama-3-8B prefill GEMMs (qkv/o/gate_up/down) at M=8192, group 128, bf16 (BASELINE configs[2])",
            us_per_step=round(tp_ * 1e6, 1), tflops=round(achieved, 1), timed_steps=nsteps,
            timed_seconds=round(tp_ * nsteps, 3), clocks=pclk,
            dense_bf16_torch_matmul=dict(us_per_step=round(td * 1e6, 1), tflops=round(fl / td / 1e12, 1)),
            roofline=dict(bound="tensor", achieved=round(achieved, 1), peak=peaks["tc"], unit="TFLOP/s",
                          frac=round(achieved / peaks["tc"], 4),
                          peak_source=f"MEASURED_PEAKS.json bf16_tflops ({peaks['src']}, burst: cuBLAS bf16 8192^3)"))
    if world == 1 and not args.no_prefill:
        res["moe"] = moe_leg(stream)
        res["attention"] = attention_leg(stream)
    if world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline()
    print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def self_launch(args):
    """`bench.py --gpus N` run directly (no torchrun): start N ranks with torch.distributed.run
    on this node (127.0.0.1 rendezvous); rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")              # communicator init (NVLink / NVLS) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


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
    ap.add_argument("--tp-reduce", default="nccl", choices=["nccl", "symm"],
                    help="row-parallel reduction at --gpus > 1: NCCL fp32 all-reduce + finalize, or the fused "
                         "symmetric-memory kernel (tm_tp_allreduce_finalize, NEXT-1)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    else:
        if int(os.environ.get("WORLD_SIZE", "1")) > 1:
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        bench_ours(args)


if __name__ == "__main__":
    main()
