"""GPU parity of the opt-in fused-scale decode variant (TM_FS=1: dequant sets apply the group
scales, cluster split-K, group 128).  The switch is read once per process, so the
cases run in a child process."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys
sys.path.insert(0, ROOT)
import torch
from oracle import compare
from oracle.gemm import gemm_f64
from paper_2508_15601_b200 import api, synth
ok = True
for M, N, K, cs in ((16, 512, 2048, 2), (1, 384, 3072, 3), (9, 256, 4096, 4), (5, 256, 1024, -1), (16, 512, 2048, 5)):
    api.set_decode_cluster(cs)
    d = synth.awq_like(M, N, K, group=128, seed=M + N + K + cs)
    A = torch.from_numpy(d["A"]).to(torch.bfloat16).cuda()
    q, s, z = (torch.from_numpy(d[k]).cuda() for k in ("q", "s", "z"))
    C = api.gemm_w4a16(A, api.pack_w4(q, s, z, 128), s, z)
    torch.cuda.synchronize()
    r = compare.check(C.float().cpu().numpy(), gemm_f64(d["A"], d["q"], d["s"], d["z"], 128),
                      d["A"], d["q"], d["s"], d["z"], 128, "bf16")
    cfg = api.query_gemm_config(M, N, K)
    assert cfg["kind"] == 2, cfg
    print(M, N, K, cs, cfg, r["ok"], r["relfro"])
    ok &= r["ok"]
print("all ok" if ok else "FAIL")
'''.replace("ROOT", repr(ROOT))


def test_fused_scale_variant_parity():
    env = dict(os.environ, TM_FS="1")
    r = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0 and "all ok" in r.stdout, r.stdout + r.stderr
