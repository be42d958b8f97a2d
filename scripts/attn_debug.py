"""Debug aid for the decode attention kernel: controlled inputs vs the fp64 oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.attention import decode_attention_f64  # noqa: E402
from paper_2508_15601_b200 import api, synth  # noqa: E402


def run(p):
    Q = torch.from_numpy(p["Q"]).to(torch.bfloat16).cuda()
    kc, vc = torch.from_numpy(p["kq"]).cuda(), torch.from_numpy(p["vq"]).cuda()
    ksz = api.pack_kv_sz(torch.from_numpy(p["ks"]).cuda(), torch.from_numpy(p["kz"]).cuda())
    vsz = api.pack_kv_sz(torch.from_numpy(p["vs"]).cuda(), torch.from_numpy(p["vz"]).cuda())
    sl = torch.from_numpy(p["seq_lens"]).cuda()
    B, Hq, D = Q.shape
    _, Hkv, Lmax, _ = kc.shape
    ws = api.attn_workspace(B, Hq, Hkv, Lmax)
    O = api.attn_decode_kv8(Q, kc, vc, ksz, vsz, sl, workspace=ws).float().cpu().numpy()
    ref = decode_attention_f64(p["Q"], p["kq"], p["ks"], p["kz"], p["vq"], p["vs"], p["vz"], p["seq_lens"])
    return np.linalg.norm(O - ref) / np.linalg.norm(ref), O, ref


if __name__ == "__main__":
  for name in ["random", "q0", "kconst", "vconst"]:
      for L in [2, 5, 16, 17, 64, 300]:
          p = synth.kv_decode_problem(1, 4, 1, 128, 320, [L], 8, seed=L)
          if name == "q0":
              p["Q"][:] = 0
          if name == "kconst":
              p["kq"][:] = p["kq"][:, :, :1]
              p["ks"][:] = p["ks"][:, :, :1]
              p["kz"][:] = p["kz"][:, :, :1]
          if name == "vconst":
              p["vq"][:] = 100
              p["vz"][:] = 0
              p["vs"][:] = 1.0
          rf, O, ref = run(p)
          print(f"{name:7s} L={L:4d} relfro {rf:.3e}  O[0,0,:4] {O[0, 0, :4]}  ref {ref[0, 0, :4]}")
