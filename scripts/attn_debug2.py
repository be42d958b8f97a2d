import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.attn_debug import run  # noqa
from paper_2508_15601_b200 import synth  # noqa
for G in [1, 2, 4, 8]:
    p = synth.kv_decode_problem(1, G, 1, 128, 64, [2], 8, seed=3)
    p["vq"][:] = 100; p["vz"][:] = 0; p["vs"][:] = 1.0
    rf, O, ref = run(p)
    print("G", G, "per-head O[:, 0:3]:", [O[0, h, :3].tolist() for h in range(G)])
    p = synth.kv_decode_problem(1, G, 1, 128, 64, [2], 8, seed=3)
    rf, O, ref = run(p)
    print("   random per-head relerr:", [float(np.linalg.norm(O[0, h] - ref[0, h]) / np.linalg.norm(ref[0, h])) for h in range(G)])
