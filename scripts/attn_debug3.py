import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from scripts.attn_debug import run  # noqa
from paper_2508_15601_b200 import synth  # noqa
p = synth.kv_decode_problem(1, 1, 1, 128, 64, [20], 8, seed=3)
p["Q"][:] = 0
rf, O, ref = run(p)
err = np.abs(O[0, 0] - ref[0, 0])
print("bad channels:", np.nonzero(err > 0.02)[0].tolist())
# which reference channel does each output channel match?
from oracle.attention import dequant_kv
V = dequant_kv(p["vq"][0, 0, :20], p["vs"][0, 0, :20], p["vz"][0, 0, :20]).mean(axis=0)
match = [int(np.argmin(np.abs(V - O[0, 0, d]))) for d in range(128)]
print("output channel -> matching ref channel:", match)
