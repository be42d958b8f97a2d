"""Medium M (tiled kernel): split-K sweep.   python scripts/mid_sweep.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from quick_perf import SHAPES, run  # noqa: E402

for name in ("qkv", "o", "gate_up", "down"):
    N, K = SHAPES[name]
    for M in (128, 256, 512):
        row = []
        for tile in ((128,) if M <= 128 else (128, 256)):
            for split in (1, 2, 3, 4, 6, 8):
                try:
                    r = run(M, N, K, reps=30, tile=tile, split=split)
                    row.append(f"t{tile}s{split}:{r['us']:.1f}")
                except Exception as e:  # noqa: BLE001
                    row.append(f"t{tile}s{split}:X")
        print(name, M, " ".join(row), flush=True)
