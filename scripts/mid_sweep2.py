"""Medium M: tiled kernel vs the NT=128/256 stream-K kernel (forced).   python scripts/mid_sweep2.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from quick_perf import SHAPES, run  # noqa: E402

for name in ("qkv", "o", "gate_up", "down"):
    N, K = SHAPES[name]
    for M in (128, 256, 512, 1024):
        row = []
        for tile, split in ((128, 1), (128, -148), (128, -296), (256, 1), (256, -148)):
            if M <= 128 and tile == 256:
                continue
            try:
                r = run(M, N, K, reps=30, tile=tile, split=split)
                row.append(f"t{tile}s{split}:{r['us']:.1f}")
            except Exception as e:  # noqa: BLE001
                row.append(f"t{tile}s{split}:X")
        print(name, M, " ".join(row), flush=True)
