"""Helpers shared by the GPU parity tests (test code; no method arithmetic)."""

import numpy as np
import torch


def to_dev(d, act_dtype=None):
    """synth dict (numpy) -> device tensors for the C ABI."""
    act_dtype = act_dtype or d.get("act_dtype", "bf16")
    tdt = torch.bfloat16 if act_dtype == "bf16" else torch.float16
    return dict(
        A=torch.from_numpy(np.ascontiguousarray(d["A"], dtype=np.float32)).to(tdt).cuda(),
        q=torch.from_numpy(np.ascontiguousarray(d["q"])).cuda(),
        s=torch.from_numpy(np.ascontiguousarray(d["s"])).cuda(),
        z=torch.from_numpy(np.ascontiguousarray(d["z"])).cuda(),
    )


def to_np64(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def bits16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
