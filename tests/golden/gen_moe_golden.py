"""Freeze small fused-MoE / alignment vectors from the CPU oracle.

The reference has no fused-MoE forward and no alignment code,
so these vectors are our own pin: they freeze oracle/moe_ref.py so that a
later change to it is caught.  Run HERE:  python tests/golden/gen_moe_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.moe_ref import fused_moe_ref, moe_align_ref  # noqa: E402
from tests._util import random_moe  # noqa: E402

out = {}
for tag, (S, H, I, E, k, mode) in {"a": (5, 64, 64, 4, 2, "dup"), "b": (9, 128, 64, 6, 3, None)}.items():
    x, w1, w2, w, ids = random_moe(S, H, I, E, k, seed=11, dup=mode == "dup")
    y = fused_moe_ref(x, w1, w2, w, ids)
    for key, val in dict(x=x, w1=w1, w2=w2, w=w, ids=ids, out=y).items():
        out[f"{tag}_{key}"] = val
    h, s, t, npp = moe_align_ref(ids, E, 4)
    out[f"{tag}_hist"], out[f"{tag}_sorted"], out[f"{tag}_tiles"] = h, s, t
np.savez_compressed(Path(__file__).with_name("moe_small.npz"), **out)
print("wrote moe_small.npz")
