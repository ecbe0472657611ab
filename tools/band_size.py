"""Per-phase time of the single-GPU loop kernel on one row band's worth of work: HR rows x 4096 for
rows = 4096 / g (g = 1, 2, 4, 8) -- the compute a rank of a g-GPU row partition of C3 does per phase,
without the exchange.  Prints one JSON line (median of --reps reconstructions, CUDA events)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_04315_b200 import flmisr, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
res = {}
for g in (1, 2, 4, 8):
    lr_h, lr_w = 2048 // g, 2048
    y = synth.random_fields((4, lr_h, lr_w), 2110, 0.2, 0.9)
    yd = torch.from_numpy(y).cuda()
    out = torch.empty((2 * lr_h, 2 * lr_w), device="cuda")
    pl = flmisr.Plan(k=4, lr_h=lr_h, lr_w=lr_w, shifts=synth.shift_pattern(2), psf=synth.gaussian_psf(), n_iter=20)
    for _ in range(3):
        _, rep = pl.reconstruct(yd, out=out)
    pl.profile(1)
    for _ in range(a.reps):
        pl.reconstruct(yd, out=out)
    p = pl.profile(0)
    ms = p["value_grad"]["ms"] / p["value_grad"]["launches"]   # the loop kernel (prof_mode 1)
    phases = 1 + 2 * rep["accepted"] + (20 - rep["accepted"])
    res[f"rows{2 * lr_h}"] = {"loop_ms": ms, "phases": phases, "us_per_phase": ms * 1e3 / phases}
    pl.destroy()
base = res["rows4096"]["us_per_phase"]
for k, v in res.items():
    v["ideal_us"] = base * int(k[4:]) / 4096
print(json.dumps(res), flush=True)
