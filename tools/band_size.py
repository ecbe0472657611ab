"""Per-phase time of the single-GPU loop kernel on one row band's worth of work: HR rows x W for
rows = H / g (g = 1, 2, 4, 8) -- the compute a rank of a g-GPU row partition of the config does per
phase (including the on-chip grid barrier), without the cross-GPU exchange.  Prints one JSON line
(mean over --reps reconstructions, CUDA events)."""
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
ap.add_argument("--config", default="C3", help="C3 (LR 2048^2, x2), C4 (LR 2048^2, x3) or C6 (LR 4096^2, x2)")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
mag, LR = cfg["mag"], cfg["lr"]
res = {"config": a.config}
for g in (1, 2, 4, 8):
    lr_h, lr_w = LR // g, LR
    y = synth.random_fields((mag * mag, lr_h, lr_w), 2110, 0.2, 0.9)
    yd = torch.from_numpy(y).cuda()
    out = torch.empty((mag * lr_h, mag * lr_w), device="cuda")
    pl = flmisr.Plan(k=mag * mag, lr_h=lr_h, lr_w=lr_w, shifts=synth.shift_pattern(mag), psf=synth.gaussian_psf(),
                     mag=mag, n_iter=20)
    for _ in range(3):
        _, rep = pl.reconstruct(yd, out=out)
    pl.profile(1)
    for _ in range(a.reps):
        pl.reconstruct(yd, out=out)
    p = pl.profile(0)
    ms = p["value_grad"]["ms"] / p["value_grad"]["launches"]   # the loop kernel (prof_mode 1)
    phases = 1 + 2 * rep["accepted"] + (20 - rep["accepted"])
    res[f"g{g}"] = {"rows": mag * lr_h, "loop_ms": ms, "phases": phases, "us_per_phase": ms * 1e3 / phases}
    pl.destroy()
base = res["g1"]["us_per_phase"]
for g in (1, 2, 4, 8):
    v = res[f"g{g}"]
    v["ideal_us"] = base / g
    v["speedup_compute_only"] = base / v["us_per_phase"]
print(json.dumps(res), flush=True)
