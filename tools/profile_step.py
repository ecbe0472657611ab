"""Minimal driver for ncu / compute-sanitizer: a few C3 (or --config) reconstructions, nothing else."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_04315_b200 import flmisr, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--n-iter", type=int, default=None)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
n_iter = a.n_iter if a.n_iter is not None else c["n_iter"]
lr, mag = c["lr"], c["mag"]
import numpy as np  # noqa: E402
# cheap synthetic stack (phantom generation is irrelevant for profiling): smooth field + noise
y = synth.random_fields((len(c.get("shifts", ())) or mag * mag, lr, lr), c["seed"], 0.2, 0.9)
sh = np.asarray(c["shifts"], dtype=np.float64) if "shifts" in c else synth.shift_pattern(mag)
pl = flmisr.Plan(k=len(sh), lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=n_iter)
yd = torch.from_numpy(y).cuda()
for _ in range(a.reps):
    hr, rep = pl.reconstruct(yd)
torch.cuda.synchronize()
print("ok", rep["iters_run"], rep["accepted"])
