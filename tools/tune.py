"""Per-kernel timing of C3 reconstructions for tuning builds (FLMISR_LIB, FLMISR_SEG_ROWS, ...).

    FLMISR_LIB=build_variants/lib_x.so FLMISR_SEG_ROWS=31 python tools/tune.py [--config C3] [--reps 10]
Prints one JSON line: avg value+gradient / update+curvature launch us and whole-reconstruction ms."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_04315_b200 import flmisr, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C3")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
lr, mag = c["lr"], c["mag"]
y = synth.random_fields((mag * mag, lr, lr), c["seed"], 0.2, 0.9)
sh = synth.shift_pattern(mag)
pl = flmisr.Plan(k=mag * mag, lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=c["n_iter"])
yd = torch.from_numpy(y).cuda()
out = torch.empty((pl.H, pl.W), device="cuda")
flush = torch.empty(128 * 1024 * 1024, device="cuda")
for _ in range(3):
    pl.reconstruct(yd, out=out)
pl.profile(1)
for _ in range(a.reps):
    flush.zero_()
    pl.reconstruct(yd, out=out)
p = pl.profile(0)
out = {"lib": os.path.basename(flmisr.LIB_PATH), "seg_rows": os.environ.get("FLMISR_SEG_ROWS", "auto"),
       "loop_kernel": pl.loop_kernel, "recon_ms": p["reconstruct"]["ms"] / p["reconstruct"]["launches"]}
if p["update_curv"]["launches"]:
    out.update(vg_us=1000 * p["value_grad"]["ms"] / p["value_grad"]["launches"],
               uc_us=1000 * p["update_curv"]["ms"] / p["update_curv"]["launches"])
else:
    out.update(loop_ms=p["value_grad"]["ms"] / p["value_grad"]["launches"])
print(json.dumps(out), flush=True)
