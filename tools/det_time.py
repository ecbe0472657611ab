"""Median ms of one C3 reconstruction (device-resident input), default or det mode:
    DET_ROWS=6 FLMISR_EDGE_RATIO=1.8 python tools/det_time.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_04315_b200 import flmisr, synth  # noqa: E402

lr, mag = 2048, 2
y = synth.random_fields((4, lr, lr), 2110, 0.2, 0.9)
T = int(os.environ.get("DET_ROWS", "0"))
pl = flmisr.Plan(k=4, lr_h=lr, lr_w=lr, shifts=synth.shift_pattern(mag), psf=synth.gaussian_psf(), mag=mag,
                 n_iter=20, det_rows=T)
yd = torch.from_numpy(y).cuda()
out = torch.empty((mag * lr, mag * lr), device="cuda")
for _ in range(3):
    pl.reconstruct(yd, out=out)
torch.cuda.synchronize()
t = []
for _ in range(10):
    t0 = time.perf_counter()
    pl.reconstruct(yd, out=out)
    torch.cuda.synchronize()
    t.append(time.perf_counter() - t0)
print(f"T={T} ratio={os.environ.get('FLMISR_EDGE_RATIO', '-')} ms={np.median(t) * 1e3:.3f}", flush=True)
