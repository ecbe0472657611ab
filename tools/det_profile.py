"""One C3 reconstruction (default or det mode) for an ncu capture of the loop kernel:
    DET_ROWS=24 python tools/det_profile.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_04315_b200 import flmisr, synth  # noqa: E402

lr, mag = 2048, 2
y = synth.random_fields((4, lr, lr), 2110, 0.2, 0.9)
pl = flmisr.Plan(k=4, lr_h=lr, lr_w=lr, shifts=synth.shift_pattern(mag), psf=synth.gaussian_psf(), mag=mag,
                 n_iter=20, det_rows=int(os.environ.get("DET_ROWS", "0")))
yd = torch.from_numpy(y).cuda()
for _ in range(2):
    pl.reconstruct(yd)
torch.cuda.synchronize()
print("ok", pl.loop_kernel)
