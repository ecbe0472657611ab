"""Small reconstructions on every kernel family, for compute-sanitizer (memcheck / racecheck):
    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_04315_b200 import flmisr, synth  # noqa: E402

G3SH = np.array([[0.0, 0.0], [0.25, 0.5], [0.5, 0.25], [0.75, 0.75]])
cases = {
    "fast_stream": (40, 64, synth.shift_pattern(2), 2),
    "per_phase": (40, 64, G3SH, 4),
    "general_fused": (21, 30, np.array([[0, 0], [0.5, 0.5], [0.3, 0.1]]), 3),
    "tiled": (19, 21, synth.shift_pattern(2), 1),
}
for name, (lh, lw, sh, fp) in cases.items():
    truth = synth.phantom(2 * lh, 2 * lw, seed=5)
    y = synth.detector_stack(truth, 2, sh, 1 / 255, seed=5).astype(np.float32)
    pl = flmisr.Plan(k=len(sh), lr_h=lh, lr_w=lw, shifts=sh, psf=synth.gaussian_psf(), n_iter=4)
    hr, rep = pl.reconstruct(torch.from_numpy(y).cuda())
    torch.cuda.synchronize()
    print(name, "fast_path", pl.fast_path, "loop", pl.loop_kernel, "accepted", rep["accepted"], flush=True)
    pl.destroy()
# two virtual peer bands (one cooperative launch) and the virtual copies group
sh = synth.shift_pattern(2)
y = synth.detector_stack(synth.phantom(96, 128, seed=6), 2, sh, 1 / 255, seed=6).astype(np.float32)
yd = torch.from_numpy(y).cuda()
pls = [flmisr.Plan(k=4, lr_h=48, lr_w=64, shifts=sh, psf=synth.gaussian_psf(), n_iter=4, rank=h, world=2,
                   virtual=True) for h in range(2)]
flmisr.reconstruct_virtual_peer(pls, yd)
flmisr.reconstruct_virtual(pls, yd)
torch.cuda.synchronize()
print("bands ok", flush=True)
