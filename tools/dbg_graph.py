import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2108_04315_b200 import flmisr, synth
y = synth.random_fields((4, 128, 128), 1)
sh = synth.shift_pattern(2)
pl = flmisr.Plan(k=4, lr_h=128, lr_w=128, shifts=sh, psf=synth.gaussian_psf(), n_iter=5)
yd = torch.from_numpy(y).cuda()
out = torch.empty((256, 256), device="cuda")
s = torch.cuda.current_stream()
for i in range(2):
    pl.reconstruct(yd, out=out); print("plain", i, flush=True)
pl.profile(1)
for i in range(3):
    try:
        pl.reconstruct_async(yd, out, stream=s); r = pl.finish(); print("prof", i, r["iters_run"], flush=True)
    except Exception as e:
        print("prof", i, "ERR", e, flush=True)
print(pl.profile(0))
