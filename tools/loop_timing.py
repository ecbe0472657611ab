"""Phase timeline of the persistent SCG loop kernel (diagnostic build -DFLMISR_TIMING):
    FLMISR_LIB=build_variants/lib_timing.so python tools/loop_timing.py
Per phase: spread of CTA work ends, last arrival, release (first/last CTA), reduction+scalars done."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_04315_b200 import flmisr, synth  # noqa: E402

c = synth.CONFIGS[os.environ.get("CFG", "C3")]
lr, mag = c["lr"], c["mag"]
y = synth.random_fields((mag * mag, lr, lr), c["seed"], 0.2, 0.9)
pl = flmisr.Plan(k=mag * mag, lr_h=lr, lr_w=lr, shifts=synth.shift_pattern(mag), psf=synth.gaussian_psf(),
                 mag=mag, n_iter=c["n_iter"])
assert pl.loop_kernel == 1
yd = torch.from_numpy(y).cuda()
for _ in range(3):
    pl.reconstruct(yd)
torch.cuda.synchronize()
n = 64 * 256 * 4
buf = (C.c_ulonglong * n)()
assert flmisr._lib.flmisr_debug_loop_timing(buf, n) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(64, 256, 4).astype(np.int64)
G = int((a[0, :, 0] > 0).sum())
a = a[:, :G, :]
nph = int((a[:, 0, 0] > 0).sum())
a = a[:nph]
t0 = a[0, :, 0].min()
prev_done = None
rows = []
for ph in range(nph):
    we, ar, rl, dn = [(a[ph, :, k] - t0) / 1e3 for k in range(4)]
    start = prev_done if prev_done is not None else 0.0
    rows.append((ph, we.min() - start, we.max() - start, ar.max() - we.max(), rl.max() - ar.max(),
                 dn.max() - rl.max()))
    prev_done = dn.max()
print("phase  first-work-end  last-work-end  (after prev release+scalars)  last-arrive-lag  release-lag  sum+scalar")
for r in rows[:6] + rows[-3:]:
    print("%3d %12.1f %12.1f %14.1f %12.1f %12.1f" % r)
m = np.array(rows)[1:]
print("mean over phases: work span %.1f..%.1f us, arrival lag %.2f, release lag %.2f, sum+scalar %.2f" %
      (m[:, 1].mean(), m[:, 2].mean(), m[:, 3].mean(), m[:, 4].mean(), m[:, 5].mean()))
# per-CTA work-end distribution (relative to the previous phase's release), averaged over phases
rel = []
for ph in range(1, nph):
    start = ((a[ph - 1, :, 3] - t0) / 1e3).max()
    rel.append((a[ph, :, 0] - t0) / 1e3 - start)
rel = np.array(rel).mean(axis=0)
q = np.percentile(rel, [0, 10, 25, 50, 75, 90, 100])
print("CTA work end (mean over phases) percentiles:", np.round(q, 1))
o = np.argsort(-rel)[:12]
print("slowest CTAs:", [(int(i), round(float(rel[i]), 1)) for i in o])
ph_vg = [ph for ph in range(1, nph) if ph % 2 == 0]
ph_uc = [ph for ph in range(1, nph) if ph % 2 == 1]
for name, phs in (("uc", ph_uc), ("vg", ph_vg)):
    r = []
    for ph in phs:
        start = ((a[ph - 1, :, 3] - t0) / 1e3).max()
        r.append((a[ph, :, 0] - t0) / 1e3 - start)
    r = np.array(r).mean(axis=0)
    print(name, "CTA work end percentiles:", np.round(np.percentile(r, [0, 10, 50, 90, 100]), 1),
          "slowest:", [int(i) for i in np.argsort(-r)[:6]])
