"""Per-warp start/end times of the last k_vg_stream launch (diagnostic build -DFLMISR_TIMING):
    FLMISR_LIB=build_variants/lib_timing.so python tools/warp_timing.py"""
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
                 mag=mag, n_iter=2)
yd = torch.from_numpy(y).cuda()
for _ in range(3):
    pl.reconstruct(yd)
torch.cuda.synchronize()
n = 3 * 16384
buf = (C.c_ulonglong * n)()
assert flmisr._lib.flmisr_debug_warp_timing(buf, n) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 3).astype(np.int64)
live = ((a[:, 2] >> 17) & 1) == 1
a = a[live]
t0 = a[:, 0].min()
st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
dur = en - st
sm = a[:, 2] & 0xffff
border = ((a[:, 2] >> 16) & 1) == 1
print(f"warps {len(a)}  kernel span {en.max():.1f} us")
for name, v in (("start", st), ("end", en), ("duration", dur)):
    q = np.percentile(v, [0, 5, 25, 50, 75, 95, 100])
    print(f"{name:9s} " + " ".join(f"{x:7.1f}" for x in q))
print(f"border warps {border.sum()}: median dur {np.median(dur[border]):.1f} vs interior {np.median(dur[~border]):.1f}")
smd = np.array([np.median(dur[sm == s]) for s in range(sm.max() + 1) if (sm == s).any()])
sme = np.array([en[sm == s].max() for s in range(sm.max() + 1) if (sm == s).any()])
print("per-SM median duration: min %.1f max %.1f; per-SM last end: min %.1f max %.1f" % (smd.min(), smd.max(), sme.min(), sme.max()))
half = len(smd) // 2
print("SM halves median duration: %.1f / %.1f" % (np.median(smd[:half]), np.median(smd[half:])))
strip = (a[:, 2] >> 20) & 0xffff
row0 = (a[:, 2] >> 36) & 0xfffff
inter = ~border
q = np.percentile(dur[inter], [0, 5, 25, 50, 75, 95, 100])
print("interior duration " + " ".join(f"{x:7.1f}" for x in q))
# per-SM composition
nb = np.array([(border & (sm == s)).sum() for s in range(sm.max() + 1) if (sm == s).any()])
for k in sorted(set(nb)):
    print(f"SMs with {k} border warps: {np.sum(nb == k):3d}, median interior-warp duration on them "
          f"{np.median(np.concatenate([dur[(sm == s) & inter] for s in np.unique(sm)[nb == k]] or [np.zeros(1)])):.1f}")
# by strip parity / position
for name, m in (("strip<17", strip < 17), ("strip>=17", strip >= 17), ("row0<2048", row0 < 2048), ("row0>=2048", row0 >= 2048)):
    print(f"interior {name}: median {np.median(dur[inter & m]):.1f}")
# SM id correlation
sids = np.unique(sm)
med = np.array([np.median(dur[(sm == s) & inter]) if ((sm == s) & inter).any() else np.nan for s in sids])
print("interior median by SM id deciles:", " ".join(f"{np.nanmedian(med[i::10]):.1f}" for i in range(10)))
print("per-SM interior median, sorted:", np.round(np.sort(med[~np.isnan(med)])[::15], 1))
nst = strip.max()
edge = (strip == 0) | (strip == nst)
rows_per = np.diff(np.unique(row0))
print(f"border classes: edge strips median {np.median(dur[edge]):.1f} (n={edge.sum()}), "
      f"interior-strip border segs median {np.median(dur[border & ~edge]):.1f} (n={(border & ~edge).sum()}), "
      f"interior median {np.median(dur[~border]):.1f}")
print(f"strip 0 median {np.median(dur[strip == 0]):.1f}, last strip median {np.median(dur[strip == nst]):.1f}")
o = np.argsort(-dur)[:8]
print("slowest:", [(int(strip[i]), int(row0[i]), int(sm[i]), round(float(dur[i]), 1)) for i in o])
cb = (C.c_ulonglong * (3 * 2048))()
assert flmisr._lib.flmisr_debug_cta_timing(cb, 3 * 2048) == 0
ct = np.frombuffer(cb, dtype=np.uint64).reshape(-1, 3).astype(np.int64)
ct = ct[ct[:, 0] > 0]
e0 = ct[:, 0].min()
print(f"CTAs {len(ct)}: entry spread {(ct[:, 0].max() - e0) / 1e3:.1f} us; first warp start after first entry "
      f"{(t0 - e0) / 1e3:.1f} us; last warp end {(a[:, 1].max() - e0) / 1e3:.1f} us; last CTA reduction end "
      f"{(ct[:, 1].max() - e0) / 1e3:.1f} us; scalar logic end {(ct[:, 2].max() - e0) / 1e3:.1f} us")
idle = (en.max() - en).mean() / en.max()
print(f"mean idle tail fraction {idle:.3f}; mean start delay fraction {st.mean() / en.max():.3f}")
