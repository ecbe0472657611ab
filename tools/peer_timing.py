"""Phase timeline of the peer band loop (diagnostic build -DFLMISR_TIMING), C3 as g virtual bands:
    FLMISR_LIB=build_variants/lib_timing.so python tools/peer_timing.py [g]
Per phase and band: CTA work-end spread, last arrival, release seen (first/last CTA), in us."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2108_04315_b200 import flmisr, synth  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lr, mag = 2048, 2
y = synth.random_fields((4, lr, lr), 2110, 0.2, 0.9)
yd = torch.from_numpy(y).cuda()
pls = [flmisr.Plan(k=4, lr_h=lr, lr_w=lr, shifts=synth.shift_pattern(2), psf=synth.gaussian_psf(), mag=2, n_iter=20,
                   rank=h, world=g, virtual=True) for h in range(g)]
for _ in range(3):
    flmisr.reconstruct_virtual_peer(pls, yd)
n = 64 * 256 * 4
buf = (C.c_ulonglong * n)()
assert flmisr._lib.flmisr_debug_loop_timing(buf, n) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(64, 256, 4).astype(np.int64)
G = int((a[0, :, 0] > 0).sum())
ctas = G // g
a = a[:, :G, :]
nph = int((a[:, 0, 0] > 0).sum())
t0 = a[0, :, 0].min()
print(f"g={g} ctas/band={ctas} phases={nph}")
for ph in range(min(nph, 12)):
    line = [f"ph{ph:2d}"]
    for l in range(g):
        sl = slice(l * ctas, (l + 1) * ctas)
        we, ar, rl, dn = [(a[ph, sl, k] - t0) / 1e3 for k in range(4)]
        line.append(f"b{l}: work {we.min():8.1f}..{we.max():8.1f} arr {ar.max():8.1f} rel {rl.min():8.1f}..{rl.max():8.1f}")
    print(" | ".join(line))
