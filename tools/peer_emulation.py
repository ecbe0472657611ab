"""Cost of the peer-memory band protocol on one B200: C3 (HR 4096 x 4096,
20 passes) as 1 band (the persistent loop kernel) and as g = 2, 4, 8 virtual peer bands in one
cooperative launch.  Each band gets 148/g SMs, so the g-band run does the same total work on the same
SMs plus g-band synchronisation per phase; the difference per phase is the protocol's on-chip cost.
With --det-rows T every run uses det mode (fixed tiles of T rows, exact sums): the g-band images must
then equal the 1-band image bit for bit ("bit_identical").
    python tools/peer_emulation.py [--reps 10] [--det-rows T]   -> one JSON line"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2108_04315_b200 import flmisr, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--lr", type=int, default=2048)
ap.add_argument("--det-rows", type=int, default=0)
a = ap.parse_args()
lr, mag, n_iter = a.lr, 2, 20
sh = synth.shift_pattern(mag)
y = synth.random_fields((4, lr, lr), 2110, 0.2, 0.9)
yd = torch.from_numpy(y).cuda()
out = torch.empty((mag * lr, mag * lr), device="cuda")
res = {"workload": f"K=4 LR {lr}x{lr} -> x2, {n_iter} SCG passes", "reps": a.reps, "det_rows": a.det_rows}
DK = dict(det_rows=a.det_rows)


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    return float(np.median(t)) * 1e3, r


one = flmisr.Plan(k=4, lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=n_iter, **DK)
ms1, (_, r1) = timed(lambda: one.reconstruct(yd, out=out))
img1 = out.cpu().numpy().copy()
phases = 1 + 2 * r1["accepted"] + (n_iter - r1["accepted"])
res["g1"] = {"ms": ms1, "phases": phases}
for g in (2, 4, 8):
    pls = [flmisr.Plan(k=4, lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=n_iter,
                       rank=h, world=g, virtual=True, **DK) for h in range(g)]
    msg, (_, rg) = timed(lambda: flmisr.reconstruct_virtual_peer(pls, yd, out=out))
    res[f"g{g}"] = {"ms": msg, "accepted": rg["accepted"], "same_trajectory": rg["accepted"] == r1["accepted"],
                    "extra_us_per_phase": (msg - ms1) * 1e3 / phases,
                    "bit_identical": bool(np.array_equal(out.cpu().numpy(), img1)
                                          and np.array_equal(rg["trace"], r1["trace"]))}
    for p in pls:
        p.destroy()
print(json.dumps(res), flush=True)
