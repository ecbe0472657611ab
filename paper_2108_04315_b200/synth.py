"""Seeded synthetic inputs shared by the tests, bench.py and the oracle checks.

This module holds NONE of the method's arithmetic (no forward operator, objective,
gradient or SCG step): it only draws phantoms, PSFs, shift patterns and noisy LR stacks
with the shapes and value distributions of the paper's workloads.

* Phantom: flat-field-normalised CT transmission image x* = exp(-sum mu L) in ~[0.1, 1]
  ("8-16 MP CT projections"; aluminium cylinder P:339; QRM bar pattern P:359;
  concrete texture P:366).
* Detector stack (P:339 degradation protocol, "shifted ... followed by a 2x2 binning"):
  frame i integrates the HR truth over a centred r x r detector aperture at sampling
  lattice offset s_i = r * shift_i (whole HR px for every config), then adds i.i.d.
  N(0, sigma_n^2) noise with sigma_n = 1/255 ("N(0,1)" on the 8-bit scale).
  The aperture is a data-generation choice, distinct from the reconstruction's Gaussian
  PSF (as with real detectors, the model is not the generator).
All draws use numpy PCG64 (default_rng(seed)) in fp64 and are cast to fp32 once; the
oracle and the CUDA path consume the same fp32 bits.
"""
from __future__ import annotations

import numpy as np


def gaussian_psf(sigma: float = 0.5, size: int = 3) -> np.ndarray:
    """Normalised size x size Gaussian ("3x3 Gaussian blur"; sigma = 0.5 HR px, reading 2)."""
    r = size // 2
    ax = np.arange(-r, r + 1, dtype=np.float64)
    g = np.exp(-(ax[:, None] ** 2 + ax[None, :] ** 2) / (2.0 * sigma * sigma))
    return g / g.sum()


def delta_psf() -> np.ndarray:
    return np.ones((1, 1))


def shift_pattern(mag: int) -> np.ndarray:
    """K = mag^2 detector positions in LR px, frame 0 = (0,0) (reading 3).

    mag = 2: (0,0), (0,1/2), (1/2,1/2), (1/2,0) -- the right/down/left/up half-pixel cycle
    of P:258 read cumulatively.  mag = 3: (a/3, b/3) in raster order."""
    if mag == 2:
        return np.array([[0.0, 0.0], [0.0, 0.5], [0.5, 0.5], [0.5, 0.0]])
    return np.array([[a / mag, b / mag] for a in range(mag) for b in range(mag)], dtype=np.float64)


def phantom(H: int, W: int, seed: int) -> np.ndarray:
    """HR ground truth: x* = exp(-sum_k mu_k L_k) in ~[0.1, 1] (fp64, H x W)."""
    rng = np.random.default_rng(seed)
    v = np.arange(W, dtype=np.float64)[None, :]
    u = np.arange(H, dtype=np.float64)[:, None]
    att = np.zeros((H, W))
    # (i) vertical aluminium-like cylinders: chord length 2 sqrt(R^2 - (v - c)^2)
    for _ in range(int(rng.integers(3, 7))):
        c = rng.uniform(0.1, 0.9) * W
        R = rng.uniform(0.03, 0.12) * W
        mu = rng.uniform(0.3, 1.2) / max(W, 1) * 4.0
        chord = 2.0 * np.sqrt(np.clip(R * R - (v - c) ** 2, 0.0, None))
        att += mu * chord * np.ones((H, 1))
    # (ii) QRM-like bar block: periods 16 .. 2 HR px (up to HR Nyquist)
    by0, bx0 = int(0.08 * H), int(0.55 * W)
    bh, bw = max(int(0.25 * H), 1), max(int(0.35 * W), 1)
    periods = [16, 12, 8, 6, 4, 3, 2]
    seg = max(bw // len(periods), 1)
    for j, per in enumerate(periods):
        x0 = bx0 + j * seg
        x1 = min(x0 + seg, W)
        if x0 >= W:
            break
        cols = np.arange(x0, x1)
        bars = ((cols // max(per // 2, 1)) % 2).astype(np.float64)
        att[by0:min(by0 + bh, H), x0:x1] += 0.35 * bars[None, :]
    # (iii) a disk edge and a slanted edge
    cy, cx, rd = 0.7 * H, 0.3 * W, 0.12 * min(H, W)
    att += 0.5 * (((u - cy) ** 2 + (v - cx) ** 2) <= rd * rd)
    att += 0.25 * ((v - 0.75 * W) * np.cos(0.087) + (u - 0.75 * H) * np.sin(0.087) > 0) * (u > 0.6 * H)
    # (iv) seeded low-pass "concrete" texture: white noise smoothed by a separable box chain
    tex = rng.standard_normal((H, W))
    for _ in range(3):
        k = 5
        tex = (np.cumsum(np.pad(tex, ((0, 0), (k, 0)), mode="edge"), axis=1)[:, k:] -
               np.cumsum(np.pad(tex, ((0, 0), (k, 0)), mode="edge"), axis=1)[:, :-k]) / k
        tex = (np.cumsum(np.pad(tex, ((k, 0), (0, 0)), mode="edge"), axis=0)[k:, :] -
               np.cumsum(np.pad(tex, ((k, 0), (0, 0)), mode="edge"), axis=0)[:-k, :]) / k
    tex = tex / (np.abs(tex).max() + 1e-12)
    att += 0.15 * (tex + 1.0)
    x = np.exp(-att)
    return np.clip(x, 0.0, 1.0)


def detector_stack(truth: np.ndarray, mag: int, shifts: np.ndarray, sigma_n: float, seed: int) -> np.ndarray:
    """k x (H/mag) x (W/mag) fp64 LR stack from the HR truth (P:339 protocol, module docstring)."""
    H, W = truth.shape
    h, w = H // mag, W // mag
    if mag % 2 == 1:
        b = np.ones(mag) / mag
    else:
        b = np.concatenate([[0.5], np.ones(mag - 1), [0.5]]) / mag
    rb = len(b) // 2
    pad = rb + mag + 1
    xp = np.pad(truth, pad, mode="edge")
    # separable centred aperture, evaluated on the padded grid
    t1 = sum(b[j] * xp[:, j:xp.shape[1] - len(b) + 1 + j] for j in range(len(b)))
    t2 = sum(b[j] * t1[j:t1.shape[0] - len(b) + 1 + j, :] for j in range(len(b)))
    # t2[i, j] is the aperture centred at padded index (i + rb, j + rb) = HR (i + rb - pad, ...)
    off = pad - rb
    rng = np.random.default_rng(seed + 7919)
    out = np.empty((len(shifts), h, w))
    for i, (dy, dx) in enumerate(shifts):
        sy, sx = int(np.floor(mag * dy + 1e-9)), int(np.floor(mag * dx + 1e-9))
        rows = off + sy + mag * np.arange(h)
        cols = off + sx + mag * np.arange(w)
        out[i] = t2[np.ix_(rows, cols)]
    out += sigma_n * rng.standard_normal(out.shape)
    return out


def make_stack(lr: int, mag: int, seed: int, sigma_n: float = 1.0 / 255.0, lr_w: int | None = None,
               shifts=None):
    """(stack fp32 k x lr x lr_w, shifts k x 2, truth fp64) for a BASELINE config.  Fractional HR
    phases of `shifts` are sampled at the floor lattice position (inputs only need the workload's
    shape and statistics; the reconstruction models the given shifts exactly)."""
    lr_w = lr if lr_w is None else lr_w
    sh = shift_pattern(mag) if shifts is None else np.asarray(shifts, dtype=np.float64)
    truth = phantom(mag * lr, mag * lr_w, seed)
    y = detector_stack(truth, mag, sh, sigma_n, seed).astype(np.float32)
    return y, sh, truth


def box_aperture_psf(mag: int) -> np.ndarray:
    """The detector aperture detector_stack integrates over, as a centred odd PSF on the HR grid
    (reading 1: a box aperture, when wanted, is part of the PSF argument): outer(b, b) with
    b = [1/2, 1, ..., 1, 1/2] / mag for even mag (mag + 1 taps), ones(mag) / mag for odd mag."""
    b = np.ones(mag) / mag if mag % 2 else np.concatenate([[0.5], np.ones(mag - 1), [0.5]]) / mag
    return np.outer(b, b)


# ---- "natural-like" ground truths for the SR-vs-interpolation quality protocol (tab:natural,
# P:388-395; SPEC AC6 S:533 "natural/synthetic images <= 1024^2").  Values in [0.05, 0.95].
def dead_leaves(n: int, seed: int, rmin: float = 2.0, rmax: float = 80.0, count: int = 6000) -> np.ndarray:
    """Occluding discs with power-law radii (density ~ r^-3) and uniform grey levels: the classic
    scale-invariant model of natural-image statistics (edges at every scale and orientation)."""
    rng = np.random.default_rng(seed)
    img = np.full((n, n), np.nan)
    u = rng.uniform(size=count)
    rad = (rmin ** -2 - u * (rmin ** -2 - rmax ** -2)) ** -0.5
    for k in range(count):
        cy, cx = rng.uniform(-rmax, n + rmax, 2)
        g = rng.uniform(0.05, 0.95)
        r = rad[k]
        y0, y1 = int(max(0, cy - r)), int(min(n, cy + r + 1))
        x0, x1 = int(max(0, cx - r)), int(min(n, cx + r + 1))
        if y0 >= y1 or x0 >= x1:
            continue
        yy, xx = np.mgrid[y0:y1, x0:x1]
        sub = img[y0:y1, x0:x1]
        m = ((yy - cy) ** 2 + (xx - cx) ** 2 <= r * r) & np.isnan(sub)
        sub[m] = g
    img[np.isnan(img)] = 0.5
    return img


def pink_noise(n: int, seed: int, beta: float = 1.0) -> np.ndarray:
    """Gaussian texture with a 1/f^beta amplitude spectrum (natural images: beta ~ 1)."""
    rng = np.random.default_rng(seed)
    f = np.fft.fftfreq(n)
    r = np.hypot(f[None, :], f[:, None])
    r[0, 0] = 1.0
    spec = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / r ** beta
    spec[0, 0] = 0.0
    img = np.real(np.fft.ifft2(spec))
    img = (img - img.min()) / (img.max() - img.min())
    return 0.05 + 0.9 * img


def resolution_chart(n: int, seed: int) -> np.ndarray:
    """Siemens star (36 cycles), bar groups of periods 16 .. 2 HR px (the QRM bar pattern)
    and random small rectangles (text-like detail) on a grey background."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:n, 0:n].astype(np.float64)
    img = np.full((n, n), 0.5)
    cy = cx = 0.3 * n
    th = np.arctan2(yy - cy, xx - cx)
    rr = np.hypot(yy - cy, xx - cx)
    inside = rr < 0.25 * n
    img[inside] = ((np.sin(36 * th) > 0) * 0.7 + 0.15)[inside]
    x = int(0.6 * n)
    for i, per in enumerate([16, 12, 8, 6, 4, 3, 2]):
        y0 = int(0.05 * n + i * 0.13 * n)
        band = ((np.arange(int(0.35 * n)) // (per / 2)) % 2) * 0.7 + 0.15
        img[y0:y0 + int(0.1 * n), x:x + len(band)] = band[None, :]
    for _ in range(int(0.16 * n)):
        y0, x0 = rng.integers(int(0.6 * n), n - 10), rng.integers(0, int(0.55 * n))
        h, w = rng.integers(2, 9, 2)
        img[y0:y0 + h, x0:x0 + w] = rng.uniform(0.05, 0.95)
    return img


def random_fields(shape, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """Uniform O(1) fp32 test field (per-operator parity inputs)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, size=shape).astype(np.float32)


# BASELINE.json configs: name -> (lr, mag, n_iter, seed)
CONFIGS = {
    "C1": dict(lr=64, mag=2, n_iter=20, seed=2108),
    "C2": dict(lr=1024, mag=2, n_iter=50, seed=2109),
    "C3": dict(lr=2048, mag=2, n_iter=20, seed=2110),
    "C4": dict(lr=2048, mag=3, n_iter=20, seed=2111),
    # the paper's largest tab:runtime workload: 4 LR 4096^2 -> x2 (67 MP HR), 20 iterations
    "C6": dict(lr=4096, mag=2, n_iter=20, seed=2113),
    # general-geometry path at C3 size: K = 4 frames at quarter-pixel detector
    # positions (fractional HR phases, a different composed kernel per frame)
    "G3": dict(lr=2048, mag=2, n_iter=20, seed=2112,
               shifts=((0.0, 0.0), (0.25, 0.5), (0.5, 0.25), (0.75, 0.75))),
}
