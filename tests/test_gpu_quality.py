"""Multi-image interpolation fusion on the GPU (tab:runtime's interpolation row) and the
quality margin of FL-MISR over it (SPEC AC6, the tab:natural protocol P:388-395).

Protocol: three natural-like ground truths of 384^2 (<= 1024^2) -- dead leaves (occluding discs
with power-law radii), 1/f texture, resolution chart (Siemens star + bar groups down to 2 px);
LR stacks by the P:339 degradation (shift, r x r detector aperture, N(0, 1/255^2) noise) at 2x with
4 frames and 3x with 9 frames; FL-MISR with the paper's parameters (lambda 0.05, alpha 0.4, 20 SCG
passes) and the detector aperture as the PSF (reading 1).  Bar: PSNR margin >= 1.0 dB on every image
and SSIM strictly higher (the paper's margins: +1.41 .. +6.62 dB)."""
import numpy as np
import pytest

from paper_2108_04315_b200 import synth
from quality import psnr, ssim

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_04315_b200 import flmisr  # noqa: E402


@pytest.mark.parametrize("mag", [2, 3])
def test_interp_fusion_matches_oracle(orc, mag):
    """flmisr_interp_fuse (product entry) and the debug op are copies of LR pixels: bit-exact."""
    lr = 40
    sh = synth.shift_pattern(mag)
    y = synth.random_fields((mag * mag, lr, lr + 4), 80)
    pl = flmisr.Plan(k=mag * mag, lr_h=lr, lr_w=lr + 4, shifts=sh, psf=synth.gaussian_psf(), mag=mag)
    yd = torch.from_numpy(y).cuda()
    out = torch.zeros((pl.H, pl.W), device="cuda")
    pl.debug(flmisr.OP_INTERP, lr=yd, out=out)
    pb = orc.Problem(k=mag * mag, lr_h=lr, lr_w=lr + 4, shifts=sh, psf=synth.gaussian_psf(), mag=mag)
    ref = orc.interp_fuse(pb, y.astype(np.float64)).astype(np.float32)
    np.testing.assert_array_equal(out.cpu().numpy(), ref)
    np.testing.assert_array_equal(pl.interp_fuse(yd).cpu().numpy(), ref)


def test_interp_fuse_entry_general_path(orc):
    """General geometry (two integer phases + one fractional): inserted sites exact, the rest bilinear."""
    sh = np.array([[0, 0], [0.5, 0.5], [0.3, 0.1]])
    y = synth.random_fields((3, 21, 19), 81)
    pl = flmisr.Plan(k=3, lr_h=21, lr_w=19, shifts=sh, psf=synth.gaussian_psf(), mag=2)
    assert pl.fast_path in (0, 3)
    got = pl.interp_fuse(torch.from_numpy(y).cuda()).cpu().numpy()
    pb = orc.Problem(k=3, lr_h=21, lr_w=19, shifts=sh, psf=synth.gaussian_psf(), mag=2)
    np.testing.assert_allclose(got, orc.interp_fuse(pb, y.astype(np.float64)), rtol=0, atol=2e-6)


@pytest.mark.parametrize("fast", [True, False])
def test_x0_mode_interpolation_start(orc, fast):
    """x0_mode = 1: the SCG starts from the interpolation fusion image; the oracle started from its own
    interp_fuse image agrees to the final-image bar (1e-3) with the same accept sequence."""
    lr, mag = 48, 2
    sh = synth.shift_pattern(2) if fast else np.array([[0, 0], [0.5, 0.5], [0.0, 0.5], [0.3, 0.2]])
    truth = synth.phantom(mag * lr, mag * lr, seed=83)
    y = synth.detector_stack(truth, mag, sh, 1 / 255, seed=83).astype(np.float32)
    pl = flmisr.Plan(k=len(sh), lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=12,
                     x0_mode=1)
    assert (pl.fast_path == 2) == fast
    hr, rep = pl.reconstruct(torch.from_numpy(y).cuda())
    pb = orc.Problem(k=len(sh), lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag)
    y64 = y.astype(np.float64)
    xo, tr, st = orc.scg(pb, y64, 12, x0=orc.interp_fuse(pb, y64))
    h = hr.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(h - xo) <= 1e-3 * np.linalg.norm(xo)
    np.testing.assert_array_equal(rep["trace"][:, 5], tr[:, 5])
    np.testing.assert_allclose(rep["trace"][0, 1], tr[0, 1], rtol=1e-5)   # f0 = J(interp image)


IMAGES = {
    "dead_leaves": lambda n: synth.dead_leaves(n, 3),
    "pink_noise": lambda n: synth.pink_noise(n, 7),
    "chart": lambda n: synth.resolution_chart(n, 4),
}


@pytest.mark.parametrize("name", list(IMAGES))
@pytest.mark.parametrize("mag", [2, 3])
def test_flmisr_beats_interpolation_ac6(name, mag):
    n = 384
    truth = IMAGES[name](n)
    sh = synth.shift_pattern(mag)
    y = synth.detector_stack(truth, mag, sh, 1 / 255, seed=11).astype(np.float32)
    lr = n // mag
    pl = flmisr.Plan(k=mag * mag, lr_h=lr, lr_w=lr, shifts=sh, psf=synth.box_aperture_psf(mag), mag=mag, n_iter=20)
    yd = torch.from_numpy(y).cuda()
    sr, _ = pl.reconstruct(yd)
    it = pl.interp_fuse(yd)
    torch.cuda.synchronize()
    m = 4   # the outermost rows/columns follow the clamp border model, not the detector
    s, t = sr.cpu().numpy()[m:-m, m:-m], it.cpu().numpy()[m:-m, m:-m]
    g = truth[m:-m, m:-m]
    p_sr, p_it, s_sr, s_it = psnr(s, g), psnr(t, g), ssim(s, g), ssim(t, g)
    print(f"\n{name} x{mag}: PSNR FL-MISR {p_sr:.2f} dB vs interpolation {p_it:.2f} dB (+{p_sr - p_it:.2f}); "
          f"SSIM {s_sr:.4f} vs {s_it:.4f}")
    assert p_sr - p_it >= 1.0
    assert s_sr > s_it
