"""Multi-image interpolation fusion on the GPU (tab:runtime's interpolation row) and the
quality margin of FL-MISR over it on a synthetic phantom (SPEC S:533 / AC6 analogue: tab:natural
reports +1.41 .. +6.62 dB PSNR over interpolation; only the sign of the margin is asserted)."""
import numpy as np
import pytest

from paper_2108_04315_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_04315_b200 import flmisr  # noqa: E402


def psnr(a, b):
    return -10.0 * np.log10(np.mean((np.asarray(a, np.float64) - b) ** 2))


@pytest.mark.parametrize("mag", [2, 3])
def test_interp_fusion_matches_oracle(orc, mag):
    lr = 40
    sh = synth.shift_pattern(mag)
    y = synth.random_fields((mag * mag, lr, lr + 4), 80)
    pl = flmisr.Plan(k=mag * mag, lr_h=lr, lr_w=lr + 4, shifts=sh, psf=synth.gaussian_psf(), mag=mag)
    out = torch.zeros((pl.H, pl.W), device="cuda")
    pl.debug(flmisr.OP_INTERP, lr=torch.from_numpy(y).cuda(), out=out)
    pb = orc.Problem(k=mag * mag, lr_h=lr, lr_w=lr + 4, shifts=sh, psf=synth.gaussian_psf(), mag=mag)
    np.testing.assert_array_equal(out.cpu().numpy(), orc.interp_fuse(pb, y.astype(np.float64)).astype(np.float32))


def test_flmisr_beats_interpolation_psnr():
    lr, mag = 128, 2
    y, sh, truth = synth.make_stack(lr, mag, seed=81)
    pl = flmisr.Plan(k=4, lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=20)
    yd = torch.from_numpy(y).cuda()
    sr, rep = pl.reconstruct(yd)
    it = torch.zeros_like(sr)
    pl.debug(flmisr.OP_INTERP, lr=yd, out=it)
    m = 4   # ignore the outermost rows/columns (border model)
    p_sr = psnr(sr.cpu().numpy()[m:-m, m:-m], truth[m:-m, m:-m])
    p_it = psnr(it.cpu().numpy()[m:-m, m:-m], truth[m:-m, m:-m])
    assert p_sr > p_it, (p_sr, p_it)
