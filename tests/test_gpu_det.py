"""det mode (flmisr_config.det_rows): results bit-identical for every band count g (SURVEY 8(e)
"bit-stable"; P:404 -- the consensus run equals the centralised run).

The g = 1 persistent loop kernel, the g-band peer protocol (all bands in one cooperative launch on one
device, the multi-GPU kernel with local pointers) and the per-phase band kernels of the NCCL transport
(device copies in place of the allgather and the halo send/recv) cut their bands into different warp segments (one
wave each: a band of 1/g of the image on 1/g of the SMs), but every segment is a union of the same
fixed global tiles of T HR rows, each tile's sums are committed separately inside the row loop and
all sums are exact (128-bit fixed point), so the final image, the f trace and the accept sequence
must agree BIT FOR BIT at g = 1, 2, 4, 8.  The det result is also held to the usual oracle bar, and
det at g = 1 agrees with the default (fp64-tree) sums to rounding."""
import numpy as np
import pytest

from paper_2108_04315_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_04315_b200 import flmisr  # noqa: E402


def _stack(lr_h, lr_w, mag, seed):
    truth = synth.phantom(mag * lr_h, mag * lr_w, seed=seed)
    sh = synth.shift_pattern(mag)
    return sh, synth.detector_stack(truth, mag, sh, 1 / 255, seed=seed).astype(np.float32)


def _run(g, lr_h, lr_w, mag, sh, yd, n_iter, T, transport="peer", **kw):
    common = dict(k=len(sh), lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=n_iter,
                  det_rows=T, **kw)
    if g == 1:
        pl = flmisr.Plan(**common)
        assert pl.fast_path == 2 and pl.loop_kernel == 1
        h, rep = pl.reconstruct(yd)
        pl.destroy()
        return h.cpu().numpy(), rep
    pls = [flmisr.Plan(rank=r, world=g, virtual=True, **common) for r in range(g)]
    tile = T * mag // np.gcd(T, mag)
    for p in pls[:-1]:   # bands are unions of the fixed tiles
        assert p.row_lo % tile == 0 and p.row_hi % tile == 0
    # "peer": the peer-memory band loop (persistent kernels, mailboxes); "copies": the per-phase band
    # kernels with device copies in place of the NCCL allgather and halo send/recv
    run = flmisr.reconstruct_virtual_peer if transport == "peer" else flmisr.reconstruct_virtual
    h, rep = run(pls, yd)
    for p in pls:
        p.destroy()
    return h.cpu().numpy(), rep


CASES = {
    # ragged last tile (256 = 42 x 6 + 4)
    "ragged_T6": dict(lr_h=128, lr_w=256, mag=2, T=6, n_iter=20, gs=(1, 2, 4, 8)),
    # many tiles per warp segment (segment lengths differ between g = 1 and the bands)
    "long_segments_T3": dict(lr_h=1024, lr_w=1024, mag=2, T=3, n_iter=12, gs=(1, 2, 8)),
    # x3 (270 = 22 x 12 + 6 rows), p = 2, BTV window 2
    "x3_p2_w2": dict(lr_h=90, lr_w=132, mag=3, T=12, n_iter=15, gs=(1, 2, 3), p_norm=2, btv_window=2),
}


@pytest.mark.parametrize("name", list(CASES))
def test_bit_identical_across_band_counts(name):
    c = dict(CASES[name])
    gs = c.pop("gs")
    lr_h, lr_w, mag, T, n_iter = (c.pop(k) for k in ("lr_h", "lr_w", "mag", "T", "n_iter"))
    sh, y = _stack(lr_h, lr_w, mag, seed=91)
    yd = torch.from_numpy(y).cuda()
    ref, rref = _run(1, lr_h, lr_w, mag, sh, yd, n_iter, T, **c)
    assert np.isfinite(ref).all()
    for g in gs[1:]:
        for transport in ("peer", "copies"):
            h, rep = _run(g, lr_h, lr_w, mag, sh, yd, n_iter, T, transport=transport, **c)
            np.testing.assert_array_equal(rep["trace"], rref["trace"], err_msg=f"g={g} {transport}: trace differs")
            np.testing.assert_array_equal(h, ref, err_msg=f"g={g} {transport}: image differs")
            assert rep["accepted"] == rref["accepted"]


def test_det_meets_oracle_bar_and_matches_default_sums(orc):
    lr_h, lr_w, mag, n_iter = 96, 140, 2, 15
    sh, y = _stack(lr_h, lr_w, mag, seed=61)
    yd = torch.from_numpy(y).cuda()
    hd, rd = _run(1, lr_h, lr_w, mag, sh, yd, n_iter, 9)
    hd4, rd4 = _run(4, lr_h, lr_w, mag, sh, yd, n_iter, 9)
    np.testing.assert_array_equal(hd4, hd)
    pl = flmisr.Plan(k=4, lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=n_iter)
    h0, r0 = pl.reconstruct(yd)
    h0 = h0.cpu().numpy()
    pb = orc.Problem(k=4, lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf(), mag=mag)
    xo, tr, st = orc.scg(pb, y.astype(np.float64), n_iter)
    assert np.linalg.norm(hd - xo) <= 1e-3 * np.linalg.norm(xo)
    np.testing.assert_array_equal(rd["trace"][:, 5], tr[:, 5])
    np.testing.assert_allclose(rd["trace"][:, 1], tr[:, 1], rtol=1e-4)
    # det vs the default fp64-tree sums: the same trajectory to rounding
    np.testing.assert_array_equal(rd["trace"][:, 5], r0["trace"][:, 5])
    np.testing.assert_allclose(rd["trace"][:, 1], r0["trace"][:, 1], rtol=1e-6)   # fp32 tile partials
    assert np.max(np.abs(hd - h0)) <= 1e-5


def test_det_repeatable_and_config_errors():
    lr_h, lr_w, mag = 64, 96, 2
    sh, y = _stack(lr_h, lr_w, mag, seed=5)
    yd = torch.from_numpy(y).cuda()
    a, ra = _run(1, lr_h, lr_w, mag, sh, yd, 10, 15)
    b, rb = _run(1, lr_h, lr_w, mag, sh, yd, 10, 15)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(ra["trace"], rb["trace"])
    # general geometry: no streaming path -> a config error, not a silent non-det run
    with pytest.raises(flmisr.FlmisrError, match="det_rows needs the streaming path"):
        flmisr.Plan(k=3, lr_h=21, lr_w=20, shifts=np.array([[0, 0], [0.5, 0.5], [0.3, 0.1]]),
                    psf=synth.gaussian_psf(), mag=2, det_rows=6)
    # bands of different det_rows are not one configuration
    pls = [flmisr.Plan(k=4, lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf(), mag=2, rank=r, world=2,
                       virtual=True, det_rows=6 if r == 0 else 9) for r in range(2)]
    with pytest.raises(flmisr.FlmisrError, match="one configuration"):
        flmisr.reconstruct_virtual(pls, yd)
    for p in pls:
        p.destroy()
