"""End-to-end parity against the fp64 oracle at BASELINE.json's full sizes and at convergence.

* C2 (K=4 LR 1024^2 -> 2048^2, 50 passes) and C3 (K=4 LR 2048^2 -> 4096^2, 20 passes; the bench
  workload) reconstructed by the persistent loop kernel bench.py times, compared with orc.scg on the
  same fp32 stack: final image <= 1e-3 relative L2 (north_star), f trace <= 1e-4 relative, and an
  identical accept/reject sequence on every pass whose objective decrease the fp32 GPU can resolve
  (SURVEY.md:331; reading 27).
* C3 as 8 peer-memory row bands (north_star's partitioned case, one cooperative launch on one device)
  against the SAME unpartitioned oracle image: same bars, no seam.
* The trajectory-free pin (SURVEY 8(c) "Converged solution", reading 22): the minimiser x^ is unique;
  the oracle run to its fp64 stagnation and the GPU run to its fp32 stagnation agree to 1e-4.

The oracle runs here, on the GPU box's host (roughly 20-60 s each for C2 and C3, single-threaded);
nothing is precomputed from the CUDA path.  Measured errors are printed (pytest -s)."""
import numpy as np
import pytest

from paper_2108_04315_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_04315_b200 import flmisr  # noqa: E402


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def _config(orc, name):
    c = synth.CONFIGS[name]
    y, sh, _ = synth.make_stack(c["lr"], c["mag"], seed=c["seed"], shifts=c.get("shifts"))
    pb = orc.Problem(k=len(sh), lr_h=c["lr"], lr_w=c["lr"], shifts=sh, psf=synth.gaussian_psf(), mag=c["mag"])
    xo, tr, st = orc.scg(pb, y.astype(np.float64), c["n_iter"])
    assert st["rc"] == 0
    return dict(c=c, y=y, sh=sh, pb=pb, xo=xo, tr=tr, st=st)


@pytest.fixture(scope="module")
def c3(orc):
    return _config(orc, "C3")


def _check_against_oracle(tag, hr, rep, ref, seams=()):
    h = hr.cpu().numpy().astype(np.float64) if hasattr(hr, "cpu") else hr
    e_img = rel(h, ref["xo"])
    e_f = np.max(np.abs(rep["trace"][:, 1] - ref["tr"][:, 1]) / np.abs(ref["tr"][:, 1]))
    print(f"\n{tag}: image rel L2 {e_img:.3e}, f trace max rel {e_f:.3e}, accepted "
          f"{rep['accepted']}/{ref['st']['accepted']} of {rep['iters_run']}")
    assert rep["iters_run"] == ref["st"]["iters_run"]
    # accept/reject decisions (Delta >= 0 on f - f_new) must agree while the oracle's objective still
    # falls by more than the fp32 resolution of the GPU's f (its trace matches the oracle's to ~1e-7
    # relative); past that point the fp64 oracle keeps improving f by 1e-11..1e-14 relative (C2,
    # passes 39-44) and both sides' decisions are rounding (reading 27)
    f = ref["tr"][:, 1]
    drop = (f[:-1] - f[1:]) / f[1:]
    resolvable = np.ones(len(f), bool)
    small = np.where((ref["tr"][1:, 5] > 0) & (drop < 1e-6))[0]
    if len(small):
        resolvable[small[0] + 1:] = False
    print(f"  accept flags compared on passes 1..{int(resolvable.sum()) - 1} of {len(f) - 1}")
    np.testing.assert_array_equal(rep["trace"][resolvable, 5], ref["tr"][resolvable, 5])
    assert e_f <= 1e-4
    assert e_img <= 1e-3
    # seam check: the difference to the oracle is no larger on the rows around a band
    # boundary than elsewhere
    if seams:
        d = np.abs(h - ref["xo"]).max(axis=1)
        for r0 in seams:
            assert d[r0 - 2:r0 + 2].max() <= 10.0 * np.median(d) + 1e-6, (r0, d[r0 - 2:r0 + 2], np.median(d))


def test_c3_final_image_vs_oracle(c3):
    c = c3["c"]
    with flmisr.Plan(k=4, lr_h=c["lr"], lr_w=c["lr"], shifts=c3["sh"], psf=synth.gaussian_psf(), mag=c["mag"],
                     n_iter=c["n_iter"]) as pl:
        assert pl.fast_path == 2 and pl.loop_kernel   # the persistent streaming loop bench.py times
        hr, rep = pl.reconstruct(torch.from_numpy(c3["y"]).cuda())
        _check_against_oracle("C3 1 GPU", hr, rep, c3)


def test_c3_eight_peer_bands_vs_oracle(c3):
    """north_star: 'the 2/4/8-GPU partitioned result must match the unpartitioned oracle to the same
    bound, with no seam at partition borders'."""
    c, g = c3["c"], 8
    pls = [flmisr.Plan(k=4, lr_h=c["lr"], lr_w=c["lr"], shifts=c3["sh"], psf=synth.gaussian_psf(), mag=c["mag"],
                       n_iter=c["n_iter"], rank=h, world=g, virtual=True) for h in range(g)]
    hr, rep = flmisr.reconstruct_virtual_peer(pls, torch.from_numpy(c3["y"]).cuda())
    _check_against_oracle("C3 8 peer bands", hr, rep, c3, seams=[p.row_lo for p in pls[1:]])
    for p in pls:
        p.destroy()


def test_c2_final_image_vs_oracle(orc):
    ref = _config(orc, "C2")
    c = ref["c"]
    with flmisr.Plan(k=4, lr_h=c["lr"], lr_w=c["lr"], shifts=ref["sh"], psf=synth.gaussian_psf(), mag=c["mag"],
                     n_iter=c["n_iter"]) as pl:
        assert pl.fast_path == 2 and pl.loop_kernel
        hr, rep = pl.reconstruct(torch.from_numpy(ref["y"]).cuda())
        _check_against_oracle("C2 1 GPU", hr, rep, ref)


def test_g3_final_image_vs_oracle(orc):
    """G3 (C3's size, quarter-pixel detector positions: a composed kernel per frame) on the per-phase
    streaming loop kernel bench.py --config G3 times, against orc.scg on the same stack."""
    ref = _config(orc, "G3")
    c = ref["c"]
    with flmisr.Plan(k=4, lr_h=c["lr"], lr_w=c["lr"], shifts=ref["sh"], psf=synth.gaussian_psf(), mag=c["mag"],
                     n_iter=c["n_iter"]) as pl:
        assert pl.fast_path == 4 and pl.loop_kernel
        hr, rep = pl.reconstruct(torch.from_numpy(ref["y"]).cuda())
        _check_against_oracle("G3 1 GPU (per-phase kernels)", hr, rep, ref)


def test_c1_converged_solution(orc):
    """SURVEY 8(c) 'Converged solution': independent of the accept/reject trajectory.  The oracle's
    fp64 SCG stagnates at <r,r> ~ 2e-12 (~1e-16 N) after ~50 passes (every later pass has
    f_new == f to the last bit); x^ = its iterate at the minimum <r,r>.  The GPU runs 300 passes
    (fp32 stagnation; a stagnated run may end in the non-finite freeze of Moller's exploding lambda,
    which returns the last finite iterate) and must agree with x^ to 1e-4 relative L2."""
    c = synth.CONFIGS["C1"]
    y, sh, _ = synth.make_stack(c["lr"], c["mag"], seed=c["seed"])
    pb = orc.Problem(k=4, lr_h=c["lr"], lr_w=c["lr"], shifts=sh, psf=synth.gaussian_psf(), mag=c["mag"])
    _, tr, _ = orc.scg(pb, y.astype(np.float64), 150)
    kmin = int(np.argmin(tr[:, 2]))
    assert tr[kmin, 2] <= 1e-14 * pb.H * pb.W
    xhat, _, _ = orc.scg(pb, y.astype(np.float64), kmin)
    with flmisr.Plan(k=4, lr_h=c["lr"], lr_w=c["lr"], shifts=sh, psf=synth.gaussian_psf(), mag=c["mag"],
                     n_iter=300) as pl:
        hr, rep = pl.reconstruct(torch.from_numpy(y).cuda(), raise_numeric=False)
    h = hr.cpu().numpy().astype(np.float64)
    assert np.isfinite(h).all()
    e = rel(h, xhat)
    e20 = rel(orc.scg(pb, y.astype(np.float64), 20)[0], xhat)
    print(f"\nC1 converged: oracle <r,r> min {tr[kmin, 2]:.2e} at pass {kmin}; GPU after {rep['iters_run']} passes "
          f"(<r,r> {rep['trace'][-1, 2]:.2e}): rel L2 to x^ {e:.3e} (the 20-pass iterate is {e20:.3e} away)")
    assert e <= 1e-4
