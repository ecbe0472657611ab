"""Row-band partitioning (Eq. subfunction, Alg. 1, inner-outer border exchange P:197) on ONE
GPU: g bands, each a separate plan with its own buffers and halo rows, run by
flmisr_reconstruct_virtual with device-to-device copies in place of the NCCL allgather and halo
send/recv.  Every band-mode kernel path runs; only the transport differs from the multi-GPU run.

Bar (north_star): the partitioned result matches the unpartitioned oracle within 1e-3 relative L2 and
shows no seam; the consensus trace equals the single-band run."""
import numpy as np
import pytest

from paper_2108_04315_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_04315_b200 import flmisr  # noqa: E402


def rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b)


def bands(lr_h, lr_w, mag, g, n_iter, **kw):
    sh = synth.shift_pattern(mag)
    return [flmisr.Plan(k=len(sh), lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf(), mag=mag,
                        n_iter=n_iter, rank=h, world=g, virtual=True, **kw) for h in range(g)]


RUNNERS = {"copies": lambda pls, yd: flmisr.reconstruct_virtual(pls, yd),
           "peer": lambda pls, yd: flmisr.reconstruct_virtual_peer(pls, yd)}


@pytest.mark.parametrize("transport", ["copies", "peer"])
@pytest.mark.parametrize("g", [2, 3, 4, 8])
def test_bands_match_oracle_and_single_band(orc, g, transport):
    """transport "copies": per-phase band kernels with device copies in place of NCCL; "peer": the
    peer-memory band loop (each band's loop one persistent kernel, all bands in one cooperative
    launch, halo rows stored into the neighbours' buffers, band sums through mailboxes)."""
    lr_h, lr_w, mag, n_iter = 96, 140, 2, 15
    truth = synth.phantom(mag * lr_h, mag * lr_w, seed=61)
    sh = synth.shift_pattern(mag)
    y = synth.detector_stack(truth, mag, sh, 1 / 255, seed=61).astype(np.float32)
    yd = torch.from_numpy(y).cuda()
    one = flmisr.Plan(k=4, lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=n_iter)
    h1, r1 = one.reconstruct(yd)
    pls = bands(lr_h, lr_w, mag, g, n_iter)
    hg, rg = RUNNERS[transport](pls, yd)
    hg = hg.cpu().numpy()
    pb = orc.Problem(k=4, lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf(), mag=mag)
    xo, tr, st = orc.scg(pb, y.astype(np.float64), n_iter)
    assert rel(hg, xo) <= 1e-3
    # same consensus trajectory as the unpartitioned GPU run (the per-warp fp32 partial sums are
    # grouped differently per band: agreement to ~1e-9, far inside the final-image bar)
    assert rg["accepted"] == r1["accepted"] == st["accepted"]
    np.testing.assert_allclose(rg["trace"][:, 1], r1["trace"][:, 1], rtol=1e-6)
    assert np.max(np.abs(hg - h1.cpu().numpy())) <= 1e-5
    # no seam: the row differences across each band boundary look like interior rows
    d = np.abs(np.diff(hg.astype(np.float64), axis=0)).mean(axis=1)
    for p in pls[1:]:
        assert d[p.row_lo - 1] <= 3.0 * np.median(d) + 1e-6
    for p in pls:
        p.destroy()


def test_virtual_copies_graph_replay_is_deterministic():
    """The per-phase band path (kernels + copies in place of the NCCL allgather and halo send/recv +
    scalar kernels) runs as one captured CUDA graph per band set; replays reproduce the first call bit
    for bit, and the eager launch (FLMISR_NO_GRAPH) gives the same result."""
    lr_h, lr_w, mag, n_iter, g = 64, 96, 2, 12, 4
    sh = synth.shift_pattern(mag)
    y = synth.detector_stack(synth.phantom(mag * lr_h, mag * lr_w, seed=66), mag, sh, 1 / 255, seed=66)
    yd = torch.from_numpy(y.astype(np.float32)).cuda()
    pls = bands(lr_h, lr_w, mag, g, n_iter)
    outs = [flmisr.reconstruct_virtual(pls, yd) for _ in range(3)]
    for h, r in outs[1:]:
        assert torch.equal(h, outs[0][0])
        np.testing.assert_array_equal(r["trace"], outs[0][1]["trace"])
    import os
    os.environ["FLMISR_NO_GRAPH"] = "1"
    try:
        eager = bands(lr_h, lr_w, mag, g, n_iter)
    finally:
        del os.environ["FLMISR_NO_GRAPH"]
    he, re_ = flmisr.reconstruct_virtual(eager, yd)
    assert torch.equal(he, outs[0][0])
    np.testing.assert_array_equal(re_["trace"], outs[0][1]["trace"])
    for p in pls + eager:
        p.destroy()


def test_peer_barrier_timeout_is_an_error_not_a_hang(monkeypatch):
    """A band that never arrives (test hook FLMISR_PEER_TEST_DROP) makes every band abandon the loop
    after FLMISR_PEER_TIMEOUT_MS instead of trapping: the call returns FLMISR_ERR_CUDA naming the
    barrier timeout, and the device stays usable (fresh plans reconstruct normally afterwards)."""
    lr_h, lr_w, mag, n_iter, g = 32, 64, 2, 6, 2
    sh = synth.shift_pattern(mag)
    y = synth.detector_stack(synth.phantom(mag * lr_h, mag * lr_w, seed=67), mag, sh, 1 / 255, seed=67)
    yd = torch.from_numpy(y.astype(np.float32)).cuda()
    pls = bands(lr_h, lr_w, mag, g, n_iter)
    monkeypatch.setenv("FLMISR_PEER_TEST_DROP", "1")
    monkeypatch.setenv("FLMISR_PEER_TIMEOUT_MS", "200")
    with pytest.raises(flmisr.FlmisrError) as ei:
        flmisr.reconstruct_virtual_peer(pls, yd)
    assert ei.value.status == flmisr.ERR_CUDA and "timed out" in str(ei.value)
    monkeypatch.delenv("FLMISR_PEER_TEST_DROP")
    monkeypatch.delenv("FLMISR_PEER_TIMEOUT_MS")
    for p in pls:
        p.destroy()
    fresh = bands(lr_h, lr_w, mag, g, n_iter)
    h, r = flmisr.reconstruct_virtual_peer(fresh, yd)
    assert torch.isfinite(h).all() and r["iters_run"] == n_iter
    for p in fresh:
        p.destroy()


def test_band_gradient_equals_full_gradient(orc):
    """One value+gradient pass at x0 in band mode (n_iter = 0 returns x0, the trace row 0 holds
    f0 = J(x0) and <r0, r0>): identical consensus scalars to the single-band plan."""
    lr_h, lr_w = 40, 64
    y = synth.random_fields((4, lr_h, lr_w), 62)
    yd = torch.from_numpy(y).cuda()
    one = flmisr.Plan(k=4, lr_h=lr_h, lr_w=lr_w, shifts=synth.shift_pattern(2), psf=synth.gaussian_psf(), n_iter=0)
    _, r1 = one.reconstruct(yd)
    pls = bands(lr_h, lr_w, 2, 4, 0)
    _, rg = flmisr.reconstruct_virtual(pls, yd)
    np.testing.assert_allclose(rg["trace"][0, 1:3], r1["trace"][0, 1:3], rtol=1e-6)
    pb = orc.Problem(k=4, lr_h=lr_h, lr_w=lr_w, shifts=synth.shift_pattern(2), psf=synth.gaussian_psf())
    x0 = orc.init_x0(pb, y.astype(np.float64))
    assert abs(rg["trace"][0, 1] - orc.objective(pb, x0, y.astype(np.float64))) <= 1e-5 * rg["trace"][0, 1]


def test_band_needs_streaming_path():
    sh = synth.shift_pattern(2)
    with pytest.raises(flmisr.FlmisrError) as ei:
        flmisr.Plan(k=4, lr_h=32, lr_w=33, shifts=sh, psf=synth.gaussian_psf(), rank=0, world=2, virtual=True)
    assert "streaming path" in str(ei.value)


def test_peer_loop_repeated_calls_and_determinism():
    """Epochs count on across calls (no rank resets a word a peer writes): the second and third call
    on the same plans reproduce the first bit for bit."""
    lr_h, lr_w, mag, n_iter, g = 64, 96, 2, 12, 4
    sh = synth.shift_pattern(mag)
    y = synth.detector_stack(synth.phantom(mag * lr_h, mag * lr_w, seed=64), mag, sh, 1 / 255, seed=64)
    yd = torch.from_numpy(y.astype(np.float32)).cuda()
    pls = bands(lr_h, lr_w, mag, g, n_iter)
    outs = [flmisr.reconstruct_virtual_peer(pls, yd) for _ in range(3)]
    for h, r in outs[1:]:
        assert torch.equal(h, outs[0][0])
        np.testing.assert_array_equal(r["trace"], outs[0][1]["trace"])
    for p in pls:
        p.destroy()


def test_peer_loop_larger_band_matches_single_gpu(orc):
    """HR 1024 x 2048 in g = 4 peer bands vs the unpartitioned persistent loop: same trajectory and
    image (sampled oracle rows would add nothing here: the single-GPU run is parity-tested)."""
    lr_h, lr_w, mag, n_iter, g = 512, 1024, 2, 10, 4
    sh = synth.shift_pattern(mag)
    y = synth.detector_stack(synth.phantom(mag * lr_h, mag * lr_w, seed=65), mag, sh, 1 / 255, seed=65)
    yd = torch.from_numpy(y.astype(np.float32)).cuda()
    one = flmisr.Plan(k=4, lr_h=lr_h, lr_w=lr_w, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=n_iter)
    h1, r1 = one.reconstruct(yd)
    pls = bands(lr_h, lr_w, mag, g, n_iter)
    hg, rg = flmisr.reconstruct_virtual_peer(pls, yd)
    assert rg["accepted"] == r1["accepted"]
    np.testing.assert_allclose(rg["trace"][:, 1], r1["trace"][:, 1], rtol=1e-6)
    assert rel(hg.cpu().numpy(), h1.cpu().numpy().astype(np.float64)) <= 1e-5
    for p in pls:
        p.destroy()


def test_peer_loop_c3_full_size_eight_bands():
    """north_star's partitioned case at full size: C3 (16.8 MP HR, 20 passes) as 8 peer bands vs the
    unpartitioned persistent loop on the same stack -- same accept/reject trajectory, f trace to
    1e-6, image to 1e-5 relative L2, no seam at the 7 band boundaries."""
    c = synth.CONFIGS["C3"]
    lr, mag, n_iter, g = c["lr"], c["mag"], c["n_iter"], 8
    y, sh, _ = synth.make_stack(lr, mag, seed=c["seed"])
    yd = torch.from_numpy(y).cuda()
    one = flmisr.Plan(k=4, lr_h=lr, lr_w=lr, shifts=sh, psf=synth.gaussian_psf(), mag=mag, n_iter=n_iter)
    h1, r1 = one.reconstruct(yd)
    pls = bands(lr, lr, mag, g, n_iter)
    hg, rg = flmisr.reconstruct_virtual_peer(pls, yd)
    assert rg["accepted"] == r1["accepted"]
    np.testing.assert_allclose(rg["trace"][:, 1], r1["trace"][:, 1], rtol=1e-6)
    h1n = h1.cpu().numpy().astype(np.float64)
    hgn = hg.cpu().numpy().astype(np.float64)
    assert rel(hgn, h1n) <= 1e-5
    d = np.abs(np.diff(hgn - h1n, axis=0)).max(axis=1)   # seam: the band-vs-single difference is flat
    for p in pls[1:]:
        assert d[p.row_lo - 1] <= 10.0 * np.median(d) + 1e-6
    for p in pls:
        p.destroy()
