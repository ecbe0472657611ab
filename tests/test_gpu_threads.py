"""Plans created and run from several host threads at once (the C ABI releases the GIL in ctypes
calls): the one-time kernel setup (shared-memory opt-in cache, NCCL symbol loading) is thread-safe
and concurrent reconstructions on separate streams give the same bits as sequential ones."""
import threading

import numpy as np
import pytest

from paper_2108_04315_b200 import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2108_04315_b200 import flmisr  # noqa: E402

GEOMS = [
    dict(mag=2, shifts=synth.shift_pattern(2)),                                    # streaming loop kernel
    dict(mag=3, shifts=synth.shift_pattern(3)),                                    # x3 streaming
    dict(mag=2, shifts=np.array([[0, 0], [0.25, 0.25], [0.5, 0.0], [0.0, 0.5]])),  # per-phase kernels
    dict(mag=2, shifts=np.array([[0, 0], [0.5, 0.5], [0.3, 0.1]])),               # general path
]


def _case(i):
    g = GEOMS[i % len(GEOMS)]
    lr = 48 + 6 * i
    y = synth.random_fields((len(g["shifts"]), lr, lr), 300 + i, 0.2, 0.9)
    return g, lr, y


def test_concurrent_plans_match_sequential():
    n = 8
    cases = [_case(i) for i in range(n)]

    def run(i, out):
        g, lr, y = cases[i]
        with torch.cuda.stream(torch.cuda.Stream()):
            pl = flmisr.Plan(k=len(g["shifts"]), lr_h=lr, lr_w=lr, shifts=g["shifts"], psf=synth.gaussian_psf(),
                             mag=g["mag"], n_iter=8)
            h, rep = pl.reconstruct(torch.from_numpy(y).cuda(), stream=torch.cuda.current_stream())
            torch.cuda.current_stream().synchronize()
            out[i] = (h.cpu().numpy(), rep["trace"].copy())
            pl.destroy()

    seq = {}
    for i in range(n):
        run(i, seq)
    for _ in range(3):   # plan creation, graph capture, launches and destruction interleave differently
        par = {}
        errs = []

        def worker(i):
            try:
                run(i, par)
            except Exception as e:   # surfaced below
                errs.append(e)

        th = [threading.Thread(target=worker, args=(i,)) for i in range(n)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        for i in range(n):
            np.testing.assert_array_equal(par[i][0], seq[i][0])
            np.testing.assert_array_equal(par[i][1], seq[i][1])
