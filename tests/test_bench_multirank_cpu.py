"""bench.py's multi-rank host logic on CPU (gloo, world_size 2): the collective transport decision of
the partitioned mode (a rank that cannot map its peers makes EVERY rank fall back to NCCL, with the
reason; --transport peer fails loudly instead), the flags, the rank records and the parity summary
rank 0 reports.  The GPU work is replaced by a stand-in Plan; the decision logic is bench.py's own."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _FakePlan:
    made = []

    def __init__(self, **kw):
        self.kw = kw
        self.destroyed = False
        self.connected = False
        self.row_lo, self.row_hi = 0, 0
        _FakePlan.made.append(self)

    def destroy(self):
        self.destroyed = True


class _FakeFlmisr:
    """peer_connect fails on the ranks listed in fail_on (as an IPC mapping failure would)."""
    Plan = _FakePlan

    def __init__(self, rank, fail_on):
        self.rank, self.fail_on = rank, fail_on

    def broadcast_unique_id(self):
        return bytes(128)

    def peer_connect(self, pl):
        if self.rank in self.fail_on:
            raise RuntimeError("cudaIpcOpenMemHandle: peer access not supported")
        pl.connected = True


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        out = {}
        out["all_true"] = bench.collective_all(dist, True, "cpu")
        out["all_one_false"] = bench.collective_all(dist, rank != 1, "cpu")
        out["bcast"] = bench.broadcast_flag(dist, rank == 0, "cpu")       # rank 0's value everywhere
        kw = dict(k=4, n_iter=20)
        # every rank can map its peers: the peer transport, no fallback
        _FakePlan.made = []
        pl, tr, why = bench.make_band_plan(_FakeFlmisr(rank, ()), dist, kw, rank, world, "auto", "cpu")
        out["ok"] = (tr, why, pl.connected, len(_FakePlan.made))
        # rank 1 cannot: every rank rebuilds on NCCL and reports rank 1's reason
        _FakePlan.made = []
        pl, tr, why = bench.make_band_plan(_FakeFlmisr(rank, (1,)), dist, kw, rank, world, "auto", "cpu")
        out["fallback"] = (tr, why, pl.connected, len(_FakePlan.made), _FakePlan.made[0].destroyed)
        # --transport peer: no fallback, a loud error on every rank
        try:
            bench.make_band_plan(_FakeFlmisr(rank, (1,)), dist, kw, rank, world, "peer", "cpu")
            out["strict"] = None
        except RuntimeError as e:
            out["strict"] = str(e)
        # --transport nccl: no attempt
        _FakePlan.made = []
        pl, tr, why = bench.make_band_plan(_FakeFlmisr(rank, (0, 1)), dist, kw, rank, world, "nccl", "cpu")
        out["nccl"] = (tr, why, pl.connected)
        rec = bench.rank_record(rank, world, rank, 100 * rank, 100 * rank + 100, tr)
        recs = [None] * world
        dist.all_gather_object(recs, rec)
        out["ranks"] = [(r["rank"], r["world"], r["rows"]) for r in recs]
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_bench_transport_decision_and_rank_records():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    res = dict(q.get() for _ in range(world))
    for rank, out in res.items():
        assert out["all_true"] is True and out["all_one_false"] is False and out["bcast"] is True
        assert out["ok"] == ("peer", None, True, 1)
        tr, why, connected, made, first_destroyed = out["fallback"]
        assert tr == "nccl" and not connected and made == 2 and first_destroyed
        assert "rank 1" in why and "peer access not supported" in why
        assert out["strict"] is not None and "rank 1" in out["strict"]
        assert out["nccl"] == ("nccl", None, False)
        assert out["ranks"] == [(0, 2, [0, 100]), (1, 2, [100, 200])]


def test_band_parity_summary():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    rng = np.random.default_rng(0)
    img = rng.uniform(size=(32, 32))
    tr = np.zeros((5, 6))
    tr[:, 1] = [10, 9, 8, 8, 7]
    tr[:, 5] = [1, 1, 1, 0, 1]
    p = bench.band_parity(img, img, tr, tr)
    assert p["ok"] and p["image_rel_l2"] == 0 and p["same_accept_sequence"]
    tr2 = tr.copy()
    tr2[3, 5] = 1
    assert not bench.band_parity(img, img, tr2, tr)["ok"]
    assert not bench.band_parity(img * (1 + 1e-4), img, tr, tr)["ok"]
    tr3 = tr.copy()
    tr3[2, 1] *= 1 + 1e-5
    assert not bench.band_parity(img, img, tr3, tr)["ok"]
