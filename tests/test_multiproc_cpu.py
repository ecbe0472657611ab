"""Multi-process host logic of the row-band path on CPU (gloo, world_size 2): the ncclUniqueId
broadcast over the torch process group, and the band geometry every rank derives independently
(Eq. subfunction: bands tile the image, agree across ranks and with the oracle's bands)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2108_04315_b200 import flmisr
        uid = flmisr.broadcast_unique_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        bands = {}
        for H, mag in ((4096, 2), (6144, 3), (128, 2), (1002, 2), (4097 - 1, 2)):
            for g in (1, 2, 3, 4, 8):
                bands[(H, mag, g)] = [flmisr.band(H, g, h, mag) for h in range(g)]
        mine = {k: v for k, v in bands.items()}
        allb = [None] * world
        dist.all_gather_object(allb, mine)
        # peer transport: every rank's fixed-size blob, gathered in rank order (flmisr_peer_connect input)
        blob = bytes([rank]) * flmisr.PEER_BLOB_BYTES
        blobs = flmisr.gather_blobs(blob, world)
        peer_ok = blobs == [bytes([r]) * flmisr.PEER_BLOB_BYTES for r in range(world)]
        q.put((rank, len(uid), all(i == ids[0] for i in ids), allb[0] == allb[1], bands, peer_ok))
    finally:
        dist.destroy_process_group()


def test_unique_id_broadcast_and_band_agreement():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = [q.get() for _ in range(world)]
    from oracle import oracle
    for rank, nid, same_id, same_bands, bands, peer_ok in res:
        assert nid == 128 and same_id and same_bands and peer_ok
        for (H, mag, g), bb in bands.items():
            # bands tile [0, H) without gaps or overlap, boundaries are multiples of mag
            assert bb[0][0] == 0 and bb[-1][1] == H
            for (lo0, hi0), (lo1, hi1) in zip(bb, bb[1:]):
                assert hi0 == lo1 and lo1 % mag == 0
            # identical to the oracle's band simulation (oracle/flmisr_oracle.c band_bounds)
            assert bb == [oracle.band_bounds(H, g, mag, h) for h in range(g)]
