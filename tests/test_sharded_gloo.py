"""Multi-process (gloo, world size 2, CPU) test of the row-sharded path's host logic (SURVEY
§8(e)): each rank computes its rows of scale * W~ x~ (here with the oracle), pads
them into the all-gather slot, `gather_rows` exchanges and reorders, and the gathered y~ must
equal the unsharded product; then the replicated inverse RHT gives the full y."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import gemv, rht
from paper_2406_11235_b200.sharded import gather_order, gather_rows, padded_shard_rows, shard_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, m, n, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tiles = synth.random_tiles(m, n, 2, seed=21)
        p = gemv.Params(k=2, V=1, code="3inst")
        x = synth.random_x(B, n, seed=22).astype(np.float64)
        sn, sm = synth.random_sign_bytes(n, 23), synth.random_sign_bytes(m, 24)
        r0, r1 = shard_rows(m, world)[rank]
        slot = padded_shard_rows(m, world)
        # this rank's rows of scale * W~ x~ (RHT-in on the replicated x, RHT-out off)
        Wt = gemv.dense_decode(tiles[r0 // 16:r1 // 16], p)
        part = gemv.matvec(Wt, x, sn, None, scale=0.5, rht_in=True, rht_out=False)
        send = torch.zeros((B, slot), dtype=torch.float64)
        send[:, :r1 - r0] = torch.from_numpy(part)
        recv = torch.empty((world, B, slot), dtype=torch.float64)
        yt = gather_rows(send, recv, world, m).numpy()
        y = rht.rht_inverse(yt, sm, m)
        q.put((rank, yt, y))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,B", [(384, 256, 1), (640, 256, 3), (256, 128, 1)])
def test_row_sharded_allgather_matches_unsharded(m, n, B):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, B, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    tiles = synth.random_tiles(m, n, 2, seed=21)
    p = gemv.Params(k=2, V=1, code="3inst")
    x = synth.random_x(B, n, seed=22).astype(np.float64)
    sn, sm = synth.random_sign_bytes(n, 23), synth.random_sign_bytes(m, 24)
    Wt = gemv.dense_decode(tiles, p)
    full_t = gemv.matvec(Wt, x, sn, None, scale=0.5, rht_in=True, rht_out=False)
    full = gemv.matvec(Wt, x, sn, sm, scale=0.5, rht_in=True, rht_out=True)
    for rank, yt, y in res:
        # the gathered rows are the full product's rows (float64; BLAS may block a 3-column
        # product differently per shape, so equality up to rounding)
        np.testing.assert_allclose(yt, full_t, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(y, full, rtol=1e-12, atol=1e-12)


def test_shard_rows_partition():
    for m in (128, 256, 1000, 4096, 11008, 28672):
        for world in (1, 2, 4, 8):
            rows = shard_rows(m, world)
            assert rows[0][0] == 0 and rows[-1][1] == m
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            assert all(r0 % 128 == 0 for r0, _ in rows)
            slot = padded_shard_rows(m, world)
            idx = gather_order(slot, m, world)
            assert len(idx) == m and len(set(idx.tolist())) == m
