"""Multi-process (gloo, world size 2 and 3) checks of the multi-GPU
decomposition on CPU, mirroring what the device path does over NCCL
(train.cu igs_forward_backward, exchange mode): every rank computes the
per-sample losses, slot keys and contribution records of its contiguous
sample block (upstream scaled by 1/NS_total), an all-gather assembles them
in global sample order, and every rank runs the sample-ordered reduction
(fit.cpp:86-104) -- so the gradients and the loss are bit-identical to the
single-process train step.  With the sharded update each rank then owns a
1/R slice of the set (ceil(n/R)-record blocks) and an all-gather of the
updated parameters restores the replicated set: also bit-identical.  Tile-row
bands stitch to the full render.  The per-rank compute is the oracle; the
decomposition is the product's (paper_2407_01866_b200/dist.py, the C-ABI).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import oracle
    from paper_2407_01866_b200 import dist as D
    from paper_2407_01866_b200 import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = oracle.get("port")
        W, H = 64, 48
        target = synth.photo_like_image(W, H, 31011)
        params = P.initialize_set(target, 301, 0.3, 4)
        params[:, 3:5] *= 3
        sidx = synth.sample_indices(1200, W, H, seed=12)[0]
        mine = D.shard(sidx, rank, world)
        n = params.shape[0]

        def allgather(a):
            parts = [torch.empty_like(torch.from_numpy(a)) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(a)))
            return np.concatenate([p.numpy() for p in parts])

        # the map on this rank's block, 1/NS_total scaling
        losses, keys, contrib = P.train_contribs(params, target, mine, 10, 1.0 / sidx.shape[0])
        losses, keys = allgather(losses), allgather(keys.astype(np.int64))
        contrib = allgather(contrib)
        # sample-ordered reduction over the gathered slots (global order)
        loss = 0.0
        for v in losses:
            loss += v
        loss *= 1.0 / sidx.shape[0]
        grads = np.zeros((n + 1, 8))
        np.add.at(grads, keys.ravel(), contrib.reshape(-1, 8))
        grads = grads[:n]
        # sharded update: Adam on this rank's ceil(n/R) block, then all-gather
        B = (n + world - 1) // world
        lo, hi = min(n, rank * B), min(n, (rank + 1) * B)
        zeros = np.zeros_like(params)
        p1, _, _ = P.adam_step(params[lo:hi], grads[lo:hi], zeros[lo:hi], zeros[lo:hi], [2e-4, 2e-3, 1e-3, 1e-3], 1)
        block = np.zeros((B, 8))
        block[:hi - lo] = p1
        updated = allgather(block)[:n]
        # tile-row band of the render
        r0, r1 = D.row_band(H, rank, world)
        band = P.render_image(params, W, H, 10)[r0:r1]
        bands = [None] * world
        dist.all_gather_object(bands, (r0, r1, band))
        if rank == 0:
            q.put((loss, grads, updated, bands))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_reduction_sharded_update_and_row_bands(port, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    loss, grads, updated, bands = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    from paper_2407_01866_b200 import synth
    W, H = 64, 48
    target = synth.photo_like_image(W, H, 31011)
    params = port.initialize_set(target, 301, 0.3, 4)
    params[:, 3:5] *= 3
    sidx = synth.sample_indices(1200, W, H, seed=12)[0]
    want_loss, want_g = port.train_step(params, target, sidx, 10)
    assert loss == want_loss
    assert np.array_equal(grads, want_g)
    zeros = np.zeros_like(params)
    want_p, _, _ = port.adam_step(params, want_g, zeros, zeros, [2e-4, 2e-3, 1e-3, 1e-3], 1)
    assert np.array_equal(updated, want_p)
    full = port.render_image(params, W, H, 10)
    stitched = np.concatenate([b for (_, _, b) in sorted(bands, key=lambda x: x[0])], axis=0)
    assert np.array_equal(stitched, full)


def test_row_bands_cover_and_align():
    from paper_2407_01866_b200.dist import row_band
    for H in (1, 15, 16, 100, 2048, 8192):
        for world in (1, 2, 3, 4, 8):
            bands = [row_band(H, r, world) for r in range(world)]
            assert bands[0][0] == 0 and bands[-1][1] == H
            for (a0, a1), (b0, b1) in zip(bands, bands[1:]):
                assert a1 == b0 and a0 % 16 == 0


def test_shard_blocks_and_uneven_count():
    from paper_2407_01866_b200 import dist as D
    s = np.arange(24).reshape(2, 12)
    assert np.array_equal(np.concatenate([D.shard(s, r, 4) for r in range(4)], axis=1), s)
    with pytest.raises(ValueError):
        D.shard(np.arange(10), 0, 4)
