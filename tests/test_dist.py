"""Multi-process (gloo, world size 2) checks of the multi-GPU decomposition
on CPU: sharded sample sets + a sum all-reduce reproduce the single-process
train step, and tile-row bands stitch to the full render.  The per-rank
compute is the oracle; the decomposition is the one the device path uses
(paper_2407_01866_b200/dist.py, NCCL inside the C-ABI)."""
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
        params = P.initialize_set(target, 300, 0.3, 4)
        params[:, 3:5] *= 3
        sidx = synth.sample_indices(1000, W, H, seed=12)[0]
        mine = D.shard(sidx, rank, world)
        blocks = [None] * world
        dist.all_gather_object(blocks, mine)
        assert np.array_equal(np.concatenate(blocks), sidx)  # gathered blocks = the sample order
        # the oracle scales by its own shard size; rescale to 1/NS_total like the device path
        loss, g = P.train_step(params, target, mine, 10)
        scale = mine.shape[0] / sidx.shape[0]
        t = torch.from_numpy(np.concatenate([g.ravel() * scale, [loss * scale]]))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        red = t.numpy()
        # tile-row band of the render
        r0, r1 = D.row_band(H, rank, world)
        band = P.render_image(params, W, H, 10)[r0:r1]
        bands = [None] * world
        dist.all_gather_object(bands, (r0, r1, band))
        if rank == 0:
            q.put((red, bands))
    finally:
        dist.destroy_process_group()


def test_sharded_train_step_and_row_bands(port):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    red, bands = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    from paper_2407_01866_b200 import synth
    W, H = 64, 48
    target = synth.photo_like_image(W, H, 31011)
    params = port.initialize_set(target, 300, 0.3, 4)
    params[:, 3:5] *= 3
    sidx = synth.sample_indices(1000, W, H, seed=12)[0]
    loss, g = port.train_step(params, target, sidx, 10)
    np.testing.assert_allclose(red[:-1].reshape(g.shape), g, rtol=1e-12, atol=1e-18)
    assert abs(red[-1] - loss) <= 1e-12 * loss
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
