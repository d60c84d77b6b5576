"""Multi-GPU decomposition of the hot path.

* Training: one iteration's samples are split across ranks in contiguous
  equal blocks (rank r: samples [r ns, (r+1) ns)); every rank runs the exact
  global top-K + contribution epilogue on its block with the upstream scaled
  by 1 / (total samples), in-place all-gathers (NCCL over NVLink, or the
  in-process loopback group for tests; inside the C-ABI) complete the
  contribution, key and loss arrays in global sample order, every rank runs
  the sample-ordered reduction, and -- with IGS_OPT_SHARD_ADAM -- rank r
  updates its ceil(n/R) slice of the set before an all-gather of the
  parameters.  Bit-identical to one GPU.
* Eval / densify (igs_fit on every rank): each rank renders a band of the
  evaluation image, an all-gather assembles it, and metrics, alias tables
  and appends are replicated -- every rank writes the single-GPU log.
* Rendering: pixels are independent; rank r renders the band of tile rows
  [row0, row1) (igs_render_image_rows) with no communication.

The helpers here are the host-side logic; tests/test_dist.py checks the
decomposition on CPU with gloo (world size 2 and 3) against the
single-process oracle, tests/test_gpu_multirank.py the device path through
the loopback transport.
"""
from __future__ import annotations

import numpy as np

TILE = 16


def shard(sample_idx: np.ndarray, rank: int, world: int) -> np.ndarray:
    """This rank's samples of one iteration: the contiguous block
    [rank * ns, (rank + 1) * ns) of the last axis, ns = count / world (the
    device path gathers the blocks back in this order, so the count must
    divide evenly)."""
    a = np.asarray(sample_idx)
    total = a.shape[-1]
    if total % world:
        raise ValueError(f"{total} samples do not split evenly over {world} ranks")
    ns = total // world
    return np.ascontiguousarray(a[..., rank * ns:(rank + 1) * ns])


def row_band(height: int, rank: int, world: int, tile: int = TILE) -> tuple[int, int]:
    """Rows [row0, row1) of a tile-row-aligned split of `height` into `world` bands."""
    tiles = (height + tile - 1) // tile
    t0 = tiles * rank // world
    t1 = tiles * (rank + 1) // world
    return min(height, t0 * tile), min(height, t1 * tile)


class DistTrainer:
    """Drives a Context as one rank of a data-parallel training job.

    `uid` is the NCCL unique id broadcast by rank 0 (Context.comm_unique_id);
    any process-group plumbing (torch.distributed, MPI, a file) can carry it.
    """

    def __init__(self, ctx, uid: bytes, rank: int, world: int):
        self.ctx, self.rank, self.world = ctx, rank, world
        if world > 1 or uid is not None:
            ctx.comm_init(uid, world, rank)

    def iteration(self, sample_idx_all: np.ndarray, k: int, lr, t: int) -> float:
        """One fit iteration over the full sample set (every rank passes the
        same array); returns the global loss."""
        return self.ctx.train_iteration(shard(sample_idx_all, self.rank, self.world), k, lr, t)
