"""Multi-GPU decomposition of the hot path.

* Training: one iteration's samples are split across ranks (strided shard);
  every rank runs the exact global top-K + backward on its share with the
  upstream scaled by 1 / (total samples), the per-Gaussian gradients and the
  loss are summed with one NCCL all-reduce over NVLink (inside the C-ABI,
  igs_comm_init), and every rank applies the identical Adam step -- the
  replicated sets stay bit-identical across ranks.
* Rendering: pixels are independent; rank r renders the band of tile rows
  [row0, row1) (igs_render_image_rows) with no communication.

The helpers here are the host-side logic; tests/test_dist.py checks the
decomposition on CPU with gloo (world size 2) against the single-process
oracle.
"""
from __future__ import annotations

import numpy as np

TILE = 16


def shard(sample_idx: np.ndarray, rank: int, world: int) -> np.ndarray:
    """This rank's samples of one iteration (strided: balanced for any count)."""
    return np.ascontiguousarray(np.asarray(sample_idx)[..., rank::world])


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
