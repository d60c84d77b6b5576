"""Certified tile culling (kernel 2).

CPU (no GPU): the predicate restated in the oracle (orc_cull_lists) is
SOUND against the reference's own top-K: for every pixel of every tile,
the reference's selected indices are members of the tile's list, on sets
where culling is hardest (fit-start sigma = 2 px, theta = 0) and on
anisotropic random sets.

GPU: the device's lists equal the restatement bit for bit (same members,
same tau) given the device's prepared records.
"""
import numpy as np
import pytest

from paper_2407_01866_b200 import synth


def _check_sound(port, ref_like, params, W, H, k, T=16):
    scan6 = port.prepare_scan(params)
    off, mem, tau = port.cull_lists(scan6, W, H, k, T)
    _, topk = ref_like.render_image(params, W, H, k, want_topk=True)
    TX = (W + T - 1) // T
    n = params.shape[0]
    sizes = np.diff(off.astype(np.int64))
    for h in range(H):
        for w in range(W):
            t = (h // T) * TX + (w // T)
            lst = set(mem[off[t]:off[t + 1]].tolist())
            for i in topk[h, w]:
                if i != 0xFFFFFFFF:
                    assert int(i) in lst, (h, w, int(i))
    return sizes.mean(), n


@pytest.mark.parametrize("kind,seed", [("init", 1), ("init", 2), ("local", 3), ("aniso", 4)])
def test_predicate_sound_vs_reference_topk(port, kind, seed):
    W, H = 96, 80
    if kind == "init":
        params = synth.init_set(1500, W, H, seed=seed)
    elif kind == "local":
        params = synth.random_local_set(1200, W, H, seed=seed)
    else:
        params = synth.random_set(800, seed, 0.002, 0.08)  # strongly anisotropic, random theta
    mean, n = _check_sound(port, port, params, W, H, 10)
    assert mean < 0.5 * n  # the lists actually cull


def test_predicate_sound_small_k_and_tiny_sets(port):
    for n, k in [(1, 10), (5, 3), (12, 10), (40, 1)]:
        params = synth.random_set(n, 50 + n, 0.01, 0.2)
        _check_sound(port, port, params, 40, 33, k)


def test_predicate_sound_clusters(port):
    """Coincident centres and a huge Gaussian: tau from dense seeds, wide reach."""
    params = synth.random_set(600, 9, 0.003, 0.02)
    params[:300, 0:2] = [0.3, 0.6]  # exact coincidence
    params[599, 3:5] = [0.7, 0.9]   # covers everything
    _check_sound(port, port, params, 64, 64, 10)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["init", "local", "aniso"])
def test_device_lists_equal_restatement(gctx, port, kind):
    W, H = 160, 120
    if kind == "init":
        params = synth.init_set(4000, W, H, seed=5)
    elif kind == "local":
        params = synth.random_local_set(3000, W, H, seed=6)
    else:
        params = synth.random_set(2000, 7, 0.002, 0.06)
    gctx.set_params(params)
    scan6 = gctx.get_prepared()
    off, mem, tau = gctx.tile_lists(W, H, 10)
    woff, wmem, wtau = port.cull_lists(scan6, W, H, 10)
    assert np.array_equal(tau, wtau)
    assert np.array_equal(off, woff)
    assert np.array_equal(mem, wmem)
