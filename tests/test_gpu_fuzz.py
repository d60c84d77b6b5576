"""Randomised parity sweep over the search paths (seed windows and their
widening, the flat-start descent, batch merges, hard points, the patch
render, the refit after Adam): random set sizes, scale ranges, anisotropy,
clusters, image shapes and K -- top-K indices bit-exact against the oracle,
at sampled points and over whole renders."""
import os

import numpy as np
import pytest

from paper_2407_01866_b200 import synth
from paper_2407_01866_b200.igs import PROF_KNN_HARD

pytestmark = pytest.mark.gpu

# IGS_FUZZ_SEEDS widens the two random sweeps (default: the quick set)
N_FUZZ = int(os.environ.get("IGS_FUZZ_SEEDS", "12"))

LR = np.array([2e-4, 2e-3, 1e-3, 1e-3])


def random_case(rng):
    n = int(rng.choice([7, 50, 400, 3000, 12000]))
    smin = float(rng.choice([0.0003, 0.002, 0.01]))
    smax = smin * float(rng.choice([1.5, 10, 100]))
    params = synth.random_set(n, int(rng.integers(1 << 30)), smin, min(smax, 0.4))
    if rng.random() < 0.3:  # a dense cluster
        m = max(1, n // 3)
        params[:m, 0:2] = rng.random(2) * 0.8 + 0.1 + rng.normal(0, 0.01, (m, 2))
    if rng.random() < 0.3:  # strong anisotropy
        params[:, 3] *= rng.uniform(0.02, 1.0, n)
    params[:, 0:2] = np.clip(params[:, 0:2], 0.0, 1.0)
    return params


@pytest.mark.parametrize("seed", range(N_FUZZ))
def test_fuzz_points_and_render(gctx, port, seed):
    rng = np.random.default_rng(1000 + seed)
    params = random_case(rng)
    n = params.shape[0]
    gctx.set_params(params)
    k = int(rng.choice([1, 3, 10, 17, 32]))
    uv = rng.random((300, 2))
    if rng.random() < 0.5:
        uv[:50] = rng.uniform(0.95, 1.0, (50, 2))  # corners
    idx, w, cnt = gctx.select_top_k(uv, k)
    for p in range(0, uv.shape[0], 11):
        wi, ww = port.select_top_k(params, uv[p, 0], uv[p, 1], k)
        assert np.array_equal(idx[p, :cnt[p]], wi), (seed, n, k, p)
    W, H = int(rng.integers(9, 70)), int(rng.integers(9, 70))
    want, wtk = port.render_image(params, W, H, k, want_topk=True)
    got, gtk = gctx.render_image(W, H, k, want_topk=True)
    assert np.array_equal(gtk, wtk), (seed, n, k, W, H)
    assert np.max(np.abs(got.astype(np.float64) - want)) <= 1e-4


@pytest.mark.parametrize("seed", [0, 3, 5, 8])
def test_fuzz_points_hard_inwarp(gctx, port, monkeypatch, seed):
    """The same sweep with frontier overflows scanned by the overflowing
    half-warp (IGS_KNN_HARD_INWARP) instead of the split hard-point scan."""
    monkeypatch.setenv("IGS_KNN_HARD_INWARP", "1")
    test_fuzz_points_and_render(gctx, port, seed)


@pytest.mark.parametrize("seed,k", [(9, 10), (26, 16), (27, 16)])
def test_frontier_overflow_both_paths(gctx, port, monkeypatch, seed, k):
    """Sweep cases whose search frontier overflows at some points (counted by
    the device): both overflow paths -- the split hard-point scan
    (default), the whole set scanned by the overflowing half-warp
    (IGS_KNN_HARD_INWARP) -- return the oracle's top-K."""
    params = random_case(np.random.default_rng(1000 + seed))
    gctx.set_params(params)
    uv = np.random.default_rng(seed).random((300, 2))
    for inwarp in (False, True):
        if inwarp:
            monkeypatch.setenv("IGS_KNN_HARD_INWARP", "1")
        gctx.profile_enable(True)
        idx, w, cnt = gctx.select_top_k(uv, k)
        hard = gctx.profile_read(PROF_KNN_HARD)[2]
        gctx.profile_enable(False)
        assert hard > 0  # the case does overflow
        for p in range(uv.shape[0]):
            wi, _ = port.select_top_k(params, uv[p, 0], uv[p, 1], k)
            assert np.array_equal(idx[p, :cnt[p]], wi), (inwarp, p)


@pytest.mark.parametrize("seed", range(max(4, N_FUZZ // 3)))
def test_fuzz_after_training(gctx, port, seed):
    """Searches after Adam steps (tree refits between re-bucketings)."""
    rng = np.random.default_rng(2000 + seed)
    W, H = 80, 64
    target = synth.photo_like_image(W, H, 31100 + seed)
    params = port.initialize_set(target, int(rng.choice([300, 2000])), 0.3, 50 + seed)
    steps = synth.sample_indices(1500, W, H, seed=60 + seed, steps=8)
    gctx.set_params(params)
    gctx.set_target(target)
    gctx.upload_samples(steps)
    gctx.train_iterations(int(rng.integers(3, 20)), 10, LR * float(rng.choice([1, 10, 30])), 1)
    p = gctx.get_params()
    _, wtk = port.render_image(p, W, H, 10, want_topk=True)
    _, gtk = gctx.render_image(W, H, 10, want_topk=True)
    assert np.array_equal(gtk, wtk)
    uv = rng.random((200, 2))
    idx, w, cnt = gctx.select_top_k(uv, 10)
    for q in range(0, 200, 13):
        wi, ww = port.select_top_k(p, uv[q, 0], uv[q, 1], 10)
        assert np.array_equal(idx[q, :cnt[q]], wi)


@pytest.mark.parametrize("seed", [9, 26])
def test_frontier_overflow_in_training_step(gctx, port, seed):
    """A training step whose samples overflow the search frontier: the hard
    points go through the fused hard-point scan + reduction-offsets launch
    (hard_offsets_kernel); loss and gradients match the oracle's train_step."""
    params = random_case(np.random.default_rng(1000 + seed))
    W, H = 96, 80
    target = synth.photo_like_image(W, H, 31200 + seed)
    sidx = synth.sample_indices(3000, W, H, seed=seed)[0]
    gctx.set_params(params)
    gctx.set_target(target)
    gctx.profile_enable(True)
    loss, grads = gctx.train_step(sidx, 10)
    hard = gctx.profile_read(PROF_KNN_HARD)[2]
    gctx.profile_enable(False)
    assert hard > 0  # the step does overflow
    wl, wg = port.train_step(params, target, sidx, 10)
    assert abs(loss - wl) <= 1e-12 * abs(wl)
    scale = np.maximum(np.abs(wg), np.max(np.abs(wg), axis=0) * 1e-3)
    assert np.max(np.abs(grads - wg) / np.maximum(scale, 1e-300)) <= 1e-12


@pytest.mark.parametrize("seed", [9, 26])
def test_frontier_overflow_in_fused_iterations(gctx, ref, seed):
    """Fused iterations (search -> segment buckets -> hard-point / overflow /
    long-segment launch -> update with the loss) on sets whose searches
    overflow the frontier: the hard points' contributions land in the
    buckets before the update, and losses, parameters and moments match the
    reference's train_iteration bit for bit."""
    params = np.ascontiguousarray(random_case(np.random.default_rng(1000 + seed)))
    W, H = 96, 80
    target = synth.photo_like_image(W, H, 31200 + seed)
    steps = synth.sample_indices(3000, W, H, seed=seed, steps=3)
    gctx.set_params(params)
    gctx.set_target(target)
    gctx.profile_enable(True)
    got = [gctx.train_iteration(steps[t], 10, LR, t + 1) for t in range(3)]
    hard = gctx.profile_read(PROF_KNN_HARD)[2]
    gctx.profile_enable(False)
    assert hard > 0  # the iterations do overflow
    p = params.copy(); m = np.zeros_like(p); v = np.zeros_like(p)
    want = [ref.train_iteration(p, m, v, target, steps[t], 10, LR, t + 1) for t in range(3)]
    gm, gv = gctx.get_adam_state()
    assert got == want
    assert np.array_equal(gctx.get_params(), p) and np.array_equal(gm, m) and np.array_equal(gv, v)
