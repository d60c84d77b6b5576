"""The R-rank training exchange on one GPU through the
in-process loopback transport (igs_comm_init_loopback): R contexts, one host
thread each, the same collectives NCCL carries between GPUs (in-place
all-gather of rank blocks, rank-ordered sum all-reduce) as device copies.

Bar: every rank's result is bit-identical to the single-context run -- the
sample blocks are gathered back in global sample order and the reduction is
the reference's sample-ordered sum (fit.cpp:86-104), so the number of ranks
cannot change a bit.  The fp64-atomics mode (an all-reduce of per-rank
gradients) is order-dependent and is held to 1e-12.
"""
import threading

import numpy as np
import pytest

from paper_2407_01866_b200 import Context, OPT_DETERMINISTIC, OPT_SHARD_ADAM, synth
from paper_2407_01866_b200 import dist as D

pytestmark = pytest.mark.gpu

K = 10
LR = np.array([2e-4, 2e-3, 1e-3, 1e-3])


def run_ranks(ctxs, fn):
    """fn(rank, ctx) on one thread per rank; re-raises the first failure."""
    out, err = [None] * len(ctxs), []

    def body(r):
        try:
            out[r] = fn(r, ctxs[r])
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(len(ctxs))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


@pytest.fixture(scope="module")
def problem():
    W, H = 1024, 768
    params = synth.random_local_set(30_000, W, H, seed=21)
    params[:, 3:5] *= 0.5
    target = synth.photo_like_image(W, H, 31021)
    samples = synth.sample_indices(12_000, W, H, seed=23, steps=6)
    return W, H, params, target, samples


def single(params, target, samples, steps, det=True):
    with Context(0) as c:
        c.set_option(OPT_DETERMINISTIC, 1 if det else 0)
        c.set_params(params)
        c.set_target(target)
        losses = [c.train_iteration(samples[t], K, LR, t + 1) for t in range(steps)]
        return losses, c.get_params()


@pytest.mark.parametrize("world,shard", [(2, 1), (3, 1), (2, 0), (4, 1)])
def test_exchange_iterations_bit_identical(problem, world, shard):
    """Fused iterations at R ranks, with the update sharded (each rank
    reduces + updates its slice, then the parameters are all-gathered) or
    replicated: the same bits as one context."""
    W, H, params, target, samples = problem
    want_l, want_p = single(params, target, samples, 6)
    ctxs = [Context(0) for _ in range(world)]
    try:
        Context.comm_init_loopback(ctxs)

        def rank(r, c):
            c.set_option(OPT_SHARD_ADAM, shard)
            c.set_params(params)
            c.set_target(target)
            mine = D.shard(samples, r, world)
            losses = [c.train_iteration(mine[t], K, LR, t + 1) for t in range(6)]
            return losses, c.get_params()

        res = run_ranks(ctxs, rank)
    finally:
        for c in ctxs:
            c.close()
    for losses, p in res:
        assert losses == want_l
        assert np.array_equal(p, want_p)


def test_exchange_async_pipelined(problem):
    """igs_train_iteration_async two deep on each rank (the fit driver's
    pattern): same bits as the synchronous single-context run."""
    W, H, params, target, samples = problem
    want_l, want_p = single(params, target, samples, 6)
    ctxs = [Context(0) for _ in range(2)]
    try:
        Context.comm_init_loopback(ctxs)

        def rank(r, c):
            c.set_params(params)
            c.set_target(target)
            mine = D.shard(samples, r, 2)
            losses = []
            for t in range(6):
                c.train_iteration_async(mine[t], K, LR, t + 1)
                if t > 0:
                    losses.append(c.train_wait())
            losses.append(c.train_wait())
            return losses, c.get_params()

        res = run_ranks(ctxs, rank)
    finally:
        for c in ctxs:
            c.close()
    for losses, p in res:
        assert losses == want_l
        assert np.array_equal(p, want_p)


def test_train_step_gradients_and_fp64_allreduce(problem):
    W, H, params, target, samples = problem
    with Context(0) as c:
        c.set_params(params)
        c.set_target(target)
        want_loss, want_g = c.train_step(samples[0], K)
    for det in (1, 0):
        ctxs = [Context(0) for _ in range(2)]
        try:
            Context.comm_init_loopback(ctxs)

            def rank(r, c):
                c.set_option(OPT_DETERMINISTIC, det)
                c.set_params(params)
                c.set_target(target)
                return c.train_step(D.shard(samples[0], r, 2), K)

            res = run_ranks(ctxs, rank)
        finally:
            for c in ctxs:
                c.close()
        for loss, g in res:
            if det:
                assert loss == want_loss and np.array_equal(g, want_g)
            else:
                assert abs(loss - want_loss) <= 1e-12 * want_loss
                np.testing.assert_allclose(g, want_g, rtol=1e-9, atol=1e-15)
        assert np.array_equal(res[0][1], res[1][1])  # ranks agree with each other in both modes


def test_sharded_moments_gather_and_densify(problem):
    """After sharded iterations: the gathered Adam moments equal the single
    context's, and an append (densification: the slices move) followed by
    more iterations stays bit-identical."""
    W, H, params, target, samples = problem
    extra = synth.random_local_set(777, W, H, seed=29)
    with Context(0) as c:
        c.set_params(params)
        c.set_target(target)
        for t in range(3):
            c.train_iteration(samples[t], K, LR, t + 1)
        c.append_params(extra)
        want_l = [c.train_iteration(samples[t], K, LR, t + 1) for t in range(3, 6)]
        want_p = c.get_params()
        want_m, want_v = c.get_adam_state()
    ctxs = [Context(0) for _ in range(2)]
    try:
        Context.comm_init_loopback(ctxs)

        def rank(r, c):
            c.set_params(params)
            c.set_target(target)
            mine = D.shard(samples, r, 2)
            for t in range(3):
                c.train_iteration(mine[t], K, LR, t + 1)
            c.append_params(extra)
            losses = [c.train_iteration(mine[t], K, LR, t + 1) for t in range(3, 6)]
            c.comm_gather_moments()
            m, v = c.get_adam_state()
            return losses, c.get_params(), m, v

        res = run_ranks(ctxs, rank)
    finally:
        for c in ctxs:
            c.close()
    for losses, p, m, v in res:
        assert losses == want_l
        assert np.array_equal(p, want_p)
        assert np.array_equal(m, want_m) and np.array_equal(v, want_v)


@pytest.mark.parametrize("world", [2, 4])
def test_fit_multirank_log_identical(world):
    """SURVEY.md 8e eval/densify split: igs_fit on R ranks (each trains on its
    sample block, renders its band of every evaluation image, all-gathers the
    image; metrics, alias tables and appends replicated) writes the same
    FitReport log and ends with the same set as one context -- and so as the
    reference's fit() (test_gpu_fit)."""
    cfg = dict(budget=400, k=10, iterations=300, samples_per_iter=4000, eval_interval=50, warmup_iters=60,
               densify_interval=40, seed=5, plateau_patience=2)
    target = synth.photo_like_image(96, 80, 31031)
    with Context(0) as c:
        want = c.fit(target, Context.fit_config(**cfg))
        want_p = c.get_params()
    ctxs = [Context(0) for _ in range(world)]
    try:
        Context.comm_init_loopback(ctxs)
        res = run_ranks(ctxs, lambda r, c: (c.fit(target, Context.fit_config(**cfg)), c.get_params()))
    finally:
        for c in ctxs:
            c.close()
    for rep, p in res:
        assert rep["log"] == want["log"]
        assert np.array_equal(p, want_p)
