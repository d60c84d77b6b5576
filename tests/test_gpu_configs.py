"""GPU parity at the BASELINE.json configuration sizes (SURVEY.md 8(d) inputs),
against the UNMODIFIED reference library (oracle/_ref, OpenMP) on the same
inputs:

* C1  512x512, random-local 10k G, K=10: full-image global top-K dump +
      pixels (renderer.cpp:161-191), one train_step_gradients (fit.cpp:51-106)
      and adam_step t=1 (adam.cpp:10-52);
* C2  2048x2048, the bench's fit-start state (100k G, sigma = 2 px, theta = 0),
      10k samples: top-K at every sample, loss + gradients, Adam, then a
      10-iteration trajectory on both sides;
* C3  4096x4096, random-local 250k G: build_partition(64) (bsp.cpp:153-176),
      IGS2 encode -> decode -> rebuild_partition (codec.cpp:141-224,
      bsp.cpp:197-218), blocked render (bsp.cpp:289-341), 10k point queries;
* C4  8192x8192, random-local 1M G: top-K at the 10k samples + one train step;
* C5  one 1024x1024 texture share, 50k G: the five LoD prefixes, blocked.

Each test records its mismatch counts in a JSON report when IGS_PARITY_OUT
names a file (the round's run keeps it under profiles/).

Bars (north_star): top-K indices and partitions bit-exact; pixels and
gradients within 1e-4 relative and PSNR(GPU vs CPU) >= 80 dB.  With the
glibc-exact exp/sincos (csrc/glibc_math.cuh) the results are expected to be
bit-identical, and the tests require that.
"""
import json
import os
import time

import numpy as np
import pytest

from paper_2407_01866_b200 import synth

pytestmark = pytest.mark.gpu

K = 10
LR = np.array([2e-4, 2e-3, 1e-3, 1e-3])


def record(name, **kv):
    path = os.environ.get("IGS_PARITY_OUT")
    kv = {k: (v.item() if hasattr(v, "item") else v) for k, v in kv.items()}
    print(name, json.dumps(kv))
    if not path:
        return
    try:
        d = json.loads(open(path).read())
    except Exception:
        d = {}
    d[name] = kv
    with open(path, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)


def pixel_stats(got, want):
    got = np.asarray(got, np.float32)
    want = np.asarray(want, np.float32)
    same = got == want
    diff = np.abs(got.astype(np.float64) - want.astype(np.float64))
    mse = float(np.mean(diff ** 2))
    return {"pixels": int(got.shape[0] * got.shape[1]),
            "pixels_bit_identical": int(np.all(same, axis=-1).sum()),
            "channels_differing": int((~same).sum()),
            "max_abs_err": float(diff.max()),
            "psnr_gpu_vs_cpu_db": float("inf") if mse == 0 else 10 * np.log10(1.0 / mse)}


def grad_stats(got, want):
    groups = {"mu": [0, 1], "theta": [2], "scale": [3, 4], "color": [5, 6, 7]}
    out = {"elements_differing": int((got != want).sum()), "bit_identical": bool(np.array_equal(got, want))}
    worst = 0.0
    for name, g in groups.items():
        a, b = got[:, g], want[:, g]
        floor = max(np.max(np.abs(b)), 1e-300) * 1e-3
        err = float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)))
        out[f"rel_err_{name}"] = err
        worst = max(worst, err)
    out["rel_err_max"] = worst
    return out


def check_pixels(st):
    assert st["max_abs_err"] <= 1e-4, st
    assert st["psnr_gpu_vs_cpu_db"] >= 80, st
    assert st["pixels_bit_identical"] == st["pixels"], st


def check_grads(st):
    assert st["rel_err_max"] <= 1e-4, st
    assert st["bit_identical"], st


def topk_at_samples(gctx, ref, params, sidx, W, H):
    """Device top-K (igs_select_top_k) vs the reference's global scan at the
    sampled pixel centres (image.hpp:18-20)."""
    h, w = np.divmod(sidx.astype(np.int64), W)
    uv = np.stack([(w + 0.5) / W, (h + 0.5) / H], axis=1)
    gctx.set_params(params)
    got, _, _ = gctx.select_top_k(uv, K)
    want, _ = ref.topk_points(params, uv, K)
    rows = int(np.any(got != want, axis=1).sum())
    return rows, uv.shape[0]


def train_compare(gctx, ref, params, target, sidx, tag):
    gctx.set_params(params)
    gctx.set_target(target)
    t0 = time.perf_counter()
    loss, grads = gctx.train_step(sidx, K)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    wl, wg = ref.train_step(params, target, sidx, K)
    t_ref = time.perf_counter() - t0
    gs = grad_stats(grads, wg)
    gctx.adam_step(LR, 1)
    p1 = gctx.get_params()
    m1, v1 = gctx.get_adam_state()
    wp, wm, wv = ref.adam_step(params, wg, np.zeros_like(params), np.zeros_like(params), LR, 1)
    rec = dict(loss=loss, loss_ref=wl, loss_bit_identical=loss == wl, **gs,
               adam_params_differing=int((p1 != wp).sum()), adam_m_differing=int((m1 != wm).sum()),
               adam_v_differing=int((v1 != wv).sum()), seconds_gpu_call=t_gpu, seconds_ref=t_ref)
    record(tag, **rec)
    assert loss == wl
    check_grads(gs)
    assert rec["adam_params_differing"] == 0 and rec["adam_m_differing"] == 0 and rec["adam_v_differing"] == 0


# ------------------------------------------------------------------------- C1
def test_c1_render_topk(gctx, ref):
    W = H = 512
    params = synth.random_local_set(10_000, W, H, seed=7)
    gctx.set_params(params)
    img, topk = gctx.render_image(W, H, K, want_topk=True)
    t0 = time.perf_counter()
    want, wtk = ref.render_image(params, W, H, K, want_topk=True)
    t_ref = time.perf_counter() - t0
    mism = int(np.any(topk != wtk, axis=-1).sum())
    st = pixel_stats(img, want)
    record("c1_render", topk_pixels_mismatched=mism, seconds_ref=t_ref, **st)
    assert mism == 0
    check_pixels(st)


def test_c1_train_step_adam(gctx, ref):
    W = H = 512
    params = synth.random_local_set(10_000, W, H, seed=7)
    target = synth.photo_like_image(W, H, 31001)
    sidx = synth.sample_indices(10_000, W, H, seed=99)[0]
    train_compare(gctx, ref, params, target, sidx, "c1_train_step")


# ------------------------------------------------------------------------- C2
@pytest.fixture(scope="module")
def c2():
    W = H = 2048
    params = synth.init_set(100_000, W, H, seed=11)
    target = synth.photo_like_image(W, H, 31001)
    samples = synth.sample_indices(10_000, W, H, seed=99, steps=10)
    return W, H, params, target, samples


def test_c2_topk_at_samples(gctx, ref, c2):
    W, H, params, _, samples = c2
    rows, n = topk_at_samples(gctx, ref, params, samples[0], W, H)
    record("c2_topk_samples", samples=n, topk_rows_mismatched=rows)
    assert rows == 0


def test_c2_train_step_adam(gctx, ref, c2):
    W, H, params, target, samples = c2
    train_compare(gctx, ref, params, target, samples[0], "c2_train_step")


def test_c2_trajectory_10_iterations(gctx, ref, c2):
    """Ten fused iterations (select, blend, loss, backward, ordered reduction,
    Adam, constrain, re-prepare) on both sides from the same state."""
    W, H, params, target, samples = c2
    gctx.set_params(params)
    gctx.set_target(target)
    p = np.ascontiguousarray(params.copy()); m = np.zeros_like(p); v = np.zeros_like(p)
    losses, wlosses = [], []
    for t in range(1, 11):
        losses.append(gctx.train_iteration(samples[t - 1], K, LR, t))
        wlosses.append(ref.train_iteration(p, m, v, target, samples[t - 1], K, LR, t))
    got = gctx.get_params()
    gm, gv = gctx.get_adam_state()
    rec = dict(iterations=10, losses_bit_identical=losses == wlosses,
               params_differing=int((got != p).sum()), m_differing=int((gm != m).sum()),
               v_differing=int((gv != v).sum()),
               max_param_abs_diff=float(np.max(np.abs(got - p))), loss_last=losses[-1], loss_last_ref=wlosses[-1])
    record("c2_trajectory", **rec)
    assert losses == wlosses
    assert rec["params_differing"] == 0 and rec["m_differing"] == 0 and rec["v_differing"] == 0


# ------------------------------------------------------------------------- C3
def test_c3_partition_codec_blocked(gctx, ref):
    W = H = 4096
    params = synth.random_local_set(250_000, W, H, seed=7)
    gctx.set_params(params)
    gctx.partition_build(64)
    blocks, shells, off, mem = gctx.partition_get()
    t0 = time.perf_counter()
    rp = ref.partition_build(params, 64)
    t_build = time.perf_counter() - t0
    wb, ws = rp.rects()
    woff, wmem = rp.shell_members()
    part_exact = (np.array_equal(blocks, wb) and np.array_equal(shells, ws) and np.array_equal(off, woff)
                  and np.array_equal(mem, wmem))
    # IGS2 encode (device binary16 pack) == the reference's bytes
    data = gctx.encode(W, H, K, with_partition=True)
    wdata = ref.encode(params, W, H, K, rp)
    # decode -> rebuild_partition on both sides
    gctx.decode(data)
    dset = gctx.get_params()
    dblocks, dshells, doff, dmem = gctx.partition_get()
    t0 = time.perf_counter()
    wset, _, _, _, wpart = ref.decode(wdata)
    t_decode = time.perf_counter() - t0
    wdb, wds = wpart.rects()
    wdoff, wdmem = wpart.shell_members()
    decode_exact = (np.array_equal(dset, wset) and np.array_equal(dblocks, wdb) and np.array_equal(dshells, wds)
                    and np.array_equal(doff, wdoff) and np.array_equal(dmem, wdmem))
    # blocked render of the decoded set through the rebuilt partition
    img = gctx.render_image_blocked(W, H, K)
    t0 = time.perf_counter()
    want = ref.render_image_blocked(wset, wpart, W, H, K)
    t_render = time.perf_counter() - t0
    st = pixel_stats(img, want)
    # random-access point queries (bench_render shape, bsp.cpp:343-406)
    uv = np.random.default_rng(1).random((10_000, 2))
    pts = gctx.render_points_blocked(uv, K)
    wpts = ref.render_points_blocked(wset, wpart, uv, K)
    record("c3", n_blocks=int(blocks.shape[0]), shell_pairs=int(mem.size), partition_bit_exact=part_exact,
           igs2_bytes=len(data), igs2_byte_identical=data == wdata, decode_bit_exact=decode_exact,
           points=10_000, points_differing=int(np.any(pts != wpts, axis=1).sum()),
           points_max_abs_err=float(np.max(np.abs(pts - wpts))), seconds_ref_build=t_build,
           seconds_ref_decode=t_decode, seconds_ref_blocked_render=t_render, **st)
    assert part_exact and data == wdata and decode_exact
    check_pixels(st)
    assert np.array_equal(pts, wpts)


# ------------------------------------------------------------------------- C4
@pytest.fixture(scope="module")
def c4():
    W = H = 8192
    params = synth.random_local_set(1_000_000, W, H, seed=7)
    small = synth.photo_like_image(2048, 2048, 31004)
    target = np.ascontiguousarray(small.repeat(4, axis=0).repeat(4, axis=1))
    sidx = synth.sample_indices(10_000, W, H, seed=99)[0]
    return W, H, params, target, sidx


def test_c4_topk_at_samples(gctx, ref, c4):
    W, H, params, _, sidx = c4
    rows, n = topk_at_samples(gctx, ref, params, sidx, W, H)
    record("c4_topk_samples", samples=n, topk_rows_mismatched=rows)
    assert rows == 0


def test_c4_train_step_adam(gctx, ref, c4):
    W, H, params, target, sidx = c4
    train_compare(gctx, ref, params, target, sidx, "c4_train_step")


# ------------------------------------------------------------------------- C5
def test_c5_lod_prefixes_blocked(gctx, ref):
    W = H = 1024
    full = synth.random_local_set(50_000, W, H, seed=100)
    worst = None
    for m in (25_000, 31_250, 37_500, 43_750, 50_000):
        p = np.ascontiguousarray(full[:m])
        gctx.set_params(p)
        gctx.partition_build(64)
        img = gctx.render_image_blocked(W, H, K)
        want = ref.render_image_blocked(p, ref.partition_build(p, 64), W, H, K)
        st = pixel_stats(img, want)
        record(f"c5_lod_{m}", **st)
        check_pixels(st)
