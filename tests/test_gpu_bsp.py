"""GPU parity of the BSP path (bsp.cpp): partition structure, shell
binning (kernel 2), locate_block, blocked raster and point queries, rebuilt
partitions from quantized corners, against golden vectors from the
reference and the oracle."""
import numpy as np
import pytest

from paper_2407_01866_b200 import IgsError, synth

pytestmark = pytest.mark.gpu


def check_image(got, want):
    assert np.max(np.abs(got.astype(np.float64) - want)) <= 1e-4
    assert np.mean(got == want) >= 0.9999


def test_golden_partition_and_blocked_render(gctx, golden):
    g = golden("bsp")
    gctx.set_params(g["params"])
    gctx.partition_build(int(g["n_max"]))
    b, s, off, mem = gctx.partition_get()
    assert np.array_equal(b, g["blocks"]) and np.array_equal(s, g["shells"])
    assert np.array_equal(off, g["shell_off"]) and np.array_equal(mem, g["shell_mem"])
    assert np.array_equal(gctx.locate_blocks(g["uv"]), g["locate"])
    check_image(gctx.render_image_blocked(int(g["W"]), int(g["H"]), int(g["k"])), g["blocked"])
    np.testing.assert_allclose(gctx.render_points_blocked(g["uv"], int(g["k"])), g["points"], rtol=1e-12,
                               atol=1e-14)


@pytest.mark.parametrize("seed,n,n_max", [(1, 900, 16), (2, 2500, 64), (3, 40, 1), (4, 7, 8), (5, 100_000, 64),
                                          (6, 5000, 4), (7, 300, 8), (8, 2000, 16)])
def test_partition_vs_oracle(gctx, port, seed, n, n_max):
    """The device tree build (bsp.cu build_tree_device) against the reference's
    recursive Builder: uniform sets, a coincident cluster, quantized
    coordinates (ties everywhere), all points identical (forced splits), and
    signed zeros (which the reference's comparator treats as equal)."""
    params = synth.random_set(n, 6000 + seed, 0.005, 0.06)
    if seed == 2:
        params[:600, 0:2] = params[0, 0:2]  # coincident cluster (tie-aware split)
    if seed == 6:
        params[:, 0:2] = np.floor(params[:, 0:2] * 16) / 16  # a 16 x 16 lattice
    if seed == 7:
        params[:, 0:2] = 0.25
    if seed == 8:
        params[:700, 0] = 0.0
        params[300:700, 0] = -0.0
        params[100:900, 1] = params[100, 1]
    gctx.set_params(params)
    gctx.partition_build(n_max)
    part = port.partition_build(params, n_max)
    b, s, off, mem = gctx.partition_get()
    wb, ws = part.rects()
    woff, wmem = part.shell_members()
    assert np.array_equal(b, wb) and np.array_equal(s, ws)
    assert np.array_equal(off, woff) and np.array_equal(mem, wmem)
    uv = np.random.default_rng(seed).random((300, 2))
    assert list(gctx.locate_blocks(uv)) == [part.locate(u, v) for u, v in uv]
    check_image(gctx.render_image_blocked(53, 41, 10), port.render_image_blocked(params, part, 53, 41, 10))
    np.testing.assert_allclose(gctx.render_points_blocked(uv, 5), port.render_points_blocked(params, part, uv, 5),
                               rtol=1e-12, atol=1e-14)


def test_rebuild_from_quantized_corners(gctx, port):
    """bsp.cpp:197-218: corners through binary16 (the IGS2 decode path), grid
    locator with gap/overlap fallbacks, shell membership by rectangle test."""
    params = synth.random_set(1500, 5013, 0.005, 0.05)
    part = port.partition_build(params, 64)
    rects = part.rects()[0].astype(np.float16).astype(np.float64)
    gctx.set_params(params)
    gctx.partition_rebuild(rects)
    q = port.partition_rebuild(rects, params)
    _, _, off, mem = gctx.partition_get()
    woff, wmem = q.shell_members()
    assert np.array_equal(off, woff) and np.array_equal(mem, wmem)
    uv = np.random.default_rng(5014).random((2000, 2))
    assert list(gctx.locate_blocks(uv)) == [q.locate(u, v) for u, v in uv]
    check_image(gctx.render_image_blocked(96, 96, 10), port.render_image_blocked(params, q, 96, 96, 10))


def test_single_block_equals_global(gctx):
    """test_bsp.cpp:146-153: N_b = 1 blocked render == global render."""
    params = synth.random_set(200, 5007)
    gctx.set_params(params)
    gctx.partition_build(200)
    nb, _ = gctx.partition_info()
    assert nb == 1
    assert np.array_equal(gctx.render_image_blocked(64, 48, 10), gctx.render_image(64, 48, 10))


def test_stale_partition_rejected(gctx):
    """test_bsp.cpp:201-207."""
    params = synth.random_set(50, 5010)
    gctx.set_params(params)
    gctx.partition_build(8)
    gctx.append_params(params[:1])
    with pytest.raises(IgsError) as e:
        gctx.render_image_blocked(16, 16, 10)
    assert e.value.kind == "invalid_parameter" and "stale" in str(e.value)
    with pytest.raises(IgsError):
        gctx.render_points_blocked([[0.5, 0.5]], 10)


def test_bench_render_rows_match_reference(gctx, ref):
    """a18: bench_render (bsp.cpp:343-406) -- the same random points, the same
    partitions per n_max, so N_b and the mean candidate count per point
    equal the reference's exactly; the times are device times."""
    params = synth.random_local_set(20_000, 1024, 1024, seed=7)
    n_max = [8, 32, 64, 128]
    gctx.set_params(params)
    rows = gctx.bench_render(10_000, n_max, seed=5, trials=5, warmup=1)
    want = ref.bench_render(params, 10_000, n_max, seed=5, trials=1, warmup=0)
    assert [r["n_max"] for r in rows] == [0] + n_max
    assert [r["n_b"] for r in rows] == [int(w) for w in want[:, 1]]
    assert [r["mean_candidates"] for r in rows] == list(want[:, 4])
    assert all(r["mean_ms_per_10k"] > 0 and r["std_ms"] >= 0 for r in rows)
