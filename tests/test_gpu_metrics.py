"""GPU error map (Eq. 8 add_distribution, sampling.cpp:77-94 -- the
kernel-5 reduction that drives error-guided addition) and PSNR
(metrics.cpp:12-27) against golden vectors from the reference."""
import numpy as np
import pytest

from paper_2407_01866_b200 import IgsError, synth

pytestmark = pytest.mark.gpu


def test_golden_add_distribution_and_psnr(gctx, golden):
    g = golden("metrics")
    H, W, _ = g["target"].shape
    gctx.set_target(g["target"])
    p = gctx.add_distribution(W, H, g["rendered"])
    # device total = exact double-double sum rounded once; the reference's
    # Kahan total agrees to the last ulp or so
    np.testing.assert_allclose(p, g["add"], rtol=4e-16, atol=0)
    assert abs(gctx.psnr(W, H, g["rendered"]) - float(g["psnr"])) <= 1e-12 * abs(float(g["psnr"]))


def test_error_map_of_last_render(gctx, port):
    params = synth.random_set(800, 17, 0.01, 0.08)
    target = synth.photo_like_image(80, 60, 31005)
    gctx.set_params(params)
    gctx.set_target(target)
    img = gctx.render_image(80, 60, 10)
    p = gctx.add_distribution(80, 60)  # rendered = resident last image
    np.testing.assert_allclose(p, port.add_distribution(img, target), rtol=4e-16, atol=0)
    assert abs(p.sum() - 1.0) < 1e-9


def test_identical_images(gctx):
    target = synth.texture_like_image(32, 24, 5)
    gctx.set_target(target)
    p = gctx.add_distribution(32, 24, target)
    assert np.all(p == 1.0 / (32 * 24))  # uniform when the error is zero
    assert gctx.psnr(32, 24, target) == float("inf")


def test_dimension_mismatch(gctx):
    gctx.set_target(synth.texture_like_image(32, 24, 5))
    with pytest.raises(IgsError) as e:
        gctx.add_distribution(31, 24, np.zeros((24, 31, 3), np.float32))
    assert e.value.kind == "dimension_mismatch"
