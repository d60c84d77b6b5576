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
    # device map, the reference's sequential Kahan total on the host:
    # the table is bit-identical
    assert np.array_equal(p, g["add"])
    assert abs(gctx.psnr(W, H, g["rendered"]) - float(g["psnr"])) <= 1e-12 * abs(float(g["psnr"]))


def test_error_map_of_last_render(gctx, port):
    params = synth.random_set(800, 17, 0.01, 0.08)
    target = synth.photo_like_image(80, 60, 31005)
    gctx.set_params(params)
    gctx.set_target(target)
    img = gctx.render_image(80, 60, 10)
    p = gctx.add_distribution(80, 60)  # rendered = resident last image
    assert np.array_equal(p, port.add_distribution(img, target))
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


@pytest.mark.parametrize("shape", [(2048, 2048), (37, 23), (1, 1), (5, 1), (1, 7)])
def test_sobel_magnitude_bit_identical(gctx, ref, shape):
    """f3: image_gradient_magnitude (sampling.cpp:44-67) on the device."""
    W, H = shape
    img = synth.photo_like_image(W, H, 31011)
    assert np.array_equal(gctx.image_gradient_magnitude(img), ref.image_gradient_magnitude(img))


@pytest.mark.parametrize("lam", [0.3, 0.8, 0.0, 1.0])
def test_gradient_mixture_bit_identical(gctx, ref, lam):
    """init/opt_distribution: device magnitude, the reference's Kahan total."""
    img = synth.photo_like_image(512, 384, 31012)
    assert np.array_equal(gctx.gradient_mixture(img, lam), ref.gradient_mixture(img, lam))
    flat = np.full((16, 16, 3), 0.25, np.float32)  # zero gradient field -> uniform
    assert np.array_equal(gctx.gradient_mixture(flat, lam), ref.gradient_mixture(flat, lam))
    with pytest.raises(IgsError):
        gctx.gradient_mixture(img, 1.5)


@pytest.mark.parametrize("shape", [(2048, 2048), (37, 23), (11, 11)])
def test_ssim_and_psnr_match_reference(gctx, ref, shape):
    """SSIM (metrics.cpp:33-112): the map is op for op on the device and each
    channel's mean is summed on the host in pixel order -- bit-identical.
    PSNR: the device's exact (double-double) squared-error total equals the
    reference's Kahan total whenever the true sum is not within ~n*u^2 of a
    rounding midpoint."""
    W, H = shape
    target = synth.photo_like_image(W, H, 31013)
    rendered = np.clip(target + np.random.default_rng(3).normal(0, 0.05, target.shape), 0, 1).astype(np.float32)
    gctx.set_target(target)
    assert gctx.ssim(W, H, rendered) == ref.ssim(rendered, target)
    assert gctx.psnr(W, H, rendered) == ref.psnr(rendered, target)
