"""IGS2 container (codec.cpp): the device binary16
packing and the host framing against the unmodified reference library --
byte-identical files, identical decoded sets and rebuilt partitions,
quantize_set, and the reference's error kinds."""
import numpy as np
import pytest

from paper_2407_01866_b200 import IgsError, synth

pytestmark = pytest.mark.gpu


def _set(n, seed, extreme=False):
    p = synth.random_set(n, seed, 0.002, 0.2)
    if extreme:  # binary16 subnormals, rounding ties, the largest finite half
        p[:8, 3] = [1e-4, 6.1e-5, 5.96e-8, 3e-8, 2.0, 1.0009765625, 0.00048828125 * 1.5, 2.0]
        p[8:16, 2] = [0.0, 3.14159, 2.5e-6, 1e-7, 65504.0, 3.0, 0.333, 1.5]
        p[16:24, 0] = -0.0
    return p


@pytest.mark.parametrize("n,extreme", [(1, False), (777, False), (3000, True)])
def test_encode_bytes_match_reference(gctx, ref, n, extreme):
    params = _set(n, 40 + n, extreme)
    gctx.set_params(params)
    assert gctx.encode(640, 480, 10) == ref.encode(params, 640, 480, 10)
    gctx.partition_build(16)
    part = ref.partition_build(params, 16)
    assert gctx.encode(640, 480, 7, with_partition=True) == ref.encode(params, 640, 480, 7, part)


def test_decode_set_and_partition_match_reference(gctx, ref):
    params = _set(2500, 9, True)
    part = ref.partition_build(params, 32)
    data = ref.encode(params, 96, 80, 10, part)
    hdr = gctx.decode(data)
    want, w, h, k, wpart = ref.decode(data)
    assert (hdr["width"], hdr["height"], hdr["k"], hdr["n_blocks"]) == (w, h, k, wpart.n_blocks)
    assert np.array_equal(gctx.get_params(), want)
    b, s, off, mem = gctx.partition_get()
    wb, ws = wpart.rects()
    woff, wmem = wpart.shell_members()
    assert np.array_equal(b, wb) and np.array_equal(s, ws)
    assert np.array_equal(off, woff) and np.array_equal(mem, wmem)
    # the decode path's render (blocked) equals the reference's on the decoded set
    got = gctx.render_image_blocked(96, 80, 10)
    exp = ref.render_image_blocked(want, wpart, 96, 80, 10)
    assert np.max(np.abs(got.astype(np.float64) - exp)) <= 1e-4 and np.mean(got == exp) >= 0.9999


def test_quantize_set_matches_reference(gctx, ref):
    params = _set(1500, 17, True)
    gctx.set_params(params)
    gctx.quantize_set()
    assert np.array_equal(gctx.get_params(), ref.quantize_set(params))


def test_codec_errors_match_reference(gctx, ref):
    params = _set(50, 3)
    data = bytearray(ref.encode(params, 32, 32, 10))
    gctx.set_params(params)
    cases = [(bytes(data[:10]), "truncated"), (b"XGS2" + bytes(data[4:]), "bad_magic"),
             (bytes(data[:4]) + b"\x07" + bytes(data[5:]), "bad_version"), (bytes(data[:-2]), "truncated")]
    for bad, kind in cases:
        with pytest.raises(IgsError) as e:
            gctx.decode(bad)
        assert e.value.kind == kind
        with pytest.raises(Exception):
            ref.decode(bad)
    p = params.copy()
    p[7, 4] = 7e4  # beyond binary16
    gctx.set_params(p)
    with pytest.raises(IgsError) as e:
        gctx.encode(32, 32, 10)
    assert e.value.kind == "invalid_parameter"
    with pytest.raises(Exception):
        ref.encode(p, 32, 32, 10)
    gctx.set_params(np.zeros((0, 8)))
    with pytest.raises(IgsError) as e:
        gctx.encode(32, 32, 10)
    assert e.value.kind == "empty_set"


def test_failed_decode_and_quantize_leave_the_set(gctx, ref):
    """The reference's decode() and quantize_set() are pure functions: a file
    with a NaN half, or a parameter beyond binary16, raises and the caller's
    set is untouched -- so the resident set must be too."""
    params = _set(60, 5)
    data = bytearray(ref.encode(params, 32, 32, 10))
    data[20:22] = (0x7e00).to_bytes(2, "little")  # the first Gaussian's mu_u: a NaN half
    other = _set(40, 6)
    gctx.set_params(other)
    with pytest.raises(IgsError):
        gctx.decode(bytes(data))
    with pytest.raises(Exception):
        ref.decode(bytes(data))
    assert np.array_equal(gctx.get_params(), other)
    # the search over the untouched set still answers exactly
    uv = np.random.default_rng(3).random((50, 2))
    idx, _, cnt = gctx.select_top_k(uv, 10)
    gctx.set_params(other)
    idx2, _, _ = gctx.select_top_k(uv, 10)
    assert np.array_equal(idx, idx2)
    p = other.copy()
    p[3, 3] = 7e4  # beyond binary16
    gctx.set_params(p)
    with pytest.raises(IgsError):
        gctx.quantize_set()
    with pytest.raises(Exception):
        ref.quantize_set(p)
    assert np.array_equal(gctx.get_params(), p)
