"""ctypes front-end for the TEST-ONLY checkers under oracle/.

TEST INFRASTRUCTURE: only tests/, ``__graft_entry__.smoke()`` and bench.py's
CPU-baseline legs may import this module.  The product package
(``paper_2407_01866_b200``) never does.

Two back-ends expose the same functions:

* ``Oracle("port")``       -- liboracle.so, our plain-C restatement
                              (oracle/igs_oracle.c, citations inside);
* ``Oracle("reference")``  -- oracle/_ref/libigs_ref.so, the unmodified
                              reference library compiled from
                              /root/reference/proj/src (oracle/Makefile) with a
                              C shim (oracle/ref_shim.cpp).

Arrays are numpy; layouts follow igs_oracle.h (Gaussian = 8 doubles, image =
float32 H x W x 3, sample = 5 doubles, rect = 4 doubles).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libigs_ref.so"

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_up = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p

ERROR_KINDS = {
    1: "invalid_parameter",
    2: "dimension_mismatch",
    3: "bad_magic",
    4: "bad_version",
    5: "truncated",
    6: "empty_set",
    7: "io",
    8: "unsupported_format",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        self.kind = ERROR_KINDS.get(code, f"code{code}")
        super().__init__(f"{self.kind}: {what}")


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


def build(quiet: bool = True) -> None:
    """Compile liboracle.so and (when /root/reference exists) _ref/."""
    import subprocess

    subprocess.run(["make", "-C", str(HERE)], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


# (name, restype, argtypes) shared by both back-ends.
_SIGS = [
    ("render_image", C.c_int, [_dp, C.c_uint32, C.c_int, C.c_int, C.c_int, _fp, _up]),
    ("select_top_k", C.c_int, [_dp, C.c_uint32, C.c_double, C.c_double, C.c_int, _up, _dp, _ip]),
    ("render_topk", C.c_int, [_dp, C.c_uint32, _dp, C.c_uint32, C.c_int, _dp]),
    ("render_naive", C.c_int, [_dp, C.c_uint32, _dp, C.c_uint32, _dp]),
    ("backward", C.c_int, [_dp, C.c_uint32, _dp, C.c_uint32, C.c_int, _dp]),
    ("train_step", C.c_int, [_dp, C.c_uint32, _fp, C.c_int, C.c_int, _up, C.c_uint32, C.c_int, _dp, _dp]),
    ("adam_step", C.c_int, [_dp, _dp, _dp, _dp, C.c_uint32, _dp, C.c_longlong, _i64p]),
    ("constrain", C.c_int, [_dp, C.c_uint32]),
    ("density", C.c_double, [_dp, C.c_double, C.c_double]),
    ("image_gradient_magnitude", None, [_fp, C.c_int, C.c_int, _dp]),
    ("gradient_mixture", C.c_int, [_fp, C.c_int, C.c_int, C.c_double, _dp]),
    ("add_distribution", C.c_int, [_fp, _fp, C.c_int, C.c_int, _dp]),
    ("initialize_set", C.c_int, [_fp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, _dp]),
    ("psnr", C.c_double, [_fp, _fp, C.c_size_t]),
    ("rng_stream", None, [C.c_uint64, C.c_uint64, C.c_uint32, _u64p]),
    ("partition_build", _vp, [_dp, C.c_uint32, C.c_int, _ip]),
    ("partition_rebuild", _vp, [_dp, C.c_uint32, _dp, C.c_uint32, _ip]),
    ("partition_free", None, [_vp]),
    ("partition_nblocks", C.c_uint32, [_vp]),
    ("partition_shell_total", C.c_uint64, [_vp]),
    ("partition_rects", None, [_vp, _dp, _dp]),
    ("partition_shell_members", None, [_vp, _up, _up]),
    ("partition_block_members", None, [_vp, _up, _up]),
    ("locate_block", C.c_int, [_vp, C.c_double, C.c_double]),
    ("render_image_blocked", C.c_int, [_dp, C.c_uint32, _vp, C.c_int, C.c_int, C.c_int, _fp]),
    ("render_points_blocked", C.c_int, [_dp, C.c_uint32, _vp, _dp, C.c_uint32, C.c_int, _dp]),
]

_PORT_ONLY = [
    ("random_set", None, [C.c_uint32, C.c_uint64, C.c_double, C.c_double, _dp]),
    ("random_image", None, [C.c_int, C.c_int, C.c_uint64, _fp]),
    ("photo_like_image", None, [C.c_int, C.c_int, C.c_uint64, _fp]),
    ("vector_like_image", None, [C.c_int, C.c_int, C.c_uint64, _fp]),
    ("texture_like_image", None, [C.c_int, C.c_int, C.c_uint64, _fp]),
    ("alias_build", C.c_int, [_dp, C.c_size_t, _dp, _up]),
    ("cull_lists", C.c_uint64, [_dp, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int, _up, _up, _dp]),
    ("prepare_scan", None, [_dp, C.c_uint32, _dp]),
    ("train_contribs", C.c_int, [_dp, C.c_uint32, _fp, C.c_int, C.c_int, _up, C.c_uint32, C.c_int, C.c_double, _dp,
                                 _up, _dp]),
]

class RefFitConfig(C.Structure):
    _fields_ = [("budget", C.c_int), ("k", C.c_int), ("lambda_init", C.c_double), ("lambda_opt", C.c_double),
                ("iterations", C.c_int), ("samples_per_iter", C.c_int), ("lr", C.c_double * 4),
                ("eval_interval", C.c_int), ("plateau_patience", C.c_int), ("lr_decay", C.c_double),
                ("warmup_iters", C.c_int), ("densify_interval", C.c_int), ("seed", C.c_uint64),
                ("compute_ssim", C.c_int)]


_REF_ONLY = [
    ("fit", C.c_int, [_fp, C.c_int, C.c_int, C.POINTER(RefFitConfig), _dp, C.c_uint32, _up, C.c_char_p,
                      C.c_size_t]),
    ("backward_mode", C.c_int, [_dp, C.c_uint32, _dp, C.c_uint32, C.c_int, _dp, C.c_int]),
    ("sample_pixel_indices", C.c_int, [_dp, C.c_int, C.c_int, C.c_int, C.c_uint64, _up]),
    ("ssim", C.c_double, [_fp, _fp, C.c_int, C.c_int]),
    ("train_iteration", C.c_int, [_dp, C.c_uint32, _dp, _dp, _fp, C.c_int, C.c_int, _up, C.c_uint32,
                                  C.c_int, _dp, C.c_longlong, _dp]),
    ("topk_points", C.c_int, [_dp, C.c_uint32, _dp, C.c_uint32, C.c_int, _up, _dp]),
    ("bench_render", C.c_int, [_dp, C.c_uint32, C.c_int, _ip, C.c_int, C.c_uint64, C.c_int, C.c_int, _dp]),
]


def available(kind: str) -> bool:
    return (PORT_LIB if kind == "port" else REF_LIB).exists()


class Partition:
    """Owning handle of an orc_/ref_ partition."""

    def __init__(self, lib, handle, prefix):
        self._lib, self.h, self._p = lib, handle, prefix

    def __del__(self):
        if getattr(self, "h", None):
            getattr(self._lib, self._p + "partition_free")(self.h)
            self.h = None

    @property
    def n_blocks(self) -> int:
        return int(getattr(self._lib, self._p + "partition_nblocks")(self.h))

    def rects(self):
        nb = self.n_blocks
        b = np.zeros((nb, 4)); s = np.zeros((nb, 4))
        getattr(self._lib, self._p + "partition_rects")(self.h, _ptr(b, _dp), _ptr(s, _dp))
        return b, s

    def _csr(self, fn, total):
        nb = self.n_blocks
        off = np.zeros(nb + 1, np.uint32)
        mem = np.zeros(max(total, 1), np.uint32)
        getattr(self._lib, self._p + fn)(self.h, _ptr(off, _up), _ptr(mem, _up))
        return off, mem[:total]

    def shell_members(self):
        total = int(getattr(self._lib, self._p + "partition_shell_total")(self.h))
        return self._csr("partition_shell_members", total)

    def block_members(self, n_gaussians: int):
        return self._csr("partition_block_members", n_gaussians)

    def locate(self, u: float, v: float) -> int:
        return int(getattr(self._lib, self._p + "locate_block")(self.h, float(u), float(v)))


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_LIB if kind == "port" else REF_LIB
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run make -C oracle)")
        self.lib = C.CDLL(str(path))
        self.p = "orc_" if kind == "port" else "ref_"
        sigs = _SIGS + (_PORT_ONLY if kind == "port" else _REF_ONLY)
        for name, res, args in sigs:
            f = getattr(self.lib, self.p + name)
            f.restype = res
            f.argtypes = args


    # ---- IGS2 codec (reference library only) ------------------------------------------
    def encode(self, params, width, height, k, part=None):
        params = np.ascontiguousarray(params, np.float64)
        size = C.c_size_t(0)
        f = self.lib.ref_encode
        f.restype = C.c_int
        f.argtypes = [_dp, C.c_uint32, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int, C.POINTER(C.c_uint8), C.c_size_t,
                      C.POINTER(C.c_size_t)]
        code = f(_ptr(params, _dp), params.shape[0], part.h if part is not None else None, width, height, k, None, 0,
                 C.byref(size))
        self._chk(code, "encode")
        out = np.zeros(size.value, np.uint8)
        self._chk(f(_ptr(params, _dp), params.shape[0], part.h if part is not None else None, width, height, k,
                    out.ctypes.data_as(C.POINTER(C.c_uint8)), out.size, C.byref(size)), "encode")
        return out.tobytes()

    def decode(self, data, max_n=1 << 24):
        buf = np.frombuffer(bytes(data), np.uint8).copy()
        f = self.lib.ref_decode
        f.restype = C.c_int
        f.argtypes = [C.POINTER(C.c_uint8), C.c_size_t, _dp, C.c_uint32, _up, _up, _up, _ip, C.POINTER(C.c_void_p)]
        n = C.c_uint32(0); w = C.c_uint32(0); h = C.c_uint32(0); k = C.c_int(0); part = C.c_void_p()
        n_hdr = int.from_bytes(bytes(data)[12:16], "little") if len(data) >= 16 else 0
        out = np.zeros((max(min(n_hdr, max_n), 1), 8))
        self._chk(f(buf.ctypes.data_as(C.POINTER(C.c_uint8)), buf.size, _ptr(out, _dp), out.shape[0], C.byref(n),
                    C.byref(w), C.byref(h), C.byref(k), C.byref(part)), "decode")
        p = Partition(self.lib, part.value, self.p) if part.value else None
        return out[:n.value], w.value, h.value, k.value, p

    def quantize_set(self, params):
        p = np.ascontiguousarray(params, np.float64).copy()
        f = self.lib.ref_quantize_set
        f.restype = C.c_int
        f.argtypes = [_dp, C.c_uint32]
        self._chk(f(_ptr(p, _dp), p.shape[0]), "quantize_set")
        return p

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    @staticmethod
    def _chk(code, what=""):
        if code:
            raise OracleError(code, what)

    # ---- generators (port back-end; deterministic mt19937_64) ----------
    def random_set(self, n, seed, smin=0.01, smax=0.3):
        out = np.zeros((n, 8))
        self._f("random_set")(n, seed, smin, smax, _ptr(out, _dp))
        return out

    def image(self, kind, W, H, seed):
        out = np.zeros((H, W, 3), np.float32)
        self._f(kind + "_image")(W, H, seed, _ptr(out, _fp))
        return out

    def rng_stream(self, seed, count, skip=0):
        out = np.zeros(count, np.uint64)
        self._f("rng_stream")(seed, skip, count, _ptr(out, _u64p))
        return out

    # ---- renderer ------------------------------------------------------
    def render_image(self, params, W, H, k, want_topk=False):
        params = np.ascontiguousarray(params, np.float64)
        n = params.shape[0]
        out = np.zeros((H, W, 3), np.float32)
        kk = min(k, n) if k >= 1 else 1
        topk = np.zeros((H, W, kk), np.uint32) if want_topk else None
        self._chk(self._f("render_image")(_ptr(params, _dp), n, W, H, k, _ptr(out, _fp), _ptr(topk, _up)),
                  "render_image")
        return (out, topk) if want_topk else out

    def select_top_k(self, params, u, v, k):
        params = np.ascontiguousarray(params, np.float64)
        n = params.shape[0]
        kk = max(1, min(k, n))
        idx = np.zeros(kk, np.uint32); w = np.zeros(kk); cnt = C.c_int(0)
        self._chk(self._f("select_top_k")(_ptr(params, _dp), n, u, v, k, _ptr(idx, _up), _ptr(w, _dp),
                                          C.byref(cnt)), "select_top_k")
        return idx[:cnt.value], w[:cnt.value]

    def topk_points(self, params, uv, k):
        """(reference back-end) global top-K indices and q at many points, OpenMP."""
        params = np.ascontiguousarray(params, np.float64)
        uv = np.ascontiguousarray(uv, np.float64).reshape(-1, 2)
        kk = max(1, min(k, params.shape[0]))
        idx = np.zeros((uv.shape[0], kk), np.uint32); q = np.zeros((uv.shape[0], kk))
        self._chk(self._f("topk_points")(_ptr(params, _dp), params.shape[0], _ptr(uv, _dp), uv.shape[0], k,
                                         _ptr(idx, _up), _ptr(q, _dp)), "topk_points")
        return idx, q

    def bench_render(self, params, pixels, n_max_values, seed, trials=20, warmup=3):
        """(reference back-end) bench_render rows: [baseline] + one per n_max, each
        (n_max, n_b, mean_ms_per_10k, std_ms, mean_candidates)."""
        params = np.ascontiguousarray(params, np.float64)
        nm = np.ascontiguousarray(n_max_values, np.int32)
        out = np.zeros((len(nm) + 1, 5))
        self._chk(self._f("bench_render")(_ptr(params, _dp), params.shape[0], pixels,
                                          nm.ctypes.data_as(_ip), len(nm), seed, trials, warmup, _ptr(out, _dp)),
                  "bench_render")
        return out

    def train_iteration(self, params, m, v, target, sample_idx, k, lr4, t):
        """(reference back-end) train_step_gradients + adam_step in place on params/m/v; returns the loss."""
        for a in (params, m, v):
            assert a.flags.c_contiguous and a.dtype == np.float64
        target = np.ascontiguousarray(target, np.float32)
        sidx = np.ascontiguousarray(sample_idx, np.uint32)
        lr = np.ascontiguousarray(lr4, np.float64)
        H, W, _ = target.shape
        loss = C.c_double(0)
        self._chk(self._f("train_iteration")(_ptr(params, _dp), params.shape[0], _ptr(m, _dp), _ptr(v, _dp),
                                             _ptr(target, _fp), W, H, _ptr(sidx, _up), sidx.shape[0], k,
                                             _ptr(lr, _dp), t, C.byref(loss)), "train_iteration")
        return loss.value

    def render_topk(self, params, uv, k):
        params = np.ascontiguousarray(params, np.float64)
        uv = np.ascontiguousarray(uv, np.float64).reshape(-1, 2)
        out = np.zeros((uv.shape[0], 3))
        self._chk(self._f("render_topk")(_ptr(params, _dp), params.shape[0], _ptr(uv, _dp), uv.shape[0], k,
                                         _ptr(out, _dp)), "render_topk")
        return out

    def render_naive(self, params, uv):
        params = np.ascontiguousarray(params, np.float64)
        uv = np.ascontiguousarray(uv, np.float64).reshape(-1, 2)
        out = np.zeros((uv.shape[0], 3))
        self._chk(self._f("render_naive")(_ptr(params, _dp), params.shape[0], _ptr(uv, _dp), uv.shape[0],
                                          _ptr(out, _dp)), "render_naive")
        return out

    def backward(self, params, samples, k):
        params = np.ascontiguousarray(params, np.float64)
        samples = np.ascontiguousarray(samples, np.float64).reshape(-1, 5)
        g = np.zeros_like(params)
        self._chk(self._f("backward")(_ptr(params, _dp), params.shape[0], _ptr(samples, _dp), samples.shape[0],
                                      k, _ptr(g, _dp)), "backward")
        return g

    def train_step(self, params, target, sample_idx, k):
        params = np.ascontiguousarray(params, np.float64)
        target = np.ascontiguousarray(target, np.float32)
        sidx = np.ascontiguousarray(sample_idx, np.uint32)
        H, W, _ = target.shape
        g = np.zeros_like(params)
        loss = C.c_double(0)
        self._chk(self._f("train_step")(_ptr(params, _dp), params.shape[0], _ptr(target, _fp), W, H,
                                        _ptr(sidx, _up), sidx.shape[0], k, C.byref(loss), _ptr(g, _dp)),
                  "train_step")
        return loss.value, g

    def train_contribs(self, params, target, sample_idx, k, inv_n):
        """(port) per-sample losses, slot keys (n = empty) and [ns][kk][8]
        contributions of a sample block, upstream scaled by inv_n."""
        params = np.ascontiguousarray(params, np.float64)
        target = np.ascontiguousarray(target, np.float32)
        sidx = np.ascontiguousarray(sample_idx, np.uint32)
        H, W, _ = target.shape
        kk = max(1, min(k, params.shape[0]))
        ns = sidx.shape[0]
        losses = np.zeros(ns); keys = np.zeros((ns, kk), np.uint32); contrib = np.zeros((ns, kk, 8))
        self._chk(self._f("train_contribs")(_ptr(params, _dp), params.shape[0], _ptr(target, _fp), W, H,
                                            _ptr(sidx, _up), ns, k, inv_n, _ptr(losses, _dp), _ptr(keys, _up),
                                            _ptr(contrib, _dp)), "train_contribs")
        return losses, keys, contrib

    def adam_step(self, params, grads, m, v, lr4, t):
        """In-place on copies; returns (params, m, v) or raises with .bad set."""
        params = np.array(params, np.float64, copy=True)
        m = np.array(m, np.float64, copy=True)
        v = np.array(v, np.float64, copy=True)
        grads = np.ascontiguousarray(grads, np.float64)
        lr = np.ascontiguousarray(lr4, np.float64)
        bad = C.c_int64(-1)
        code = self._f("adam_step")(_ptr(params, _dp), _ptr(grads, _dp), _ptr(m, _dp), _ptr(v, _dp),
                                    params.shape[0], _ptr(lr, _dp), t, C.byref(bad))
        if code:
            e = OracleError(code, "adam_step")
            e.bad = bad.value
            raise e
        return params, m, v

    def constrain(self, params):
        params = np.array(params, np.float64, copy=True)
        self._chk(self._f("constrain")(_ptr(params, _dp), params.shape[0]), "constrain")
        return params

    def density(self, g8, u, v):
        g8 = np.ascontiguousarray(g8, np.float64)
        return float(self._f("density")(_ptr(g8, _dp), u, v))

    # ---- sampling / metrics -------------------------------------------------
    def image_gradient_magnitude(self, img):
        img = np.ascontiguousarray(img, np.float32)
        H, W, _ = img.shape
        out = np.zeros((H, W))
        self._f("image_gradient_magnitude")(_ptr(img, _fp), W, H, _ptr(out, _dp))
        return out

    def gradient_mixture(self, img, lam):
        img = np.ascontiguousarray(img, np.float32)
        H, W, _ = img.shape
        out = np.zeros((H, W))
        self._chk(self._f("gradient_mixture")(_ptr(img, _fp), W, H, lam, _ptr(out, _dp)), "gradient_mixture")
        return out

    def add_distribution(self, rendered, target):
        rendered = np.ascontiguousarray(rendered, np.float32)
        target = np.ascontiguousarray(target, np.float32)
        if rendered.shape != target.shape:
            raise OracleError(2, "add_distribution")
        H, W, _ = target.shape
        out = np.zeros((H, W))
        self._chk(self._f("add_distribution")(_ptr(rendered, _fp), _ptr(target, _fp), W, H, _ptr(out, _dp)),
                  "add_distribution")
        return out

    def initialize_set(self, img, count, lam, seed):
        img = np.ascontiguousarray(img, np.float32)
        H, W, _ = img.shape
        out = np.zeros((count, 8))
        self._chk(self._f("initialize_set")(_ptr(img, _fp), W, H, count, lam, seed, _ptr(out, _dp)),
                  "initialize_set")
        return out

    def ssim(self, a, b):
        """(reference back-end) ssim(a, b) (metrics.cpp:71-112)."""
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        H, W, _ = a.shape
        return float(self._f("ssim")(_ptr(a, _fp), _ptr(b, _fp), W, H))

    def psnr(self, a, b):
        a = np.ascontiguousarray(a, np.float32).ravel()
        b = np.ascontiguousarray(b, np.float32).ravel()
        return float(self._f("psnr")(_ptr(a, _fp), _ptr(b, _fp), a.size))

    # ---- certified culling (port back-end only) ----------------------------------
    def prepare_scan(self, params):
        params = np.ascontiguousarray(params, np.float64)
        out = np.zeros((params.shape[0], 6))
        self._f("prepare_scan")(_ptr(params, _dp), params.shape[0], _ptr(out, _dp))
        return out

    def cull_lists(self, scan6, W, H, k, T=16):
        scan6 = np.ascontiguousarray(scan6, np.float64)
        n = scan6.shape[0]
        nt = ((W + T - 1) // T) * ((H + T - 1) // T)
        off = np.zeros(nt + 1, np.uint32); tau = np.zeros(nt)
        total = int(self._f("cull_lists")(_ptr(scan6, _dp), n, W, H, k, T, _ptr(off, _up), None, _ptr(tau, _dp)))
        mem = np.zeros(max(total, 1), np.uint32)
        self._f("cull_lists")(_ptr(scan6, _dp), n, W, H, k, T, _ptr(off, _up), _ptr(mem, _up), _ptr(tau, _dp))
        return off, mem[:total], tau

    # ---- encoder (reference back-end) -----------------------------------------
    def fit(self, target, **cfg):
        """The reference's fit(); cfg keys as FitConfig; returns (set, log)."""
        target = np.ascontiguousarray(target, np.float32)
        H, W, _ = target.shape
        c = RefFitConfig(budget=0, k=10, lambda_init=0.3, lambda_opt=0.8, iterations=50000, samples_per_iter=10000,
                         eval_interval=1000, plateau_patience=3, lr_decay=0.1, warmup_iters=10000,
                         densify_interval=5000, seed=0, compute_ssim=1)
        for i, x in enumerate((2e-4, 2e-3, 1e-3, 1e-3)):
            c.lr[i] = x
        for k, v in cfg.items():
            if k == "lr":
                for i, x in enumerate(v):
                    c.lr[i] = x
            else:
                setattr(c, k, v)
        cap = max(c.budget, 8) * 2
        out = np.zeros((cap, 8)); n = C.c_uint32(0); log = C.create_string_buffer(1 << 20)
        self._chk(self._f("fit")(_ptr(target, _fp), W, H, C.byref(c), _ptr(out, _dp), cap, C.byref(n), log,
                                 len(log)), "fit")
        return out[:n.value], log.value.decode()

    # ---- BSP ------------------------------------------------------------------
    def partition_build(self, params, n_max):
        params = np.ascontiguousarray(params, np.float64)
        err = C.c_int(0)
        h = self._f("partition_build")(_ptr(params, _dp), params.shape[0], n_max, C.byref(err))
        self._chk(err.value, "partition_build")
        return Partition(self.lib, h, self.p)

    def partition_rebuild(self, rects, params):
        params = np.ascontiguousarray(params, np.float64)
        rects = np.ascontiguousarray(rects, np.float64).reshape(-1, 4)
        err = C.c_int(0)
        h = self._f("partition_rebuild")(_ptr(rects, _dp), rects.shape[0], _ptr(params, _dp), params.shape[0],
                                         C.byref(err))
        self._chk(err.value, "partition_rebuild")
        return Partition(self.lib, h, self.p)

    def render_image_blocked(self, params, part, W, H, k):
        params = np.ascontiguousarray(params, np.float64)
        out = np.zeros((H, W, 3), np.float32)
        self._chk(self._f("render_image_blocked")(_ptr(params, _dp), params.shape[0], part.h, W, H, k,
                                                  _ptr(out, _fp)), "render_image_blocked")
        return out

    def render_points_blocked(self, params, part, uv, k):
        params = np.ascontiguousarray(params, np.float64)
        uv = np.ascontiguousarray(uv, np.float64).reshape(-1, 2)
        out = np.zeros((uv.shape[0], 3))
        self._chk(self._f("render_points_blocked")(_ptr(params, _dp), params.shape[0], part.h, _ptr(uv, _dp),
                                                   uv.shape[0], k, _ptr(out, _dp)), "render_points_blocked")
        return out


_cache: dict[str, Oracle] = {}


def get(kind: str = "port") -> Oracle:
    if kind not in _cache:
        _cache[kind] = Oracle(kind)
    return _cache[kind]
