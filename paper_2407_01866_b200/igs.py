"""Python binding of the B200 C-ABI (include/igs_b200.h) via ctypes.

Mirrors the reference's hot-path API (proj/include/igs/*.hpp) with the same
names, argument meaning and error kinds:

    reference (C++)                            here (Python)
    render_image(set, W, H, k)                 Context.render_image(W, H, k)
    select_top_k(set, x, k)                    Context.select_top_k(uv, k)
    render_topk(set, x, k)                     Context.render_points(uv, k)
    backward(set, samples, k)                  Context.backward(samples, k)
    train_step_gradients(ps, target, idx, k)   Context.train_step(idx, k)
    adam_step(set, grads, state, lr, t)        Context.adam_step(lr, t)
    add_distribution(rendered, target)         Context.add_distribution(W, H)
    psnr(rendered, target)                     Context.psnr(W, H)
    build_partition(set, n_max)                Context.partition_build(n_max)
    rebuild_partition(blocks, set)             Context.partition_rebuild(rects)
    render_image_blocked(set, p, W, H, k)      Context.render_image_blocked(W, H, k)
    render_topk_blocked(set, p, x, k)          Context.render_points_blocked(uv, k)
    locate_block(p, x)                         Context.locate_blocks(uv)

The Gaussian set is device-resident in the Context (set_params /
append_params / get_params); records are the reference's 8-double layout.
Errors raise IgsError whose .kind is the reference ErrorKind name.

There is no CPU fallback: importing this module without the built CUDA
extension raises, and every call runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

# IGS_B200_LIB: an alternative build of the same library (kernel-tuning
# experiments); it must exist -- there is no fallback.
LIB_PATH = Path(os.environ.get("IGS_B200_LIB") or Path(__file__).resolve().parent / "libigs_b200.so")

ERROR_KINDS = {
    1: "invalid_parameter",
    2: "dimension_mismatch",
    3: "bad_magic",
    4: "bad_version",
    5: "truncated",
    6: "empty_set",
    7: "io",
    8: "unsupported_format",
    100: "cuda",
}

OPT_CULL, OPT_DETERMINISTIC, OPT_TILE, OPT_RASTER, OPT_SHARD_ADAM = 1, 2, 3, 4, 5
PROF_SCAN, PROF_FINISH, PROF_REDUCE, PROF_ADAM, PROF_CULL, PROF_BLOCKED, PROF_KNN_HARD = range(7)
PROF_NAMES = ["scan", "finish", "reduce", "adam", "cull", "blocked", "knn_hard"]

# Learning rates in the reference's LearningRates field order (adam.hpp:11-16).
DEFAULT_LR = (2e-4, 2e-3, 1e-3, 1e-3)  # mu, color, scale, theta
DEFAULT_K = 10  # renderer.hpp:16 kDefaultTopK


class FitConfig(C.Structure):
    """igs_fit_config == FitConfig (fit.hpp:19-33) + compute_ssim."""
    _fields_ = [("budget", C.c_int), ("k", C.c_int), ("lambda_init", C.c_double), ("lambda_opt", C.c_double),
                ("iterations", C.c_int), ("samples_per_iter", C.c_int), ("lr", C.c_double * 4),
                ("eval_interval", C.c_int), ("plateau_patience", C.c_int), ("lr_decay", C.c_double),
                ("warmup_iters", C.c_int), ("densify_interval", C.c_int), ("seed", C.c_uint64),
                ("compute_ssim", C.c_int)]


class EvalRecord(C.Structure):
    _fields_ = [("iteration", C.c_int), ("count", C.c_int), ("loss", C.c_double), ("psnr", C.c_double),
                ("ssim", C.c_double), ("best_psnr", C.c_double)]


CHECKPOINT_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.POINTER(C.c_double), C.c_uint32)


class BenchRow(C.Structure):
    _fields_ = [("n_max", C.c_int), ("n_b", C.c_int), ("mean_ms_per_10k", C.c_double), ("std_ms", C.c_double),
                ("mean_candidates", C.c_double)]


class IgsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        self.kind = ERROR_KINDS.get(code, f"code{code}")
        super().__init__(f"[{self.kind}] {msg}")


_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_up = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p

# name -> (restype, argtypes); the full export set of include/igs_b200.h
SIGNATURES = {
    "igs_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "igs_ctx_destroy": (None, [_vp]),
    "igs_last_error": (C.c_char_p, [_vp]),
    "igs_sync": (C.c_int, [_vp]),
    "igs_kernel_launches": (C.c_uint64, [_vp]),
    "igs_set_option": (C.c_int, [_vp, C.c_int, C.c_int64]),
    "igs_get_option": (C.c_int64, [_vp, C.c_int]),
    "igs_set_params": (C.c_int, [_vp, _dp, C.c_uint32]),
    "igs_append_params": (C.c_int, [_vp, _dp, C.c_uint32]),
    "igs_get_params": (C.c_int, [_vp, _dp, C.c_uint32]),
    "igs_num_gaussians": (C.c_uint32, [_vp]),
    "igs_device_params": (_vp, [_vp]),
    "igs_render_image": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _fp, _up]),
    "igs_render_image_rows": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _fp]),
    "igs_device_image": (_vp, [_vp]),
    "igs_select_top_k": (C.c_int, [_vp, _dp, C.c_uint32, C.c_int, _up, _dp, _i32p]),
    "igs_render_points": (C.c_int, [_vp, _dp, C.c_uint32, C.c_int, _dp]),
    "igs_backward": (C.c_int, [_vp, _dp, C.c_uint32, C.c_int, _dp]),
    "igs_set_target": (C.c_int, [_vp, _fp, C.c_int, C.c_int]),
    "igs_train_step": (C.c_int, [_vp, _up, C.c_uint32, C.c_int, _dp, _dp]),
    "igs_adam_step": (C.c_int, [_vp, _dp, C.c_longlong]),
    "igs_train_iteration": (C.c_int, [_vp, _up, C.c_uint32, C.c_int, _dp, C.c_longlong, _dp]),
    "igs_upload_samples": (C.c_int, [_vp, _up, C.c_uint32, C.c_uint32]),
    "igs_train_iterations": (C.c_int, [_vp, C.c_uint32, C.c_int, _dp, C.c_longlong, _dp]),
    "igs_device_grads": (_vp, [_vp]),
    "igs_get_grads": (C.c_int, [_vp, _dp, C.c_uint32]),
    "igs_set_grads": (C.c_int, [_vp, _dp, C.c_uint32]),
    "igs_get_adam_state": (C.c_int, [_vp, _dp, _dp, C.c_uint32]),
    "igs_set_adam_state": (C.c_int, [_vp, _dp, _dp, C.c_uint32]),
    "igs_add_distribution": (C.c_int, [_vp, _fp, C.c_int, C.c_int, _dp]),
    "igs_psnr": (C.c_int, [_vp, _fp, C.c_int, C.c_int, _dp]),
    "igs_partition_build": (C.c_int, [_vp, C.c_int]),
    "igs_partition_rebuild": (C.c_int, [_vp, _dp, C.c_uint32]),
    "igs_partition_info": (C.c_int, [_vp, _up, _u64p]),
    "igs_partition_get": (C.c_int, [_vp, _dp, _dp, _up, _up]),
    "igs_encode": (C.c_int, [_vp, C.c_int, C.c_uint32, C.c_uint32, C.c_int, _u8p, C.c_size_t,
                             C.POINTER(C.c_size_t)]),
    "igs_decode": (C.c_int, [_vp, _u8p, C.c_size_t, _up, _up, C.POINTER(C.c_int), _up]),
    "igs_quantize_set": (C.c_int, [_vp]),
    "igs_locate_blocks": (C.c_int, [_vp, _dp, C.c_uint32, _i32p]),
    "igs_partition_export": (C.c_int, [_vp, C.POINTER(C.c_int), _up, _i32p, _up, C.POINTER(C.c_int), _up]),
    "igs_partition_get_tree": (C.c_int, [_vp, _i32p, _dp]),
    "igs_partition_get_grid": (C.c_int, [_vp, _up, _up]),
    "igs_partition_block_members": (C.c_int, [_vp, _up, _up]),
    "igs_partition_set": (C.c_int, [_vp, _dp, C.c_uint32, _i32p, _dp, C.c_uint32, C.c_int32, C.c_int, C.c_uint32]),
    "igs_render_image_blocked": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _fp]),
    "igs_render_image_blocked_rows": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _fp]),
    "igs_render_points_blocked": (C.c_int, [_vp, _dp, C.c_uint32, C.c_int, _dp]),
    "igs_get_prepared": (C.c_int, [_vp, _dp, C.c_uint32]),
    "igs_tile_lists": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, _up, _u64p, _up, _up, _dp]),
    "igs_timer_begin": (C.c_int, [_vp]),
    "igs_timer_end": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "igs_timer_mark": (C.c_int, [_vp, C.c_uint32]),
    "igs_timer_between": (C.c_int, [_vp, C.c_uint32, C.c_uint32, C.POINTER(C.c_float)]),
    "igs_flush_l2": (C.c_int, [_vp, C.c_size_t]),
    "igs_fp64_peak": (C.c_int, [_vp, _dp]),
    "igs_libm_eval": (C.c_int, [_vp, _dp, C.c_uint32, _dp]),
    "igs_debug_scan": (C.c_int, [_vp, _up, C.c_uint32, _up]),
    "igs_debug_sort_pairs": (C.c_int, [_vp, _u64p, _up, C.c_uint32, C.c_int, _u64p, _up]),
    "igs_bench_render": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_int), C.c_int, C.c_uint64, C.c_int, C.c_int,
                                   C.POINTER(BenchRow)]),
    "igs_profile_enable": (C.c_int, [_vp, C.c_int]),
    "igs_profile_read": (C.c_int, [_vp, C.c_int, _dp, _u64p, _dp]),
    "igs_train_iteration_async": (C.c_int, [_vp, _up, C.c_uint32, C.c_int, _dp, C.c_longlong]),
    "igs_train_wait": (C.c_int, [_vp, _dp]),
    "igs_ssim": (C.c_int, [_vp, _fp, C.c_int, C.c_int, _dp]),
    "igs_image_gradient_magnitude": (C.c_int, [_vp, _fp, C.c_int, C.c_int, _dp]),
    "igs_gradient_mixture": (C.c_int, [_vp, _fp, C.c_int, C.c_int, C.c_double, _dp]),
    "igs_initialize_set": (C.c_int, [_vp, _fp, C.c_int, C.c_int, C.c_int, C.c_double, _u64p, _dp]),
    "igs_fit_config_default": (None, [C.POINTER(FitConfig)]),
    "igs_fit": (C.c_int, [_vp, _fp, C.c_int, C.c_int, C.POINTER(FitConfig), CHECKPOINT_FN, C.c_void_p,
                          C.POINTER(EvalRecord), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                          C.POINTER(C.c_int), C.c_char_p, C.c_size_t]),
    "igs_comm_unique_id": (C.c_int, [_u8p]),
    "igs_comm_init": (C.c_int, [_vp, _u8p, C.c_int, C.c_int]),
    "igs_comm_destroy": (C.c_int, [_vp]),
    "igs_comm_init_loopback": (C.c_int, [C.POINTER(_vp), C.c_int]),
    "igs_comm_gather_moments": (C.c_int, [_vp]),
}

_lib = None


def load_library() -> C.CDLL:
    """Loads libigs_b200.so; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _f64(a, shape_last=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape_last is not None:
        a = a.reshape(-1, shape_last)
    return a


class Context:
    """One GPU context (igs_ctx): device-resident set, Adam state, images."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = _vp()
        code = self.lib.igs_ctx_create(device, C.byref(h))
        if code:
            raise IgsError(code, f"igs_ctx_create(device={device}) failed (no CUDA device?)")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.igs_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _chk(self, code):
        if code:
            raise IgsError(code, (self.lib.igs_last_error(self.h) or b"").decode())

    # ---- options / diagnostics ---------------------------------------------
    def set_option(self, opt: int, value: int):
        self._chk(self.lib.igs_set_option(self.h, opt, int(value)))

    def get_option(self, opt: int) -> int:
        return int(self.lib.igs_get_option(self.h, opt))

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.igs_kernel_launches(self.h))

    def sync(self):
        self._chk(self.lib.igs_sync(self.h))

    # ---- set -----------------------------------------------------------------
    @property
    def n(self) -> int:
        return int(self.lib.igs_num_gaussians(self.h))

    def set_params(self, params):
        p = _f64(params, 8)
        self._chk(self.lib.igs_set_params(self.h, _p(p, _dp), p.shape[0]))

    def append_params(self, params):
        p = _f64(params, 8)
        self._chk(self.lib.igs_append_params(self.h, _p(p, _dp), p.shape[0]))

    def get_params(self):
        out = np.zeros((self.n, 8))
        self._chk(self.lib.igs_get_params(self.h, _p(out, _dp), out.shape[0]))
        return out

    # ---- renderer ---------------------------------------------------------------
    def render_image(self, width: int, height: int, k: int = DEFAULT_K, want_topk: bool = False, host: bool = True):
        out = np.zeros((height, width, 3), np.float32) if host else None
        topk = None
        if want_topk:
            kk = max(1, min(k, self.n))
            topk = np.zeros((height, width, kk), np.uint32)
        self._chk(self.lib.igs_render_image(self.h, width, height, k, _p(out, _fp), _p(topk, _up)))
        return (out, topk) if want_topk else out

    def render_image_rows(self, width: int, height: int, k: int, row0: int, row1: int, host: bool = True):
        out = np.zeros((row1 - row0, width, 3), np.float32) if host else None
        self._chk(self.lib.igs_render_image_rows(self.h, width, height, k, row0, row1, _p(out, _fp)))
        return out

    def select_top_k(self, uv, k: int = DEFAULT_K):
        uv = _f64(uv, 2)
        kk = max(1, min(k, self.n))
        idx = np.zeros((uv.shape[0], kk), np.uint32)
        w = np.zeros((uv.shape[0], kk))
        cnt = np.zeros(uv.shape[0], np.int32)
        self._chk(self.lib.igs_select_top_k(self.h, _p(uv, _dp), uv.shape[0], k, _p(idx, _up), _p(w, _dp),
                                            _p(cnt, _i32p)))
        return idx, w, cnt

    def render_points(self, uv, k: int = DEFAULT_K):
        uv = _f64(uv, 2)
        out = np.zeros((uv.shape[0], 3))
        self._chk(self.lib.igs_render_points(self.h, _p(uv, _dp), uv.shape[0], k, _p(out, _dp)))
        return out

    def backward(self, samples, k: int = DEFAULT_K):
        s = _f64(samples, 5)
        out = np.zeros((self.n, 8))
        self._chk(self.lib.igs_backward(self.h, _p(s, _dp), s.shape[0], k, _p(out, _dp)))
        return out

    # ---- training -------------------------------------------------------------------
    def set_target(self, img):
        img = np.ascontiguousarray(img, np.float32)
        H, W, _ = img.shape
        self._chk(self.lib.igs_set_target(self.h, _p(img, _fp), W, H))

    def train_step(self, sample_idx, k: int = DEFAULT_K, want_grads: bool = True):
        s = np.ascontiguousarray(sample_idx, np.uint32)
        loss = C.c_double(0)
        g = np.zeros((self.n, 8)) if want_grads else None
        self._chk(self.lib.igs_train_step(self.h, _p(s, _up), s.shape[0], k, C.byref(loss), _p(g, _dp)))
        return loss.value, g

    def adam_step(self, lr=DEFAULT_LR, t: int = 1):
        lr = np.ascontiguousarray(lr, np.float64)
        self._chk(self.lib.igs_adam_step(self.h, _p(lr, _dp), int(t)))

    def train_iteration(self, sample_idx, k: int = DEFAULT_K, lr=DEFAULT_LR, t: int = 1) -> float:
        s = np.ascontiguousarray(sample_idx, np.uint32)
        lr = np.ascontiguousarray(lr, np.float64)
        loss = C.c_double(0)
        self._chk(self.lib.igs_train_iteration(self.h, _p(s, _up), s.shape[0], k, _p(lr, _dp), int(t),
                                               C.byref(loss)))
        return loss.value

    def upload_samples(self, sample_idx_steps):
        s = np.ascontiguousarray(sample_idx_steps, np.uint32)
        steps, ns = s.shape
        self._chk(self.lib.igs_upload_samples(self.h, _p(s, _up), ns, steps))

    def train_iterations(self, steps: int, k: int = DEFAULT_K, lr=DEFAULT_LR, t0: int = 1, want_losses=True):
        lr = np.ascontiguousarray(lr, np.float64)
        losses = np.zeros(steps) if want_losses else None
        self._chk(self.lib.igs_train_iterations(self.h, steps, k, _p(lr, _dp), int(t0), _p(losses, _dp)))
        return losses

    def get_grads(self):
        out = np.zeros((self.n, 8))
        self._chk(self.lib.igs_get_grads(self.h, _p(out, _dp), out.shape[0]))
        return out

    def set_grads(self, grads):
        g = _f64(grads, 8)
        self._chk(self.lib.igs_set_grads(self.h, _p(g, _dp), g.shape[0]))

    def get_adam_state(self):
        m = np.zeros((self.n, 8)); v = np.zeros((self.n, 8))
        self._chk(self.lib.igs_get_adam_state(self.h, _p(m, _dp), _p(v, _dp), self.n))
        return m, v

    def set_adam_state(self, m, v):
        m = _f64(m, 8); v = _f64(v, 8)
        self._chk(self.lib.igs_set_adam_state(self.h, _p(m, _dp), _p(v, _dp), m.shape[0]))

    # ---- error map / metrics -----------------------------------------------------------
    def add_distribution(self, width: int, height: int, rendered=None):
        r = None if rendered is None else np.ascontiguousarray(rendered, np.float32)
        out = np.zeros((height, width))
        self._chk(self.lib.igs_add_distribution(self.h, _p(r, _fp), width, height, _p(out, _dp)))
        return out

    def psnr(self, width: int, height: int, rendered=None) -> float:
        r = None if rendered is None else np.ascontiguousarray(rendered, np.float32)
        out = C.c_double(0)
        self._chk(self.lib.igs_psnr(self.h, _p(r, _fp), width, height, C.byref(out)))
        return out.value

    def ssim(self, width: int, height: int, rendered=None) -> float:
        r = None if rendered is None else np.ascontiguousarray(rendered, np.float32)
        out = C.c_double(0)
        self._chk(self.lib.igs_ssim(self.h, _p(r, _fp), width, height, C.byref(out)))
        return out.value

    def image_gradient_magnitude(self, img=None, width: int = 0, height: int = 0):
        """sampling.cpp:44-67 on the device; img None = the resident target."""
        if img is not None:
            img = np.ascontiguousarray(img, np.float32)
            height, width = img.shape[:2]
        out = np.zeros((height, width))
        self._chk(self.lib.igs_image_gradient_magnitude(self.h, _p(img, _fp), width, height, _p(out, _dp)))
        return out

    def gradient_mixture(self, img, lam: float):
        """init/opt_distribution (sampling.cpp:25-40)."""
        img = np.ascontiguousarray(img, np.float32)
        H, W = img.shape[:2]
        out = np.zeros((H, W))
        self._chk(self.lib.igs_gradient_mixture(self.h, _p(img, _fp), W, H, lam, _p(out, _dp)))
        return out

    def initialize_set(self, img, count: int, lam: float, raw2):
        """initialize_set (sampling.cpp:154-174) drawing from 2*count raw engine outputs."""
        img = np.ascontiguousarray(img, np.float32)
        H, W = img.shape[:2]
        raw2 = np.ascontiguousarray(raw2, np.uint64)
        out = np.zeros((count, 8))
        self._chk(self.lib.igs_initialize_set(self.h, _p(img, _fp), W, H, count, lam, _p(raw2, _u64p), _p(out, _dp)))
        return out

    def train_iteration_async(self, sample_idx, k: int = DEFAULT_K, lr=DEFAULT_LR, t: int = 1):
        self._async_keep = np.ascontiguousarray(sample_idx, np.uint32)
        lr = np.ascontiguousarray(lr, np.float64)
        self._chk(self.lib.igs_train_iteration_async(self.h, _p(self._async_keep, _up), self._async_keep.shape[0],
                                                     k, _p(lr, _dp), int(t)))

    def train_wait(self) -> float:
        loss = C.c_double(0)
        self._chk(self.lib.igs_train_wait(self.h, C.byref(loss)))
        return loss.value

    # ---- encoder (fit.cpp) -----------------------------------------------------------------
    @staticmethod
    def fit_config(**overrides) -> FitConfig:
        cfg = FitConfig()
        load_library().igs_fit_config_default(C.byref(cfg))
        for k, v in overrides.items():
            if k == "lr":
                for i, x in enumerate(v):
                    cfg.lr[i] = x
            else:
                setattr(cfg, k, v)
        return cfg

    def fit(self, target, config: FitConfig, on_checkpoint=None, max_evals: int = 4096):
        """fit() on the device; returns a dict like FitReport + the log text.
        on_checkpoint(stage, iteration, id, params (n, 8)) mirrors CheckpointFn."""
        target = np.ascontiguousarray(target, np.float32)
        H, W, _ = target.shape

        def _cb(user, stage, iteration, cid, p, n):
            if on_checkpoint is not None:
                arr = np.ctypeslib.as_array(p, shape=(n * 8,)).reshape(n, 8).copy() if n else np.zeros((0, 8))
                on_checkpoint(stage, iteration, cid.decode(), arr)

        cb = CHECKPOINT_FN(_cb)
        evals = (EvalRecord * max_evals)()
        n_evals = C.c_int(0); decay = C.c_int(-1); final = C.c_int(0)
        log = C.create_string_buffer(1 << 20)
        self._chk(self.lib.igs_fit(self.h, _p(target, _fp), W, H, C.byref(config), cb, None, evals, max_evals,
                                   C.byref(n_evals), C.byref(decay), C.byref(final), log, len(log)))
        recs = [dict(iteration=e.iteration, count=e.count, loss=e.loss, psnr=e.psnr, ssim=e.ssim,
                     best_psnr=e.best_psnr) for e in evals[:n_evals.value]]
        return {"evals": recs, "lr_decay_iteration": decay.value, "final_count": final.value,
                "log": log.value.decode()}

    # ---- BSP ------------------------------------------------------------------------------
    def partition_build(self, n_max: int):
        self._chk(self.lib.igs_partition_build(self.h, n_max))

    def partition_rebuild(self, rects):
        r = _f64(rects, 4)
        self._chk(self.lib.igs_partition_rebuild(self.h, _p(r, _dp), r.shape[0]))

    def partition_info(self):
        nb = C.c_uint32(0); tot = C.c_uint64(0)
        self._chk(self.lib.igs_partition_info(self.h, C.byref(nb), C.byref(tot)))
        return nb.value, tot.value

    def partition_get(self):
        nb, tot = self.partition_info()
        b = np.zeros((nb, 4)); s = np.zeros((nb, 4))
        off = np.zeros(nb + 1, np.uint32); mem = np.zeros(max(tot, 1), np.uint32)
        self._chk(self.lib.igs_partition_get(self.h, _p(b, _dp), _p(s, _dp), _p(off, _up), _p(mem, _up)))
        return b, s, off, mem[:tot]

    # ---- IGS2 container (codec.cpp) ---------------------------------------------------------
    def encode(self, width: int, height: int, k: int = DEFAULT_K, with_partition: bool = False) -> bytes:
        size = C.c_size_t(0)
        self._chk(self.lib.igs_encode(self.h, int(with_partition), width, height, k, None, 0, C.byref(size)))
        out = np.zeros(size.value, np.uint8)
        self._chk(self.lib.igs_encode(self.h, int(with_partition), width, height, k, _p(out, _u8p), out.size,
                                      C.byref(size)))
        return out.tobytes()

    def decode(self, data: bytes) -> dict:
        """The set becomes the resident set (and the partition, if the file has
        blocks); returns the header fields."""
        buf = np.frombuffer(bytes(data), np.uint8).copy()
        w = C.c_uint32(0); h = C.c_uint32(0); k = C.c_int(0); nb = C.c_uint32(0)
        self._chk(self.lib.igs_decode(self.h, _p(buf, _u8p) if buf.size else None, buf.size, C.byref(w), C.byref(h),
                                      C.byref(k), C.byref(nb)))
        return {"width": w.value, "height": h.value, "k": k.value, "n_blocks": nb.value}

    def quantize_set(self):
        self._chk(self.lib.igs_quantize_set(self.h))

    def partition_block_members(self):
        nb, _ = self.partition_info()
        off = np.zeros(nb + 1, np.uint32)
        self._chk(self.lib.igs_partition_block_members(self.h, _p(off, _up), None))
        mem = np.zeros(max(int(off[-1]), 1), np.uint32)
        self._chk(self.lib.igs_partition_block_members(self.h, _p(off, _up), _p(mem, _up)))
        return off, mem[:int(off[-1])]

    def partition_tree(self):
        """(root, nodes [n x 4: axis, low, high, block], lines) of a built partition."""
        n_max = C.c_int(0); src = C.c_uint32(0); root = C.c_int32(0); nn = C.c_uint32(0)
        gd = C.c_int(0); gt = C.c_uint32(0)
        self._chk(self.lib.igs_partition_export(self.h, C.byref(n_max), C.byref(src), C.byref(root), C.byref(nn),
                                                C.byref(gd), C.byref(gt)))
        nodes = np.zeros((max(nn.value, 1), 4), np.int32); lines = np.zeros(max(nn.value, 1))
        self._chk(self.lib.igs_partition_get_tree(self.h, _p(nodes, _i32p), _p(lines, _dp)))
        return root.value, nodes[:nn.value], lines[:nn.value]

    def partition_set(self, blocks, nodes=None, lines=None, root=-1, n_max=0, source_size=None):
        b = _f64(blocks, 4)
        nn = 0 if nodes is None else len(nodes)
        nd = None if nodes is None else np.ascontiguousarray(nodes, np.int32)
        ln = None if lines is None else np.ascontiguousarray(lines, np.float64)
        self._chk(self.lib.igs_partition_set(self.h, _p(b, _dp), b.shape[0], _p(nd, _i32p), _p(ln, _dp), nn, root,
                                             n_max, self.n if source_size is None else source_size))

    def locate_blocks(self, uv):
        uv = _f64(uv, 2)
        out = np.zeros(uv.shape[0], np.int32)
        self._chk(self.lib.igs_locate_blocks(self.h, _p(uv, _dp), uv.shape[0], _p(out, _i32p)))
        return out

    def render_image_blocked(self, width: int, height: int, k: int = DEFAULT_K, host: bool = True):
        out = np.zeros((height, width, 3), np.float32) if host else None
        self._chk(self.lib.igs_render_image_blocked(self.h, width, height, k, _p(out, _fp)))
        return out

    def render_image_blocked_rows(self, width: int, height: int, k: int, row0: int, row1: int):
        out = np.zeros((row1 - row0, width, 3), np.float32)
        self._chk(self.lib.igs_render_image_blocked_rows(self.h, width, height, k, row0, row1, _p(out, _fp)))
        return out

    def render_points_blocked(self, uv, k: int = DEFAULT_K):
        uv = _f64(uv, 2)
        out = np.zeros((uv.shape[0], 3))
        self._chk(self.lib.igs_render_points_blocked(self.h, _p(uv, _dp), uv.shape[0], k, _p(out, _dp)))
        return out

    def get_prepared(self):
        out = np.zeros((self.n, 6))
        self._chk(self.lib.igs_get_prepared(self.h, _p(out, _dp), out.shape[0]))
        return out

    # ---- culling introspection -------------------------------------------------------------
    def tile_lists(self, width: int, height: int, k: int = DEFAULT_K):
        nt = C.c_uint32(0); tot = C.c_uint64(0)
        self._chk(self.lib.igs_tile_lists(self.h, width, height, k, C.byref(nt), C.byref(tot), None, None, None))
        off = np.zeros(nt.value + 1, np.uint32); mem = np.zeros(max(tot.value, 1), np.uint32)
        tau = np.zeros(nt.value)
        self._chk(self.lib.igs_tile_lists(self.h, width, height, k, C.byref(nt), C.byref(tot), _p(off, _up),
                                          _p(mem, _up), _p(tau, _dp)))
        return off, mem[:tot.value], tau

    # ---- benchmark support ----------------------------------------------------------------------
    def timer_begin(self):
        self._chk(self.lib.igs_timer_begin(self.h))

    def timer_end(self) -> float:
        ms = C.c_float(0)
        self._chk(self.lib.igs_timer_end(self.h, C.byref(ms)))
        return ms.value

    def timer_mark(self, idx: int):
        self._chk(self.lib.igs_timer_mark(self.h, idx))

    def timer_between(self, a: int, b: int) -> float:
        ms = C.c_float(0)
        self._chk(self.lib.igs_timer_between(self.h, a, b, C.byref(ms)))
        return ms.value

    def flush_l2(self, nbytes: int = 512 << 20):
        self._chk(self.lib.igs_flush_l2(self.h, nbytes))

    def fp64_peak(self) -> float:
        out = C.c_double(0)
        self._chk(self.lib.igs_fp64_peak(self.h, C.byref(out)))
        return out.value

    def bench_render(self, pixels: int, n_max_values, seed: int, trials: int = 20, warmup: int = 3):
        """bench_render (bsp.cpp:343-406): [baseline] + one row per n_max as dicts."""
        nm = (C.c_int * max(len(n_max_values), 1))(*n_max_values)
        rows = (BenchRow * (len(n_max_values) + 1))()
        self._chk(self.lib.igs_bench_render(self.h, pixels, nm, len(n_max_values), seed, trials, warmup, rows))
        return [{f: getattr(r, f) for f, _ in BenchRow._fields_} for r in rows]

    def debug_scan(self, a):
        """Device exclusive scan (kernel 2's primitive) of a u32 array."""
        a = np.ascontiguousarray(a, np.uint32)
        out = np.zeros_like(a)
        self._chk(self.lib.igs_debug_scan(self.h, _p(a, _up), a.size, _p(out, _up)))
        return out

    def debug_sort_pairs(self, keys, vals, bits: int = 64):
        """Device stable LSD radix sort of (u64 key, u32 value) pairs."""
        keys = np.ascontiguousarray(keys, np.uint64)
        vals = np.ascontiguousarray(vals, np.uint32)
        ko, vo = np.zeros_like(keys), np.zeros_like(vals)
        self._chk(self.lib.igs_debug_sort_pairs(self.h, _p(keys, _u64p), _p(vals, _up), keys.size, bits,
                                                _p(ko, _u64p), _p(vo, _up)))
        return ko, vo

    def libm_eval(self, x):
        """Device glibc-exact (exp, sin, cos) of each x (parity diagnostics)."""
        x = np.ascontiguousarray(x, np.float64).ravel()
        out = np.zeros((x.size, 3))
        self._chk(self.lib.igs_libm_eval(self.h, _p(x, _dp), x.size, _p(out, _dp)))
        return out

    def profile_enable(self, on: bool = True):
        self._chk(self.lib.igs_profile_enable(self.h, 1 if on else 0))

    def profile_read(self, family: int):
        ms = C.c_double(0); n = C.c_uint64(0); work = C.c_double(0)
        self._chk(self.lib.igs_profile_read(self.h, family, C.byref(ms), C.byref(n), C.byref(work)))
        return ms.value, n.value, work.value

    # ---- multi-GPU ---------------------------------------------------------------------------
    @staticmethod
    def comm_unique_id() -> bytes:
        lib = load_library()
        buf = (C.c_uint8 * 128)()
        code = lib.igs_comm_unique_id(buf)
        if code:
            raise IgsError(code, "ncclGetUniqueId failed")
        return bytes(buf)

    def comm_init(self, uid: bytes, nranks: int, rank: int):
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        self._chk(self.lib.igs_comm_init(self.h, buf, nranks, rank))

    @staticmethod
    def comm_init_loopback(ctxs):
        """Joins the contexts into one in-process loopback group (rank = list
        position); drive each from its own thread afterwards."""
        arr = (_vp * len(ctxs))(*[c.h for c in ctxs])
        code = load_library().igs_comm_init_loopback(arr, len(ctxs))
        if code:
            raise IgsError(code, ctxs[0].lib.igs_last_error(ctxs[0].h).decode() if ctxs else "")

    def comm_gather_moments(self):
        """(collective) re-replicate the sharded Adam moments on every rank."""
        self._chk(self.lib.igs_comm_gather_moments(self.h))

    def comm_destroy(self):
        self._chk(self.lib.igs_comm_destroy(self.h))
