"""Python mirror of the reference engine API over the C-ABI (include/gridshift_c.h).

The reference's boundary is the C++ call ``gridshift::run(Dataset, EngineConfig) ->
ClusterLabeling`` (types :107-114) with the exception
taxonomy of /root/reference/proj/include/gridshift/errors.hpp.  This module keeps those names
(``EngineConfig``, ``ClusterLabeling``, ``run``, ``InvalidBandwidthError`` ...) so the parity
tests read like the reference's own, and routes every call to ``libgridshift_cuda.so``.  There
is no CPU fallback: without the library or a device the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libgridshift_cuda.so")

# ----------------------------------------------------------------------------- errors
class Error(RuntimeError):
    """gridshift::Error (errors.hpp:9-11)."""


class InvalidInputError(Error):
    """errors.hpp:14-16."""


class InvalidBandwidthError(InvalidInputError):
    """errors.hpp:18-20 (h <= 0)."""


class EmptyInputError(InvalidInputError):
    """errors.hpp:22-24 (n == 0)."""


class InvalidParameterError(InvalidInputError):
    """errors.hpp:26-28."""


class InternalInvariantError(Error):
    """errors.hpp:31-33."""


class UndefinedScoreError(Error):
    """errors.hpp:36-38 (silhouette of fewer than 2 clusters)."""


class TuningFailureError(Error):
    """errors.hpp:41-43 (no bandwidth gave a scorable clustering)."""


class InvalidWindowError(InvalidInputError):
    """errors.hpp:55-57 (tracking window outside the frame)."""


class SelectionError(InvalidInputError):
    """errors.hpp:59-61 (selected cluster does not exist)."""


GS_OK = 0
_STATUS = {
    1: InvalidInputError,
    2: InvalidBandwidthError,
    3: EmptyInputError,
    4: InvalidParameterError,
    5: InternalInvariantError,
    6: InvalidParameterError,  # GS_E_KEY_RANGE
    7: Error,  # GS_E_CUDA
    8: Error,  # GS_E_OOM
    9: Error,  # GS_E_NCCL
    10: Error,  # GS_E_NO_DEVICE
    11: TuningFailureError,
    12: UndefinedScoreError,
    13: InvalidWindowError,
    14: SelectionError,
}
STATUS_NAMES = {
    0: "GS_OK", 1: "GS_E_INVALID_INPUT", 2: "GS_E_INVALID_BANDWIDTH", 3: "GS_E_EMPTY_INPUT",
    4: "GS_E_INVALID_PARAMETER", 5: "GS_E_INTERNAL_INVARIANT", 6: "GS_E_KEY_RANGE",
    7: "GS_E_CUDA", 8: "GS_E_OOM", 9: "GS_E_NCCL", 10: "GS_E_NO_DEVICE",
    11: "GS_E_TUNING_FAILED", 12: "GS_E_UNDEFINED_SCORE", 13: "GS_E_INVALID_WINDOW",
    14: "GS_E_SELECTION",
}

GS_F32, GS_F64, GS_U8 = 0, 1, 2
GS_RECORD_HISTORY, GS_DEVICE_OUTPUTS = 0x1, 0x2
GS_TIME_PHASES, GS_TIME_KERNEL = 0x4, 0x8
GS_NO_PIPELINE = 0x10
GS_DEBUG_GLOBAL_PATH = 0x80000000
GS_DEBUG_PIPELINE = 0x40000000
GS_DEBUG_SWEEP_FLOW = 0x20000000
GS_DEBUG_SWEEP_LEVELS = 0x10000000
GS_DEBUG_SWEEP_SINGLE = 0x08000000

# every symbol include/gridshift_c.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "gs_validate", "gs_create", "gs_destroy", "gs_run", "gs_get_centroids", "gs_get_history",
    "gs_get_stats", "gs_last_error", "gs_status_string", "gs_debug_build",
    "gs_debug_iterate_once", "gs_debug_resident_once", "gs_fixed_shift", "gs_shard_keybounds", "gs_shard_bin",
    "gs_shard_run", "gs_render", "gs_tuner_create", "gs_tuner_destroy", "gs_tuner_last_error",
    "gs_tune_bandwidth", "gs_silhouette_subsampled", "gs_tracker_create", "gs_tracker_destroy",
    "gs_tracker_last_error", "gs_track_init", "gs_track_sequence", "gs_mspp_run",
    "gs_dist_create", "gs_dist_destroy", "gs_dist_last_error", "gs_dist_run_frames",
    "gs_dist_run_slabs", "gs_dist_get_centroids", "gs_dist_get_history",
]


class GsInput(C.Structure):
    _fields_ = [("points", C.c_void_p), ("n", C.c_int64), ("d", C.c_int32),
                ("dtype", C.c_int32), ("batch", C.c_int64), ("on_device", C.c_int32),
                ("reserved", C.c_int32)]


class GsConfig(C.Structure):
    _fields_ = [("h", C.c_double), ("max_iter", C.c_int32), ("flags", C.c_uint32)]


class GsResult(C.Structure):
    _fields_ = [("labels", C.c_void_p), ("k", C.c_void_p), ("iterations", C.c_void_p),
                ("converged", C.c_void_p)]


class GsStats(C.Structure):
    _fields_ = [("ms_total", C.c_double), ("ms_bin", C.c_double), ("ms_iterate", C.c_double),
                ("ms_label", C.c_double), ("ms_h2d", C.c_double), ("ms_d2h", C.c_double),
                ("cells_swept", C.c_int64), ("m0", C.c_int64), ("k_total", C.c_int64),
                ("kernel_launches", C.c_int64), ("max_iterations", C.c_int32),
                ("fixed_shift", C.c_int32), ("dense_cells", C.c_int64),
                ("ms_k_bin", C.c_double), ("ms_k_label", C.c_double), ("lib_calls", C.c_int64),
                ("sweep_modes", C.c_int64 * 3), ("resident_cycles", C.c_int64 * 8),
                ("slot_bytes", C.c_int32), ("predicted_box", C.c_int32)]


class GsSweepEntry(C.Structure):
    _fields_ = [("h", C.c_double), ("score", C.c_double), ("k", C.c_int64),
                ("iterations", C.c_int32), ("converged", C.c_int32), ("valid", C.c_int32),
                ("reserved", C.c_int32)]


class GsWindow(C.Structure):
    _fields_ = [("ox", C.c_double), ("oy", C.c_double), ("l", C.c_double), ("w", C.c_double)]


class GsTrackerConfig(C.Structure):
    _fields_ = [("h", C.c_double), ("f", C.c_double), ("eta", C.c_double),
                ("max_inner_iters", C.c_int32), ("engine_max_iter", C.c_int32),
                ("top_k", C.c_int32), ("n_ids", C.c_int32), ("ids", C.c_void_p)]


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libgridshift_cuda.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise Error(f"{path} missing: run __graft_entry__.build() (no CPU fallback exists)")
    lib = C.CDLL(path)
    P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    lib.gs_validate.argtypes = [C.POINTER(GsInput), C.POINTER(GsConfig)]
    lib.gs_create.argtypes = [C.c_int, P, C.POINTER(P)]
    lib.gs_destroy.argtypes = [P]
    lib.gs_destroy.restype = None
    lib.gs_run.argtypes = [P, C.POINTER(GsInput), C.POINTER(GsConfig), C.POINTER(GsResult)]
    lib.gs_get_centroids.argtypes = [P, I64, P, I64]
    lib.gs_get_history.argtypes = [P, I64, P, P, I32]
    lib.gs_get_stats.argtypes = [P, C.POINTER(GsStats)]
    lib.gs_last_error.argtypes = [P]
    lib.gs_last_error.restype = C.c_char_p
    lib.gs_status_string.argtypes = [C.c_int]
    lib.gs_status_string.restype = C.c_char_p
    lib.gs_debug_build.argtypes = [P, C.POINTER(GsInput), D, I64, P, P, P, P, P]
    lib.gs_debug_iterate_once.argtypes = [P, I32, D, I64, P, P, P, P, P, P, P, P, P, P, P, P]
    lib.gs_debug_resident_once.argtypes = [P, I32, D, I64, P, P, P, P, P, P, P, P, P, P]
    lib.gs_fixed_shift.argtypes = [I64, D]
    lib.gs_fixed_shift.restype = I32
    lib.gs_render.argtypes = [P, I64, P, I32]
    lib.gs_shard_keybounds.argtypes = [P, C.POINTER(GsInput), D, P, P]
    lib.gs_shard_bin.argtypes = [P, C.POINTER(GsInput), D, I64, P, P, I64, P, P, P, P]
    lib.gs_shard_run.argtypes = [P, I64, P, P, P, I64, C.POINTER(GsConfig), C.POINTER(GsResult)]
    lib.gs_tuner_create.argtypes = [C.c_int, I32, C.POINTER(P)]
    lib.gs_tuner_destroy.argtypes = [P]
    lib.gs_tuner_destroy.restype = None
    lib.gs_tuner_last_error.argtypes = [P]
    lib.gs_tuner_last_error.restype = C.c_char_p
    lib.gs_tune_bandwidth.argtypes = [P, C.POINTER(GsInput), P, I32, I32, I64, C.c_uint64,
                                      C.POINTER(GsSweepEntry), C.POINTER(D)]
    lib.gs_silhouette_subsampled.argtypes = [P, C.POINTER(GsInput), P, I32, I64, C.c_uint64,
                                             C.POINTER(D)]
    lib.gs_mspp_run.argtypes = [P, C.POINTER(GsInput), D, D, I32, C.POINTER(GsResult), P]
    lib.gs_dist_create.argtypes = [C.c_int, P, C.POINTER(P)]
    lib.gs_dist_destroy.argtypes = [P]
    lib.gs_dist_destroy.restype = None
    lib.gs_dist_last_error.argtypes = [P]
    lib.gs_dist_last_error.restype = C.c_char_p
    lib.gs_dist_run_frames.argtypes = [P, C.POINTER(GsInput), C.POINTER(GsConfig), C.POINTER(GsResult)]
    lib.gs_dist_run_slabs.argtypes = [P, C.POINTER(GsInput), C.POINTER(GsConfig), C.POINTER(GsResult)]
    lib.gs_dist_get_centroids.argtypes = [P, I64, P, I64]
    lib.gs_dist_get_history.argtypes = [P, P, P, I32]
    lib.gs_tracker_create.argtypes = [C.c_int, C.POINTER(P)]
    lib.gs_tracker_destroy.argtypes = [P]
    lib.gs_tracker_destroy.restype = None
    lib.gs_tracker_last_error.argtypes = [P]
    lib.gs_tracker_last_error.restype = C.c_char_p
    lib.gs_track_init.argtypes = [P, P, I32, I32, I32, C.POINTER(GsWindow),
                                  C.POINTER(GsTrackerConfig), C.POINTER(I64)]
    lib.gs_track_sequence.argtypes = [P, P, I64, I32, C.POINTER(GsWindow), P, P]
    _lib = lib
    return lib


def _raise(status: int, detail: str = "") -> None:
    if status == GS_OK:
        return
    exc = _STATUS.get(status, Error)
    raise exc(f"{STATUS_NAMES.get(status, status)}: {detail}")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ----------------------------------------------------------------------------- types
@dataclass
class EngineConfig:
    """SPEC.md:111-114."""
    h: float
    max_iterations: int = 1000
    record_history: bool = False
    debug_flags: int = 0          # test hooks (GS_DEBUG_GLOBAL_PATH)


@dataclass
class ClusterLabeling:
    """SPEC.md:107-110 (one frame)."""
    labels: np.ndarray
    centroids: np.ndarray
    iterations: int
    converged: bool
    history: Optional[List[tuple]] = None


@dataclass
class BatchLabeling:
    labels: np.ndarray          # [batch, n] int32
    k: np.ndarray               # [batch] int64
    iterations: np.ndarray      # [batch] int32
    converged: np.ndarray       # [batch] int32
    centroids: List[np.ndarray] = field(default_factory=list)
    history: Optional[List[List[tuple]]] = None


def validate(n: int, d: int, h: float, max_iter: int = 1000, batch: int = 1,
             dtype: int = GS_F64) -> None:
    """Host-only contract check through gs_validate (no device needed)."""
    lib = load_library()
    dummy = C.c_double(0.0)
    inp = GsInput(C.addressof(dummy), n, d, dtype, batch, 0, 0)
    cfg = GsConfig(h, max_iter, 0)
    _raise(lib.gs_validate(C.byref(inp), C.byref(cfg)), "gs_validate")


class Engine:
    """A GridShift engine bound to one CUDA device (owns a gs_ctx)."""

    def __init__(self, device: int = 0, stream: int = 0):
        self._lib = load_library()
        h = C.c_void_p()
        _raise(self._lib.gs_create(device, C.c_void_p(stream or None), C.byref(h)), "gs_create")
        self._ctx = h

    def close(self) -> None:
        if getattr(self, "_ctx", None):
            self._lib.gs_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> str:
        return self._lib.gs_last_error(self._ctx).decode()

    def _check(self, status: int) -> None:
        if status != GS_OK:
            _raise(status, self.last_error())

    # -- raw run over host numpy or device pointers --------------------------------------
    def run_raw(self, points_ptr: int, n: int, d: int, dtype: int, batch: int, on_device: bool,
                cfg: EngineConfig, labels_ptr: int, device_outputs: bool = False):
        k = np.zeros(batch, np.int64)
        it = np.zeros(batch, np.int32)
        cv = np.zeros(batch, np.int32)
        flags = (GS_RECORD_HISTORY if cfg.record_history else 0) | (
            GS_DEVICE_OUTPUTS if device_outputs else 0) | cfg.debug_flags
        inp = GsInput(points_ptr, n, d, dtype, batch, 1 if on_device else 0, 0)
        c = GsConfig(cfg.h, cfg.max_iterations, flags)
        res = GsResult(labels_ptr, _ptr(k), _ptr(it), _ptr(cv))
        self._check(self._lib.gs_run(self._ctx, C.byref(inp), C.byref(c), C.byref(res)))
        self._last_n = n
        return k, it, cv

    def run_batch(self, X: np.ndarray, cfg: EngineConfig, want_centroids: bool = True
                  ) -> BatchLabeling:
        """Independent frames X[batch, n, d] (float32 or float64, host memory)."""
        X = np.ascontiguousarray(X)
        if X.ndim == 2:
            X = X[None]
        if X.ndim != 3:
            raise InvalidParameterError("X must be [n, d] or [batch, n, d]")
        if X.dtype == np.float32:
            dt = GS_F32
        elif X.dtype == np.float64:
            dt = GS_F64
        else:
            X = X.astype(np.float64)
            dt = GS_F64
        b, n, d = X.shape
        labels = np.zeros((b, n), np.int32)
        k, it, cv = self.run_raw(_ptr(X), n, d, dt, b, False, cfg, _ptr(labels))
        out = BatchLabeling(labels, k, it, cv)
        if want_centroids:
            for f in range(b):
                out.centroids.append(self.centroids(f, int(k[f]), d))
        if cfg.record_history:
            out.history = [self.history(f, int(it[f])) for f in range(b)]
        return out

    def run(self, X: np.ndarray, cfg: EngineConfig) -> ClusterLabeling:
        """engine.run on one dataset X[n, d]."""
        X = np.asarray(X)
        if X.ndim != 2:
            raise InvalidParameterError("X must be [n, d]")
        r = self.run_batch(X[None], cfg)
        return ClusterLabeling(r.labels[0], r.centroids[0], int(r.iterations[0]),
                               bool(r.converged[0]), r.history[0] if r.history else None)

    def mspp(self, X: np.ndarray, h: float, tol: Optional[float] = None,
             max_iter: int = 300) -> ClusterLabeling:
        """MS++ baseline, mspp_run on the GPU: Jacobi grid mean shift."""
        X = np.ascontiguousarray(X)
        if X.dtype not in (np.float32, np.float64):
            X = X.astype(np.float64)
        n, d = X.shape
        tol = 1e-6 * h if tol is None else tol
        dt = GS_F32 if X.dtype == np.float32 else GS_F64
        inp = GsInput(X.ctypes.data, n, d, dt, 1, 0, 0)
        labels = np.zeros(n, np.int32)
        k = np.zeros(1, np.int64)
        it = np.zeros(1, np.int32)
        cv = np.zeros(1, np.int32)
        disp = np.zeros(max(max_iter, 1), np.float64)
        res = GsResult(labels.ctypes.data, k.ctypes.data, it.ctypes.data, cv.ctypes.data)
        self._check(self._lib.gs_mspp_run(self._ctx, C.byref(inp), h, tol, max_iter, C.byref(res),
                                          disp.ctypes.data))
        cen = self.centroids(0, int(k[0]), d)
        return ClusterLabeling(labels=labels, centroids=cen, iterations=int(it[0]),
                               converged=bool(cv[0]),
                               history=[(None, float(v)) for v in disp[:int(it[0])]])

    def centroids(self, frame: int, k: int, d: int) -> np.ndarray:
        out = np.zeros((k, d), np.float64)
        self._check(self._lib.gs_get_centroids(self._ctx, frame, _ptr(out), k))
        return out

    def history(self, frame: int, iters: int) -> List[tuple]:
        m = np.zeros(max(iters, 1), np.int64)
        dsp = np.zeros(max(iters, 1), np.float64)
        self._check(self._lib.gs_get_history(self._ctx, frame, _ptr(m), _ptr(dsp), iters))
        return [(int(m[t]), float(dsp[t])) for t in range(iters)]

    def stats(self) -> dict:
        s = GsStats()
        self._check(self._lib.gs_get_stats(self._ctx, C.byref(s)))
        out = {name: getattr(s, name) for name, _ in GsStats._fields_}
        out["sweep_modes"] = list(out["sweep_modes"])
        out["resident_cycles"] = list(out["resident_cycles"])
        return out

    # -- segmentation front end / render, fused into K1/K2 and K7 ---------
    def run_image(self, img: np.ndarray, cfg: EngineConfig, mode: str = "rgb") -> ClusterLabeling:
        """segment(): 8-bit RGB image [H, W, 3] (or a batch [B, H, W, 3]); features (r,g,b)/255
        (mode "rgb", d = 3) or + (col/(W-1), row/(H-1)) ("rgbxy", d = 5) are formed on the
        device from the 3-byte pixels.  Returns frame 0's labelling (labels [H*W])."""
        img = np.ascontiguousarray(img, np.uint8)
        if img.ndim == 3:
            img = img[None]
        if img.ndim != 4 or img.shape[3] != 3:
            raise InvalidParameterError("image must be [H, W, 3] or [B, H, W, 3] uint8")
        B, H, W, _ = img.shape
        d = 3 if mode == "rgb" else 5
        if mode not in ("rgb", "rgbxy"):
            raise InvalidParameterError("mode is rgb or rgbxy")
        n = H * W
        labels = np.zeros((B, n), np.int32)
        k = np.zeros(B, np.int64)
        it = np.zeros(B, np.int32)
        cv = np.zeros(B, np.int32)
        flags = (GS_RECORD_HISTORY if cfg.record_history else 0) | cfg.debug_flags
        inp = GsInput(_ptr(img), n, d, GS_U8, B, 0, W if d == 5 else 0)
        c = GsConfig(cfg.h, cfg.max_iterations, flags)
        res = GsResult(_ptr(labels), _ptr(k), _ptr(it), _ptr(cv))
        self._check(self._lib.gs_run(self._ctx, C.byref(inp), C.byref(c), C.byref(res)))
        self._last_n = n
        return ClusterLabeling(labels[0], self.centroids(0, int(k[0]), d), int(it[0]),
                               bool(cv[0]), None)

    def render(self, frame: int = 0) -> np.ndarray:
        """render(): every pixel of `frame` replaced by its segment's mean colour (uint8
        [n, 3]; centroid rgb * 255 rounded half-up)."""
        n = getattr(self, "_last_n", 0)
        out = np.zeros((n, 3), np.uint8)
        self._check(self._lib.gs_render(self._ctx, frame, _ptr(out), 0))
        return out

    # -- one point cloud over several ranks (gridshift_c.h gs_shard_*; driven by dist.py) ----
    @staticmethod
    def _shard_input(X):
        """numpy (host) or a contiguous torch CUDA tensor (device-resident shard)."""
        if hasattr(X, "is_cuda") and X.is_cuda:
            import torch
            assert X.is_contiguous() and X.dtype in (torch.float32, torch.float64)
            n, d = X.shape
            dt = GS_F32 if X.dtype == torch.float32 else GS_F64
            return X, GsInput(X.data_ptr(), n, d, dt, 1, 1, 0)
        X = np.ascontiguousarray(X)
        if X.dtype not in (np.float32, np.float64):
            X = X.astype(np.float64)
        n, d = X.shape
        dt = GS_F32 if X.dtype == np.float32 else GS_F64
        return X, GsInput(_ptr(X), n, d, dt, 1, 0, 0)

    def shard_keybounds(self, X: np.ndarray, h: float):
        """Per-dim cell-key range [klo, khi] of this rank's shard (to be all-reduced)."""
        X, inp = self._shard_input(X)
        d = X.shape[1]
        lo, hi = np.zeros(d, np.int64), np.zeros(d, np.int64)
        self._check(self._lib.gs_shard_keybounds(self._ctx, C.byref(inp), h, _ptr(lo), _ptr(hi)))
        return lo, hi

    def shard_bin(self, X: np.ndarray, h: float, n_global: int, klo, khi):
        """This shard's partial cells over the global key box: (keys u32, counts u32,
        sums int64 [m, d]) -- integers, merged exactly by shard_run."""
        X, inp = self._shard_input(X)
        n, d = X.shape
        klo = np.ascontiguousarray(klo, np.int64)
        khi = np.ascontiguousarray(khi, np.int64)
        cap = max(1, n)
        keys = np.zeros(cap, np.uint32)
        counts = np.zeros(cap, np.uint32)
        sums = np.zeros((cap, d), np.int64)
        m = C.c_int64()
        self._check(self._lib.gs_shard_bin(self._ctx, C.byref(inp), h, int(n_global), _ptr(klo),
                                           _ptr(khi), cap, C.byref(m), _ptr(keys),
                                           _ptr(counts), _ptr(sums)))
        m = m.value
        return keys[:m].copy(), counts[:m].copy(), sums[:m].copy()

    def shard_run(self, keys, counts, sums, n_shard: int, cfg: EngineConfig) -> ClusterLabeling:
        """Merge every rank's partial cells, iterate, label this rank's shard."""
        keys = np.ascontiguousarray(keys, np.uint32)
        counts = np.ascontiguousarray(counts, np.uint32)
        sums = np.ascontiguousarray(sums, np.int64)
        d = sums.shape[1]
        labels = np.zeros(n_shard, np.int32)
        k = np.zeros(1, np.int64)
        it = np.zeros(1, np.int32)
        cv = np.zeros(1, np.int32)
        flags = (GS_RECORD_HISTORY if cfg.record_history else 0) | cfg.debug_flags
        c = GsConfig(cfg.h, cfg.max_iterations, flags)
        res = GsResult(_ptr(labels), _ptr(k), _ptr(it), _ptr(cv))
        self._check(self._lib.gs_shard_run(self._ctx, len(keys), _ptr(keys), _ptr(counts),
                                           _ptr(sums), n_shard, C.byref(c), C.byref(res)))
        hist = self.history(0, int(it[0])) if cfg.record_history else None
        return ClusterLabeling(labels, self.centroids(0, int(k[0]), d), int(it[0]),
                               bool(cv[0]), hist)

    # -- test hooks --------------------------------------------------------------------------
    def debug_build(self, X: np.ndarray, h: float):
        X = np.ascontiguousarray(X)
        n, d = X.shape
        dt = GS_F32 if X.dtype == np.float32 else GS_F64
        if dt == GS_F64:
            X = X.astype(np.float64)
        cap = n
        keys = np.zeros((cap, d), np.int64)
        counts = np.zeros(cap, np.int64)
        cent = np.zeros((cap, d), np.float64)
        slot = np.zeros(n, np.int64)
        m = C.c_int64()
        inp = GsInput(_ptr(X), n, d, dt, 1, 0, 0)
        self._check(self._lib.gs_debug_build(self._ctx, C.byref(inp), h, cap, C.byref(m),
                                             _ptr(keys), _ptr(counts), _ptr(cent), _ptr(slot)))
        m = m.value
        return keys[:m], counts[:m], cent[:m], slot

    def debug_iterate_once(self, keys: np.ndarray, counts: np.ndarray, cent: np.ndarray,
                           h: float) -> dict:
        keys = np.ascontiguousarray(keys, np.int64)
        counts = np.ascontiguousarray(counts, np.int64)
        cent = np.ascontiguousarray(cent, np.float64)
        m, d = keys.shape
        ko = np.zeros((m, d), np.int64)
        co = np.zeros(m, np.int64)
        so = np.zeros((m, d), np.float64)
        sw = np.zeros((m, d), np.float64)
        par = np.zeros(m, np.int64)
        mo = C.c_int64()
        ch = C.c_int32()
        cv = C.c_int32()
        md = C.c_double()
        self._check(self._lib.gs_debug_iterate_once(
            self._ctx, d, h, m, _ptr(keys), _ptr(counts), _ptr(cent), C.byref(mo), _ptr(ko),
            _ptr(co), _ptr(so), _ptr(sw), _ptr(par), C.byref(ch), C.byref(cv), C.byref(md)))
        mn = mo.value
        return dict(keys=ko[:mn], counts=co[:mn], centroids=so[:mn], swept=sw, parent=par,
                    changed=bool(ch.value), converged=bool(cv.value), maxdisp=md.value)

    def debug_resident_once(self, keys: np.ndarray, counts: np.ndarray, cent: np.ndarray,
                            h: float) -> dict:
        """One iteration of K8 (the CTA-resident engine) on an injected state."""
        keys = np.ascontiguousarray(keys, np.int64)
        counts = np.ascontiguousarray(counts, np.int64)
        cent = np.ascontiguousarray(cent, np.float64)
        m, d = keys.shape
        ko = np.zeros((m, d), np.int64)
        co = np.zeros(m, np.int64)
        so = np.zeros((m, d), np.float64)
        par = np.zeros(m, np.int64)
        mo = C.c_int64()
        stop = C.c_int32()
        md = C.c_double()
        self._check(self._lib.gs_debug_resident_once(
            self._ctx, d, h, m, _ptr(keys), _ptr(counts), _ptr(cent), C.byref(mo), _ptr(ko),
            _ptr(co), _ptr(so), _ptr(par), C.byref(stop), C.byref(md)))
        mn = mo.value
        return dict(keys=ko[:mn], counts=co[:mn], centroids=so[:mn], parent=par,
                    stop=bool(stop.value), maxdisp=md.value)


class Dist:
    """Multi-GPU driver (gridshift_c.h gs_dist_*): one host thread drives R ranks, each an
    engine context on devices[r] (a device may repeat: loopback ranks share a GPU)."""

    def __init__(self, devices):
        self._lib = load_library()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _raise(self._lib.gs_dist_create(len(devices), devs, C.byref(h)), "gs_dist_create")
        self._d = h
        self.R = len(devices)

    def close(self) -> None:
        if getattr(self, "_d", None):
            self._lib.gs_dist_destroy(self._d)
            self._d = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, status: int) -> None:
        _raise(status, self._lib.gs_dist_last_error(self._d).decode() if self._d else "")

    @staticmethod
    def _input(X):
        X = np.ascontiguousarray(X)
        dt = GS_F32 if X.dtype == np.float32 else GS_F64
        if X.dtype not in (np.float32, np.float64):
            X = X.astype(np.float64)
        return X, dt

    def run_slabs(self, X: np.ndarray, cfg: EngineConfig) -> ClusterLabeling:
        """ONE cloud X[n, d] over the ranks: point shards, dim-0 slab ownership of the cells,
        per-iteration halo exchange; equal to Engine.run on one GPU."""
        X, dt = self._input(X)
        n, d = X.shape
        labels = np.zeros(n, np.int32)
        k = np.zeros(1, np.int64)
        it = np.zeros(1, np.int32)
        cv = np.zeros(1, np.int32)
        flags = (GS_RECORD_HISTORY if cfg.record_history else 0) | cfg.debug_flags
        inp = GsInput(X.ctypes.data, n, d, dt, 1, 0, 0)
        c = GsConfig(cfg.h, cfg.max_iterations, flags)
        res = GsResult(labels.ctypes.data, k.ctypes.data, it.ctypes.data, cv.ctypes.data)
        self._check(self._lib.gs_dist_run_slabs(self._d, C.byref(inp), C.byref(c), C.byref(res)))
        cen = np.zeros((int(k[0]), d), np.float64)
        self._check(self._lib.gs_dist_get_centroids(self._d, 0, cen.ctypes.data, int(k[0])))
        hist = None
        if cfg.record_history:
            mt = np.zeros(int(it[0]), np.int64)
            md = np.zeros(int(it[0]), np.float64)
            self._check(self._lib.gs_dist_get_history(self._d, mt.ctypes.data, md.ctypes.data,
                                                      int(it[0])))
            hist = [(int(a), float(b)) for a, b in zip(mt, md)]
        return ClusterLabeling(labels, cen, int(it[0]), bool(cv[0]), hist)

    def run_frames(self, X: np.ndarray, cfg: EngineConfig) -> BatchLabeling:
        """Independent frames X[batch, n, d] in contiguous blocks per rank."""
        X, dt = self._input(X)
        b, n, d = X.shape
        labels = np.zeros((b, n), np.int32)
        k = np.zeros(b, np.int64)
        it = np.zeros(b, np.int32)
        cv = np.zeros(b, np.int32)
        inp = GsInput(X.ctypes.data, n, d, dt, b, 0, 0)
        c = GsConfig(cfg.h, cfg.max_iterations, cfg.debug_flags)
        res = GsResult(labels.ctypes.data, k.ctypes.data, it.ctypes.data, cv.ctypes.data)
        self._check(self._lib.gs_dist_run_frames(self._d, C.byref(inp), C.byref(c), C.byref(res)))
        out = BatchLabeling(labels, k, it, cv)
        for f in range(b):
            cen = np.zeros((int(k[f]), d), np.float64)
            self._check(self._lib.gs_dist_get_centroids(self._d, f, cen.ctypes.data, int(k[f])))
            out.centroids.append(cen)
        return out


_default_engine: Optional[Engine] = None


def run(X, cfg: EngineConfig) -> ClusterLabeling:
    """engine.run(X, cfg) on device 0."""
    if not (cfg.h > 0) or not np.isfinite(cfg.h):
        raise InvalidBandwidthError("h must be > 0")
    X = np.asarray(X, dtype=np.float64 if np.asarray(X).dtype != np.float32 else np.float32)
    if X.size == 0:
        raise EmptyInputError("empty dataset")
    global _default_engine
    if _default_engine is None:
        _default_engine = Engine(0)
    return _default_engine.run(X, cfg)


def fixed_shift(n: int, h: float) -> int:
    return int(load_library().gs_fixed_shift(n, h))


# ----------------------------------------------------------------------------- metrics
@dataclass
class SweepEntry:
    """One (h, silhouette score, cluster count) pair of BandwidthSweepResult."""
    h: float
    score: Optional[float]   # None: undefined (< 2 clusters in the sample), skipped
    k: int
    iterations: int
    converged: bool


@dataclass
class BandwidthSweepResult:
    """evaluated pairs and best_h."""
    entries: List[SweepEntry]
    best_h: float


class Tuner:
    """tune_bandwidth with the GPU engine as the clusterer and
    silhouette_subsampled as the score, over gs_tune_bandwidth: up to
    ``max_concurrent`` sweep entries run at once on one GPU, each on its own engine context."""

    def __init__(self, device: int = 0, max_concurrent: int = 8):
        self._lib = load_library()
        h = C.c_void_p()
        _raise(self._lib.gs_tuner_create(device, max_concurrent, C.byref(h)), "gs_tuner_create")
        self._t = h

    def close(self) -> None:
        if self._t:
            self._lib.gs_tuner_destroy(self._t)
            self._t = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, status: int) -> None:
        if status != GS_OK:
            _raise(status, (self._lib.gs_tuner_last_error(self._t) or b"").decode())

    @staticmethod
    def _input(X: np.ndarray):
        if X.ndim != 2:
            raise InvalidParameterError("X must be n x d")
        if X.dtype not in (np.float32, np.float64):
            X = X.astype(np.float64)
        X = np.ascontiguousarray(X)
        dt = GS_F32 if X.dtype == np.float32 else GS_F64
        return X, GsInput(X.ctypes.data, X.shape[0], X.shape[1], dt, 1, 0, 0)

    def tune_bandwidth(self, X: np.ndarray, h_grid=None, max_iter: int = 1000, cap: int = 10000,
                       seed: int = 0) -> BandwidthSweepResult:
        if h_grid is None:  # SPEC.md:347 default grid {0.05, 0.10, ..., 1.00}
            h_grid = [round(0.05 * i, 2) for i in range(1, 21)]
        X, inp = self._input(X)
        hs = np.ascontiguousarray(h_grid, np.float64)
        out = (GsSweepEntry * max(len(hs), 1))()
        best = C.c_double()
        self._check(self._lib.gs_tune_bandwidth(self._t, C.byref(inp), hs.ctypes.data, len(hs),
                                                max_iter, cap, seed, out, C.byref(best)))
        ents = [SweepEntry(e.h, e.score if e.valid else None, e.k, e.iterations,
                           bool(e.converged)) for e in out[:len(hs)]]
        return BandwidthSweepResult(ents, best.value)

    def silhouette_subsampled(self, X: np.ndarray, labels: np.ndarray, cap: int,
                              seed: int = 0) -> float:
        X, inp = self._input(X)
        lab = np.ascontiguousarray(labels, np.int32)
        if lab.shape != (X.shape[0],):
            raise InvalidInputError("labels must have one entry per point")
        sc = C.c_double()
        self._check(self._lib.gs_silhouette_subsampled(self._t, C.byref(inp), lab.ctypes.data, 0,
                                                       cap, seed, C.byref(sc)))
        return sc.value


# ----------------------------------------------------------------------------- tracker
@dataclass
class TrackerConfig:
    """TrackerConfig with the ledger defaults."""
    h: float
    f: float = 1.0
    eta: float = 1.0
    max_inner_iters: int = 20
    engine_max_iter: int = 1000
    top_k: int = 1
    ids: Optional[List[int]] = None


class Tracker:
    """init_tracker / track_frame / track_sequence over gs_track_*: the
    engine on the GPU for init, the whole tracked sequence in one kernel launch."""

    def __init__(self, device: int = 0):
        self._lib = load_library()
        h = C.c_void_p()
        _raise(self._lib.gs_tracker_create(device, C.byref(h)), "gs_tracker_create")
        self._t = h
        self._ids = None

    def close(self) -> None:
        if self._t:
            self._lib.gs_tracker_destroy(self._t)
            self._t = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, status: int) -> None:
        if status != GS_OK:
            _raise(status, (self._lib.gs_tracker_last_error(self._t) or b"").decode())

    def init(self, frame0: np.ndarray, window, cfg: TrackerConfig) -> int:
        """init_tracker: returns the number of clusters found in the window."""
        fr = np.ascontiguousarray(frame0, np.uint8)
        if fr.ndim != 3 or fr.shape[2] != 3:
            raise InvalidInputError("frame must be H x W x 3 uint8")
        ids = np.ascontiguousarray(cfg.ids or [], np.int32)
        self._ids = ids
        c = GsTrackerConfig(cfg.h, cfg.f, cfg.eta, cfg.max_inner_iters, cfg.engine_max_iter,
                            cfg.top_k, len(ids), ids.ctypes.data if len(ids) else None)
        w = GsWindow(*[float(v) for v in window])
        k = C.c_int64()
        self._check(self._lib.gs_track_init(self._t, fr.ctypes.data, fr.shape[0], fr.shape[1], 0,
                                            C.byref(w), C.byref(c), C.byref(k)))
        return k.value

    def track_sequence(self, frames: np.ndarray):
        """track_sequence over frames [T][H][W][3]: (windows T x 4, lost T, inner T)."""
        fr = np.ascontiguousarray(frames, np.uint8)
        T = fr.shape[0]
        out = (GsWindow * T)()
        lost = np.zeros(T, np.int32)
        inner = np.zeros(T, np.int32)
        self._check(self._lib.gs_track_sequence(self._t, fr.ctypes.data, T, 0, out,
                                                lost.ctypes.data, inner.ctypes.data))
        win = np.array([[o.ox, o.oy, o.l, o.w] for o in out])
        return win, lost.astype(bool), inner
