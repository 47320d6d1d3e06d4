"""ctypes binding of the CPU oracle (oracle/gs_oracle.cpp).  TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl reference``
legs may import this module; the product path never does.  The oracle restates
/root/reference/SPEC.md:17-181 (grid-core + engine) — see the header of gs_oracle.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
BUILD_SPEC, BUILD_FIXED = 0, 1
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        P, I64, I32, D = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        L.gso_build.argtypes = [P, I64, I32, D, I32, P, P, P, P, P]
        L.gso_iterate_once.argtypes = [I32, D, I64, P, P, P, P, P, P, P, P, P, P, P, P]
        L.gso_has_converged.argtypes = [I32, I64, P, P]
        L.gso_run.argtypes = [P, I64, I32, D, I32, I32, P, P, P, P, P, P, P]
        L.gso_fixed_shift.argtypes = [I64, D]
        L.gso_sample_indices.argtypes = [I64, I64, C.c_uint64, P]
        L.gso_sample_indices.restype = I64
        L.gso_silhouette.argtypes = [P, P, I64, I32, P, P, P]
        L.gso_track.argtypes = [P, I64, I32, I32, P, D, D, D, I32, I32, I32, P, I32, I32, P, P, P]
        L.gso_mspp.argtypes = [P, I64, I32, D, D, I32, P, P, P, P, P, P]
        L.gso_tune.argtypes = [P, I64, I32, P, I32, I32, I64, C.c_uint64, I32, P, P, P, P, P]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, status: int):
        super().__init__(f"oracle status {status}")
        self.status = status


def _chk(rc: int) -> None:
    if rc != 0:
        raise OracleError(rc)


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def build_grid(X: np.ndarray, h: float, mode: int = BUILD_FIXED):
    """build_active_grid: lex-sorted keys, counts, centroids, point->rank."""
    X = np.ascontiguousarray(X, np.float64)
    n, d = X.shape
    keys = np.zeros((n, d), np.int64)
    cnt = np.zeros(n, np.int64)
    cen = np.zeros((n, d), np.float64)
    slot = np.zeros(n, np.int64)
    m = C.c_int64()
    _chk(lib().gso_build(_p(X), n, d, h, mode, C.byref(m), _p(keys), _p(cnt), _p(cen), _p(slot)))
    m = m.value
    return keys[:m], cnt[:m], cen[:m], slot


def iterate_once(keys, counts, cent, h: float) -> dict:
    """iterate_once on an injected lex-sorted state."""
    keys = np.ascontiguousarray(keys, np.int64)
    counts = np.ascontiguousarray(counts, np.int64)
    cent = np.ascontiguousarray(cent, np.float64)
    m, d = keys.shape
    ko = np.zeros((m, d), np.int64)
    co = np.zeros(m, np.int64)
    so = np.zeros((m, d), np.float64)
    sw = np.zeros((m, d), np.float64)
    par = np.zeros(m, np.int64)
    mo, ch, cv, md = C.c_int64(), C.c_int32(), C.c_int32(), C.c_double()
    _chk(lib().gso_iterate_once(d, h, m, _p(keys), _p(counts), _p(cent), C.byref(mo), _p(ko),
                                _p(co), _p(so), _p(sw), _p(par), C.byref(ch), C.byref(cv),
                                C.byref(md)))
    mn = mo.value
    return dict(keys=ko[:mn], counts=co[:mn], centroids=so[:mn], swept=sw, parent=par,
                changed=bool(ch.value), converged=bool(cv.value), maxdisp=md.value)


def has_converged(keys) -> bool:
    keys = np.ascontiguousarray(keys, np.int64)
    m, d = keys.shape
    out = C.c_int32()
    _chk(lib().gso_has_converged(d, m, _p(keys), C.byref(out)))
    return bool(out.value)


def run(X: np.ndarray, h: float, max_iter: int = 1000, mode: int = BUILD_SPEC) -> dict:
    """engine.run on one frame."""
    X = np.ascontiguousarray(X, np.float64)
    n, d = X.shape
    labels = np.zeros(n, np.int32)
    cen = np.zeros((n, d), np.float64)
    hm = np.zeros(max(max_iter, 1), np.int64)
    hd = np.zeros(max(max_iter, 1), np.float64)
    k, it, cv = C.c_int64(), C.c_int32(), C.c_int32()
    _chk(lib().gso_run(_p(X), n, d, h, max_iter, mode, _p(labels), C.byref(k), C.byref(it),
                       C.byref(cv), _p(cen), _p(hm), _p(hd)))
    k, it = k.value, it.value
    return dict(labels=labels, k=k, iterations=it, converged=bool(cv.value), centroids=cen[:k],
                history=[(int(hm[t]), float(hd[t])) for t in range(it)])


def fixed_shift(n: int, h: float) -> int:
    return int(lib().gso_fixed_shift(n, h))


def sample_indices(n: int, cap: int, seed: int) -> np.ndarray:
    """Pin S1 of silhouette_subsampled."""
    out = np.zeros(min(n, cap), np.int64)
    lib().gso_sample_indices(n, cap, seed, _p(out))
    return out


def silhouette(X: np.ndarray, labels: np.ndarray):
    """silhouette (pin S2): (score, valid, per-point values)."""
    X = np.ascontiguousarray(X, np.float64)
    lab = np.ascontiguousarray(labels, np.int32)
    s, d = X.shape
    sc, va = C.c_double(), C.c_int32()
    per = np.zeros(s, np.float64)
    _chk(lib().gso_silhouette(_p(X), _p(lab), s, d, C.byref(sc), C.byref(va), _p(per)))
    return sc.value, bool(va.value), per


def silhouette_subsampled(X: np.ndarray, labels: np.ndarray, cap: int, seed: int = 0):
    idx = sample_indices(X.shape[0], cap, seed)
    return silhouette(np.asarray(X, np.float64)[idx], np.asarray(labels)[idx])


def tune(X: np.ndarray, hs, max_iter: int = 1000, cap: int = 10000, seed: int = 0,
         mode: int = BUILD_FIXED) -> dict:
    """tune_bandwidth with the oracle engine (build `mode`)."""
    X = np.ascontiguousarray(X, np.float64)
    n, d = X.shape
    hs = np.ascontiguousarray(hs, np.float64)
    nh = len(hs)
    sc = np.zeros(max(nh, 1)); ks = np.zeros(max(nh, 1), np.int64)
    it = np.zeros(max(nh, 1), np.int32); va = np.zeros(max(nh, 1), np.int32)
    best = C.c_double()
    _chk(lib().gso_tune(_p(X), n, d, _p(hs), nh, max_iter, cap, seed, mode, _p(sc), _p(ks),
                        _p(it), _p(va), C.byref(best)))
    return dict(scores=sc[:nh], k=ks[:nh], iterations=it[:nh], valid=va[:nh].astype(bool),
                best_h=best.value)


def track(frames: np.ndarray, window, h: float, f: float = 1.0, eta: float = 1.0,
          max_inner: int = 20, engine_max_iter: int = 1000, top_k: int = 1, ids=None,
          mode: int = BUILD_FIXED) -> dict:
    """tracker (pins T1-T5): frames [T][H][W][3] u8; frames[0] initialises.
    Returns per tracked frame the window (ox, oy, l, w), the lost flag and inner iterations."""
    fr = np.ascontiguousarray(frames, np.uint8)
    T, H, W, _ = fr.shape
    w0 = np.ascontiguousarray(window, np.float64)
    ida = np.ascontiguousarray([] if ids is None else ids, np.int32)
    out = np.zeros((max(T - 1, 1), 4))
    lost = np.zeros(max(T - 1, 1), np.int32)
    inner = np.zeros(max(T - 1, 1), np.int32)
    _chk(lib().gso_track(_p(fr), T, H, W, _p(w0), h, f, eta, max_inner, engine_max_iter, top_k,
                         _p(ida) if len(ida) else None, len(ida), mode, _p(out), _p(lost),
                         _p(inner)))
    return dict(windows=out[:T - 1], lost=lost[:T - 1].astype(bool), inner=inner[:T - 1])


def mspp(X: np.ndarray, h: float, tol: float = None, max_iter: int = 300) -> dict:
    """mspp_run (pins M1-M5): MS++ parallel grid mean shift."""
    X = np.ascontiguousarray(X, np.float64)
    n, d = X.shape
    tol = 1e-6 * h if tol is None else tol
    labels = np.zeros(n, np.int32)
    cen = np.zeros((n, d))
    disp = np.zeros(max(max_iter, 1))
    k, it, cv = C.c_int64(), C.c_int32(), C.c_int32()
    _chk(lib().gso_mspp(_p(X), n, d, h, tol, max_iter, _p(labels), C.byref(k), C.byref(it),
                        C.byref(cv), _p(cen), _p(disp)))
    return dict(labels=labels, k=k.value, iterations=it.value, converged=bool(cv.value),
                centroids=cen[:k.value], disp=disp[:it.value])
