"""The five BASELINE.json configs as seeded synthetic workloads.

Inputs are generated on the host by ``_lib/libgs_gen.so`` (counter-based SplitMix64, fp64
Box-Muller), so the GPU engine and the CPU oracle read identical bytes.  The paper's datasets
(UCI sensor sets, BSDS500, OTB100) are absent; these generators stand in for them with the
shapes, sizes and value distributions BASELINE.json names.  Base seed 2206 + config index.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
GEN_PATH = os.path.join(_HERE, "_lib", "libgs_gen.so")
_gen = None


def _lib():
    global _gen
    if _gen is None:
        if not os.path.exists(GEN_PATH):
            raise RuntimeError(f"{GEN_PATH} missing: run __graft_entry__.build()")
        g = C.CDLL(GEN_PATH)
        U64, I64, I32, D, P = C.c_uint64, C.c_int64, C.c_int32, C.c_double, C.c_void_p
        g.gsgen_blobs.argtypes = [U64, I64, I32, I32, D, D, D, P]
        g.gsgen_voronoi_rgb.argtypes = [U64, I32, I32, I32, D, P]
        g.gsgen_voronoi_rgbxy.argtypes = [U64, I32, I32, I32, D, D, P]
        g.gsgen_ellipse_frames.argtypes = [U64, I32, I32, I32, D, D, D, D, I64, I64, P]
        g.gsgen_gmm3.argtypes = [U64, I64, I64, I32, D, D, D, D, P]
        _gen = g
    return _gen


def _chk(rc):
    if rc != 0:
        raise ValueError("generator rejected its parameters")


def blobs(seed=2207, n=100_000, d=2, k=5, sigma=0.5, lo=0.0, hi=10.0) -> np.ndarray:
    out = np.empty((n, d), np.float64)
    _chk(_lib().gsgen_blobs(seed, n, d, k, sigma, lo, hi, out.ctypes.data))
    return out


def voronoi_rgb(seed=2208, W=481, H=321, sites=16, sigma=8.0 / 255.0) -> np.ndarray:
    out = np.empty((W * H, 3), np.float32)
    _chk(_lib().gsgen_voronoi_rgb(seed, W, H, sites, sigma, out.ctypes.data))
    return out


def voronoi_rgbxy(seed=2209, W=1920, H=1080, sites=64, grad=0.3, sigma=0.02) -> np.ndarray:
    out = np.empty((W * H, 5), np.float32)
    _chk(_lib().gsgen_voronoi_rgbxy(seed, W, H, sites, grad, sigma, out.ctypes.data))
    return out


def ellipse_frames(seed=2210, W=640, H=480, ne=12, f0=0, nf=256, amin=20.0, amax=80.0,
                   vmax=4.0, bg_sigma=0.05) -> np.ndarray:
    out = np.empty((nf, W * H, 3), np.float32)
    _chk(_lib().gsgen_ellipse_frames(seed, W, H, ne, amin, amax, vmax, bg_sigma, f0, nf,
                                     out.ctypes.data))
    return out


def gmm3(seed=2211, n=64_000_000, p0=0, k=64, lo=0.0, hi=100.0, smin=0.3, smax=2.0
         ) -> np.ndarray:
    out = np.empty((n, 3), np.float32)
    _chk(_lib().gsgen_gmm3(seed, p0, n, k, lo, hi, smin, smax, out.ctypes.data))
    return out


@dataclass(frozen=True)
class Config:
    name: str
    h: float
    max_iter: int
    n: int          # points per frame
    d: int
    batch: int
    dtype: str
    desc: str


CONFIGS = {
    "cfg1": Config("cfg1", 0.5, 300, 100_000, 2, 1, "f64",
                   "2D Gaussian blobs: 5 x 20,000 points, sigma 0.5, centres U[0,10]^2"),
    "cfg2": Config("cfg2", 0.08, 100, 481 * 321, 3, 1, "f32",
                   "481x321 RGB image, 16 Voronoi regions, noise sigma 8/255"),
    "cfg3": Config("cfg3", 0.06, 50, 1920 * 1080, 5, 1, "f32",
                   "1920x1080 (x/W, y/H, r, g, b), 64 gradient Voronoi regions, noise 0.02"),
    "cfg4": Config("cfg4", 0.08, 50, 640 * 480, 3, 256, "f32",
                   "256 frames 640x480 RGB, 12 moving solid ellipses, noisy background"),
    "cfg5": Config("cfg5", 1.0, 100, 64_000_000, 3, 1, "f32",
                   "64M-point 3D cloud, 64 anisotropic Gaussians, Dirichlet(1) weights"),
}


def generate(name: str, scale: Optional[float] = None, frames: Optional[int] = None,
             frame0: int = 0) -> np.ndarray:
    """Input of config `name` as [batch, n, d].  `scale` shrinks the point count (tests);
    `frames`/`frame0` select a frame range of cfg4 (sharding)."""
    if name == "cfg1":
        n = 100_000 if scale is None else max(5, int(100_000 * scale))
        return blobs(n=n)[None]
    if name == "cfg2":
        if scale is None:
            return voronoi_rgb()[None]
        W, H = max(8, int(481 * scale ** 0.5)), max(8, int(321 * scale ** 0.5))
        return voronoi_rgb(W=W, H=H)[None]
    if name == "cfg3":
        if scale is None:
            return voronoi_rgbxy()[None]
        W, H = max(8, int(1920 * scale ** 0.5)), max(8, int(1080 * scale ** 0.5))
        return voronoi_rgbxy(W=W, H=H)[None]
    if name == "cfg4":
        nf = 256 if frames is None else frames
        if scale is None:
            return ellipse_frames(f0=frame0, nf=nf)
        W, H = max(8, int(640 * scale ** 0.5)), max(8, int(480 * scale ** 0.5))
        a = 20.0 * scale ** 0.5, 80.0 * scale ** 0.5
        return ellipse_frames(W=W, H=H, f0=frame0, nf=nf, amin=a[0], amax=a[1])
    if name == "cfg5":
        n = 64_000_000 if scale is None else max(64, int(64_000_000 * scale))
        return gmm3(n=n)[None]
    raise KeyError(name)
