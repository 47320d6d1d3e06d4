import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import oracle as O
from paper_2206_02200_b200 import gridshift as G

rng = np.random.default_rng(11)
eng = G.Engine(0)
for trial in range(25):
    d = int(rng.integers(1, 6))
    n = int(rng.integers(1, 3000))
    X = rng.normal(size=(n, d)) * rng.uniform(0.1, 5) + rng.uniform(-20, 20)
    if trial % 3 == 0:
        X = X.astype(np.float32)
    h = float(rng.uniform(0.05, 2.0))
    Xd = np.asarray(X, np.float64)
    ext = np.floor(Xd.max(0) / h) - np.floor(Xd.min(0) / h) + 5
    if np.prod(ext) > 2 ** 28:
        continue
    o = O.run(Xd, h, 500, O.BUILD_FIXED)
    for tag, e in (("shared", eng), ("fresh", G.Engine(0))):
        g = e.run(X, G.EngineConfig(h, 500))
        bad = np.flatnonzero(g.labels != o["labels"])
        print(trial, tag, "d", d, "n", n, "h", round(h, 3), "k", len(g.centroids), o["k"], "it", g.iterations,
              o["iterations"], "lab_bad", len(bad), "cent_eq",
              g.centroids.shape == o["centroids"].shape and np.array_equal(g.centroids, o["centroids"]),
              "stats", {k: e.stats()[k] for k in ("m0", "sweep_modes", "kernel_launches")})
        if len(bad):
            print("   first bad", bad[:10], g.labels[bad[:10]], o["labels"][bad[:10]])
    if trial > 4:
        break
