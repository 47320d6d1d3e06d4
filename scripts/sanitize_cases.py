"""Small engine runs for compute-sanitizer (memcheck / racecheck / synccheck): each case drives
one kernel family at a size the sanitizer finishes in seconds, and checks the result against
the oracle.  Usage: python scripts/sanitize_cases.py <case>
  k2dense   K2 dense per-frame tables (3 image frames) + K3 + K8 + K7
  k2hash    K2 hash table (a wide cloud: the key box far exceeds a CTA's table)
  cluster   global path, level-synchronous 16-CTA cluster sweep (d = 3)
  flow      global path, dataflow cluster sweep (d = 5)
  single    global path, single-CTA sweep (d = 2)
  resident  K8 state injection"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402  (checker)
from paper_2206_02200_b200 import configs as CF  # noqa: E402
from paper_2206_02200_b200 import gridshift as G  # noqa: E402


def check(eng, X, h, flags=0):
    g = eng.run(X, G.EngineConfig(h, 100, debug_flags=flags))
    o = O.run(X.astype(np.float64), h, 100, O.BUILD_FIXED)
    assert np.array_equal(g.labels, o["labels"]) and g.iterations == o["iterations"]
    assert np.array_equal(g.centroids.view(np.int64), o["centroids"].view(np.int64))


def mixture(seed, n, d, span=4.0, sig=0.3):
    rng = np.random.default_rng(seed)
    c = rng.uniform(0, span, (6, d))
    return (c[rng.integers(0, 6, n)] + sig * rng.standard_normal((n, d))).astype(np.float32)


case = sys.argv[1]
eng = G.Engine(0)
if case == "k2dense":
    X = CF.generate("cfg4", scale=0.02, frames=3)
    r = eng.run_batch(X, G.EngineConfig(0.08, 50))
    for f in range(X.shape[0]):
        o = O.run(X[f].astype(np.float64), 0.08, 50, O.BUILD_FIXED)
        assert np.array_equal(r.labels[f], o["labels"])
    r = eng.run_batch(X, G.EngineConfig(0.08, 50))  # second run: the predicted key box
elif case == "k2hash":
    check(eng, mixture(1, 20000, 3, span=60.0, sig=2.0), 0.5)
elif case == "cluster":
    check(eng, mixture(2, 3000, 3), 0.3, G.GS_DEBUG_GLOBAL_PATH | G.GS_DEBUG_SWEEP_LEVELS)
elif case == "flow":
    check(eng, mixture(3, 1500, 5), 0.5, G.GS_DEBUG_GLOBAL_PATH | G.GS_DEBUG_SWEEP_FLOW)
elif case == "single":
    check(eng, mixture(4, 3000, 2), 0.3, G.GS_DEBUG_GLOBAL_PATH | G.GS_DEBUG_SWEEP_SINGLE)
elif case == "resident":
    X = mixture(5, 3000, 3).astype(np.float64)
    keys, cnt, cen, _ = O.build_grid(X, 0.3, O.BUILD_FIXED)
    g = eng.debug_resident_once(keys, cnt, cen, 0.3)
    o = O.iterate_once(keys, cnt, cen, 0.3)
    assert np.array_equal(g["keys"], o["keys"])
else:
    raise SystemExit(f"unknown case {case}")
eng.close()
print(f"case {case} ok")
