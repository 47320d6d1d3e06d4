"""gs_dist on loopback ranks (one GPU): host wall per call of Engine.run vs Dist.run_slabs /
run_frames at R ranks, to calibrate DESIGN.md §5's multi-GPU cost model (on one GPU the ranks'
kernels serialise, so this measures the exchange/orchestration overhead, not a speed-up)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2206_02200_b200 import configs as CF  # noqa: E402
from paper_2206_02200_b200 import gridshift as G  # noqa: E402


def wall(f, reps=3):
    f()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)


X = CF.generate("cfg5")[0]
cfg = G.EngineConfig(1.0, 100)
eng = G.Engine(0)
r1 = eng.run(X, cfg)
print(f"cfg5 Engine.run (host input, 1 GPU): {wall(lambda: eng.run(X, cfg)):.1f} ms, "
      f"iterations {r1.iterations}")
eng.close()
for R in (2, 4, 8):
    D = G.Dist([0] * R)
    got = D.run_slabs(X, cfg)
    assert np.array_equal(got.labels, r1.labels)
    print(f"cfg5 Dist.run_slabs R={R} loopback: {wall(lambda: D.run_slabs(X, cfg), 2):.1f} ms")
    D.close()
F = CF.generate("cfg4", frames=32)
eng = G.Engine(0)
print(f"cfg4 32 frames Engine.run_batch: {wall(lambda: eng.run_batch(F, G.EngineConfig(0.08, 50), False)):.1f} ms")
eng.close()
for R in (2, 4):
    D = G.Dist([0] * R)
    print(f"cfg4 32 frames Dist.run_frames R={R} loopback: "
          f"{wall(lambda: D.run_frames(F, G.EngineConfig(0.08, 50))):.1f} ms")
    D.close()
