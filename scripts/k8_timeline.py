"""K8 per-iteration phase timeline (GS_TRACE_LEVELS) of one workload run: python scripts/k8_timeline.py cfg2"""
import os
import sys

os.environ.setdefault("GS_TRACE_LEVELS", "1")
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
from paper_2206_02200_b200 import gridshift as G  # noqa: E402
from paper_2206_02200_b200.configs import generate, CONFIGS  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[w]
X = generate(w)
X = X[0] if X.ndim == 3 else X
eng = G.Engine(0)
for _ in range(2):
    r = eng.run(X, G.EngineConfig(cfg.h, cfg.max_iter))
print(w, "k", r.k if hasattr(r, "k") else None, file=sys.stderr)
