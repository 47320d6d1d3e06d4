"""Timing probe: K8's first sweep under GS_SWEEP_VARIANT knobs (results are wrong when != 0)."""
import os, subprocess, sys
code = r'''
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2206_02200_b200 import gridshift as G, configs as CF
w = sys.argv[1]
X = CF.generate(w)[0]; cfg = CF.CONFIGS[w]
e = G.Engine(0)
for r in range(3):
    try:
        e.run(X, G.EngineConfig(cfg.h, cfg.max_iter))
    except Exception as ex:
        print("run failed:", type(ex).__name__, file=sys.stderr)
'''
w = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
for v in [0, 32, 1, 2, 4, 8, 3, 7, 15, 16, 48]:
    env = dict(os.environ, GS_SWEEP_VARIANT=str(v), GS_TRACE_LEVELS="1")
    out = subprocess.run([sys.executable, "-c", code, w], env=env, capture_output=True, text=True).stderr
    it0 = [l for l in out.splitlines() if l.startswith("iter  0")]
    lv = [l for l in out.splitlines() if l.startswith("level")]
    print(f"variant {v:3d}: {it0[-1] if it0 else 'no trace'}  | levels {len(lv)//max(1,len(it0))}")
