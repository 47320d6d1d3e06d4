"""Where does a device-resident run's time go?  host wall per call vs CUDA-event step time."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2206_02200_b200 import gridshift as G  # noqa: E402
from paper_2206_02200_b200.configs import generate, CONFIGS  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = CONFIGS[w]
X = generate(w)
X = X[None] if X.ndim == 2 else X
B, n, d = X.shape
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(device=dev)
eng = G.Engine(0, stream.cuda_stream)
Xd = torch.from_numpy(np.ascontiguousarray(X)).to(dev)
lab = torch.empty((B, n), dtype=torch.int32, device=dev)
dt = G.GS_F32 if X.dtype == np.float32 else G.GS_F64
ec = G.EngineConfig(cfg.h, cfg.max_iter)
for _ in range(5):
    eng.run_raw(Xd.data_ptr(), n, d, dt, B, True, ec, lab.data_ptr(), device_outputs=True)
torch.cuda.synchronize()
N = 200
t0 = time.perf_counter()
for _ in range(N):
    eng.run_raw(Xd.data_ptr(), n, d, dt, B, True, ec, lab.data_ptr(), device_outputs=True)
t1 = time.perf_counter()
print(f"{w}: run_raw host wall {1e6 * (t1 - t0) / N:.1f} us/call")
# bare ctypes with prebuilt structs
k = np.zeros(B, np.int64); it = np.zeros(B, np.int32); cv = np.zeros(B, np.int32)
inp = G.GsInput(Xd.data_ptr(), n, d, dt, B, 1, 0)
c = G.GsConfig(cfg.h, cfg.max_iter, G.GS_DEVICE_OUTPUTS)
res = G.GsResult(lab.data_ptr(), k.ctypes.data, it.ctypes.data, cv.ctypes.data)
f = eng._lib.gs_run
t0 = time.perf_counter()
for _ in range(N):
    f(eng._ctx, C.byref(inp), C.byref(c), C.byref(res))
t1 = time.perf_counter()
print(f"{w}: bare gs_run host wall {1e6 * (t1 - t0) / N:.1f} us/call")
s = eng.stats()
print({kk: s[kk] for kk in ("ms_bin", "ms_iterate", "ms_label", "ms_total") if kk in s})
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
for i in range(N):
    ev[i][0].record(stream)
    f(eng._ctx, C.byref(inp), C.byref(c), C.byref(res))
    ev[i][1].record(stream)
torch.cuda.synchronize()
print(f"{w}: event step {1e3 * np.mean([a.elapsed_time(b) for a, b in ev]):.1f} us")
