"""Box probe: host cores/CPU model, PCIe H2D / D2H / concurrent bandwidth from pinned memory."""
import os, subprocess, torch, time
print("nproc", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
try:
    print([l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].strip())
except Exception as e:
    print(e)
N = 512 << 20
h = torch.empty(N, dtype=torch.uint8).pin_memory(); h2 = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device="cuda"); d2 = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def t(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); return time.perf_counter() - t0
a = t(lambda: d.copy_(h, non_blocking=True)); print("H2D GB/s", N / a / 1e9)
b = t(lambda: h2.copy_(d2, non_blocking=True)); print("D2H GB/s", N / b / 1e9)
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
c = t(both); print("concurrent H2D+D2H GB/s each", N / c / 1e9)
