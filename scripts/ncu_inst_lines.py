"""Instructions executed per source line from `ncu --page source --csv --print-source=cuda,sass`
(gzip ok): top lines by warp-level instructions executed, with average active threads."""
import csv, gzip, io, sys
path = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
cur = None; out = []; tot = 0
for r in csv.reader(f):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if len(r) < 9 or r[0] == "Line No" or not r[0]:
        continue
    try:
        ie = int(r[7]); thr = float(r[10]) if r[10] not in ("", "-") else 0
    except ValueError:
        continue
    tot += ie
    out.append((ie, thr, cur, r[0], r[1].strip()[:80]))
out.sort(reverse=True)
print(f"total warp instructions {tot}")
for ie, thr, fn, ln, src in out[:top]:
    print(f"{ie:12d} {100*ie/tot:5.1f}% thr={thr:5.1f} {fn}:{ln} {src}")
