"""Top source lines by warp-stall samples from `ncu --page source --csv --print-source=cuda,sass`."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
cur_file = None
lines = []  # (samples, file, line, src)
sass = {}
last = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 7 or r[0] == "Line No":
        continue
    if r[0]:  # source line
        try:
            s = int(r[4])
        except ValueError:
            continue
        last = (cur_file, r[0], r[1].strip())
        lines.append([s, cur_file, int(r[0]), r[1].strip()[:90]])
    elif last and r[2] not in ("...", "-") and r[4] not in ("-", ""):
        sass.setdefault(last, []).append((int(r[4]), r[3].strip()[:60]))
tot = sum(l[0] for l in lines) or 1
lines.sort(key=lambda x: -x[0])
print(f"total samples {tot}")
for s, f, ln, src in lines[:top]:
    print(f"{s:7d} {100*s/tot:5.1f}%  {f}:{ln:<4d} {src}")
    ins = sorted(sass.get((f, str(ln), src), []), reverse=True)[:3] if False else None
