"""Warp instructions executed per SASS opcode (deduplicated by address) from an
`ncu --page source --csv --print-source=cuda,sass` export (gzip ok)."""
import collections, csv, gzip, sys
path = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
seen = {}
for r in csv.reader(f):
    if len(r) < 9 or not r[2].startswith("0x"):
        continue
    try:
        seen[r[2]] = (r[3].strip(), int(r[7]))
    except ValueError:
        pass
ops = collections.Counter()
for ins, n in seen.values():
    op = ins.split()[0]
    if op.startswith("@"):
        op = ins.split()[1]
    ops[op] += n
tot = sum(ops.values())
print(f"total warp instructions {tot} over {len(seen)} SASS addresses")
for op, n in ops.most_common(top):
    print(f"{n:12d} {100*n/tot:5.1f}% {op}")
