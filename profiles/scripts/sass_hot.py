"""Hot SASS instructions of an ncu source-page CSV (ncu -i rep --page source --csv --print-source sass):
stall samples per instruction, grouped by opcode, and the top individual instructions.
Usage: python profiles/scripts/sass_hot.py file.csv[.gz] [top]"""
import collections
import csv
import gzip
import io
import sys

p = sys.argv[1]
txt = (gzip.open(p, "rt") if p.endswith(".gz") else open(p)).read()
lines = txt.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
def _i(v):
    try:
        return int(v)
    except (TypeError, ValueError):
        return 0


samp = lambda r: _i(r.get("Warp Stall Sampling (All Samples)"))   # (several kernels: repeated headers count 0)
exe = lambda r: _i(r.get("Instructions Executed"))
tot = sum(samp(r) for r in rows) or 1
toti = sum(exe(r) for r in rows) or 1
by = collections.defaultdict(lambda: [0, 0])
for r in rows:
    op = r["Source"].split()[0] if r["Source"].split() else "?"
    if op.startswith("@"):
        op = r["Source"].split()[1]
    op = op.split(".")[0]
    by[op][0] += samp(r)
    by[op][1] += exe(r)
print(f"{len(rows)} SASS instructions, {tot} stall samples, {toti} warp-instructions executed")
print("opcode          samples%   executed%")
for op, (s, e) in sorted(by.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"{op:14s} {100 * s / tot:8.1f} {100 * e / toti:10.1f}")
print("\ntop instructions by stall samples:")
for r in sorted(rows, key=lambda r: -samp(r))[:top]:
    print(f"{100 * samp(r) / tot:5.1f}%  {r['Address'][-5:]}  {r['Source'].strip()[:80]}")
