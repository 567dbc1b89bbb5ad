"""Summarise an ncu --metrics gpu__time_duration.sum launch list by kernel."""
import csv, collections, io, sys
txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(txt)))
t = collections.defaultdict(float); n = collections.Counter()
for r in rows:
    if r['Metric Name'] != 'gpu__time_duration.sum': continue
    k = r['Kernel Name'].split('(')[0].replace('void ','')
    t[k] += float(r['Metric Value']); n[k] += 1
tot = sum(t.values())
print(f"{'kernel':45s} {'launches':>8s} {'total ms':>10s} {'share':>6s} {'us/launch':>10s}")
for k,v in sorted(t.items(), key=lambda kv:-kv[1]):
    print(f"{k:45s} {n[k]:8d} {v/1e6:10.3f} {v/tot:6.3f} {v/n[k]/1e3:10.1f}")
print(f"{len(rows)} launches, {tot/1e6:.3f} ms total")
