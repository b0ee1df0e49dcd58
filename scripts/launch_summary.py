"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel share."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]; data = rows[hi + 1:]
ki, mi, vi, ui = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
tot = collections.defaultdict(float); cnt = collections.Counter()
scale = {'nsecond': 1, 'usecond': 1e3, 'msecond': 1e6, 'second': 1e9}
for r in data:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
        continue
    v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1)
    name = r[ki].split('(')[0].replace('void ', '')
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
print(f"# ncu launch list {sys.argv[1]} (cold-cache, serialised per-launch times: compare shares)")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{100 * v / T:6.2f}%  {v / 1e6:10.2f} ms  {cnt[k]:6d} launches  {k}")
print(f"total {T / 1e6:.2f} ms, {sum(cnt.values())} launches")
