"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections, csv, json, re, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ui = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {'nsecond': 1.0, 'usecond': 1e3, 'msecond': 1e6, 'second': 1e9}
for r in data:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
        continue
    name = re.sub(r'\(.*', '', r[ki])
    name = re.sub(r'^void ', '', name).replace('(anonymous namespace)::', '')
    name = re.sub(r'<.*', lambda m: '<' + m.group(0)[1:40] + '>' if len(m.group(0)) > 40 else m.group(0), name)
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
tot = sum(v[1] for v in agg.values())
out = []
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append({'kernel': k, 'launches': c, 'total_ms': t / 1e6, 'share': t / tot})
    print(f"{k:70s} {c:5d} launches {t / 1e6:9.3f} ms {100 * t / tot:5.1f}%")
print(f"total {tot / 1e6:.3f} ms (cold-cache, serialised replay: compare shares)")
if len(sys.argv) > 2:
    json.dump({'source': sys.argv[1], 'kernels': out, 'total_ms': tot / 1e6}, open(sys.argv[2], 'w'), indent=1)
