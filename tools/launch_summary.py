"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel name."""
import collections, csv, io, sys
lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
F = {'ns': 1e-9, 'nsecond': 1e-9, 'us': 1e-6, 'usecond': 1e-6, 'ms': 1e-3, 'msecond': 1e-3, 's': 1, 'second': 1}
agg = collections.OrderedDict()
for r in rows:
    if r.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    k = r['Kernel Name'].split('(')[0]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += float(r['Metric Value'].replace(',', '')) * F[r['Metric Unit']]
tot = sum(a[1] for a in agg.values())
print("%-64s %8s %12s %7s %10s" % ("kernel", "launches", "total_s", "share", "avg_us"))
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%-64s %8d %12.5f %6.2f%% %10.2f" % (k[:64], c, t, 100 * t / tot, 1e6 * t / c))
print("%-64s %8d %12.5f" % ("TOTAL", sum(a[0] for a in agg.values()), tot))
