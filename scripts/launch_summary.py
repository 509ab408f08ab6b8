"""Summarise an ncu --csv launch list: per kernel (in first-sort launch order) count, mean us, DRAM bytes."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]; data = rows[hi + 1:]
ki, mi, vi, ui, ii = (hdr.index(c) for c in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
per = collections.defaultdict(dict)
names = {}
for r in data:
    if len(r) <= vi: continue
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    v *= {'ns': 1e-3, 'us': 1, 'ms': 1e3, 'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
    per[int(r[ii])][r[mi]] = v
    names[int(r[ii])] = r[ki].split('(')[0].replace('void ', '')
only = sys.argv[2] if len(sys.argv) > 2 else 'gbs::'
agg = collections.OrderedDict()
for i in sorted(per):
    n = names[i]
    if only not in n: continue
    a = agg.setdefault(n, [0, 0.0, 0.0])
    a[0] += 1; a[1] += per[i].get('gpu__time_duration.sum', 0)
    a[2] += per[i].get('dram__bytes_read.sum', 0) + per[i].get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':58s} {'n':>3s} {'us/launch':>10s} {'share':>6s} {'DRAM MB/launch':>14s}")
for n, (c, t, b) in agg.items():
    print(f"{n[:58]:58s} {c:3d} {t / c:10.1f} {100 * t / tot:5.1f}% {b / c / 1e6:14.1f}")
print(f"total {tot:.1f} us over all listed launches")
