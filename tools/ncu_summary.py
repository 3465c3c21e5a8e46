"""Summarise an ncu --csv launch list: per-launch time and DRAM bytes of the measured round
trip (after the last marker fill kernel of tools/prof_one.py; else the second half)."""
import csv, collections, sys, io
path = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(io.StringIO(''.join(lines))))
ids = sorted({int(r['ID']) for r in rows})
start = ids[int(len(ids) * (1 - frac))] if frac < 1 else 0
marks = sorted({int(r['ID']) for r in rows if 'ill' in r['Kernel Name'] and 'Fill' in r['Kernel Name'] or 'fill' in r['Kernel Name']})
if marks:  # tools/prof_one.py: the measured round trip follows the last marker fill kernel
    start = marks[-1] + 1
agg = collections.OrderedDict()
for r in rows:
    i = int(r['ID'])
    if i < start: continue
    name = r['Kernel Name'].split('(')[0].replace('void ', '')[:70]
    agg.setdefault(i, {'name': name, 'grid': r['Grid Size']})[r['Metric Name']] = float(r['Metric Value'].replace(',', ''))
tot = 0; byk = collections.OrderedDict()
for i, m in agg.items():
    t = m.get('gpu__time_duration.sum', 0) / 1e3; tot += t
    b = (m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0))
    k = byk.setdefault(m['name'], [0, 0.0, 0.0]); k[0] += 1; k[1] += t; k[2] += b
    if t > float(sys.argv[3] if len(sys.argv) > 3 else 200):
        print(f"{i:4d} {m['name']:70s} {m['grid']:>14s} {t:9.1f}us R={m.get('dram__bytes_read.sum',0)/1e9:6.3f}GB W={m.get('dram__bytes_write.sum',0)/1e9:6.3f}GB  {b/1e3/max(t,1e-9):7.0f}GB/s")
print(f"total {tot/1e3:.3f} ms over {len(agg)} launches")
for n, (c, t, b) in sorted(byk.items(), key=lambda kv: -kv[1][1]):
    print(f"  {n:70s} x{c:3d} {t/1e3:8.3f} ms {b/1e9:7.2f} GB")
