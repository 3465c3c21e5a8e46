"""Per-source-line shared-memory wavefronts (ideal / excessive) from an ncu report.
usage: ncu_smem_lines.py REPORT [LAUNCH_INDEX] [topN]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass',
                      '--launch-skip', str(idx), '--launch-count', '1'], capture_output=True, text=True).stdout
hdr = None; cur = None; src = {}
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None or len(r) < len(hdr): continue
    d = dict(zip(hdr[2:], r[2:]))
    if r[0].strip():
        cur = int(r[0]); src[cur] = r[1].strip()[:100]
    def f(k):
        try: return float((d.get(k) or '0').replace(',', ''))
        except ValueError: return 0.0
    a = agg[cur]; a[0] += f('L1 Wavefronts Shared'); a[1] += f('L1 Wavefronts Shared Ideal'); a[2] += f('L1 Wavefronts Shared Excessive')
tw = sum(v[0] for v in agg.values()); te = sum(v[2] for v in agg.values())
print(f'shared wavefronts {tw:.3e}, excessive {te:.3e} ({te / max(tw, 1) * 100:.1f}%)')
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    if v[0] == 0: continue
    print(f'{k:5d} wav {v[0]:.2e} ideal {v[1]:.2e} excess {v[2]:.2e} | {src.get(k, "")}')
