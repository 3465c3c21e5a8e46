"""Per-source-line totals (instructions executed, stall samples) from an ncu report.
usage: ncu_lines.py REPORT LAUNCH_INDEX [topN]"""
import csv, io, subprocess, sys, collections
rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass',
                      '--launch-skip', str(idx), '--launch-count', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; cur_file = None; cur_line = None; src = {}
agg = collections.defaultdict(lambda: [0, 0, 0])
for r in rows:
    if not r: continue
    if r[0] == 'Line No':
        hdr = r; continue
    if r[0] == 'File Name':
        cur_file = r[1].split('/')[-1]; continue
    if hdr is None or len(r) < len(hdr): continue
    d = dict(zip(hdr[2:], r[2:]))
    if r[0].strip():
        cur_line = (cur_file, int(r[0])); src[cur_line] = r[1].strip()[:90]
    if not d.get('Address'): continue
    try:
        ie = float(d.get('Instructions Executed', '0') or 0)
        ss = float(d.get('Warp Stall Sampling (All Samples)', '0') or 0)
    except ValueError:
        continue
    a = agg[cur_line]; a[0] += ie; a[1] += ss; a[2] += 1
tot_i = sum(v[0] for v in agg.values()); tot_s = sum(v[1] for v in agg.values())
print(f'total warp-instr {tot_i:.3e}, stall samples {tot_s:.0f}')
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f'{k[0]}:{k[1]:4d} inst {100*v[0]/tot_i:5.1f}% stall {100*v[1]/tot_s:5.1f}% nsass {v[2]:3d} | {src.get(k, "")}')
