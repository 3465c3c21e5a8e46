"""Opcode histogram (weighted by executed instructions) from an ncu report's SASS page."""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ie, st = h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
ops, stalls, tot = collections.Counter(), collections.Counter(), 0
for r in rows[2:]:
    if len(r) != len(h) or not r[1].split():
        continue
    n = float(r[ie] or 0)
    toks = r[1].split()
    op = toks[1] if toks[0].startswith('@') else toks[0]
    op = op.split('.')[0]
    ops[op] += n
    stalls[op] += float(r[st] or 0)
    tot += n
print('total warp instructions', tot)
for op, n in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f'  {op:10s} {n / tot * 100:6.2f}%  stall samples {stalls[op]:8.0f}')
