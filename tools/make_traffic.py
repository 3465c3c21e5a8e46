"""Build profiles/ncu_traffic.json (DRAM bytes per bench-bracket launch, per kernel class)
from ncu launch lists of one warm round trip (tools/gpu_round.sh): the bench's roofline
`traffic` field. usage: make_traffic.py CONFIG=launches.csv [CONFIG=launches.csv ...]"""
import csv, io, json, re, sys, collections
from pathlib import Path

CLASSES = {  # bench kind -> (kernel-name regex, bench brackets per round trip)
    "fused_decompose_level": (r"k_(level_(fused|face)|face_(slab|zload))<\w+, 0[,>]", None),
    "fused_recompose_level": (r"k_(level_(fused|face)|face_(slab|zload))<\w+, 2[,>]", None),
    "recompose_interp": (r"k_interp_(march|face)", None),
    "thomas": (r"k_thomas_(lines|rows|long|stream|planes_ws|band)", None),
    "assembly": (r"k_(scatter|merge)_even", None),
    "small_levels": (r"k_(tail_\w+|lpk|thomas|coefficients|gather|gpk_dec|gpk_rec|axpy|check_finite)<", None),
}

def per_trip(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO(''.join(lines))))
    agg = collections.OrderedDict()
    for r in rows:
        i = int(r['ID'])
        name = r['Kernel Name'].split('(')[0].replace('void ', '').replace('(int)', '')
        d = agg.setdefault(i, {'name': name})
        d[r['Metric Name']] = float(r['Metric Value'].replace(',', ''))
    ids = sorted(agg)
    # the measured round trip follows the last marker (fill) kernel of tools/prof_one.py
    marks = [i for i in ids if re.search(r"[Ff]ill", agg[i]['name'])]
    if marks:
        start = marks[-1] + 1
    else:  # older lists: the second decompose's first fused launch
        dec = [i for i in ids if re.search(r"k_level_fused<\w+, 0>", agg[i]['name'])]
        start = dec[len(dec) // 2]
    return [agg[i] for i in ids if i >= start]

out_path = Path(__file__).resolve().parent.parent / "profiles" / "ncu_traffic.json"
res = json.loads(out_path.read_text()) if out_path.exists() else {}
for arg in sys.argv[1:]:
    cfg, path = arg.split('=', 1)
    launches = per_trip(path)
    cls = {}
    for kind, (rx, _) in CLASSES.items():
        sel = [l for l in launches if re.search(rx, l['name'])]
        main = [l for l in sel if not re.search(r"face", l['name'])]
        if not main:
            continue
        tot = sum(l.get('dram__bytes_read.sum', 0) + l.get('dram__bytes_write.sum', 0) for l in sel)
        # one bench bracket per main-kernel launch (faces share their level's bracket)
        cls[kind] = round(tot / len(main))
    # the whole round trip: every launch's DRAM bytes and time (bench dram_frac)
    cls["_step"] = {
        "dram_bytes": round(sum(l.get('dram__bytes_read.sum', 0) + l.get('dram__bytes_write.sum', 0)
                                for l in launches)),
        "kernel_ms": round(sum(l.get('gpu__time_duration.sum', 0) for l in launches) / 1e6, 4),
        "launches": len(launches), "source": Path(path).name}
    res[cfg] = cls
    print(cfg, cls)
out_path.write_text(json.dumps(res, indent=1) + "\n")
