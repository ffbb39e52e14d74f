# Dev tool: per-source-line stall samples from 'ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv'. Usage: python tools/srcagg.py X.csv [N] [first_line last_line]
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None; f = None; data = []
for r in rows:
    if not r: continue
    if r[0] == 'File Path': f = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr and r[0] not in ('', 'Function Name'):
        try: s = int(r[4])
        except: continue
        data.append((s, f, r[0], r[1][:90], r))
tot = sum(d[0] for d in data)
print('total samples', tot)
sc = [i for i, h in enumerate(hdr) if h.startswith('stall') and 'Not Issued' not in h]
for s, f, l, src, r in sorted(data, key=lambda x: -x[0])[:N]:
    top = sorted(((int(r[i]) if r[i].isdigit() else 0, hdr[i][6:]) for i in sc), reverse=True)[:2]
    print(f"{s:6d} {100*s/tot:4.1f}% {f}:{l}: {src} | " + ' '.join(f"{n}={v}" for v, n in top if v))
if len(sys.argv) > 4:
    lo, hi = int(sys.argv[3]), int(sys.argv[4])
    sel = [d for d in data if d[1] == 'chains.cu' and lo <= int(d[2]) <= hi]
    t2 = sum(d[0] for d in sel)
    print('lines', lo, hi, 'samples', t2)
    agg = {}
    for s, f, l, src, r in data:
        if f == 'chains.cu' and lo <= int(l) <= hi:
            for i in sc:
                agg[hdr[i]] = agg.get(hdr[i], 0) + (int(r[i]) if r[i].isdigit() else 0)
    print(sorted(((v, k) for k, v in agg.items() if v), reverse=True)[:10])
