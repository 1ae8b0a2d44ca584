"""Top source lines by warp-stall samples from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv, sys, collections
path = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = []
fname = None; hdr = None
for r in csv.reader(open(path)):
    if not r: continue
    if r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None or r[0] in ('', 'Function Name'): continue
    d = dict(zip(hdr[4:], r[4:]))
    try: s = int(d.get('Warp Stall Sampling (All Samples)', '0') or 0)
    except ValueError: continue
    rows.append((s, fname, r[0], r[1][:80], d))
tot = sum(x[0] for x in rows)
print('total samples', tot)
keys = ['stall_barrier', 'stall_long_sb', 'stall_wait', 'stall_selected', 'stall_short_sb', 'stall_branch_resolving']
for s, f, ln, src, d in sorted(rows, key=lambda x: -x[0])[:top]:
    ks = ' '.join(f"{k[6:]}={d.get(k, '0')}" for k in keys if d.get(k, '0') not in ('0', ''))
    print(f"{100*s/tot:5.1f}% {f}:{ln:5s} {src:80s} {ks}")
