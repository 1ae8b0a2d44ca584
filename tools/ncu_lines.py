"""Top CUDA source lines by warp-stall samples from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > out.csv`."""
import collections
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
keys = ["stall_barrier", "stall_long_sb", "stall_wait", "stall_selected", "stall_short_sb",
        "stall_branch_resolving", "stall_math_pipe_throttle", "stall_lg_throttle", "stall_mio_throttle"]
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
fname, hdr = None, None
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    key = (fname, int(r[0]))
    src[key] = r[1][:90]
    for k in ["Warp Stall Sampling (All Samples)", "Instructions Executed"] + keys:
        try:
            agg[key][k] += float(d.get(k, "0") or 0)
        except ValueError:
            pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values()) or 1
print("total samples", int(tot))
for key, v in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]:
    s = v["Warp Stall Sampling (All Samples)"]
    ks = " ".join(f"{k[6:]}={int(v[k])}" for k in keys if v[k] > 0.02 * s)
    print(f"{100 * s / tot:5.1f}% {key[0]}:{key[1]:<5d} {src[key]:90s} {ks}")
