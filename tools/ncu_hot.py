"""Summarise an ncu source page (SASS) CSV: stall totals and the hottest instructions.
usage: ncu -i X.ncu-rep --page source --csv --print-source=sass > x.csv; python tools/ncu_hot.py x.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
S = ix["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
def num(x):
    try: return float(x.replace(",", ""))
    except: return 0.0
tot = {s: sum(num(r[ix[s]]) for r in data) for s in stalls}
allsamp = sum(num(r[S]) for r in data)
print("total samples", allsamp)
for s, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {s:28s} {v:10.0f} {100*v/max(allsamp,1):5.1f}%")
print("hottest:")
for r in sorted(data, key=lambda r: -num(r[S]))[:N]:
    top = sorted(((num(r[ix[s]]), s) for s in stalls), reverse=True)[:2]
    print(f"{r[ix['Address']]:>6} {num(r[S]):7.0f} {r[ix['Source']][:60]:60s} " + " ".join(f"{s[6:]}={v:.0f}" for v, s in top))
