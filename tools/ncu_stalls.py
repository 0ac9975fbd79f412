"""Summarise ncu's per-instruction warp-stall sampling (source page, SASS):
  ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv
  python tools/ncu_stalls.py X.csv [top]
Prints the stall-reason totals (barrier waits separated) and the top
instructions by non-barrier samples."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
items = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        n = int(r[idx["# Samples"]] or 0)
    except ValueError:
        continue
    if n == 0:
        continue
    d = {h[6:]: int(r[idx[h]] or 0) for h in stalls}
    tot.update(d)
    items.append((n - d.get("barrier", 0), n, r[idx["Address"]][-6:], r[idx["Source"]].strip()[:64],
                  {k: v for k, v in d.items() if v}))
allv = sum(tot.values())
print(f"samples {allv}; barrier {tot['barrier']}; non-barrier {allv - tot['barrier']}")
for k, v in tot.most_common():
    if v and k != "barrier":
        print(f"  {k:20s} {v:6d}  {v / max(1, allv - tot['barrier']):.0%}")
items.sort(key=lambda t: (t[0], t[1]), reverse=True)
for it in items[:top]:
    print(it[0], it[1], it[2], it[3], it[4])
