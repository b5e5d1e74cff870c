"""Per-region sample split of an ncu source CSV: cumulative samples between
barrier / arrive / copy instructions (identifies which warp role is busy).
usage: python tools/ncu_roles.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) >= len(hdr)]
stall = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
keys = ("TRYWAIT", "SYNCS.ARRIVE", "UBLKCP", "ARRIVES.LDGSTSBAR", "ATOMG", "BAR.SYNC", "EXIT")
cum, rs = 0, {}
for r in body:
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    cum += n
    for h in stall:
        v = int(r[ix[h]] or 0)
        if v:
            rs[h] = rs.get(h, 0) + v
    s = r[ix["Source"]]
    if any(k in s for k in keys) and cum > 50:
        top = sorted(rs.items(), key=lambda x: -x[1])[:3]
        print(f"{r[ix['Address']][-5:]} {cum:7d}  {s.strip()[:60]:60s} {[(h[6:], v) for h, v in top]}")
        cum, rs = 0, {}
