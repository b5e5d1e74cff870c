"""Summarise an ncu --page source --csv (SASS) dump: total stall reasons and the
hottest instructions.  usage: python tools/ncu_src_stalls.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: 0 for h in stall_cols}
body = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        n = int(r[ix["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    for h in stall_cols:
        try:
            tot[h] += int(r[ix[h]])
        except ValueError:
            pass
    body.append((n, r[ix["Address"]], r[ix["Source"]].strip(),
                 {h: r[ix[h]] for h in stall_cols if r[ix[h]] not in ("0", "")}))
S = sum(tot.values()) or 1
print("total samples", S)
for h, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v:
        print(f"  {h:28s} {v:8d} {100 * v / S:5.1f}%")
print("hottest instructions:")
for n, a, src, st in sorted(body, key=lambda x: -x[0])[:top]:
    print(f"{n:6d} {a[-5:]} {src[:60]:60s} {st}")
