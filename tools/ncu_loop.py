"""Stall-sample breakdown of the chain warp's stage loop in an ncu source
(SASS) CSV dump: finds the innermost backward branch enclosing the chain's
SHFL (.UP for K2, .DOWN for K3) and classifies the loop's samples.
usage: python tools/ncu_loop.py src.csv [UP|DOWN] [top]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
kind = sys.argv[2] if len(sys.argv) > 2 else "DOWN"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) >= len(hdr)]
addr = [int(r[ix["Address"]], 16) for r in body]
src = [r[ix["Source"]].strip() for r in body]
smp = [int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body]
stall = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
shfl = [i for i, s in enumerate(src) if f"SHFL.{kind} PT" in s]
if not shfl:
    sys.exit("no chain SHFL found")
lo_i, hi_i = min(shfl), max(shfl)
best = None
for i, s in enumerate(src):
    m = re.search(r"BRA (?:\S+, )?0x([0-9a-f]+)", s)
    if m and i > hi_i:
        t = int(m.group(1), 16)
        if t <= addr[lo_i] and (best is None or addr[i] - t < best[1] - best[0]):
            best = (t, addr[i])
a0, a1 = best
idx = [i for i in range(len(body)) if a0 <= addr[i] <= a1]
tot = sum(smp[i] for i in idx)
cls = {}
for i in idx:
    op = src[i].split()[0] if not src[i].startswith("@") else src[i].split()[1]
    c = ("chain" if lo_i - 3 <= i <= hi_i + 12 else
         "LDS" if op.startswith("LDS") else "STS" if op.startswith("STS") else
         "SYNCS/BRA" if op.startswith(("SYNCS", "BRA", "BSYNC", "BSSY")) else "other")
    cls[c] = cls.get(c, 0) + smp[i]
print(f"loop {a0:x}..{a1:x}: {len(idx)} instr, {tot} samples")
for c, v in sorted(cls.items(), key=lambda x: -x[1]):
    print(f"  {c:10s} {v:6d} {100 * v / max(tot, 1):5.1f}%")
rs = {}
for i in idx:
    for h in stall:
        v = int(body[i][ix[h]] or 0)
        rs[h] = rs.get(h, 0) + v
print("  reasons:", ", ".join(f"{h[6:]} {100 * v / max(tot, 1):.0f}%" for h, v in sorted(rs.items(), key=lambda x: -x[1])[:6]))
for i in sorted(idx, key=lambda i: -smp[i])[:top]:
    st = {h[6:]: body[i][ix[h]] for h in stall if body[i][ix[h]] not in ("0", "")}
    print(f"{smp[i]:6d} {addr[i] & 0xfffff:05x} {src[i][:64]:64s} {st}")
