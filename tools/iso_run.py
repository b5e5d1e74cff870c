"""Minimal isolated-tile run (16x16 x nz) for ncu source-level stall sampling."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1303_4538_b200 as sip
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
g = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "16x16x1024").split("x"))
s = sip.Solver(None, prec, 0, lattice=(g, (1, 1, 1)))
s.generate(0, 1304); s.factor(0.92); s.load_phi([sip.field(*g)])
s.iterate(3)
torch.cuda.synchronize()
print("ok")
