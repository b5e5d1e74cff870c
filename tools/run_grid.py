"""Run a few SIP iterations on one grid (for ncu captures)."""
import sys
sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
g = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "16x16x256").split("x"))
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 4
s = sip.Solver(None, prec, 0, lattice=(g, (1, 1, 1)))
s.generate(0, 1304)
s.factor(0.92)
s.load_phi([sip.field(*g)])
s.iterate(iters)
s.synchronize()
print("ok")
