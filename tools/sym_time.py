"""Symmetric fast path at full size: a kind-3 (symmetric)
256^3 system timed with the general K2 and with the flagged fast path; the
norm histories must be identical (same values, same operation order)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1303_4538_b200 as sip
for prec in ("f64", "f32"):
    g = (256, 256, 256)
    s = sip.Solver(None, prec, 0, lattice=(g, (1, 1, 1)))
    st = torch.cuda.Stream(); torch.cuda.set_stream(st); s.set_stream(st.cuda_stream)
    s.generate(3, 1309)
    s.factor(0.92)
    res = {}
    for flag in (False, True):
        s.set_symmetric(0, flag)
        s.load_phi([sip.field(*g)])  # restarts the iteration count
        s.iterate(3)
        n0 = s.read_norms(0, 3)
        s.set_profiling(True); s.iterate(10); pr = s.profile(); s.set_profiling(False)
        res[flag] = (n0, pr["fwd_ms"] / 10, pr["bwd_ms"] / 10)
    s.close()
    same = np.array_equal(res[False][0], res[True][0])
    print(f"{prec}: general K2 {res[False][1]*1e3:.1f} us, symmetric K2 {res[True][1]*1e3:.1f} us "
          f"({100*(1-res[True][1]/res[False][1]):.1f} % less), norms identical: {same}")
