"""K2 / K3 time at config 1 (256^3) for the library in $SIPB_LIB (10 iterations, CUDA events)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1303_4538_b200 as sip
tag = sys.argv[1] if len(sys.argv) > 1 else ""
out = []
for prec in ("f64", "f32"):
    g = (256, 256, 256)
    s = sip.Solver(None, prec, 0, lattice=(g, (1, 1, 1)))
    st = torch.cuda.Stream(); torch.cuda.set_stream(st); s.set_stream(st.cuda_stream)
    s.generate(0, 1304); s.factor(0.92); s.load_phi([sip.field(*g)])
    s.iterate(3)
    s.set_profiling(True); s.iterate(20); pr = s.profile(); s.set_profiling(False)
    out.append(f"{prec} fwd {pr['fwd_ms']/20*1e3:.1f} bwd {pr['bwd_ms']/20*1e3:.1f}")
    s.close()
print(f"{tag:10s} " + " | ".join(out))
