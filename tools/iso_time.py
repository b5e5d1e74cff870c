"""Untraced per-step time of an isolated tile (16x16 columns x nz) and of config 1."""
import sys
sys.path.insert(0, ".")
import torch
import paper_1303_4538_b200 as sip
for prec in ("f64", "f32"):
    for g in ((16, 16, 1024), (256, 256, 256)):
        s = sip.Solver(None, prec, 0, lattice=(g, (1, 1, 1)))
        st = torch.cuda.Stream(); torch.cuda.set_stream(st); s.set_stream(st.cuda_stream)
        s.generate(0, 1304); s.factor(0.92); s.load_phi([sip.field(*g)])
        s.iterate(3)
        s.set_profiling(True); s.iterate(10); pr = s.profile(); s.set_profiling(False)
        ns = g[2] + 30
        print(f"{prec} {g}: fwd {pr['fwd_ms']/10*1e3:.1f} us ({pr['fwd_ms']/10*1e6/ns:.0f} ns/step), "
              f"bwd {pr['bwd_ms']/10*1e3:.1f} us ({pr['bwd_ms']/10*1e6/ns:.0f} ns/step)")
        s.close()
