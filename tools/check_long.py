"""Long-run sanity: many iterate() batches on config 1; all norms must be
positive and decreasing; per-batch device time."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_1303_4538_b200 as sip
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
g = (256, 256, 256)
s = sip.Solver(None, prec, 0, lattice=(g, (1, 1, 1)))
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
s.set_stream(stream.cuda_stream)
s.generate(0, 1304); s.factor(0.92); s.load_phi([sip.field(*g)])
for b in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); s.iterate(50); e1.record(stream); torch.cuda.synchronize()
    print(f"batch {b}: {e0.elapsed_time(e1):.2f} ms -> {16777216*50/e0.elapsed_time(e1)/1e3:.0f} MLUP/s")
n = s.read_norms(0, 400)
print("norms[0,1,50,100,200,399]:", n[[0, 1, 50, 100, 200, 399]])
print("zeros:", int((n == 0).sum()), "non-decreasing steps:", int((np.diff(n) >= 0).sum()))
