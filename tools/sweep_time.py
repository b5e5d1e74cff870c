"""K2 / K3 launch times (CUDA events, no tracing) of a single block.

usage: python tools/sweep_time.py [f64|f32] [n | nxXnyXnz] [iters] [pxXpyXpz]
Prints ms per launch and ns per slice of one brick for the isolated-brick
grid 8x32xnz (one brick) and per-launch ms for bigger grids."""
import sys

sys.path.insert(0, ".")
import paper_1303_4538_b200 as sip  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
dims = [int(x) for x in sys.argv[2].split("x")] if len(sys.argv) > 2 else [256]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
pd = tuple(int(x) for x in sys.argv[4].split("x")) if len(sys.argv) > 4 else (1, 1, 1)
nx, ny, nz = dims if len(dims) == 3 else dims * 3
s = sip.Solver(None, prec, 0, lattice=((nx, ny, nz), pd))
s.generate(0, 1304)
s.factor(0.92)
s.load_phi([sip.field(*d) for (_, d, _) in s.blocks])
s.iterate(3)
s.set_profiling(True)
s.iterate(iters)
p = s.profile()
g = s.geometry()
slices = g["slices"] // g["bricks"]
f, b = p["fwd_ms"] / iters, p["bwd_ms"] / iters
print(f"{prec} {nx}x{ny}x{nz} / {pd}: K2 {f * 1e3:.1f} us  K3 {b * 1e3:.1f} us  "
      f"({f * 1e6 / slices:.1f} / {b * 1e6 / slices:.1f} ns per brick slice)")
s.close()
