"""Python mirror of the reference's sip module interface on
top of the B200 C-ABI library (include/sip_c.h, libsip_b200.so).

Names, argument meaning and error behaviour follow the specification:

    StencilSystem   -> StencilSystem
    SipFactors   -> SipFactors (device-resident, stamped)
    SipConfig   -> SipConfig
    SolveReport   -> SolveReport
    sip_factor   -> sip_factor
    residual_general -> residual_general
    residual_symmetric -> residual_symmetric
    sip_sweep   -> sip_sweep
    solve   -> solve
    errors         (error.hpp:34-50)   -> SingularFactorError, StaleFactorsError, MisuseError
    assemble_poisson -> assemble_poisson / Solver.assemble_poisson
    FlowState   -> Flow (device-resident u, v, w, p)
    pressure_correct -> pressure_correct / Flow.pressure_correct

Arrays are numpy float64 Field3 arrays (proj/include/bsfv/field.hpp:25-44):
shape (nz+2, ny+2, nx+2), i fastest, interior 1..n.  Coefficients use the
matrix-entry sign convention (A_nb = -a_nb).

There is no CPU fallback: every operation runs the sm_100a kernels; when the
shared library or a CUDA device is missing the calls raise.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import time
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SIPB_LIB") or os.path.join(_HERE, "libsip_b200.so")

SIP_OK, SIP_ERR_SINGULAR, SIP_ERR_STALE, SIP_ERR_MISUSE = 0, 1, 2, 3
SIP_ERR_CONFIG, SIP_ERR_CUDA, SIP_ERR_NCCL, SIP_ERR_NOMEM = 4, 5, 6, 7
SIP_ERR_FORMAT, SIP_ERR_PROTOCOL, SIP_ERR_NOCONV = 8, 9, 10
BC = {"wall": 0, "periodic": 1, "symmetry": 2}
FLOW_FIELDS = {"u": 0, "v": 1, "w": 2, "p": 3}
PREC = {"f64": 0, "double": 0, "f32": 1, "single": 1}

ARRAYS = ("AP", "AW", "AE", "AS", "AN", "AB", "AT", "Q")

# Exported symbols declared by include/sip_c.h (checked by the CPU tests).
EXPORTS = (
    "sip_version", "sip_status_string", "sip_last_error", "sip_create", "sip_create_lattice",
    "sip_destroy", "sip_num_local_blocks", "sip_local_block", "sip_set_system", "sip_set_source",
    "sip_generate_system", "sip_factor", "sip_solve", "sip_load_phi", "sip_store_phi",
    "sip_iterate", "sip_read_norms", "sip_synchronize", "sip_residual", "sip_set_symmetric",
    "sip_set_stream",
    "sip_get_stream", "sip_set_profiling", "sip_get_profile", "sip_launch_count", "sip_geometry",
    "sip_nccl_unique_id", "sip_generate_host", "sip_plan_block_ranks", "sip_plan_halo",
    "sip_ftt1_read", "sip_ftt1_write", "sip_ftt1_validate", "sip_set_halo_tables",
    "sip_plan_halo_periodic", "sip_assemble_poisson", "sip_flow_create", "sip_flow_destroy",
    "sip_flow_set", "sip_flow_get", "sip_flow_divergence", "sip_pressure_correct",
    "sip_factor_count", "sip_num_global_blocks", "sip_solve_ex", "sip_set_source_async",
    "sip_solve_async", "sip_wait_async",
)


class Error(RuntimeError):
    """bsfv::Error (error.hpp:10-14)."""


class ConfigError(Error):
    """bsfv::ConfigError (error.hpp:16-19)."""


class SingularFactorError(Error):
    """bsfv::SingularFactorError (error.hpp:34-37): names the cell."""


class StaleFactorsError(Error):
    """bsfv::StaleFactorsError (error.hpp:40-43)."""


class MisuseError(Error):
    """bsfv::MisuseError (error.hpp:47-50)."""


class FormatError(Error):
    """bsfv::FormatError (error.hpp:22-31): malformed FTT1 file; `offset` = byte offset."""

    def __init__(self, what: str, offset: int = -1):
        super().__init__(what)
        self.offset = offset


class ProtocolError(Error):
    """bsfv::ProtocolError (error.hpp:53-57): unmatched transfer-table entries."""


class NonConvergenceError(Error):
    """bsfv::NonConvergenceError (error.hpp:72-80): the pressure-correction outer
    loop hit its cap with the divergence above the threshold; `defect` = last L1."""

    def __init__(self, what: str, defect: float = float("nan")):
        super().__init__(what)
        self.defect = defect


_EXC = {SIP_ERR_SINGULAR: SingularFactorError, SIP_ERR_STALE: StaleFactorsError,
        SIP_ERR_MISUSE: MisuseError, SIP_ERR_CONFIG: ConfigError, SIP_ERR_FORMAT: FormatError,
        SIP_ERR_PROTOCOL: ProtocolError}

_lib = None
_dp = ctypes.POINTER(ctypes.c_double)


def lib():
    """Load libsip_b200.so (built by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = ctypes.CDLL(LIB_PATH)
        L.sip_version.restype = ctypes.c_char_p
        L.sip_status_string.restype = ctypes.c_char_p
        L.sip_last_error.restype = ctypes.c_char_p
        L.sip_last_error.argtypes = [ctypes.c_void_p]
        L.sip_get_stream.restype = ctypes.c_void_p
        L.sip_get_stream.argtypes = [ctypes.c_void_p]
        L.sip_launch_count.restype = ctypes.c_longlong
        L.sip_launch_count.argtypes = [ctypes.c_void_p]
        L.sip_factor_count.restype = ctypes.c_longlong
        L.sip_factor_count.argtypes = [ctypes.c_void_p]
        for name in ("sip_destroy", "sip_synchronize"):
            getattr(L, name).argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


def _check(ctx, status: int, what: str):
    if status == SIP_OK:
        return
    msg = lib().sip_last_error(ctx).decode(errors="replace") if True else ""
    cls = _EXC.get(status, Error)
    raise cls(f"{what}: {lib().sip_status_string(status).decode()}: {msg}")


def _ptr(a: np.ndarray):
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise MisuseError("arrays must be C-contiguous float64 Field3 arrays")
    return a.ctypes.data_as(_dp)


def field(nx: int, ny: int, nz: int) -> np.ndarray:
    """Zero Field3 array (one ghost layer)."""
    return np.zeros((nz + 2, ny + 2, nx + 2), dtype=np.float64)


# ----------------------------------------------------------------- types
@dataclasses.dataclass
class StencilSystem:
    """Seven diagonals + source of one block, matrix-entry signs."""
    AP: np.ndarray
    AW: np.ndarray
    AE: np.ndarray
    AS: np.ndarray
    AN: np.ndarray
    AB: np.ndarray
    AT: np.ndarray
    Q: np.ndarray
    symmetric: bool = False

    @property
    def dims(self):
        nz, ny, nx = (s - 2 for s in self.AP.shape)
        return nx, ny, nz

    def arrays(self):
        return [getattr(self, n) for n in ARRAYS]

    @classmethod
    def from_dict(cls, d: dict, symmetric: bool = False) -> "StencilSystem":
        return cls(*(np.ascontiguousarray(d[n], dtype=np.float64) for n in ARRAYS),
                   symmetric=symmetric)


@dataclasses.dataclass
class SipConfig:
    """alpha in [0,1), max_iters >= 1, target reduction, precision."""
    alpha: float = 0.92
    max_iters: int = 50
    target: float = 0.0          # <= 0: fixed iteration count
    precision: str = "f64"       # "f64" | "f32" (single-precision relaxation)

    def validate(self):
        if not (0.0 <= self.alpha < 1.0):
            raise ConfigError("alpha must be in [0, 1)")
        if self.max_iters < 1:
            raise ConfigError("max_iters must be >= 1")
        if self.precision not in PREC:
            raise ConfigError(f"unknown precision {self.precision!r}")


@dataclasses.dataclass
class SolveReport:
    """SPEC.md:128-131."""
    iterations: int
    norms: np.ndarray
    factor_seconds: float = 0.0
    relax_seconds: float = 0.0

    @property
    def initial_norm(self):
        return float(self.norms[0]) if len(self.norms) else 0.0

    @property
    def final_norm(self):
        return float(self.norms[-1]) if len(self.norms) else 0.0


# ----------------------------------------------------------------- device context
class Solver:
    """One C-ABI context: a single block (dims) or a block lattice."""

    def __init__(self, dims=None, precision: str = "f64", device: int = 0, *, lattice=None,
                 block_rank: Optional[Sequence[int]] = None, rank: int = 0, nranks: int = 1,
                 nccl_id: Optional[bytes] = None):
        L = lib()
        self._ctx = ctypes.c_void_p()
        p = PREC[precision]
        self.precision = precision
        if lattice is None:
            nx, ny, nz = dims
            st = L.sip_create(device, nx, ny, nz, p, ctypes.byref(self._ctx))
        else:
            (gx, gy, gz), (px, py, pz) = lattice
            br = None
            if block_rank is not None:
                br = (ctypes.c_int * len(block_rank))(*block_rank)
            nid = None if nccl_id is None else ctypes.create_string_buffer(nccl_id, 128)
            st = L.sip_create_lattice(device, gx, gy, gz, px, py, pz, br, rank, nranks, nid, p,
                                      ctypes.byref(self._ctx))
        if st != SIP_OK:
            raise _EXC.get(st, Error)(
                f"sip_create: {L.sip_status_string(st).decode()}: {L.sip_last_error(None).decode()}")
        n = ctypes.c_int()
        L.sip_num_local_blocks(self._ctx, ctypes.byref(n))
        self.blocks = []
        for lb in range(n.value):
            bid = ctypes.c_int()
            d = (ctypes.c_int * 3)()
            o = (ctypes.c_int * 3)()
            L.sip_local_block(self._ctx, lb, ctypes.byref(bid), d, o)
            self.blocks.append((bid.value, tuple(d), tuple(o)))

    # -- plumbing
    @property
    def handle(self):
        return self._ctx

    def close(self):
        for fl in list(getattr(self, "_flows", ())):  # flows live on this context: free them first
            fl.close()
        if self._ctx:
            lib().sip_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, st, what):
        _check(self._ctx, st, what)

    # -- system / factor
    def set_system(self, local: int, A: StencilSystem):
        self._c(lib().sip_set_system(self._ctx, local, *[_ptr(a) for a in A.arrays()]),
                "sip_set_system")

    def set_symmetric(self, local: int, symmetric: bool = True):
        """Flag the system of a local block symmetric (checked on the device)."""
        self._c(lib().sip_set_symmetric(self._ctx, local, int(symmetric)), "sip_set_symmetric")

    def set_halo_tables(self, tables):
        """Drive the face-halo exchange by an FTT1 table set (ftt1_read output:
        one (n, 12) int array per rank), e.g. periodic decompositions."""
        counts, flat = _tables_flat(tables)
        self._c(lib().sip_set_halo_tables(self._ctx, len(tables), counts, flat),
                "sip_set_halo_tables")

    def set_source(self, local: int, q: np.ndarray):
        self._c(lib().sip_set_source(self._ctx, local, _ptr(q)), "sip_set_source")

    def set_source_async(self, local: int, q: np.ndarray):
        """sip_set_source_async: q is copied on the copy stream (keep it alive
        and unchanged until the next synchronize; pinned memory overlaps)."""
        self._keep = getattr(self, "_keep", []) + [q]
        self._c(lib().sip_set_source_async(self._ctx, local, _ptr(q)), "sip_set_source_async")

    def solve_async(self, phis: Sequence[np.ndarray], iters: int, norms: np.ndarray):
        """sip_solve_async: fixed iteration count, no host synchronisation;
        phis and norms[iters] are complete after synchronize()."""
        self._keep = getattr(self, "_keep", []) + [phis, norms]
        self._c(lib().sip_solve_async(self._ctx, self._phis(phis), int(iters), norms.ctypes.data_as(_dp)),
                "sip_solve_async")

    def wait_async(self):
        """sip_wait_async: the oldest pending solve_async is complete."""
        self._c(lib().sip_wait_async(self._ctx), "sip_wait_async")

    def generate(self, kind: int, seed: int):
        self._c(lib().sip_generate_system(self._ctx, kind, ctypes.c_uint64(seed)),
                "sip_generate_system")

    def assemble_poisson(self, lengths, bc=("wall",) * 6):
        """assemble_poisson: 7-point pressure Laplacian of the
        lattice over a domain of `lengths` (lx, ly, lz); bc per face W,E,S,N,B,T
        ("wall" | "periodic" | "symmetry").  Global cell (0,0,0) is pinned."""
        codes = [BC[b] if isinstance(b, str) else int(b) for b in bc]
        if len(codes) != 6:
            raise ConfigError("assemble_poisson: bc needs 6 faces (W,E,S,N,B,T)")
        self._c(lib().sip_assemble_poisson(self._ctx, (ctypes.c_double * 3)(*lengths),
                                           (ctypes.c_int * 6)(*codes)), "sip_assemble_poisson")

    def factor(self, alpha: float):
        global _factor_count
        _factor_count += 1
        bb, bc = ctypes.c_longlong(-1), ctypes.c_longlong(-1)
        st = lib().sip_factor(self._ctx, ctypes.c_double(alpha), ctypes.byref(bb), ctypes.byref(bc))
        if st == SIP_ERR_SINGULAR:
            raise SingularFactorError(
                f"singular factorization at block {bb.value}, Field3 index {bc.value}")
        self._c(st, "sip_factor")

    # -- relaxation
    def _phis(self, phis):
        arr = (_dp * len(phis))(*[_ptr(p) for p in phis])
        return arr

    def solve(self, phis: Sequence[np.ndarray], max_iters: int, target: float = 0.0,
              check_every: Optional[int] = None):
        """solve; check_every: norm-evaluation interval of the
        target mode (None: sip_solve's default)."""
        norms = np.zeros(max(max_iters, 1))
        used = ctypes.c_int(0)
        if check_every is None:
            st = lib().sip_solve(self._ctx, self._phis(phis), max_iters, ctypes.c_double(target),
                                 norms.ctypes.data_as(_dp), ctypes.byref(used))
        else:
            st = lib().sip_solve_ex(self._ctx, self._phis(phis), max_iters, ctypes.c_double(target),
                                    int(check_every), norms.ctypes.data_as(_dp), ctypes.byref(used))
        self._c(st, "sip_solve")
        return norms[:used.value]

    def load_phi(self, phis):
        self._c(lib().sip_load_phi(self._ctx, self._phis(phis)), "sip_load_phi")

    def store_phi(self, phis):
        self._c(lib().sip_store_phi(self._ctx, self._phis(phis)), "sip_store_phi")

    def iterate(self, iters: int):
        self._c(lib().sip_iterate(self._ctx, iters), "sip_iterate")

    def read_norms(self, first: int, count: int, per_block: bool = False):
        n = np.zeros(max(count, 1))
        nb = self.num_global_blocks() if per_block else 0
        bn = np.zeros((max(count, 1), max(nb, 1)))
        self._c(lib().sip_read_norms(self._ctx, first, count, n.ctypes.data_as(_dp),
                                     bn.ctypes.data_as(_dp) if per_block else None),
                "sip_read_norms")
        return (n[:count], bn[:count]) if per_block else n[:count]

    def num_global_blocks(self) -> int:
        """Blocks of the whole lattice (all ranks): the width of read_norms' per-block rows."""
        n = ctypes.c_int()
        self._c(lib().sip_num_global_blocks(self._ctx, ctypes.byref(n)), "sip_num_global_blocks")
        return n.value

    def factor_count(self) -> int:
        """Library-side factorisation counter: K1 launches of this context."""
        return int(lib().sip_factor_count(self._ctx))

    def synchronize(self):
        self._c(lib().sip_synchronize(self._ctx), "sip_synchronize")
        self._keep = []

    def residual(self, symmetric: bool = False):
        outs = [field(*d) for (_, d, _) in self.blocks]
        self._c(lib().sip_residual(self._ctx, int(symmetric), self._phis(outs)), "sip_residual")
        return outs

    # -- measurement helpers
    def set_stream(self, stream_ptr: int):
        self._c(lib().sip_set_stream(self._ctx, ctypes.c_void_p(stream_ptr)), "sip_set_stream")

    def set_profiling(self, on: bool):
        self._c(lib().sip_set_profiling(self._ctx, int(on)), "sip_set_profiling")

    def profile(self):
        f, b, h = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        n = ctypes.c_longlong()
        self._c(lib().sip_get_profile(self._ctx, ctypes.byref(f), ctypes.byref(b), ctypes.byref(h),
                                      ctypes.byref(n)), "sip_get_profile")
        return {"fwd_ms": f.value, "bwd_ms": b.value, "halo_ms": h.value, "launches": n.value}

    def launch_count(self) -> int:
        return int(lib().sip_launch_count(self._ctx))

    def geometry(self):
        ti, tj = ctypes.c_int(), ctypes.c_int()
        nt, ns = ctypes.c_longlong(), ctypes.c_longlong()
        lib().sip_geometry(self._ctx, ctypes.byref(ti), ctypes.byref(tj), ctypes.byref(nt),
                           ctypes.byref(ns))
        return {"brick_i": ti.value, "brick_j": tj.value, "bricks": nt.value, "slices": ns.value}


# ----------------------------------------------------------------- SPEC operations
class Flow:
    """FlowState of a Solver whose system was assembled by
    assemble_poisson: u, v, w, p as fp64 Field3 arrays per local block, kept in
    device memory; set / get copy host arrays in and out."""

    def __init__(self, solver: "Solver"):
        import weakref
        self.solver = solver
        self._h = ctypes.c_void_p()
        _check(solver.handle, lib().sip_flow_create(solver.handle, ctypes.byref(self._h)),
               "sip_flow_create")
        if not hasattr(solver, "_flows"):
            solver._flows = weakref.WeakSet()
        solver._flows.add(self)

    def close(self):
        if self._h:
            lib().sip_flow_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _c(self, st, what):
        if st == SIP_ERR_NOCONV:
            raise NonConvergenceError(
                f"{what}: {lib().sip_last_error(self.solver.handle).decode(errors='replace')}")
        _check(self.solver.handle, st, what)

    def set(self, name: str, arrays: Sequence[np.ndarray]):
        self._c(lib().sip_flow_set(self._h, FLOW_FIELDS[name], self.solver._phis(arrays)),
                "sip_flow_set")

    def get(self, name: str, arrays: Sequence[np.ndarray]):
        self._c(lib().sip_flow_get(self._h, FLOW_FIELDS[name], self.solver._phis(arrays)),
                "sip_flow_get")

    def divergence(self) -> float:
        """L1 of the co-located central divergence, sum |div u| * cell volume."""
        d = ctypes.c_double()
        self._c(lib().sip_flow_divergence(self._h, ctypes.byref(d)), "sip_flow_divergence")
        return d.value

    def pressure_correct(self, dt: float, threshold: float, max_outer: int = 20,
                         sweeps: int = 5):
        """pressure_correct with the factors of the assembled
        system reused.  Returns (outer iterations, divergence L1 history);
        raises NonConvergenceError (with .defect) at the outer cap."""
        hist = np.zeros(max_outer + 1)
        used = ctypes.c_int(0)
        st = lib().sip_pressure_correct(self._h, ctypes.c_double(dt), ctypes.c_double(threshold),
                                        max_outer, sweeps, ctypes.byref(used),
                                        hist.ctypes.data_as(_dp))
        if st == SIP_ERR_NOCONV:
            raise NonConvergenceError(
                lib().sip_last_error(self.solver.handle).decode(errors="replace"),
                float(hist[used.value]))
        self._c(st, "sip_pressure_correct")
        return used.value, hist[:used.value + 1]


def assemble_poisson(solver: "Solver", lengths, bc=("wall",) * 6, dt: Optional[float] = None):
    """SPEC.md:134-142 (dt does not enter the coefficients; kept for the signature)."""
    solver.assemble_poisson(lengths, bc)
    return solver


def pressure_correct(flow: Flow, dt: float, threshold: float, max_outer: int = 20,
                     sweeps: int = 5):
    """see Flow.pressure_correct."""
    return flow.pressure_correct(dt, threshold, max_outer, sweeps)


class SipFactors:
    """Factors of one StencilSystem, resident on the device and stamped with
    the system revision they were computed from."""

    def __init__(self, solver: Solver, system: StencilSystem, alpha: float, revision: int):
        self.solver = solver
        self.system = system
        self.alpha = alpha
        self.revision = revision
        self.precision = solver.precision


_factor_count = 0


def factorization_count() -> int:
    """Number of sip_factor calls made through this module (work-avoidance check)."""
    return _factor_count


def sip_factor(A: StencilSystem, cfg: SipConfig, device: int = 0) -> SipFactors:
    """SPEC.md:143-151.  Raises SingularFactorError naming the cell."""
    global _factor_count
    cfg.validate()
    s = Solver(A.dims, cfg.precision, device)
    s.set_system(0, A)
    s.factor(cfg.alpha)
    _factor_count += 1
    return SipFactors(s, A, cfg.alpha, _revision(A))


def _revision(A: StencilSystem) -> int:
    # content stamp of the coefficient arrays (the source Q may change freely)
    h = 0
    for a in A.arrays()[:7]:
        h = hash((h, a.tobytes()[:4096], a.sum()))
    return h


def residual_general(A: StencilSystem, fi: np.ndarray, device: int = 0) -> np.ndarray:
    """res = sum a_nb*fi_nb + su - ap*fi at interior cells."""
    s = Solver(A.dims, "f64", device)
    s.set_system(0, A)
    s.load_phi([np.ascontiguousarray(fi, dtype=np.float64)])
    return s.residual()[0]


def residual_symmetric(A: StencilSystem, fi: np.ndarray, device: int = 0) -> np.ndarray:
    """SPEC.md:161-169 / Listing 1: the residual reading only ae, an, at
    (+ shifted), ap and su.  MisuseError unless A is flagged symmetric;
    ConfigError if the flag contradicts the coefficients."""
    if not A.symmetric:
        raise MisuseError("residual_symmetric: system not flagged symmetric")
    s = Solver(A.dims, "f64", device)
    s.set_system(0, A)
    s.set_symmetric(0, True)
    s.load_phi([np.ascontiguousarray(fi, dtype=np.float64)])
    return s.residual(symmetric=True)[0]


def sip_sweep(A: StencilSystem, F: SipFactors, fi: np.ndarray) -> float:
    """one iteration in place on fi; returns the L1 norm."""
    if _revision(A) != F.revision:
        raise StaleFactorsError("factors were computed from a different system revision")
    s = F.solver
    s.set_source(0, A.Q)
    norms = s.solve([fi], 1, 0.0)
    return float(norms[0])


def solve(A: StencilSystem, fi0: np.ndarray, cfg: SipConfig, F: Optional[SipFactors] = None):
    """SPEC.md:179-187.  Returns (fi, SolveReport); factorises at most once
    (zero times on the reuse path, when F is given and its stamp matches)."""
    cfg.validate()
    fi = np.array(fi0, dtype=np.float64, copy=True, order="C")
    t0 = time.perf_counter()
    if F is None:
        F = sip_factor(A, cfg)
    elif _revision(A) != F.revision:
        raise StaleFactorsError("factors were computed from a different system revision")
    elif F.precision != cfg.precision:
        raise MisuseError("factors were computed for another precision")
    t1 = time.perf_counter()
    if cfg.target >= 1.0:
        return fi, SolveReport(0, np.zeros(0), t1 - t0, 0.0)
    F.solver.set_source(0, A.Q)
    norms = F.solver.solve([fi], cfg.max_iters, cfg.target)
    t2 = time.perf_counter()
    return fi, SolveReport(len(norms), norms, t1 - t0, t2 - t1)


def version() -> str:
    return lib().sip_version().decode()


# ----------------------------------------------------------------- FTT1 tables
def _tables_flat(tables):
    counts = (ctypes.c_int * max(1, len(tables)))(*[len(t) for t in tables])
    rows = [np.asarray(t, dtype=np.int32).reshape(-1, 12) for t in tables]
    flat = np.ascontiguousarray(np.concatenate(rows) if rows else np.zeros((0, 12), np.int32),
                                dtype=np.int32)
    return counts, flat.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def ftt1_read(data: bytes):
    """FTT1 image -> per-rank (n, 12) int arrays (tables.cpp:140-183 semantics;
    FormatError with the reference's message and byte offset)."""
    buf = ctypes.create_string_buffer(bytes(data), len(data))
    nranks, total, off = ctypes.c_int(0), ctypes.c_longlong(0), ctypes.c_longlong(-1)
    st = lib().sip_ftt1_read(buf, ctypes.c_size_t(len(data)), ctypes.byref(nranks), None, None,
                             ctypes.c_longlong(0), ctypes.byref(total), ctypes.byref(off))
    if st == SIP_ERR_FORMAT:
        raise FormatError(lib().sip_last_error(None).decode(), off.value)
    _check(None, st, "sip_ftt1_read")
    counts = (ctypes.c_int * max(1, nranks.value))()
    ent = np.zeros((max(1, total.value), 12), dtype=np.int32)
    st = lib().sip_ftt1_read(buf, ctypes.c_size_t(len(data)), ctypes.byref(nranks), counts,
                             ent.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                             ctypes.c_longlong(total.value), ctypes.byref(total), ctypes.byref(off))
    _check(None, st, "sip_ftt1_read")
    out, at = [], 0
    for r in range(nranks.value):
        out.append(ent[at:at + counts[r]].copy())
        at += counts[r]
    return out


def ftt1_write(tables) -> bytes:
    counts, flat = _tables_flat(tables)
    n = ctypes.c_size_t(0)
    _check(None, lib().sip_ftt1_write(len(tables), counts, flat, None, ctypes.c_size_t(0),
                                      ctypes.byref(n)), "sip_ftt1_write")
    buf = ctypes.create_string_buffer(n.value)
    _check(None, lib().sip_ftt1_write(len(tables), counts, flat, buf, n, ctypes.byref(n)),
           "sip_ftt1_write")
    return buf.raw[: n.value]


def ftt1_validate(tables) -> None:
    """Send/recv matching (tables.cpp:185-235); ProtocolError on a violation."""
    counts, flat = _tables_flat(tables)
    st = lib().sip_ftt1_validate(len(tables), counts, flat)
    if st == SIP_ERR_PROTOCOL:
        raise ProtocolError(lib().sip_last_error(None).decode())
    _check(None, st, "sip_ftt1_validate")
