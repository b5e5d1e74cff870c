"""Independent pure-Python restatement of SIP, used only to cross-check the C
oracle (oracle/sip_oracle.c) on small grids.  TEST INFRASTRUCTURE ONLY.

Written directly from the normative text (SPEC.md:146, SPEC.md:155,
SPEC.md:173) with the sign mapping a_nb = -A_nb,
using Python floats (IEEE binary64, no contraction) and, for the fp32 path,
numpy float32 scalars.  Loop order is SPEC's "j fastest, then i, then k"
(SPEC.md design decision, Listing 1) -- deliberately different from the C
oracle's i-fastest order: any topological order gives identical values.
"""
from __future__ import annotations

import numpy as np


def _get(a, i, j, k):
    return a[k, j, i]


def factor(A, alpha):
    nz, ny, nx = (s - 2 for s in A["AP"].shape)
    F = {n: np.zeros_like(A["AP"]) for n in ("LB", "LW", "LS", "LP", "UN", "UE", "UT")}
    UN, UE, UT = F["UN"], F["UE"], F["UT"]
    for k in range(1, nz + 1):
        for i in range(1, nx + 1):
            for j in range(1, ny + 1):
                unb, ueb, utb = float(UN[k - 1, j, i]), float(UE[k - 1, j, i]), float(UT[k - 1, j, i])
                unw, uew, utw = float(UN[k, j, i - 1]), float(UE[k, j, i - 1]), float(UT[k, j, i - 1])
                uns, ues, uts = float(UN[k, j - 1, i]), float(UE[k, j - 1, i]), float(UT[k, j - 1, i])
                lb = float(A["AB"][k, j, i]) / (1.0 + alpha * (unb + ueb))
                lw = float(A["AW"][k, j, i]) / (1.0 + alpha * (unw + utw))
                ls = float(A["AS"][k, j, i]) / (1.0 + alpha * (ues + uts))
                p1 = alpha * (lb * unb + lw * unw)
                p2 = alpha * (lb * ueb + ls * ues)
                p3 = alpha * (lw * utw + ls * uts)
                den = float(A["AP"][k, j, i]) + p1 + p2 + p3 - lb * utb - lw * uew - ls * uns
                if not abs(den) >= 1e-30:
                    raise ValueError(f"singular at {(i, j, k)}")
                lp = 1.0 / den
                F["LB"][k, j, i], F["LW"][k, j, i], F["LS"][k, j, i], F["LP"][k, j, i] = lb, lw, ls, lp
                UN[k, j, i] = (float(A["AN"][k, j, i]) - p1) * lp
                UE[k, j, i] = (float(A["AE"][k, j, i]) - p2) * lp
                UT[k, j, i] = (float(A["AT"][k, j, i]) - p3) * lp
    return F


def sweep(A, F, phi):
    """One SIP iteration in place; dtype of phi selects fp64 / fp32 arithmetic.
    In fp32 mode A and F must already be float32 arrays."""
    nz, ny, nx = (s - 2 for s in A["AP"].shape)
    T = phi.dtype.type
    w = np.zeros_like(phi)
    norm = 0.0
    for k in range(1, nz + 1):
        for i in range(1, nx + 1):
            for j in range(1, ny + 1):
                c = (k, j, i)
                r = -(A["AE"][c] * phi[k, j, i + 1])
                r = T(r - A["AW"][c] * phi[k, j, i - 1])
                r = T(r - A["AN"][c] * phi[k, j + 1, i])
                r = T(r - A["AS"][c] * phi[k, j - 1, i])
                r = T(r - A["AT"][c] * phi[k + 1, j, i])
                r = T(r - A["AB"][c] * phi[k - 1, j, i])
                r = T(r + A["Q"][c])
                r = T(r - A["AP"][c] * phi[c])
                norm += abs(float(r))
                t = T(r - F["LB"][c] * w[k - 1, j, i])
                t = T(t - F["LW"][c] * w[k, j, i - 1])
                t = T(t - F["LS"][c] * w[k, j - 1, i])
                w[c] = T(t * F["LP"][c])
    for k in range(nz, 0, -1):
        for i in range(nx, 0, -1):
            for j in range(ny, 0, -1):
                c = (k, j, i)
                d = T(w[c] - F["UN"][c] * w[k, j + 1, i])
                d = T(d - F["UE"][c] * w[k, j, i + 1])
                d = T(d - F["UT"][c] * w[k + 1, j, i])
                w[c] = d
                phi[c] = T(phi[c] + d)
    return norm
