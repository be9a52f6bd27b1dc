"""O1: the GCN propagation values P_vu (TEST INFRASTRUCTURE ONLY, see oracle/__init__).

P is "the propagation matrix following the definition of GCN" (§3.1 after
Eq. 5; appendix Preliminaries).  Reading A1: Kipf's
P = D~^{-1/2} (A + I) D~^{-1/2} with unit edge weights and GLOBAL degrees
(S:42), so that P_in + P_out = P_m holds.
Reading A2 (rounding, paper silent): each stored value is
    P_vu = fp32( 1 / sqrt( double(deg v + 1) * double(deg u + 1) ) )
with IEEE round-to-nearest double multiply, sqrt and divide, then one rounding
to fp32.
"""
import numpy as np


def degrees(indptr: np.ndarray) -> np.ndarray:
    """deg(v) = number of stored neighbours of v (raw adjacency, no self loop)."""
    return np.diff(np.asarray(indptr, dtype=np.int64))


def prop_values(deg_v, deg_u) -> np.ndarray:
    """P_vu for arrays of (deg v, deg u) pairs, as fp32 (reading A2)."""
    dv = np.asarray(deg_v, dtype=np.float64) + 1.0
    du = np.asarray(deg_u, dtype=np.float64) + 1.0
    return (1.0 / np.sqrt(dv * du)).astype(np.float32)
