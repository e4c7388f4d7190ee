"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the engine's QMC mode
(the north_star's Sobol + AS241 + Brownian bridge).  The reference has no
QMC: parity for this mode is pinned to third-party
references instead -- Sobol integers to scipy.stats.qmc.Sobol(scramble=False,
bits=32) (Joe-Kuo new-joe-kuo-6.21201 direction numbers), AS241 to
scipy.special.ndtri -- and the bridge to its covariance min(s, t).
"""
from __future__ import annotations

import numpy as np

# Wichura (1988), Algorithm AS 241 "PPND16", Appl. Statist. 37(3):477-484.
A = [3.3871328727963666080e0, 1.3314166789178437745e+2, 1.9715909503065514427e+3,
     1.3731693765509461125e+4, 4.5921953931549871457e+4, 6.7265770927008700853e+4,
     3.3430575583588128105e+4, 2.5090809287301226727e+3]
B = [1.0, 4.2313330701600911252e+1, 6.8718700749205790830e+2, 5.3941960214247511077e+3,
     2.1213794301586595867e+4, 3.9307895800092710610e+4, 2.8729085735721942674e+4,
     5.2264952788528545610e+3]
C = [1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0,
     3.64784832476320460504e0, 1.27045825245236838258e0, 2.41780725177450611770e-1,
     2.27238449892691845833e-2, 7.74545014278341407640e-4]
D = [1.0, 2.05319162663775882187e0, 1.67638483018380384940e0, 6.89767334985100004550e-1,
     1.48103976427480074590e-1, 1.51986665636164571966e-2, 5.47593808499534494600e-4,
     1.05075007164441684324e-9]
E_ = [6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0,
      2.96560571828504891230e-1, 2.65321895265761230930e-2, 1.24266094738807843860e-3,
      2.71155556874348757815e-5, 2.01033439929228813265e-7]
F = [1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1, 1.48753612908506148525e-2,
     7.86869131145613259100e-4, 1.84631831751005468180e-5, 1.42151175831644588870e-7,
     2.04426310338993978564e-15]


def _poly(c, x):
    r = np.zeros_like(x) + c[7]
    for k in range(6, -1, -1):
        r = r * x + c[k]
    return r


def as241(p):
    p = np.asarray(p, dtype=np.float64)
    q = p - 0.5
    out = np.empty_like(p)
    cen = np.abs(q) <= 0.425
    r = 0.180625 - q[cen] * q[cen]
    out[cen] = q[cen] * _poly(A, r) / _poly(B, r)
    t = ~cen
    r = np.where(q[t] < 0, p[t], 1.0 - p[t])
    r = np.sqrt(-np.log(r))
    near = r <= 5.0
    v = np.where(near, _poly(C, r - 1.6) / _poly(D, r - 1.6), _poly(E_, r - 5.0) / _poly(F, r - 5.0))
    out[t] = np.where(q[t] < 0, -v, v)
    return out


# ---- Sobol (gray-code form over the engine's shipped direction numbers) ----
def load_direction_numbers(path: str) -> np.ndarray:
    """Parse csrc/sobol_table.cpp (generated) into v[d][k]."""
    import re
    txt = open(path).read()
    body = txt[txt.index("kSobolV"):]
    vals = [int(x, 16) for x in re.findall(r"0x[0-9a-f]{8}", body)]
    v = np.array(vals, dtype=np.uint32)
    return v.reshape(-1, 32)


def sobol_int(v: np.ndarray, dims, n: np.ndarray) -> np.ndarray:
    """x[len(n)][len(dims)]: point n, dimension d = XOR of v[d][k] over set bits k of gray(n)."""
    n = np.asarray(n, dtype=np.uint64)
    g = n ^ (n >> np.uint64(1))
    dims = np.asarray(dims)
    x = np.zeros((len(n), len(dims)), dtype=np.uint32)
    for k in range(32):
        bit = ((g >> np.uint64(k)) & np.uint64(1)).astype(bool)
        x[bit] ^= v[dims, k][None, :].repeat(bit.sum(), axis=0)
    return x


# ---- Brownian bridge, built directly (breadth-first node numbering) --------
def bridge_nodes(nD: int):
    """node[m], left[m], right[m] for grid indices m in [0, nD); -1 = origin."""
    node = [-1] * nD
    L = [-2] * nD
    R = [-2] * nD
    node[nD - 1] = 0
    nxt = 1
    q = [(-1, nD - 1)]
    h = 0
    while h < len(q):
        l, r = q[h]
        h += 1
        if r - l < 2:
            continue
        m = l + (r - l) // 2
        node[m], L[m], R[m] = nxt, l, r
        nxt += 1
        q += [(l, m), (m, r)]
    return node, L, R


def bridge_paths(tau: np.ndarray, Z: np.ndarray) -> np.ndarray:
    """W[K][nD][nA] from Z[K][nD nodes][nA] (node-indexed normals)."""
    nD = len(tau)
    node, L, R = bridge_nodes(nD)
    T = lambda i: 0.0 if i < 0 else tau[i]
    W = np.zeros((Z.shape[0], nD, Z.shape[2]))
    W[:, nD - 1] = np.sqrt(tau[nD - 1]) * Z[:, 0]
    # parents are always built before children in BFS node order
    order = sorted(range(nD - 1), key=lambda m: node[m])
    for m in order:
        l, r = L[m], R[m]
        tl, tr, tm = T(l), T(r), T(m)
        Wl = 0.0 if l < 0 else W[:, l]
        W[:, m] = ((tr - tm) * Wl + (tm - tl) * W[:, r]) / (tr - tl) \
            + np.sqrt((tm - tl) * (tr - tm) / (tr - tl)) * Z[:, node[m]]
    return W
