"""Philox4x32-10 and the Brownian-increment map of the oracle (TEST INFRASTRUCTURE ONLY).

P:64 (Eq. 5, "ΔW_n ~ N(0, Δt_n)") asks for Gaussian increments; the paper does
not say how they are drawn.  Reading R8: a counter-based
Philox4x32-10 generator (Salmon et al., SC'11) keyed by the seed, with counter
(q = j // 4, m = global path, n = time step, it = global iteration), and a
Box-Muller map of each 4 x uint32 block to 4 standard normals.

This is a plain vectorised numpy transcription of the published algorithm:
10 rounds of   (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0))
with the Weyl key bump (k0 += W0, k1 += W1) between rounds.
"""
import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)

# Counter word c3 reserved values (R8 / R7): training uses the global iteration
# (< 2^31); evaluation streams set the top bit; the initialisation stream uses
# 0xC0000000.
EVAL_BIT = 0x80000000
INIT_STREAM = 0xC0000000


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 on broadcastable uint32 arrays; returns 4 uint32 arrays."""
    c0 = np.asarray(c0, dtype=np.uint64) & MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & MASK32
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for r in range(10):
        if r:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c0                      # < 2^64, exact in uint64
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1,
                          hi0 ^ c3 ^ np.uint64(k1), lo0)
    return tuple(x.astype(np.uint32) for x in (c0, c1, c2, c3))


def seed_key(seed):
    """key = (seed mod 2^32, seed >> 32) (R8)."""
    seed = int(seed)
    return seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF


def uint_to_unit(x):
    """u = ((x >> 9) + 0.5) * 2^-23 in (0, 1) (R8, exact in fp32 and fp64)."""
    x = np.asarray(x, dtype=np.uint32)
    return ((x >> np.uint32(9)).astype(np.float64) + 0.5) * 2.0 ** -23


def box_muller(u1, u2):
    """(r cos 2πu2, r sin 2πu2), r = sqrt(-2 ln u1): two N(0,1) draws (R8)."""
    r = np.sqrt(-2.0 * np.log(u1))
    a = 2.0 * np.pi * u2
    return r * np.cos(a), r * np.sin(a)


def standard_normals(seed, it, n, m, d):
    """z[i, j] ~ N(0,1) for global path m[i], step n, component j < d (R8).

    Normal 4q+0/4q+1 come from outputs (x0, x1) of block q, 4q+2/4q+3 from
    (x2, x3).  Shape [len(m), d], float64.
    """
    m = np.asarray(m, dtype=np.uint64).reshape(-1, 1)
    nq = (d + 3) // 4
    q = np.arange(nq, dtype=np.uint64).reshape(1, -1)
    k0, k1 = seed_key(seed)
    x0, x1, x2, x3 = philox4x32_10(q, m, np.uint64(n), np.uint64(it), k0, k1)
    za, zb = box_muller(uint_to_unit(x0), uint_to_unit(x1))
    zc, zd = box_muller(uint_to_unit(x2), uint_to_unit(x3))
    z = np.stack([za, zb, zc, zd], axis=-1).reshape(m.shape[0], 4 * nq)
    return z[:, :d]


def brownian_increments(seed, it, n, m, d, dt):
    """ΔW_n^m = sqrt(Δt) z  (Eq. 5)."""
    return np.sqrt(dt) * standard_normals(seed, it, n, m, d)


def coupled_increments(seed, it, n, m, d, dt, factor):
    """Coupled multilevel paths ("coarsen_increments",
    PAPER.md §3.2 fig:multilevel: the levels simulate the same underlying path): the
    increment of coarse step n (Δt = T/N) is the sum of the `factor` increments of the
    finest grid (Δt/factor) that it spans, fine steps n·factor .. n·factor + factor - 1,
    each drawn with its own fine step index in the counter (R8).  factor = 1 is
    brownian_increments."""
    if factor < 1:
        raise ValueError("factor must be >= 1")
    acc = np.zeros((len(np.atleast_1d(m)), d))
    for j in range(factor):
        acc = acc + brownian_increments(seed, it, n * factor + j, m, d, dt / factor)
    return acc


def init_uniforms(seed, tensor_id, count):
    """Uniforms of the initialisation stream (R7): ctr = (idx//4, tensor_id, 0, INIT_STREAM)."""
    idx = np.arange(count, dtype=np.uint64)
    k0, k1 = seed_key(seed)
    outs = philox4x32_10(idx // np.uint64(4), np.uint64(tensor_id), np.uint64(0),
                         np.uint64(INIT_STREAM), k0, k1)
    sel = (idx % np.uint64(4)).astype(np.int64)
    x = np.choose(sel, outs)
    return uint_to_unit(x)
