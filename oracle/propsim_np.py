"""numpy restatement of the reference's hot-path arithmetic (TEST ORACLE ONLY).

Each function cites the reference code it restates (paths relative to
/root/reference/pkg/src/propsim). Summation order is the reference's:
every output element is a sequential ascending-q fold from +0 in the run
dtype (mingemm.py:79-91), realised here as a Python loop over q of
whole-matrix numpy adds -- the same scalar add sequence per element, so
results are bitwise those of the reference on any NaN-free input.
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)


def mix64(x):
    """verify.py:36-55 (scalar and vectorised)."""
    a = np.asarray(x, dtype=np.uint64).copy()
    with np.errstate(over="ignore"):
        a ^= a >> np.uint64(30)
        a *= C1
        a ^= a >> np.uint64(27)
        a *= C2
        a ^= a >> np.uint64(31)
    return a


def random_exact(seed: int, n_f: int, n_v: int, bits: int, dtype=np.float64,
                 f0: int = 0, f1: int | None = None, v0: int = 0, v1: int | None = None):
    """SyntheticSpec.local_block, random-exact (verify.py:131-147): (n_f, n_v) Fortran."""
    f1 = n_f if f1 is None else f1
    v1 = n_v if v1 is None else v1
    q = np.arange(f0, f1, dtype=np.uint64)[:, None]
    i = np.arange(v0, v1, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        h = mix64((q * np.uint64(n_v) + i) ^ np.uint64(seed & MASK64))
    return np.asfortranarray((h & np.uint64((1 << bits) - 1)).astype(dtype))


def random_exact_cols(seed: int, n_f: int, n_v: int, bits: int, cols, dtype=np.float64):
    """Selected global columns of the random-exact matrix (sampled parity)."""
    q = np.arange(n_f, dtype=np.uint64)[:, None]
    i = np.asarray(cols, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        h = mix64((q * np.uint64(n_v) + i) ^ np.uint64(seed & MASK64))
    return np.asfortranarray((h & np.uint64((1 << bits) - 1)).astype(dtype))


def analytic(n_f: int, n_v: int, dtype=np.float64):
    """SyntheticSpec.local_block, analytic: 1 + [q mod n_v == i] (verify.py:143-145)."""
    q = np.arange(n_f, dtype=np.uint64)[:, None]
    i = np.arange(n_v, dtype=np.uint64)[None, :]
    return np.asfortranarray(((q % np.uint64(n_v) == i).astype(np.uint64) + 1).astype(dtype))


def uniform(seed: int, n_f: int, n_v: int, dtype=np.float64):
    """General-FP input of SURVEY 8d: (mix64(seed^(q*n_v+i)) >> 11) * 2^-53 (FP64),
    (>> 40) * 2^-24 (FP32). Mirrors psim_gen_uniform."""
    q = np.arange(n_f, dtype=np.uint64)[:, None]
    i = np.arange(n_v, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        h = mix64((q * np.uint64(n_v) + i) ^ np.uint64(seed & MASK64))
    if np.dtype(dtype) == np.float64:
        return np.asfortranarray((h >> np.uint64(11)).astype(np.float64) * 2.0**-53)
    return np.asfortranarray((h >> np.uint64(40)).astype(np.float32) * np.float32(2.0**-24))


def column_sums(V):
    """_colsum_kernel (mingemm.py:120-127): sequential ascending q from +0."""
    V = np.asarray(V)
    acc = np.zeros(V.shape[1], dtype=V.dtype)
    for q in range(V.shape[0]):
        acc = acc + V[q]
    return acc


def mgemm(W, V):
    """_naive_kernel (mingemm.py:79-91): M[i,j] = sum_q (w if w < v else v), ascending q."""
    W, V = np.asarray(W), np.asarray(V)
    M = np.zeros((W.shape[1], V.shape[1]), dtype=W.dtype)
    for q in range(W.shape[0]):
        w = W[q][:, None]
        v = V[q][None, :]
        M = M + np.where(w < v, w, v)
    return M


def triple_min(V):
    """_triple_num_kernel (mingemm.py:146-162) as a dense cube T[i,j,k]."""
    V = np.asarray(V)
    n = V.shape[1]
    T = np.zeros((n, n, n), dtype=V.dtype)
    for q in range(V.shape[0]):
        a = V[q][:, None, None]
        b = V[q][None, :, None]
        c = V[q][None, None, :]
        ab = np.where(a < b, a, b)
        T = T + np.where(ab < c, ab, c)
    return T


def values_2way(V):
    """All pair values in canonical order + degenerate mask (oracle_2way, verify.py:216-237;
    expression metrics2.py:77-89)."""
    V = np.asarray(V)
    dt = V.dtype.type
    N = mgemm(V, V)
    s = column_sums(V)
    iu, ju = np.triu_indices(V.shape[1], k=1)
    d = s[iu] + s[ju]
    zero = d == 0
    vals = (dt(2) * N[iu, ju]) / np.where(zero, dt(1), d)
    return np.where(zero, dt(0), vals).astype(V.dtype), zero


def triple_ids(n: int):
    """Canonical (lexicographic) i<j<k id arrays."""
    ii, jj, kk = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    m = (ii < jj) & (jj < kk)
    return ii[m], jj[m], kk[m]


def values_3way(V):
    """All triple values in canonical order + degenerate mask (oracle_3way,
    verify.py:240-272; expression metrics3.py:38-44)."""
    V = np.asarray(V)
    dt = V.dtype.type
    N = mgemm(V, V)
    T = triple_min(V)
    s = column_sums(V)
    i, j, k = triple_ids(V.shape[1])
    n3 = ((N[i, j] + N[i, k]) + N[j, k]) - T[i, j, k]
    d = (s[i] + s[j]) + s[k]
    zero = d == 0
    vals = (dt(1.5) * n3) / np.where(zero, dt(1), d)
    return np.where(zero, dt(0), vals).astype(V.dtype), zero


def value_bits(vals):
    """verify.py:58-65: FP32 zero-extended to 64 bits."""
    vals = np.asarray(vals)
    if vals.dtype == np.float32:
        return vals.view(np.uint32).astype(np.uint64)
    return vals.view(np.uint64)


def _sum_u64(x) -> int:
    x = np.asarray(x, dtype=np.uint64)
    return int(np.sum(x & np.uint64(0xFFFFFFFF), dtype=np.uint64)) + (
        int(np.sum(x >> np.uint64(32), dtype=np.uint64)) << 32)


def checksum(canonical_indices, vals) -> int:
    """Checksum128 of (index, value) terms (verify.py:68-96), vectorised:
    sum of mix64(idx) * (mix64(bits) | 1) mod 2^128 via 32-bit limb products."""
    a = mix64(np.asarray(canonical_indices, dtype=np.uint64))
    b = mix64(value_bits(vals)) | np.uint64(1)
    m32 = np.uint64(0xFFFFFFFF)
    a0, a1 = a & m32, a >> np.uint64(32)
    b0, b1 = b & m32, b >> np.uint64(32)
    total = (_sum_u64(a0 * b0) + ((_sum_u64(a1 * b0) + _sum_u64(a0 * b1)) << 32)
             + (_sum_u64(a1 * b1) << 64))
    return total & MASK128


def checksum_hex(canonical_indices, vals) -> str:
    return format(checksum(canonical_indices, vals), "032x")


def values_field_split(V, arity: int, n_pf: int):
    """Values of a run whose field axis is split into n_pf slabs: every
    numerator and column sum is a per-slab sequential sum, folded in
    ascending p_f order (engine.py:197-216; metrics2.py:135-156,
    metrics3.py:88-164)."""
    V = np.asarray(V)
    dt = V.dtype.type
    w = V.shape[0] // n_pf
    slabs = [V[p * w:(p + 1) * w] for p in range(n_pf)]

    def fold(parts):
        total = parts[0]
        for p in parts[1:]:
            total = total + p
        return total

    N = fold([mgemm(s, s) for s in slabs])
    s = fold([column_sums(x) for x in slabs])
    if arity == 2:
        iu, ju = np.triu_indices(V.shape[1], k=1)
        d = s[iu] + s[ju]
        zero = d == 0
        vals = (dt(2) * N[iu, ju]) / np.where(zero, dt(1), d)
        return np.where(zero, dt(0), vals).astype(V.dtype), zero
    T = fold([triple_min(x) for x in slabs])
    i, j, k = triple_ids(V.shape[1])
    n3 = ((N[i, j] + N[i, k]) + N[j, k]) - T[i, j, k]
    d = (s[i] + s[j]) + s[k]
    zero = d == 0
    vals = (dt(1.5) * n3) / np.where(zero, dt(1), d)
    return np.where(zero, dt(0), vals).astype(V.dtype), zero


def run_2way(V):
    """(values, degenerate mask, checksum hex) of a full single-rank 2-way run."""
    vals, zero = values_2way(V)
    return vals, zero, checksum_hex(np.arange(len(vals)), vals)


def run_3way(V):
    vals, zero = values_3way(V)
    return vals, zero, checksum_hex(np.arange(len(vals)), vals)


def pair_values_sampled(V, pairs):
    """Values of selected pairs only (columns-only recomputation)."""
    V = np.asarray(V)
    dt = V.dtype.type
    out = np.empty(len(pairs), dtype=V.dtype)
    for t, (i, j) in enumerate(pairs):
        a, b = V[:, i], V[:, j]
        zero = np.zeros(1, dtype=V.dtype)
        # np.cumsum is a strict left-to-right scan: a sequential sum from +0
        n = np.cumsum(np.concatenate([zero, np.where(a < b, a, b)]))[-1]
        si = np.cumsum(np.concatenate([zero, a]))[-1]
        sj = np.cumsum(np.concatenate([zero, b]))[-1]
        d = si + sj
        out[t] = dt(0) if d == 0 else (dt(2) * n) / d
    return out


def _seq_sum(x, slabs: int = 1):
    """Sequential ascending sum from +0 (np.cumsum is a strict left-to-right
    scan); with slabs > 1, per-slab sums folded in ascending slab order
    (reduce_field_axis, engine.py:197-216)."""
    x = np.asarray(x)
    w = len(x) // slabs
    total = None
    for p in range(slabs):
        part = np.cumsum(np.concatenate([np.zeros(1, x.dtype), x[p * w:(p + 1) * w]]))[-1]
        total = part if total is None else total + part
    return total


def pair_values_sampled_slabs(V, pairs, n_pf: int = 1):
    """Selected 2-way values recomputed from their two columns only."""
    V = np.asarray(V)
    dt = V.dtype.type
    out = np.empty(len(pairs), dtype=V.dtype)
    for t, (i, j) in enumerate(pairs):
        a, b = V[:, i], V[:, j]
        n = _seq_sum(np.where(a < b, a, b), n_pf)
        d = _seq_sum(a, n_pf) + _seq_sum(b, n_pf)
        out[t] = dt(0) if d == 0 else (dt(2) * n) / d
    return out


def triple_values_sampled(V, triples, n_pf: int = 1):
    """Selected 3-way values recomputed from their three columns only
    (pair_numerators / triple_min_numerators / metric3_value)."""
    V = np.asarray(V)
    dt = V.dtype.type
    out = np.empty(len(triples), dtype=V.dtype)
    for t, (i, j, k) in enumerate(triples):
        a, b, c = V[:, i], V[:, j], V[:, k]
        nij = _seq_sum(np.where(a < b, a, b), n_pf)
        nik = _seq_sum(np.where(a < c, a, c), n_pf)
        njk = _seq_sum(np.where(b < c, b, c), n_pf)
        ab = np.where(a < b, a, b)
        n3p = _seq_sum(np.where(ab < c, ab, c), n_pf)
        d = (_seq_sum(a, n_pf) + _seq_sum(b, n_pf)) + _seq_sum(c, n_pf)
        n3 = ((nij + nik) + njk) - n3p
        out[t] = dt(0) if d == 0 else (dt(1.5) * n3) / d
    return out


def _seq_sum_cols(X, slabs: int = 1):
    """Per-column sequential ascending sums of X (n_f, k) from +0 (np.cumsum
    along axis 0 is a strict left-to-right scan per column); with slabs > 1,
    per-slab sums folded in ascending slab order (engine.py:197-216)."""
    X = np.asarray(X)
    w = X.shape[0] // slabs
    total = None
    for p in range(slabs):
        part = np.cumsum(np.concatenate([np.zeros((1, X.shape[1]), X.dtype),
                                         X[p * w:(p + 1) * w]]), axis=0)[-1]
        total = part if total is None else total + part
    return total


def pair_values_grid(VR, VC, n_pf: int = 1):
    """2-way values of every (row column r, col column c) combination,
    recomputed from those columns only: pair_numerators (mingemm.py:237-247),
    column_sums (212-222) and metric2_value (metrics2.py:77-82). Returns an
    (a, b) array for VR (n_f, a) and VC (n_f, b)."""
    VR, VC = np.asarray(VR), np.asarray(VC, dtype=np.asarray(VR).dtype)
    dt = VR.dtype.type
    sr, sc = _seq_sum_cols(VR, n_pf), _seq_sum_cols(VC, n_pf)
    out = np.empty((VR.shape[1], VC.shape[1]), dtype=VR.dtype)
    for r in range(VR.shape[1]):
        x = VR[:, r:r + 1]
        num = _seq_sum_cols(np.where(x < VC, x, VC), n_pf)
        d = sr[r] + sc
        with np.errstate(divide="ignore", invalid="ignore"):
            v = (dt(2) * num) / d
        out[r] = np.where(d == 0, dt(0), v)
    return out


def triple_values_grid(VI, xj, VK, n_pf: int = 1):
    """3-way values of every (i, j, k) with one pivot column xj (n_f,), rows
    VI (n_f, a) and columns VK (n_f, b), recomputed from those columns only:
    pair_numerators / triple_min_numerators (mingemm.py:237-260), column_sums
    and metric3_value (metrics3.py:38-44) with the canonical roles i < j < k
    (the caller passes i < j < k). Returns an (a, b) array."""
    VI = np.asarray(VI)
    dt = VI.dtype.type
    xj = np.asarray(xj, dtype=VI.dtype)[:, None]
    VK = np.asarray(VK, dtype=VI.dtype)
    si, sk = _seq_sum_cols(VI, n_pf), _seq_sum_cols(VK, n_pf)
    sj = _seq_sum_cols(xj, n_pf)[0]
    nij = _seq_sum_cols(np.where(VI < xj, VI, xj), n_pf)          # (a,)
    njk = _seq_sum_cols(np.where(xj < VK, xj, VK), n_pf)          # (b,)
    ab = np.where(VI < xj, VI, xj)                                # min(v_i, x_j)
    out = np.empty((VI.shape[1], VK.shape[1]), dtype=VI.dtype)
    for r in range(VI.shape[1]):
        a, m = VI[:, r:r + 1], ab[:, r:r + 1]
        nik = _seq_sum_cols(np.where(a < VK, a, VK), n_pf)
        n3p = _seq_sum_cols(np.where(m < VK, m, VK), n_pf)
        n3 = ((nij[r] + nik) + njk) - n3p
        d = (si[r] + sj) + sk
        with np.errstate(divide="ignore", invalid="ignore"):
            v = (dt(1.5) * n3) / d
        out[r] = np.where(d == 0, dt(0), v)
    return out


def uniform_cols(seed: int, n_f: int, n_v: int, cols, dtype=np.float64):
    """Selected global columns of the uniform matrix."""
    q = np.arange(n_f, dtype=np.uint64)[:, None]
    i = np.asarray(cols, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        h = mix64((q * np.uint64(n_v) + i) ^ np.uint64(seed & MASK64))
    if np.dtype(dtype) == np.float64:
        return np.asfortranarray((h >> np.uint64(11)).astype(np.float64) * 2.0**-53)
    return np.asfortranarray((h >> np.uint64(40)).astype(np.float32) * np.float32(2.0**-24))


def n_pairs(n_v: int) -> int:
    return math.comb(n_v, 2)
