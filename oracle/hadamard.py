"""Hadamard matrices and the online Hadamard transforms — oracle (TEST INFRASTRUCTURE).

Definitions followed (§3.1 "Orthogonal, Rotation and Hadamard Matrices"):

* P:59    a Hadamard matrix is orthogonal with entries from {+1, -1} (after scaling).
* P:60-63 Eq. (1): H_2 = (1/sqrt 2)[[1,1],[1,-1]],  H_{2^n} = H_2 (x) H_{2^{n-1}}.
* P:67    for d != 2^n: d = 2^n m with m the size of a *known* Hadamard matrix,
          H_d = H_{2^n} (x) H_m.
* P:69    randomized Hadamard  H~ = H diag(s), s in {+1,-1}^d.
* P:204-208 Eq. (9): H_{n_h d_h} = (I (x) H_{d_h}) (H_{n_h} (x) I)  ("Hadamard heads").
* P:219-223 Eqs. (13)-(14): per-head H_{d_h} on post-RoPE queries and keys.

Everything here is *dense*: the transform of a vector is a plain matrix-vector
product with the explicit +-1 matrix, divided by sqrt(d) (reading Z5).  The fast
algorithms (FWHT butterflies, fused kernels) live only in the CUDA path.

Readings: Z1 Sylvester/natural order; Z2 Kronecker order
H_{2^n} (x) H_m exactly as P:67 writes it (index i = a*m + b, H_m acting on the
contiguous b); Z3 the specific H_20 / H_28 / H_108 / H_172 instances below; Z4 y = H x (row i of
H dotted with x); Z5 orthonormal scaling 1/sqrt(d).
"""
from __future__ import annotations

import hashlib
import math
from functools import lru_cache

import numpy as np

# --------------------------------------------------------------------------------------
# Sylvester (Walsh) matrices, Eq. (1)
# --------------------------------------------------------------------------------------


@lru_cache(maxsize=None)
def sylvester(p: int) -> np.ndarray:
    """Unnormalized Walsh-Hadamard matrix of order p = 2^n, by the recursion of
    Eq. (1): H_{2^n} = H_2 (x) H_{2^{n-1}}, H_1 = [1].  int64 entries +-1."""
    if p < 1 or p & (p - 1):
        raise ValueError(f"sylvester order must be a power of two, got {p}")
    h = np.ones((1, 1), dtype=np.int64)
    h2 = np.array([[1, 1], [1, -1]], dtype=np.int64)
    while h.shape[0] < p:
        h = np.kron(h2, h)  # H_2 (x) H_{2^{n-1}}
    h.setflags(write=False)
    return h


# --------------------------------------------------------------------------------------
# Known non-power-of-two Hadamard matrices ("a list of known Hadamard matrices").
# The cited list is not available offline; we construct the two sizes the Llama-2
# FFN widths need with classical constructions (reading Z3).  Any Hadamard matrix of
# the right order satisfies the paper; the pins (tests) are H H^T = m I.
# --------------------------------------------------------------------------------------


def _quadratic_character(q: int) -> np.ndarray:
    """chi(x) for x in GF(q), q prime: 0 at 0, +1 on non-zero squares, -1 otherwise."""
    squares = {(x * x) % q for x in range(1, q)}
    return np.array([0] + [1 if x in squares else -1 for x in range(1, q)], dtype=np.int64)


@lru_cache(maxsize=None)
def h28() -> np.ndarray:
    """H_28 by Paley's second construction with q = 13 (q = 1 mod 4).

    Jacobsthal Q_ij = chi(j - i) over GF(13); conference matrix
    S = [[0, 1^T], [1, Q]] (order 14, symmetric);
    H_28 = S (x) [[1,1],[1,-1]] + I_14 (x) [[1,-1],[-1,-1]].  Symmetric."""
    q = 13
    chi = _quadratic_character(q)
    jac = np.array([[chi[(j - i) % q] for j in range(q)] for i in range(q)], dtype=np.int64)
    s = np.zeros((q + 1, q + 1), dtype=np.int64)
    s[0, 1:] = 1
    s[1:, 0] = 1
    s[1:, 1:] = jac
    h = np.kron(s, np.array([[1, 1], [1, -1]])) + np.kron(np.eye(q + 1, dtype=np.int64), np.array([[1, -1], [-1, -1]]))
    h = h.astype(np.int64)
    h.setflags(write=False)
    return h


def _paley1(q: int) -> np.ndarray:
    """Paley's first construction, q prime with q = 3 mod 4: Jacobsthal Q_ij = chi(j - i) is
    antisymmetric; S = [[0, 1^T], [-1, Q]] (skew conference matrix of order q + 1); H = I + S."""
    chi = _quadratic_character(q)
    jac = np.array([[chi[(j - i) % q] for j in range(q)] for i in range(q)], dtype=np.int64)
    s = np.zeros((q + 1, q + 1), dtype=np.int64)
    s[0, 1:] = 1
    s[1:, 0] = -1
    s[1:, 1:] = jac
    h = (np.eye(q + 1, dtype=np.int64) + s).astype(np.int64)
    h.setflags(write=False)
    return h


@lru_cache(maxsize=None)
def h20() -> np.ndarray:
    """H_20 by Paley I with q = 19 (Llama-2-13B hidden 5120 = 256 x 20).  Not symmetric."""
    return _paley1(19)


@lru_cache(maxsize=None)
def h108() -> np.ndarray:
    """H_108 by Paley I with q = 107 (Llama-2-13B FFN 13824 = 128 x 108).  Not symmetric."""
    return _paley1(107)


# Williamson quadruple of order 43 from the cyclotomic classes of index 7 of GF(43),
# generator 3.  Each of A, B, C, D is the symmetric circulant with first row
# v[0] = a0 and v[j] = -1 iff j lies in the union of the classes selected by `mask`
# (bit i selects C_i), else +1.  (mask, a0) found by exhaustive search over the
# 2 * 128 candidates per matrix for A^2 + B^2 + C^2 + D^2 = 172 I.
_WILLIAMSON_43 = ((7, +1), (25, +1), (44, +1), (50, -1))


def _cyclotomic_classes(p: int = 43, g: int = 3, e: int = 7):
    f = (p - 1) // e
    return [sorted({pow(g, e * k + i, p) for k in range(f)}) for i in range(e)]


def _williamson_circulant(mask: int, a0: int, p: int = 43) -> np.ndarray:
    classes = _cyclotomic_classes(p)
    neg = set()
    for i, c in enumerate(classes):
        if mask >> i & 1:
            neg.update(c)
    v = np.array([a0] + [(-1 if j in neg else 1) for j in range(1, p)], dtype=np.int64)
    return np.array([[v[(j - i) % p] for j in range(p)] for i in range(p)], dtype=np.int64)


@lru_cache(maxsize=None)
def h172() -> np.ndarray:
    """H_172 by the Williamson array on a cyclotomic Williamson quadruple of order 43:
    H = [[A,B,C,D], [-B,A,-D,C], [-C,D,A,-B], [-D,-C,B,A]].  NOT symmetric (Z4)."""
    a, b, c, d = (_williamson_circulant(m, s) for m, s in _WILLIAMSON_43)
    h = np.block([[a, b, c, d], [-b, a, -d, c], [-c, d, a, -b], [-d, -c, b, a]]).astype(np.int64)
    h.setflags(write=False)
    return h


BASE_SIZES = (1, 20, 28, 108, 172)


def base_matrix(m: int) -> np.ndarray:
    """The stored small Hadamard H_m, m in BASE_SIZES (int64 +-1)."""
    if m == 1:
        return np.ones((1, 1), dtype=np.int64)
    if m == 20:
        return h20()
    if m == 28:
        return h28()
    if m == 108:
        return h108()
    if m == 172:
        return h172()
    raise ValueError(f"no stored Hadamard matrix of order {m}; supported {BASE_SIZES}")


def base_checksum(m: int) -> str:
    """SHA-256 of the int8 row-major bytes of H_m (reading Z3 pins the instance)."""
    return hashlib.sha256(base_matrix(m).astype(np.int8).tobytes()).hexdigest()


def factorize(d: int) -> tuple[int, int]:
    """d = 2^n * m with m in BASE_SIZES, choosing the smallest admissible m
    (largest power of two), P:67 and SPEC S:197.  Returns (2^n, m)."""
    if d <= 0:
        raise ValueError(f"dimension must be positive, got {d}")
    best = None
    for m in BASE_SIZES:
        if d % m == 0:
            p = d // m
            if p & (p - 1) == 0:
                if best is None or m < best[1]:
                    best = (p, m)
    if best is None:
        raise ValueError(
            f"unsupported Hadamard size {d}: need d = 2^n * m with m in {BASE_SIZES}")
    return best


def hadamard_unnormalized(d: int) -> np.ndarray:
    """Dense H_d = H_{2^n} (x) H_m, int64 +-1, d x d.  Memory d^2 * 8 bytes."""
    p, m = factorize(d)
    return np.kron(sylvester(p), base_matrix(m))


def hadamard_rows(d: int, rows: slice) -> np.ndarray:
    """Rows `rows` of H_d = H_{2^n} (x) H_m, built from the Kronecker definition
    entry-wise: H_d[a*m+b, a'*m+b'] = H_{2^n}[a,a'] * H_m[b,b'].  Used so the dense
    oracle can stream H_d for d = 28672 without a 6.6 GB matrix."""
    p, m = factorize(d)
    idx = np.arange(d)[rows]
    a, b = idx // m, idx % m
    syl, hm = sylvester(p), base_matrix(m)
    # outer structure: for each selected row (a,b): kron(syl[a], hm[b])
    out = (syl[a][:, :, None] * hm[b][:, None, :]).reshape(len(idx), d)
    return out


def hadamard(d: int) -> np.ndarray:
    """Orthonormal Hadamard H^_d = H_d / sqrt(d) (Z5), fp64 dense."""
    return hadamard_unnormalized(d).astype(np.float64) / math.sqrt(d)


# --------------------------------------------------------------------------------------
# Online transforms (the three modes of the hot path), computed as dense matvecs.
# --------------------------------------------------------------------------------------

_DENSE_LIMIT = 12288  # above this, stream rows of H_d in blocks (same arithmetic)


def apply_full(x: np.ndarray) -> np.ndarray:
    """FULL mode (down_proj input, Stage 1b P:182-185): y = H^_K x for every row x of
    x[..., K].  Column convention y_i = sum_j H^_ij x_j (Z4).  fp64."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    flat = x.reshape(-1, d)
    if d <= _DENSE_LIMIT:
        y = flat @ hadamard(d).T
    else:
        y = np.empty_like(flat)
        blk = 2048
        for r0 in range(0, d, blk):
            rows = hadamard_rows(d, slice(r0, min(d, r0 + blk))).astype(np.float64)
            y[:, r0:r0 + rows.shape[0]] = flat @ rows.T
        y /= math.sqrt(d)
    return y.reshape(x.shape)


def apply_across_heads(z: np.ndarray, head_dim: int) -> np.ndarray:
    """ACROSS_HEADS mode ("Hadamard heads", Stage 1c P:204-208, Eq. 9):
    y = (H^_{n_h} (x) I_{d_h}) z with z indexed i = h*d_h + j.  n_h, d_h powers of 2
    (P:208).  Dense: the matrix kron(H^_{n_h}, I) applied to each row."""
    z = np.asarray(z, dtype=np.float64)
    k = z.shape[-1]
    if head_dim <= 0 or k % head_dim:
        raise ValueError(f"width {k} is not a multiple of head_dim {head_dim}")
    n_h = k // head_dim
    if n_h & (n_h - 1) or head_dim & (head_dim - 1):
        raise ValueError("Hadamard heads needs n_h and d_h powers of two (P:208)")
    mat = np.kron(sylvester(n_h).astype(np.float64) / math.sqrt(n_h), np.eye(head_dim))
    return (z.reshape(-1, k) @ mat.T).reshape(z.shape)


def apply_per_head(x: np.ndarray, head_dim: int) -> np.ndarray:
    """PER_HEAD (post-RoPE Q/K rotation, Stage 1d P:219-223 Eqs. 13-14):
    y = (I_{n_h} (x) H^_{d_h}) x.  Dense."""
    x = np.asarray(x, dtype=np.float64)
    k = x.shape[-1]
    if head_dim <= 0 or k % head_dim:
        raise ValueError(f"width {k} is not a multiple of head_dim {head_dim}")
    n_h = k // head_dim
    mat = np.kron(np.eye(n_h), hadamard(head_dim))
    return (x.reshape(-1, k) @ mat.T).reshape(x.shape)


def randomized(d: int, signs: np.ndarray) -> np.ndarray:
    """H~ = H^ diag(s).  Used only offline (global Q fused into weights)."""
    s = np.asarray(signs, dtype=np.float64)
    if s.shape != (d,) or not np.all(np.abs(s) == 1):
        raise ValueError("signs must be a +-1 vector of length d")
    return hadamard(d) * s[None, :]


def incoherence(w: np.ndarray) -> float:
    """mu such that max|W| = mu ||W||_F / sqrt(mn) (Eq. 2)."""
    w = np.asarray(w, dtype=np.float64)
    fro = np.linalg.norm(w)
    if fro == 0:
        raise ValueError("incoherence of a zero matrix is undefined")
    return float(np.max(np.abs(w)) * math.sqrt(w.size) / fro)
