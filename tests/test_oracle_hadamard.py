"""Pins for oracle/hadamard.py against what the paper and mathematics fix (CPU only)."""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg

from oracle import hadamard as had
from oracle import layer

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


@pytest.mark.parametrize("n", range(0, 11))
def test_sylvester_matches_scipy(n):
    # P2: Eq. (1) recursion == textbook Sylvester construction (scipy).
    assert np.array_equal(had.sylvester(2**n), scipy.linalg.hadamard(2**n))


def test_h2_definition():
    # P:60-61 Eq. (1)
    g = GOLD["hadamard_2"]
    assert np.allclose(had.hadamard(2) * math.sqrt(2), np.array(g["dense_times_sqrt2"]), atol=1e-15)


@pytest.mark.parametrize("m", [20, 28, 108, 172])
def test_base_matrices_are_hadamard(m):
    # P1 / P:59: entries +-1 and H H^T = m I exactly (int64).
    h = had.base_matrix(m)
    assert set(np.unique(h)) == {-1, 1}
    assert np.array_equal(h @ h.T, m * np.eye(m, dtype=np.int64))


def test_base_checksums_recorded():
    # Z3: the instances are pinned by checksum (recorded independently in SURVEY App. A).
    rec = {}
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "hadamard_checksums.txt")):
        if line.strip() and not line.startswith("#"):
            m, pre = line.split()
            rec[int(m)] = pre
    for m, pre in rec.items():
        assert had.base_checksum(m).startswith(pre)


def test_h28_symmetric_h172_not():
    # Z4: orientation only matters for the non-symmetric H_172 (and the Paley I H_20 / H_108,
    # which are I + skew: H + H^T = 2 I).
    assert np.array_equal(had.h28(), had.h28().T)
    assert not np.array_equal(had.h172(), had.h172().T)
    for m in (20, 108):
        h = had.base_matrix(m)
        assert np.array_equal(h + h.T, 2 * np.eye(m, dtype=np.int64))


@pytest.mark.parametrize("d,expect", [(256, (256, 1)), (4096, (4096, 1)), (8192, (8192, 1)),
                                      (11008, (64, 172)), (28672, (1024, 28)), (128, (128, 1)),
                                      (5120, (256, 20)), (13824, (128, 108))])
def test_factorize_llama_sizes(d, expect):
    # d = 2^n m; Llama-2 FFN widths (BASELINE configs).
    assert had.factorize(d) == expect


@pytest.mark.parametrize("d", [12, 100, 3, 0, 5120 * 3])
def test_factorize_rejects_unsupported(d):
    with pytest.raises(ValueError):
        had.factorize(d)


@pytest.mark.parametrize("d", [2, 16, 256, 28 * 4, 172 * 4, 28 * 64])
def test_dense_orthogonality(d):
    # P1: H_d H_d^T = d I for the Kronecker construction.
    h = had.hadamard_unnormalized(d)
    assert np.array_equal(h @ h.T, d * np.eye(d, dtype=np.int64))


@pytest.mark.parametrize("d", [11008, 28672])
def test_large_rows_orthogonal_sampled(d):
    # P1 at the Llama sizes, on sampled rows against every row.
    rng = np.random.default_rng(0)
    sample = rng.choice(d, size=3, replace=False)
    hs = np.stack([had.hadamard_rows(d, slice(i, i + 1))[0] for i in sample]).astype(np.float64)
    gram = np.zeros((3, d))
    for r0 in range(0, d, 4096):
        blk = had.hadamard_rows(d, slice(r0, min(d, r0 + 4096))).astype(np.float64)
        gram[:, r0:r0 + blk.shape[0]] = hs @ blk.T
    expect = np.zeros((3, d))
    expect[np.arange(3), sample] = d
    assert np.array_equal(gram, expect)


def test_kron_rows_entrywise_definition():
    # H_d[a m + b, a' m + b'] = H_{2^n}[a,a'] H_m[b,b'], sampled entries.
    d = 28672
    p, m = had.factorize(d)
    rng = np.random.default_rng(1)
    rows = rng.choice(d, 5, replace=False)
    for i in rows:
        r = had.hadamard_rows(d, slice(i, i + 1))[0]
        for j in rng.choice(d, 50, replace=False):
            assert r[j] == had.sylvester(p)[i // m, j // m] * had.base_matrix(m)[i % m, j % m]


def test_fwht_worked_examples():
    # P3
    for key in ("fwht_basis", "fwht_constant"):
        g = GOLD[key]
        assert np.allclose(had.apply_full(np.array([g["x"]], dtype=np.float64))[0], g["y"], atol=1e-15)


@pytest.mark.parametrize("d", [256, 28 * 8, 172 * 4, 11008])
def test_norm_preserved_and_inverse(d):
    # orthonormality: ||H^ x|| = ||x||; H^T H^ x = x (Z5)
    rng = np.random.default_rng(d)
    x = rng.standard_normal((3, d))
    y = had.apply_full(x)
    assert np.allclose(np.linalg.norm(y, axis=1), np.linalg.norm(x, axis=1), rtol=1e-12)
    h = had.hadamard(d) if d <= 12288 else None
    back = y @ h  # H^T applied to column vectors == row @ H
    assert np.allclose(back, x, atol=1e-10)


def test_full_streaming_equals_dense_path():
    # the blocked-row path used above _DENSE_LIMIT computes the same matvec
    d = 28 * 512  # 14336 > _DENSE_LIMIT
    rng = np.random.default_rng(7)
    x = rng.standard_normal((2, d))
    y = had.apply_full(x)
    # independent: dense mixed-product identity (A (x) B) vec(X) = vec(A X B^T)
    p, m = had.factorize(d)
    xm = x.reshape(2, p, m)
    y2 = np.einsum("ab,nbc,dc->nad", had.sylvester(p).astype(float), xm, had.base_matrix(m).astype(float))
    assert np.allclose(y, y2.reshape(2, d) / math.sqrt(d), atol=1e-11)


@pytest.mark.parametrize("n_h,d_h", [(4, 8), (8, 16), (2, 2), (64, 128), (32, 128)])
def test_eq9_heads_identity(n_h, d_h):
    # P4: H_{n_h d_h} = (I (x) H_{d_h})(H_{n_h} (x) I) (Eq. 9)
    rng = np.random.default_rng(n_h * 1000 + d_h)
    x = rng.standard_normal((3, n_h * d_h))
    two_step = had.apply_per_head(had.apply_across_heads(x, d_h), d_h)
    assert np.allclose(two_step, had.apply_full(x), atol=1e-12)


def test_headwise_degenerate_cases():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 64))
    assert np.allclose(had.apply_per_head(x, 64), had.apply_full(x), atol=1e-13)  # n_h = 1
    assert np.allclose(had.apply_across_heads(x, 1), had.apply_full(x), atol=1e-13)  # d_h = 1
    assert np.array_equal(had.apply_across_heads(np.zeros((1, 64)), 8), np.zeros((1, 64)))


def test_incoherence_examples():
    assert had.incoherence(np.eye(4)) == pytest.approx(GOLD["incoherence_identity"]["mu"])
    assert had.incoherence(np.full((5, 7), 3.0)) == pytest.approx(1.0)


def test_outliers_removed_by_rotation():
    # P13 (Fig. activation_dist, Eq. 2): planted x50 channels -> rotation spreads
    # them; max/rms and kurtosis drop in >= 95 of 100 seeds.
    wins = 0
    for seed in range(100):
        rng = np.random.default_rng(seed)
        x = rng.standard_normal((4, 256))
        x[:, rng.choice(256, 4, replace=False)] *= 50
        y = had.apply_full(x)

        def peak(v):
            return np.max(np.abs(v)) / np.sqrt(np.mean(v**2))

        def kurt(v):
            v = v.ravel()
            return np.mean((v - v.mean())**4) / np.var(v)**2

        if peak(y) < peak(x) and kurt(y) < kurt(x) and had.incoherence(y) < had.incoherence(x):
            wins += 1
    assert wins >= 95


def _random_orthogonal(d, rng):
    q, r = np.linalg.qr(rng.standard_normal((d, d)))
    return q * np.sign(np.diag(r))[None, :]


@pytest.mark.parametrize("f", [172 * 4, 28 * 16])
def test_computational_invariance_ffn(f):
    # P12: rotated full-precision FFN (Fig. ffn_quarot, Eqs. 3-4) reproduces the
    # original FFN output: YQ Q^T == Y within 1e-9 (north_star bar 1e-5).
    rng = np.random.default_rng(f)
    d = 64
    x = rng.standard_normal((5, d))
    wg, wu = rng.standard_normal((f, d)) / 8, rng.standard_normal((f, d)) / 8
    wd = rng.standard_normal((d, f)) / 16
    alpha = rng.uniform(0.5, 1.5, d)
    q = had.randomized(d, rng.choice([-1.0, 1.0], d))
    y = layer.ffn_reference(x, wg, wu, wd, alpha)
    yq = layer.ffn_quarot_fullprecision(x @ q, wg, wu, wd, alpha, q)
    rel = np.linalg.norm(yq @ q.T - y) / np.linalg.norm(y)
    assert rel < 1e-9


def test_rmsnorm_commutation_eq3():
    # Eq. (3): RMSNorm(X) = RMSNorm(X Q^T) Q for orthogonal Q
    rng = np.random.default_rng(11)
    x = rng.standard_normal((4, 32))
    q = _random_orthogonal(32, rng)
    assert np.allclose(layer.rmsnorm_noscale(x), layer.rmsnorm_noscale(x @ q.T) @ q, atol=1e-13)


def _linear_invariance_error(k, online, weight):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((6, k))
    w = rng.standard_normal((9, k))
    return np.linalg.norm(online(x) @ weight(w).T - x @ w.T) / np.linalg.norm(x @ w.T)


@pytest.mark.parametrize("k", [688, 448, 256])
def test_linear_invariance_and_negative_controls(k):
    # P12 on the linear level: (x H^T)(H W)-pairing is exact ...
    ok = _linear_invariance_error(k, lambda x: layer.online_transform(x, "full"),
                                  lambda w: layer.rotate_weight(w, "full"))
    assert ok < 1e-12
    # P16 negative controls must FAIL by >> 1e-2: skip the online H
    bad = _linear_invariance_error(k, lambda x: x, lambda w: layer.rotate_weight(w, "full"))
    assert bad > 1e-1
    p, m = had.factorize(k)
    if m == 172:
        # transposed H_172 (wrong orientation, Z4)
        ht = np.kron(had.sylvester(p), had.h172().T) / math.sqrt(k)
        bad_t = _linear_invariance_error(k, lambda x: x @ ht.T, lambda w: layer.rotate_weight(w, "full"))
        assert bad_t > 1e-1
    if m > 1:
        # wrong Kronecker order H_m (x) H_{2^n} (Z2)
        hw = np.kron(had.base_matrix(m), had.sylvester(p)) / math.sqrt(k)
        bad_o = _linear_invariance_error(k, lambda x: x @ hw.T, lambda w: layer.rotate_weight(w, "full"))
        assert bad_o > 1e-1


def test_across_heads_pairing():
    # Stage 1c: Z <- Z (H_{n_h} (x) I) online with W_out rotated identically
    err = _linear_invariance_error(512, lambda x: layer.online_transform(x, "across_heads", 64),
                                   lambda w: layer.rotate_weight(w, "across_heads", 64))
    assert err < 1e-12
