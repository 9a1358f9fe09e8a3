"""Pins of the oracle's RSC/turbo encoder and its constituent SISO against
closed forms (GF(2) polynomial identities), hand-worked values and brute-force
max-log-MAP over all input sequences.  CPU only."""
import itertools
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
G0 = [1, 0, 1, 1]     # 1 + D^2 + D^3 (feedback)
G1 = [1, 1, 0, 1]     # 1 + D + D^3   (feed-forward)


def polymul2(a, b):
    return np.convolve(np.asarray(a, np.int64), np.asarray(b, np.int64)) % 2


def split_tails(d0, d1, d2, K):
    """Stream layout of DESIGN.md R11 (36.212 5.1.3.2.2 column-wise tails)."""
    t = [d0[K], d1[K], d2[K], d0[K + 1], d1[K + 1], d2[K + 1],
         d0[K + 2], d1[K + 2], d2[K + 2], d0[K + 3], d1[K + 3], d2[K + 3]]
    return t[0:6], t[6:12]      # (x_K, z_K, x_K+1, z_K+1, x_K+2, z_K+2), (x', z', ...)


def test_rsc_impulse_response_power_series(orc):
    exp = [int(x) for x in open(os.path.join(GOLD, "rsc_impulse.txt")).read().split("\n")[-2].split()]
    # independent: power series g1/g0 over GF(2) by long division
    n = 16
    q = []
    rem = G1 + [0] * (n + 4)
    for k in range(n):
        q.append(rem[k])
        if rem[k]:
            for j, g in enumerate(G0):
                rem[k + j] ^= g
    assert q == exp
    K = 40
    c = np.zeros(K, np.uint8)
    c[0] = 1
    d0, d1, d2 = orc.turbo_encode(c)
    assert list(d1[:16]) == exp


@pytest.mark.parametrize("K", [40, 48, 104, 1056, 6144])
def test_turbo_encoder_polynomial_identities(orc, K):
    """Both constituents satisfy z(D) g0(D) = u(D) g1(D) over the terminated
    K+3-step sequence (u includes the tail inputs): termination returns the
    register to 0 exactly when this holds as a finite identity."""
    rng = np.random.default_rng(K)
    pi = orc.qpp_perm(K)
    for _ in range(3):
        c = rng.integers(0, 2, K, dtype=np.uint8)
        d0, d1, d2 = orc.turbo_encode(c)
        assert d0.size == d1.size == d2.size == K + 4          # 3K+12 in total
        assert np.array_equal(d0[:K], c)
        t1, t2 = split_tails(d0, d1, d2, K)
        u1 = np.r_[c, t1[0::2]]
        z1 = np.r_[d1[:K], t1[1::2]]
        u2 = np.r_[c[pi], t2[0::2]]
        z2 = np.r_[d2[:K], t2[1::2]]
        for u, z in ((u1, z1), (u2, z2)):
            assert np.array_equal(polymul2(z, G0), polymul2(u, G1))


def test_encoder_zero_and_linearity(orc):
    K = 40
    d = orc.turbo_encode(np.zeros(K, np.uint8))
    assert sum(int(x.sum()) for x in d) == 0 and sum(x.size for x in d) == 132
    rng = np.random.default_rng(7)
    for K in (40, 512, 2048):
        a = rng.integers(0, 2, K, dtype=np.uint8)
        b = rng.integers(0, 2, K, dtype=np.uint8)
        for x, y, z in zip(orc.turbo_encode(a), orc.turbo_encode(b), orc.turbo_encode(a ^ b)):
            assert np.array_equal(x ^ y, z)


# ------------------------------------------------------------------ brute-force SISO
def rsc_paths(n):
    """All 2^n inputs of one constituent: (u [P,n], z [P,n], tail x [P,3], tail z [P,3],
    state after step k [P,n+1]) by the polynomial description a = u/g0, z = a*g1."""
    U = np.array(list(itertools.product([0, 1], repeat=n)), np.int64)
    P = U.shape[0]
    A = np.zeros((P, n + 3), np.int64)          # a_{k} at index k+3 (three leading zeros)
    for k in range(n):
        A[:, k + 3] = U[:, k] ^ A[:, k + 1] ^ A[:, k]        # a_k = u_k + a_{k-2} + a_{k-3}
    Z = A[:, 3:] ^ A[:, 2:-1] ^ A[:, 0:-3]                    # z_k = a_k + a_{k-1} + a_{k-3}
    S = np.zeros((P, n + 1), np.int64)
    for k in range(n + 1):                                    # S = 4 a_{k-1} + 2 a_{k-2} + a_{k-3}
        S[:, k] = 4 * A[:, k + 2] + 2 * A[:, k + 1] + A[:, k]
    r = [A[:, n + 2], A[:, n + 1], A[:, n]]                   # (r1, r2, r3) after n steps
    tx, tz = [], []
    for _ in range(3):
        tx.append(r[1] ^ r[2])
        tz.append(r[0] ^ r[2])
        r = [np.zeros(P, np.int64), r[0], r[1]]
    return U, Z, np.stack(tx, 1), np.stack(tz, 1), S


def brute(lsys, lpar, la, tail, W):
    n = lsys.size
    U, Z, TX, TZ, S = rsc_paths(n)
    Lu = lsys + la
    g = U * Lu + Z * lpar                                     # per-step metric [P, n]
    tm = TX @ tail[0::2] + TZ @ tail[1::2]
    tot = g.sum(1) + tm
    le = np.array([tot[U[:, k] == 1].max() - tot[U[:, k] == 0].max() - Lu[k] for k in range(n)])
    pre = np.concatenate([np.zeros((U.shape[0], 1), np.int64), np.cumsum(g, 1)], 1)
    suf = tot[:, None] - pre
    M = n // W
    alpha = np.zeros((M + 1, 8), np.int64)
    beta = np.zeros((M + 1, 8), np.int64)
    for j in range(M + 1):
        k = j * W
        a = np.array([pre[S[:, k] == s, k].max() if np.any(S[:, k] == s) else -10**9 for s in range(8)])
        b = np.array([suf[S[:, k] == s, k].max() if np.any(S[:, k] == s) else -10**9 for s in range(8)])
        alpha[j] = a - a.max()
        beta[j] = b - b.max()
    return le, alpha, beta, tot, U


@pytest.mark.parametrize("n,W", [(12, 12), (12, 3), (12, 4), (12, 6), (14, 7), (14, 14), (10, 5)])
def test_siso_equals_bruteforce_maxlog(orc, n, W):
    """Le(k) = max_{u_k=1} metric - max_{u_k=0} metric - Lu_k exactly (small LLRs:
    no clamp or floor is active), for the full block (M=1) and for windows whose
    NII boundary states are the exact normalised forward/backward metrics."""
    rng = np.random.default_rng(100 * n + W)
    for _ in range(6):
        lsys, lpar, la = (rng.integers(-100, 101, n) for _ in range(3))
        tail = rng.integers(-100, 101, 6)
        le_b, alpha, beta, tot, U = brute(lsys, lpar, la, tail, W)
        M = n // W
        ai = np.zeros((M, 8), np.int64)
        bi = np.zeros((M, 8), np.int64)
        for j in range(M):
            ai[j] = alpha[j]
            bi[j] = beta[j + 1]
        le, ao, bo, ops, viol = orc.siso(lsys, lpar, la, tail, W, ai, bi)
        assert viol == 0
        assert np.array_equal(le, le_b)
        for j in range(M - 1):
            assert np.array_equal(ao[j], alpha[j + 1])          # alpha_{(j+1)W}
        for j in range(1, M):
            assert np.array_equal(bo[j], beta[j])               # beta_{jW}
        # op count: 129 per trellis step + 90 for the three tail steps
        assert ops == 129 * n + 90
        # Viterbi special case: sign(Lu + Le) is the ML sequence where the optimum is unique
        best = tot.max()
        if np.sum(tot == best) == 1:
            ml = U[np.argmax(tot)]
            lapp = lsys + la + le
            assert np.array_equal((lapp > 0)[lapp != 0], ml.astype(bool)[lapp != 0])


@pytest.mark.parametrize("n,W", [(96, 32), (12, 3), (200, 40), (64, 32)])
def test_nii_iterations_converge_to_full_block(orc, n, W):
    """With the inputs held fixed, repeating the windowed SISO with the oracle's
    NII hand-over (window j starts from what window j-1 / j+1 produced in the
    previous pass) reaches the exact full-block max-log-MAP after M passes:
    window 0 starts from the known state and the last from the tail, so exact
    boundary states advance one window per pass (R13)."""
    rng = np.random.default_rng(n + W)
    for lim in (100, 3000):
        lsys, lpar, la = (rng.integers(-lim, lim + 1, n) for _ in range(3))
        tail = rng.integers(-lim, lim + 1, 6)
        full = orc.siso(lsys, lpar, la, tail, n)[0]
        M = n // W
        ai = bi = None
        for t in range(M):
            le, ao, bo, _, v = orc.siso(lsys, lpar, la, tail, W, ai, bi)
            assert v == 0
            ai, bi = orc.nii_update(ao, bo)
        assert np.array_equal(le, full)
