"""Pins of the oracle's CRC24A/B, 36.212 segmentation and QPP interleaver
against the CRC catalogue, hand-worked 36.212 examples, closed forms and
invariants.  CPU only."""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [l.split() for l in f if l.strip() and not l.startswith("#")]


def _ascii_bits(s):
    return np.array([(b >> (7 - i)) & 1 for b in s.encode() for i in range(8)], np.uint8)


# ------------------------------------------------------------------ CRC
def test_crc_catalogue_check_values(orc):
    bits = _ascii_bits("123456789")
    for name, kind, check in _rows("crc_catalogue.txt"):
        k = orc.CRC24A if kind == "A" else orc.CRC24B
        assert orc.crc24(k, bits) == int(check, 16), name


@pytest.mark.parametrize("kind", [1, 2])
def test_crc_attach_check_and_single_flips(orc, kind):
    rng = np.random.default_rng(1)
    x = rng.integers(0, 2, 64, dtype=np.uint8)
    cw = orc.crc_attach(kind, x)
    assert cw.size == 88 and orc.crc24(kind, cw) == 0
    for n in range(cw.size):                      # every single flip detected
        e = cw.copy()
        e[n] ^= 1
        assert orc.crc24(kind, e) != 0


@pytest.mark.parametrize("kind", [1, 2])
def test_crc_odd_weight_linearity_leading_zeros(orc, kind):
    rng = np.random.default_rng(2)
    for _ in range(50):
        n = int(rng.integers(30, 300))
        cw = orc.crc_attach(kind, rng.integers(0, 2, n, dtype=np.uint8))
        w = 2 * int(rng.integers(0, 4)) + 1       # both generators have a (1+D) factor
        e = np.zeros_like(cw)
        e[rng.choice(cw.size, w, replace=False)] = 1
        assert orc.crc24(kind, cw ^ e) != 0
        a = rng.integers(0, 2, n, dtype=np.uint8)
        b = rng.integers(0, 2, n, dtype=np.uint8)
        assert orc.crc24(kind, a ^ b) == orc.crc24(kind, a) ^ orc.crc24(kind, b)
        z = np.concatenate([np.zeros(int(rng.integers(1, 40)), np.uint8), a])
        assert orc.crc24(kind, z) == orc.crc24(kind, a)


def test_crc_equals_polynomial_remainder(orc):
    """Register = M(x) x^24 mod g(x): long division over GF(2) on Python ints."""
    g = {1: (1 << 24) | 0x864CFB, 2: (1 << 24) | 0x800063}
    rng = np.random.default_rng(3)
    for kind in (1, 2):
        for _ in range(20):
            bits = rng.integers(0, 2, int(rng.integers(1, 200)), dtype=np.uint8)
            m = int("".join(map(str, bits)), 2) << 24
            while m.bit_length() > 24:
                m ^= g[kind] << (m.bit_length() - 25)
            assert orc.crc24(kind, bits) == m


# ------------------------------------------------------------------ K table / segmentation
def test_k_table_closed_form(orc):
    exp = (list(range(40, 513, 8)) + list(range(528, 1025, 16)) + list(range(1056, 2049, 32))
           + list(range(2112, 6145, 64)))
    assert orc.k_table() == exp and len(exp) == 188


def test_segmentation_worked_examples(orc):
    for r in _rows("segmentation_36212.txt"):
        tbs, C, Kp, Km, Cp, Cm, F, L = map(int, r)
        s = orc.segment(tbs)
        assert (s["C"], s["Kplus"], s["Kminus"], s["Cplus"], s["Cminus"], s["F"], s["L"]) == \
            (C, Kp, Km, Cp, Cm, F, L), tbs


def test_segmentation_invariants(orc):
    ks = orc.k_table()
    rng = np.random.default_rng(4)
    for tbs in list(rng.integers(1, 200000, 400)) + [6119, 6120, 6121, 12240, 75376]:
        s = orc.segment(int(tbs))
        B = tbs + 24
        Bp = B if s["C"] == 1 else B + 24 * s["C"]
        assert (s["C"] == 1) == (B <= 6144)
        assert s["C"] == (1 if B <= 6144 else math.ceil(B / 6120))
        assert s["Kplus"] in ks and s["Cplus"] + s["Cminus"] == s["C"]
        assert s["Cplus"] * s["Kplus"] + s["Cminus"] * s["Kminus"] == Bp + s["F"]
        assert 0 <= s["F"] < (s["Kplus"] - s["Kminus"] if s["C"] > 1 else s["Kplus"])
        # K+ is the smallest table size with C*K >= B'
        assert s["C"] * s["Kplus"] >= Bp
        i = ks.index(s["Kplus"])
        assert i == 0 or s["C"] * ks[i - 1] < Bp


def test_tb_segment_reassemble_roundtrip(orc):
    rng = np.random.default_rng(5)
    for tbs in (16, 1000, 4000, 6120, 6121, 12000, 40000, 75376):
        a = rng.integers(0, 2, tbs, dtype=np.uint8)
        cbs, Fs, seg = orc.segment_tb_bits(a)
        assert len(cbs) == seg["C"]
        for c, F in zip(cbs, Fs):
            assert np.all(c[:F] == 0)
            if seg["C"] > 1:
                assert orc.crc24b(c) == 0
        assert np.array_equal(orc.reassemble_tb(cbs, Fs, seg), a)
        if seg["C"] > 1:                          # one failed CB loses the TB
            bad = [c.copy() for c in cbs]
            bad[-1][-30] ^= 1
            assert orc.reassemble_tb(bad, Fs, seg) is None


# ------------------------------------------------------------------ QPP
def test_qpp_k40_example(orc):
    exp = [int(x) for x in _rows("qpp_k40.txt")[0]]
    assert orc.qpp_params(40) == (3, 10)
    assert list(orc.qpp_perm(40)) == exp


def _primes(n):
    p, d = set(), 2
    while d * d <= n:
        while n % d == 0:
            p.add(d)
            n //= d
        d += 1
    if n > 1:
        p.add(n)
    return p


def test_qpp_all_sizes_permutation_and_contention_free(orc):
    for K in orc.k_table():
        f1, f2 = orc.qpp_params(K)
        pi = orc.qpp_perm(K)
        assert sorted(pi) == list(range(K)), K                       # bijection
        assert math.gcd(f1, K) == 1 and all(f2 % p == 0 for p in _primes(K))
        assert np.all(pi % 2 == np.arange(K) % 2)                    # parity preserving
        M = orc.num_windows(K, 32)
        W = K // M
        assert K % W == 0 and W >= 32 and (M == 1 or K // (M + 1) < 32 or K % (M + 1))
        # contention-free: at every step i, the M windows hit M distinct windows
        # and all hit the same in-window offset (Pi(jW+i) = Pi(i) mod W)
        pw = pi.reshape(M, W)
        assert np.all(pw % W == pw[0] % W)
        assert all(len(set(pw[:, i] // W)) == M for i in range(W))
        # deinterleave(interleave(x)) = x
        x = np.arange(K)
        y = x[pi]
        z = np.empty_like(y)
        z[pi] = y
        assert np.array_equal(z, x)


def test_qpp_forward_recurrence(orc):
    for K in (40, 1056, 6144, 248, 4224):
        f1, f2 = orc.qpp_params(K)
        pi = orc.qpp_perm(K)
        g = (f1 + f2) % K
        p = 0
        for x in range(K):
            assert p == pi[x]
            p = (p + g) % K
            g = (g + 2 * f2) % K


def test_window_examples(orc):
    # SURVEY.md 8c.4 / A.3 examples of M_K x W_K
    for K, M in ((40, 1), (64, 2), (120, 3), (504, 14), (528, 16), (1008, 28), (1056, 33),
                 (2112, 66), (5824, 182), (6144, 192)):
        assert orc.num_windows(K, 32) == M, K
    Ws = [K // orc.num_windows(K, 32) for K in orc.k_table()]
    assert min(Ws) == 32 and max(Ws) == 62
