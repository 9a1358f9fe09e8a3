"""Pins of the oracle's rate matching / de-matching (TS 36.212 5.1.4.1; row f4,
DESIGN.md R30).  CPU only.

* the inter-column permutation P is the 5-bit bit reversal;
* the sub-block interleaver + bit collection + bit selection order equals an
  independent construction (the R x 32 matrix written row by row, columns
  permuted, read column by column, with numpy) for several K and every rv;
* with E = 3(K+4) every coded bit is sent exactly once (a bijection);
* repetition counts, puncturing zeros, HARQ combining = sum, int16 saturation;
* a noiseless rate-1/2 round trip through the decoder.
"""
import numpy as np
import pytest


def _bitrev5(c):
    return int(f"{c:05b}"[::-1], 2)


def test_perm_is_bit_reversal(orc):
    assert [orc.rm_perm(c) for c in range(32)] == [_bitrev5(c) for c in range(32)]
    assert orc.rm_perm(32) == -1


@pytest.mark.parametrize("K", [40, 1056, 6144])
def test_params_closed_form(orc, K):
    for rv in range(4):
        p = orc.rm_params(K, rv)
        R = -(-(K + 4) // 32)
        assert p["R"] == R and p["ND"] == 32 * R - K - 4 and 0 <= p["ND"] < 32
        assert p["k0"] == R * (2 * 12 * rv + 2)            # ceil(Ncb / 8R) = 12 for Ncb = 96R


def _reference_order(K, rv):
    """(stream, d index) of every selected position, built from the matrix picture."""
    D = K + 4
    R = -(-D // 32)
    Kpi, ND = 32 * R, 32 * R - D
    y = np.arange(Kpi) - ND                                  # y index -> d index (negative = <NULL>)
    perm = [_bitrev5(c) for c in range(32)]
    mat = y.reshape(R, 32)[:, perm]                          # written row by row, columns permuted
    v01 = mat.T.reshape(-1)                                  # read column by column
    k = np.arange(Kpi)
    v2 = y[(np.array(perm)[k // R] + 32 * (k % R) + 1) % Kpi]
    w = [(0, x) for x in v01] + [item for i in range(Kpi) for item in ((1, v01[i]), (2, v2[i]))]
    k0 = R * (24 * rv + 2)
    order = [w[(k0 + j) % (3 * Kpi)] for j in range(3 * Kpi)]
    return [o for o in order if o[1] >= 0]


def _probe_positions(orc, K, E, rv):
    """Where each of the E transmitted values lands, via single-impulse de-matching."""
    pos = []
    for k in range(E):
        e = np.zeros(E, np.int16)
        e[k] = 1
        h = orc.rate_dematch(e, K, rv)
        hit = [(s, int(n)) for s in range(3) for n in np.flatnonzero(h[s])]
        assert len(hit) == 1
        pos.append(hit[0])
    return pos


@pytest.mark.parametrize("K", [40, 48, 88])
def test_selection_order_matches_matrix_construction(orc, K):
    for rv in range(4):
        ref = _reference_order(K, rv)
        assert len(ref) == 3 * (K + 4)
        assert _probe_positions(orc, K, len(ref), rv) == ref
        rng = np.random.default_rng(K + rv)
        d = [rng.integers(0, 2, K + 4, dtype=np.uint8) for _ in range(3)]
        e = orc.rate_match(d, len(ref), rv)
        assert np.array_equal(e, np.array([d[s][n] for s, n in ref], np.uint8))


@pytest.mark.parametrize("K", [40, 512, 6144])
def test_repetition_puncturing_and_bijection(orc, K):
    N = 3 * (K + 4)
    ones = lambda E: np.ones(E, np.int16)  # noqa: E731
    h = orc.rate_dematch(ones(N), K)
    assert all(np.all(x == 1) for x in h)                    # every coded bit exactly once
    E = N * 5 // 2
    h = orc.rate_dematch(ones(E), K, rv=2)
    cnt = np.concatenate(h)
    assert set(np.unique(cnt)) == {2, 3} and cnt.sum() == E
    E = N * 2 // 3
    h = orc.rate_dematch(ones(E), K, rv=1)
    cnt = np.concatenate(h)
    assert (cnt == 0).sum() == N - E and (cnt == 1).sum() == E


def test_harq_combining_and_saturation(orc):
    K, rng = 1056, np.random.default_rng(3)
    N = 3 * (K + 4)
    e1 = rng.integers(-3000, 3001, N // 2).astype(np.int16)
    e2 = rng.integers(-3000, 3001, N).astype(np.int16)
    a = orc.rate_dematch(e1, K, rv=0)
    b = orc.rate_dematch(e2, K, rv=2)
    c = orc.rate_dematch(e2, K, rv=2, h=a)
    for s in range(3):
        assert np.array_equal(c[s], np.clip(a[s].astype(np.int32) + b[s], -32768, 32767).astype(np.int16))
    big = np.full(4 * N, 20000, np.int16)
    h = orc.rate_dematch(big, K)
    assert all(np.all(x == 32767) for x in h)


@pytest.mark.parametrize("K", [40, 1056])
def test_noiseless_rate_half_roundtrip(orc, K):
    rng = np.random.default_rng(K)
    c = orc.crc_attach(orc.CRC24B, rng.integers(0, 2, K - 24, dtype=np.uint8))
    d = orc.turbo_encode(c)
    E = 2 * K                                                # about rate 1/2: parity punctured
    e = orc.rate_match(d, E, rv=0)
    soft = ((2 * e.astype(np.int32) - 1) * 64).astype(np.int16)
    h = orc.rate_dematch(soft, K, rv=0)
    r = orc.decode_cb(*h, max_iters=8, early_term=True)
    assert r["crc_ok"] == 1 and np.array_equal(r["bits"], c)
