"""Pins of the oracle's decoder variants, CPU only:
the scaled-extrinsic max-log-MAP (R28: the extrinsic each SISO
hands on is floor(3 Le / 4)) and the paper's average-MI stopping rule
(R29).  Scaled variant:

* the scaling map against the definition of the floor (4 s <= 3x < 4 s + 4);
* one iteration equals the composition of the brute-force-pinned SISO
  (tests/test_oracle_encoder_siso.py) with that map and the QPP permutation;
* noiseless round trips, zero-evidence failure, int16 safety, ET prefix;
* the known behaviour of scaling max-log-MAP extrinsics (it offsets the
  max-log over-estimate): fewer block errors and iterations at the same Eb/N0.
MI rule: its table against the definition of binary entropy (via a second
closed form) and special values; libcrn's independent table equals it; the
rule never stops at iteration 1, stops at 2 when the statistic is saturated
(noiseless) or identically 0 (no evidence); an MI-stopped run is a prefix of
the fixed-iteration run.
"""
import numpy as np
import pytest

from paper_1905_01141_b200 import workload as wlmod
from tests._inputs import offsets, oracle_llrs


def test_ext_scale_is_floor_of_three_quarters(orc):
    xs = np.arange(-4096, 4097)
    s = np.array([orc.ext_scale(int(x)) for x in xs])
    assert np.all(4 * s <= 3 * xs) and np.all(3 * xs < 4 * s + 4)     # s = floor(3x/4) by definition
    assert np.all(np.diff(s) >= 0) and s[0] == -3072 and s[-1] == 3072
    assert [orc.ext_scale(x) for x in (-1, 0, 1, 2, -2)] == [-1, 0, 0, 1, -2]


@pytest.mark.parametrize("K", [40, 1056])
def test_one_iteration_is_composition_of_pinned_parts(orc, K):
    """DEC1 -> scale -> interleave -> DEC2 -> scale -> de-interleave."""
    rng = np.random.default_rng(K)
    d = [rng.integers(-5000, 5001, K + 4).astype(np.int16) for _ in range(3)]
    r = orc.decode_cb(*d, max_iters=1, variant=orc.VAR_SCALED)
    W = K // orc.num_windows(K)
    cl = [np.clip(x.astype(np.int32), -4096, 4096) for x in d]
    Ls, Lp1, Lp2 = cl[0][:K], cl[1][:K], cl[2][:K]
    t1 = [cl[0][K], cl[1][K], cl[2][K], cl[0][K + 1], cl[1][K + 1], cl[2][K + 1]]
    t2 = [cl[0][K + 2], cl[1][K + 2], cl[2][K + 2], cl[0][K + 3], cl[1][K + 3], cl[2][K + 3]]
    Pi = orc.qpp_perm(K)
    sc = np.vectorize(orc.ext_scale)
    le1 = sc(orc.siso(Ls, Lp1, np.zeros(K), t1, W)[0])
    le2 = sc(orc.siso(Ls[Pi], Lp2, le1[Pi], t2, W)[0])
    la1n = np.zeros(K, np.int64)
    la1n[Pi] = le2
    assert np.array_equal(r["ext"].astype(np.int64), la1n)
    lapp = Ls + le1 + la1n
    assert np.array_equal(r["bits"], (lapp >= 0).astype(np.uint8))


def _noiseless(orc, c, amp):
    return [((2 * x.astype(np.int32) - 1) * amp).astype(np.int16) for x in orc.turbo_encode(c)]


@pytest.mark.parametrize("K", [40, 104, 1056, 6144])
def test_scaled_noiseless_zero_and_range(orc, K):
    rng = np.random.default_rng(K + 1)
    c = orc.crc_attach(orc.CRC24B, rng.integers(0, 2, K - 24, dtype=np.uint8))
    for amp in (4096, 8):
        r = orc.decode_cb(*_noiseless(orc, c, amp), max_iters=8, early_term=True, variant=orc.VAR_SCALED)
        assert np.array_equal(r["bits"], c) and r["crc_ok"] == 1 and r["violations"] == 0
    z = [np.zeros(K + 4, np.int16)] * 3
    r = orc.decode_cb(*z, max_iters=4, early_term=True, variant=orc.VAR_SCALED)
    assert r["crc_ok"] == 0 and r["iters"] == 4 and np.all(r["bits"] == 1)
    ll = [rng.integers(-32768, 32768, K + 4).astype(np.int16) for _ in range(3)]
    r = orc.decode_cb(*ll, max_iters=4, variant=orc.VAR_SCALED)
    assert r["violations"] == 0 and np.all(np.abs(r["ext"]) <= 3072)


def test_scaled_et_is_prefix_of_fixed(orc):
    wl = wlmod.make_workload(5, seed=4)
    cbs, ll = oracle_llrs(wl)
    lo, _ = offsets([cb["K"] for cb in cbs])
    for cb, o in list(zip(cbs, lo))[:60]:
        K = cb["K"]
        x = [t[o:o + K + 4].numpy() for t in ll]
        r = orc.decode_cb(*x, F=cb["F"], crc_kind=cb["crc"], max_iters=8, early_term=True, variant=orc.VAR_SCALED)
        f = orc.decode_cb(*x, F=cb["F"], crc_kind=cb["crc"], max_iters=r["iters"], variant=orc.VAR_SCALED)
        assert np.array_equal(r["bits"], f["bits"]) and np.array_equal(r["ext"], f["ext"])


def test_scaling_lowers_bler_and_iterations(orc):
    """128 CBs of K=1056 at Eb/N0 = 0.9 dB, CRC ET at max 8 (seeded)."""
    wl = wlmod.make_workload(1, seed=5, scale=4.0)
    wl.tb_ebn0_db[:] = 0.9
    cbs, ll = oracle_llrs(wl)
    K = np.array([c["K"] for c in cbs], np.int32)
    lo, bo = offsets(K)
    res = []
    for v in (orc.VAR_MAXLOG, orc.VAR_SCALED):
        r = orc.decode_batch(K, np.zeros_like(K), np.full_like(K, 2), lo, bo, *(x.numpy() for x in ll),
                             max_iters=8, early_term=True, nthreads=4, variant=v, want_ext=False)
        res.append((1 - r["crc_ok"].mean(), r["iters"].mean()))
    assert res[1][0] < res[0][0] and res[1][1] < res[0][1], res


# ---------------------------------------------------------------- MI stopping rule (R29)
def test_mi_table_pins(orc):
    """Q16 MI of a consistent LLR of magnitude a/8: I(0) = 0 exactly (a fair coin
    carries no information), nondecreasing, saturating at 1, and equal (to one
    Q16 unit) to the identity I(L) = 1 - log2(1 + e^L) + (L / ln 2) e^L / (1 + e^L),
    a different closed form of 1 - Hb(1 / (1 + e^L))."""
    import math
    t = np.array([orc.mi_table(a) for a in range(256)])
    assert t[0] == 0 and t[255] == 65536 and np.all(np.diff(t) >= 0)
    assert orc.mi_table(1000) == t[255] and orc.mi_table(-1) == -1
    for a in range(256):
        L = a / 8.0
        alt = 1.0 - math.log2(1.0 + math.exp(L)) + (L / math.log(2.0)) * math.exp(L) / (1.0 + math.exp(L))
        assert abs(t[a] - 65536.0 * alt) <= 1.0, a
    # I(L) for L = 1 (a = 8): 1 - Hb(0.268941...) = 0.16007...
    assert abs(t[8] / 65536.0 - 0.16007) < 1e-4


def test_mi_table_product_equals_oracle(orc):
    """libcrn computes the same table independently (crn_mi_table, host side)."""
    from paper_1905_01141_b200 import crn
    assert np.array_equal(crn.mi_table(), np.array([orc.mi_table(a) for a in range(256)], np.int32))


def test_mi_stop_special_cases(orc):
    rng = np.random.default_rng(7)
    for K in (40, 1056):
        c = orc.crc_attach(orc.CRC24B, rng.integers(0, 2, K - 24, dtype=np.uint8))
        r = orc.decode_cb(*_noiseless(orc, c, 4096), max_iters=8, early_term=orc.ET_MI)
        assert r["iters"] == 2 and r["crc_ok"] == 1 and np.array_equal(r["bits"], c)   # saturated from t=1
        z = [np.zeros(K + 4, np.int16)] * 3
        r = orc.decode_cb(*z, max_iters=8, early_term=orc.ET_MI)
        assert r["iters"] == 2 and r["crc_ok"] == 0          # the MI stays 0: converged, CB lost
        r = orc.decode_cb(*z, max_iters=1, early_term=orc.ET_MI)
        assert r["iters"] == 1


def test_mi_stop_is_prefix_of_fixed(orc):
    wl = wlmod.make_workload(5, seed=6)
    cbs, ll = oracle_llrs(wl)
    lo, _ = offsets([cb["K"] for cb in cbs])
    its = []
    for cb, o in list(zip(cbs, lo))[:60]:
        K = cb["K"]
        x = [t[o:o + K + 4].numpy() for t in ll]
        r = orc.decode_cb(*x, F=cb["F"], crc_kind=cb["crc"], max_iters=8, early_term=orc.ET_MI)
        f = orc.decode_cb(*x, F=cb["F"], crc_kind=cb["crc"], max_iters=r["iters"])
        assert np.array_equal(r["bits"], f["bits"]) and np.array_equal(r["ext"], f["ext"])
        assert r["crc_ok"] == f["crc_ok"] and r["iters"] >= 2
        its.append(r["iters"])
    assert min(its) < 8                                       # it does stop early somewhere


# ---------------------------------------------------------------- Log-MAP (R32)
# max*(a, b) = max(a, b) + LUT[min(|a-b| >> 2, 7)], values in 1/8 nat.  Pinned against
# the exact Jacobian logarithm 8 ln(e^(a/8) + e^(b/8)) -- not against the table --
# and, at SISO level, against exact MAP (log-sum-exp over every path by brute force).
LOGMAP_EPS = 0.82     # max |LUT bucket value - 8 ln(1 + e^(-d/8))| over d >= 0 (bucket 0 at d = 3)


def test_max_star_is_jacobian_log_within_table_error(orc):
    a = np.arange(-200, 201, 3)
    for x in a:
        for y in (-211, -40, -9, -3, 0, 1, 2, 5, 13, 31, 32, 77, 200):
            m = orc.max_star(int(x), int(y))
            exact = 8 * np.logaddexp(x / 8, y / 8)
            assert abs(m - exact) <= LOGMAP_EPS, (x, y, m, exact)
            assert m == orc.max_star(int(y), int(x))                       # symmetric
            assert orc.max_star(int(x) + 17, int(y) + 17) == m + 17       # shift-invariant
            assert m >= max(x, y)
    # far apart the correction vanishes: max* = max (the max-log-MAP limit)
    assert all(orc.max_star(d, 0) == d for d in range(32, 400, 7))
    assert orc.logmap_correction(0) == 5 and orc.logmap_correction(-1) == -1


def _exact_map_le(lsys, lpar, la, tail):
    """Exact APP extrinsics (float64) of one terminated constituent by enumerating paths."""
    from tests.test_oracle_encoder_siso import rsc_paths
    n = lsys.size
    U, Z, TX, TZ, S = rsc_paths(n)
    Lu = lsys + la
    tot = (U * Lu + Z * lpar).sum(1) + TX @ tail[0::2] + TZ @ tail[1::2]
    lse = lambda v: np.logaddexp.reduce(v / 8.0) * 8.0
    return np.array([lse(tot[U[:, k] == 1]) - lse(tot[U[:, k] == 0]) - Lu[k] for k in range(n)])


@pytest.mark.parametrize("n", [8, 11, 13])
def test_logmap_siso_is_exact_map_within_bound(orc, n):
    """Every Le of the Log-MAP SISO is within the accumulated table error of exact
    MAP (alpha chain + beta chain + the 7-term Lambda fold, both Lambdas), and on
    average far closer to it than max-log-MAP is (a missing or wrong-signed
    correction fails this)."""
    rng = np.random.default_rng(7 + n)
    bound = 2 * (n + 7) * LOGMAP_EPS + 1
    err_log, err_max = [], []
    for _ in range(12):
        lsys, lpar, la = (rng.integers(-40, 41, n) for _ in range(3))
        tail = rng.integers(-40, 41, 6)
        ex = _exact_map_le(lsys, lpar, la, tail)
        le_l, _, _, _, v = orc.siso(lsys, lpar, la, tail, n, variant=orc.VAR_LOGMAP)
        le_m = orc.siso(lsys, lpar, la, tail, n)[0]
        assert v == 0
        assert np.all(np.abs(le_l - ex) <= bound), np.abs(le_l - ex).max()
        err_log.append(np.abs(le_l - ex).mean())
        err_max.append(np.abs(le_m - ex).mean())
    assert np.mean(err_log) < 0.4 * np.mean(err_max), (np.mean(err_log), np.mean(err_max))


def test_logmap_zero_evidence_and_noiseless(orc):
    """No evidence: Le = 0 everywhere by symmetry of max*; noiseless (+-800 LLRs):
    every selection is decided by >= 32 units, so Log-MAP = max-log-MAP."""
    for n in (9, 12):
        z = np.zeros(n, np.int64)
        assert np.all(orc.siso(z, z, z, np.zeros(6, np.int64), n, variant=orc.VAR_LOGMAP)[0] == 0)
    c = np.random.default_rng(3).integers(0, 2, 40).astype(np.uint8)
    d = [800 * (2 * x.astype(np.int16) - 1) for x in orc.turbo_encode(c)]
    a = orc.decode_cb(*d, F=0, crc_kind=0, max_iters=3, variant=orc.VAR_LOGMAP)
    b = orc.decode_cb(*d, F=0, crc_kind=0, max_iters=3)
    assert np.array_equal(a["bits"], c) and np.array_equal(a["ext"], b["ext"])


def test_logmap_lowers_bler_and_iterations(orc):
    """Same seeded CBs as the scaled-variant pin: Log-MAP decodes at least as many
    and stops earlier on average than max-log-MAP (its known gain)."""
    wl = wlmod.make_workload(1, seed=5, scale=4.0)
    wl.tb_ebn0_db[:] = 0.9
    cbs, ll = oracle_llrs(wl)
    K = np.array([c["K"] for c in cbs], np.int32)
    lo, bo = offsets(K)
    res = []
    for v in (orc.VAR_MAXLOG, orc.VAR_LOGMAP):
        r = orc.decode_batch(K, np.zeros_like(K), np.full_like(K, 2), lo, bo, *(x.numpy() for x in ll),
                             max_iters=8, early_term=True, nthreads=4, variant=v, want_ext=False)
        assert r["violations"] == 0
        res.append((1 - r["crc_ok"].mean(), r["iters"].mean()))
    assert res[1][0] < res[0][0] and res[1][1] < res[0][1], res
