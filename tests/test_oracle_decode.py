"""Pins of the oracle's iterative decoder: noiseless round
trip, zero-evidence failure (tie rule R16), ET prefix
consistency, exact-ML agreement at K=40 by branch-and-bound, BLER monotone in
Eb/N0, int16 range safety, determinism, TB round trip.  CPU only."""
import numpy as np
import pytest

from paper_1905_01141_b200 import workload as wlmod
from tests._inputs import offsets, oracle_llrs


def noiseless(orc, c, amp=4096):
    return [((2 * x.astype(np.int32) - 1) * amp).astype(np.int16) for x in orc.turbo_encode(c)]


@pytest.mark.parametrize("K", [40, 56, 104, 248, 1056, 2112, 6144])
def test_noiseless_roundtrip(orc, K):
    rng = np.random.default_rng(K)
    for amp in (4096, 8192, 3):
        c = orc.crc_attach(orc.CRC24B, rng.integers(0, 2, K - 24, dtype=np.uint8))
        r = orc.decode_cb(*noiseless(orc, c, amp), max_iters=8, early_term=True)
        assert r["violations"] == 0
        assert np.array_equal(r["bits"], c) and r["crc_ok"] == 1 and r["iters"] <= 2


@pytest.mark.parametrize("tbs", [1000, 4000, 6121, 12000])
def test_noiseless_fillers(orc, tbs):
    rng = np.random.default_rng(tbs)
    cbs, Fs, seg = orc.segment_tb_bits(rng.integers(0, 2, tbs, dtype=np.uint8))
    kind = orc.CRC24A if seg["C"] == 1 else orc.CRC24B
    out = []
    for c, F in zip(cbs, Fs):
        r = orc.decode_cb(*noiseless(orc, c, 40), F=F, crc_kind=kind, max_iters=8, early_term=True)
        assert r["crc_ok"] == 1 and np.array_equal(r["bits"], c) and np.all(r["bits"][:F] == 0)
        out.append(r["bits"])
    assert orc.reassemble_tb(out, Fs, seg) is not None


@pytest.mark.parametrize("K,F,kind", [(40, 0, 2), (1056, 0, 2), (4032, 8, 1), (6144, 0, 1)])
def test_zero_llrs_fail_at_max(orc, K, F, kind):
    z = [np.zeros(K + 4, np.int16)] * 3
    for et in (False, True):
        r = orc.decode_cb(*z, F=F, crc_kind=kind, max_iters=5, early_term=et)
        assert r["crc_ok"] == 0 and r["iters"] == 5
        assert np.all(r["bits"][F:] == 1) and np.all(r["bits"][:F] == 0)   # tie -> 1 (R16)
        assert np.all(r["ext"] == 0)


def test_fixed_iteration_op_count(orc):
    rng = np.random.default_rng(0)
    for K in (40, 528, 1056):
        ll = [rng.integers(-8192, 8193, K + 4).astype(np.int16) for _ in range(3)]
        for I in (1, 3):
            r = orc.decode_cb(*ll, max_iters=I)
            assert r["ops"] == 2 * I * (129 * K + 90)


def test_int16_range_adversarial(orc):
    """Every intermediate stays in int16 (DESIGN.md int16 safety) for arbitrary,
    saturated and out-of-range inputs."""
    rng = np.random.default_rng(1)
    for K in (40, 64, 1056, 6144):
        for lim in (8192, 32767, 200):
            ll = [rng.integers(-lim, lim + 1, K + 4).astype(np.int16) for _ in range(3)]
            r = orc.decode_cb(*ll, F=min(8, K - 25), max_iters=4)
            assert r["violations"] == 0
            assert np.all(np.abs(r["ext"]) <= 4096)
        ll = [np.full(K + 4, s, np.int16) for s in (32767, -32768, 32767)]
        assert orc.decode_cb(*ll, max_iters=3)["violations"] == 0


def test_early_termination_is_prefix_of_fixed(orc):
    wl = wlmod.make_workload(5, seed=3, scale=1.0)
    cbs, (l0, l1, l2) = oracle_llrs(wl)
    lo, _ = offsets([cb["K"] for cb in cbs])
    n = 0
    for cb, o in zip(cbs, lo):
        K = cb["K"]
        ll = [x[o:o + K + 4].numpy() for x in (l0, l1, l2)]
        r = orc.decode_cb(*ll, F=cb["F"], crc_kind=cb["crc"], max_iters=8, early_term=True)
        f = orc.decode_cb(*ll, F=cb["F"], crc_kind=cb["crc"], max_iters=r["iters"], early_term=False)
        assert f["crc_ok"] == r["crc_ok"] and f["iters"] == r["iters"]
        assert np.array_equal(f["bits"], r["bits"]) and np.array_equal(f["ext"], r["ext"])
        n += r["crc_ok"]
        if r["crc_ok"]:
            assert np.array_equal(r["bits"], cb["c"])
    assert n > 0


def test_ber_bler_monotone_in_ebn0(orc):
    rng = np.random.default_rng(9)
    K, n = 104, 150
    bler = []
    for ebn0 in (0.0, 1.5, 3.0):
        fails = 0
        for _ in range(n):
            c = orc.crc_attach(orc.CRC24B, rng.integers(0, 2, K - 24, dtype=np.uint8))
            a, s2 = wlmod.noise_sigma2(np.array([K]), np.array([ebn0]), "bpsk")
            ll = []
            for x in orc.turbo_encode(c):
                y = (1 - 2.0 * x) + np.sqrt(s2[0]) * rng.standard_normal(x.size)
                ll.append(np.clip(np.sign(-2 * y / s2[0]) * np.floor(np.abs(16 * y / s2[0]) + .5),
                                  -8192, 8192).astype(np.int16))
            r = orc.decode_cb(*ll, max_iters=8, early_term=True)
            fails += int(not (r["crc_ok"] and np.array_equal(r["bits"], c)))
        bler.append(fails / n)
    assert bler[0] >= bler[1] >= bler[2] and bler[0] > bler[2]


def test_batch_determinism_threads(orc):
    wl = wlmod.make_workload(5, seed=1)
    cbs, ll = oracle_llrs(wl)
    K = np.array([cb["K"] for cb in cbs])
    lo, bo = offsets(K)
    args = (K, [cb["F"] for cb in cbs], [cb["crc"] for cb in cbs], lo, bo, *(x.numpy() for x in ll))
    a = orc.decode_batch(*args, max_iters=8, early_term=True, nthreads=1)
    b = orc.decode_batch(*args, max_iters=8, early_term=True, nthreads=4)
    for k in ("bits", "crc_ok", "iters", "ext"):
        assert np.array_equal(a[k], b[k])
    assert a["ops"] == b["ops"] and a["violations"] == 0
    # batch == per-CB
    for i in (0, 7, len(cbs) - 1):
        r = orc.decode_cb(*(x.numpy()[lo[i]:lo[i] + K[i] + 4] for x in ll), F=cbs[i]["F"],
                          crc_kind=cbs[i]["crc"], max_iters=8, early_term=True)
        assert np.array_equal(r["bits"], a["bits"][bo[i]:bo[i] + K[i]])


# ------------------------------------------------------------------ exact ML at K=40
def _ml_branch_and_bound(orc, L0, L1, L2, K=40):
    """Exact ML info word of the terminated turbo code: maximise sum_n L_n (2b_n-1)/2
    (equivalently sum over coded 1-bits of L) by breadth-first branch and bound with
    the admissible bound partial + sum |L| over undetermined coded bits."""
    pi = orc.qpp_perm(K)
    L0, L1, L2 = (np.asarray(x, np.int64) for x in (L0, L1, L2))
    # value of coded bit b at LLR L: b*L (positive => 1); optimistic bound max(L, 0)
    pos = lambda L: np.maximum(L, 0)
    p2 = [0] * (K + 1)          # d2 prefix length decided once info bits < m are known
    for m in range(K + 1):
        p = 0
        while p < K and pi[p] < m:
            p += 1
        p2[m] = p
    tail_opt = int(pos(np.r_[L0[K:], L1[K:], L2[K:]]).sum())
    rem = [int(pos(L0[m:K]).sum() + pos(L1[m:K]).sum() + pos(L2[p2[m]:K]).sum()) + tail_opt
           for m in range(K + 1)]

    def rsc_step(s, u):
        r1, r2, r3 = (s >> 2) & 1, (s >> 1) & 1, s & 1
        a = u ^ r2 ^ r3
        return (a << 2) | (r1 << 1) | r2, a ^ r1 ^ r3

    # incumbent: the transmitted-like guess from the oracle decoder (any codeword works)
    best = -10**18
    frontier = [(0, 0, 0, 0)]   # (bits as int, rsc1 state, rsc2 state, partial metric)
    inc = _INCUMBENT[0]
    if inc is not None:
        best = inc
    for m in range(K):
        nxt = []
        for bits, s1, s2, val in frontier:
            for u in (0, 1):
                b2 = bits | (u << m)
                n1, z1 = rsc_step(s1, u)
                v = val + u * L0[m] + z1 * L1[m]
                n2 = s2
                for i in range(p2[m], p2[m + 1]):
                    ui = (b2 >> int(pi[i])) & 1
                    n2, zz = rsc_step(n2, ui)
                    v += zz * L2[i]
                if v + rem[m + 1] >= best:
                    nxt.append((b2, n1, n2, v))
        frontier = nxt
    res = None
    for bits, s1, s2, v in frontier:
        # tails (R11 layout)
        tl = []
        for s in (s1, s2):
            xs, zs = [], []
            for _ in range(3):
                r1, r2, r3 = (s >> 2) & 1, (s >> 1) & 1, s & 1
                xs.append(r2 ^ r3)
                zs.append(r1 ^ r3)
                s = (r1 << 1) | r2
            tl += [xs[0], zs[0], xs[1], zs[1], xs[2], zs[2]]
        Lt = [L0[K], L1[K], L2[K], L0[K + 1], L1[K + 1], L2[K + 1],
              L0[K + 2], L1[K + 2], L2[K + 2], L0[K + 3], L1[K + 3], L2[K + 3]]
        v += sum(int(a) * int(b) for a, b in zip(tl, Lt))
        if v > best or (res is None and v >= best):
            best, res = v, bits
    return res, best


_INCUMBENT = [None]


def _metric(orc, c, L):
    return sum(int((d.astype(np.int64) * l).sum()) for d, l in zip(orc.turbo_encode(c), L))


def test_k40_high_snr_equals_exact_ml(orc):
    rng = np.random.default_rng(40)
    K, agree, total = 40, 0, 0
    for _ in range(6):
        c = orc.crc_attach(orc.CRC24B, rng.integers(0, 2, K - 24, dtype=np.uint8))
        a, s2 = wlmod.noise_sigma2(np.array([K]), np.array([4.0]), "bpsk")
        L = []
        for x in orc.turbo_encode(c):
            y = (1 - 2.0 * x) + np.sqrt(s2[0]) * rng.standard_normal(x.size)
            L.append(np.clip(np.round(-16 * y / s2[0]), -8192, 8192).astype(np.int16))
        r = orc.decode_cb(*L, max_iters=8)
        _INCUMBENT[0] = _metric(orc, r["bits"], L)
        ml, _ = _ml_branch_and_bound(orc, *L)
        total += 1
        mlbits = np.array([(ml >> i) & 1 for i in range(K)], np.uint8)
        agree += int(np.array_equal(mlbits, r["bits"]))
        assert np.array_equal(mlbits, c)           # at 4 dB the ML word is the transmitted one
    assert agree == total
