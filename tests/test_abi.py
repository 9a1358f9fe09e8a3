"""CPU tests of the C-ABI library: it builds, loads, exports every symbol
include/crn.h declares, its host helpers agree with the oracle, and its decode
entry points refuse to run without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest
import torch

from paper_1905_01141_b200 import build as crn_build
from paper_1905_01141_b200 import crn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    crn_build.build()
    return crn.lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "crn.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(crn_\w+)\s*\(", txt)))


def test_exports_every_declared_symbol(L):
    syms = header_symbols()
    assert len(syms) >= 19
    out = subprocess.check_output(["nm", "-D", "--defined-only", crn.SO]).decode()
    exported = set(re.findall(r"\sT\s(crn_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert hasattr(L, s)


def test_sm100a_sass_present(L):
    out = subprocess.check_output(["cuobjdump", "--list-elf", crn.SO]).decode()
    assert "sm_100a" in out


def test_qpp_table_matches_oracle_copy(L, orc):
    for K in orc.k_table():
        assert crn.qpp_params(K) == orc.qpp_params(K)
        M, W = crn.windows(K)
        assert M == orc.num_windows(K, 32) and M * W == K
    for K in (0, 39, 41, 6145, 520):
        with pytest.raises(crn.CrnError):
            crn.qpp_params(K)


def test_segmentation_and_crc_match_oracle(L, orc):
    rng = np.random.default_rng(0)
    for tbs in list(rng.integers(1, 200000, 300)) + [16, 6120, 6121, 75376]:
        assert crn.segment_tb(int(tbs)) == orc.segment(int(tbs))
    for n in (1, 7, 8, 9, 64, 1000, 6143):
        b = rng.integers(0, 2, n, dtype=np.uint8)
        assert crn.crc24a(b) == orc.crc24a(b) and crn.crc24b(b) == orc.crc24b(b)


def test_tb_build_and_reassemble_match_oracle(L, orc):
    rng = np.random.default_rng(1)
    for tbs in (16, 1000, 4000, 6121, 12000, 75376):
        a = rng.integers(0, 2, tbs, dtype=np.uint8)
        bits, desc = crn.tb_build_cbs(a)
        cbs, Fs, seg = orc.segment_tb_bits(a)
        assert np.array_equal(bits, np.concatenate(cbs))
        assert list(desc["F"]) == Fs and list(desc["K"]) == [c.size for c in cbs]
        # pack LSB-first as the decoder does, then reassemble
        words = np.zeros(int((desc["bit_off"] + (desc["K"] + 31) // 32).max()), np.uint32)
        for d, c in zip(desc, cbs):
            for k, v in enumerate(c):
                words[d["bit_off"] + k // 32] |= np.uint32(int(v) << (k % 32))
        ok = np.ones(desc.size, np.uint8)
        assert np.array_equal(crn.tb_reassemble(words, desc, ok, tbs), a)
        ok[-1] = 0
        assert crn.tb_reassemble(words, desc, ok, tbs) is None


def test_counted_ops_matches_oracle_counter(L, orc):
    rng = np.random.default_rng(2)
    Ks = [40, 528, 1056]
    tot = 0
    for K in Ks:
        ll = [rng.integers(-300, 301, K + 4).astype(np.int16) for _ in range(3)]
        tot += orc.decode_cb(*ll, max_iters=3)["ops"]
    assert crn.counted_ops(Ks, 3) == tot
    assert crn.counted_ops(Ks, 8, iters_used=[3, 3, 3]) == tot


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1905_01141_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "oracle.h" not in txt and "liboracle" not in txt, f


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_decode_refuses_without_gpu(L):
    import ctypes as C
    K = np.array([1056], np.int32)
    rc = L.crn_decode_batch(None, None, None, K.ctypes.data_as(C.POINTER(C.c_int32)), 1, 6, None, None)
    assert rc in (crn.CRN_EINVAL, crn.CRN_ENODEV)
    d = np.zeros(1, crn.DESC_DTYPE)
    d["K"] = 1056
    rc = L.crn_decode_batch_ex(d.ctypes.data, 1, 1, 1, 1, 6, 0, 0, 1, 1, None, None, None, 0, None)
    assert rc == crn.CRN_ENODEV
    assert L.crn_workspace_bytes(None, 100) == 0


def test_tb_verdict_batch_validation():
    """crn_tb_verdict_batch rejects TB tables that do not match 36.212 segmentation
    before touching a device (host-side validation)."""
    import ctypes as C
    tb_bits = np.random.default_rng(1).integers(0, 2, 12000, dtype=np.uint8)
    cbb, desc = crn.tb_build_cbs(tb_bits)
    tbs = np.zeros(1, crn.TB_DTYPE)
    tbs[0] = (0, desc.size, 12000, 0)
    fake = C.c_void_p(16)
    def call(t, d):
        t = np.ascontiguousarray(t, crn.TB_DTYPE)
        d = np.ascontiguousarray(d, crn.DESC_DTYPE)
        return crn.lib().crn_tb_verdict_batch(t.ctypes.data, t.size, d.ctypes.data, d.size, fake, fake, fake,
                                              None, None)
    assert call(tbs, desc) in (crn.CRN_ENODEV, crn.CRN_OK)        # valid (no device here)
    bad = tbs.copy(); bad["tbs"] = 12001
    assert call(bad, desc) == crn.CRN_EINVAL                       # wrong segmentation
    bad = tbs.copy(); bad["n_cb"] = 3
    assert call(bad, desc) == crn.CRN_EINVAL                       # range outside desc
    d2 = desc.copy(); d2["F"][0] += 1
    assert call(tbs, d2) == crn.CRN_EINVAL                         # filler mismatch
    d2 = desc.copy(); d2["crc_kind"][1] = crn.CRC24A
    assert call(tbs, d2) == crn.CRN_EINVAL


def test_new_entry_points_validate_on_host():
    """Argument checks of the runtime, variant and rate-matching entry points run
    before any device access (CRN_EINVAL here, CRN_ENODEV only for valid calls)."""
    import ctypes as C
    L = crn.lib()
    fake = C.c_void_p(16)
    rm = np.zeros(1, crn.RM_DTYPE)
    rm["K"], rm["E"], rm["rv"] = 1056, 3000, 0
    ok = L.crn_rate_dematch_batch(rm.ctypes.data, 1, fake, 0, fake, fake, fake, None)
    assert ok in (crn.CRN_ENODEV, crn.CRN_OK)
    for field, bad in (("K", 1057), ("rv", 4), ("E", 0), ("e_off", -1)):
        b = rm.copy()
        b[field] = bad
        assert L.crn_rate_dematch_batch(b.ctypes.data, 1, fake, 0, fake, fake, fake, None) == crn.CRN_EINVAL
        assert L.crn_rate_match_batch(b.ctypes.data, 1, fake, fake, fake, fake, None) == crn.CRN_EINVAL
    d = np.zeros(1, crn.DESC_DTYPE)
    d["K"], d["crc_kind"] = 1056, crn.CRC24B
    assert L.crn_decode_batch_ex(d.ctypes.data, 1, fake, fake, fake, 8, 3, 0, fake, fake, None, None, None, 0,
                                 None) == crn.CRN_EINVAL                    # unknown stopping rule
    assert L.crn_decode_batch_ex(d.ctypes.data, 1, fake, fake, fake, 8, 1, 8, fake, fake, None, None, None, 0,
                                 None) == crn.CRN_EINVAL                    # unknown flag bit
    tim = (crn.TtiTiming * 1)()
    grp = (crn.TtiGroup * 1)()
    assert L.crn_stream_run_ex(grp, 1, 1, 1000.0, 8, 1, 16, tim) == crn.CRN_EINVAL  # unknown stream flag
    assert L.crn_stream_run_ex(grp, 1, 1, 1000.0, 8, 1, 3 << 8, tim) == crn.CRN_EINVAL   # shift without LLR8
    assert L.crn_stream_run_ex(grp, 1, 1, 1000.0, 8, 1, 8 | (9 << 8), tim) == crn.CRN_EINVAL   # shift > 8
    assert L.crn_stream_run_ex(grp, 1, 1, 1000.0, 8, 1, 8 | 1, tim) == crn.CRN_EINVAL    # int8 + merged
    assert L.crn_stream_run_ex(grp, 1, 1, 1000.0, 8, 1, 8 | 4, tim) == crn.CRN_EINVAL    # int8 + zero copy
    assert L.crn_stream_run_ex(grp, 1, 1, 1000.0, 8, 1, 5, tim) == crn.CRN_EINVAL   # merged + zero copy
    assert L.crn_stream_run_ex(grp, 1, 1, 1000.0, 8, 5, 0, tim) == crn.CRN_EINVAL   # unknown stopping rule


def test_llr_format_validation(L):
    """crn_plan_set_llr_format (row f4 int8 ingest): only a NULL-plan check is
    reachable without a GPU (plans need a device)."""
    assert L.crn_plan_set_llr_format(None, 8, 3) == crn.CRN_EINVAL
    assert L.crn_plan_llr_bytes(None) == crn.CRN_EINVAL


def test_logmap_lut_matches_oracle(L, orc):
    """libcrn's Log-MAP table (its own computation) equals the oracle's."""
    lut = crn.logmap_lut()
    assert [int(x) for x in lut] == [orc.logmap_correction(4 * b) for b in range(8)]
    assert lut[6] == 0 and lut[7] == 0          # the kernel's PRMT zero filler (R32)


def test_kpi_iterations_paper_convention():
    """crn_kpi_iterations follows PAPER.md:411 (Performance captor): the
    registered value is the iteration count of a successful CB and a value
    greater than the maximum for a failure, so the loss rate read from the KPI
    (share of values > max) equals the CRC failure rate."""
    rng = np.random.default_rng(4)
    for I in (1, 6, 8, 32):
        it = rng.integers(1, I + 1, 1000).astype(np.uint8)
        ok = (rng.random(1000) < 0.8).astype(np.uint8)
        k = crn.kpi_iterations(it, ok, I)
        assert np.array_equal(k[ok == 1], it[ok == 1])
        assert np.all(k[ok == 0] == I + 1) and np.all(k <= I + 1)
        assert int((k > I).sum()) == int((ok == 0).sum())
    assert crn.kpi_iterations([], [], 8).size == 0
    L = crn.lib()
    z = np.zeros(1, np.uint8)
    p = z.ctypes.data_as(C.POINTER(C.c_uint8))
    assert L.crn_kpi_iterations(p, p, 1, 0, p) == crn.CRN_EINVAL
    assert L.crn_kpi_iterations(p, p, 1, 33, p) == crn.CRN_EINVAL
    assert L.crn_kpi_iterations(None, p, 1, 8, p) == crn.CRN_EINVAL
    assert L.crn_kpi_iterations(p, p, -1, 8, p) == crn.CRN_EINVAL


def test_stream_run_binding_refuses_mismatched_llr_dtypes():
    """The binding checks the LLR dtype against CRN_STREAM_LLR8 before the C call
    (the runtime would copy n_llr elements of the flag's width), the three
    streams' lengths and the output dtypes."""
    d = np.zeros(1, crn.DESC_DTYPE)
    d["K"] = 40

    def grp(dt, n=(44, 44, 44)):
        return dict(desc=d, l0=torch.zeros(n[0], dtype=dt), l1=torch.zeros(n[1], dtype=dt),
                    l2=torch.zeros(n[2], dtype=dt), bits=torch.zeros(2, dtype=torch.int32),
                    ok=torch.zeros(1, dtype=torch.uint8), it=None)
    with pytest.raises(crn.CrnError):
        crn.stream_run([grp(torch.int8)], 1, 1, 1000.0, 8, True, flags=0)
    with pytest.raises(crn.CrnError):
        crn.stream_run([grp(torch.int16)], 1, 1, 1000.0, 8, True, flags=crn.STREAM_LLR8)
    with pytest.raises(crn.CrnError):
        crn.stream_run([grp(torch.int16, (44, 44, 40))], 1, 1, 1000.0, 8, True, flags=0)
    g = grp(torch.int16)
    g["bits"] = torch.zeros(2, dtype=torch.int64)
    with pytest.raises(crn.CrnError):
        crn.stream_run([g], 1, 1, 1000.0, 8, True, flags=0)


def _dense_desc(Ks):
    K = np.asarray(Ks, np.int64)
    d = np.zeros(K.size, crn.DESC_DTYPE)
    d["K"] = K
    d["crc_kind"] = crn.CRC24B
    d["llr_off"] = np.concatenate([[0], np.cumsum(K + 4)[:-1]])
    d["bit_off"] = np.concatenate([[0], np.cumsum((K + 31) // 32)[:-1]])
    d["ext_off"] = np.concatenate([[0], np.cumsum(K)[:-1]])
    return d


@pytest.mark.timeout(120)
def test_task_layout_invariants(L):
    """Row a1 on the host (crn_task_layout, no GPU): every CB in exactly one task,
    at most two CBs of one K per pair, tasks within their window / sum-K budget
    (whole-CTA: <= 192 windows, sum K <= 6144; group tasks: W = 32, <= 64
    windows, sum K <= 2048), group tasks after every whole-CTA task, the units
    formula, and termination of the small-batch spreading for every batch shape
    (np = 16, per = 4 once looped forever: floor((np + cur) / (cur + 1)) = per)."""
    rng = np.random.default_rng(5)
    import oracle
    Ktab = [int(k) for k in oracle.k_table()]
    cases = [[1056] * 32, [1056] * 33, [64] * 500, [6144] * 5, [40] * 1000, [2048] * 7 + [512] * 9,
             list(rng.choice(Ktab, 200)), list(rng.choice(Ktab, 3000)), [1024] * 31 + [6144] * 300]
    cases += [[int(k)] * int(n) for k, n in zip(rng.choice(Ktab, 40), rng.integers(1, 400, 40))]
    for Ks in cases:
        d = _dense_desc(Ks)
        units0 = None
        for spread in (0, 1, 7, 148, 1000):
            tof, info, units = crn.task_layout(d, spread)
            units0 = units if units0 is None else units0
            nt = info.shape[0]
            assert tof.min() >= 0 and tof.max() < nt
            K = d["K"]
            cnt = np.bincount(tof, minlength=nt)
            assert np.all(cnt >= 1) and np.all(cnt <= 2 * info[:, 1])
            for t in range(nt):                                  # one K per task
                assert np.all(K[tof == t] == info[t, 0])
            W32 = (info[:, 0] % 32 == 0) & (info[:, 0] >= 64)
            grp = info[:, 3] == 1
            assert np.all(W32[grp]) and np.all(info[grp, 2] <= 64) and np.all(info[grp, 0] * info[grp, 1] <= 2048)
            assert np.all(info[~grp, 2] <= 192) and np.all(info[~grp, 0] * info[~grp, 1] <= 6144)
            if grp.any():
                assert np.all(grp[np.argmax(grp):]), "group tasks must come last"
            assert units == int((~grp).sum()) + (int(grp.sum()) + 2) // 3
            assert units <= max(spread, units0)                   # spreading stays within spread_to CTAs
