"""GPU parity: libcrn (CUDA, sm_100a) vs the CPU oracle, bit-exact on packed
hard decisions, int16 extrinsics, iteration counts and CRC flags, for every
BASELINE config (every CB of cfg3 and cfg4 at full size) and the edge cases."""
import numpy as np
import pytest
import torch

from paper_1905_01141_b200 import batch as bmod
from paper_1905_01141_b200 import build as crn_build
from paper_1905_01141_b200 import crn
from paper_1905_01141_b200 import workload as wlmod
from tests._gpu import assert_parity, run_gpu, run_oracle, unpack
from tests._inputs import oracle_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    crn_build.build()
    crn.lib()
    assert torch.cuda.is_available()


def _full(cfg, scale=1.0, seed=0, cells=None):
    """Parity inputs: the oracle's CBs and coded bits on the shared channel."""
    wl = wlmod.make_workload(cfg, seed=seed, device="cuda", scale=scale, cells=cells)
    return oracle_batch(wl)


def _full_gpu_encoded(cfg, scale=1.0, seed=0):
    """The product's own batch assembly (libcrn segmentation + GPU encoder), for
    the tests of that assembly against the oracle."""
    wl = wlmod.make_workload(cfg, seed=seed, device="cuda", scale=scale)
    return bmod.build(wl)


def test_encoder_matches_oracle(orc):
    for cfg, scale in ((1, 1.0), (2, 1.0), (3, 0.2), (5, 1.0)):
        b = _full_gpu_encoded(cfg, scale)
        info = b.info.cpu().numpy()
        coded = [x.cpu().numpy() for x in b.coded]
        for i in range(b.n_cb):
            d = b.desc[i]
            c = info[d["ext_off"]:d["ext_off"] + d["K"]].copy()
            if b.wl.tb_kind == "cb":
                c = orc.crc_attach(orc.CRC24B, c[:-24])
            e = orc.turbo_encode(c)
            for s in range(3):
                assert np.array_equal(coded[s][d["llr_off"]:d["llr_off"] + d["K"] + 4], e[s]), (cfg, i, s)


@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (2, 1.0), (3, 0.2), (5, 1.0)])
def test_product_batch_equals_oracle_batch(orc, cfg, scale):
    """The product's batch assembly (libcrn segmentation / CRC / fillers, GPU
    encoder) produces exactly the oracle's CBs, layout, coded bits and LLRs."""
    p = _full_gpu_encoded(cfg, scale)
    o = _full(cfg, scale)
    for f in ("K", "F", "crc_kind", "llr_off", "bit_off", "ext_off"):
        assert np.array_equal(p.desc[f], o.desc[f]), f
    pi, oi = p.info.cpu().numpy(), o.info.cpu().numpy()
    if p.wl.tb_kind == "cb":                     # the product attaches the CRC24B while encoding
        keep = np.ones(pi.size, bool)
        for d in p.desc:
            keep[d["ext_off"] + d["K"] - 24:d["ext_off"] + d["K"]] = False
        assert np.array_equal(pi[keep], oi[keep])
    else:
        assert np.array_equal(pi, oi)
    for x, y in zip(p.coded + p.llr, o.coded + o.llr):
        assert torch.equal(x, y)


@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (2, 1.0), (3, 1.0), (5, 1.0)])
def test_config_parity_full(orc, cfg, scale):
    """BASELINE configs 1, 2, 3 (the whole pooled TTI: 1,000 TBs, ~6,700 CBs of
    mixed K with fillers) and 5 (one TTI) at full size: every CB, every output."""
    b = _full(cfg, scale)
    I, et = b.wl.max_iters, b.wl.early_term
    g = run_gpu(b, I, et)
    idx = np.arange(b.n_cb)
    r = run_oracle(b, idx, I, et)
    assert_parity(b, g, r, idx)


def test_cfg4_full_size_all_cbs(orc):
    """BASELINE cfg 4 at its full size (65,536 CBs, K=6144, 8 fixed iterations) in
    the launch configuration bench.py times (one plan, one persistent launch):
    every CB's bits, int16 extrinsics, CRC flag and iteration count against the
    oracle (about a minute of oracle time on the box's host cores)."""
    b = _full(4)
    assert b.n_cb == 65536
    bits, ok, it, ext = bmod.outputs(b)
    p = crn.Plan(b.desc)
    p.decode(*b.llr, 8, False, bits, ok, it, ext)
    torch.cuda.synchronize()
    g = dict(words=bits.cpu().numpy().view(np.uint32), crc_ok=ok.cpu().numpy()[:b.n_cb],
             iters=it.cpu().numpy()[:b.n_cb], ext=ext.cpu().numpy())
    p.close()
    del bits, ok, it, ext
    idx = np.arange(b.n_cb)
    r = run_oracle(b, idx, 8, False)
    assert_parity(b, g, r, idx)
    assert np.all(g["iters"] == 8)
    assert 0.9 * b.n_cb < int(g["crc_ok"].sum()) < b.n_cb      # 1 dB: a few failures, not all


def _desc_for(K_list, F_list=None, kinds=None):
    K = np.asarray(K_list, np.int64)
    d = np.zeros(K.size, crn.DESC_DTYPE)
    d["K"] = K
    d["F"] = 0 if F_list is None else F_list
    d["crc_kind"] = crn.CRC24B if kinds is None else kinds
    d["llr_off"] = np.concatenate([[0], np.cumsum(K + 4)[:-1]])
    d["bit_off"] = np.concatenate([[0], np.cumsum((K + 31) // 32)[:-1]])
    d["ext_off"] = np.concatenate([[0], np.cumsum(K)[:-1]])
    return d


class _B:
    """A raw batch (descriptor + LLR buffers) not produced by the workload."""

    def __init__(self, desc, llr):
        self.desc, self.llr = desc, llr
        self.n_cb = desc.size
        self.n_words = int((desc["bit_off"] + (desc["K"] + 31) // 32).max())
        self.wl = None


def _random_llr(desc, rng, lim):
    n = int((desc["llr_off"] + desc["K"] + 4).max())
    return tuple(torch.from_numpy(rng.integers(-lim, lim + 1, n).astype(np.int16)).cuda() for _ in range(3))


def _raw_parity(desc, llr, I, et):
    b = _B(desc, llr)
    bits = torch.zeros(b.n_words, dtype=torch.int32, device="cuda")
    ok = torch.zeros(desc.size, dtype=torch.uint8, device="cuda")
    it = torch.zeros(desc.size, dtype=torch.uint8, device="cuda")
    ext = torch.zeros(int(desc["K"].sum()), dtype=torch.int16, device="cuda")
    crn.decode_batch_ex(desc, desc.size, *llr, I, et, 0, bits, ok, it, ext)
    torch.cuda.synchronize()
    g = dict(words=bits.cpu().numpy().view(np.uint32), crc_ok=ok.cpu().numpy(), iters=it.cpu().numpy(),
             ext=ext.cpu().numpy())
    idx = np.arange(desc.size)
    r = run_oracle(b, idx, I, et)
    assert_parity(b, g, r, idx)
    return g


def test_every_k_ragged_and_adversarial(orc):
    """All 188 sizes once (odd buckets -> dummy partner lanes, every window
    length 32..62), random fillers up to K-25, all CRC kinds, saturated and
    out-of-range LLRs (clamp path)."""
    rng = np.random.default_rng(7)
    Ks = orc.k_table()
    F = [int(rng.integers(0, K - 24)) if i % 3 == 0 else 0 for i, K in enumerate(Ks)]
    kinds = [i % 3 for i in range(len(Ks))]
    d = _desc_for(Ks, F, kinds)
    for lim in (300, 32767):
        _raw_parity(d, _random_llr(d, rng, lim), 3, False)


def test_many_small_blocks_multi_pair_tasks(orc):
    rng = np.random.default_rng(8)
    Ks = [40] * 301 + [48] * 7 + [64] * 130 + [1056] * 5
    d = _desc_for(list(rng.permutation(Ks)))
    _raw_parity(d, _random_llr(d, rng, 200), 4, False)


def test_full_multi_pair_tasks_beyond_one_wave(orc):
    """Enough small CBs that the tasks stay fully packed (96 pairs of K=64 per
    task, more tasks than CTAs: no spreading) next to a spread small remainder,
    with early termination."""
    rng = np.random.default_rng(18)
    Ks = [64] * (2 * 96 * 160) + [40] * 97 + [2112] * 3
    d = _desc_for(list(rng.permutation(Ks)))
    _raw_parity(d, _random_llr(d, rng, 60), 6, True)


def test_group_tasks_beyond_one_wave(orc):
    """Group tasks (W = 32, sum K <= 2048: three per CTA, one per four-warp group
    with its own named barrier) well beyond one wave of 3 x 148 group slots,
    behind whole-CTA tasks (K = 6144 pairs and split-path sizes), every group
    geometry from one pair of K = 2048 (64 windows) to 32 pairs of K = 64 and a
    lone K = 1056 (33 windows, a dummy partner lane); early termination, so the
    groups of a CTA finish their tasks at different times."""
    rng = np.random.default_rng(19)
    Ks = ([64] * 640 + [96] * 300 + [512] * 257 + [1024] * 401 + [1056] * 1 + [1088] * 150 + [2048] * 333 +
          [6144] * 61 + [1008] * 20 + [40] * 9)
    d = _desc_for(list(rng.permutation(Ks)))
    llr = _random_llr(d, rng, 70)
    # every third CB leans to the all-zero codeword (CRC 0): it stops after 1-3 iterations, the rest run to 8
    n = int((d["llr_off"] + d["K"] + 4).max())
    lean = np.zeros(n, np.int16)
    for o, K in zip(d["llr_off"][::3], d["K"][::3]):
        lean[o:o + K + 4] = -60 - int(rng.integers(0, 40))
    llr = tuple((x + torch.from_numpy(lean).cuda()).clamp(-32767, 32767) for x in llr)
    g = _raw_parity(d, llr, 8, True)
    assert 0 < int(g["crc_ok"].sum()) < d.size and len(set(g["iters"].tolist())) > 2


def test_iteration_extremes_and_et(orc):
    rng = np.random.default_rng(9)
    d = _desc_for([6144, 6144, 6144, 512, 40])
    llr = _random_llr(d, rng, 100)
    _raw_parity(d, llr, 1, False)
    _raw_parity(d, llr, 32, True)


def test_zero_llrs_fail_at_max(orc):
    d = _desc_for([40, 1056, 6144], [0, 8, 100], [2, 1, 2])
    n = int((d["llr_off"] + d["K"] + 4).max())
    z = tuple(torch.zeros(n, dtype=torch.int16, device="cuda") for _ in range(3))
    g = _raw_parity(d, z, 5, True)
    assert np.all(g["crc_ok"] == 0) and np.all(g["iters"] == 5)


def test_batch_order_and_composition_invariance(orc):
    b = _full(5)
    g = run_gpu(b, 8, True)
    rng = np.random.default_rng(3)
    perm = rng.permutation(b.n_cb)
    d2 = b.desc[perm].copy()
    g2 = run_gpu(b, 8, True, desc=d2)
    for i in range(b.n_cb):
        assert np.array_equal(unpack(g["words"], b.desc, i), unpack(g2["words"], b.desc, i))
    assert np.array_equal(g["crc_ok"][perm], g2["crc_ok"]) and np.array_equal(g["iters"][perm], g2["iters"])
    sub = b.desc[perm[:37]].copy()
    g3 = run_gpu(b, 8, True, desc=sub)
    assert np.array_equal(g3["iters"], g["iters"][perm[:37]])
    g4 = run_gpu(b, 8, True)                                    # run twice: identical
    assert np.array_equal(g4["words"], g["words"]) and np.array_equal(g4["ext"], g["ext"])


def test_plan_simple_api_and_device_descriptors(orc):
    b = _full(1)
    g = run_gpu(b, 6, False)
    # plan API
    bits, ok, it, ext = bmod.outputs(b)
    p = crn.Plan(b.desc)
    assert p.launches == 1
    p.decode(*b.llr, 6, False, bits, ok, it, ext)
    torch.cuda.synchronize()
    assert np.array_equal(bits.cpu().numpy().view(np.uint32), g["words"])
    assert np.array_equal(ext.cpu().numpy(), g["ext"])
    p.close()
    # BASELINE.json form (dense layout, CRC24B, fixed iterations)
    bits2 = torch.zeros_like(bits)
    ok2 = torch.zeros_like(ok)
    crn.decode_batch(*b.llr, b.K, b.n_cb, 6, bits2, ok2)
    torch.cuda.synchronize()
    assert np.array_equal(bits2.cpu().numpy().view(np.uint32), g["words"])
    assert np.array_equal(ok2.cpu().numpy()[:b.n_cb], g["crc_ok"])
    # descriptors in device memory
    dd = torch.from_numpy(b.desc.view(np.uint8).copy()).cuda()
    bits3 = torch.zeros_like(bits)
    crn.decode_batch_ex(dd, b.n_cb, *b.llr, 6, False, crn.DESC_ON_DEVICE, bits3, ok)
    torch.cuda.synchronize()
    assert np.array_equal(bits3.cpu().numpy().view(np.uint32), g["words"])


def test_device_descriptors_bucketed_on_device(orc):
    """CRN_DESC_ON_DEVICE: row a1 runs on the device (crn_tasks.cu) -- a mixed-K
    TTI with CRC early termination through device descriptors equals the oracle
    on every output; invalid descriptors (bad K, F, crc_kind, offsets) are not
    decoded (crc_ok = iters_used = 0) while their neighbours are; a caller
    workspace of exactly crn_workspace_bytes(n_cb) works; host descriptors
    decoded twice (plan cache hit) and a same-size different layout (miss) agree."""
    b = _full(5)
    g = run_gpu(b, 8, True)
    idx = np.arange(b.n_cb)
    r = run_oracle(b, idx, 8, True)
    assert_parity(b, g, r, idx)
    dd = torch.from_numpy(b.desc.view(np.uint8).copy()).cuda()
    bits, ok, it, ext = bmod.outputs(b)
    ws = torch.zeros(crn.workspace_bytes(b.n_cb), dtype=torch.uint8, device="cuda")
    for w in (None, ws):
        bits.zero_(); ok.fill_(7); it.fill_(7); ext.zero_()
        crn.decode_batch_ex(dd, b.n_cb, *b.llr, 8, True, crn.DESC_ON_DEVICE, bits, ok, it, ext,
                            workspace=w, workspace_bytes=0 if w is None else w.numel())
        torch.cuda.synchronize()
        gd = dict(words=bits.cpu().numpy().view(np.uint32), crc_ok=ok.cpu().numpy()[:b.n_cb],
                  iters=it.cpu().numpy()[:b.n_cb], ext=ext.cpu().numpy())
        assert_parity(b, gd, r, idx)
    # invalid descriptors in device memory
    bad = b.desc.copy()
    kill = np.arange(0, b.n_cb, 7)
    for n, i in enumerate(kill):
        if n % 4 == 0: bad["K"][i] = 41
        elif n % 4 == 1: bad["F"][i] = bad["K"][i]
        elif n % 4 == 2: bad["crc_kind"][i] = 3
        else: bad["llr_off"][i] = -1
    dd = torch.from_numpy(bad.view(np.uint8).copy()).cuda()
    bits.zero_(); ok.fill_(7); it.fill_(7)
    crn.decode_batch_ex(dd, b.n_cb, *b.llr, 8, True, crn.DESC_ON_DEVICE, bits, ok, it)
    torch.cuda.synchronize()
    okh, ith = ok.cpu().numpy()[:b.n_cb], it.cpu().numpy()[:b.n_cb]
    assert np.all(okh[kill] == 0) and np.all(ith[kill] == 0)
    keep = np.setdiff1d(idx, kill)
    assert np.array_equal(okh[keep], r["crc_ok"][keep]) and np.array_equal(ith[keep], r["iters"][keep])
    words = bits.cpu().numpy().view(np.uint32)
    for i in keep[::5]:
        assert np.array_equal(unpack(words, b.desc, i), r["bits"][r["bo"][i]:r["bo"][i] + b.desc["K"][i]])
    # host descriptors: a cache hit and a same-size layout change
    g2 = run_gpu(b, 8, True)
    assert np.array_equal(g2["words"], g["words"]) and np.array_equal(g2["iters"], g["iters"])
    perm = np.random.default_rng(4).permutation(b.n_cb)
    d2 = b.desc[perm].copy()
    g3 = run_gpu(b, 8, True, desc=d2)
    assert np.array_equal(g3["iters"], g["iters"][perm]) and np.array_equal(g3["crc_ok"], g["crc_ok"][perm])


def test_streams_and_invalid_args(orc):
    b = _full(5)
    g = run_gpu(b, 8, True)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        g2 = run_gpu(b, 8, True, stream=s)
    assert np.array_equal(g["words"], g2["words"])
    bits, ok, it, ext = bmod.outputs(b)
    bad = b.desc.copy()
    bad["K"][0] = 41
    with pytest.raises(crn.CrnError):
        crn.decode_batch_ex(bad, bad.size, *b.llr, 8, True, 0, bits, ok)
    bad = b.desc.copy()
    bad["llr_off"][1] = bad["llr_off"][0]          # overlapping inputs
    with pytest.raises(crn.CrnError):
        crn.decode_batch_ex(bad, bad.size, *b.llr, 8, True, 0, bits, ok)
    with pytest.raises(crn.CrnError):
        crn.decode_batch_ex(b.desc, b.n_cb, *b.llr, 33, True, 0, bits, ok)
    crn.decode_batch_ex(b.desc[:0], 0, *b.llr, 8, True, 0, bits, ok)   # n_cb == 0 no-op


def test_tb_configs_tb_verdict(orc):
    """cfg2/cfg3 transport blocks: TB success iff all CBs pass and the TB CRC24A
    passes; successful TBs reproduce the payload."""
    for cfg, scale in ((2, 1.0), (3, 0.1)):
        b = _full(cfg, scale)
        g = run_gpu(b, 8, True)
        n_ok = 0
        for t in range(b.wl.n_tb):
            idx = np.flatnonzero(b.cb_tb == t)
            pay = crn.tb_reassemble(g["words"], b.desc[idx], g["crc_ok"][idx], int(b.wl.tbs[t]))
            if pay is not None:
                n_ok += 1
                assert np.array_equal(pay, b.wl.payload[t].cpu().numpy())
            else:
                assert not np.all(g["crc_ok"][idx])
        assert n_ok >= 1


def _host(t):
    return t.cpu().pin_memory()


@pytest.mark.parametrize("n_chunks", [0, 1, 3, 7])
def test_plan_decode_host_pipeline(orc, n_chunks):
    """crn_plan_decode_host (host buffers, chunked upload/decode/download overlap)
    equals the oracle on a mixed-K, filler-carrying TB batch for any chunking."""
    b = _full(3, 0.1)
    idx = np.arange(b.n_cb)
    r = run_oracle(b, idx, 8, True)
    p = crn.Plan(b.desc)
    hl = [_host(x) for x in b.llr]
    hb = torch.zeros(b.n_words, dtype=torch.int32).pin_memory()
    hok = torch.full((b.n_cb,), 7, dtype=torch.uint8).pin_memory()
    hit = torch.zeros(b.n_cb, dtype=torch.uint8).pin_memory()
    for rep in range(2):                        # second call reuses the staging buffers
        hb.zero_()
        p.decode_host(*hl, 8, True, hb, hok, hit, n_chunks=n_chunks)
        torch.cuda.synchronize()
        g = dict(words=hb.numpy().view(np.uint32), crc_ok=hok.numpy(), iters=hit.numpy(), ext=None)
        assert_parity(b, g, r, idx)
    assert p.chunks >= 1 and (n_chunks == 0 or p.chunks <= n_chunks)
    with pytest.raises(crn.CrnError):
        p.decode_host(*b.llr, 8, True, hb, hok)            # device tensors refused
    p.close()


@pytest.mark.parametrize("flags,packed", [(0, False), (0, True), (1, False), (2, True), (4, False), (6, True),
                                          (8, True), (8 | (3 << 8), False), (10 | (5 << 8), True)])
def test_stream_run_cfg5(orc, flags, packed):
    """crn_stream_run_ex: paced TTIs of cfg5, one stream per cell group (per-group
    decode launches, or one merged launch per TTI; int16 or -- CRN_STREAM_LLR8 --
    int8 LLRs read as x * 2^shift); every CB of every TTI bit-exact against the
    oracle (on the widened input for int8); timestamps ordered."""
    import dataclasses
    n_tti, n_groups = 3, 4
    llr8, sh = bool(flags & 8), (flags >> 8) & 0xF
    groups, checks = [], []
    for t in range(n_tti):
        b = _full(5, seed=100 + t)
        src = b.llr
        if llr8:
            src = tuple(torch.clamp(torch.round(x.float() / (1 << sh)), -128, 127).to(torch.int8) for x in b.llr)
            b = dataclasses.replace(b, llr=tuple(x.to(torch.int16) * (1 << sh) for x in src))
        r = run_oracle(b, np.arange(b.n_cb), 8, True)
        cells = np.unique(b.cb_cell)
        for gi in range(n_groups):
            sel = np.flatnonzero(np.isin(b.cb_cell, cells[gi::n_groups]))
            d = b.desc[sel].copy()
            K = d["K"].astype(np.int64)
            d["llr_off"] = np.concatenate([[0], np.cumsum(K + 4)[:-1]])
            d["bit_off"] = np.concatenate([[0], np.cumsum((K + 31) // 32)[:-1]])
            hl = [torch.cat([x[int(o):int(o) + int(k) + 4] for o, k in zip(b.desc["llr_off"][sel], K)]).cpu()
                  .pin_memory() if sel.size else torch.zeros(1, dtype=x.dtype).pin_memory() for x in src]
            nw, nc = max(int(((K + 31) // 32).sum()), 1), max(sel.size, 1)
            if packed:                      # one host block: bits | crc_ok | iters_used
                ob = torch.zeros(4 * nw + 2 * nc, dtype=torch.uint8).pin_memory()
                bits, ok, it = ob[:4 * nw].view(torch.int32), ob[4 * nw:4 * nw + nc], ob[4 * nw + nc:]
            else:
                bits = torch.zeros(nw, dtype=torch.int32).pin_memory()
                ok = torch.zeros(nc, dtype=torch.uint8).pin_memory()
                it = torch.zeros(nc, dtype=torch.uint8).pin_memory()
            g = dict(desc=d, l0=hl[0], l1=hl[1], l2=hl[2], bits=bits, ok=ok, it=it)
            groups.append(g)
            checks.append((b, r, sel, d, g))
    tim = crn.stream_run(groups, n_tti, n_groups, 1000.0, 8, True, flags=flags)
    for b, r, sel, d, g in checks:
        words = g["bits"].numpy().view(np.uint32)
        for n, i in enumerate(sel):
            K = int(d["K"][n])
            ob = r["bits"][r["bo"][i]:r["bo"][i] + K]
            assert np.array_equal(unpack(words, d, n), ob)
            assert g["ok"].numpy()[n] == r["crc_ok"][i] and g["it"].numpy()[n] == r["iters"][i]
    assert np.all(tim["latency_us"] > 0) and np.all(tim["device_us"] > 0)
    if flags & 3:                           # stage split recorded
        assert np.all(tim["decode_end_us"] > tim["decode_start_us"]) and np.all(tim["upload_us"] > 0)
    else:
        assert np.all(tim["upload_us"] == -1.0)
    assert np.all(np.diff(tim["release_us"]) > 900)
    assert np.all(tim["complete_us"] > tim["release_us"])


@pytest.mark.parametrize("llr8", [False, True])
def test_stream_run_cfg5_50_ttis_contiguous(orc, llr8):
    """BASELINE cfg5 as bench.py runs it: 50 distinct TTIs (cells 20t..20t+19),
    2 cell groups, each group's three LLR streams one pinned [3, n] block (the
    runtime's single-copy upload: int8, and int16 with n a multiple of 128) and
    bits | crc_ok | iters one host block (single download).  Every CB of every
    TTI against the oracle (int8: on the widened input)."""
    import dataclasses
    n_tti, n_groups, cpt = 50, 2, 20
    groups, checks = [], []
    for t in range(n_tti):
        b = _full(5, cells=range(cpt * t, cpt * (t + 1)))
        if llr8:
            q = tuple(torch.clamp(x, -128, 127).to(torch.int8) for x in b.llr)
            b = dataclasses.replace(b, llr=tuple(x.to(torch.int16) for x in q))
        checks.append([b, run_oracle(b, np.arange(b.n_cb), 8, True)])
        for gi in range(n_groups):
            sel = np.flatnonzero((b.cb_cell % cpt) // (cpt // n_groups) == gi)
            K = b.desc["K"][sel].astype(np.int64)
            ext = int((K + 4).sum())
            pad = 0 if llr8 else (-ext) % 128            # int16: stream stride a multiple of 256 B
            d = b.desc[sel].copy()
            d["llr_off"] = pad + np.concatenate([[0], np.cumsum(K + 4)[:-1]])
            d["bit_off"] = np.concatenate([[0], np.cumsum((K + 31) // 32)[:-1]])
            src = np.concatenate([np.arange(int(o), int(o) + int(k) + 4) for o, k in zip(b.desc["llr_off"][sel], K)])
            src = torch.from_numpy(src).cuda()
            dt = torch.int8 if llr8 else torch.int16
            buf = torch.zeros(3, pad + ext, dtype=dt)
            for s in range(3):
                buf[s, pad:] = b.llr[s][src].to(dt).cpu()
            buf = buf.pin_memory()
            nw, nc = int(((K + 31) // 32).sum()), sel.size
            ob = torch.zeros(4 * nw + 2 * nc, dtype=torch.uint8).pin_memory()
            g = dict(desc=d, l0=buf[0], l1=buf[1], l2=buf[2], bits=ob[:4 * nw].view(torch.int32),
                     ok=ob[4 * nw:4 * nw + nc], it=ob[4 * nw + nc:])
            groups.append(g)
            checks[-1].append((sel, d, g))
    tim = crn.stream_run(groups, n_tti, n_groups, 1000.0, 8, True, flags=crn.STREAM_LLR8 if llr8 else 0)
    assert tim.size == n_tti and np.all(tim["latency_us"] > 0)
    n = 0
    for b, r, *parts in checks:
        for sel, d, g in parts:
            words = g["bits"].numpy().view(np.uint32)
            gg = dict(words=np.zeros(b.n_words, np.uint32), crc_ok=np.zeros(b.n_cb, np.uint8),
                      iters=np.zeros(b.n_cb, np.uint8), ext=None)
            for m, i in enumerate(sel):                  # back to the TTI's own layout
                k = int(d["K"][m])
                gg["words"][b.desc["bit_off"][i]:b.desc["bit_off"][i] + (k + 31) // 32] = \
                    words[d["bit_off"][m]:d["bit_off"][m] + (k + 31) // 32]
            gg["crc_ok"][sel] = g["ok"].numpy()
            gg["iters"][sel] = g["it"].numpy()
            r_sel = dict(bits=r["bits"], crc_ok=r["crc_ok"][sel], iters=r["iters"][sel], bo=r["bo"][sel], ext=None)
            assert_parity(b, gg, r_sel, sel)
            n += sel.size
    assert n == sum(c[0].n_cb for c in checks) and n >= 50 * 150


def _tb_table(b):
    """TB descriptors of a TB-config batch (CBs of TB t are contiguous, in segment order)."""
    tbs = np.zeros(b.wl.n_tb, crn.TB_DTYPE)
    w = 0
    for t in range(b.wl.n_tb):
        idx = np.flatnonzero(b.cb_tb == t)
        tbs[t] = (idx[0], idx.size, int(b.wl.tbs[t]), w)
        w += (int(b.wl.tbs[t]) + 31) // 32
    return tbs, w


@pytest.mark.parametrize("cfg,scale,kill", [(2, 1.0, False), (3, 0.2, False), (3, 0.1, True)])
def test_tb_verdict_batch_matches_oracle(orc, cfg, scale, kill):
    """Row f1: device TB post-processing (strip fillers + CB CRCs, concatenate, TB
    CRC24A, all-CBs rule of PAPER.md:369) equals the oracle's reassembly of the
    oracle's own decoded bits, payload words included."""
    b = _full(cfg, scale)
    if kill:                                     # zero the LLRs of every 3rd CB's systematic stream
        for i in range(0, b.n_cb, 3):
            o, K = int(b.desc["llr_off"][i]), int(b.desc["K"][i])
            for x in b.llr:
                x[o:o + K + 4] = 0
    g = run_gpu(b, 8, True, want_ext=False)
    idx = np.arange(b.n_cb)
    r = run_oracle(b, idx, 8, True)
    tbs, nw = _tb_table(b)
    words = torch.from_numpy(g["words"].view(np.int32).copy()).cuda()
    ok = torch.from_numpy(g["crc_ok"].copy()).cuda()
    tb_ok = torch.full((tbs.size,), 9, dtype=torch.uint8, device="cuda")
    tb_words = torch.zeros(max(nw, 1), dtype=torch.int32, device="cuda")
    crn.tb_verdict_batch(tbs, b.desc, words, ok, tb_ok, tb_words)
    torch.cuda.synchronize()
    tb_ok, tb_words = tb_ok.cpu().numpy(), tb_words.cpu().numpy().view(np.uint32)
    n_fail = 0
    for t in range(tbs.size):
        cb = np.arange(tbs["cb0"][t], tbs["cb0"][t] + tbs["n_cb"][t])
        seg = orc.segment(int(tbs["tbs"][t]))
        bits = [r["bits"][r["bo"][i]:r["bo"][i] + r["K"][i]] for i in cb]
        Fs = [int(b.desc["F"][i]) for i in cb]
        pay = orc.reassemble_tb(bits, Fs, seg)
        want = bool(np.all(r["crc_ok"][cb]) and pay is not None)
        assert bool(tb_ok[t]) == want, t
        n_fail += not want
        L = seg["L"]
        full = np.concatenate([c[F:c.size - L] for c, F in zip(bits, Fs)])[:int(tbs["tbs"][t])]
        w0 = int(tbs["word_off"][t])
        got = ((tb_words[w0:w0 + (full.size + 31) // 32, None] >> np.arange(32, dtype=np.uint32)) & 1)
        assert np.array_equal(got.astype(np.uint8).reshape(-1)[:full.size], full), t
        if want:
            assert np.array_equal(full, b.wl.payload[t].cpu().numpy())
    if kill:
        assert n_fail >= 1


@pytest.mark.parametrize("cfg,scale,I,et", [(1, 1.0, 6, False), (5, 1.0, 8, True), (3, 0.1, 8, True)])
def test_scaled_variant_parity(orc, cfg, scale, I, et):
    """Row f2: the scaled-extrinsic variant (CRN_EXT_SCALED, R28) is
    bit-exact against the oracle's variant on both kernel paths (W = 32 and
    generic W), and the plan API selects it too."""
    b = _full(cfg, scale)
    g = run_gpu(b, I, et, flags=crn.EXT_SCALED)
    idx = np.arange(b.n_cb)
    r = run_oracle(b, idx, I, et, variant=orc.VAR_SCALED)
    assert_parity(b, g, r, idx)
    p = crn.Plan(b.desc)
    p.set_variant(crn.VARIANT_SCALED)
    bits, ok, it, ext = bmod.outputs(b)
    p.decode(*b.llr, I, et, bits, ok, it, ext)
    torch.cuda.synchronize()
    assert np.array_equal(bits.cpu().numpy().view(np.uint32), g["words"])
    assert np.array_equal(ext.cpu().numpy(), g["ext"])
    with pytest.raises(crn.CrnError):
        p.set_variant(7)


def test_outputs_write_only_their_ranges(orc):
    """Memcheck substitute (compute-sanitizer is unavailable on this pool): CBs are
    laid out with gaps between their LLR, output-word and ext ranges, every output
    buffer is pre-filled with a sentinel, and after decoding (fast + generic paths,
    ET, ext_out) everything outside the described ranges still holds the sentinel
    while every CB is bit-exact against the oracle."""
    b = _full(5, 1.0)
    rng = np.random.default_rng(11)
    K = b.desc["K"].astype(np.int64)
    gl = rng.integers(1, 40, b.n_cb)
    gw = rng.integers(1, 5, b.n_cb)
    ge = rng.integers(1, 40, b.n_cb)
    d = b.desc.copy()
    lo = np.zeros(b.n_cb, np.int64); wo = np.zeros(b.n_cb, np.int64); eo = np.zeros(b.n_cb, np.int64)
    a = c = e = 0
    for i in range(b.n_cb):
        a += gl[i]; lo[i] = a; a += K[i] + 4
        c += gw[i]; wo[i] = c; c += (K[i] + 31) // 32
        e += ge[i]; eo[i] = e; e += K[i]
    d["llr_off"], d["bit_off"], d["ext_off"] = lo, wo, eo
    n_llr, n_w, n_e = a + 17, c + 9, e + 23
    ll = [torch.full((n_llr,), 0x5A5A, dtype=torch.int16, device="cuda") for _ in range(3)]
    for s in range(3):
        for i in range(b.n_cb):
            o = int(b.desc["llr_off"][i])
            ll[s][int(lo[i]):int(lo[i]) + int(K[i]) + 4] = b.llr[s][o:o + int(K[i]) + 4]
    SENT = 0x3C3C3C3C
    bits = torch.full((n_w,), SENT, dtype=torch.int64, device="cuda").to(torch.int32)
    ok = torch.full((b.n_cb + 7,), 0xA5, dtype=torch.uint8, device="cuda")
    it = torch.full((b.n_cb + 7,), 0xA5, dtype=torch.uint8, device="cuda")
    ext = torch.full((n_e,), 0x7B7B, dtype=torch.int16, device="cuda")
    crn.decode_batch_ex(d, b.n_cb, *ll, 8, True, 0, bits, ok, it, ext)
    torch.cuda.synchronize()
    words = bits.cpu().numpy().view(np.uint32)
    r = run_oracle(b, np.arange(b.n_cb), 8, True)
    g = dict(words=words, crc_ok=ok.cpu().numpy()[:b.n_cb], iters=it.cpu().numpy()[:b.n_cb], ext=ext.cpu().numpy())

    class _B:
        desc = d
    assert_parity(_B, g, r, np.arange(b.n_cb))
    wmask = np.ones(n_w, bool)
    emask = np.ones(n_e, bool)
    for i in range(b.n_cb):
        wmask[wo[i]:wo[i] + (K[i] + 31) // 32] = False
        emask[eo[i]:eo[i] + K[i]] = False
    assert np.all(words[wmask] == SENT)
    assert np.all(g["ext"][emask] == 0x7B7B)
    assert np.all(ok.cpu().numpy()[b.n_cb:] == 0xA5) and np.all(it.cpu().numpy()[b.n_cb:] == 0xA5)


@pytest.mark.parametrize("cfg,scale", [(5, 1.0), (3, 0.1), (1, 1.0)])
def test_mi_stopping_rule_parity(orc, cfg, scale):
    """The paper's MI stopping rule (CRN_ET_MI, R29) on
    both kernel paths: bits, extrinsics, iteration counts and CRC flags equal the
    oracle's; the plain and scaled variants both."""
    b = _full(cfg, scale)
    idx = np.arange(b.n_cb)
    for flags, var in ((0, orc.VAR_MAXLOG), (crn.EXT_SCALED, orc.VAR_SCALED)):
        g = run_gpu(b, 8, crn.ET_MI, flags=flags)
        r = run_oracle(b, idx, 8, orc.ET_MI, variant=var)
        assert_parity(b, g, r, idx)
        assert np.all(g["iters"] >= 2)


def _rm_case(rng, n, ks):
    K = rng.choice(ks, n)
    N = 3 * (K + 4)
    E = np.maximum(1, (N * rng.choice([0.31, 0.5, 1.0, 1.7, 2.6], n)).astype(np.int64))
    rv = rng.integers(0, 4, n)
    d = np.zeros(n, crn.RM_DTYPE)
    d["K"], d["E"], d["rv"] = K, E, rv
    d["e_off"] = np.concatenate([[0], np.cumsum(E)[:-1]]) + 3 * np.arange(n)          # gaps between CBs
    d["llr_off"] = np.concatenate([[0], np.cumsum(K + 4)[:-1]]) + 5 * np.arange(n)
    return d


def test_rate_dematch_and_match_parity(orc):
    """Row f4: device rate de-matching (with and without HARQ combining) and rate
    matching equal the oracle's for mixed K (both kernel geometries), E from
    heavy puncturing to repetition and every redundancy version."""
    rng = np.random.default_rng(21)
    ks = np.array([40, 48, 56, 104, 112, 120, 248, 512, 1008, 528, 1056, 2112, 4096, 6144])   # ND in {4, 12, 20, 28}
    d = _rm_case(rng, 80, ks)
    n_e = int((d["e_off"] + d["E"]).max())
    n_l = int((d["llr_off"] + d["K"] + 4).max())
    e = rng.integers(-3000, 3001, n_e).astype(np.int16)
    h_prev = [rng.integers(-30000, 30001, n_l).astype(np.int16) for _ in range(3)]
    for combine in (False, True):
        hg = [torch.from_numpy(x.copy()).cuda() for x in h_prev]
        crn.rate_dematch_batch(d, torch.from_numpy(e).cuda(), combine, *hg)
        torch.cuda.synchronize()
        hg = [x.cpu().numpy() for x in hg]
        for i in range(d.size):
            K, lo, eo, E = int(d["K"][i]), int(d["llr_off"][i]), int(d["e_off"][i]), int(d["E"][i])
            prev = [x[lo:lo + K + 4] for x in h_prev] if combine else None
            ho = orc.rate_dematch(e[eo:eo + E], K, int(d["rv"][i]), h=prev)
            for s in range(3):
                assert np.array_equal(hg[s][lo:lo + K + 4], ho[s]), (combine, i, s)
    bits = [rng.integers(0, 2, n_l, dtype=np.uint8) for _ in range(3)]
    eg = torch.zeros(n_e, dtype=torch.uint8, device="cuda")
    crn.rate_match_batch(d, *(torch.from_numpy(x).cuda() for x in bits), eg)
    torch.cuda.synchronize()
    eg = eg.cpu().numpy()
    for i in range(d.size):
        K, lo, eo, E = int(d["K"][i]), int(d["llr_off"][i]), int(d["e_off"][i]), int(d["E"][i])
        ref = orc.rate_match([x[lo:lo + K + 4] for x in bits], E, int(d["rv"][i]))
        assert np.array_equal(eg[eo:eo + E], ref), i


def test_rate_matched_chain_decodes_like_oracle(orc):
    """Rate match -> noisy int16 soft values -> de-match -> decode: the GPU chain
    (crn_rate_match_batch, crn_rate_dematch_batch, decode) against the oracle's
    chain on the same soft values, which are made from the ORACLE's rate-matched
    bits (the GPU's are checked equal to them), every stage compared."""
    b = _full(5, 0.5)
    rng = np.random.default_rng(5)
    K = b.desc["K"].astype(np.int64)
    d = np.zeros(b.n_cb, crn.RM_DTYPE)
    d["K"] = K
    d["E"] = (3 * (K + 4) * 0.75).astype(np.int64)                    # rate about 0.45
    d["rv"] = 0
    d["e_off"] = np.concatenate([[0], np.cumsum(d["E"])[:-1]])
    d["llr_off"] = b.desc["llr_off"]
    n_e = int(d["E"].sum())
    coded = [x.cpu().numpy() for x in b.coded]                        # the oracle's coded bits (_full)
    eo_bits = np.concatenate([orc.rate_match([x[lo:lo + k + 4] for x in coded], int(E), 0)
                              for k, lo, E in zip(K, d["llr_off"], d["E"])])
    eb = torch.zeros(n_e, dtype=torch.uint8, device="cuda")
    crn.rate_match_batch(d, *b.coded, eb)
    torch.cuda.synchronize()
    assert np.array_equal(eb.cpu().numpy(), eo_bits)
    x = (2 * eo_bits.astype(np.int32) - 1) * 40 + rng.normal(0, 25, n_e).round().astype(np.int32)
    soft = np.clip(x, -32768, 32767).astype(np.int16)
    hg = [torch.zeros_like(t) for t in b.llr]
    crn.rate_dematch_batch(d, torch.from_numpy(soft).cuda(), False, *hg)
    g = run_gpu(b, 8, True, l=hg)
    hh = [t.cpu().numpy() for t in hg]
    ho_all = [np.zeros_like(t) for t in hh]
    for i in range(b.n_cb):
        k, lo, eo, E = int(K[i]), int(d["llr_off"][i]), int(d["e_off"][i]), int(d["E"][i])
        ho = orc.rate_dematch(soft[eo:eo + E], k, 0)
        for s in range(3):
            assert np.array_equal(hh[s][lo:lo + k + 4], ho[s])
            ho_all[s][lo:lo + k + 4] = ho[s]
    b2 = type("B", (), {})()
    b2.llr, b2.desc = tuple(torch.from_numpy(x) for x in ho_all), b.desc   # the oracle's de-matched streams
    r = run_oracle(b2, np.arange(b.n_cb), 8, True)
    assert_parity(b, g, r, np.arange(b.n_cb))
    assert g["crc_ok"].mean() > 0.5


def test_tb_purge_of_waiting_cbs(orc):
    """The paper's purge (crn_plan_set_purge): with the TB id in
    each descriptor, a CB that has not started when a sibling fails is not
    decoded (crc_ok = 0, iters_used = 0); every decoded CB equals the oracle and
    the no-purge run, purged CBs belong to TBs with a failed decoded CB, and the
    TB verdicts do not change.  A one-CTA grid makes the order strict, so purges
    must happen; the full grid is checked for consistency only."""
    b = _full(3, 0.3)
    for i in range(0, b.n_cb, 4):                          # kill a quarter of the CBs: they fail at max
        o, K = int(b.desc["llr_off"][i]), int(b.desc["K"][i])
        for x in b.llr:
            x[o:o + K + 4] = 0
    desc = b.desc.copy()
    desc["reserved"] = b.cb_tb
    idx = np.arange(b.n_cb)
    r = run_oracle(b, idx, 8, True)
    tbs, nw = _tb_table(b)
    verdicts = []
    for grid in (0, 1):
        for purge in (False, True):
            p = crn.Plan(desc)
            p.set_grid(grid)
            p.set_purge(purge)
            bits, ok, it, ext = bmod.outputs(b)
            p.decode(*b.llr, 8, True, bits, ok, it, ext)
            tb_ok = torch.zeros(tbs.size, dtype=torch.uint8, device="cuda")
            crn.tb_verdict_batch(tbs, b.desc, bits, ok, tb_ok)
            torch.cuda.synchronize()
            g = dict(words=bits.cpu().numpy().view(np.uint32), crc_ok=ok.cpu().numpy()[:b.n_cb],
                     iters=it.cpu().numpy()[:b.n_cb], ext=ext.cpu().numpy())
            verdicts.append(tb_ok.cpu().numpy())
            dec = np.flatnonzero(g["iters"] > 0)
            purged = np.flatnonzero(g["iters"] == 0)
            assert_parity(b, g, r if dec.size == b.n_cb else run_oracle(b, dec, 8, True), dec)
            if not purge:
                assert purged.size == 0
            else:
                failed_tb = set(b.cb_tb[dec[g["crc_ok"][dec] == 0]])
                assert all(b.cb_tb[i] in failed_tb for i in purged)
                assert np.all(g["crc_ok"][purged] == 0)
                if grid == 1:
                    assert purged.size > 0
            p.close()
    assert all(np.array_equal(v, verdicts[0]) for v in verdicts)


@pytest.mark.parametrize("cfg,scale,shift,pad", [(1, 1.0, 4, 0), (5, 1.0, 5, 1), (3, 0.1, 3, 0), (2, 1.0, 8, 3)])
def test_int8_llr_ingest_parity(orc, cfg, scale, shift, pad):
    """Row f4 int8 ingest (crn_plan_set_llr_format, R31): int8 LLRs x
    decode exactly as the int16 LLRs x * 2^shift -- the GPU int8 path against the
    oracle on the widened int16 input, every output, through the device path and
    the host-buffer pipeline; pad shifts every offset off 4-byte alignment."""
    import dataclasses
    b = _full(cfg, scale)
    I, et = b.wl.max_iters, b.wl.early_term
    q = [torch.clamp(torch.round(x.float() / (1 << shift)), -128, 127).to(torch.int8) for x in b.llr]
    desc = b.desc.copy()
    if pad:
        desc["llr_off"] += pad
        q = [torch.cat([torch.full((pad,), 77, dtype=torch.int8, device=x.device), x]) for x in q]
    wide = tuple(x.to(torch.int16)[pad:] * (1 << shift) for x in q)
    b16 = dataclasses.replace(b, llr=wide)
    plan = crn.Plan(desc)
    plan.set_llr_format(8, shift)
    with pytest.raises(crn.CrnError):
        plan.decode(*b.llr, I, et, *bmod.outputs(b, want_ext=False)[:3])      # int16 tensors refused
    bits, ok, it, _ = bmod.outputs(b, want_ext=False)
    plan.decode(*q, I, et, bits, ok, it)
    torch.cuda.synchronize()
    g = dict(words=bits.cpu().numpy().view(np.uint32), crc_ok=ok.cpu().numpy()[:b.n_cb],
             iters=it.cpu().numpy()[:b.n_cb], ext=None)
    idx = np.arange(b.n_cb)
    r = run_oracle(b16, idx, I, et)
    assert_parity(b16, g, r, idx)
    hq = [x.cpu().pin_memory() for x in q]
    hb = torch.zeros(bits.numel(), dtype=torch.int32).pin_memory()
    hok = torch.zeros(ok.numel(), dtype=torch.uint8).pin_memory()
    hit = torch.zeros(it.numel(), dtype=torch.uint8).pin_memory()
    plan.decode_host(*hq, I, et, hb, hok, hit, n_chunks=3)
    torch.cuda.synchronize()
    assert np.array_equal(hb.numpy().view(np.uint32)[:b.n_words], g["words"][:b.n_words])
    assert np.array_equal(hok.numpy()[:b.n_cb], g["crc_ok"])
    assert np.array_equal(hit.numpy()[:b.n_cb], g["iters"])


@pytest.mark.parametrize("cfg,scale,I,et", [(1, 1.0, 6, False), (5, 1.0, 8, True), (3, 0.1, 8, True)])
def test_logmap_variant_parity(orc, cfg, scale, I, et):
    """Row f2: Log-MAP (CRN_VARIANT_LOGMAP, R32) is bit-exact against the
    oracle's Log-MAP -- bits, int16 extrinsics, iteration counts, CRC flags -- on
    both kernel paths (W = 32 and generic W), device and host-buffer plans."""
    b = _full(cfg, scale)
    p = crn.Plan(b.desc)
    p.set_variant(crn.VARIANT_LOGMAP)
    bits, ok, it, ext = bmod.outputs(b)
    p.decode(*b.llr, I, et, bits, ok, it, ext)
    torch.cuda.synchronize()
    g = dict(words=bits.cpu().numpy().view(np.uint32), crc_ok=ok.cpu().numpy()[:b.n_cb],
             iters=it.cpu().numpy()[:b.n_cb], ext=ext.cpu().numpy())
    idx = np.arange(b.n_cb)
    r = run_oracle(b, idx, I, et, variant=orc.VAR_LOGMAP)
    assert_parity(b, g, r, idx)
    hl = [x.cpu().pin_memory() for x in b.llr]
    hb = torch.zeros(bits.numel(), dtype=torch.int32).pin_memory()
    hok = torch.zeros(ok.numel(), dtype=torch.uint8).pin_memory()
    p.decode_host(*hl, I, et, hb, hok, None, n_chunks=2)
    torch.cuda.synchronize()
    assert np.array_equal(hb.numpy().view(np.uint32)[:b.n_words], g["words"][:b.n_words])
    assert np.array_equal(hok.numpy()[:b.n_cb], g["crc_ok"])


def test_tb_build_cbs_batch_matches_oracle(orc):
    """Row f3 (DL conditioning on the device): crn_tb_build_cbs_batch -- TB
    CRC24A, 36.212 segmentation, fillers, CB CRC24B -- equals the oracle's
    segment_tb_bits for every TB: descriptors, and every CB bit.  TBS cover C = 1
    with and without fillers, the C = 1 / C = 2 boundary (6120 / 6121), the
    smallest K, cfg2's 13 CBs, the largest LTE TBS and 4-layer sizes (C up to
    64), random sizes; payloads sit at odd byte offsets."""
    rng = np.random.default_rng(31)
    tbs = [16, 17, 40, 1000, 4000, 6119, 6120, 6121, 12000, 75376, 97896, 391656, 1, 2, 3, 5, 8]
    tbs += list(rng.integers(1, 75377, 60)) + list(rng.integers(75377, 391657, 4))
    pays = [rng.integers(0, 2, int(t), dtype=np.uint8) for t in tbs]
    gaps = rng.integers(0, 7, len(tbs))
    off, buf, o = [], [], 0
    for p, gp in zip(pays, gaps):
        buf.append(np.full(int(gp), 9, np.uint8))               # junk between payloads (bit 0 of 9 is 1)
        o += int(gp)
        off.append(o)
        buf.append(p)
        o += p.size
    payload = torch.from_numpy(np.concatenate(buf)).cuda()
    desc, cb_bits = crn.tb_build_cbs_batch(np.array(tbs, np.int64), np.array(off, np.int64), payload)
    torch.cuda.synchronize()
    got = cb_bits.cpu().numpy()
    n = 0
    bit = llr = word = 0
    for t, p in enumerate(pays):
        cbs, Fs, seg = orc.segment_tb_bits(p)
        assert seg["C"] == len(cbs)
        for r, (c, F) in enumerate(zip(cbs, Fs)):
            d = desc[n]
            K = c.size
            assert (d["K"], d["F"], d["reserved"]) == (K, F, t)
            assert d["crc_kind"] == (crn.CRC24A if seg["C"] == 1 else crn.CRC24B)
            assert (d["ext_off"], d["llr_off"], d["bit_off"]) == (bit, llr, word)
            assert np.array_equal(got[bit:bit + K], c), (t, r, np.flatnonzero(got[bit:bit + K] != c)[:8])
            bit += K
            llr += K + 4
            word += (K + 31) // 32
            n += 1
    assert n == desc.size and got.size == bit
    # a CB buffer that is not 8-byte aligned takes the kernel's byte-by-byte write
    # path; payload bytes with their upper bits set count by bit 0 only (include/crn.h)
    for shift in (1, 4):
        raw = torch.full((got.size + 16,), 7, dtype=torch.uint8, device="cuda")
        d2, cb2 = crn.tb_build_cbs_batch(np.array(tbs, np.int64), np.array(off, np.int64), payload | 0xFE,
                                         cb_bits=raw[shift:shift + got.size + 8], max_cb=desc.size)
        torch.cuda.synchronize()
        assert np.array_equal(d2, desc) and np.array_equal(cb2.cpu().numpy(), got)
        r = raw.cpu().numpy()
        assert (r[:shift] == 7).all() and (r[shift + got.size:] == 7).all()
    with pytest.raises(crn.CrnError):
        crn.tb_build_cbs_batch(np.array([0], np.int64), np.array([0], np.int64), payload)


def test_race_stress_grids_repeats_variants(orc):
    """Stand-in for a race detector (compute-sanitizer is closed on this GPU pool,
    DESIGN.md §5b): the single-buffered shared state (NII boundaries, the hard
    decision's window words, the CRC / MI atomics, the group tasks' named barriers
    and next-task slots) is exercised under many different interleavings -- one
    mixed early-terminated batch (whole-CTA W = 32 tasks, split-path tasks, group
    tasks, dummy partner lanes, fillers) decoded on persistent grids of 1, 2, 3, 5,
    17, 61 and all CTAs (so every CTA runs a different task sequence) and 12 times
    on the full grid, each decoder variant and stopping rule.  Every run must equal
    the oracle's outputs for that variant, element by element."""
    rng = np.random.default_rng(23)
    Ks = ([6144] * 9 + [5824] * 4 + [3072] * 5 + [2048] * 7 + [1056] * 11 + [1088] * 3 + [512] * 30 + [64] * 70 +
          [1008] * 5 + [488] * 7 + [40] * 13 + [104] * 3)
    K = list(rng.permutation(Ks))
    F = [int(rng.integers(0, min(64, k - 24))) if i % 5 == 0 else 0 for i, k in enumerate(K)]
    d = _desc_for(K, F, [crn.CRC24A if i % 7 == 0 else crn.CRC24B for i in range(len(K))])
    llr = _random_llr(d, rng, 90)
    n = int((d["llr_off"] + d["K"] + 4).max())
    lean = np.zeros(n, np.int16)                 # a third lean to the all-zero codeword: early stops
    for o, k in zip(d["llr_off"][::3], d["K"][::3]):
        lean[o:o + k + 4] = -70
    llr = tuple((x + torch.from_numpy(lean).cuda()).clamp(-32767, 32767) for x in llr)
    b = _B(d, llr)
    idx = np.arange(d.size)
    plan = crn.Plan(d)
    for variant, et, ov, oet in ((crn.VARIANT_MAXLOG, crn.ET_CRC, orc.VAR_MAXLOG, orc.ET_CRC),
                                 (crn.VARIANT_SCALED, crn.ET_CRC, orc.VAR_SCALED, orc.ET_CRC),
                                 (crn.VARIANT_MAXLOG, crn.ET_MI, orc.VAR_MAXLOG, orc.ET_MI),
                                 (crn.VARIANT_LOGMAP, crn.ET_CRC, orc.VAR_LOGMAP, orc.ET_CRC)):
        plan.set_variant(variant)
        r = run_oracle(b, idx, 8, oet, variant=ov)
        runs = [(g, 1) for g in (1, 2, 3, 5, 17, 61)] + [(0, 12)]
        for grid, reps in runs:
            plan.set_grid(grid)
            for _ in range(reps):
                bits = torch.full((b.n_words,), -1, dtype=torch.int32, device="cuda")
                ok = torch.full((d.size,), 7, dtype=torch.uint8, device="cuda")
                it = torch.zeros(d.size, dtype=torch.uint8, device="cuda")
                ext = torch.zeros(int(d["K"].sum()), dtype=torch.int16, device="cuda")
                plan.decode(*llr, 8, et, bits, ok, it, ext)
                torch.cuda.synchronize()
                g = dict(words=bits.cpu().numpy().view(np.uint32), crc_ok=ok.cpu().numpy(), iters=it.cpu().numpy(),
                         ext=ext.cpu().numpy())
                assert_parity(b, g, r, idx)
        assert 0 < int(r["crc_ok"].sum()) < d.size and len(set(r["iters"].tolist())) > 2
    plan.set_grid(0)


def _bits_to_words(bits, n_words):
    """uint8 0/1 array -> packed LSB-first uint32 words (numpy), zero-padded."""
    b = np.zeros(32 * n_words, np.uint8)
    b[:bits.size] = bits
    return np.packbits(b, bitorder="little").view(np.uint32).copy()


def _words_to_bits(words):
    return np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")


def test_packed_encoder_and_rate_match_parity(orc):
    """Row f3/f4 packed-bit forms (crn_encode_batch_packed, crn_rate_match_batch_packed):
    one bit per bit at unaligned BIT offsets with gaps between CBs (neighbouring CBs
    share words), mixed K over every K mod 32 residue, CRC attach on and off; the
    coded streams equal the oracle encoder's and the rate-matched bits the oracle's,
    bit for bit, and every bit outside the CBs' ranges keeps its previous value."""
    rng = np.random.default_rng(29)
    Ks = np.array(list(rng.choice(orc.k_table(), 60)) + [6144, 6144, 40, 1056, 1088, 1008, 1024])
    n = Ks.size
    kinds = np.where(np.arange(n) % 4 == 0, crn.CRC24A, crn.CRC24B)
    d = np.zeros(n, crn.DESC_DTYPE)
    d["K"], d["crc_kind"] = Ks, kinds
    d["ext_off"] = np.concatenate([[5], np.cumsum(Ks + 3)[:-1] + 5])               # bit offsets, odd gaps
    d["llr_off"] = np.concatenate([[3], np.cumsum(Ks + 4 + 7)[:-1] + 3])
    n_info = int((d["ext_off"] + Ks).max()) + 40
    n_code = int((d["llr_off"] + Ks + 4).max()) + 40
    info_bits = rng.integers(0, 2, n_info).astype(np.uint8)
    info = torch.from_numpy(_bits_to_words(info_bits, (n_info + 31) // 32).view(np.int32)).cuda()
    nw = (n_code + 31) // 32
    for attach in (False, True):
        fill = [rng.integers(0, 2, 32 * nw).astype(np.uint8) for _ in range(3)]
        outs = [torch.from_numpy(_bits_to_words(f, nw).view(np.int32)).cuda() for f in fill]
        crn.encode_batch_packed(d, info, attach, *outs)
        torch.cuda.synchronize()
        got = [_words_to_bits(o.cpu().numpy()) for o in outs]
        inside = np.zeros(32 * nw, bool)
        for i in range(n):
            K, eo, lo = int(Ks[i]), int(d["ext_off"][i]), int(d["llr_off"][i])
            c = info_bits[eo:eo + K].copy()
            if attach:
                c = orc.crc_attach(int(kinds[i]), c[:-24])
            ref = orc.turbo_encode(c)
            for s in range(3):
                assert np.array_equal(got[s][lo:lo + K + 4], ref[s]), (attach, i, s)
            inside[lo:lo + K + 4] = True
        for s in range(3):
            assert np.array_equal(got[s][~inside], fill[s][~inside]), (attach, s)
    # packed rate matching of random coded streams
    dm = _rm_case(rng, 70, np.array([40, 48, 56, 104, 112, 120, 248, 512, 1008, 528, 1056, 2112, 4096, 6144]))
    dm["llr_off"] = np.concatenate([[9], np.cumsum(dm["K"] + 4 + 13)[:-1] + 9])     # bit offsets
    dm["e_off"] = np.concatenate([[17], np.cumsum(dm["E"] + 5)[:-1] + 17])
    n_l = int((dm["llr_off"] + dm["K"] + 4).max()) + 40
    n_e = int((dm["e_off"] + dm["E"]).max()) + 40
    coded = [rng.integers(0, 2, n_l).astype(np.uint8) for _ in range(3)]
    cw = [torch.from_numpy(_bits_to_words(x, (n_l + 31) // 32).view(np.int32)).cuda() for x in coded]
    nwe = (n_e + 31) // 32
    efill = rng.integers(0, 2, 32 * nwe).astype(np.uint8)
    eg = torch.from_numpy(_bits_to_words(efill, nwe).view(np.int32)).cuda()
    crn.rate_match_batch_packed(dm, *cw, eg)
    torch.cuda.synchronize()
    got = _words_to_bits(eg.cpu().numpy())
    inside = np.zeros(32 * nwe, bool)
    for i in range(dm.size):
        K, lo, eo, E = int(dm["K"][i]), int(dm["llr_off"][i]), int(dm["e_off"][i]), int(dm["E"][i])
        ref = orc.rate_match([x[lo:lo + K + 4] for x in coded], E, int(dm["rv"][i]))
        assert np.array_equal(got[eo:eo + E], ref), i
        inside[eo:eo + E] = True
    assert np.array_equal(got[~inside], efill[~inside])
