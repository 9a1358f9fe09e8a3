"""GPU-side helpers for the parity tests: run libcrn on a product-built batch and
the oracle on the very same LLR buffers, then compare element by element."""
import os

import numpy as np
import torch

from paper_1905_01141_b200 import batch as bmod
from paper_1905_01141_b200 import crn


def run_gpu(b, max_iters, et, want_ext=True, stream=None, desc=None, l=None, flags=0):
    desc = b.desc if desc is None else desc
    bits, ok, it, ext = bmod.outputs(b, want_ext=want_ext)
    l0, l1, l2 = b.llr if l is None else l
    crn.decode_batch_ex(desc, desc.size, l0, l1, l2, max_iters, et, flags, bits, ok, it, ext, stream=stream)
    torch.cuda.synchronize()
    return dict(words=bits.cpu().numpy().view(np.uint32), crc_ok=ok.cpu().numpy()[:desc.size],
                iters=it.cpu().numpy()[:desc.size], ext=None if ext is None else ext.cpu().numpy())


def unpack(words, desc, i):
    K, o = int(desc["K"][i]), int(desc["bit_off"][i])
    w = words[o:o + (K + 31) // 32]
    return ((w[:, None] >> np.arange(32, dtype=np.uint32)) & 1).astype(np.uint8).reshape(-1)[:K]


def run_oracle(b, idx, max_iters, et, variant=0):
    import oracle
    host = [x.cpu().numpy() for x in b.llr]
    d = b.desc[np.asarray(idx)]
    K = d["K"].astype(np.int32)
    lo = np.concatenate([[0], np.cumsum(K + 4)[:-1]]).astype(np.int64)
    bo = np.concatenate([[0], np.cumsum(K)[:-1]]).astype(np.int64)
    ll = [np.concatenate([h[o:o + k + 4] for o, k in zip(d["llr_off"], K)]) if K.size else h[:0] for h in host]
    r = oracle.decode_batch(K, d["F"], d["crc_kind"], lo, bo, *ll, max_iters=max_iters, early_term=et,
                            nthreads=os.cpu_count() or 1, variant=variant)
    assert r["violations"] == 0
    r["bo"], r["K"] = bo, K
    return r


def assert_parity(b, g, r, idx):
    """Element-by-element comparison of the GPU outputs g (words at desc.bit_off,
    crc_ok / iters per CB, ext at desc.ext_off) with the oracle's r for the CBs
    idx (r in idx order).  Equal-K groups are compared vectorised."""
    desc = b.desc
    idx = np.asarray(idx)
    if idx.size > 64:
        _assert_parity_vec(desc, g, r, idx)
        return
    _assert_parity_loop(desc, g, r, idx)


def _assert_parity_vec(desc, g, r, idx, chunk=1024):
    K = desc["K"][idx].astype(np.int64)
    okg, ito = g["crc_ok"][idx], g["iters"][idx]
    bad = np.flatnonzero(okg != r["crc_ok"])
    assert bad.size == 0, f"crc_ok differs at CBs {idx[bad[:8]]}"
    bad = np.flatnonzero(ito != r["iters"])
    assert bad.size == 0, f"iters differ at CBs {idx[bad[:8]]}: {ito[bad[:4]]} vs {r['iters'][bad[:4]]}"
    words = g["words"].view(np.uint32)
    for k in np.unique(K):
        sel = np.flatnonzero(K == k)
        nw = (int(k) + 31) // 32
        for c0 in range(0, sel.size, chunk):
            s = sel[c0:c0 + chunk]
            wo = desc["bit_off"][idx[s]].astype(np.int64)
            gw = words[wo[:, None] + np.arange(nw)]                               # [n, nw] packed LSB-first
            gb = np.unpackbits(gw.view(np.uint8), axis=1, bitorder="little")[:, :k]
            ob = r["bits"][r["bo"][s][:, None] + np.arange(k)]
            bad = np.flatnonzero(np.any(gb != ob, axis=1))
            assert bad.size == 0, f"bits differ: CB {idx[s[bad[0]]]} K={k} at {np.flatnonzero(gb[bad[0]] != ob[bad[0]])[:8]}"
            if g.get("ext") is not None:
                eo = desc["ext_off"][idx[s]].astype(np.int64)
                ge = g["ext"][eo[:, None] + np.arange(k)]
                oe = r["ext"][r["bo"][s][:, None] + np.arange(k)]
                bad = np.flatnonzero(np.any(ge != oe, axis=1))
                assert bad.size == 0, f"ext differs: CB {idx[s[bad[0]]]} K={k}"


def count_mismatches(desc, g, r, idx, chunk=1024) -> int:
    """Number of CBs in idx whose packed bits, crc_ok or iters (when g has them)
    differ from the oracle's r (r in idx order) -- bench.py's self-check."""
    idx = np.asarray(idx)
    K = desc["K"][idx].astype(np.int64)
    bad = g["crc_ok"][idx] != r["crc_ok"]
    if g.get("iters") is not None:
        bad |= g["iters"][idx] != r["iters"]
    words = g["words"].view(np.uint32)
    for k in np.unique(K):
        sel = np.flatnonzero(K == k)
        nw = (int(k) + 31) // 32
        for c0 in range(0, sel.size, chunk):
            s = sel[c0:c0 + chunk]
            wo = desc["bit_off"][idx[s]].astype(np.int64)
            gb = np.unpackbits(words[wo[:, None] + np.arange(nw)].view(np.uint8), axis=1, bitorder="little")[:, :k]
            ob = r["bits"][r["bo"][s][:, None] + np.arange(k)]
            bad[s] |= np.any(gb != ob, axis=1)
    return int(bad.sum())


def _assert_parity_loop(desc, g, r, idx):
    for n, i in enumerate(idx):
        K = int(desc["K"][i])
        ob = r["bits"][r["bo"][n]:r["bo"][n] + K]
        gb = unpack(g["words"], desc, i)
        assert np.array_equal(gb, ob), f"bits CB {i} K={K}: {np.flatnonzero(gb != ob)[:8]}"
        assert g["crc_ok"][i] == r["crc_ok"][n], f"crc_ok CB {i}"
        assert g["iters"][i] == r["iters"][n], f"iters CB {i}: {g['iters'][i]} vs {r['iters'][n]}"
        if g["ext"] is not None:
            e = int(desc["ext_off"][i])
            ge, oe = g["ext"][e:e + K], r["ext"][r["bo"][n]:r["bo"][n] + K]
            assert np.array_equal(ge, oe), f"ext CB {i}: {np.flatnonzero(ge != oe)[:8]}"
