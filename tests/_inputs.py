"""Test-side input assembly: oracle CRC/segmentation/encoder + the shared
workload generator's channel.  Test infrastructure only."""
import numpy as np
import torch

from paper_1905_01141_b200 import workload as wlmod


def oracle_cbs(wl):
    """Per CB: dict(c=bits incl. CRC and fillers, K, F, crc, cell, ebn0, tb)."""
    import oracle
    out = []
    for t in range(wl.n_tb):
        a = wl.payload[t].cpu().numpy().astype(np.uint8)
        if wl.tb_kind == "cb":
            c = oracle.crc_attach(oracle.CRC24B, a)
            out.append(dict(c=c, K=c.size, F=0, crc=oracle.CRC24B, cell=int(wl.tb_cell[t]),
                            ebn0=float(wl.tb_ebn0_db[t]), tb=t))
        else:
            cbs, Fs, seg = oracle.segment_tb_bits(a)
            kind = oracle.CRC24A if seg["C"] == 1 else oracle.CRC24B
            for c, F in zip(cbs, Fs):
                out.append(dict(c=c, K=c.size, F=F, crc=kind, cell=int(wl.tb_cell[t]),
                                ebn0=float(wl.tb_ebn0_db[t]), tb=t, seg=seg))
    return out


def oracle_llrs(wl, cbs=None, device="cpu"):
    """Dense int16 LLR streams (CB i's K_i+4 values at sum_{j<i}(K_j+4))."""
    import oracle
    cbs = oracle_cbs(wl) if cbs is None else cbs
    enc = [oracle.turbo_encode(cb["c"]) for cb in cbs]
    d = tuple(torch.from_numpy(np.concatenate([e[s] for e in enc])).to(device) for s in range(3))
    K = np.array([cb["K"] for cb in cbs])
    l0, l1, l2 = wlmod.channel_llr(wl, np.array([cb["cell"] for cb in cbs]), K,
                                   np.array([cb["ebn0"] for cb in cbs]), d)
    return cbs, (l0, l1, l2)


def offsets(K):
    K = np.asarray(K, np.int64)
    llr_off = np.concatenate([[0], np.cumsum(K + 4)[:-1]]) if K.size else np.zeros(0, np.int64)
    bit_off = np.concatenate([[0], np.cumsum(K)[:-1]]) if K.size else np.zeros(0, np.int64)
    return llr_off, bit_off


def oracle_batch(wl, device="cuda"):
    """A product Batch whose CB contents (segmentation, CRC, fillers) and coded
    bits are the oracle's -- the parity tests' inputs never come from the CUDA
    path -- on the shared workload channel."""
    import oracle
    from paper_1905_01141_b200 import batch as bmod
    cbs = oracle_cbs(wl)
    enc = [oracle.turbo_encode(cb["c"]) for cb in cbs]
    return bmod.from_cbs(wl, cbs, enc, device)
