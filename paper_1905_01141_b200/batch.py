"""Product-side batch assembly for a synthetic workload: CB packing via libcrn
(crn_tb_build_cbs_batch on the device for transport blocks, descriptors, row
a1), device encoding via crn_encode_batch
(the paper's encoding function), then the shared workload
channel (``build``, used by bench.py); or the same dense layout around CB
contents and coded bits the caller supplies (``from_cbs``: the parity tests
pass the oracle's, so no oracle input comes from the CUDA path).  Never
touches oracle/.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import crn
from . import workload as wlmod


@dataclass
class Batch:
    wl: wlmod.Workload
    desc: np.ndarray          # crn.DESC_DTYPE [n_cb] (host)
    cb_cell: np.ndarray
    cb_tb: np.ndarray         # TB index per CB
    cb_ebn0: np.ndarray
    info: torch.Tensor        # uint8 [sum K] CB contents (device)
    coded: tuple              # d0, d1, d2 uint8 [sum (K+4)] (device)
    llr: tuple                # l0, l1, l2 int16 [sum (K+4)] (device)

    @property
    def n_cb(self) -> int:
        return int(self.desc.size)

    @property
    def K(self) -> np.ndarray:
        return self.desc["K"].astype(np.int32)

    @property
    def n_words(self) -> int:
        return int((self.desc["bit_off"] + (self.desc["K"] + 31) // 32).max()) if self.n_cb else 0

    @property
    def n_llr(self) -> int:
        return int((self.desc["llr_off"] + self.desc["K"] + 4).max()) if self.n_cb else 0

    def info_bits(self) -> int:
        """Decoded information bits per CB: K - F - 24 (DESIGN.md metric)."""
        return int((self.desc["K"] - self.desc["F"] - 24).sum())


def build(wl: wlmod.Workload, device="cuda") -> Batch:
    if wl.tb_kind == "tb":
        return _build_tb(wl, device)
    dev = torch.device(device)
    descs, infos, cells, tbs, ebn0 = [], [], [], [], []
    bit = llr = word = 0
    for t in range(wl.n_tb):
        if wl.tb_kind == "cb":
            K = int(wl.tb_K[t])
            d = np.zeros(1, crn.DESC_DTYPE)
            d["K"], d["F"], d["crc_kind"] = K, 0, crn.CRC24B
            d["ext_off"], d["llr_off"], d["bit_off"] = bit, llr, word
            infos.append(torch.cat([wl.payload[t].to(dev), torch.zeros(24, dtype=torch.uint8, device=dev)]))
        else:
            cbb, d = crn.tb_build_cbs(wl.payload[t].cpu().numpy(), base_bit=bit, base_llr=llr, base_word=word)
            infos.append(torch.from_numpy(cbb).to(dev))
        descs.append(d)
        n = d.size
        cells += [int(wl.tb_cell[t])] * n
        tbs += [t] * n
        ebn0 += [float(wl.tb_ebn0_db[t])] * n
        bit += int(d["K"].sum())
        llr += int((d["K"] + 4).sum())
        word += int(((d["K"] + 31) // 32).sum())
    desc = np.concatenate(descs) if descs else np.zeros(0, crn.DESC_DTYPE)
    info = torch.cat(infos) if infos else torch.zeros(0, dtype=torch.uint8, device=dev)
    coded = tuple(torch.empty(llr, dtype=torch.uint8, device=dev) for _ in range(3))
    crn.encode_batch(desc, info, wl.tb_kind == "cb", *coded)
    cell = np.array(cells, np.int32)
    e = np.array(ebn0, np.float64)
    l0, l1, l2 = wlmod.channel_llr(wl, cell, desc["K"], e, coded)
    return Batch(wl=wl, desc=desc, cb_cell=cell, cb_tb=np.array(tbs, np.int64), cb_ebn0=e, info=info,
                 coded=coded, llr=(l0, l1, l2))


def _build_tb(wl: wlmod.Workload, device="cuda") -> Batch:
    """Transport-block configs on the device: TB CRC24A, 36.212 segmentation with
    fillers and CB CRC24B (crn_tb_build_cbs_batch), then the turbo encoder."""
    dev = torch.device(device)
    tbs = np.asarray(wl.tbs, np.int64)
    pay = torch.cat([p.to(dev) for p in wl.payload]) if wl.n_tb else torch.zeros(1, dtype=torch.uint8, device=dev)
    off = np.concatenate([[0], np.cumsum(tbs)[:-1]]).astype(np.int64) if wl.n_tb else np.zeros(0, np.int64)
    desc, info = crn.tb_build_cbs_batch(tbs, off, pay)
    llr = int((desc["K"] + 4).sum())
    coded = tuple(torch.empty(max(llr, 1), dtype=torch.uint8, device=dev) for _ in range(3))
    crn.encode_batch(desc, info, False, *coded)
    cb_tb = desc["reserved"].astype(np.int64)
    cell = np.asarray(wl.tb_cell, np.int32)[cb_tb]
    e = np.asarray(wl.tb_ebn0_db, np.float64)[cb_tb]
    coded = tuple(x[:llr] for x in coded)
    l0, l1, l2 = wlmod.channel_llr(wl, cell, desc["K"], e, coded)
    desc["reserved"] = 0
    return Batch(wl=wl, desc=desc, cb_cell=cell, cb_tb=cb_tb, cb_ebn0=e, info=info, coded=coded, llr=(l0, l1, l2))


def outputs(b: Batch, device="cuda", want_ext: bool = True):
    dev = torch.device(device)
    bits = torch.zeros(max(b.n_words, 1), dtype=torch.int32, device=dev)
    ok = torch.zeros(max(b.n_cb, 1), dtype=torch.uint8, device=dev)
    it = torch.zeros(max(b.n_cb, 1), dtype=torch.uint8, device=dev)
    ext = torch.zeros(max(int(b.desc["K"].sum()), 1), dtype=torch.int16, device=dev) if want_ext else None
    return bits, ok, it, ext


def from_cbs(wl: wlmod.Workload, cbs, coded, device="cuda") -> Batch:
    """Batch of the given CBs in the dense layout ``build`` uses (CB i's K_i bits
    at sum K, K_i+4 coded bits / LLRs at sum (K+4), ceil(K_i/32) words at the
    word sum).  cbs: per CB a dict with c (uint8 bits incl. CRC and fillers), K,
    F, crc, cell, ebn0, tb; coded: per CB (d0, d1, d2) uint8 arrays of K+4."""
    dev = torch.device(device)
    n = len(cbs)
    desc = np.zeros(n, crn.DESC_DTYPE)
    K = np.array([cb["K"] for cb in cbs], np.int64)
    desc["K"], desc["F"], desc["crc_kind"] = K, [cb["F"] for cb in cbs], [cb["crc"] for cb in cbs]
    z = np.zeros(1, np.int64)
    desc["ext_off"] = np.concatenate([z, np.cumsum(K)[:-1]]) if n else K
    desc["llr_off"] = np.concatenate([z, np.cumsum(K + 4)[:-1]]) if n else K
    desc["bit_off"] = np.concatenate([z, np.cumsum((K + 31) // 32)[:-1]]) if n else K
    info = torch.from_numpy(np.concatenate([cb["c"] for cb in cbs]).astype(np.uint8)).to(dev)
    cd = tuple(torch.from_numpy(np.concatenate([e[s] for e in coded]).astype(np.uint8)).to(dev) for s in range(3))
    cell = np.array([cb["cell"] for cb in cbs], np.int32)
    e = np.array([cb["ebn0"] for cb in cbs], np.float64)
    l0, l1, l2 = wlmod.channel_llr(wl, cell, desc["K"], e, cd)
    return Batch(wl=wl, desc=desc, cb_cell=cell, cb_tb=np.array([cb["tb"] for cb in cbs], np.int64), cb_ebn0=e,
                 info=info, coded=cd, llr=(l0, l1, l2))
