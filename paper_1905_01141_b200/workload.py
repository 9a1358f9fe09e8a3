"""Seeded synthetic workload generator -- shared by the oracle side (tests,
cpu baseline) and the CUDA side (bench, GPU tests).

This module holds NONE of the method's arithmetic: no CRC, no segmentation,
no encoding, no decoding.  It only draws what the paper's workload draws
(UEs of cells sending transport blocks over a radio channel)
and maps already-encoded bits to quantised channel LLRs:

* cell / UE / code-block structure of BASELINE.json configs 1-5 (DESIGN.md
  "input recipe"; readings R21-R24);
* uniform random information bits, Eb/N0 draws, TBS draws;
* BPSK / QPSK over AWGN and the LLR quantiser (R8-R10):
  L = -2*a*y/sigma^2 (positive => bit 1), Lq = clamp(round_half_away(8L), +-8192).

Randomness is one ``torch.Generator`` per (config, seed, cell) so a shard of
cells generates the same values whatever the number of ranks (SPEC.md:290
determinism).  Values are identical for a given device type; parity tests
always feed the SAME stored buffer to both sides.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

# The 188 interleaver sizes of the LTE turbo code (closed form:
# 40..512 step 8, 528..1024 step 16, 1056..2048 step 32, 2112..6144 step 64).
# Used only to DRAW a K for config 5 -- the (f1, f2) values live elsewhere.
K_SIZES = (list(range(40, 513, 8)) + list(range(528, 1025, 16)) + list(range(1056, 2049, 32))
           + list(range(2112, 6145, 64)))

CRC_NONE, CRC24A, CRC24B = 0, 1, 2
LLR_SCALE = 8.0
LLR_SAT = 8192


def _cell_seed(cfg: int, seed: int, cell: int, stream: int) -> int:
    """SplitMix64 finaliser of the key (cfg, seed, cell, stream) -> 63-bit seed."""
    x = (cfg * 0x9E3779B97F4A7C15 + seed * 0xBF58476D1CE4E5B9 + cell * 0x94D049BB133111EB
         + stream * 0xD6E8FEB86659FD93) & 0xFFFFFFFFFFFFFFFF
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    x ^= x >> 31
    return x & 0x7FFFFFFFFFFFFFFF


def generator(cfg: int, seed: int, cell: int, stream: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(_cell_seed(cfg, seed, cell, stream))
    return g


@dataclass
class Workload:
    """A batch of code blocks.  Standalone CBs carry K-24 info bits (+CRC24B);
    TB configs carry whole transport blocks that each side segments itself."""
    name: str
    cfg: int
    seed: int
    max_iters: int
    early_term: bool
    modulation: str                      # "bpsk" | "qpsk"
    cells: list[int]
    # per transport block (standalone CBs are 1-CB "TBs" with tbs = K - 24, kind "cb")
    tb_kind: str                         # "cb" (standalone CBs, CRC24B) | "tb" (36.212 TBs)
    tbs: np.ndarray                      # int64 [n_tb] info bits per TB
    tb_cell: np.ndarray                  # int32 [n_tb]
    tb_ebn0_db: np.ndarray               # float64 [n_tb]  (per-CB draws: one TB per CB)
    tb_K: np.ndarray | None = None       # int32 [n_tb] (kind "cb" only)
    payload: list = field(default_factory=list)   # per TB: uint8 tensor [tbs]

    @property
    def n_tb(self) -> int:
        return int(self.tbs.size)


def _uniform(g, lo, hi, n, device):
    return (lo + (hi - lo) * torch.rand(n, generator=g, dtype=torch.float64, device=device)).cpu().numpy()


def make_workload(cfg: int, seed: int = 0, cells=None, device="cpu", scale: float = 1.0) -> Workload:
    """BASELINE.json configs 1-5 (one TTI for 5).  ``cells`` selects a shard of
    cells (multi-GPU); ``scale`` < 1 shrinks the per-cell CB count for small
    CPU tests while keeping every other distribution."""
    dev = torch.device(device)
    if cfg == 1:        # 32 CBs K=1056, BPSK 1.5 dB, 6 fixed iterations
        n_cells, per_cell, mod, I, et = 1, max(1, int(32 * scale)), "bpsk", 6, False
    elif cfg == 2:      # one subframe: TB 75376, QPSK, Eb/N0 ~ U[1.0,2.5] per TB, ET max 8
        n_cells, per_cell, mod, I, et = 1, 1, "qpsk", 8, True
    elif cfg == 3:      # 100 cells x 10 UEs, TBS ~ U{1000..75376}, Eb/N0 ~ U[0.5,3] per UE
        n_cells, per_cell, mod, I, et = 100, max(1, int(10 * scale)), "qpsk", 8, True
    elif cfg == 4:      # 256 cells x 256 CBs K=6144, BPSK 1.0 dB, 8 fixed iterations
        n_cells, per_cell, mod, I, et = 256, max(1, int(256 * scale)), "bpsk", 8, False
    elif cfg == 5:      # one TTI: 20 cells x 10 CBs, K ~ U(table), Eb/N0 ~ U[0.5,3] per CB
        n_cells, per_cell, mod, I, et = 20, max(1, int(10 * scale)), "qpsk", 8, True
    else:
        raise ValueError(f"unknown config {cfg}")
    cells = list(range(n_cells)) if cells is None else list(cells)
    tbs, tb_cell, ebn0, tbK, payload = [], [], [], [], []
    for cell in cells:
        g = generator(cfg, seed, cell, 0, "cpu")          # structure draws: always on CPU
        if cfg == 1:
            Ks = np.full(per_cell, 1056)
            e = np.full(per_cell, 1.5)
        elif cfg == 4:
            Ks = np.full(per_cell, 6144)
            e = np.full(per_cell, 1.0)
        elif cfg == 5:
            Ks = np.array(K_SIZES)[torch.randint(0, len(K_SIZES), (per_cell,), generator=g).numpy()]
            e = _uniform(g, 0.5, 3.0, per_cell, "cpu")
        elif cfg == 2:
            Ks = None
            t = np.array([75376])
            e = _uniform(g, 1.0, 2.5, 1, "cpu")
        else:  # cfg 3
            Ks = None
            t = torch.randint(1000, 75377, (per_cell,), generator=g).numpy()
            e = _uniform(g, 0.5, 3.0, per_cell, "cpu")
        if Ks is not None:
            t = Ks - 24
            tbK.extend(int(k) for k in Ks)
        gb = generator(cfg, seed, cell, 1, dev)            # payload bits
        for n in t:
            payload.append(torch.randint(0, 2, (int(n),), generator=gb, device=dev, dtype=torch.uint8))
        tbs.extend(int(x) for x in t)
        tb_cell.extend([cell] * len(t))
        ebn0.extend(float(x) for x in e)
    return Workload(name=f"cfg{cfg}", cfg=cfg, seed=seed, max_iters=I, early_term=et, modulation=mod,
                    cells=cells, tb_kind="cb" if cfg in (1, 4, 5) else "tb",
                    tbs=np.array(tbs, np.int64), tb_cell=np.array(tb_cell, np.int32),
                    tb_ebn0_db=np.array(ebn0, np.float64),
                    tb_K=np.array(tbK, np.int32) if tbK else None, payload=payload)


def noise_sigma2(K: np.ndarray, ebn0_db: np.ndarray, modulation: str) -> tuple[np.ndarray, np.ndarray]:
    """(amplitude a, per-dimension noise variance sigma^2) per CB (R10):
    R = K/(3K+12); BPSK a = 1, N0 = 1/(R*ebn0); QPSK a = 1/sqrt2, N0 = 1/(2R*ebn0); sigma^2 = N0/2."""
    K = np.asarray(K, np.float64)
    R = K / (3 * K + 12)
    ebn0 = 10.0 ** (np.asarray(ebn0_db, np.float64) / 10.0)
    if modulation == "bpsk":
        a = np.ones_like(R)
        n0 = 1.0 / (R * ebn0)
    else:
        a = np.full_like(R, 1.0 / math.sqrt(2.0))
        n0 = 1.0 / (2.0 * R * ebn0)
    return a, n0 / 2.0


def quantise(L: torch.Tensor) -> torch.Tensor:
    """Lq = clamp(round_half_away_from_zero(8 L), -8192, 8192) as int16 (BASELINE cfg 1)."""
    q = torch.sign(L) * torch.floor(torch.abs(L) * LLR_SCALE + 0.5)
    return q.clamp_(-LLR_SAT, LLR_SAT).to(torch.int16)


def channel_llr(wl: Workload, cb_cell: np.ndarray, cb_K: np.ndarray, cb_ebn0_db: np.ndarray,
                d: tuple[torch.Tensor, torch.Tensor, torch.Tensor], device=None):
    """Map coded bits d0,d1,d2 (uint8, dense layout: CB i's K_i+4 bits at
    sum_{j<i}(K_j+4)) to int16 LLRs with noise drawn per cell (cells in the
    order they appear).  Returns (l0, l1, l2) on ``device`` (default: d's)."""
    dev = d[0].device if device is None else torch.device(device)
    cb_cell = np.asarray(cb_cell)
    lens = np.asarray(cb_K, np.int64) + 4
    offs = np.concatenate([[0], np.cumsum(lens)])
    a, s2 = noise_sigma2(cb_K, cb_ebn0_db, wl.modulation)
    out = [torch.empty(int(offs[-1]), dtype=torch.int16, device=dev) for _ in range(3)]
    # CBs of a cell are contiguous
    starts = np.flatnonzero(np.r_[True, cb_cell[1:] != cb_cell[:-1]]) if cb_cell.size else []
    bounds = list(starts) + [cb_cell.size]
    for ci in range(len(bounds) - 1):
        i0, i1 = bounds[ci], bounds[ci + 1]
        cell = int(cb_cell[i0])
        g = generator(wl.cfg, wl.seed, cell, 2, dev)
        lo, hi = int(offs[i0]), int(offs[i1])
        rep = torch.from_numpy(lens[i0:i1]).to(dev)
        amp = torch.repeat_interleave(torch.from_numpy(a[i0:i1]).to(dev), rep)
        sig2 = torch.repeat_interleave(torch.from_numpy(s2[i0:i1]).to(dev), rep)
        n = torch.randn((3, hi - lo), generator=g, dtype=torch.float64, device=dev)
        for s in range(3):
            x = amp * (1.0 - 2.0 * d[s][lo:hi].to(dev, torch.float64))     # bit 0 -> +a, 1 -> -a
            y = x + torch.sqrt(sig2) * n[s]
            L = -2.0 * amp * y / sig2                                      # positive => bit 1
            out[s][lo:hi] = quantise(L)
    return tuple(out)


def make_cb_workload(Ks, ebn0_db=1.0, seed=0, modulation="qpsk", device="cpu", max_iters=8,
                     early_term=False, cfg=9) -> Workload:
    """Standalone CBs of the given sizes (K-24 random bits + CRC24B each), all on
    one synthetic cell, one Eb/N0 for all: probes and tests of single sizes."""
    Ks = [int(k) for k in Ks]
    dev = torch.device(device)
    gb = generator(cfg, seed, 0, 1, dev)
    payload = [torch.randint(0, 2, (k - 24,), generator=gb, device=dev, dtype=torch.uint8) for k in Ks]
    n = len(Ks)
    return Workload(name=f"cb{n}", cfg=cfg, seed=seed, max_iters=max_iters, early_term=early_term,
                    modulation=modulation, cells=[0], tb_kind="cb", tbs=np.array([k - 24 for k in Ks], np.int64),
                    tb_cell=np.zeros(n, np.int32), tb_ebn0_db=np.full(n, float(ebn0_db)),
                    tb_K=np.array(Ks, np.int32), payload=payload)
