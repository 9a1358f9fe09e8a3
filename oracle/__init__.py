"""ctypes binding of the CPU oracle (oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
``paper_1905_01141_b200`` never imports it (a test greps for that).

Arrays are numpy; bits are one per uint8.  See oracle.h for the definitions and
PAPER.md citations of each function.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

CRC_NONE, CRC24A, CRC24B = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc -O2 (scalar C11, no intrinsics)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-fPIC", "-shared", "-pthread",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        P = C.POINTER
        i16p, i32p, i64p, u8p, u64p = (P(C.c_int16), P(C.c_int32), P(C.c_int64), P(C.c_uint8),
                                       P(C.c_uint64))
        L.oracle_num_k.restype = C.c_int
        L.oracle_k_at.argtypes = [C.c_int]
        L.oracle_qpp_params.argtypes = [C.c_int, P(C.c_int), P(C.c_int)]
        L.oracle_qpp_index.argtypes = [C.c_int, C.c_int]
        L.oracle_crc24.argtypes = [C.c_int, u8p, C.c_int64]
        L.oracle_crc24.restype = C.c_uint32
        L.oracle_segment.argtypes = [C.c_int64, P(_Seg)]
        L.oracle_num_windows.argtypes = [C.c_int, C.c_int]
        L.oracle_turbo_encode.argtypes = [u8p, C.c_int, u8p, u8p, u8p]
        L.oracle_siso.argtypes = [i32p, i32p, i32p, i32p, C.c_int, C.c_int, i32p, i32p, i32p, i32p,
                                  i32p, u64p]
        L.oracle_siso.restype = C.c_int64
        L.oracle_siso_v.argtypes = [i32p, i32p, i32p, i32p, C.c_int, C.c_int, i32p, i32p, i32p, i32p,
                                    i32p, u64p, C.c_int]
        L.oracle_siso_v.restype = C.c_int64
        L.oracle_max_star.argtypes = [C.c_int32, C.c_int32]
        L.oracle_max_star.restype = C.c_int32
        L.oracle_logmap_correction.argtypes = [C.c_int32]
        L.oracle_logmap_correction.restype = C.c_int32
        L.oracle_nii_update.argtypes = [C.c_int, i32p, i32p, i32p, i32p]
        L.oracle_nii_update.restype = None
        L.oracle_decode_cb.argtypes = [i16p, i16p, i16p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                       C.c_int, u8p, u8p, u8p, i16p, u64p]
        L.oracle_decode_cb.restype = C.c_int64
        L.oracle_decode_cb_v.argtypes = [i16p, i16p, i16p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_int, u8p, u8p, u8p, i16p, u64p]
        L.oracle_decode_cb_v.restype = C.c_int64
        L.oracle_rm_perm.argtypes = [C.c_int]
        L.oracle_rm_params.argtypes = [C.c_int, C.c_int, P(C.c_int), P(C.c_int), P(C.c_int), P(C.c_int)]
        L.oracle_rate_match.argtypes = [u8p, u8p, u8p, C.c_int, C.c_int, C.c_int, u8p]
        L.oracle_rate_dematch.argtypes = [i16p, C.c_int, C.c_int, C.c_int, C.c_int, i16p, i16p, i16p]
        L.oracle_mi_table.argtypes = [C.c_int32]
        L.oracle_mi_table.restype = C.c_int32
        L.oracle_ext_scale.argtypes = [C.c_int32]
        L.oracle_ext_scale.restype = C.c_int32
        L.oracle_decode_batch.argtypes = [C.c_int, i32p, i32p, i32p, i64p, i64p, i16p, i16p, i16p,
                                          C.c_int, C.c_int, C.c_int, u8p, u8p, u8p, i16p, u64p]
        L.oracle_decode_batch.restype = C.c_int64
        L.oracle_decode_batch_v.argtypes = [C.c_int, i32p, i32p, i32p, i64p, i64p, i16p, i16p, i16p,
                                            C.c_int, C.c_int, C.c_int, C.c_int, u8p, u8p, u8p, i16p, u64p]
        L.oracle_decode_batch_v.restype = C.c_int64
        _lib = L
    return _lib


class _Seg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("C", "Kplus", "Kminus", "Cplus", "Cminus", "F", "L")]


def _p(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def k_table() -> list[int]:
    L = lib()
    return [L.oracle_k_at(i) for i in range(L.oracle_num_k())]


def qpp_params(K: int) -> tuple[int, int]:
    f1, f2 = C.c_int(), C.c_int()
    if lib().oracle_qpp_params(K, C.byref(f1), C.byref(f2)) != 0:
        raise ValueError(f"unsupported K={K}")
    return f1.value, f2.value


def qpp_index(K: int, i: int) -> int:
    r = lib().oracle_qpp_index(K, i)
    if r < 0:
        raise ValueError(f"bad K={K} or i={i}")
    return r


def qpp_perm(K: int) -> np.ndarray:
    return np.array([qpp_index(K, i) for i in range(K)], dtype=np.int64)


def crc24(kind: int, bits) -> int:
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    return int(lib().oracle_crc24(kind, _p(b, C.c_uint8), b.size))


def crc24a(bits) -> int:
    return crc24(CRC24A, bits)


def crc24b(bits) -> int:
    return crc24(CRC24B, bits)


def crc_attach(kind: int, bits) -> np.ndarray:
    """bits || CRC (24 parity bits, MSB first) -- the register after the payload."""
    b = np.ascontiguousarray(bits, dtype=np.uint8)
    r = crc24(kind, b)
    par = np.array([(r >> (23 - i)) & 1 for i in range(24)], dtype=np.uint8)
    return np.concatenate([b, par])


def segment(tbs: int) -> dict:
    s = _Seg()
    if lib().oracle_segment(tbs, C.byref(s)) != 0:
        raise ValueError(f"bad tbs={tbs}")
    return {n: getattr(s, n) for n, _ in _Seg._fields_}


def num_windows(K: int, wmin: int = 32) -> int:
    return lib().oracle_num_windows(K, wmin)


def segment_tb_bits(tb_payload) -> tuple[list[np.ndarray], list[int], dict]:
    """TB payload -> list of CB bit arrays (36.212 5.1.1-5.1.2: TB CRC24A, then
    CB CRC24B per CB if C > 1, leading filler zeros in CB 0).  Returns
    (cb_bits, F per CB, seg)."""
    a = np.ascontiguousarray(tb_payload, dtype=np.uint8)
    b = crc_attach(CRC24A, a)
    seg = segment(a.size)
    C_, L = seg["C"], seg["L"]
    cbs, Fs, s = [], [], 0
    for r in range(C_):
        Kr = seg["Kminus"] if r < seg["Cminus"] else seg["Kplus"]
        F = seg["F"] if r == 0 else 0
        n = Kr - L - F
        c = np.concatenate([np.zeros(F, np.uint8), b[s:s + n]])
        s += n
        if C_ > 1:
            c = crc_attach(CRC24B, c)
        cbs.append(c)
        Fs.append(F)
    assert s == b.size
    return cbs, Fs, seg


def reassemble_tb(cb_bits: list[np.ndarray], Fs: list[int], seg: dict):
    """Strip fillers and CB CRCs, concatenate, check the TB CRC24A.  Returns
    (payload or None).  A TB succeeds only if every CB does."""
    L = seg["L"]
    parts = [np.asarray(c[F:c.size - L], np.uint8) for c, F in zip(cb_bits, Fs)]
    b = np.concatenate(parts)
    if crc24a(b) != 0:
        return None
    return b[:-24]


def turbo_encode(c) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    c = np.ascontiguousarray(c, dtype=np.uint8)
    K = c.size
    d = [np.zeros(K + 4, np.uint8) for _ in range(3)]
    if lib().oracle_turbo_encode(_p(c, C.c_uint8), K, *(_p(x, C.c_uint8) for x in d)) != 0:
        raise ValueError(f"unsupported K={K}")
    return d[0], d[1], d[2]


def siso(lsys, lpar, la, tail, W: int, alpha_in=None, beta_in=None, variant: int = 0):
    """One constituent half-iteration.  Returns (le, alpha_out, beta_out, ops, violations)."""
    lsys, lpar, la = (np.ascontiguousarray(x, np.int32) for x in (lsys, lpar, la))
    tail = np.ascontiguousarray(tail, np.int32)
    K = lsys.size
    M = K // W
    ai = np.zeros((M, 8), np.int32) if alpha_in is None else np.ascontiguousarray(alpha_in, np.int32)
    bi = np.zeros((M, 8), np.int32) if beta_in is None else np.ascontiguousarray(beta_in, np.int32)
    ao, bo = np.zeros((M, 8), np.int32), np.zeros((M, 8), np.int32)
    le = np.zeros(K, np.int32)
    ops = C.c_uint64(0)
    v = lib().oracle_siso_v(_p(lsys, C.c_int32), _p(lpar, C.c_int32), _p(la, C.c_int32),
                            _p(tail, C.c_int32), K, W, _p(ai, C.c_int32), _p(bi, C.c_int32),
                            _p(ao, C.c_int32), _p(bo, C.c_int32), _p(le, C.c_int32), C.byref(ops), variant)
    return le, ao, bo, ops.value, v


def nii_update(alpha_out, beta_out):
    """NII hand-over: returns (alpha_in, beta_in) for the next iteration."""
    ao = np.ascontiguousarray(alpha_out, np.int32)
    bo = np.ascontiguousarray(beta_out, np.int32)
    M = ao.shape[0]
    ai, bi = np.zeros_like(ao), np.zeros_like(bo)
    lib().oracle_nii_update(M, _p(ao, C.c_int32), _p(bo, C.c_int32), _p(ai, C.c_int32), _p(bi, C.c_int32))
    return ai, bi


VAR_MAXLOG, VAR_SCALED, VAR_LOGMAP = 0, 1, 2


def max_star(a: int, b: int) -> int:
    """Log-MAP's max*(a, b) = max(a, b) + LUT correction (R32)."""
    return int(lib().oracle_max_star(int(a), int(b)))


def logmap_correction(d: int) -> int:
    return int(lib().oracle_logmap_correction(int(d)))
ET_NONE, ET_CRC, ET_MI = 0, 1, 2
MI_EPS = 66


def rm_perm(c: int) -> int:
    """Sub-block interleaver inter-column permutation P(c) (36.212 5.1.4.1.1)."""
    return int(lib().oracle_rm_perm(int(c)))


def rm_params(K: int, rv: int = 0) -> dict:
    R, ND, Kpi, k0 = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    if lib().oracle_rm_params(K, rv, C.byref(R), C.byref(ND), C.byref(Kpi), C.byref(k0)):
        raise ValueError("bad K / rv")
    return dict(R=R.value, ND=ND.value, Kpi=Kpi.value, k0=k0.value, Ncb=3 * Kpi.value)


def rate_match(d, E: int, rv: int = 0) -> np.ndarray:
    """d = (d0, d1, d2) coded bits (K+4 each) -> E selected bits."""
    d0, d1, d2 = (np.ascontiguousarray(x, np.uint8) for x in d)
    e = np.zeros(E, np.uint8)
    if lib().oracle_rate_match(_p(d0, C.c_uint8), _p(d1, C.c_uint8), _p(d2, C.c_uint8), d0.size - 4, E, rv,
                               _p(e, C.c_uint8)):
        raise ValueError("bad arguments")
    return e


def rate_dematch(e, K: int, rv: int = 0, h=None):
    """E soft values -> (h0, h1, h2) soft buffers (K+4 each); h: previous buffers (HARQ) or None."""
    e = np.ascontiguousarray(e, np.int16)
    hs = [np.zeros(K + 4, np.int16) for _ in range(3)] if h is None else [np.array(x, np.int16) for x in h]
    if lib().oracle_rate_dematch(_p(e, C.c_int16), K, e.size, rv, int(h is not None), *(_p(x, C.c_int16) for x in hs)):
        raise ValueError("bad arguments")
    return tuple(hs)


def mi_table(a: int) -> int:
    """Q16 MI of an LLR of magnitude a/8 (R29)."""
    return int(lib().oracle_mi_table(int(a)))


def ext_scale(x: int) -> int:
    """The scaled variant's extrinsic map floor(3x/4) (R28)."""
    return int(lib().oracle_ext_scale(int(x)))


def decode_cb(d0, d1, d2, F: int = 0, crc_kind: int = CRC24B, max_iters: int = 8,
              early_term: bool = False, wmin: int = 32, variant: int = VAR_MAXLOG) -> dict:
    d0, d1, d2 = (np.ascontiguousarray(x, np.int16) for x in (d0, d1, d2))
    K = d0.size - 4
    bits = np.zeros(K, np.uint8)
    ext = np.zeros(K, np.int16)
    ok, it, ops = C.c_uint8(), C.c_uint8(), C.c_uint64(0)
    v = lib().oracle_decode_cb_v(_p(d0, C.c_int16), _p(d1, C.c_int16), _p(d2, C.c_int16), K, F,
                                 crc_kind, max_iters, int(early_term), wmin, variant, _p(bits, C.c_uint8),
                               C.byref(ok), C.byref(it), _p(ext, C.c_int16), C.byref(ops))
    if v < 0:
        raise ValueError("invalid arguments")
    return {"bits": bits, "crc_ok": ok.value, "iters": it.value, "ext": ext, "ops": ops.value,
            "violations": v}


def decode_batch(K, F, crc_kind, llr_off, bit_off, d0, d1, d2, max_iters: int, early_term: bool,
                 nthreads: int, want_ext: bool = True, variant: int = VAR_MAXLOG) -> dict:
    K = np.ascontiguousarray(K, np.int32)
    n = K.size
    F = np.ascontiguousarray(F, np.int32)
    crc_kind = np.ascontiguousarray(crc_kind, np.int32)
    llr_off = np.ascontiguousarray(llr_off, np.int64)
    bit_off = np.ascontiguousarray(bit_off, np.int64)
    d0, d1, d2 = (np.ascontiguousarray(x, np.int16) for x in (d0, d1, d2))
    nbits = int((bit_off + K).max()) if n else 0
    bits = np.zeros(nbits, np.uint8)
    ext = np.zeros(nbits, np.int16) if want_ext else None
    ok = np.zeros(n, np.uint8)
    it = np.zeros(n, np.uint8)
    ops = C.c_uint64(0)
    v = lib().oracle_decode_batch_v(n, _p(K, C.c_int32), _p(F, C.c_int32), _p(crc_kind, C.c_int32),
                                    _p(llr_off, C.c_int64), _p(bit_off, C.c_int64),
                                    _p(d0, C.c_int16), _p(d1, C.c_int16), _p(d2, C.c_int16),
                                    max_iters, int(early_term), variant, nthreads, _p(bits, C.c_uint8),
                                  _p(ok, C.c_uint8), _p(it, C.c_uint8),
                                  _p(ext, C.c_int16) if want_ext else None, C.byref(ops))
    return {"bits": bits, "crc_ok": ok, "iters": it, "ext": ext, "ops": ops.value, "violations": v}
