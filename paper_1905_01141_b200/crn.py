"""Thin ctypes binding of libcrn (include/crn.h) -- argument marshalling only.

Every function here has the same name as its C entry point minus the ``crn_``
prefix.  Device buffers are passed as torch CUDA tensors (``data_ptr()``),
host buffers as numpy arrays; streams default to torch's current stream.  No
step of the decoding path runs in Python: if libcrn.so is missing or no sm_100
device is present the calls raise -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("CRN_LIB") or os.path.join(HERE, "libcrn.so")   # CRN_LIB: A/B experiments only

CRN_OK, CRN_EINVAL, CRN_ECUDA, CRN_ENOMEM, CRN_ENODEV = 0, -1, -2, -3, -4
CRC_NONE, CRC24A, CRC24B = 0, 1, 2
DESC_ON_DEVICE = 1
EXT_SCALED = 2
PURGE = 4
VARIANT_MAXLOG, VARIANT_SCALED, VARIANT_LOGMAP = 0, 1, 2
ET_NONE, ET_CRC, ET_MI = 0, 1, 2

DESC_DTYPE = np.dtype([("K", "<i4"), ("F", "<i4"), ("crc_kind", "<i4"), ("reserved", "<i4"),
                       ("llr_off", "<i8"), ("bit_off", "<i8"), ("ext_off", "<i8")])


class Seg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("C", "Kplus", "Kminus", "Cplus", "Cminus", "F", "L")]


class TtiGroup(C.Structure):
    _fields_ = [("desc", C.c_void_p), ("n_cb", C.c_int32), ("reserved", C.c_int32),
                ("llr_sys", C.c_void_p), ("llr_p1", C.c_void_p), ("llr_p2", C.c_void_p),
                ("n_llr", C.c_int64), ("out_bits", C.c_void_p), ("n_words", C.c_int64),
                ("crc_ok", C.c_void_p), ("iters_used", C.c_void_p)]


class TtiTiming(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("release_us", "submitted_us", "complete_us", "latency_us",
                                          "device_us", "upload_us", "decode_start_us", "decode_end_us")]


class CrnError(RuntimeError):
    pass


_lib = None
P = C.POINTER
vp, i16p, i32p, i64p, u8p, u32p = C.c_void_p, P(C.c_int16), P(C.c_int32), P(C.c_int64), P(C.c_uint8), P(C.c_uint32)

_SIGS = {
    "crn_decode_batch": (C.c_int, [vp, vp, vp, i32p, C.c_int32, C.c_int32, vp, vp]),
    "crn_decode_batch_ex": (C.c_int, [vp, C.c_int32, vp, vp, vp, C.c_int32, C.c_int32, C.c_int32,
                                      vp, vp, vp, vp, vp, C.c_size_t, vp]),
    "crn_workspace_bytes": (C.c_size_t, [vp, C.c_int32]),
    "crn_plan_create": (C.c_int, [vp, C.c_int32, P(vp)]),
    "crn_plan_decode": (C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, vp, vp, vp, vp, vp]),
    "crn_plan_launches": (C.c_int, [vp]),
    "crn_task_layout": (C.c_int, [vp, C.c_int32, C.c_int32, i32p, i32p, i32p]),
    "crn_plan_layout": (C.c_int, [vp, i32p, C.c_int32]),
    "crn_plan_set_variant": (C.c_int, [vp, C.c_int32]),
    "crn_plan_set_purge": (C.c_int, [vp, C.c_int32]),
    "crn_plan_set_grid": (C.c_int, [vp, C.c_int32]),
    "crn_plan_set_llr_format": (C.c_int, [vp, C.c_int32, C.c_int32]),
    "crn_plan_llr_bytes": (C.c_int, [vp]),
    "crn_plan_decode_host": (C.c_int, [vp, vp, vp, vp, C.c_int32, C.c_int32, vp, vp, vp, C.c_int32, vp]),
    "crn_plan_chunks": (C.c_int, [vp]),
    "crn_stream_run": (C.c_int, [vp, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_int32, vp]),
    "crn_stream_run_ex": (C.c_int, [vp, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_int32, C.c_int32, vp]),
    "crn_plan_destroy": (None, [vp]),
    "crn_counted_ops": (C.c_int64, [i32p, C.c_int32, u8p, C.c_int32]),
    "crn_kpi_iterations": (C.c_int, [u8p, u8p, C.c_int32, C.c_int32, u8p]),
    "crn_encode_batch": (C.c_int, [vp, C.c_int32, vp, C.c_int32, vp, vp, vp, vp]),
    "crn_encode_batch_packed": (C.c_int, [vp, C.c_int32, vp, C.c_int32, vp, vp, vp, vp]),
    "crn_tb_build_cbs": (C.c_int, [u8p, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_int64, u8p, vp,
                                   i32p]),
    "crn_tb_build_cbs_batch": (C.c_int, [i64p, i64p, C.c_int32, vp, C.c_int32, vp, vp, i32p, vp]),
    "crn_rate_dematch_batch": (C.c_int, [vp, C.c_int32, vp, C.c_int32, vp, vp, vp, vp]),
    "crn_rate_match_batch": (C.c_int, [vp, C.c_int32, vp, vp, vp, vp, vp]),
    "crn_rate_match_batch_packed": (C.c_int, [vp, C.c_int32, vp, vp, vp, vp, vp]),
    "crn_tb_verdict_batch": (C.c_int, [vp, C.c_int32, vp, C.c_int32, vp, vp, vp, vp, vp]),
    "crn_tb_reassemble": (C.c_int, [u32p, vp, u8p, C.c_int32, C.c_int64, u8p]),
    "crn_segment_tb": (C.c_int, [C.c_int64, P(Seg)]),
    "crn_qpp_params": (C.c_int, [C.c_int32, i32p, i32p]),
    "crn_windows": (C.c_int, [C.c_int32, i32p, i32p]),
    "crn_crc24a": (C.c_uint32, [u8p, C.c_int64]),
    "crn_crc24b": (C.c_uint32, [u8p, C.c_int64]),
    "crn_strerror": (C.c_char_p, [C.c_int]),
    "crn_last_error": (C.c_char_p, []),
    "crn_device_info": (C.c_int, [i32p, i32p, i32p, i32p]),
    "crn_mi_table": (C.c_int, [i32p]),
    "crn_logmap_lut": (C.c_int, [i32p]),
    "crn_decode_kernel_info": (C.c_int, [i32p, i32p, i32p, i32p]),
    "crn_ubench_int16x2": (C.c_int, [C.c_int32, i64p, P(C.c_float), i64p]),
}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise CrnError(f"{SO} is not built: run paper_1905_01141_b200.build.build() (no CPU fallback)")
        L = C.CDLL(SO)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("CRN_LIB") and not hasattr(L, name):
                continue                    # A/B experiments may load an older build
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _chk(rc: int, what: str):
    if rc < 0:
        detail = lib().crn_last_error().decode()
        raise CrnError(f"{what}: {lib().crn_strerror(rc).decode()} ({rc})" + (f" [{detail}]" if detail else ""))
    return rc


def _ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def _np(a, ct):
    return a.ctypes.data_as(P(ct))


def _stream(stream):
    if stream is not None:
        return stream if isinstance(stream, int) else stream.cuda_stream
    import torch
    return torch.cuda.current_stream().cuda_stream


def _cuda_dev(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise CrnError("device buffers must be CUDA tensors (no CPU fallback)")


# ------------------------------------------------------------------ decode
def decode_batch(l0, l1, l2, K, n_cb: int, iters: int, out_bits, crc_ok) -> None:
    _cuda_dev(l0, l1, l2, out_bits, crc_ok)
    Kh = np.ascontiguousarray(K, np.int32)
    _chk(lib().crn_decode_batch(_ptr(l0), _ptr(l1), _ptr(l2), _np(Kh, C.c_int32), n_cb, iters,
                                _ptr(out_bits), _ptr(crc_ok)), "crn_decode_batch")


def decode_batch_ex(desc, n_cb: int, l0, l1, l2, max_iters: int, early_term: bool, flags: int, out_bits,
                    crc_ok, iters_used=None, ext_out=None, workspace=None, workspace_bytes: int = 0,
                    stream=None) -> None:
    _cuda_dev(l0, l1, l2, out_bits, crc_ok, iters_used, ext_out)
    if flags & DESC_ON_DEVICE:
        dptr = desc.data_ptr()
    else:
        desc = np.ascontiguousarray(desc, DESC_DTYPE)
        dptr = desc.ctypes.data
    _chk(lib().crn_decode_batch_ex(dptr, n_cb, _ptr(l0), _ptr(l1), _ptr(l2), max_iters, int(early_term),
                                   flags, _ptr(out_bits), _ptr(crc_ok), _ptr(iters_used), _ptr(ext_out),
                                   _ptr(workspace), workspace_bytes, _stream(stream)),
         "crn_decode_batch_ex")


def task_layout(desc: np.ndarray, spread_to: int = 0):
    """crn_task_layout (host only): (task_of_cb[n_cb], task_info[n_tasks, 4] = K, n_pairs,
    windows, group flag, units)."""
    desc = np.ascontiguousarray(desc, DESC_DTYPE)
    n = desc.size
    tof = np.zeros(max(n, 1), np.int32)
    info = np.zeros((n + 1, 4), np.int32)
    units = np.zeros(1, np.int32)
    nt = lib().crn_task_layout(desc.ctypes.data if n else None, n, spread_to, _np(tof, C.c_int32),
                               _np(info, C.c_int32), _np(units, C.c_int32))
    _chk(nt if nt < 0 else 0, "crn_task_layout")
    return tof[:n], info[:nt], int(units[0])


def workspace_bytes(n_cb: int = 0) -> int:
    """crn_workspace_bytes(NULL, n_cb): caller workspace for a batch of n_cb CBs."""
    return int(lib().crn_workspace_bytes(None, n_cb))


class Plan:
    """crn_plan_create / crn_plan_decode / crn_plan_destroy."""

    def __init__(self, desc):
        self.desc = np.ascontiguousarray(desc, DESC_DTYPE)
        h = C.c_void_p()
        _chk(lib().crn_plan_create(self.desc.ctypes.data, self.desc.size, C.byref(h)), "crn_plan_create")
        self.h = h

    def decode(self, l0, l1, l2, max_iters: int, early_term: bool, out_bits, crc_ok, iters_used=None,
               ext_out=None, stream=None) -> None:
        _cuda_dev(l0, l1, l2, out_bits, crc_ok, iters_used, ext_out)
        self._check_llr(l0, l1, l2)
        _chk(lib().crn_plan_decode(self.h, _ptr(l0), _ptr(l1), _ptr(l2), max_iters, int(early_term),
                                   _ptr(out_bits), _ptr(crc_ok), _ptr(iters_used), _ptr(ext_out),
                                   _stream(stream)), "crn_plan_decode")

    def decode_host(self, h0, h1, h2, max_iters: int, early_term: bool, h_bits, h_ok, h_iters=None,
                    n_chunks: int = 0, stream=None) -> None:
        """crn_plan_decode_host: every buffer is a HOST (CPU, ideally pinned) torch tensor."""
        for t in (h0, h1, h2, h_bits, h_ok, h_iters):
            if t is not None and t.is_cuda:
                raise CrnError("crn_plan_decode_host takes host buffers")
        self._check_llr(h0, h1, h2)
        _chk(lib().crn_plan_decode_host(self.h, _ptr(h0), _ptr(h1), _ptr(h2), max_iters, int(early_term),
                                        _ptr(h_bits), _ptr(h_ok), _ptr(h_iters), n_chunks, _stream(stream)),
             "crn_plan_decode_host")

    def set_variant(self, variant: int) -> None:
        _chk(lib().crn_plan_set_variant(self.h, variant), "crn_plan_set_variant")

    def set_purge(self, on: bool) -> None:
        _chk(lib().crn_plan_set_purge(self.h, int(on)), "crn_plan_set_purge")

    def set_grid(self, max_ctas: int) -> None:
        _chk(lib().crn_plan_set_grid(self.h, max_ctas), "crn_plan_set_grid")

    def set_llr_format(self, bits: int, shift: int = 0) -> None:
        """crn_plan_set_llr_format: 16 (int16 LLRs) or 8 (int8 LLRs read as x * 2^shift);
        the LLR tensors of later decode / decode_host calls must then be int8."""
        _chk(lib().crn_plan_set_llr_format(self.h, bits, shift), "crn_plan_set_llr_format")

    @property
    def llr_bytes(self) -> int:
        return int(lib().crn_plan_llr_bytes(self.h))

    def _check_llr(self, *ts):
        import torch
        want = torch.int8 if self.llr_bytes == 1 else torch.int16
        for t in ts:
            if t.dtype != want:
                raise CrnError(f"LLR tensors must be {want} for this plan's LLR format, got {t.dtype}")

    @property
    def chunks(self) -> int:
        return int(lib().crn_plan_chunks(self.h))

    def layout(self) -> np.ndarray:
        """crn_plan_layout: the task index of every CB (diagnostic)."""
        out = np.zeros(self.desc.size, np.int32)
        _chk(lib().crn_plan_layout(self.h, _np(out, C.c_int32), self.desc.size), "crn_plan_layout")
        return out

    @property
    def launches(self) -> int:
        return int(lib().crn_plan_launches(self.h))

    def close(self):
        if self.h:
            lib().crn_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


STREAM_MERGED = 1
STREAM_STAGES = 2
STREAM_ZEROCOPY = 4
STREAM_LLR8 = 8


def stream_llr8_shift(s: int) -> int:
    return s << 8


def stream_run(groups, n_tti: int, n_groups: int, period_us: float, max_iters: int, early_term: bool,
               flags: int = 0):
    """crn_stream_run.  groups: list (length n_tti * n_groups, TTI-major) of dicts with
    HOST arrays desc (numpy DESC_DTYPE), l0/l1/l2 (int16 tensors, pinned), bits (int32 tensor),
    ok (uint8 tensor), it (uint8 tensor or None).  Returns a numpy structured array of timings."""
    import torch
    arr = (TtiGroup * len(groups))()
    keep = []
    want = torch.int8 if flags & STREAM_LLR8 else torch.int16
    for x, g in enumerate(groups):
        d = np.ascontiguousarray(g["desc"], DESC_DTYPE)
        keep.append(d)
        for k in ("l0", "l1", "l2", "bits", "ok", "it"):
            if g.get(k) is not None and g[k].is_cuda:
                raise CrnError("crn_stream_run takes host buffers")
        # the runtime copies n_llr elements of the flag's width from each stream
        for k in ("l0", "l1", "l2"):
            if g[k].dtype != want:
                raise CrnError(f"group {x}: LLR tensors must be {want} for these flags, got {g[k].dtype}")
        if not (g["l0"].numel() == g["l1"].numel() == g["l2"].numel()):
            raise CrnError(f"group {x}: the three LLR streams differ in length")
        if g["bits"].dtype != torch.int32 or g["ok"].dtype != torch.uint8 or \
                (g.get("it") is not None and g["it"].dtype != torch.uint8):
            raise CrnError(f"group {x}: bits must be int32, ok / it uint8")
        arr[x] = TtiGroup(d.ctypes.data if d.size else None, d.size, 0, _ptr(g["l0"]), _ptr(g["l1"]),
                          _ptr(g["l2"]), g["l0"].numel(), _ptr(g["bits"]), g["bits"].numel(), _ptr(g["ok"]),
                          _ptr(g.get("it")))
    tim = (TtiTiming * n_tti)()
    _chk(lib().crn_stream_run_ex(arr, n_tti, n_groups, period_us, max_iters, int(early_term), flags, tim),
         "crn_stream_run_ex")
    out = np.zeros(n_tti, [(n, "f8") for n, _ in TtiTiming._fields_])
    for i in range(n_tti):
        for n, _ in TtiTiming._fields_:
            out[n][i] = getattr(tim[i], n)
    return out


def counted_ops(K, max_iters: int, iters_used=None) -> int:
    Kh = np.ascontiguousarray(K, np.int32)
    it = None if iters_used is None else np.ascontiguousarray(iters_used, np.uint8)
    return int(lib().crn_counted_ops(_np(Kh, C.c_int32), Kh.size, None if it is None else _np(it, C.c_uint8),
                                     max_iters))


def kpi_iterations(iters_used, crc_ok, max_iters: int) -> np.ndarray:
    """crn_kpi_iterations: the paper's per-CB iteration KPI (failures -> max_iters + 1)."""
    it = np.ascontiguousarray(iters_used, np.uint8)
    ok = np.ascontiguousarray(crc_ok, np.uint8)
    if it.size != ok.size:
        raise CrnError("iters_used and crc_ok differ in length")
    out = np.zeros(it.size, np.uint8)
    _chk(lib().crn_kpi_iterations(_np(it, C.c_uint8), _np(ok, C.c_uint8), it.size, max_iters, _np(out, C.c_uint8)),
         "crn_kpi_iterations")
    return out


# ------------------------------------------------------------------ encode / TB helpers
def encode_batch(desc, info, attach_crc: bool, d0, d1, d2, stream=None) -> None:
    _cuda_dev(info, d0, d1, d2)
    desc = np.ascontiguousarray(desc, DESC_DTYPE)
    _chk(lib().crn_encode_batch(desc.ctypes.data, desc.size, _ptr(info), int(attach_crc), _ptr(d0), _ptr(d1),
                                _ptr(d2), _stream(stream)), "crn_encode_batch")


def encode_batch_packed(desc, info, attach_crc: bool, d0, d1, d2, stream=None) -> None:
    """crn_encode_batch_packed: info / d* int32 CUDA tensors of packed LSB-first bits;
    ext_off / llr_off are BIT offsets."""
    _cuda_dev(info, d0, d1, d2)
    _need_i32(info, d0, d1, d2)
    desc = np.ascontiguousarray(desc, DESC_DTYPE)
    _chk(lib().crn_encode_batch_packed(desc.ctypes.data, desc.size, _ptr(info), int(attach_crc), _ptr(d0), _ptr(d1),
                                       _ptr(d2), _stream(stream)), "crn_encode_batch_packed")


def _need_i32(*ts):
    for t in ts:
        if t.dtype != __import__("torch").int32:
            raise CrnError("packed-bit buffers are int32 tensors")


def tb_build_cbs(tb_bits, base_bit: int = 0, base_llr: int = 0, base_word: int = 0, max_cb: int = 64):
    """-> (cb_bits uint8 [sum K], desc array [C])."""
    tb = np.ascontiguousarray(tb_bits, np.uint8)
    out = np.zeros(max_cb * 6144, np.uint8)
    desc = np.zeros(max_cb, DESC_DTYPE)
    n = C.c_int32()
    _chk(lib().crn_tb_build_cbs(_np(tb, C.c_uint8), tb.size, max_cb, base_bit, base_llr, base_word,
                                _np(out, C.c_uint8), desc.ctypes.data, C.byref(n)), "crn_tb_build_cbs")
    desc = desc[:n.value].copy()
    return out[:int(desc["K"].sum())].copy(), desc


def tb_build_cbs_batch(tbs_bits, payload_off, payload, cb_bits=None, max_cb=None, stream=None):
    """crn_tb_build_cbs_batch: TB payloads (one bit per byte in the CUDA uint8
    tensor ``payload``, TB t at payload_off[t]) -> (desc [n_cb] host array, cb_bits
    CUDA uint8 tensor of sum K bytes).  cb_bits may be preallocated (>= sum K)."""
    import torch
    _cuda_dev(payload, cb_bits)
    tb = np.ascontiguousarray(tbs_bits, np.int64)
    po = np.ascontiguousarray(payload_off, np.int64)
    if tb.size != po.size:
        raise CrnError("tbs_bits and payload_off differ in length")
    if max_cb is None:
        max_cb = int(sum(segment_tb(int(x))["C"] for x in tb)) if tb.size else 0
    desc = np.empty(max(max_cb, 1), DESC_DTYPE)          # the call writes every field of its n_cb records
    if cb_bits is None:
        cb_bits = torch.empty(max(max_cb, 1) * 6144, dtype=torch.uint8, device=payload.device)
    n = C.c_int32()
    _chk(lib().crn_tb_build_cbs_batch(_np(tb, C.c_int64), _np(po, C.c_int64), tb.size, _ptr(payload), max_cb,
                                      _ptr(cb_bits), desc.ctypes.data, C.byref(n), _stream(stream)),
         "crn_tb_build_cbs_batch")
    desc = desc[:n.value]                                # a view: copying a structured array goes field by field
    n_bytes = int(desc["ext_off"][-1]) + int(desc["K"][-1]) if n.value else 0      # = sum K (dense layout)
    return desc, cb_bits[:n_bytes]


RM_DTYPE = np.dtype([("K", "<i4"), ("E", "<i4"), ("rv", "<i4"), ("reserved", "<i4"), ("e_off", "<i8"),
                     ("llr_off", "<i8")])


def rate_dematch_batch(desc, e, combine: bool, h0, h1, h2, stream=None) -> None:
    """crn_rate_dematch_batch: desc (RM_DTYPE) host array; e, h* CUDA tensors."""
    _cuda_dev(e, h0, h1, h2)
    desc = np.ascontiguousarray(desc, RM_DTYPE)
    _chk(lib().crn_rate_dematch_batch(desc.ctypes.data, desc.size, _ptr(e), int(combine), _ptr(h0), _ptr(h1),
                                      _ptr(h2), _stream(stream)), "crn_rate_dematch_batch")


def rate_match_batch(desc, d0, d1, d2, e, stream=None) -> None:
    """crn_rate_match_batch: desc (RM_DTYPE) host array; d*, e CUDA uint8 tensors."""
    _cuda_dev(d0, d1, d2, e)
    desc = np.ascontiguousarray(desc, RM_DTYPE)
    _chk(lib().crn_rate_match_batch(desc.ctypes.data, desc.size, _ptr(d0), _ptr(d1), _ptr(d2), _ptr(e),
                                    _stream(stream)), "crn_rate_match_batch")


def rate_match_batch_packed(desc, d0, d1, d2, e, stream=None) -> None:
    """crn_rate_match_batch_packed: desc (RM_DTYPE, llr_off / e_off in BITS) host array;
    d*, e int32 CUDA tensors of packed LSB-first bits."""
    _cuda_dev(d0, d1, d2, e)
    _need_i32(d0, d1, d2, e)
    desc = np.ascontiguousarray(desc, RM_DTYPE)
    _chk(lib().crn_rate_match_batch_packed(desc.ctypes.data, desc.size, _ptr(d0), _ptr(d1), _ptr(d2), _ptr(e),
                                           _stream(stream)), "crn_rate_match_batch_packed")


TB_DTYPE = np.dtype([("cb0", "<i4"), ("n_cb", "<i4"), ("tbs", "<i8"), ("word_off", "<i8")])


def tb_verdict_batch(tbs, desc, cb_words, crc_ok, tb_ok, tb_words=None, stream=None) -> None:
    """crn_tb_verdict_batch: tbs (TB_DTYPE) and desc host arrays; the rest CUDA tensors."""
    _cuda_dev(cb_words, crc_ok, tb_ok, tb_words)
    tbs = np.ascontiguousarray(tbs, TB_DTYPE)
    desc = np.ascontiguousarray(desc, DESC_DTYPE)
    _chk(lib().crn_tb_verdict_batch(tbs.ctypes.data, tbs.size, desc.ctypes.data, desc.size, _ptr(cb_words),
                                    _ptr(crc_ok), _ptr(tb_ok), _ptr(tb_words), _stream(stream)),
         "crn_tb_verdict_batch")


def tb_reassemble(cb_words, desc, crc_ok, tbs: int):
    """-> payload (uint8 bits) or None if the TB is lost."""
    w = np.ascontiguousarray(cb_words, np.uint32)
    desc = np.ascontiguousarray(desc, DESC_DTYPE)
    ok = np.ascontiguousarray(crc_ok, np.uint8)
    out = np.zeros(tbs, np.uint8)
    r = _chk(lib().crn_tb_reassemble(_np(w, C.c_uint32), desc.ctypes.data, _np(ok, C.c_uint8), desc.size, tbs,
                                     _np(out, C.c_uint8)), "crn_tb_reassemble")
    return out if r == 1 else None


def segment_tb(tbs: int) -> dict:
    s = Seg()
    _chk(lib().crn_segment_tb(tbs, C.byref(s)), "crn_segment_tb")
    return {n: getattr(s, n) for n, _ in Seg._fields_}


def qpp_params(K: int) -> tuple[int, int]:
    f1, f2 = C.c_int32(), C.c_int32()
    _chk(lib().crn_qpp_params(K, C.byref(f1), C.byref(f2)), "crn_qpp_params")
    return f1.value, f2.value


def windows(K: int) -> tuple[int, int]:
    M, W = C.c_int32(), C.c_int32()
    _chk(lib().crn_windows(K, C.byref(M), C.byref(W)), "crn_windows")
    return M.value, W.value


def crc24a(bits) -> int:
    b = np.ascontiguousarray(bits, np.uint8)
    return int(lib().crn_crc24a(_np(b, C.c_uint8), b.size))


def crc24b(bits) -> int:
    b = np.ascontiguousarray(bits, np.uint8)
    return int(lib().crn_crc24b(_np(b, C.c_uint8), b.size))


def strerror(code: int) -> str:
    return lib().crn_strerror(code).decode()


def logmap_lut() -> np.ndarray:
    """crn_logmap_lut: the Log-MAP correction table LUT[0..7] (R32)."""
    out = np.zeros(8, np.int32)
    _chk(lib().crn_logmap_lut(_np(out, C.c_int32)), "crn_logmap_lut")
    return out


def mi_table() -> np.ndarray:
    out = np.zeros(256, np.int32)
    _chk(lib().crn_mi_table(_np(out, C.c_int32)), "crn_mi_table")
    return out


def device_info() -> dict:
    v = [C.c_int32() for _ in range(4)]
    _chk(lib().crn_device_info(*(C.byref(x) for x in v)), "crn_device_info")
    return dict(num_sms=v[0].value, clock_khz=v[1].value, cc=(v[2].value, v[3].value))


def decode_kernel_info() -> dict:
    v = [C.c_int32() for _ in range(4)]
    _chk(lib().crn_decode_kernel_info(*(C.byref(x) for x in v)), "crn_decode_kernel_info")
    return dict(static_smem=v[0].value, dyn_smem=v[1].value, max_dyn_attr=v[2].value, regs=v[3].value)


def ubench_int16x2(op: int) -> dict:
    li, ms, cyc = C.c_int64(), C.c_float(), C.c_int64()
    _chk(lib().crn_ubench_int16x2(op, C.byref(li), C.byref(ms), C.byref(cyc)), "crn_ubench_int16x2")
    return dict(lane_instr=li.value, ms=ms.value, max_block_cycles=cyc.value)
