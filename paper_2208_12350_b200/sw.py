"""Thin ctypes binding of the C ABI in include/sw.h (argument marshalling only).

Every step of the alignment runs in ``libsw_b200.so`` (sm_100a kernels).  There
is no CPU fallback: if the library cannot be loaded, the calls raise.  The
function names mirror the C ABI (``sw_init``, ``sw_align_batch``,
``sw_align_batch_host``, ``sw_free``, ``sw_batch_status``, ``sw_plan_shards``,
...); ``Aligner`` is a convenience wrapper over torch tensors (PyTorch is used
only for device memory and streams).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

SW_OK = 0
SW_ERR_INVALID_ARGUMENT = 1
SW_ERR_INVALID_SCORING = 2
SW_ERR_CUDA = 3
SW_ERR_OUT_OF_MEMORY = 4
SW_ERR_WRONG_DEVICE = 5
SW_ERR_BAD_PAIRS = 6
SW_ERR_INTERNAL = 7

SW_ALPHABET_DNA = 0
SW_ALPHABET_PROTEIN = 1
SW_MAX_SEQ_LEN = 65535
SW_STAGE_NAMES = ("pack", "sort", "fwd", "mid", "rev", "finish")
SW_MODE_FULL = 0
SW_MODE_END_ONLY = 1
SW_MODE_AFFINE_ONLY = 2
SW_MODE_TB_INT32 = 4
SW_MODE_POISON = 8
SW_MODE_NO_BAND = 16
SW_MODE_BAND_ALWAYS = 32

EXPORTED = ("sw_init", "sw_reserve", "sw_align_batch", "sw_align_query_db", "sw_align_batch_host", "sw_submit_host", "sw_wait", "sw_set_mode", "sw_traceback", "sw_batch_status", "sw_free",
            "sw_status_string", "sw_last_error_message", "sw_plan_shards", "sw_enable_stage_timing",
            "sw_get_stage_ms", "sw_last_launch_count", "sw_last_cell_counts", "sw_last_reverse_cells", "sw_dpx_peak")


class sw_scoring_t(ctypes.Structure):
    _fields_ = [("alphabet", ctypes.c_int32), ("match", ctypes.c_int32), ("mismatch", ctypes.c_int32),
                ("gap_open", ctypes.c_int32), ("gap_extend", ctypes.c_int32)]


class sw_result_t(ctypes.Structure):
    _fields_ = [("score", ctypes.c_void_p), ("q_end", ctypes.c_void_p), ("r_end", ctypes.c_void_p),
                ("q_start", ctypes.c_void_p), ("r_start", ctypes.c_void_p)]


class SWError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"{status_string(status)}: {msg}")
        self.status = status


_lib = None


def library_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libsw_b200.so (building it with nvcc if absent).  Raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    # SW_B200_LIB: an alternative build of the same library (kernel-variant experiments)
    path = os.environ.get("SW_B200_LIB", _build.LIB)
    if not os.path.exists(path):
        if not build_if_missing:
            raise OSError(f"{path} not built (run __graft_entry__.build())")
        _build.build()
    lib = ctypes.CDLL(path)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    sp = ctypes.POINTER(sw_scoring_t)
    rp = ctypes.POINTER(sw_result_t)
    lib.sw_init.argtypes = [ctypes.POINTER(vp), ctypes.c_int]
    lib.sw_align_batch.argtypes = [vp, vp, vp, vp, vp, i64, sp, rp, vp]
    lib.sw_reserve.argtypes = [vp, i64, i64, i64, i32, i32]
    lib.sw_align_batch_host.argtypes = [vp, vp, vp, vp, vp, i64, sp, rp, vp]
    lib.sw_align_query_db.argtypes = [vp, vp, i64, vp, vp, i64, sp, rp, vp]
    lib.sw_submit_host.argtypes = [vp, vp, vp, vp, vp, i64, sp, rp, vp]
    lib.sw_wait.argtypes = [vp]
    lib.sw_set_mode.argtypes = [vp, ctypes.c_int32]
    lib.sw_traceback.argtypes = [vp, vp, vp, vp, vp, i64, sp, rp, vp, vp, vp]
    lib.sw_batch_status.argtypes = [vp, ctypes.POINTER(i64)]
    lib.sw_free.argtypes = [vp]
    lib.sw_status_string.argtypes = [ctypes.c_int]
    lib.sw_status_string.restype = ctypes.c_char_p
    lib.sw_last_error_message.argtypes = [vp]
    lib.sw_last_error_message.restype = ctypes.c_char_p
    lib.sw_plan_shards.argtypes = [vp, vp, i64, i32, vp]
    lib.sw_enable_stage_timing.argtypes = [vp, ctypes.c_int]
    lib.sw_get_stage_ms.argtypes = [vp, ctypes.POINTER(ctypes.c_float)]
    lib.sw_last_launch_count.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    lib.sw_last_cell_counts.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    lib.sw_last_reverse_cells.argtypes = [vp, ctypes.POINTER(i64)]
    lib.sw_dpx_peak.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.POINTER(ctypes.c_double), vp]
    for name in EXPORTED:
        if name not in ("sw_status_string", "sw_last_error_message"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def status_string(st: int) -> str:
    try:
        return load().sw_status_string(int(st)).decode()
    except OSError:
        return f"status {st}"


def make_scoring(scoring: dict) -> sw_scoring_t:
    a = scoring.get("alphabet", "dna")
    a = {"dna": SW_ALPHABET_DNA, "protein": SW_ALPHABET_PROTEIN}[a] if isinstance(a, str) else int(a)
    return sw_scoring_t(a, int(scoring.get("match", 0)), int(scoring.get("mismatch", 0)),
                        int(scoring["gap_open"]), int(scoring["gap_extend"]))


# ------------------------------------------------------------ C-ABI mirrors

def sw_init(device: int) -> int:
    lib = load()
    h = ctypes.c_void_p()
    st = lib.sw_init(ctypes.byref(h), int(device))
    if st != SW_OK:
        raise SWError(st, "sw_init")
    return h.value


def sw_free(handle: int) -> None:
    st = load().sw_free(ctypes.c_void_p(handle))
    if st != SW_OK:
        raise SWError(st, "sw_free")


def sw_last_error_message(handle: int) -> str:
    return load().sw_last_error_message(ctypes.c_void_p(handle)).decode()


def sw_align_batch(handle: int, queries, q_offsets, refs, r_offsets, n_pairs: int, scoring: dict, out: dict,
                   stream: int = 0) -> int:
    """Device pointers (ints) in, device pointers in ``out`` (dict of 5). Returns the status."""
    lib = load()
    sc = make_scoring(scoring)
    res = sw_result_t(out["score"], out["q_end"], out["r_end"], out["q_start"], out["r_start"])
    return lib.sw_align_batch(ctypes.c_void_p(handle), ctypes.c_void_p(queries), ctypes.c_void_p(q_offsets),
                              ctypes.c_void_p(refs), ctypes.c_void_p(r_offsets), int(n_pairs), ctypes.byref(sc),
                              ctypes.byref(res), ctypes.c_void_p(stream))


def sw_align_batch_host(handle: int, queries, q_offsets, refs, r_offsets, n_pairs: int, scoring: dict, out: dict,
                        stream: int = 0) -> int:
    lib = load()
    sc = make_scoring(scoring)
    res = sw_result_t(out["score"], out["q_end"], out["r_end"], out["q_start"], out["r_start"])
    return lib.sw_align_batch_host(ctypes.c_void_p(handle), ctypes.c_void_p(queries), ctypes.c_void_p(q_offsets),
                                   ctypes.c_void_p(refs), ctypes.c_void_p(r_offsets), int(n_pairs),
                                   ctypes.byref(sc), ctypes.byref(res), ctypes.c_void_p(stream))


def sw_submit_host(handle: int, queries, q_offsets, refs, r_offsets, n_pairs: int, scoring: dict, out: dict,
                   stream: int = 0) -> int:
    """Asynchronous host-buffer batch (include/sw.h): returns once enqueued; sw_wait completes it."""
    lib = load()
    sc = make_scoring(scoring)
    res = sw_result_t(out["score"], out["q_end"], out["r_end"], out["q_start"], out["r_start"])
    return lib.sw_submit_host(ctypes.c_void_p(handle), ctypes.c_void_p(queries), ctypes.c_void_p(q_offsets),
                              ctypes.c_void_p(refs), ctypes.c_void_p(r_offsets), int(n_pairs),
                              ctypes.byref(sc), ctypes.byref(res), ctypes.c_void_p(stream))


def sw_wait(handle: int) -> int:
    return load().sw_wait(ctypes.c_void_p(handle))


def sw_batch_status(handle: int) -> tuple[int, int]:
    n = ctypes.c_int64(0)
    st = load().sw_batch_status(ctypes.c_void_p(handle), ctypes.byref(n))
    return st, n.value


def sw_plan_shards(q_offsets: np.ndarray, r_offsets: np.ndarray, n_shards: int) -> np.ndarray:
    """Host-only cell-count shard plan: n_shards + 1 contiguous cut indices."""
    qo = np.ascontiguousarray(q_offsets, dtype=np.int64)
    ro = np.ascontiguousarray(r_offsets, dtype=np.int64)
    n = qo.size - 1
    out = np.zeros(int(n_shards) + 1, dtype=np.int64)
    st = load().sw_plan_shards(qo.ctypes.data, ro.ctypes.data, n, int(n_shards), out.ctypes.data)
    if st != SW_OK:
        raise SWError(st, "sw_plan_shards")
    return out


def sw_dpx_peak(device: int, milliseconds: float = 200.0, stream: int = 0) -> float:
    cups = ctypes.c_double(0)
    st = load().sw_dpx_peak(int(device), float(milliseconds), ctypes.byref(cups), ctypes.c_void_p(stream))
    if st != SW_OK:
        raise SWError(st, "sw_dpx_peak")
    return cups.value


# ------------------------------------------------------ torch convenience

class Aligner:
    """Owns one sw handle on one device; aligns batches held in torch tensors."""

    def __init__(self, device: int = 0, poison: bool = False):
        """poison=True keeps SW_MODE_POISON on (tests and soaks): every call first fills its outputs
        and the handle's workspace with poison bytes, so an unwritten value cannot pass as a result."""
        import torch
        self.torch = torch
        self.device = int(device)
        torch.cuda.set_device(self.device)
        self.handle = sw_init(self.device)
        self.poison = SW_MODE_POISON if poison else 0
        if self.poison:
            self.set_mode(SW_MODE_FULL)

    def reserve(self, max_pairs: int, max_query_bytes: int, max_ref_bytes: int, max_query_len: int, max_ref_len: int):
        """sw_reserve: afterwards calls within these bounds enqueue without a host round trip."""
        st = load().sw_reserve(ctypes.c_void_p(self.handle), int(max_pairs), int(max_query_bytes), int(max_ref_bytes),
                               int(max_query_len), int(max_ref_len))
        if st != SW_OK:
            raise SWError(st, sw_last_error_message(self.handle))

    def reserve_for(self, batch, pairs_slack: float = 1.0):
        """Reservation sized for `batch` (times `pairs_slack` on counts and bytes)."""
        n, m = batch.lengths()
        k = max(pairs_slack, 1.0)
        self.reserve(int(batch.n_pairs * k) + 1, int(n.sum() * k) + 1, int(m.sum() * k) + 1,
                     int(n.max()) if n.size else 0, int(m.max()) if m.size else 0)

    def close(self):
        if self.handle:
            sw_free(self.handle)
            self.handle = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def to_device(self, batch):
        t = self.torch
        dev = f"cuda:{self.device}"
        q = t.from_numpy(np.ascontiguousarray(batch.queries)).to(dev) if batch.queries.size else t.zeros(1, dtype=t.uint8, device=dev)
        r = t.from_numpy(np.ascontiguousarray(batch.refs)).to(dev) if batch.refs.size else t.zeros(1, dtype=t.uint8, device=dev)
        qo = t.from_numpy(np.ascontiguousarray(batch.q_offsets)).to(dev)
        ro = t.from_numpy(np.ascontiguousarray(batch.r_offsets)).to(dev)
        return q, qo, r, ro

    def alloc_out(self, n: int):
        t = self.torch
        buf = t.empty((5, max(n, 1)), dtype=t.int32, device=f"cuda:{self.device}")
        return buf

    def align_tensors(self, q, qo, r, ro, scoring: dict, out=None, stream=None, check=True):
        t = self.torch
        n = qo.numel() - 1
        if out is None:
            out = self.alloc_out(n)
        s = stream if stream is not None else t.cuda.current_stream(self.device)
        ptrs = {k: out[i].data_ptr() for i, k in enumerate(("score", "q_end", "r_end", "q_start", "r_start"))}
        st = sw_align_batch(self.handle, q.data_ptr(), qo.data_ptr(), r.data_ptr(), ro.data_ptr(), n, scoring, ptrs,
                            s.cuda_stream)
        if check and st != SW_OK:
            raise SWError(st, sw_last_error_message(self.handle))
        return out, st

    def align(self, batch, check=True) -> dict:
        """Align a synth.Batch; returns dict of five int32 numpy arrays."""
        q, qo, r, ro = self.to_device(batch)
        out, st = self.align_tensors(q, qo, r, ro, batch.scoring, check=check)
        self.torch.cuda.synchronize(self.device)
        n = batch.n_pairs
        o = out[:, :n].cpu().numpy()
        return {k: o[i] for i, k in enumerate(("score", "q_end", "r_end", "q_start", "r_start"))}

    def align_query_db(self, query: bytes, refs, scoring: dict) -> dict:
        """One query against a list of references (include/sw.h sw_align_query_db); returns the
        five int32 numpy arrays, one entry per reference."""
        t = self.torch
        dev = f"cuda:{self.device}"
        rb = [x.encode() if isinstance(x, str) else bytes(x) for x in refs]
        ro = np.zeros(len(rb) + 1, dtype=np.int64)
        ro[1:] = np.cumsum([len(x) for x in rb]) if rb else []
        ra = np.frombuffer(b"".join(rb), dtype=np.uint8) if rb else np.zeros(0, np.uint8)
        qa = np.frombuffer(bytes(query), dtype=np.uint8)
        qd = t.from_numpy(qa.copy()).to(dev) if qa.size else t.zeros(1, dtype=t.uint8, device=dev)
        rd = t.from_numpy(ra.copy()).to(dev) if ra.size else t.zeros(1, dtype=t.uint8, device=dev)
        rod = t.from_numpy(ro).to(dev)
        n = len(rb)
        out = self.alloc_out(n)
        res = sw_result_t(*[out[i].data_ptr() for i in range(5)])
        st = load().sw_align_query_db(ctypes.c_void_p(self.handle), ctypes.c_void_p(qd.data_ptr()), int(qa.size),
                                      ctypes.c_void_p(rd.data_ptr()), ctypes.c_void_p(rod.data_ptr()), n,
                                      ctypes.byref(make_scoring(scoring)), ctypes.byref(res),
                                      ctypes.c_void_p(t.cuda.current_stream(self.device).cuda_stream))
        if st != SW_OK:
            raise SWError(st, sw_last_error_message(self.handle))
        t.cuda.synchronize(self.device)
        o = out[:, :n].cpu().numpy()
        return {k: o[i] for i, k in enumerate(("score", "q_end", "r_end", "q_start", "r_start"))}

    def batch_status(self):
        return sw_batch_status(self.handle)

    def stage_ms(self) -> dict:
        arr = (ctypes.c_float * 6)()
        st = load().sw_get_stage_ms(ctypes.c_void_p(self.handle), arr)
        if st != SW_OK:
            raise SWError(st, sw_last_error_message(self.handle))
        return dict(zip(SW_STAGE_NAMES, list(arr)))

    def enable_stage_timing(self, on: bool = True):
        load().sw_enable_stage_timing(ctypes.c_void_p(self.handle), 1 if on else 0)

    def launch_count(self):
        a, b = ctypes.c_int32(0), ctypes.c_int32(0)
        load().sw_last_launch_count(ctypes.c_void_p(self.handle), ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value

    def traceback_tensors(self, q, qo, r, ro, scoring: dict, res, ops=None, n_ops=None):
        """Alignment ops of an aligned batch (include/sw.h sw_traceback); res = the (5, n) result
        tensor of align_tensors.  Returns (ops uint8 tensor, n_ops int32 tensor), on the device."""
        import torch
        n = qo.numel() - 1
        if ops is None:
            ops = torch.zeros(int(q.numel() + r.numel()) + 1, dtype=torch.uint8, device=q.device)
        if n_ops is None:
            n_ops = torch.empty(max(n, 1), dtype=torch.int32, device=q.device)
        rr = sw_result_t(res[0].data_ptr(), res[1].data_ptr(), res[2].data_ptr(), res[3].data_ptr(), res[4].data_ptr())
        st = load().sw_traceback(ctypes.c_void_p(self.handle), ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(qo.data_ptr()),
                                 ctypes.c_void_p(r.data_ptr()), ctypes.c_void_p(ro.data_ptr()), int(n),
                                 ctypes.byref(make_scoring(scoring)), ctypes.byref(rr), ctypes.c_void_p(ops.data_ptr()),
                                 ctypes.c_void_p(n_ops.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        if st != SW_OK:
            raise SWError(st, sw_last_error_message(self.handle))
        return ops, n_ops

    def traceback(self, batch) -> list:
        """Align a host batch and return each pair's op string ('' for S == 0, None for invalid)."""
        return self.align_and_traceback(batch)[1]

    def align_and_traceback(self, batch):
        """One sw_align_batch call and the sw_traceback of ITS results: returns (the five int32
        numpy arrays, each pair's op string ('' for S == 0, None for invalid))."""
        import torch
        q, qo, r, ro = self.to_device(batch)
        out, _ = self.align_tensors(q, qo, r, ro, batch.scoring)
        ops, n_ops = self.traceback_tensors(q, qo, r, ro, batch.scoring, out)
        torch.cuda.synchronize()
        n = batch.n_pairs
        o = out[:, :n].cpu().numpy()
        fields = {k: o[i] for i, k in enumerate(("score", "q_end", "r_end", "q_start", "r_start"))}
        ops_h = ops.cpu().numpy().tobytes()
        n_h = n_ops.cpu().numpy()
        qoff, roff = batch.q_offsets, batch.r_offsets
        res = []
        for p in range(batch.n_pairs):
            k = int(n_h[p])
            if k < 0:
                res.append(None)
                continue
            at = int(qoff[p] - qoff[0] + roff[p] - roff[0])
            res.append(ops_h[at:at + k].decode())
        return fields, res

    def set_mode(self, mode: int):
        """SW_MODE_FULL (forward + reverse) or SW_MODE_END_ONLY (forward only; starts not written),
        optionally OR-ed with SW_MODE_AFFINE_ONLY (linear-gap scorings stay on the affine kernels)."""
        st = load().sw_set_mode(ctypes.c_void_p(self.handle), int(mode) | self.poison)
        if st != SW_OK:
            raise SWError(st, sw_last_error_message(self.handle))

    def reverse_cells(self):
        a = ctypes.c_int64(0)
        load().sw_last_reverse_cells(ctypes.c_void_p(self.handle), ctypes.byref(a))
        return a.value

    def cell_counts(self):
        a, b = ctypes.c_int64(0), ctypes.c_int64(0)
        load().sw_last_cell_counts(ctypes.c_void_p(self.handle), ctypes.byref(a), ctypes.byref(b))
        return a.value, b.value
