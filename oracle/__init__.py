"""CPU oracle for batched Smith-Waterman with affine (Gotoh) gaps.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_2208_12350_b200``) never imports it, and this
package imports nothing from the product.

The arithmetic lives in ``sw_oracle.c`` (plain full-matrix int32 Gotoh, see
the header there for the PAPER.md passages it follows); this module only
compiles it with gcc and marshals arguments through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sw_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK = 0
BAD_PAIR = 1
BAD_SCORING = 2
NO_MEMORY = 4
REVERSE_MISMATCH = 99

DNA = 0
PROTEIN = 1
PROT_ORDER = "ARNDCQEGHILKMFPSTWYVBZX*"


class _Scoring(ctypes.Structure):
    _fields_ = [("alphabet", ctypes.c_int32), ("match", ctypes.c_int32),
                ("mismatch", ctypes.c_int32), ("gap_open", ctypes.c_int32),
                ("gap_extend", ctypes.c_int32)]


def build(force: bool = False) -> str:
    """Compile sw_oracle.c into liboracle.so (plain -O2, no SIMD intrinsics)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-shared", "-fPIC",
                                   "-pthread", _SRC, "-o", tmp])
            os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        i64p = ctypes.POINTER(ctypes.c_int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        sp = ctypes.POINTER(_Scoring)
        lib.oracle_align.argtypes = [u8p, ctypes.c_int64, u8p, ctypes.c_int64, sp, i32p]
        lib.oracle_align.restype = ctypes.c_int
        lib.oracle_fill_H.argtypes = [u8p, ctypes.c_int64, u8p, ctypes.c_int64, sp, i32p]
        lib.oracle_fill_H.restype = ctypes.c_int
        lib.oracle_check_scoring.argtypes = [sp]
        lib.oracle_check_scoring.restype = ctypes.c_int
        lib.oracle_blosum62.argtypes = [ctypes.c_int, ctypes.c_int]
        lib.oracle_blosum62.restype = ctypes.c_int
        lib.oracle_align_batch.argtypes = [u8p, i64p, u8p, i64p, ctypes.c_int64, sp,
                                           i32p, i32p, i32p, i32p, i32p, ctypes.c_int]
        lib.oracle_align_batch.restype = ctypes.c_int
        lib.oracle_traceback.argtypes = [u8p, ctypes.c_int64, u8p, ctypes.c_int64, sp, i32p, ctypes.c_char_p]
        lib.oracle_traceback.restype = ctypes.c_int
        _lib = lib
    return _lib


def scoring(alphabet="dna", match=0, mismatch=0, gap_open=-1, gap_extend=-1) -> _Scoring:
    """Build the oracle's own scoring struct.  ``alphabet`` is 'dna' or 'protein'."""
    a = {"dna": DNA, "protein": PROTEIN}[alphabet] if isinstance(alphabet, str) else int(alphabet)
    return _Scoring(a, int(match), int(mismatch), int(gap_open), int(gap_extend))


def _as_scoring(sc) -> _Scoring:
    if isinstance(sc, _Scoring):
        return sc
    if isinstance(sc, dict):
        return scoring(**sc)
    raise TypeError(f"unsupported scoring {sc!r}")


def _u8(buf) -> np.ndarray:
    if isinstance(buf, str):
        buf = buf.encode("ascii")
    a = np.frombuffer(bytes(buf), dtype=np.uint8) if isinstance(buf, (bytes, bytearray)) else np.ascontiguousarray(buf, dtype=np.uint8)
    if a.size == 0:
        a = np.zeros(1, dtype=np.uint8)[:0]
    return np.ascontiguousarray(a)


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def align(q, r, sc) -> tuple:
    """(score, q_end, r_end, q_start, r_start) for one pair; all -1 if invalid."""
    lib = _load()
    qa, ra = _u8(q), _u8(r)
    qa_b = qa if qa.size else np.zeros(1, np.uint8)
    ra_b = ra if ra.size else np.zeros(1, np.uint8)
    out = np.zeros(5, dtype=np.int32)
    s = _as_scoring(sc)
    st = lib.oracle_align(_ptr(qa_b, ctypes.c_uint8), qa.size, _ptr(ra_b, ctypes.c_uint8), ra.size,
                          ctypes.byref(s), _ptr(out, ctypes.c_int32))
    if st == BAD_SCORING:
        raise ValueError("invalid scoring")
    if st in (NO_MEMORY, REVERSE_MISMATCH):
        raise RuntimeError(f"oracle failure status {st}")
    return tuple(int(x) for x in out)


def traceback(q, r, sc, res=None) -> str | None:
    """Alignment ops ('M' aligned pair, 'I' query residue vs gap, 'D' reference residue vs gap)
    from start to end of the pair's reported alignment (sw_oracle.c oracle_traceback, reading R20).
    '' for S == 0, None for an invalid pair.  ``res`` = align(q, r, sc) if already known."""
    lib = _load()
    qa, ra = _u8(q), _u8(r)
    if res is None:
        res = align(qa, ra, sc)
    qa_b = qa if qa.size else np.zeros(1, np.uint8)
    ra_b = ra if ra.size else np.zeros(1, np.uint8)
    rv = np.asarray(res, dtype=np.int32)
    buf = ctypes.create_string_buffer(max(1, qa.size + ra.size))
    k = lib.oracle_traceback(_ptr(qa_b, ctypes.c_uint8), qa.size, _ptr(ra_b, ctypes.c_uint8), ra.size,
                             ctypes.byref(_as_scoring(sc)), _ptr(rv, ctypes.c_int32), buf)
    if k == -2:
        raise RuntimeError("oracle traceback: global optimum differs from S")
    if k < 0:
        return None
    return buf.raw[:k].decode()


def cigar(ops: str) -> str:
    """Run-length form of an op string ('MMMID' -> '3M1I1D')."""
    out, k = [], 0
    while k < len(ops):
        t = k
        while t < len(ops) and ops[t] == ops[k]:
            t += 1
        out.append(f"{t - k}{ops[k]}")
        k = t
    return "".join(out)


def fill_H(q, r, sc) -> np.ndarray:
    """Full (n+1) x (m+1) H matrix of one pair (tests only)."""
    lib = _load()
    qa, ra = _u8(q), _u8(r)
    H = np.zeros((qa.size + 1, ra.size + 1), dtype=np.int32)
    qa_b = qa if qa.size else np.zeros(1, np.uint8)
    ra_b = ra if ra.size else np.zeros(1, np.uint8)
    s = _as_scoring(sc)
    st = lib.oracle_fill_H(_ptr(qa_b, ctypes.c_uint8), qa.size, _ptr(ra_b, ctypes.c_uint8), ra.size,
                           ctypes.byref(s), _ptr(H, ctypes.c_int32))
    if st != OK:
        raise ValueError(f"oracle_fill_H status {st}")
    return H


def check_scoring(sc) -> bool:
    s = _as_scoring(sc)
    return _load().oracle_check_scoring(ctypes.byref(s)) == OK


def blosum62(a: str, b: str) -> int:
    return int(_load().oracle_blosum62(PROT_ORDER.index(a), PROT_ORDER.index(b)))


def align_batch(queries, q_offsets, refs, r_offsets, sc, threads: int | None = None) -> dict:
    """Batch over host CSR arrays.  Returns dict of five int32 numpy arrays."""
    lib = _load()
    qa = np.ascontiguousarray(queries, dtype=np.uint8)
    ra = np.ascontiguousarray(refs, dtype=np.uint8)
    qo = np.ascontiguousarray(q_offsets, dtype=np.int64)
    ro = np.ascontiguousarray(r_offsets, dtype=np.int64)
    n = qo.size - 1
    if qa.size == 0:
        qa = np.zeros(1, np.uint8)
    if ra.size == 0:
        ra = np.zeros(1, np.uint8)
    outs = {k: np.full(max(n, 0), -1, dtype=np.int32) for k in ("score", "q_end", "r_end", "q_start", "r_start")}
    if n <= 0:
        return outs
    s = _as_scoring(sc)
    th = threads if threads else (os.cpu_count() or 1)
    st = lib.oracle_align_batch(_ptr(qa, ctypes.c_uint8), _ptr(qo, ctypes.c_int64),
                                _ptr(ra, ctypes.c_uint8), _ptr(ro, ctypes.c_int64), n, ctypes.byref(s),
                                *[_ptr(outs[k], ctypes.c_int32) for k in ("score", "q_end", "r_end", "q_start", "r_start")],
                                int(th))
    if st == BAD_SCORING:
        raise ValueError("invalid scoring")
    if st != OK:
        raise RuntimeError(f"oracle_align_batch status {st}")
    return outs
