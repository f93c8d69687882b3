"""Thin ctypes binding of include/simcov.h: the SIMCoV diffusion stencil on a zero-padded
grid (reading R22).

Argument marshalling only: every step runs in ``libsw_b200.so`` (sm_100a kernels); there is
no CPU fallback.  ``Grid`` is a convenience wrapper that owns the padded device buffers
(torch tensors are used only as device memory and for the stream).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import sw

SIMCOV_MAX_FIELDS = 8
SIMCOV_MAX_RATE = 1 << 30
SIMCOV_MAX_TBLOCK = 8

EXPORTED = ("simcov_grid_pitch", "simcov_grid_words", "simcov_pad", "simcov_unpad", "simcov_diffuse",
            "simcov_set_schedule", "simcov_last_launch_count", "simcov_last_error_message")

_ready = False


def load():
    """The library with the simcov_* prototypes set (raises if it cannot be loaded)."""
    global _ready
    lib = sw.load()
    if not _ready:
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        lib.simcov_grid_pitch.argtypes = [i64]
        lib.simcov_grid_pitch.restype = i64
        lib.simcov_grid_words.argtypes = [i64, i64]
        lib.simcov_grid_words.restype = i64
        lib.simcov_pad.argtypes = [vp, vp, i64, i64, i32, i64, vp]
        lib.simcov_unpad.argtypes = [vp, vp, i64, i64, i32, i64, vp]
        lib.simcov_diffuse.argtypes = [vp, vp, i64, i64, i32, i64, vp, i32, vp]
        lib.simcov_set_schedule.argtypes = [i32]
        for f in ("simcov_pad", "simcov_unpad", "simcov_diffuse", "simcov_set_schedule",
                  "simcov_last_launch_count"):
            getattr(lib, f).restype = ctypes.c_int
        lib.simcov_last_error_message.restype = ctypes.c_char_p
        _ready = True
    return lib


def _check(st: int, what: str) -> None:
    if st != sw.SW_OK:
        raise sw.SWError(st, f"{what}: {load().simcov_last_error_message().decode()}")


def simcov_grid_pitch(W: int) -> int:
    return int(load().simcov_grid_pitch(int(W)))


def simcov_grid_words(H: int, W: int) -> int:
    return int(load().simcov_grid_words(int(H), int(W)))


def simcov_pad(dense_ptr: int, padded_ptr: int, H: int, W: int, n_fields: int, field_stride: int,
               stream: int | None = None) -> None:
    _check(load().simcov_pad(dense_ptr, padded_ptr, H, W, n_fields, field_stride, stream), "simcov_pad")


def simcov_unpad(padded_ptr: int, dense_ptr: int, H: int, W: int, n_fields: int, field_stride: int,
                 stream: int | None = None) -> None:
    _check(load().simcov_unpad(padded_ptr, dense_ptr, H, W, n_fields, field_stride, stream), "simcov_unpad")


def simcov_diffuse(grid_ptr: int, scratch_ptr: int, H: int, W: int, n_fields: int, field_stride: int,
                   rates, steps: int, stream: int | None = None) -> None:
    arr = (ctypes.c_uint32 * max(1, len(rates)))(*[int(a) for a in rates])
    _check(load().simcov_diffuse(grid_ptr, scratch_ptr, H, W, n_fields, field_stride, arr, int(steps), stream),
           "simcov_diffuse")


def simcov_set_schedule(steps_per_launch: int) -> None:
    _check(load().simcov_set_schedule(int(steps_per_launch)), "simcov_set_schedule")


def simcov_last_launch_count() -> int:
    return int(load().simcov_last_launch_count())


def rate_fixed(r: float) -> int:
    """Fixed-point rate a = floor(r * 2^32) of a fraction 0 <= r <= 1/4 (R22)."""
    a = int(np.floor(float(r) * 4294967296.0))
    if not 0 <= a <= SIMCOV_MAX_RATE:
        raise ValueError("rate must lie in [0, 1/4]")
    return a


class Grid:
    """n_fields padded H x W uint32 fields (and their ping-pong scratch) on one CUDA device."""

    def __init__(self, H: int, W: int, n_fields: int = 2, device: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("simcov.Grid needs a CUDA device (there is no CPU fallback)")
        load()
        self.H, self.W, self.n_fields = int(H), int(W), int(n_fields)
        self.device = torch.device("cuda", device)
        self.pitch = simcov_grid_pitch(W)
        words = simcov_grid_words(H, W)
        if self.pitch < 0 or words < 0:
            raise ValueError("bad grid size")
        self.field_stride = (words + 31) // 32 * 32
        n = self.field_stride * self.n_fields
        # int32 storage (torch has no uint32 arithmetic on CUDA); the kernels see uint32 words
        self.grid = torch.zeros(n, dtype=torch.int32, device=self.device)
        self.scratch = torch.zeros(n, dtype=torch.int32, device=self.device)

    def _stream(self):
        import torch
        return torch.cuda.current_stream(self.device).cuda_stream

    def upload(self, fields) -> None:
        """Copy n_fields H x W arrays (uint32-valued) into the padded grid (simcov_pad)."""
        import torch
        dense = np.ascontiguousarray(np.stack([np.asarray(f, dtype=np.uint32) for f in fields]))
        assert dense.shape == (self.n_fields, self.H, self.W)
        d = torch.from_numpy(dense.view(np.int32)).to(self.device)
        simcov_pad(d.data_ptr(), self.grid.data_ptr(), self.H, self.W, self.n_fields, self.field_stride,
                   self._stream())
        self._keep = d

    def download(self) -> list:
        """The n_fields H x W fields as uint32 numpy arrays (simcov_unpad)."""
        import torch
        d = torch.empty(self.n_fields * self.H * self.W, dtype=torch.int32, device=self.device)
        simcov_unpad(self.grid.data_ptr(), d.data_ptr(), self.H, self.W, self.n_fields, self.field_stride,
                     self._stream())
        out = d.cpu().numpy().view(np.uint32).reshape(self.n_fields, self.H, self.W)
        return [out[f] for f in range(self.n_fields)]

    def diffuse(self, rates, steps: int) -> None:
        simcov_diffuse(self.grid.data_ptr(), self.scratch.data_ptr(), self.H, self.W, self.n_fields,
                       self.field_stride, rates, steps, self._stream())

    def padded(self) -> np.ndarray:
        """The raw padded buffer as (n_fields, H + 2, pitch) uint32 (layout checks)."""
        a = self.grid.cpu().numpy().view(np.uint32).reshape(self.n_fields, self.field_stride)
        return a[:, :(self.H + 2) * self.pitch].reshape(self.n_fields, self.H + 2, self.pitch)
