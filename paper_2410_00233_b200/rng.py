"""Device-side ``default_rng(seed).standard_normal`` (kernels in csrc/kb_rng.cu).

The reference draws its random start vector (lowrank.py:199-201) and the RSVD
test matrix (lowrank.py:361-362) on the host with numpy.  ``standard_normal``
here returns the SAME values (PCG64 + numpy's float64 ziggurat, bit-exact
after the reference's ``astype``), generated on the GPU, so results stay
identical to the reference while the host never touches n^2 draws.
"""

from __future__ import annotations

import ctypes as C
import functools

import numpy as np
import torch

from . import _lib
from . import device as D


@functools.lru_cache(maxsize=64)
def _seeded_state(seed: int) -> tuple[int, int]:
    st = np.random.PCG64(seed).state["state"]        # SeedSequence hashing: ~50 us, cached
    return int(st["state"]), int(st["inc"])


def pcg64_state(seed) -> tuple[int, int]:
    """(state, inc) of ``np.random.default_rng(seed)``'s PCG64 before any draw."""
    if isinstance(seed, (int, np.integer)) and not isinstance(seed, bool) and seed >= 0:
        return _seeded_state(int(seed))
    if isinstance(seed, np.random.Generator):
        bg = seed.bit_generator
    elif isinstance(seed, np.random.BitGenerator):
        bg = seed
    else:
        bg = np.random.PCG64(seed)
    if not isinstance(bg, np.random.PCG64):
        raise TypeError(f"device draws need a PCG64 stream, got {type(bg).__name__}")
    st = bg.state
    if st.get("has_uint32"):
        raise ValueError("PCG64 stream has a buffered 32-bit half draw; not reproducible here")
    return int(st["state"]["state"]), int(st["state"]["inc"])


def _pair(v: int):
    arr = (C.c_uint64 * 2)(v & 0xFFFFFFFFFFFFFFFF, (v >> 64) & 0xFFFFFFFFFFFFFFFF)
    return arr


def standard_normal(seed, shape, dtype=np.float32, transpose: bool = False) -> torch.Tensor:
    """``np.random.default_rng(seed).standard_normal(shape).astype(dtype)`` on the device.

    ``transpose=True`` (2-D shapes) returns the transposed matrix, contiguous.
    """
    shape = (int(shape),) if np.isscalar(shape) else tuple(int(s) for s in shape)
    count = int(np.prod(shape)) if shape else 1
    cols = 0
    out_shape = shape
    if transpose:
        if len(shape) != 2:
            raise ValueError("transpose needs a 2-D shape")
        cols = shape[1]
        out_shape = (shape[1], shape[0])
    out = D.empty(out_shape, dtype)
    if count == 0:
        return out
    state, inc = pcg64_state(seed)
    lib = _lib.load()
    nb = C.c_size_t()
    _lib.check(lib.kb_normal_workspace_bytes(count, C.byref(nb)), "kb_normal_workspace_bytes")
    ws, ws_n = D.WORKSPACE.get(nb.value)
    code = _lib.KB_F32 if np.dtype(dtype) == np.float32 else _lib.KB_F64
    _lib.check(lib.kb_normal_pcg64(_pair(state), _pair(inc), count, code, cols, out.data_ptr(), ws, ws_n,
                                   D.stream_ptr()), "kb_normal_pcg64")
    return out
