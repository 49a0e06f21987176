"""Device plumbing: torch owns device memory and streams; the kernels are ours.

Host numpy inputs (the reference's drop-in surface) are uploaded once; torch
CUDA tensors are used in place.  Every product call runs on the current torch
stream of ``cuda:0`` (or the tensor's device).
"""

from __future__ import annotations

import numpy as np
import torch

from .exceptions import KronblurError, ValidationError

_TORCH_OF = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}
_NP_OF = {torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64)}


_CUDA_OK = False


def device() -> torch.device:
    global _CUDA_OK
    if not _CUDA_OK:   # the driver query costs a few us per call; once available it stays available
        if not torch.cuda.is_available():
            raise KronblurError("no CUDA device: the kronblur_b200 path runs on B200 (sm_100a) only")
        _CUDA_OK = True
    return torch.device("cuda", torch.cuda.current_device())


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_ptr() -> int:
    """cudaStream_t of torch's current stream on the current device (the raw query
    skips building a Stream object: a few us per call on the launch paths)."""
    if _RAW_STREAM is not None:
        return _RAW_STREAM(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def torch_dtype(dt) -> torch.dtype:
    try:
        return _TORCH_OF[np.dtype(dt)]
    except (KeyError, TypeError):
        raise ValidationError(f"unsupported dtype {dt}; expected float32 or float64") from None


def np_dtype(t: torch.Tensor) -> np.dtype:
    return _NP_OF[t.dtype]


def is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


def to_device(x, dtype=None, contiguous=True) -> torch.Tensor:
    """Host array / tensor -> contiguous CUDA tensor of ``dtype``."""
    dev = device()
    if isinstance(x, torch.Tensor):
        t = x
        if dtype is not None and t.dtype != torch_dtype(dtype):
            t = t.to(torch_dtype(dtype))
        if t.device != dev:
            t = t.to(dev)
    else:
        a = np.asarray(x)
        if dtype is not None:
            a = a.astype(dtype, copy=False)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(dev, non_blocking=False)
    return t.contiguous() if contiguous else t


def upload(a: np.ndarray, dtype) -> torch.Tensor:
    """Host array -> device tensor of ``dtype`` through pinned staging (cast while staging)."""
    a = np.asarray(a)
    stage = torch.empty(a.shape, dtype=torch_dtype(dtype), pin_memory=True)
    np.copyto(stage.numpy(), a, casting="same_kind")
    return stage.to(device(), non_blocking=True)


class _PinnedStage:
    """One reusable pinned staging buffer for small stream-ordered uploads
    (a fresh pinned allocation per call costs ~50-80 us of host time).  The
    buffer is rewritten only after the previous copy out of it has finished
    (event), so an in-flight upload is never clobbered."""

    def __init__(self):
        self._buf = None
        self._event = None

    def upload(self, host: np.ndarray) -> torch.Tensor:
        host = np.ascontiguousarray(host).view(np.uint8).reshape(-1)
        n = host.size
        if self._buf is None or self._buf.numel() < n:
            if self._event is not None:
                self._event.synchronize()
            self._buf = torch.empty(max(n, 1 << 16), dtype=torch.uint8, pin_memory=True)
            self._event = None
        if self._event is not None:
            self._event.synchronize()
        self._buf.numpy()[:n] = host
        dev = torch.empty(n, dtype=torch.uint8, device=device())
        dev.copy_(self._buf[:n], non_blocking=True)
        if self._event is None:
            self._event = torch.cuda.Event()
        self._event.record()
        return dev


PINNED = _PinnedStage()


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=torch_dtype(dtype), device=device())


def zeros(shape, dtype) -> torch.Tensor:
    return torch.zeros(shape, dtype=torch_dtype(dtype), device=device())


class Workspace:
    """Grow-only scratch buffer per device (zero-filled on growth)."""

    def __init__(self):
        self._buf: dict[int, torch.Tensor] = {}

    def get(self, nbytes: int) -> tuple[int, int]:
        dev = device()
        key = dev.index or 0
        buf = self._buf.get(key)
        if buf is None or buf.numel() < nbytes:
            size = max(int(nbytes), 1 << 20)
            buf = torch.zeros(size, dtype=torch.uint8, device=dev)
            self._buf[key] = buf
        return buf.data_ptr(), buf.numel()


WORKSPACE = Workspace()


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()
