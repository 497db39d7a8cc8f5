"""Device plumbing: the CUDA device, streams and tensor helpers (torch)."""
from __future__ import annotations

import numpy as np
import torch


class DeviceUnavailable(RuntimeError):
    """Raised when a device entry point runs without a CUDA device."""


_available = False
_devices: dict = {}


def require_cuda() -> torch.device:
    global _available
    if not _available:
        if not torch.cuda.is_available():
            raise DeviceUnavailable(
                "the condensed-space solve path runs on the GPU only (no CPU fallback); "
                "no CUDA device is visible")
        _available = True
    i = torch._C._cuda_getDevice()
    d = _devices.get(i)
    if d is None:
        d = _devices[i] = torch.device("cuda", i)
    return d


def stream_ptr(stream=None) -> int:
    """cudaStream_t of `stream` or of the current stream (the raw lookup:
    torch.cuda.current_stream() costs ~15 us of Python per call, and the
    driver asks for the stream at every launch)."""
    if stream is not None:
        return stream.cuda_stream
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


TRANSFER = {"h2d": 0, "d2h": 0}   # bytes moved by these helpers (bench accounting)


def to_dev(a, dtype=torch.float64):
    """numpy / list / tensor -> contiguous CUDA tensor of ``dtype``."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        if a.device.type != "cuda":
            TRANSFER["h2d"] += a.numel() * a.element_size()
        return a.to(device=dev, dtype=dtype).contiguous()
    t = torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device=dev)
    TRANSFER["h2d"] += t.numel() * t.element_size()
    return t


def trim_plan_cache() -> int:
    """Return the native plan allocator's cached blocks to the driver
    (gn_alloc_trim) and torch's cached blocks too; returns the native cache
    size before trimming (bytes)."""
    import ctypes

    from . import _lib as L

    before = ctypes.c_int64()
    L.check(L.lib().gn_alloc_trim(ctypes.byref(before)))
    torch.cuda.empty_cache()
    return before.value


def _retry_oom(fn):
    try:
        return fn()
    except torch.OutOfMemoryError:   # the plan cache may hold the memory torch needs
        trim_plan_cache()
        return fn()


def empty(n, dtype=torch.float64):
    return _retry_oom(lambda: torch.empty(int(n), dtype=dtype, device=require_cuda()))


def zeros(n, dtype=torch.float64):
    return _retry_oom(lambda: torch.zeros(int(n), dtype=dtype, device=require_cuda()))


def is_tensor(a) -> bool:
    return isinstance(a, torch.Tensor)


def to_host(t) -> np.ndarray:
    TRANSFER["d2h"] += t.numel() * t.element_size()
    return t.detach().cpu().numpy()
