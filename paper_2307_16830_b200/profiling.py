"""Optional CUDA-event phase timing (off by default; used by bench.py).

``with span("refactor"):`` records a start/stop event pair on the current
stream when profiling is enabled; ``summary()`` turns the pairs into
milliseconds per phase (count, total, mean).
"""
from __future__ import annotations

import contextlib
from collections import defaultdict

import torch

_enabled = False
_spans: dict = defaultdict(list)


def enable(on: bool = True) -> None:
    global _enabled
    _enabled = on


def reset() -> None:
    _spans.clear()


_NULL = contextlib.nullcontext()


@contextlib.contextmanager
def _span(name: str):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    try:
        yield
    finally:
        b.record()
        _spans[name].append((a, b))


def span(name: str):
    """Event pair around a phase when profiling is on; a shared no-op otherwise."""
    return _span(name) if _enabled else _NULL


def summary() -> dict:
    torch.cuda.synchronize()
    out = {}
    for k, v in _spans.items():
        ms = [a.elapsed_time(b) for a, b in v]
        out[k] = {"count": len(ms), "total_ms": sum(ms), "mean_ms": sum(ms) / max(1, len(ms))}
    return out
