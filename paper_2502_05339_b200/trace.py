"""Stage tracing: NVTX ranges (visible to ncu/nsys) plus optional CUDA-event
stage timers on the launching stream. Disabled by default (no events, no
syncs); bench.py enables it to attribute fit time to stages."""

from __future__ import annotations

import time
from contextlib import contextmanager

import torch

_rec = None


def enable():
    global _rec
    _rec = []


def disable():
    global _rec
    r, _rec = _rec, None
    return r or []


@contextmanager
def stage(name: str):
    nvtx = torch.cuda.is_available()
    if nvtx:
        torch.cuda.nvtx.range_push(name)
    if _rec is None:
        try:
            yield
        finally:
            if nvtx:
                torch.cuda.nvtx.range_pop()
        return
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    try:
        yield
    finally:
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record()
        _rec.append((name, e0, e1, time.perf_counter() - h0))
        if nvtx:
            torch.cuda.nvtx.range_pop()


def summarize(rec, steps: int = 1) -> dict:
    """{stage: ms per step} (stages may nest; each is its own interval)."""
    torch.cuda.synchronize()
    out: dict = {}
    for name, e0, e1, _ in rec:
        out[name] = out.get(name, 0.0) + e0.elapsed_time(e1)
    return {k: round(v / steps, 2) for k, v in out.items()}


def summarize_host(rec, steps: int = 1) -> dict:
    """{stage: host wall ms per step} (time the launching thread spent inside)."""
    out: dict = {}
    for name, _, _, h in rec:
        out[name] = out.get(name, 0.0) + h * 1e3
    return {k: round(v / steps, 2) for k, v in out.items()}
