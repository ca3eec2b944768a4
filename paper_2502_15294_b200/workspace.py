"""Grow-only, zero-initialised device scratch shared by the librk entry points.

The split-K kernels keep per-(row, kv-head) arrival counters in the scratch and
reset them themselves, so the buffer is zeroed exactly once when it grows.
One arena per (device, stream, tag) keeps concurrently-queued calls apart.
"""

from __future__ import annotations

import torch

_ARENAS: dict = {}


def scratch(nbytes: int, device=None, tag: str = "default") -> torch.Tensor:
    dev = torch.device(device if device is not None else "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    key = (dev.index, torch.cuda.current_stream(dev).cuda_stream, tag)
    buf = _ARENAS.get(key)
    need = max(256, int(nbytes))
    if buf is None or buf.numel() < need:
        if buf is not None:
            torch.cuda.current_stream(dev).synchronize()
        buf = torch.zeros(need + (need >> 2), dtype=torch.uint8, device=dev)
        _ARENAS[key] = buf
    return buf
