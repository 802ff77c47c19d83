"""Device plumbing: CUDA device/stream handles and reusable workspaces (torch allocations)."""

from __future__ import annotations

import torch

_ws: dict[tuple, torch.Tensor] = {}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("bastion needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def workspace(tag: str, nbytes: int) -> torch.Tensor:
    """Grow-only byte workspace per (tag, device)."""
    dev = require_cuda()
    key = (tag, dev.index)
    buf = _ws.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
        _ws[key] = buf
    return buf


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()
