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


def graph_kernel_nodes(graph) -> int:
    """Number of kernel nodes in a captured torch CUDAGraph (exact launch count per replay)."""
    import ctypes as C
    import glob
    import os

    global _cudart
    try:
        _cudart
    except NameError:
        _cudart = None
    if _cudart is None:
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                       "libcudart.so.*"))
        _cudart = C.CDLL(cands[0] if cands else "libcudart.so")
    raw = C.c_void_p(graph.raw_cuda_graph())
    n = C.c_size_t(0)
    if _cudart.cudaGraphGetNodes(raw, None, C.byref(n)) != 0:
        return -1
    nodes = (C.c_void_p * n.value)()
    _cudart.cudaGraphGetNodes(raw, nodes, C.byref(n))
    kernels = 0
    for i in range(n.value):
        t = C.c_int(-1)
        _cudart.cudaGraphNodeGetType(C.c_void_p(nodes[i]), C.byref(t))
        kernels += t.value == 0  # cudaGraphNodeTypeKernel
    return kernels
