"""Device plumbing: tensors, streams, host<->device staging.

PyTorch is used only for device memory, streams and the caching allocator;
all arithmetic runs in the CUDA library (``_lib``).  There is no CPU path:
anything that needs the GPU raises ``RuntimeError`` when CUDA is absent.
"""

from __future__ import annotations

import numpy as np
import torch

U64 = torch.uint64


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2209_01290_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")


_get_device = getattr(torch._C, "_cuda_getDevice", None)


def index() -> int:
    """Current CUDA device index (the raw getter: no lazy-init bookkeeping)."""
    if _get_device is not None and torch.cuda.is_initialized():
        return _get_device()
    require_cuda()
    return torch.cuda.current_device()


def device() -> torch.device:
    return torch.device("cuda", index())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_ptr() -> int:
    """cudaStream_t of torch's current stream (the launch stream) - the raw
    handle without building a torch.cuda.Stream object (a few us per call)."""
    if _raw_stream is not None:
        return _raw_stream(index())
    return torch.cuda.current_stream().cuda_stream


def is_device_tensor(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def host_u64(values) -> np.ndarray:
    """Coerce a list / ndarray / CPU tensor to a contiguous uint64 ndarray."""
    if isinstance(values, torch.Tensor):
        if values.dtype != U64:
            raise ValueError(f"expected uint64 tensor, got {values.dtype}")
        return values.detach().cpu().numpy()
    if isinstance(values, np.ndarray):
        if values.dtype != np.uint64:
            if not np.issubdtype(values.dtype, np.integer):
                raise ValueError(f"expected integer array, got {values.dtype}")
        return np.ascontiguousarray(values, dtype=np.uint64)
    return np.array([int(v) for v in values], dtype=np.uint64)


def to_device(values) -> torch.Tensor:
    """A contiguous uint64 CUDA tensor holding ``values`` (no copy if it is one)."""
    if isinstance(values, torch.Tensor) and values.is_cuda:
        if values.dtype != U64:
            raise ValueError(f"expected uint64 tensor, got {values.dtype}")
        return values if values.is_contiguous() else values.contiguous()
    arr = host_u64(values)
    return torch.from_numpy(arr).to(device(), non_blocking=False)


def empty(shape, like: torch.Tensor | None = None) -> torch.Tensor:
    dev = like.device if like is not None else device()
    return torch.empty(shape, dtype=U64, device=dev)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()
