"""Device plumbing: torch for memory and streams only (no torch compute)."""

import numpy as np

from .errors import NativeError

try:
    import torch
except Exception as e:  # pragma: no cover
    torch = None
    _torch_err = e


def require_cuda(device=None):
    if torch is None:
        raise NativeError(f"torch unavailable: {_torch_err}")
    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the B200 hydro path has no CPU fallback")
    return torch.device(device if device is not None else "cuda")


def stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes_void(s.cuda_stream)


def ctypes_void(x):
    import ctypes

    return ctypes.c_void_p(int(x))


def to_device(arr, device):
    a = np.ascontiguousarray(arr, dtype=np.float64)
    return torch.from_numpy(a).to(device, non_blocking=False)


def ptr(t):
    return None if t is None else t.data_ptr()
