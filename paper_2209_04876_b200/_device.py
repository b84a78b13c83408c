"""Device plumbing: torch owns HBM allocations and streams; kernels come from the C-ABI.

Inputs are accepted as anything ``np.asarray(..., float64)`` accepts (the reference's
convention, e.g. tensor.py:35-52) or as torch tensors (CPU or CUDA).  Results are returned as
fresh NumPy arrays when the primary input lived on the host, and as CUDA tensors when it
already lived on the device (zero-copy pipelines)."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import InvalidInputError

F64 = torch.float64
I64 = torch.int64


_READY = [False]


def require_cuda():
    if _READY[0]:
        return
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2209_04876_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    _lib.load()
    _READY[0] = True


# the raw current device / stream without building torch Stream objects (every C-ABI call passes
# the current stream; the Python wrappers cost microseconds per call on the host-bound small paths)
_GET_DEVICE = getattr(torch._C, "_cuda_getDevice", None)
_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_DEVICES: dict = {}


def dev() -> torch.device:
    i = _GET_DEVICE() if (_GET_DEVICE is not None and _READY[0]) else torch.cuda.current_device()
    d = _DEVICES.get(i)
    if d is None:
        d = _DEVICES.setdefault(i, torch.device("cuda", i))
    return d


def stream() -> ctypes.c_void_p:
    if _GET_DEVICE is not None and _RAW_STREAM is not None and _READY[0]:
        return ctypes.c_void_p(_RAW_STREAM(_GET_DEVICE()))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def on_device(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_dev(x, dtype=F64) -> torch.Tensor:
    """Contiguous CUDA tensor of ``dtype`` (copies host data; no-op for matching CUDA input)."""
    require_cuda()
    if isinstance(x, torch.Tensor):
        if x.is_cuda and x.dtype == dtype and x.is_contiguous() and x.device.index == torch.cuda.current_device():
            return x  # already where and what it needs to be (the common device-resident case)
        return x.to(device=dev(), dtype=dtype).contiguous()
    npdt = np.float64 if dtype == F64 else np.int64
    a = np.ascontiguousarray(np.asarray(x, dtype=npdt))
    t = torch.from_numpy(a)
    if a.nbytes >= (1 << 20):
        t = t.pin_memory()
        return t.to(dev(), non_blocking=True)
    return t.to(dev())


def empty(*shape, dtype=F64) -> torch.Tensor:
    return torch.empty(*shape, dtype=dtype, device=dev())


def zeros(*shape, dtype=F64) -> torch.Tensor:
    return torch.zeros(*shape, dtype=dtype, device=dev())


def p(t) -> ctypes.c_void_p:
    """Device pointer of a tensor (None -> NULL)."""
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def out(t: torch.Tensor, host: bool):
    return t.detach().cpu().numpy() if host else t


def check_flags(flags: torch.Tensor, name: str, need_nonzero: bool = False):
    f = flags.cpu().tolist()
    if f[0]:
        raise InvalidInputError(f"{name} contains non-finite entries")
    if need_nonzero and not f[1]:
        raise InvalidInputError(f"{name} is identically zero")


def finite_flags(t: torch.Tensor) -> torch.Tensor:
    flags = torch.zeros(2, dtype=torch.int32, device=t.device)
    _lib.call("ks_check_finite_nonzero", p(t), t.numel(), p(flags), stream())
    return flags


def scalar(t: torch.Tensor) -> float:
    return float(t.item())
