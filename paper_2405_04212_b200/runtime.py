"""Device plumbing: PyTorch supplies device memory and streams; the compute is
libtmb200.so.  Every helper raises if no CUDA device is present -- the
package never silently computes on the CPU."""

from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _lib

_checked = False


def require_device():
    """Raise unless a CUDA (sm_100) device and libtmb200.so are usable."""
    global _checked
    if _checked:
        return
    import torch
    if not torch.cuda.is_available():
        raise _lib.TmbError(_lib.TMB_E_NO_DEVICE,
                            "no CUDA device: the B200 path has no CPU fallback")
    torch.cuda.init()
    lib = _lib.load()
    sm = ct.c_int()
    major = ct.c_int()
    minor = ct.c_int()
    l2 = ct.c_int64()
    smem = ct.c_int()
    _lib.call("tmb_device_info", torch.cuda.current_device(), ct.byref(sm), ct.byref(major),
              ct.byref(minor), ct.byref(l2), ct.byref(smem))
    if major.value != 10:
        raise _lib.TmbError(_lib.TMB_E_NO_DEVICE,
                            f"device is sm_{major.value}{minor.value}; built for sm_100a")
    assert lib.tmb_abi_version() == 1
    _checked = True


def device():
    import torch
    require_device()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr():
    import torch
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


def to_dev(a: np.ndarray, dtype=None):
    """numpy -> contiguous device tensor (pinned staging for large arrays)."""
    import torch
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    t = torch.from_numpy(a)
    if a.nbytes >= (1 << 20):
        t = t.pin_memory()
    return t.to(device(), non_blocking=True)


def empty(shape, dtype):
    import torch
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype):
    import torch
    return torch.zeros(shape, dtype=dtype, device=device())


def ptr(t) -> ct.c_void_p:
    return ct.c_void_p(t.data_ptr()) if t is not None else ct.c_void_p(0)


def np_ptr(a: np.ndarray) -> ct.c_void_p:
    return a.ctypes.data_as(ct.c_void_p)


def to_host(t) -> np.ndarray:
    return t.cpu().numpy()
