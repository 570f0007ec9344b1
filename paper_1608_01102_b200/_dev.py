"""Device-buffer plumbing: numpy/torch inputs -> contiguous CUDA tensors.

PyTorch is used only for device memory and the current stream.  Every
compute call goes through libsmk.so; a missing library or device raises
``errors.ExtensionMissing`` (there is no CPU fallback on the product path).
"""

import numpy as np
import torch

from . import _lib, errors

_DT = {torch.float64: _lib.SMK_F64, torch.float32: _lib.SMK_F32}


def require_device():
    if not torch.cuda.is_available():
        raise errors.ExtensionMissing("libsmk needs a CUDA device (no CPU fallback)")
    _lib.load()


def stream():
    return torch.cuda.current_stream().cuda_stream


def torch_dtype(dtype):
    if dtype is None:
        return torch.float64
    if isinstance(dtype, torch.dtype):
        return dtype
    return {"float64": torch.float64, "f64": torch.float64, "fp64": torch.float64,
            "float32": torch.float32, "f32": torch.float32, "fp32": torch.float32}[str(dtype)]


def as_dev(x, dtype=None):
    """Contiguous CUDA tensor (copy only when needed)."""
    if isinstance(x, torch.Tensor):
        t = x
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if not t.is_cuda:
            t = t.cuda()
        return t.contiguous()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def infer_dtype(*xs):
    for x in xs:
        if isinstance(x, torch.Tensor):
            return x.dtype
        if isinstance(x, (tuple, list)) and x:
            d = infer_dtype(*x)
            if d is not None:
                return d
    return None


def any_numpy(*xs):
    for x in xs:
        if isinstance(x, np.ndarray):
            return True
        if isinstance(x, (tuple, list)) and any_numpy(*x):
            return True
    return False


def out(t, numpy):
    if isinstance(t, tuple):
        return tuple(out(x, numpy) for x in t)
    if numpy:
        return t.detach().cpu().numpy()
    return t


def grid(spec, dtype):
    g = _lib.smk_grid()
    g.dim = spec.dim
    for a in range(3):
        g.res[a] = spec.res[a] if a < spec.dim else 1
    g.h = float(spec.h)
    g.boundary = _lib.SMK_PERIODIC if spec.periodic else _lib.SMK_NEUMANN
    g.dtype = _DT[dtype]
    return g
