"""Helpers for GPU tests: call C-ABI kernel entry points on torch device tensors."""
import ctypes

import numpy as np


def ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def call(name, *args):
    """Call p2r_<name>(*args, stream); tensors are passed as device pointers."""
    import torch
    from paper_2110_03888_b200 import _lib
    conv = []
    for a in args:
        if isinstance(a, torch.Tensor):
            conv.append(ptr(a))
        elif isinstance(a, float):
            conv.append(ctypes.c_float(a))
        elif isinstance(a, np.floating):
            conv.append(ctypes.c_float(float(a)))
        elif isinstance(a, ctypes._SimpleCData) or a is None:
            conv.append(a)
        else:
            conv.append(ctypes.c_int(int(a)))
    fn = getattr(_lib.lib(), "p2r_" + name)
    fn.restype = ctypes.c_int
    st = fn(*conv, stream())
    _lib.check(st)
    torch.cuda.synchronize()


def dev(a, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
