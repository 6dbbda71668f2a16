"""Helpers shared by the GPU parity tests (test infrastructure)."""

import ctypes

import numpy as np
import torch

from paper_2505_21404_b200 import _lib, kernels


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def class_descs(classes):
    """oracle OpClass list -> (ctypes ClassDesc array, keep-alive device tensors)."""
    arr = (_lib.ClassDesc * len(classes))()
    keep = []
    for k, c in enumerate(classes):
        d = arr[k]
        pts = dev(c.points)
        f = dev(c.f)
        keep += [pts, f]
        d.count = c.count
        d.ngrad = len(c.grad_dims)
        d.nlap = len(c.lap_dims)
        for g, gd in enumerate(c.grad_dims):
            d.grad_dims[g] = gd
            d.cg[g] = c.cg[g]
        for l, ld in enumerate(c.lap_dims):
            d.lap_grad[l] = c.grad_dims.index(ld)
        d.cu, d.cl, d.weight = c.cu, c.cl, c.weight
        d.points = pts.data_ptr()
        d.f = f.data_ptr()
        d.c3 = getattr(c, "c3", 0.0)
        if getattr(c, "inputs", None) is not None:
            inp = dev(c.inputs)
            keep.append(inp)
            d.inputs = inp.data_ptr()
        if getattr(c, "pgrad", None) is not None:
            gi = torch.as_tensor(np.ascontiguousarray(c.pgrad, dtype=np.int32), device="cuda")
            keep.append(gi)
            d.grad_idx = gi.data_ptr()
        if getattr(c, "pcoef", None) is not None:
            co = dev(c.pcoef)
            keep.append(co)
            d.coefs = co.data_ptr()
    return arr, keep
