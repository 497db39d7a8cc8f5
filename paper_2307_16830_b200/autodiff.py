"""Objective/constraint evaluation and sparse derivatives on the GPU.

API of reference src/gridnlp/autodiff.py:22-142.  Each call launches the
pattern-block AD kernels (``csrc/ad.cu``): one record-parallel pass over
every pattern block plus a deterministic gather into the fixed COO slots.
numpy inputs are copied to HBM and results copied back (drop-in for the
reference); CUDA-tensor inputs stay on the device.  Non-finite results
raise ``NonFiniteResult`` exactly where the reference raises.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .model import CompiledModel

F, C, GRAD, JAC, HESS = 1, 2, 4, 8, 16
RESET = 256   # zero the flag word inside the same C call (no separate fill launch)
_WHAT_NAME = ((F, "objective"), (C, "constraint"), (GRAD, "gradient"), (JAC, "jacobian"),
              (HESS, "hessian"))


class NonFiniteResult(ArithmeticError):
    """Evaluation produced NaN or infinity (point outside the domain)."""


class DerivativeBuffers:
    """Preallocated output arrays matching a model's fixed sparsity (autodiff.py:26-33)."""

    def __init__(self, model: CompiledModel):
        self.gradient = np.zeros(model.n_var)
        self.jacobian_values = np.zeros(model.nnz_jac)
        self.hessian_values = np.zeros(model.nnz_hess)
        self.constraint_values = np.zeros(model.n_con)


class DeviceEvaluator:
    """Device buffers + launcher for one compiled model."""

    def __init__(self, model: CompiledModel):
        self.model = model
        self.handle = model.device_plan()
        self.contrib = D.empty(max(1, model.n_contrib))
        self.flags = torch.zeros(1, dtype=torch.int32, device=self.contrib.device)

    def launch(self, x, what, y=None, obj_weight=1.0, con_scale=None, obj_scale=1.0,
               f=None, c=None, grad=None, jac=None, hess=None, flags=None):
        """Enqueue one evaluation; outputs are caller-provided CUDA tensors.
        `flags` (an int32 CUDA tensor) receives the non-finite bits instead of
        the evaluator's own word (the solver's scalar mailbox)."""
        L.check(L.lib().gn_ad_eval(
            self.handle, L.ptr(x), L.ptr(y), float(obj_weight), L.ptr(con_scale), float(obj_scale),
            L.ptr(f), L.ptr(c), L.ptr(grad), L.ptr(jac), L.ptr(hess), what, L.ptr(self.contrib),
            L.ptr(self.flags if flags is None else flags), D.stream_ptr()))

    def raise_on_flags(self, flags_value: int, order=(F, C, GRAD, JAC, HESS)):
        for bit in order:
            if flags_value & bit:
                name = dict(_WHAT_NAME)[bit]
                raise NonFiniteResult(f"{name} evaluation produced a non-finite value")


def evaluator(model: CompiledModel) -> DeviceEvaluator:
    ev = getattr(model, "_evaluator", None)
    if ev is None:
        ev = DeviceEvaluator(model)
        model._evaluator = ev
    return ev


def _run(model, x, what, n_out, y=None, obj_weight=1.0, out=None):
    ev = evaluator(model)
    xd = D.to_dev(x)
    yd = None if y is None else D.to_dev(y)
    ev.flags.zero_()
    res = D.empty(n_out) if (out is None or not D.is_tensor(out)) else out
    kw = {F: "f", C: "c", GRAD: "grad", JAC: "jac", HESS: "hess"}
    ev.launch(xd, what, y=yd, obj_weight=obj_weight, **{kw[what]: res})
    ev.raise_on_flags(int(ev.flags.item()))
    if D.is_tensor(x) or D.is_tensor(out):
        return res
    host = D.to_host(res)
    if out is not None:
        out[...] = host
        return out
    return host


def eval_objective(model: CompiledModel, x) -> float:
    r = _run(model, x, F, 1)
    return float(r[0]) if not D.is_tensor(r) else float(r[0].item())


def eval_constraints(model: CompiledModel, x, out=None):
    return _run(model, x, C, model.n_con, out=out)


def eval_gradient(model: CompiledModel, x, out=None):
    return _run(model, x, GRAD, model.n_var, out=out)


def eval_jacobian(model: CompiledModel, x, out=None):
    return _run(model, x, JAC, model.nnz_jac, out=out)


def eval_lagrangian_hessian(model: CompiledModel, x, y, obj_weight: float = 1.0, out=None):
    """Lower-triangle values of obj_weight*H(f) + sum_i y_i H(g_i)."""
    if y is None or (not D.is_tensor(y) and np.asarray(y).size == 0):
        y = np.zeros(max(1, model.n_con))
    return _run(model, x, HESS, model.nnz_hess, y=y, obj_weight=obj_weight, out=out)


def pattern_source(model: CompiledModel) -> str:
    """CUDA source generated from the model's pattern tapes (one device
    function per distinct pattern; compiled with NVRTC at upload)."""
    import ctypes

    need = ctypes.c_size_t()
    L.check(L.lib().gn_model_pattern_source(model._handle, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    L.check(L.lib().gn_model_pattern_source(model._handle, buf, need.value, None))
    return buf.value.decode()


def ad_backend(model: CompiledModel) -> str:
    """'patterns' (generated kernels) or 'interpreter: <reason>'."""
    import ctypes

    model.device_plan()
    buf = ctypes.create_string_buffer(512)
    L.check(L.lib().gn_model_ad_backend(model._handle, buf, 512))
    return buf.value.decode()
