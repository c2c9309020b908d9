"""B200-native recycled GMRES(m) for sequences of convection-diffusion systems (arXiv:1807.09467).

The product is ``lib/librg.so`` (C ABI in ``include/rg.h``; fp64 CUDA kernels for sm_100a in
``csrc/``).  ``rg`` is its thin ctypes binding (same function names); ``Context`` is a small
convenience wrapper over it that keeps the argument arrays alive.  Importing this package fails
loudly when the CUDA library has not been built: there is no CPU fallback.
"""
from __future__ import annotations

from . import rg
from .rg import RgError  # noqa: F401

__all__ = ["rg", "Context", "RgError"]


class Context:
    """One rg_ctx: a sequence solver for systems of dimension n (marshalling only)."""

    def __init__(self, n, row_ptr, col_idx, val, fmt="csr", block=1, sell_C=0, max_m=64,
                 max_snapshots=32, max_k=32, stream=None, flags=0, sell_sigma=1):
        keep = []
        self.n, self.fmt, self.block, self.sell_C = int(n), fmt, int(block), int(sell_C)
        self.sell_sigma = int(sell_sigma)
        A = rg.make_matrix(n, row_ptr, col_idx, val, fmt, block, sell_C, keep, self.sell_sigma)
        self.max_snapshots = max_snapshots
        self.ctx = rg.rg_create(n, A, max_m, max_snapshots, max_k, stream, flags)

    def update_matrix(self, val, row_ptr=None, col_idx=None):
        keep = []
        A = rg.make_matrix(self.n, row_ptr, col_idx, val, self.fmt, self.block, self.sell_C, keep, self.sell_sigma)
        rg.rg_update_matrix(self.ctx, A)

    def values_ptr(self):
        """Device pointer / length of the library-owned matrix values (rg_matrix_values)."""
        return rg.rg_matrix_values(self.ctx)

    def update_values_inplace(self, nnz):
        """The values behind values_ptr() were rewritten on the context's stream."""
        rg.rg_update_values_inplace(self.ctx, self.n, nnz, self.fmt, self.block, self.sell_C, self.sell_sigma)

    def push_snapshot(self, x):
        rg.rg_push_snapshot(self.ctx, x)

    def clear_snapshots(self):
        rg.rg_clear_snapshots(self.ctx)

    def build_recycle(self, k, modes="largest", deferred=False):
        if modes == "largest":
            return rg.rg_build_recycle(self.ctx, k, self.max_snapshots, deferred)
        return rg.rg_build_recycle_modes(self.ctx, k, modes, self.max_snapshots)

    def solve(self, b, x_out, x0=None, m=30, variant="plain", tol=1e-8, max_iters=20000, history_cap=0):
        return rg.rg_solve(self.ctx, b, x_out, x0, m, variant, tol, max_iters, history_cap)

    def apply(self, x, y):
        rg.rg_apply(self.ctx, x, y)

    def set_preconditioner(self, kind="ssor", omega=1.0, colors=None):
        """Right SSOR(omega) preconditioner in a multicolour order (None kind removes it); returns
        the number of colours."""
        if colors is not None:
            if hasattr(colors, "is_cuda"):        # torch tensor
                import torch
                colors = colors.to(dtype=torch.int32).contiguous()
            else:
                import numpy as np
                colors = np.ascontiguousarray(colors, dtype=np.int32)
        return rg.rg_set_preconditioner(self.ctx, kind, omega, colors)

    def apply_preconditioner(self, x, y):
        rg.rg_apply_preconditioner(self.ctx, x, y)

    def export(self, which, out):
        return rg.rg_export(self.ctx, which, out)

    def kernel_stats(self):
        return rg.rg_kernel_stats(self.ctx)

    def kernel_trace(self, cap=65536):
        return rg.rg_kernel_trace(self.ctx, cap)

    def reset_kernel_stats(self):
        rg.rg_reset_kernel_stats(self.ctx)

    def close(self):
        if self.ctx is not None:
            rg.rg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
