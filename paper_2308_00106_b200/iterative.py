"""Iterative drivers on the permuted matrix (C5).

The paper's premise is that the matrix is reused many times, so the one-time
permutation cost amortises over iterations.  The
reference has no solver; its oracle is a numpy loop over spmv_csr.  Here one
iteration is a fixed launch sequence with every scalar in device memory
(blas1.cu), so K iterations are captured once in a CUDA graph and replayed.

PermutedOperator keeps the iterate in permuted coordinates:
    z_k = P_c^-1 x_k   (z[p_c[i]] = x[i], i.e. permute_vector(x, p_c))
    B z_k = P_r A x_k  (the permuted matrix of permute_csr)
    z_{k+1} = P_c^-1 (A x_k) = (B z_k)[q],  q = p_r o inverse(p_c)
so an iteration costs one SpMV on B plus one gather, instead of two vector
permutations; with a symmetric permutation (p_c = p_r, B = P A P^T) q is the
identity and no gather is needed (the SPD case CG requires).

Folding (default).  The gather by q is a FIXED permutation, so it can be folded
into the matrix once instead of being paid every iteration: iterating in row-
permuted coordinates u_k = P_r x_k gives u_{k+1} = (P_r A P_r^-1) u_k, i.e. the
row+column permuted operator of a ROW_COLUMN_PERMUTE strategy is, for repeated
application, the symmetric permutation by p_r (a random row AND column
relabelling: the same maximal-entropy structure).  The operator then builds
permute_csr(A, p_r, p_r) once and an iteration is just the SpMV (fold=False
keeps B = P_r A P_c and the per-iteration gather).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _cuda, _lib
from ._cuda import ptr, stream
from .kernels import spmv_into
from .matio import CsrMatrix
from .permute import Permutation, compose, inverse, permute_csr, permute_vector


def _scratch(dev) -> tuple[torch.Tensor, torch.Tensor]:
    n_part = _lib.query_i64("sme_blas_partials")
    return (torch.zeros(4, dtype=torch.float64, device=dev),
            torch.zeros(n_part, dtype=torch.float64, device=dev))


class PermutedOperator:
    """y = A x applied through B = P_r A P_c in permuted coordinates."""

    def __init__(self, A: CsrMatrix, p_r: Permutation | None = None, p_c: Permutation | None = None,
                 kernel: str = "auto", fold: bool = True):
        if A.n_rows != A.n_cols:
            raise ValueError("iterative drivers need a square matrix")
        self.A, self.kernel = A, kernel
        self.folded = fold and p_r is not None and p_c is not None and not (p_r == p_c)
        if self.folded:
            p_c = p_r  # the gather by q = p_r o p_c^-1 folded into the columns (module docstring)
        self.p_r, self.p_c = p_r, p_c
        self.B = permute_csr(A, p_r, p_c) if (p_r is not None or p_c is not None) else A
        self.q = None  # gather index mapping B z back into permuted coordinates
        if p_r is not None or p_c is not None:
            same = p_r is not None and p_c is not None and p_r == p_c
            if not same:
                pr = p_r if p_r is not None else _ident(A.n_rows)
                pc = p_c if p_c is not None else _ident(A.n_cols)
                self.q = compose(pr, inverse(pc)).d_forward
        self.n = A.n_rows
        self.dtype = A.dtype
        self.dev = A.d_row_ptr.device
        self._tmp = torch.empty(self.n, dtype=self.dtype, device=self.dev)

    def to_permuted(self, x) -> torch.Tensor:
        """z = P_c^-1 x (x in original coordinates)."""
        xd = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float64))
        xd = xd.to(self.dev, self.dtype)
        return permute_vector(xd, self.p_c) if self.p_c is not None else xd.clone()

    def from_permuted(self, z: torch.Tensor) -> torch.Tensor:
        """x = P_c z."""
        if self.p_c is None:
            return z.clone()
        out = torch.empty_like(z)
        _lib.call("sme_gather", _cuda.sme_dtype(z), self.n, ptr(self.p_c.d_forward), ptr(z), ptr(out), stream())
        return out

    def fused_layout(self):
        """The fused-epilogue SpMV of this operator: the seg layout (with the full last
        panel) for 'seg', VectorEpi for 'vector' (no gather by q); None otherwise or
        when values are not f64."""
        from .kernels import auto_kernel, default_lanes
        from .seg import seg_of

        kern = auto_kernel(self.B) if self.kernel == "auto" else self.kernel
        if self.dtype != torch.float64:
            return None
        if not hasattr(self, "_qinv"):
            self._qinv = Permutation(self.q, _trusted=True).d_inverse if self.q is not None else None
        if kern == "seg":
            return seg_of(self.B, full_last=True)
        if kern == "vector" and self.q is None and not self.B.wide:  # VectorEpi: int32 row_ptr only
            return VectorEpi(self.B, default_lanes(self.B))
        return None

    def apply(self, z: torch.Tensor, out: torch.Tensor) -> None:
        """out = P_c^-1 A P_c z (stream-ordered; no allocation: graph-capturable)."""
        if self.q is None:
            spmv_into(self.B, z, out, self.kernel)
        else:
            spmv_into(self.B, z, self._tmp, self.kernel)
            _lib.call("sme_gather", _cuda.sme_dtype(out), self.n, ptr(self.q), ptr(self._tmp), ptr(out), stream())


class VectorEpi:
    """The CSR-vector twin of the seg fused epilogue (sme_spmv_vector_epi): one launch
    computes out = s * (A x) and the iteration's reduction (same interface as
    SegLayout.epi_pass / epi_cg_pass)."""

    n_panels = 1
    full_last = True

    def __init__(self, B: CsrMatrix, lanes: int):
        self.B, self.lanes = B, int(lanes)
        self.n_warps = _lib.query_i64("sme_spmv_vector_epi_blocks", B.n_rows, self.lanes)  # partials length

    def epi_pass(self, xd, y, out, qinv, scal, partials, ticket, result) -> None:
        if qinv is not None:
            raise ValueError("the CSR-vector epilogue does not scatter: fold the operator")
        B = self.B
        _lib.call("sme_spmv_vector_epi", self.lanes, B.n_rows, ptr(B.d_row_ptr), ptr(B.d_col_idx), ptr(B.d_values),
                  ptr(xd), ptr(out), ptr(scal), None, ptr(partials), ptr(ticket), ptr(result), 0, stream())

    def epi_cg_pass(self, p, y, out, partials, ticket, scal) -> None:
        B = self.B
        _lib.call("sme_spmv_vector_epi", self.lanes, B.n_rows, ptr(B.d_row_ptr), ptr(B.d_col_idx), ptr(B.d_values),
                  ptr(p), ptr(out), None, ptr(p), ptr(partials), ptr(ticket), ptr(scal), 1, stream())


def _ident(n: int) -> Permutation:
    from .permute import identity_permutation

    return identity_permutation(n)


class PowerIteration:
    """x_{k+1} = A x_k / ||A x_k|| (2-norm); eigenvalue estimate ||A x_k||.

    Fused mode (seg or CSR-vector operators, f64): one step is the operator's passes with
    the BLAS-1 work folded into the last pass (sme_spmv_seg_epi): the iterate is
    kept unnormalised, w_{k+1} = (B w_k) / ||w_k|| scattered straight into
    permuted coordinates, and ||w_{k+1}||^2 (the eigenvalue estimate squared) and
    the next scale come out of the same launch — no gather, dot or scale kernels.
    Otherwise: SpMV, gather, dot, scale (blas1.cu)."""

    def __init__(self, op: PermutedOperator, x0, fused: bool | None = None):
        self.op = op
        self.z = op.to_permuted(x0)
        self.y = torch.empty_like(self.z)
        self.scal, self.partial = _scratch(op.dev)
        self.norm2 = torch.zeros(1, dtype=torch.float64, device=op.dev)
        self.graph: torch.cuda.CUDAGraph | None = None
        self.graph_steps = 0
        dt = _cuda.sme_dtype(self.z)
        s = stream()
        # normalise x0
        _lib.call("sme_dot", dt, op.n, ptr(self.z), ptr(self.z), ptr(self.partial), ptr(self.norm2), ptr(self.scal), 3, s)
        _lib.call("sme_scale", dt, op.n, ptr(self.z), ptr(self.z), ptr(self.scal), 3, s)
        self.lay = op.fused_layout() if fused is not False else None
        if fused and self.lay is None:
            raise ValueError("the fused power iteration needs a 'seg' or 'vector' operator with f64 values")
        self.fused = self.lay is not None
        if self.fused:
            self.w = [self.z, self.y]  # iterate ping-pongs between the two
            self.cur = 0
            self.res = torch.tensor([1.0, 0.0], dtype=torch.float64, device=op.dev)  # {scale, ||w||^2}
            self.epi_partials = torch.zeros(getattr(self.lay, "epi_partials_len", self.lay.n_warps),
                                            dtype=torch.float64, device=op.dev)
            self.ticket = torch.zeros(1, dtype=torch.int32, device=op.dev)

    def _step(self) -> None:
        if self.fused:
            a, b = self.w[self.cur], self.w[1 - self.cur]
            self.lay.epi_pass(a, self.op._tmp, b, self.op._qinv, self.res, self.epi_partials, self.ticket, self.res)
            self.cur = 1 - self.cur
            return
        dt = _cuda.sme_dtype(self.z)
        self.op.apply(self.z, self.y)
        _lib.call("sme_dot", dt, self.op.n, ptr(self.y), ptr(self.y), ptr(self.partial), ptr(self.norm2),
                  ptr(self.scal), 3, stream())
        _lib.call("sme_scale", dt, self.op.n, ptr(self.z), ptr(self.y), ptr(self.scal), 3, stream())

    def capture(self, steps: int) -> None:
        """Record `steps` iterations into one CUDA graph (after one eager warm-up step);
        fused mode alternates two buffers, so it records an even number of steps."""
        if self.fused and steps % 2:
            raise ValueError("the fused power iteration captures an even number of steps")
        self._step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        start = getattr(self, "cur", 0)
        with torch.cuda.graph(g):
            for _ in range(steps):
                self._step()
        if self.fused:
            self.cur = start  # capture does not run the steps; replays leave the iterate where it was
        self.graph, self.graph_steps = g, steps

    def run(self, steps: int) -> None:
        if self.graph is not None and steps % self.graph_steps == 0:
            for _ in range(steps // self.graph_steps):
                self.graph.replay()
        else:
            for _ in range(steps):
                self._step()

    @property
    def eigenvalue(self) -> float:
        return math.sqrt(float((self.res[1] if self.fused else self.norm2).item()))

    def x(self) -> torch.Tensor:
        if self.fused:  # the stored iterate is unnormalised: x = w / ||w||
            z = self.w[self.cur] * self.res[0]
            return self.op.from_permuted(z)
        return self.op.from_permuted(self.z)


class ConjugateGradient:
    """CG for SPD A (use a symmetric permutation p_c = p_r so that B = P A P^T is SPD).

    Fused mode (seg or CSR-vector operators, f64): p.Ap is reduced inside the SpMV's last pass
    and alpha written by its last CTA (sme_spmv_seg_epi_cg), so a step is the
    panel passes + the x/r update + the p update."""

    def __init__(self, op: PermutedOperator, b, x0=None, fused: bool | None = None):
        if op.q is not None:
            raise ValueError("CG needs a symmetric permutation (p_c == p_r) so that B stays SPD")
        self.op = op
        dev, dt = op.dev, op.dtype
        self.b = op.to_permuted(b)
        self.x = torch.zeros_like(self.b) if x0 is None else op.to_permuted(x0)
        self.r = self.b.clone()
        if x0 is not None:  # r = b - B x
            tmp = torch.empty_like(self.b)
            op.apply(self.x, tmp)
            _lib.call("sme_axpby", _cuda.sme_dtype(tmp), op.n, -1.0, ptr(tmp), 1.0, ptr(self.r), stream())
        self.p = self.r.clone()
        self.ap = torch.empty_like(self.b)
        self.scal, self.partial = _scratch(dev)
        self.graph: torch.cuda.CUDAGraph | None = None
        self.graph_steps = 0
        _lib.call("sme_dot", _cuda.sme_dtype(self.r), op.n, ptr(self.r), ptr(self.r), ptr(self.partial),
                  ptr(self.scal), ptr(self.scal), 0, stream())  # scal[0] = r.r
        del dt
        self.lay = op.fused_layout() if fused is not False else None
        if fused and self.lay is None:
            raise ValueError("the fused CG needs a 'seg' or 'vector' operator with f64 values")
        self.fused = self.lay is not None
        if self.fused:
            self.epi_partials = torch.zeros(getattr(self.lay, "epi_partials_len", self.lay.n_warps),
                                            dtype=torch.float64, device=dev)
            self.ticket = torch.zeros(1, dtype=torch.int32, device=dev)

    def _step(self) -> None:
        dt = _cuda.sme_dtype(self.r)
        if self.fused:
            self.lay.epi_cg_pass(self.p, self.op._tmp, self.ap, self.epi_partials, self.ticket, self.scal)
        else:
            self.op.apply(self.p, self.ap)
            _lib.call("sme_dot", dt, self.op.n, ptr(self.p), ptr(self.ap), ptr(self.partial), None, ptr(self.scal),
                      1, stream())
        _lib.call("sme_cg_update", dt, self.op.n, ptr(self.x), ptr(self.r), ptr(self.p), ptr(self.ap),
                  ptr(self.scal), ptr(self.partial), stream())

    def capture(self, steps: int) -> None:
        self._step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(steps):
                self._step()
        self.graph, self.graph_steps = g, steps

    def run(self, steps: int) -> None:
        if self.graph is not None and steps % self.graph_steps == 0:
            for _ in range(steps // self.graph_steps):
                self.graph.replay()
        else:
            for _ in range(steps):
                self._step()

    @property
    def residual_norm2(self) -> float:
        return float(self.scal[0].item())

    def solution(self) -> torch.Tensor:
        return self.op.from_permuted(self.x)
