"""Restarted GMRES on the device around the FDA apply (the
system A x = b solved with GMRES whose main cost is the matrix-vector product, and PAPER.md:981-982).

The operator is the C-ABI apply (`fda_apply`, all of it in libfda's CUDA kernels); the Krylov
vectors live in device memory as torch complex128 tensors and the small Hessenberg least-squares
problem is solved with Givens rotations on the host (restart-length scalars only).  This is solver
plumbing: with the synthetic singular corrections the system has no physical
meaning, and the corrected weights it would need are out of scope.
"""
from __future__ import annotations

import math

import torch

from . import fda


def gmres(plan_handle, b: torch.Tensor, tol: float = 1e-6, restart: int = 50, maxiter: int = 500,
          x0: torch.Tensor | None = None):
    """Solve H x = b with H the plan's operator.  b: complex128 CUDA tensor (n,).  Returns
    (x, residual history relative to ||b||, number of operator applies)."""
    if not (b.is_cuda and b.dtype == torch.complex128 and b.dim() == 1):
        raise ValueError("b must be a 1-D complex128 CUDA tensor")
    n = b.shape[0]
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    tmp = torch.empty_like(b)

    def apply(v, out):
        fda.fda_apply(plan_handle, torch.view_as_real(v), torch.view_as_real(out))

    bnorm = torch.linalg.vector_norm(b).item()
    if bnorm == 0.0:
        return x, [0.0], 0
    hist = []
    napply = 0
    V = torch.empty((restart + 1, n), dtype=b.dtype, device=b.device)
    while napply < maxiter:
        apply(x, tmp)
        napply += 1
        r = b - tmp
        beta = torch.linalg.vector_norm(r).item()
        hist.append(beta / bnorm)
        if beta / bnorm <= tol:
            break
        V[0] = r / beta
        H = [[0j] * restart for _ in range(restart + 1)]
        cs, sn = [0j] * restart, [0j] * restart
        g = [0j] * (restart + 1)
        g[0] = complex(beta)
        j_last = 0
        for j in range(restart):
            apply(V[j], tmp)
            napply += 1
            w = tmp.clone()
            for i in range(j + 1):  # modified Gram-Schmidt
                hij = torch.vdot(V[i], w)
                w -= hij * V[i]
                H[i][j] = complex(hij.item())
            hn = torch.linalg.vector_norm(w).item()
            H[j + 1][j] = complex(hn)
            if hn > 0:
                V[j + 1] = w / hn
            for i in range(j):  # previous Givens rotations
                t = cs[i].conjugate() * H[i][j] + sn[i].conjugate() * H[i + 1][j]
                H[i + 1][j] = -sn[i] * H[i][j] + cs[i] * H[i + 1][j]
                H[i][j] = t
            a, c = H[j][j], H[j + 1][j]
            den = math.sqrt(abs(a) ** 2 + abs(c) ** 2)
            cs[j], sn[j] = (a / den, c / den) if den > 0 else (1.0 + 0j, 0j)
            H[j][j] = cs[j].conjugate() * a + sn[j].conjugate() * c
            H[j + 1][j] = 0j
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j].conjugate() * g[j]
            j_last = j
            hist.append(abs(g[j + 1]) / bnorm)
            if hist[-1] <= tol or napply >= maxiter:
                break
        # back substitution and update
        m = j_last + 1
        y = [0j] * m
        for i in range(m - 1, -1, -1):
            s = g[i] - sum(H[i][l] * y[l] for l in range(i + 1, m))
            y[i] = s / H[i][i]
        yt = torch.tensor(y, dtype=b.dtype, device=b.device)
        x = x + (yt[:, None] * V[:m]).sum(dim=0)
        if hist[-1] <= tol:
            apply(x, tmp)
            napply += 1
            hist.append(torch.linalg.vector_norm(b - tmp).item() / bnorm)
            if hist[-1] <= 10 * tol:
                break
    return x, hist, napply
