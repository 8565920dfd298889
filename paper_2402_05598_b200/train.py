"""Training the SNO preconditioner on the GPU: the scheme of the paper's Fig. 3,
every step a libfcgno.so call.

  (a) FCG with B = I on the training systems: a tight solve gives u_exact, and the solve stopped
      after i iterations gives the CG iterate u_i (Krylov-subspace residuals, Eq. 8-9);
  (b) training pairs (r_i, e_i) = (f - A u_i, u_exact - u_i) (fcgno_krylov_pair);
  (c) minibatch AdamW on the Notay loss in error form (Eq. notay_loss_with_error) with
      Table 6's schedule (lr 1e-3 halved every 50 epochs, weight decay 1e-2);
  (d) the trained weights feed fcgno_fcg_solve (FCG with B = NO) on held-out systems.

This module sequences library calls and draws the permutations (the random numbers the method
uses); all arithmetic runs in the library's kernels.
"""
from __future__ import annotations

import numpy as np
import torch

from . import fcgno


def lr_at_epoch(epoch: int, lr0: float = 1e-3, decay: float = 0.5, every: int = 50) -> float:
    """Table 6."""
    return lr0 * decay ** (epoch // every)


def krylov_dataset(problem: fcgno.Problem, f: torch.Tensor, u0: torch.Tensor, sample_iters, m: int = 5,
                   tol_exact: float = 1e-12, maxit_exact: int = 20000, e_scale: float = 1.0):
    """Training pairs of every system of `problem` at the CG iterations `sample_iters` (Fig. 3 (a)-(b)).
    Returns (r, e, ksys): r, e [S][n][n] fp64 with S = len(sample_iters) * B (sample s belongs to system
    s % B), ksys [S] int32, and the per-system iteration count of the tight solve."""
    exact = fcgno.fcg_solve(problem, f, u0, m=m, tol=tol_exact, maxit=maxit_exact, history=False)
    u_star = exact.u
    rs, es = [], []
    for i in sample_iters:
        u_i = fcgno.fcg_solve(problem, f, u0, m=m, tol=0.0, maxit=int(i), history=False).u
        r, e = fcgno.krylov_pair(problem, f, u_star, u_i, e_scale=e_scale)
        rs.append(r)
        es.append(e)
    B = problem.B
    ksys = torch.arange(len(rs) * B, dtype=torch.int32, device=f.device) % B
    return torch.cat(rs), torch.cat(es), ksys, exact.iters


def train(trainer: fcgno.Trainer, k: torch.Tensor, r: torch.Tensor, e: torch.Tensor, ksys: torch.Tensor,
          epochs: int, seed: int = 0, lr0: float = 1e-3, log=None):
    """Fig. 3 (c): `epochs` passes over the samples in seeded random order.  Returns the mean loss per
    epoch (a host list; one device->host read per epoch)."""
    gen = torch.Generator().manual_seed(seed)
    S = int(r.shape[0])
    curve = []
    for ep in range(epochs):
        perm = torch.randperm(S, generator=gen).to(dtype=torch.int32, device=r.device)
        loss = trainer.epoch(k, r, e, perm, ksys, lr=lr_at_epoch(ep, lr0))
        curve.append(float(loss.mean()))
        if log is not None:
            log(ep, curve[-1])
    return curve


def trained_operator(trainer: fcgno.Trainer, precision: int = fcgno.FP32, device="cuda") -> fcgno.NeuralOperator:
    """Fig. 3 (d): the trained weights as a NeuralOperator for fcgno_fcg_solve."""
    return fcgno.NeuralOperator(trainer.width, np.ascontiguousarray(trainer.blob()), precision=precision,
                                device=device)
