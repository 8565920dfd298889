"""Thin ctypes binding of libfcgno.so (include/fcgno.h).

Argument marshalling only: every step of the hot path runs in the library's CUDA kernels.
PyTorch supplies device memory (tensors) and the current stream.  There is no CPU fallback:
importing this module fails loudly when the shared library is missing, and every call raises
``FcgnoError`` on a non-OK return.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfcgno.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2402_05598_b200.build` "
                      "(or __graft_entry__.build()); there is no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

FP32, FP64 = 0, 1
JACOBI, SGS_RB = 1, 2   # classical preconditioners (fcgno_precond_kind)
FOURIER, CHEBYSHEV = 0, 1  # SNO basis (fcgno_basis)
SCHEDULE_PAPER, SCHEDULE_SLIDING = 0, 1
RUNNING, CONVERGED, MAXIT, BREAKDOWN, NONFINITE = 0, 1, 2, 3, 4
K_MODES = 20
LOSS_NOTAY, LOSS_L2 = 0, 1
ERRORS = {1: "EINVAL", 2: "ENONPOS_K", 3: "ECUDA", 4: "EWORKSPACE", 5: "EUNSUPPORTED"}


class FcgnoError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fcgno {ERRORS.get(code, code)}: {msg}")
        self.code = code


class Grid(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("batch", ctypes.c_int32)]


class NoDesc(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("precision", ctypes.c_int32), ("use_gelu", ctypes.c_int32),
                ("basis", ctypes.c_int32)]


class TrainDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("width", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("loss", ctypes.c_int32)]


class AdamWOpts(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("weight_decay", ctypes.c_double)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int32), ("maxit", ctypes.c_int32), ("tol", ctypes.c_double),
                ("schedule", ctypes.c_int32), ("check_every", ctypes.c_int32),
                ("profile_mask", ctypes.c_int32), ("vec_fp32", ctypes.c_int32)]


_vp, _sz, _i = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
_P = ctypes.POINTER
EXPORTS = {
    "fcgno_problem_workspace_bytes": (_sz, [Grid]),
    "fcgno_assemble": (_i, [Grid, _vp, _vp, _sz, _vp, _P(_vp)]),
    "fcgno_problem_destroy": (None, [_vp]),
    "fcgno_apply_A": (_i, [_vp, _vp, _vp, _vp]),
    "fcgno_dot_workspace_bytes": (_sz, [Grid]),
    "fcgno_batched_dot": (_i, [_vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "fcgno_no_packed_bytes": (_sz, [NoDesc]),
    "fcgno_no_pack": (_i, [NoDesc, _vp, _vp, _vp]),
    "fcgno_no_uses_tensor_cores": (_i, [Grid, NoDesc]),
    "fcgno_apply_no_workspace_bytes": (_sz, [Grid, NoDesc]),
    "fcgno_apply_NO": (_i, [_vp, NoDesc, _vp, _vp, _vp, _vp, _sz, _vp]),
    "fcgno_solve_workspace_bytes": (_sz, [Grid, _P(NoDesc), SolveOpts]),
    "fcgno_fcg_solve": (_i, [_vp, _P(NoDesc), _vp, _vp, _vp, SolveOpts, _vp, _vp, _vp, _vp, _sz, _vp]),
    "fcgno_solve_diag_workspace_bytes": (_sz, [Grid, _P(NoDesc), SolveOpts]),
    "fcgno_fcg_solve_diag": (_i, [_vp, _P(NoDesc), _vp, _vp, _vp, SolveOpts, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                                  _vp]),
    "fcgno_notay_workspace_bytes": (_sz, [Grid, _P(NoDesc)]),
    "fcgno_stationary_workspace_bytes": (_sz, [Grid]),
    "fcgno_apply_stationary": (_i, [_vp, _i, _i, _vp, _vp, _vp, _sz, _vp]),
    "fcgno_solve_stationary_workspace_bytes": (_sz, [Grid, SolveOpts]),
    "fcgno_fcg_solve_stationary": (_i, [_vp, _i, _i, _vp, _vp, SolveOpts, _vp, _vp, _vp, _vp, _sz, _vp]),
    "fcgno_notay_ratio": (_i, [_vp, _P(NoDesc), _vp, _vp, _vp, _i, _vp, _vp, _sz, _vp]),
    "fcgno_solve_host_workspace_bytes": (_sz, [Grid, _P(NoDesc), SolveOpts]),
    "fcgno_solve_host": (_i, [Grid, _vp, _vp, _vp, _P(NoDesc), _vp, SolveOpts, _vp, _vp, _vp, _vp, _sz, _vp]),
    "fcgno_profile_get": (_i, [_i, _P(ctypes.c_double), _P(ctypes.c_int64)]),
    "fcgno_profile_reset": (None, []),
    "fcgno_profile_name": (ctypes.c_char_p, [_i]),
    "fcgno_kernel_launches": (ctypes.c_uint64, []),
    "fcgno_debug_px_trace": (_i, [_vp, _i]),
    "fcgno_train_param_count": (_sz, [ctypes.c_int32]),
    "fcgno_train_workspace_bytes": (_sz, [TrainDesc]),
    "fcgno_train_loss_grad": (_i, [TrainDesc, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "fcgno_adamw_step": (_i, [_sz, _vp, _vp, _vp, _vp, ctypes.c_int32, AdamWOpts, _vp]),
    "fcgno_train_epoch": (_i, [TrainDesc, ctypes.c_int32, _vp, _vp, _vp, _vp, _P(ctypes.c_int32), AdamWOpts, _vp,
                               _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "fcgno_krylov_pair": (_i, [_vp, _vp, _vp, _vp, ctypes.c_double, _vp, _vp, _vp]),
    "fcgno_last_error": (ctypes.c_char_p, []),
    "fcgno_abi_version": (_i, []),
}
for _name, (_res, _args) in EXPORTS.items():
    _fn = getattr(_lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def _check(code: int):
    if code != 0:
        raise FcgnoError(code, _lib.fcgno_last_error().decode())


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return ctypes.c_void_p(t.data_ptr())
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(ctypes.c_void_p)
    raise TypeError(type(t))


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _workspace(nbytes: int, device, stream=None) -> torch.Tensor:
    """Device workspace (torch's caching allocator returns 512-byte aligned blocks).  When the
    library call runs on `stream` rather than torch's current stream, the block is allocated on
    `stream`, so the allocator cannot hand it to other work while the call's kernels still use it."""
    if stream is None:
        return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)
    with torch.cuda.stream(stream):
        return torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=device)


def _on(stream, make):
    """Allocate an output with `make()` on `stream` (see _workspace)."""
    if stream is None:
        return make()
    with torch.cuda.stream(stream):
        return make()


def _require(t: torch.Tensor, shape, name):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError(f"{name} must be a contiguous float64 CUDA tensor")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


def kernel_launches() -> int:
    return int(_lib.fcgno_kernel_launches())


def abi_version() -> int:
    return int(_lib.fcgno_abi_version())


PROF_NCLASS = 10
PROF_NO_LAYER, PROF_NO_MIX, PROF_NO_OUT, PROF_NO_INPUT, PROF_WINDOW, PROF_PFORM, PROF_STENCIL, PROF_UPDATE, \
    PROF_FINALIZE, PROF_NO_YDIR = range(PROF_NCLASS)


def no_uses_tensor_cores(problem: "Problem", no: "NeuralOperator") -> bool:
    """True when the NO's operator layers run on the tcgen05 tensor-core kernels for this grid."""
    return bool(_lib.fcgno_no_uses_tensor_cores(problem.grid, no.desc))


def profile_reset() -> None:
    _lib.fcgno_profile_reset()


def profile_read() -> dict:
    """{class name: (total device ms, timed launches)} accumulated since the last reset."""
    out = {}
    for c in range(PROF_NCLASS):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        _check(_lib.fcgno_profile_get(c, ctypes.byref(ms), ctypes.byref(n)))
        out[_lib.fcgno_profile_name(c).decode()] = (ms.value, n.value)
    return out


class Problem:
    """assemble(k): a batch of B independent n x n systems."""

    def __init__(self, k: torch.Tensor, stream=None):
        if k.dim() != 3 or k.shape[1] != k.shape[2]:
            raise ValueError("k must be [B, n, n]")
        _require(k, k.shape, "k")
        self.B, self.n = int(k.shape[0]), int(k.shape[1])
        self.grid = Grid(self.n, self.B)
        self.k = k
        self.device = k.device
        self._ws = _workspace(_lib.fcgno_problem_workspace_bytes(self.grid), self.device)
        h = ctypes.c_void_p()
        _check(_lib.fcgno_assemble(self.grid, _ptr(k), _ptr(self._ws), self._ws.numel(), _stream(stream),
                                   ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.fcgno_problem_destroy(h)
            except (AttributeError, TypeError):   # interpreter shutdown
                pass
            self._h = None

    @property
    def shape(self):
        return (self.B, self.n, self.n)

    def apply_A(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        _require(x, self.shape, "x")
        y = _on(stream, lambda: torch.empty_like(x)) if out is None else out
        _check(_lib.fcgno_apply_A(self._h, _ptr(x), _ptr(y), _stream(stream)))
        return y

    def dot(self, x: torch.Tensor, y: torch.Tensor, stream=None) -> torch.Tensor:
        _require(x, self.shape, "x")
        _require(y, self.shape, "y")
        out = _on(stream, lambda: torch.empty(self.B, dtype=torch.float64, device=self.device))
        ws = _workspace(_lib.fcgno_dot_workspace_bytes(self.grid), self.device, stream)
        _check(_lib.fcgno_batched_dot(self._h, _ptr(x), _ptr(y), _ptr(out), _ptr(ws), ws.numel(), _stream(stream)))
        return out


class NeuralOperator:
    """Packed SNO weights resident on the device."""

    def __init__(self, width: int, blob: np.ndarray, precision: int = FP32, use_gelu: bool = True,
                 device="cuda", stream=None, basis: int = FOURIER):
        self.desc = NoDesc(int(width), int(precision), int(bool(use_gelu)), int(basis))
        blob = np.ascontiguousarray(blob, dtype=np.float64)
        nbytes = _lib.fcgno_no_packed_bytes(self.desc)
        if nbytes == 0:
            raise ValueError("bad NO descriptor")
        self.packed = _workspace(nbytes, device)
        _check(_lib.fcgno_no_pack(self.desc, _ptr(blob), _ptr(self.packed), _stream(stream)))
        self.width, self.precision = int(width), int(precision)

    def apply(self, problem: Problem, r: torch.Tensor, stream=None) -> torch.Tensor:
        _require(r, problem.shape, "r")
        w = _on(stream, lambda: torch.empty_like(r))
        ws = _workspace(_lib.fcgno_apply_no_workspace_bytes(problem.grid, self.desc), problem.device, stream)
        _check(_lib.fcgno_apply_NO(problem._h, self.desc, _ptr(self.packed), _ptr(r), _ptr(w), _ptr(ws), ws.numel(),
                                   _stream(stream)))
        return w


@dataclass
class SolveResult:
    u: torch.Tensor
    iters: torch.Tensor
    status: torch.Tensor
    history: torch.Tensor | None


class Solver:
    """fcg_solve(k, f, m, tol, maxit): Algorithm 1 over the batch.

    Holds the workspace so repeated solves allocate nothing."""

    def __init__(self, problem: Problem, m: int, tol: float, maxit: int, no: NeuralOperator | None = None,
                 schedule: int = SCHEDULE_PAPER, check_every: int = 16, history: bool = True,
                 profile_mask: int = 0, vec_fp32: bool = False):
        self.problem, self.no = problem, no
        self.opts = SolveOpts(int(m), int(maxit), float(tol), int(schedule), int(check_every), int(profile_mask),
                              int(bool(vec_fp32)))
        self._desc = ctypes.byref(no.desc) if no is not None else None
        nbytes = _lib.fcgno_solve_workspace_bytes(problem.grid, self._desc, self.opts)
        if nbytes == 0:
            raise ValueError("bad solve options")
        dev = problem.device
        self.ws = _workspace(nbytes, dev)
        self.iters = torch.empty(problem.B, dtype=torch.int32, device=dev)
        self.status = torch.empty(problem.B, dtype=torch.int32, device=dev)
        self.history = (torch.full((problem.B, maxit + 1), float("nan"), dtype=torch.float64, device=dev)
                        if history else None)

    def solve(self, f: torch.Tensor, u: torch.Tensor, stream=None) -> SolveResult:
        """u: in = u0, out = final iterate (updated in place)."""
        p = self.problem
        _require(f, p.shape, "f")
        _require(u, p.shape, "u")
        _check(_lib.fcgno_fcg_solve(p._h, self._desc, _ptr(self.no.packed) if self.no else None, _ptr(f), _ptr(u),
                                    self.opts, _ptr(self.iters), _ptr(self.status), _ptr(self.history),
                                    _ptr(self.ws), self.ws.numel(), _stream(stream)))
        return SolveResult(u, self.iters, self.status, self.history)


def fcg_solve(problem: Problem, f: torch.Tensor, u0: torch.Tensor | None = None, *, m: int, tol: float, maxit: int,
              no: NeuralOperator | None = None, schedule: int = SCHEDULE_PAPER, history: bool = True,
              check_every: int = 16, vec_fp32: bool = False) -> SolveResult:
    u = torch.zeros_like(f) if u0 is None else u0.clone()
    return Solver(problem, m, tol, maxit, no, schedule, check_every, history, vec_fp32=vec_fp32).solve(f, u)


class HostSolver:
    """End-to-end entry point with HOST buffers (fcgno_solve_host): H2D copies, assemble, solve
    and D2H copies inside one call."""

    def __init__(self, n: int, batch: int, m: int, tol: float, maxit: int, no: NeuralOperator | None = None,
                 schedule: int = SCHEDULE_PAPER, check_every: int = 16, device="cuda", vec_fp32: bool = False):
        self.grid = Grid(int(n), int(batch))
        self.no = no
        self.opts = SolveOpts(int(m), int(maxit), float(tol), int(schedule), int(check_every), 0, int(bool(vec_fp32)))
        self._desc = ctypes.byref(no.desc) if no is not None else None
        self.ws = _workspace(_lib.fcgno_solve_host_workspace_bytes(self.grid, self._desc, self.opts), device)
        self.n, self.B = int(n), int(batch)

    def solve(self, k: np.ndarray, f: np.ndarray, u: np.ndarray, iters: np.ndarray, status: np.ndarray,
              stream=None):
        for name, a, dt in (("k", k, np.float64), ("f", f, np.float64), ("u", u, np.float64),
                            ("iters", iters, np.int32), ("status", status, np.int32)):
            if not (isinstance(a, np.ndarray) and a.dtype == dt and a.flags.c_contiguous):
                raise TypeError(f"{name} must be a C-contiguous {dt} array")
        _check(_lib.fcgno_solve_host(self.grid, _ptr(k), _ptr(f), _ptr(u), self._desc,
                                     _ptr(self.no.packed) if self.no else None, self.opts, _ptr(iters),
                                     _ptr(status), None, _ptr(self.ws), self.ws.numel(), _stream(stream)))


def notay_ratio(problem: Problem, r: torch.Tensor, e: torch.Tensor, no: NeuralOperator | None = None,
                stream=None, optimal_scale: bool = False) -> torch.Tensor:
    """Theorem-1 / Notay diagnostic (PAPER.md Eq. final_loss):
    eps_b = ||c B(r_b) - e_b||_A / ||e_b||_A with e = A^{-1} r supplied by the caller and c = 1, or the
    minimiser c* (optimal_scale).  fcgno_notay_ratio, computed entirely in the library's kernels."""
    _require(r, problem.shape, "r")
    _require(e, problem.shape, "e")
    desc = ctypes.byref(no.desc) if no is not None else None
    ws = _workspace(_lib.fcgno_notay_workspace_bytes(problem.grid, desc), problem.device, stream)
    eps = _on(stream, lambda: torch.empty(problem.B, dtype=torch.float64, device=problem.device))
    _check(_lib.fcgno_notay_ratio(problem._h, desc, _ptr(no.packed) if no is not None else None, _ptr(r), _ptr(e),
                                  int(bool(optimal_scale)), _ptr(eps), _ptr(ws), ws.numel(), _stream(stream)))
    return eps


def fcg_solve_diag(problem: Problem, f: torch.Tensor, u_star: torch.Tensor, u0: torch.Tensor | None = None, *,
                   m: int, tol: float, maxit: int, no: NeuralOperator | None = None,
                   schedule: int = SCHEDULE_PAPER, check_every: int = 16, vec_fp32: bool = False):
    """fcg_solve with per-iteration Theorem-1 diagnostics (fcgno_fcg_solve_diag): returns
    (SolveResult, eps[B][maxit], err_a[B][maxit]) with eps[b][i] = ||w_i - e_i||_A / ||e_i||_A and
    err_a[b][i] = ||e_i||_A, e_i = u_star - u_i, for i < iters[b] (NaN beyond)."""
    _require(f, problem.shape, "f")
    _require(u_star, problem.shape, "u_star")
    opts = SolveOpts(int(m), int(maxit), float(tol), int(schedule), int(check_every), 0, int(bool(vec_fp32)))
    desc = ctypes.byref(no.desc) if no is not None else None
    nbytes = _lib.fcgno_solve_diag_workspace_bytes(problem.grid, desc, opts)
    if nbytes == 0:
        raise ValueError("bad solve options")
    dev = problem.device
    ws = _workspace(nbytes, dev)
    u = torch.zeros_like(f) if u0 is None else u0.clone()
    iters = torch.empty(problem.B, dtype=torch.int32, device=dev)
    status = torch.empty(problem.B, dtype=torch.int32, device=dev)
    hist = torch.full((problem.B, maxit + 1), float("nan"), dtype=torch.float64, device=dev)
    eps = torch.full((problem.B, max(maxit, 1)), float("nan"), dtype=torch.float64, device=dev)
    err_a = torch.full((problem.B, max(maxit, 1)), float("nan"), dtype=torch.float64, device=dev)
    _check(_lib.fcgno_fcg_solve_diag(problem._h, desc, _ptr(no.packed) if no is not None else None, _ptr(f), _ptr(u),
                                     opts, _ptr(iters), _ptr(status), _ptr(hist), _ptr(u_star), _ptr(eps),
                                     _ptr(err_a), _ptr(ws), ws.numel(), _stream()))
    return SolveResult(u, iters, status, hist), eps, err_a


def apply_stationary(problem: Problem, r: torch.Tensor, kind: int, sweeps: int, stream=None) -> torch.Tensor:
    """w = Jacobi(sweeps) r (kind JACOBI, Eq. 15) or red-black symmetric Gauss-Seidel(sweeps) r (SGS_RB),
    from x^0 = 0 (fcgno_apply_stationary)."""
    _require(r, problem.shape, "r")
    w = _on(stream, lambda: torch.empty_like(r))
    ws = _workspace(_lib.fcgno_stationary_workspace_bytes(problem.grid), problem.device, stream)
    _check(_lib.fcgno_apply_stationary(problem._h, int(kind), int(sweeps), _ptr(r), _ptr(w), _ptr(ws), ws.numel(),
                                       _stream(stream)))
    return w


def fcg_solve_stationary(problem: Problem, f: torch.Tensor, u0: torch.Tensor | None = None, *, kind: int,
                         sweeps: int, m: int, tol: float, maxit: int, schedule: int = SCHEDULE_PAPER,
                         check_every: int = 16, vec_fp32: bool = False) -> SolveResult:
    """Algorithm 1 with the classical preconditioner B = Jacobi(sweeps) / SGS_RB(sweeps)
    (fcgno_fcg_solve_stationary)."""
    _require(f, problem.shape, "f")
    opts = SolveOpts(int(m), int(maxit), float(tol), int(schedule), int(check_every), 0, int(bool(vec_fp32)))
    nbytes = _lib.fcgno_solve_stationary_workspace_bytes(problem.grid, opts)
    if nbytes == 0:
        raise ValueError("bad solve options")
    dev = problem.device
    ws = _workspace(nbytes, dev)
    u = torch.zeros_like(f) if u0 is None else u0.clone()
    iters = torch.empty(problem.B, dtype=torch.int32, device=dev)
    status = torch.empty(problem.B, dtype=torch.int32, device=dev)
    hist = torch.full((problem.B, maxit + 1), float("nan"), dtype=torch.float64, device=dev)
    _check(_lib.fcgno_fcg_solve_stationary(problem._h, int(kind), int(sweeps), _ptr(f), _ptr(u), opts, _ptr(iters),
                                           _ptr(status), _ptr(hist), _ptr(ws), ws.numel(), _stream()))
    return SolveResult(u, iters, status, hist)


# ------------------------------------------------------------------ training
def krylov_pair(problem: Problem, f: torch.Tensor, u_star: torch.Tensor, u: torch.Tensor, e_scale: float = 1.0,
                stream=None):
    """Training pair of every system (Eq. 8-9; fcgno_krylov_pair): r = f - A u,
    e = e_scale (u_star - u)."""
    for name, t in (("f", f), ("u_star", u_star), ("u", u)):
        _require(t, problem.shape, name)
    r = _on(stream, lambda: torch.empty_like(f))
    e = _on(stream, lambda: torch.empty_like(f))
    _check(_lib.fcgno_krylov_pair(problem._h, _ptr(f), _ptr(u_star), _ptr(u), float(e_scale), _ptr(r), _ptr(e),
                                  _stream(stream)))
    return r, e


def train_param_count(width: int) -> int:
    return int(_lib.fcgno_train_param_count(int(width)))


class Trainer:
    """fp32 SNO weights, AdamW state and the training workspace (fcgno_train_*).  The weights use the
    canonical blob order (include/fcgno.h), so `blob()` feeds NeuralOperator directly."""

    def __init__(self, n: int, width: int, batch: int, blob: np.ndarray, loss: int = LOSS_NOTAY, device="cuda",
                 lr: float = 1e-3, weight_decay: float = 1e-2, betas=(0.9, 0.999), eps: float = 1e-8):
        self.desc = TrainDesc(int(n), int(width), int(batch), int(loss))
        nbytes = _lib.fcgno_train_workspace_bytes(self.desc)
        if nbytes == 0:
            raise FcgnoError(1, _lib.fcgno_last_error().decode())
        self.P = train_param_count(width)
        blob = np.ascontiguousarray(blob, dtype=np.float64)
        if blob.size != self.P:
            raise ValueError("weight blob size mismatch")
        self.width, self.n, self.batch = int(width), int(n), int(batch)
        self.params = torch.tensor(blob, dtype=torch.float32, device=device)
        self.grad = torch.zeros_like(self.params)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.t = ctypes.c_int32(0)
        self.opts = AdamWOpts(float(lr), float(betas[0]), float(betas[1]), float(eps), float(weight_decay))
        self.ws = _workspace(nbytes, device)
        self.device = device

    def blob(self) -> np.ndarray:
        """Canonical fp64 blob of the current weights (for NeuralOperator / the oracle)."""
        return self.params.double().cpu().numpy()

    def loss_grad(self, k, r, e, perm=None, ksys=None, count=None, grad=True, stream=None):
        """Per-sample losses [count] (and self.grad = d mean loss / d theta) of samples perm[:count]."""
        count = int(perm.numel() if perm is not None else (count or r.shape[0]))
        loss = _on(stream, lambda: torch.empty(count, dtype=torch.float64, device=self.device))
        _check(_lib.fcgno_train_loss_grad(self.desc, count, _ptr(self.params), _ptr(k), _ptr(r), _ptr(e), _ptr(perm),
                                          _ptr(ksys), _ptr(loss), _ptr(self.grad) if grad else None, _ptr(self.ws),
                                          self.ws.numel(), _stream(stream)))
        return loss

    def adamw_step(self, lr: float | None = None, stream=None):
        if lr is not None:
            self.opts.lr = float(lr)
        self.t.value += 1
        _check(_lib.fcgno_adamw_step(self.P, _ptr(self.params), _ptr(self.grad), _ptr(self.m), _ptr(self.v),
                                     self.t.value, self.opts, _stream(stream)))

    def epoch(self, k, r, e, perm, ksys=None, lr: float | None = None, stream=None) -> torch.Tensor:
        """One pass over the samples in the order perm (int32 device): minibatch loss/grad + AdamW steps.
        Returns the per-sample losses (before each minibatch's step), in perm order."""
        if lr is not None:
            self.opts.lr = float(lr)
        ns = int(perm.numel())
        loss = _on(stream, lambda: torch.empty(ns, dtype=torch.float64, device=self.device))
        _check(_lib.fcgno_train_epoch(self.desc, ns, _ptr(self.params), _ptr(self.grad), _ptr(self.m), _ptr(self.v),
                                      ctypes.byref(self.t), self.opts, _ptr(k), _ptr(r), _ptr(e), _ptr(perm),
                                      _ptr(ksys), _ptr(loss), _ptr(self.ws), self.ws.numel(), _stream(stream)))
        return loss
