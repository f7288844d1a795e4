"""Thin Python binding over libaz (argument marshalling only; every step runs in libaz kernels).

Tensors are torch.float64 CUDA tensors in COLUMN-MAJOR layout: shape (rows, ncols) with
stride (1, ld).  `colmajor(t)` produces that layout; 1-D tensors are one column.
PyTorch provides device memory and streams only.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import check, lib


def colmajor(t: torch.Tensor) -> torch.Tensor:
    if t.dim() == 1:
        return t.contiguous()
    if t.stride(0) == 1 and t.stride(1) >= max(1, t.shape[0]):
        return t
    return t.t().contiguous().t()


def empty_colmajor(rows: int, cols: int, device="cuda") -> torch.Tensor:
    return torch.empty((cols, rows), dtype=torch.float64, device=device).t()


def _mat(t: torch.Tensor):
    """(pointer, ld, ncols) of a column-major float64 CUDA tensor."""
    if t.dtype != torch.float64 or not t.is_cuda:
        raise TypeError("expected a float64 CUDA tensor")
    if t.dim() == 1:
        if t.stride(0) != 1:
            raise ValueError("1-D tensor must be contiguous")
        return t.data_ptr(), max(1, t.shape[0]), 1
    if t.stride(0) != 1:
        raise ValueError("2-D tensor must be column-major (stride(0) == 1); use colmajor()")
    return t.data_ptr(), max(t.stride(1), t.shape[0], 1), t.shape[1]


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _keep(stream, *tensors):
    """Tensors allocated on the current stream but used by libaz work enqueued on another `stream`:
    tell the caching allocator, so their memory is not reused before that work completes."""
    if stream is None or stream == torch.cuda.current_stream():
        return
    for t in tensors:
        if t is not None and t.is_cuda:
            t.record_stream(stream)


class Plan:
    """An AZ plan (az_plan_create): geometry, symbols of B and B^dag, scratch."""

    def __init__(self, *, dim: int, n: int, L: int, T: float, eps: float, op: int = 0,
                 row_scale: float = 1.0, mask: np.ndarray, boundary_xy: Optional[np.ndarray] = None,
                 boundary_weight: float = 0.0, zstar_rcond: float = 1e-10, seed: int = 0, k0sq: float = 0.0,
                 n_y: int = 0, T_y: float = 0.0, boundary_coef: Optional[np.ndarray] = None, stream=None):
        self._mask = np.ascontiguousarray(mask, dtype=np.uint8)
        bxy = np.zeros((0, 2)) if boundary_xy is None else boundary_xy
        self._bxy = np.ascontiguousarray(bxy, dtype=np.float64)
        d = _lib.PlanDesc()
        d.dim, d.n, d.L, d.T, d.eps = dim, n, L, T, eps
        d.op, d.row_scale = op, row_scale
        d.k0sq = k0sq
        d.n_y, d.T_y = n_y, T_y
        self._bcoef = None if boundary_coef is None else np.ascontiguousarray(boundary_coef, dtype=np.float64)
        if self._bcoef is not None and self._bcoef.shape != (self._bxy.shape[0], 4):
            raise ValueError("boundary_coef must be (n_boundary, 4): [a, b, n_x, n_y] per point")
        d.boundary_coef = self._bcoef.ctypes.data if self._bcoef is not None else None
        d.mask = self._mask.ctypes.data
        d.n_boundary = self._bxy.shape[0]
        d.boundary_xy = self._bxy.ctypes.data if self._bxy.shape[0] else None
        d.boundary_weight = boundary_weight
        d.zstar_rcond = zstar_rcond
        d.seed = seed
        h = C.c_void_p()
        check("az_plan_create", lib().az_plan_create(C.byref(d), _stream(stream), C.byref(h)))
        self._h = h
        info = _lib.PlanInfo()
        check("az_plan_query", lib().az_plan_query(h, C.byref(info)))
        self.N, self.M, self.Mb = info.N, info.M, info.Mb
        self.rows = self.M + self.Mb
        self.sigma_max, self.sigma_min_kept = info.sigma_max, info.sigma_min_kept
        self.n_dropped, self.zstar_norm = info.n_dropped, info.zstar_norm
        self.seed = seed

    @classmethod
    def from_config(cls, cfg, stream=None) -> "Plan":
        from . import inputs as I
        return cls(dim=cfg.dim, n=cfg.n, L=cfg.s, T=cfg.T, eps=cfg.eps, op=cfg.row_op,
                   row_scale=cfg.row_scale, mask=I.mask(cfg).reshape(-1),
                   boundary_xy=I.boundary_points(cfg) if cfg.n_boundary else None,
                   boundary_weight=cfg.boundary_weight, zstar_rcond=cfg.tol, seed=cfg.seed,
                   k0sq=getattr(cfg, "k0sq", 0.0), n_y=cfg.n_y if cfg.dim == 2 else 0,
                   T_y=cfg.T_y if cfg.dim == 2 else 0.0, boundary_coef=I.boundary_coefs(cfg), stream=stream)

    def close(self):
        if getattr(self, "_h", None):
            lib().az_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- operators
    def _op(self, name, x, rows_in, rows_out, out=None, stream=None):
        px, ldx, k = _mat(x)
        if x.shape[0] != rows_in:
            raise ValueError(f"{name}: expected {rows_in} rows, got {x.shape[0]}")
        if out is None:
            out = empty_colmajor(rows_out, k, x.device) if x.dim() == 2 else torch.empty(rows_out, dtype=torch.float64, device=x.device)
        py, ldy, _ = _mat(out)
        check(name, getattr(lib(), name)(self._h, C.c_void_p(px), ldx, C.c_void_p(py), ldy, k, _stream(stream)))
        _keep(stream, x, out)
        return out

    def apply_A(self, x, out=None, stream=None):
        return self._op("az_apply_A", x, self.N, self.rows, out, stream)

    def apply_At(self, y, out=None, stream=None):
        return self._op("az_apply_At", y, self.rows, self.N, out, stream)

    def apply_Zstar(self, y, out=None, stream=None):
        return self._op("az_apply_Zstar", y, self.rows, self.N, out, stream)

    def apply_step1(self, v, out=None, stream=None):
        return self._op("az_apply_step1", v, self.N, self.rows, out, stream)

    def apply_resid(self, b, out=None, stream=None):
        return self._op("az_apply_resid", b, self.rows, self.rows, out, stream)

    def sketch(self, col0: int, ncols: int, out=None, stream=None):
        if out is None:
            out = empty_colmajor(self.rows, ncols)
        p, ld, _ = _mat(out)
        check("az_sketch", lib().az_sketch(self._h, col0, ncols, C.c_void_p(p), ld, _stream(stream)))
        _keep(stream, out)
        return out

    def omega_apply(self, col0: int, y, out=None, accumulate=False, stream=None):
        py, ldy, nrhs = _mat(y)
        ncols = y.shape[0]
        if out is None:
            out = empty_colmajor(self.N, nrhs)
        px, ldx, _ = _mat(out)
        check("az_omega_apply", lib().az_omega_apply(self._h, col0, ncols, C.c_void_p(py), ldy, nrhs,
                                                     C.c_void_p(px), ldx, int(accumulate), _stream(stream)))
        _keep(stream, y, out)
        return out

    def step2(self, x2, b, out=None, stream=None):
        """x = x2 + Z* (b - A x2) (az_step2: steps 2-3 of Alg. 1 for a given step-1 solution)."""
        p2, ld2, nrhs = _mat(x2)
        pb, ldb, nb = _mat(b)
        if nb != nrhs or x2.shape[0] != self.N or b.shape[0] != self.rows:
            raise ValueError("az_step2: shapes")
        if out is None:
            out = empty_colmajor(self.N, nrhs, x2.device) if x2.dim() == 2 else torch.empty(self.N, dtype=torch.float64,
                                                                                           device=x2.device)
        px, ldx, _ = _mat(out)
        need = C.c_size_t()
        check("az_step2_workspace_size", lib().az_step2_workspace_size(self._h, nrhs, C.byref(need)))
        ws = torch.empty(max(need.value, 1), dtype=torch.uint8, device=x2.device)
        check("az_step2", lib().az_step2(self._h, C.c_void_p(p2), ld2, C.c_void_p(pb), ldb, C.c_void_p(px), ldx, nrhs,
                                         C.c_void_p(ws.data_ptr()), ws.numel(), _stream(stream)))
        _keep(stream, x2, b, out, ws)
        return out

    # ---------------------------------------------------------------- solve
    def solve_workspace_bytes(self, nrhs: int, R: int, max_blocks: int) -> int:
        b = C.c_size_t()
        check("az_solve_workspace_size", lib().az_solve_workspace_size(self._h, nrhs, R, max_blocks, C.byref(b)))
        return b.value

    def solve(self, b, theta: float, R: int, max_blocks: int = 1, x=None, workspace=None, stream=None):
        pb, ldb, nrhs = _mat(b)
        if x is None:
            x = empty_colmajor(self.N, nrhs) if b.dim() == 2 else torch.empty(self.N, dtype=torch.float64, device=b.device)
        px, ldx, _ = _mat(x)
        need = self.solve_workspace_bytes(nrhs, R, max_blocks)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=b.device)
        rep = _lib.SolveReport()
        st = check("az_solve", lib().az_solve(self._h, C.c_void_p(pb), ldb, C.c_void_p(px), ldx, nrhs, theta, R,
                                              max_blocks, C.c_void_p(workspace.data_ptr()), workspace.numel(),
                                              C.byref(rep), _stream(stream)),
                   allow=(_lib.AZ_OK, _lib.AZ_WARN_SKETCH_SATURATED))
        # az_solve synchronises its stream before returning: the workspace is free to go
        return x, _report(rep, st, workspace)

    def solve_host(self, b, theta: float, R: int, max_blocks: int = 1, x=None, stream=None):
        """End-to-end solve on HOST buffers (host->device copy of b, solve, device->host copy of x
        inside the call).  b, x: numpy arrays or CPU torch tensors in column-major layout; pinned
        torch tensors (pin_memory=True) are copied by DMA directly."""
        if isinstance(b, torch.Tensor):
            nrhs = 1 if b.dim() == 1 else b.shape[1]
            if b.dim() == 2 and b.stride(0) != 1:
                raise ValueError("b must be column-major")
            pb = b.data_ptr()
            if x is None:
                x = torch.empty((nrhs, self.N), dtype=torch.float64, pin_memory=True).t()
            px = x.data_ptr()
        else:
            b = np.asfortranarray(b, dtype=np.float64)
            nrhs = 1 if b.ndim == 1 else b.shape[1]
            if x is None:
                x = np.empty((self.N, nrhs), dtype=np.float64, order="F")
            pb, px = b.ctypes.data, x.ctypes.data
        rep = _lib.SolveReport()
        st = check("az_solve_host", lib().az_solve_host(self._h, C.c_void_p(pb), C.c_void_p(px),
                                                        nrhs, theta, R, max_blocks, C.byref(rep), _stream(stream)),
                   allow=(_lib.AZ_OK, _lib.AZ_WARN_SKETCH_SATURATED))
        return x, _report(rep, st)


class Comm:
    """An NCCL communicator inside libaz (az_comm_create) for az_solve_sharded.  Collective: every
    rank of a torch.distributed process group builds it with `Comm.from_process_group()` (rank 0's
    unique id is broadcast over the group: torch.distributed is the bootstrap plumbing only)."""

    def __init__(self, world: int, rank: int, uid: bytes):
        h = C.c_void_p()
        buf = C.create_string_buffer(bytes(uid), 128)
        check("az_comm_create", lib().az_comm_create(world, rank, buf, C.byref(h)))
        self._h = h
        self.world, self.rank = world, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check("az_comm_unique_id", lib().az_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        t = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            t = torch.frombuffer(bytearray(cls.unique_id()), dtype=torch.uint8).clone()
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0, group=group)
        return cls(world, rank, bytes(t.cpu().numpy().tobytes()))

    def close(self):
        if getattr(self, "_h", None):
            lib().az_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_sharded(plan: "Plan", comm: Comm, b, theta: float, R: int, max_blocks: int = 1, x=None, stream=None):
    """az_solve_sharded: the multi-GPU AZ solve inside libaz (NCCL), collective over `comm`;
    b replicated on every rank, x returned replicated."""
    pb, ldb, nrhs = _mat(b)
    if x is None:
        x = empty_colmajor(plan.N, nrhs, b.device) if b.dim() == 2 else torch.empty(plan.N, dtype=torch.float64,
                                                                                   device=b.device)
    px, ldx, _ = _mat(x)
    rep = _lib.SolveReport()
    st = check("az_solve_sharded", lib().az_solve_sharded(plan._h, comm._h, C.c_void_p(pb), ldb, C.c_void_p(px), ldx,
                                                          nrhs, theta, R, max_blocks, C.byref(rep), _stream(stream)),
               allow=(_lib.AZ_OK, _lib.AZ_WARN_SKETCH_SATURATED))
    return x, _report(rep, st)


class Factor:
    """A factored step-1 sketch (az_factorize): solve for new right-hand sides without redrawing,
    re-factoring or re-decomposing the sketch."""

    def __init__(self, plan: "Plan", theta: float, R: int, max_blocks: int = 1, stream=None):
        self.plan = plan
        h = C.c_void_p()
        rep = _lib.SolveReport()
        st = check("az_factorize", lib().az_factorize(plan._h, theta, R, max_blocks, C.byref(h), C.byref(rep),
                                                       _stream(stream)),
                   allow=(_lib.AZ_OK, _lib.AZ_WARN_SKETCH_SATURATED))
        self._h = h
        self.report = _report(rep, st)

    def close(self):
        if getattr(self, "_h", None):
            lib().az_factor_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def workspace_bytes(self, nrhs: int) -> int:
        b = C.c_size_t()
        check("az_factor_workspace_size", lib().az_factor_workspace_size(self._h, nrhs, C.byref(b)))
        return b.value

    def solve(self, b, x=None, workspace=None, stream=None):
        pb, ldb, nrhs = _mat(b)
        if x is None:
            x = empty_colmajor(self.plan.N, nrhs) if b.dim() == 2 else torch.empty(self.plan.N, dtype=torch.float64,
                                                                                  device=b.device)
        px, ldx, _ = _mat(x)
        need = self.workspace_bytes(nrhs)
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=b.device)
        rep = _lib.SolveReport()
        st = check("az_solve_factored", lib().az_solve_factored(self._h, C.c_void_p(pb), ldb, C.c_void_p(px), ldx, nrhs,
                                                                C.c_void_p(workspace.data_ptr()), workspace.numel(),
                                                                C.byref(rep), _stream(stream)))
        return x, _report(rep, st)


def _host_ptr(t, what):
    if not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{what}: expected a float64 CPU (pinned) tensor")
    if t.dim() == 2 and t.stride(0) != 1:
        raise ValueError(f"{what}: must be column-major")
    return t.data_ptr()


def solve_host_pipelined(plan: "Plan", b, x, theta: float, R: int, max_blocks: int = 1, stream=None):
    """az_solve_host_pipelined: enqueue upload of b (pinned host), solve, download into x (pinned
    host) and return; call plan_sync(plan) before reading x."""
    nrhs = 1 if b.dim() == 1 else b.shape[1]
    check("az_solve_host_pipelined", lib().az_solve_host_pipelined(
        plan._h, C.c_void_p(_host_ptr(b, "b")), C.c_void_p(_host_ptr(x, "x")), nrhs, theta, R, max_blocks,
        _stream(stream)), allow=(_lib.AZ_OK, _lib.AZ_WARN_SKETCH_SATURATED))
    return x


def plan_sync(plan: "Plan") -> str:
    """az_plan_sync: wait for the plan's pipelined solves; returns "AZ_OK" or "AZ_WARN_SKETCH_SATURATED"
    (some single-block pipelined solve since the last sync saturated its sketch)."""
    st = check("az_plan_sync", lib().az_plan_sync(plan._h), allow=(_lib.AZ_OK, _lib.AZ_WARN_SKETCH_SATURATED))
    return _lib.STATUS.get(st, st)


def _report(rep, status, workspace=None):
    out = {"rank": rep.rank_used, "probes": rep.probes_used, "saturated": bool(rep.saturated),
           "sigma_first": rep.sigma_first, "sigma_last_kept": rep.sigma_last_kept,
           "ms_rhs": rep.ms_rhs, "ms_sketch": rep.ms_sketch, "ms_qr": rep.ms_qr, "ms_svd": rep.ms_svd,
           "ms_step2": rep.ms_step2, "ms_total": rep.ms_total, "status": _lib.STATUS.get(status, status)}
    if workspace is not None and rep.sigma and rep.n_sigma > 0:
        # the sketch's singular values live in the caller's workspace: copy them out
        off = rep.sigma - workspace.data_ptr()
        if 0 <= off and off + 8 * rep.n_sigma <= workspace.numel():
            out["sigma"] = workspace[off:off + 8 * rep.n_sigma].view(torch.float64).clone()
    return out


def qr_r(A: torch.Tensor, stream=None) -> torch.Tensor:
    """R factor (k x k) of a tall column-major matrix A (m x k); A is overwritten."""
    pa, lda, k = _mat(A)
    m = A.shape[0]
    ws = C.c_size_t()
    check("az_qr_workspace_size", lib().az_qr_workspace_size(m, k, C.byref(ws)))
    w = torch.empty(max(ws.value, 1), dtype=torch.uint8, device=A.device)
    R = empty_colmajor(k, k, A.device)
    pr, ldr, _ = _mat(R)
    check("az_qr_r", lib().az_qr_r(None, C.c_void_p(pa), m, k, lda, C.c_void_p(pr), ldr,
                                   C.c_void_p(w.data_ptr()), w.numel(), _stream(stream)))
    _keep(stream, A, w, R)
    return R


def qr_r_partial(A: torch.Tensor, k1: int, stream=None) -> torch.Tensor:
    """[R_11 | (Q^T A[:, k1:])[:k1]] (k1 x k) of a tall column-major A (m x k, k <= 128);
    A is overwritten."""
    pa, lda, k = _mat(A)
    m = A.shape[0]
    ws = C.c_size_t()
    check("az_qr_workspace_size", lib().az_qr_workspace_size(m, k, C.byref(ws)))
    w = torch.empty(max(ws.value, 1), dtype=torch.uint8, device=A.device)
    R = empty_colmajor(k1, k, A.device)
    pr, ldr, _ = _mat(R)
    check("az_qr_r_partial", lib().az_qr_r_partial(None, C.c_void_p(pa), m, k, k1, lda, C.c_void_p(pr), ldr,
                                                   C.c_void_p(w.data_ptr()), w.numel(), _stream(stream)))
    _keep(stream, A, w, R)
    return R


def tsvd_solve(Rf: torch.Tensor, r: int, nrhs: int, theta: float, stream=None):
    """y = V_k Sigma_k^-1 U_k^T c from Rf = [R_S | c] (r x (r + nrhs)); returns (y, sigma, k)."""
    pr, ldr, _ = _mat(Rf)
    ws = C.c_size_t()
    check("az_tsvd_workspace_size", lib().az_tsvd_workspace_size(r, nrhs, C.byref(ws)))
    w = torch.empty(max(ws.value, 1), dtype=torch.uint8, device=Rf.device)
    y = empty_colmajor(r, nrhs, Rf.device)
    sig = torch.empty(r, dtype=torch.float64, device=Rf.device)
    py, ldy, _ = _mat(y)
    k = C.c_int64()
    check("az_tsvd_solve", lib().az_tsvd_solve(C.c_void_p(pr), ldr, r, nrhs, theta, C.c_void_p(py), ldy,
                                               C.c_void_p(sig.data_ptr()), C.byref(k),
                                               C.c_void_p(w.data_ptr()), w.numel(), _stream(stream)))
    _keep(stream, Rf, w, y, sig)
    return y, sig, k.value


def launch_count(reset: bool = False) -> int:
    return lib().az_launch_count(int(reset))


def trace_enable(on: bool = True) -> None:
    """Bracket every libaz launch with CUDA events on its stream (measurement only)."""
    lib().az_trace_enable(int(on))


def trace_report() -> dict:
    """{kernel name: (launches, total ms, units)} since trace_enable (synchronises the events)."""
    n = lib().az_trace_report(None, 0)
    buf = C.create_string_buffer(n + 1)
    lib().az_trace_report(buf, n + 1)
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms, units = line.split()
        out[name] = (int(cnt), float(ms), int(units))
    return out
