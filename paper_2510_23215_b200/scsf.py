"""Thin ctypes binding of libscsf.so (include/scsf.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module
allocates device memory with torch, passes raw pointers and the current CUDA
stream, and converts status codes to exceptions.  There is no CPU fallback:
if the shared library is missing, or no CUDA device is present, the calls
raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SCSF_LIB: another in-tree build of the same library (A/B measurements of a kernel variant)
LIB_PATH = os.environ.get("SCSF_LIB") or os.path.join(_HERE, "lib", "libscsf.so")

SCSF_OK, SCSF_ERR_ARG, SCSF_ERR_NUMERICAL, SCSF_ERR_DEVICE, SCSF_ERR_NOT_IMPLEMENTED, SCSF_ERR_WORKSPACE = range(6)
_STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_NUMERICAL", 3: "ERR_DEVICE", 4: "ERR_NOT_IMPLEMENTED", 5: "ERR_WORKSPACE"}

EXPORTED = [
    "scsf_sort_workspace_bytes", "scsf_sort", "scsf_signatures", "scsf_assemble",
    "scsf_filter_workspace_bytes", "scsf_cheb_filter", "scsf_solve_workspace_bytes",
    "scsf_solve_one", "scsf_solve_queue", "scsf_last_error", "scsf_abi_version",
    "scsf_launch_count", "scsf_set_timing", "scsf_solve_chains",
    "scsf_dev_workspace_bytes", "scsf_gemm_tn", "scsf_gemm_nn", "scsf_chol_inv", "scsf_syev_small",
    "scsf_comm_unique_id", "scsf_comm_create", "scsf_comm_create_loopback", "scsf_comm_destroy",
    "scsf_comm_rank", "scsf_slab_rows", "scsf_solve_dist_workspace_bytes", "scsf_solve_queue_dist",
    "scsf_filter_kind", "scsf_solve_chains_host_workspace_bytes", "scsf_solve_chains_host",
    "scsf_chain_state_doubles", "scsf_solve_chains_resume", "scsf_grf_workspace_bytes", "scsf_grf_fields",
    "scsf_assemble_vibration",
]


ABI_VERSION = 2                         # include/scsf.h SCSF_ABI_VERSION


class ScsfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"scsf {_STATUS.get(code, code)}: {msg}")
        self.code = code


class NotConverged(ScsfError):
    pass


class scsf_ops(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("nz", ctypes.c_int32), ("n_ops", ctypes.c_int32), ("stencil", ctypes.c_int32),
                ("ld", ctypes.c_int64), ("coef", ctypes.c_void_p)]


class scsf_stats(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("filter_steps", ctypes.c_int32), ("cholqr_fallbacks", ctypes.c_int32),
                ("n_locked", ctypes.c_int32), ("warm", ctypes.c_int32),
                ("spmm_columns", ctypes.c_int64), ("max_rel_resid", ctypes.c_double),
                ("beta", ctypes.c_double), ("t_filter_ms", ctypes.c_double), ("t_ortho_ms", ctypes.c_double),
                ("t_rr_ms", ctypes.c_double), ("filter_bytes", ctypes.c_double),
                ("jacobi_sweeps", ctypes.c_int32), ("cold_retry", ctypes.c_int32),
                ("t_gemm_ms", ctypes.c_double), ("gemm_flops", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libscsf.so; raise loudly if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libscsf.so not found at {path}: run `python -m paper_2510_23215_b200.build`")
    lib = ctypes.CDLL(path)
    P, I32, I64, D, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
    OPS = ctypes.POINTER(scsf_ops)
    ST = ctypes.POINTER(scsf_stats)
    sig = {
        "scsf_sort_workspace_bytes": (SZ, [I32, I32, I32, I32, I32]),
        "scsf_sort": (ctypes.c_int, [P, I32, I32, I32, I32, I32, I32, P, P, P, P, SZ, P]),
        "scsf_signatures": (ctypes.c_int, [P, I32, I32, I32, I32, I32, P, P, SZ, P]),
        "scsf_assemble": (ctypes.c_int, [OPS, D, P, P, P, P, P, P]),
        "scsf_filter_workspace_bytes": (SZ, [OPS, I32, I64]),
        "scsf_cheb_filter": (ctypes.c_int, [OPS, I32, P, I64, I32, I32, D, D, D, P, P, SZ, P]),
        "scsf_solve_workspace_bytes": (SZ, [OPS, I32, I32]),
        "scsf_solve_one": (ctypes.c_int, [OPS, I32, I32, I32, I32, D, I32, P, ctypes.c_uint64, P, P, I64, ST,
                                          P, SZ, P]),
        "scsf_solve_queue": (ctypes.c_int, [OPS, P, I32, I32, I32, I32, D, I32, ctypes.c_uint64, P, P, I64, ST,
                                            P, SZ, P]),
        "scsf_last_error": (ctypes.c_char_p, []),
        "scsf_abi_version": (ctypes.c_int, []),
        "scsf_launch_count": (ctypes.c_int64, []),
        "scsf_set_timing": (ctypes.c_int, [I32]),
        "scsf_solve_chains": (ctypes.c_int, [OPS, P, P, I32, I32, I32, I32, D, I32, ctypes.c_uint64, P, P, I64,
                                             ST, P, SZ, P]),
        "scsf_dev_workspace_bytes": (SZ, [I64, I32, I32]),
        "scsf_gemm_tn": (ctypes.c_int, [P, I64, I32, P, I64, I32, I64, D, I32, P, I64, P, SZ, P]),
        "scsf_gemm_nn": (ctypes.c_int, [P, I64, I64, I32, P, I64, I32, D, D, P, I64, P]),
        "scsf_chol_inv": (ctypes.c_int, [P, I64, I32, I64, P, P, SZ, P]),
        "scsf_syev_small": (ctypes.c_int, [P, I64, I32, P, P, P, P, SZ, P]),
        "scsf_filter_kind": (ctypes.c_int, [OPS]),
        "scsf_solve_chains_host_workspace_bytes": (SZ, [OPS, I32, I32]),
        "scsf_solve_chains_host": (ctypes.c_int, [OPS, P, P, I32, I32, I32, I32, D, I32, ctypes.c_uint64, P, P, I64,
                                                  ST, P, SZ, P]),
        "scsf_chain_state_doubles": (I64, [OPS, I32, I32]),
        "scsf_grf_workspace_bytes": (SZ, [I32, I32]),
        "scsf_assemble_vibration": (ctypes.c_int, [OPS, D, P, P, I64, P, P]),
        "scsf_grf_fields": (ctypes.c_int, [I32, I32, I32, D, D, D, I32, I32, P, P, P, P, P, P, P, SZ, P]),
        "scsf_solve_chains_resume": (ctypes.c_int, [OPS, P, P, I32, I32, I32, I32, D, I32, ctypes.c_uint64, P, P,
                                                    P, P, I64, ST, P, SZ, P]),
        "scsf_comm_unique_id": (ctypes.c_int, [P]),
        "scsf_comm_create": (ctypes.c_int, [I32, I32, P, ctypes.POINTER(P)]),
        "scsf_comm_create_loopback": (ctypes.c_int, [I32, P]),
        "scsf_comm_destroy": (ctypes.c_int, [P]),
        "scsf_comm_rank": (ctypes.c_int, [P, ctypes.POINTER(I32), ctypes.POINTER(I32)]),
        "scsf_slab_rows": (None, [I32, I32, I32, ctypes.POINTER(I32), ctypes.POINTER(I32)]),
        "scsf_solve_dist_workspace_bytes": (SZ, [OPS, I32, I32, I32, I32, I32]),
        "scsf_solve_queue_dist": (ctypes.c_int, [OPS, I32, I32, P, I32, I32, I32, I32, D, I32, ctypes.c_uint64, P,
                                                 P, I64, ST, P, P, SZ, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.scsf_abi_version() != ABI_VERSION:       # the ctypes structs below must match include/scsf.h
        raise ImportError(f"libscsf.so ABI {lib.scsf_abi_version()} != binding ABI {ABI_VERSION}: rebuild")
    _lib = lib
    return lib


def _check(code: int):
    if code == SCSF_OK:
        return
    msg = load_library().scsf_last_error().decode(errors="replace")
    if code == SCSF_ERR_NUMERICAL:
        raise NotConverged(code, msg)
    raise ScsfError(code, msg)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _require_cuda_f64(t: torch.Tensor, name: str):
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def launch_count() -> int:
    return int(load_library().scsf_launch_count())


FILTER_KERNELS = {3: "k_filter_rp (cluster-resident whole filter, register patches, Alg. 1)",
                  2: "k_filter_cl (cluster-resident whole filter, Alg. 1)",
                  1: "k_filter_res2d (single-CTA resident whole filter, Alg. 1)",
                  0: "k_stencil_v4 (one streaming launch per filter step, Alg. 1)"}


def filter_kind(ops: "Operators") -> int:
    st = ops.c_struct()
    return int(load_library().scsf_filter_kind(ctypes.byref(st)))


def set_timing(on: bool) -> bool:
    """Enable the library's per-phase CUDA-event timers (stats t_*_ms); returns the old state."""
    return bool(load_library().scsf_set_timing(1 if on else 0))


def ld_for(n: int) -> int:
    return (n + 31) // 32 * 32


# ------------------------------------------------------------------ operators ----
STENCIL_FLUX, STENCIL_VIB13 = 0, 1


@dataclass
class Operators:
    """A device batch of symmetric DIA stencils (include/scsf.h `scsf_ops`)."""
    dim: int
    nx: int
    ny: int
    nz: int
    n_ops: int
    ld: int
    coef: torch.Tensor          # [n_ops, ncoef, ld] float64 on the device (ncoef = 1+dim, or 7 for VIB13)
    stencil: int = 0            # STENCIL_FLUX or STENCIL_VIB13 (include/scsf.h)

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz

    def c_struct(self) -> scsf_ops:
        return scsf_ops(self.dim, self.nx, self.ny, self.nz, self.n_ops, self.stencil, self.ld,
                        self.coef.data_ptr())


def assemble(dim: int, nx: int, h: float, faces, c: torch.Tensor | None) -> Operators:
    """Flux-form FD assembly on the device (scsf_assemble).  faces: list of dim tensors."""
    lib = load_library()
    for i, f in enumerate(faces):
        _require_cuda_f64(f, f"faces[{i}]")
    n_ops = faces[0].shape[0]
    n = nx ** dim
    ld = ld_for(n)
    nz = nx if dim == 3 else 1
    coef = torch.empty((n_ops, 1 + dim, ld), dtype=torch.float64, device=faces[0].device)
    ops = Operators(dim, nx, nx, nz, n_ops, ld, coef)
    st = ops.c_struct()
    if c is not None:
        _require_cuda_f64(c, "c")
    fz = faces[2] if dim == 3 else None
    _check(lib.scsf_assemble(ctypes.byref(st), h, _ptr(faces[0]), _ptr(faces[1]), _ptr(fz), _ptr(c),
                             _ptr(coef), _stream()))
    return ops


GRF_FAMILIES = {"diva": 0, "lapv": 1, "divac": 2, "vib": 3}


def grf_fields(dim: int, nx: int, K: int, s: float, sigma: float | None, vscale: float, family: str,
               xi: torch.Tensor):
    """Coefficient arrays of a batch from its normal draws, on the device (scsf_grf_fields).
    xi: cuda float64 [N, F, K^dim].  Returns (faces list, c [N, n], params [N, F, n])."""
    lib = load_library()
    _require_cuda_f64(xi, "xi")
    fam = GRF_FAMILIES[family]
    F = 2 if fam >= 2 else 1
    N = xi.shape[0]
    if xi.shape[1:] != (F, K ** dim):
        raise ValueError(f"xi must be [N, {F}, {K ** dim}]")
    n = nx ** dim
    dev = xi.device
    faces = []
    for ax in range(dim if fam != 3 else 0):              # vib: nodal D, rho only
        shp = [nx] * dim
        shp[dim - 1 - ax] = nx + 1
        faces.append(torch.empty((N, *shp), dtype=torch.float64, device=dev))
    c = torch.empty((N, n), dtype=torch.float64, device=dev) if fam != 3 else None
    params = torch.empty((N, F, n), dtype=torch.float64, device=dev)
    ws = _workspace(lib.scsf_grf_workspace_bytes(nx, K), dev)
    fp = [_ptr(faces[ax]) if ax < len(faces) else None for ax in range(3)]
    _check(lib.scsf_grf_fields(dim, nx, K, s, -1.0 if sigma is None else sigma, vscale, fam, N, _ptr(xi),
                               fp[0], fp[1], fp[2], _ptr(c),
                               _ptr(params), _ptr(ws), ws.numel(), _stream()))
    return faces, c, params


def assemble_vibration(nx: int, h: float, params: torch.Tensor) -> Operators:
    """Thin-plate vibration operators B = rho^-1/2 Lh D Lh rho^-1/2 on the device
    (scsf_assemble_vibration).  params: cuda float64 [N, 2, n] with D = params[:, 0], rho = params[:, 1]."""
    lib = load_library()
    _require_cuda_f64(params, "params")
    n = nx * nx
    if params.dim() != 3 or params.shape[1] != 2 or params.shape[2] != n:
        raise ValueError(f"params must be [N, 2, {n}]")
    n_ops = params.shape[0]
    ld = ld_for(n)
    coef = torch.empty((n_ops, 7, ld), dtype=torch.float64, device=params.device)
    ops = Operators(2, nx, nx, 1, n_ops, ld, coef, STENCIL_VIB13)
    st = ops.c_struct()
    D = params[:, 0]
    rho = params[:, 1]
    _check(lib.scsf_assemble_vibration(ctypes.byref(st), h, ctypes.c_void_p(D.data_ptr()),
                                       ctypes.c_void_p(rho.data_ptr()), 2 * n, _ptr(coef), _stream()))
    return ops


# ----------------------------------------------------------------------- sort ----
def signatures(params: torch.Tensor, dim: int, p: int, p0: int) -> torch.Tensor:
    """Alg. 2 ll. 3-5: truncated DFT signatures, complex128 [N, F*p0^dim]."""
    lib = load_library()
    _require_cuda_f64(params, "params")
    N, F = params.shape[0], params.shape[1]
    ws = _workspace(lib.scsf_sort_workspace_bytes(N, dim, p, F, p0), params.device)
    sig = torch.empty((N, F * p0 ** dim, 2), dtype=torch.float64, device=params.device)
    _check(lib.scsf_signatures(_ptr(params), N, dim, p, F, p0, _ptr(sig), _ptr(ws), ws.numel(), _stream()))
    return torch.view_as_complex(sig)


def sort(params: torch.Tensor, dim: int, p: int, p0: int, start: int = 0):
    """Alg. 2: returns (perm int32[N], d2_best[N-1], d2_second[N-1]) as numpy arrays."""
    lib = load_library()
    _require_cuda_f64(params, "params")
    N, F = params.shape[0], params.shape[1]
    ws = _workspace(lib.scsf_sort_workspace_bytes(N, dim, p, F, p0), params.device)
    perm = np.empty(N, dtype=np.int32)
    best = np.empty(max(N - 1, 1), dtype=np.float64)
    second = np.empty(max(N - 1, 1), dtype=np.float64)
    _check(lib.scsf_sort(_ptr(params), N, dim, p, F, p0, start, perm.ctypes.data_as(ctypes.c_void_p),
                         best.ctypes.data_as(ctypes.c_void_p), second.ctypes.data_as(ctypes.c_void_p),
                         _ptr(ws), ws.numel(), _stream()))
    return perm, best[:N - 1], second[:N - 1]


# --------------------------------------------------------------------- filter ----
def cheb_filter(ops: Operators, op_index: int, Y0: torch.Tensor, degree: int, lam: float, c: float,
                e: float) -> torch.Tensor:
    """Alg. 1 on a block Y0 [k, ldy] (column-major n x k); returns Y_m of the same shape."""
    lib = load_library()
    _require_cuda_f64(Y0, "Y0")
    k, ldy = Y0.shape
    st = ops.c_struct()
    ws = _workspace(lib.scsf_filter_workspace_bytes(ctypes.byref(st), k, ldy), Y0.device)
    Ym = torch.empty_like(Y0)
    _check(lib.scsf_cheb_filter(ctypes.byref(st), op_index, _ptr(Y0), ldy, k, degree, lam, c, e, _ptr(Ym),
                                _ptr(ws), ws.numel(), _stream()))
    return Ym


# ---------------------------------------------------------------------- solve ----
def solve_workspace(ops: Operators, L: int, nex: int) -> torch.Tensor:
    lib = load_library()
    st = ops.c_struct()
    return _workspace(lib.scsf_solve_workspace_bytes(ctypes.byref(st), L, nex), ops.coef.device)


def solve_one(ops: Operators, op_index: int, L: int, nex: int, degree: int = 20, tol: float = 1e-8,
              max_iter: int = 200, warm: torch.Tensor | None = None, seed: int = 0, raise_on_fail=True,
              ws: torch.Tensor | None = None):
    """Alg. 3 on one operator.  Returns (evals[b], evecs[b, ld], stats dict)."""
    lib = load_library()
    b = L + nex
    st = ops.c_struct()
    if ws is None:
        ws = solve_workspace(ops, L, nex)
    evals = torch.empty(b, dtype=torch.float64, device=ops.coef.device)
    evecs = torch.empty((b, ops.ld), dtype=torch.float64, device=ops.coef.device)
    if warm is not None:
        _require_cuda_f64(warm, "warm")
        assert warm.shape == (b, ops.ld)
    stats = scsf_stats()
    code = lib.scsf_solve_one(ctypes.byref(st), op_index, L, nex, degree, tol, max_iter, _ptr(warm),
                              ctypes.c_uint64(seed), _ptr(evals), _ptr(evecs), ops.ld, ctypes.byref(stats),
                              _ptr(ws), ws.numel(), _stream())
    if raise_on_fail or code != SCSF_ERR_NUMERICAL:
        _check(code)
    return evals, evecs, stats.as_dict()


def solve_queue(ops: Operators, chain, L: int, nex: int, degree: int = 20, tol: float = 1e-8,
                max_iter: int = 200, seed: int = 0, want_vecs: bool = True, raise_on_fail=True,
                ws: torch.Tensor | None = None, evals: torch.Tensor | None = None,
                evecs: torch.Tensor | None = None):
    """SCSF chain solve.  Returns (evals[n_chain, L], evecs[n_chain, L, ld] or None, stats list)."""
    lib = load_library()
    chain = np.ascontiguousarray(np.asarray(chain, dtype=np.int32))
    nc = int(chain.shape[0])
    st = ops.c_struct()
    if ws is None:
        ws = solve_workspace(ops, L, nex)
    dev = ops.coef.device
    if evals is None:
        evals = torch.empty((nc, L), dtype=torch.float64, device=dev)
    if want_vecs and evecs is None:
        evecs = torch.empty((nc, L, ops.ld), dtype=torch.float64, device=dev)
    stats = (scsf_stats * max(nc, 1))()
    code = lib.scsf_solve_queue(ctypes.byref(st), chain.ctypes.data_as(ctypes.c_void_p), nc, L, nex, degree,
                                tol, max_iter, ctypes.c_uint64(seed), _ptr(evals),
                                _ptr(evecs) if want_vecs else None, ops.ld, stats, _ptr(ws), ws.numel(),
                                _stream())
    if raise_on_fail or code != SCSF_ERR_NUMERICAL:
        _check(code)
    return evals, (evecs if want_vecs else None), [stats[i].as_dict() for i in range(nc)]


def split_chains(length: int, n_chains: int) -> np.ndarray:
    """chain_start offsets of n_chains contiguous, near-equal slices of a queue."""
    n_chains = max(1, min(n_chains, max(length, 1)))
    return np.array([(c * length) // n_chains for c in range(n_chains + 1)], dtype=np.int32)


def solve_chains(ops: Operators, queue, n_chains: int, L: int, nex: int, degree: int = 20, tol: float = 1e-8,
                 max_iter: int = 200, seed: int = 0, want_vecs: bool = True, raise_on_fail=True,
                 ws: torch.Tensor | None = None, evals: torch.Tensor | None = None,
                 evecs: torch.Tensor | None = None, chain_start=None):
    """Concurrent warm-start chains over contiguous slices of `queue` (scsf_solve_chains).

    Returns (evals[len, L], evecs[len, L, ld] or None, stats list) by queue position.
    """
    lib = load_library()
    queue = np.ascontiguousarray(np.asarray(queue, dtype=np.int32))
    nq = int(queue.shape[0])
    starts = split_chains(nq, n_chains) if chain_start is None else np.ascontiguousarray(chain_start, dtype=np.int32)
    nc = len(starts) - 1
    st = ops.c_struct()
    per = lib.scsf_solve_workspace_bytes(ctypes.byref(st), L, nex)
    if ws is None:
        ws = _workspace(per * nc, ops.coef.device)
    dev = ops.coef.device
    if evals is None:
        evals = torch.empty((nq, L), dtype=torch.float64, device=dev)
    if want_vecs and evecs is None:
        evecs = torch.empty((nq, L, ops.ld), dtype=torch.float64, device=dev)
    stats = (scsf_stats * max(nq, 1))()
    code = lib.scsf_solve_chains(ctypes.byref(st), queue.ctypes.data_as(ctypes.c_void_p),
                                 starts.ctypes.data_as(ctypes.c_void_p), nc, L, nex, degree, tol, max_iter,
                                 ctypes.c_uint64(seed), _ptr(evals), _ptr(evecs) if want_vecs else None, ops.ld,
                                 stats, _ptr(ws), ws.numel(), _stream())
    if raise_on_fail or code != SCSF_ERR_NUMERICAL:
        _check(code)
    return evals, (evecs if want_vecs else None), [stats[i].as_dict() for i in range(nq)]


def chains_host_workspace_bytes(ops: Operators, L: int, nex: int) -> int:
    """Per-chain workspace of scsf_solve_chains_host (bytes)."""
    st = ops.c_struct()
    return int(load_library().scsf_solve_chains_host_workspace_bytes(ctypes.byref(st), L, nex))


def solve_chains_host(ops: Operators, queue, n_chains: int, L: int, nex: int, evals_host: torch.Tensor,
                      evecs_host: torch.Tensor | None, degree: int = 20, tol: float = 1e-8, max_iter: int = 200,
                      seed: int = 0, raise_on_fail=True, ws: torch.Tensor | None = None):
    """Concurrent chains with the pairs streamed into pinned host tensors while the chains run
    (scsf_solve_chains_host).  evals_host [len, L], evecs_host [len, L, ld_host] (both pinned CPU
    float64) or None.  Returns the stats list (by queue position)."""
    lib = load_library()
    queue = np.ascontiguousarray(np.asarray(queue, dtype=np.int32))
    nq = int(queue.shape[0])
    starts = split_chains(nq, n_chains)
    nc = len(starts) - 1
    for t, nm in ((evals_host, "evals_host"), (evecs_host, "evecs_host")):
        if t is not None and not (t.is_pinned() and t.dtype == torch.float64 and t.is_contiguous()):
            raise ValueError(f"{nm} must be a pinned contiguous float64 CPU tensor")
    st = ops.c_struct()
    per = lib.scsf_solve_chains_host_workspace_bytes(ctypes.byref(st), L, nex)
    if ws is None or ws.numel() < per * nc:
        ws = _workspace(per * nc, ops.coef.device)
    stats = (scsf_stats * max(nq, 1))()
    ld_host = evecs_host.shape[2] if evecs_host is not None else 0
    code = lib.scsf_solve_chains_host(ctypes.byref(st), queue.ctypes.data_as(ctypes.c_void_p),
                                      starts.ctypes.data_as(ctypes.c_void_p), nc, L, nex, degree, tol, max_iter,
                                      ctypes.c_uint64(seed), ctypes.c_void_p(evals_host.data_ptr()),
                                      ctypes.c_void_p(evecs_host.data_ptr()) if evecs_host is not None else None,
                                      ld_host, stats, _ptr(ws), ws.numel(), _stream())
    if raise_on_fail or code != SCSF_ERR_NUMERICAL:
        _check(code)
    return [stats[i].as_dict() for i in range(nq)]


def chain_state_doubles(ops: Operators, L: int, nex: int) -> int:
    """Length of one chain's resume state: b * (n + 1) doubles (scsf_chain_state_doubles)."""
    st = ops.c_struct()
    return int(load_library().scsf_chain_state_doubles(ctypes.byref(st), L, nex))


def solve_chains_resume(ops: Operators, queue, chain_start, L: int, nex: int, state_in: torch.Tensor | None,
                        state_out: torch.Tensor, degree: int = 20, tol: float = 1e-8, max_iter: int = 200,
                        seed: int = 0, want_vecs: bool = False, raise_on_fail=True, ws: torch.Tensor | None = None):
    """scsf_solve_chains_resume: chains over queue[chain_start[c]:chain_start[c+1]], chain c warm from
    state_in[c] (or cold when state_in is None); state_out [n_chains, state] receives each chain's
    state after its last operator.  Returns (evals[len, L], evecs or None, stats list)."""
    lib = load_library()
    queue = np.ascontiguousarray(np.asarray(queue, dtype=np.int32))
    starts = np.ascontiguousarray(np.asarray(chain_start, dtype=np.int32))
    nq, nc = int(queue.shape[0]), len(starts) - 1
    sd = chain_state_doubles(ops, L, nex)
    for t, nm in ((state_in, "state_in"), (state_out, "state_out")):
        if t is not None:
            _require_cuda_f64(t, nm)
            if t.numel() < nc * sd:
                raise ValueError(f"{nm} needs {nc} x {sd} doubles")
    st = ops.c_struct()
    per = lib.scsf_solve_workspace_bytes(ctypes.byref(st), L, nex)
    if ws is None or ws.numel() < per * nc:
        ws = _workspace(per * nc, ops.coef.device)
    dev = ops.coef.device
    evals = torch.empty((max(nq, 1), L), dtype=torch.float64, device=dev)
    evecs = torch.empty((nq, L, ops.ld), dtype=torch.float64, device=dev) if want_vecs else None
    stats = (scsf_stats * max(nq, 1))()
    code = lib.scsf_solve_chains_resume(ctypes.byref(st), queue.ctypes.data_as(ctypes.c_void_p),
                                        starts.ctypes.data_as(ctypes.c_void_p), nc, L, nex, degree, tol, max_iter,
                                        ctypes.c_uint64(seed), _ptr(state_in), _ptr(state_out), _ptr(evals),
                                        _ptr(evecs), ops.ld, stats, _ptr(ws), ws.numel(), _stream())
    if raise_on_fail or code != SCSF_ERR_NUMERICAL:
        _check(code)
    return evals[:nq], evecs, [stats[i].as_dict() for i in range(nq)]


# ------------------------------------------------------- component entries ----
# Blocks are column-major: a torch tensor of shape [cols, ld] holds an ld x cols block.
def gemm_tn(X: torch.Tensor, Y: torch.Tensor, n: int, alpha: float = 1.0, upper: bool = False) -> torch.Tensor:
    """C = alpha X[:n]^T Y[:n] for X [b1, ldx], Y [b2, ldy]; returns C as [b2, b1] (column-major b1 x b2)."""
    lib = load_library()
    b1, ldx = X.shape
    b2, ldy = Y.shape
    ws = _workspace(lib.scsf_dev_workspace_bytes(n, b1, b2), X.device)
    C = torch.zeros((b2, b1), dtype=torch.float64, device=X.device)
    _check(lib.scsf_gemm_tn(_ptr(X), ldx, b1, _ptr(Y), ldy, b2, n, alpha, 1 if upper else 0, _ptr(C), b1,
                            _ptr(ws), ws.numel(), _stream()))
    return C


def gemm_nn(X: torch.Tensor, M: torch.Tensor, n: int, alpha: float = 1.0, beta: float = 0.0,
            out: torch.Tensor | None = None) -> torch.Tensor:
    """Out = alpha X[:n] M + beta Out for X [b1, ldx], M [b2, b1] (column-major b1 x b2); out [b2, ldx]."""
    lib = load_library()
    b1, ldx = X.shape
    b2, ldm = M.shape
    if out is None:
        out = torch.zeros((b2, ldx), dtype=torch.float64, device=X.device)
    _check(lib.scsf_gemm_nn(_ptr(X), ldx, n, b1, _ptr(M), ldm, b2, alpha, beta, _ptr(out), out.shape[1], _stream()))
    return out


def chol_inv(S: torch.Tensor, nrows: int = 1):
    """R^{-1} of S = R^T R (upper triangle of S used); S, result [b, b] column-major."""
    lib = load_library()
    b = S.shape[0]
    ws = _workspace(lib.scsf_dev_workspace_bytes(1, b, b), S.device)
    R = torch.empty_like(S)
    _check(lib.scsf_chol_inv(_ptr(S), b, b, nrows, _ptr(R), _ptr(ws), ws.numel(), _stream()))
    return R


def syev_small(G: torch.Tensor, return_sweeps: bool = False):
    """theta ascending, Z (column-major [b, b]) with G = Z diag(theta) Z^T (upper triangle of G used)."""
    lib = load_library()
    b = G.shape[0]
    ws = _workspace(lib.scsf_dev_workspace_bytes(1, b, b), G.device)
    theta = torch.empty(b, dtype=torch.float64, device=G.device)
    Z = torch.empty_like(G)
    sw = ctypes.c_int32(0)
    _check(lib.scsf_syev_small(_ptr(G), b, b, _ptr(theta), _ptr(Z), ctypes.byref(sw), _ptr(ws), ws.numel(),
                               _stream()))
    return (theta, Z, sw.value) if return_sweeps else (theta, Z)


# ------------------------------------------------- row-partitioned solve ----
def slab_rows(ny: int, world: int, rank: int) -> tuple[int, int]:
    """Grid rows [y0, y1) owned by `rank` (scsf_slab_rows)."""
    lib = load_library()
    y0, y1 = ctypes.c_int32(0), ctypes.c_int32(0)
    lib.scsf_slab_rows(ny, world, rank, ctypes.byref(y0), ctypes.byref(y1))
    return y0.value, y1.value


class Comm:
    """Owning handle of a scsf_comm (NCCL or loopback)."""

    def __init__(self, handle):
        self.handle = ctypes.c_void_p(handle)
        r, w = ctypes.c_int32(0), ctypes.c_int32(0)
        _check(load_library().scsf_comm_rank(self.handle, ctypes.byref(r), ctypes.byref(w)))
        self.rank, self.world = r.value, w.value

    def close(self):
        if self.handle:
            load_library().scsf_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p(None)


def comm_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 makes it; broadcast it with torch.distributed)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().scsf_comm_unique_id(buf))
    return buf.raw


def comm_create(rank: int, world: int, uid: bytes) -> Comm:
    """NCCL communicator over NVLink/NVSwitch (collective: every rank calls it)."""
    buf = ctypes.create_string_buffer(bytes(uid), 128)
    h = ctypes.c_void_p(None)
    _check(load_library().scsf_comm_create(rank, world, buf, ctypes.byref(h)))
    return Comm(h.value)


def comm_create_loopback(world: int) -> list[Comm]:
    """`world` in-process virtual ranks on the current device (tests / one-GPU parity)."""
    arr = (ctypes.c_void_p * world)()
    _check(load_library().scsf_comm_create_loopback(world, arr))
    return [Comm(arr[r]) for r in range(world)]


def solve_queue_dist(ops: Operators, chain, L: int, nex: int, comm: Comm, degree: int = 20, tol: float = 1e-8,
                     max_iter: int = 200, seed: int = 0, want_vecs: bool = True, raise_on_fail=True,
                     stream: torch.cuda.Stream | None = None):
    """Row-partitioned SCSF chain solve on this rank's slab (scsf_solve_queue_dist).

    Returns (evals[n_chain, L], evecs_local[n_chain, L, ld_loc] or None, stats list, (y0, y1))."""
    lib = load_library()
    chain = np.ascontiguousarray(np.asarray(chain, dtype=np.int32))
    nc = int(chain.shape[0])
    y0, y1 = slab_rows(ops.ny, comm.world, comm.rank)
    st = ops.c_struct()
    dev = ops.coef.device
    ws = _workspace(lib.scsf_solve_dist_workspace_bytes(ctypes.byref(st), y0, y1, L, nex, comm.world), dev)
    n_loc = ops.nx * (y1 - y0)
    ld_loc = ld_for(n_loc)
    evals = torch.empty((nc, L), dtype=torch.float64, device=dev)
    evecs = torch.empty((nc, L, ld_loc), dtype=torch.float64, device=dev) if want_vecs else None
    stats = (scsf_stats * max(nc, 1))()
    s = (stream or torch.cuda.current_stream()).cuda_stream
    code = lib.scsf_solve_queue_dist(ctypes.byref(st), y0, y1, chain.ctypes.data_as(ctypes.c_void_p), nc, L, nex,
                                     degree, tol, max_iter, ctypes.c_uint64(seed), _ptr(evals), _ptr(evecs), ld_loc,
                                     stats, comm.handle, _ptr(ws), ws.numel(), s)
    if raise_on_fail or code != SCSF_ERR_NUMERICAL:
        _check(code)
    return evals, evecs, [stats[i].as_dict() for i in range(nc)], (y0, y1)
