"""ctypes binding of libwalklap.so (include/walklap.h).  Argument marshalling only.

Every numerical step runs in the library's CUDA kernels; this module converts torch CUDA
tensors to (pointer, leading dimension) pairs, numpy CSR arrays to host pointers and torch
streams to cudaStream_t handles.  Names follow walklap.h: θ (theta) = 1 - μ.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libwalklap.so")
_lib = None

WL_WALK, WL_NBT, WL_BTDW = 0, 1, 2
WL_F_EXP, WL_F_RESOLVENT, WL_F_SERIES = 0, 1, 2
_STATUS = {0: "WL_OK", 1: "WL_EINVAL", 2: "WL_EGRAPH", 3: "WL_EDIVERGE", 4: "WL_ENOCONV",
           5: "WL_ENOMEM", 6: "WL_ECUDA", 7: "WL_ENCCL", 8: "WL_EUNSUPPORTED"}


class WalkLapError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_STATUS.get(code, code)}: {msg}")
        self.code = code


class _WalkFun(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("param", ctypes.c_double),
                ("coeffs", ctypes.POINTER(ctypes.c_double)), ("ncoeffs", ctypes.c_int32),
                ("scale", ctypes.c_double)]


class _Opts(ctypes.Structure):
    _fields_ = [("krylov_dim", ctypes.c_int32), ("reorth", ctypes.c_int32),
                ("max_cols", ctypes.c_int32), ("breakdown_tol", ctypes.c_double),
                ("rho_bound", ctypes.c_double), ("relabel", ctypes.c_int32), ("solver", ctypes.c_int32),
                ("cg_tol", ctypes.c_double), ("cg_maxit", ctypes.c_int32), ("cg_check", ctypes.c_int32),
                ("tol", ctypes.c_double), ("halo_overlap", ctypes.c_int32),
                ("lanczos", ctypes.c_int32), ("krylov_adaptive", ctypes.c_int32),
                ("fp32", ctypes.c_int32)]


def load():
    """Load the in-tree CUDA library; raise loudly if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libwalklap.so not found at {LIB_PATH}; run `python -c 'import "
                          "__graft_entry__ as g; g.build()'` (nvcc, sm_100a)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    pvp = ctypes.POINTER(vp)
    sig = {
        "wl_last_error": ([], ctypes.c_char_p),
        "wl_version": ([], ctypes.c_char_p),
        "wl_launch_count": ([], i64),
        "wl_opts_default": ([ctypes.POINTER(_Opts)], None),
        "wl_nccl_unique_id": ([vp], ctypes.c_int),
        "wl_comm_create": ([i32, i32, vp, i32, pvp], ctypes.c_int),
        "wl_comm_destroy": ([vp], None),
        "wl_loopback_create": ([i32, pvp], ctypes.c_int),
        "wl_loopback_set_timeout": ([vp, dbl], ctypes.c_int),
        "wl_loopback_destroy": ([vp], None),
        "wl_comm_create_loopback": ([vp, i32, i32, pvp], ctypes.c_int),
        "wl_partition": ([i64, vp, i32, vp], ctypes.c_int),
        "wl_halo_plan": ([i64, i32, vp, i32, vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "wl_operator_create": ([vp, i64, i64, i64, vp, vp, i32, i32, vp, ctypes.POINTER(_WalkFun),
                                ctypes.POINTER(_Opts), vp, pvp], ctypes.c_int),
        "wl_operator_destroy": ([vp], None),
        "wl_operator_info": ([vp, vp, vp, vp, vp], ctypes.c_int),
        "wl_operator_active_rows": ([vp, vp], ctypes.c_int),
        "wl_operator_diag_shift": ([vp, vp, i64, vp], ctypes.c_int),
        "wl_workspace_create": ([vp, i32, pvp], ctypes.c_int),
        "wl_workspace_destroy": ([vp], None),
        "wl_workspace_stats": ([vp, vp, vp, vp], ctypes.c_int),
        "wl_apply": ([vp, i32, vp, i64, vp, i64, vp, vp], ctypes.c_int),
        "wl_phi_apply": ([vp, i32, vp, i64, vp, i64, vp, vp], ctypes.c_int),
        "wl_apply_host": ([vp, i32, vp, i64, vp, i64, vp, vp], ctypes.c_int),
        "wl_diffuse": ([vp, i32, i32, vp, vp, vp, i64, i32, vp, vp], ctypes.c_int),
        "wl_wait": ([vp, vp], ctypes.c_int),
        "wl_spectral_radius": ([vp, i32, ctypes.POINTER(dbl), vp], ctypes.c_int),
        "wl_spectral_radius_z": ([vp, i32, i32, ctypes.POINTER(dbl), vp], ctypes.c_int),
        "wl_markov": ([vp, i32, i32, vp, vp, i64, vp, vp], ctypes.c_int),
        "wl_xnystrace_exp": ([vp, i32, i32, vp, i64, i32, i32, vp, vp, vp, vp, vp], ctypes.c_int),
        "wl_xnystrace_exp_rational": ([vp, i32, i32, vp, i64, i32, vp, vp, dbl, i32, i32, vp, vp, vp, vp, vp, vp],
                                      ctypes.c_int),
        "wl_aaa_exp_poles": ([dbl, dbl, i32, vp, vp, ctypes.POINTER(i32)], ctypes.c_int),
        "wl_laplacian_bound": ([vp, i32, ctypes.POINTER(dbl)], ctypes.c_int),
        "wl_hessenberg_eigvals": ([i32, vp, vp, vp], ctypes.c_int),
        "wl_symmetric_eig": ([i32, vp, vp, i32], ctypes.c_int),
        "wl_xnystrace_curve": ([i32, i32, dbl, vp, vp, i32, vp, vp, vp], ctypes.c_int),
        "wl_profile_enable": ([i32], None),
        "wl_profile_collect": ([], ctypes.c_int),
        "wl_profile_count": ([], i32),
        "wl_profile_get": ([i32, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(dbl), ctypes.POINTER(i64)],
                           ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def _check(rc):
    if rc != 0:
        raise WalkLapError(rc, load().wl_last_error().decode())


def version() -> str:
    return load().wl_version().decode()


def launch_count() -> int:
    """Kernels launched by libwalklap in this process (monotone)."""
    return int(load().wl_launch_count())


def profile_enable(on: bool = True) -> None:
    """Bracket every library launch with CUDA events on its stream (live per-kernel timing)."""
    load().wl_profile_enable(1 if on else 0)


def profile_collect() -> dict:
    """Synchronize on the recorded events; {kernel name: (total ms, launches)}; clears the session."""
    lib = load()
    _check(lib.wl_profile_collect())
    out = {}
    for i in range(lib.wl_profile_count()):
        name, ms, cnt = ctypes.c_char_p(), ctypes.c_double(), ctypes.c_int64()
        _check(lib.wl_profile_get(i, ctypes.byref(name), ctypes.byref(ms), ctypes.byref(cnt)))
        out[name.value.decode()] = (ms.value, cnt.value)
    return out


def partition(row_ptr: np.ndarray, nranks: int) -> np.ndarray:
    """nnz-balanced contiguous row partition (wl_partition)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    out = np.empty(nranks + 1, dtype=np.int64)
    _check(load().wl_partition(len(rp) - 1, rp.ctypes.data, nranks, out.ctypes.data))
    return out


def halo_plan(n_global: int, bounds: np.ndarray, rank: int, row_ptr_local: np.ndarray,
              col_idx_local: np.ndarray):
    """Host-only halo plan (wl_halo_plan): (local column ids, halo global ids, per-rank counts)."""
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    rp = np.ascontiguousarray(row_ptr_local, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx_local, dtype=np.int32)
    nnz = int(rp[-1] - rp[0])
    col = np.empty(max(1, nnz), dtype=np.int32)
    halo = np.empty(max(1, nnz), dtype=np.int64)
    cnt = np.empty(len(b) - 1, dtype=np.int64)
    nh = ctypes.c_int64()
    _check(load().wl_halo_plan(n_global, len(b) - 1, b.ctypes.data, rank, rp.ctypes.data, ci.ctypes.data,
                               col.ctypes.data, halo.ctypes.data, ctypes.byref(nh), cnt.ctypes.data))
    return col[:nnz], halo[:nh.value], cnt


def hessenberg_eigvals(H: np.ndarray) -> np.ndarray:
    """Eigenvalues of a real upper Hessenberg matrix by the library's host QR (wl_hessenberg_eigvals)."""
    H = np.ascontiguousarray(H, dtype=np.float64)
    n = H.shape[0]
    wr, wi = np.empty(n), np.empty(n)
    _check(load().wl_hessenberg_eigvals(n, H.ctypes.data, wr.ctypes.data, wi.ctypes.data))
    return wr + 1j * wi


def symmetric_eig(A: np.ndarray, method: int = 0):
    """Eigenvalues and eigenvectors (columns) of a symmetric matrix by the library's host solver
    (wl_symmetric_eig: 0 = tridiagonal QL, 1 = Jacobi)."""
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    lam = np.empty(A.shape[0])
    _check(load().wl_symmetric_eig(A.shape[0], A.ctypes.data, lam.ctypes.data, method))
    return lam, A


def xnystrace_curve(lam, W, n: float, times):
    """The library's host XNysTrace (wl_xnystrace_curve) on eigen-coordinates lam (d), W (d x M)."""
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    W = np.ascontiguousarray(W, dtype=np.float64)
    times = np.ascontiguousarray(np.atleast_1d(times), dtype=np.float64)
    p, e = np.empty(len(times)), np.empty(len(times))
    _check(load().wl_xnystrace_curve(W.shape[0], W.shape[1], float(n), lam.ctypes.data, W.ctypes.data,
                                     len(times), times.ctypes.data, p.ctypes.data, e.ctypes.data))
    return p, e


def aaa_exp_poles(xmax: float, tol: float = 1e-13) -> np.ndarray:
    """AAA poles of exp(-x) on [0, xmax] (wl_aaa_exp_poles): one representative per conjugate pair."""
    re, im = np.empty(64), np.empty(64)
    k = ctypes.c_int32()
    _check(load().wl_aaa_exp_poles(float(xmax), float(tol), 64, re.ctypes.data, im.ctypes.data, ctypes.byref(k)))
    return re[:k.value] + 1j * im[:k.value]


def _stream_handle(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _block(t, cols, what):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
        raise TypeError(f"{what}: expected a CUDA float64 tensor")
    if t.dim() == 1:
        t = t.view(-1, 1)
    if t.shape[1] != cols or (t.shape[0] > 1 and t.stride(1) != 1):
        raise ValueError(f"{what}: expected rows x {cols} with unit column stride")
    return t, max(t.stride(0), cols)


class Comm:
    """NCCL communicator over the current torch.distributed group (one process per GPU), or a rank of
    a LoopbackGroup (Comm.loopback)."""

    @classmethod
    def loopback(cls, group: "LoopbackGroup", rank: int, device: int = 0) -> "Comm":
        """Rank `rank` of a single-process loopback group (wl_comm_create_loopback)."""
        self = cls.__new__(cls)
        h = ctypes.c_void_p()
        _check(load().wl_comm_create_loopback(group.handle, rank, device, ctypes.byref(h)))
        self.handle, self.rank, self.world, self.device = h, rank, group.nranks, device
        self._group = group  # the group must outlive its comms
        return self

    def __init__(self, rank: int, world: int, device: int, group=None):
        import torch.distributed as dist
        lib = load()
        uid = (ctypes.c_char * 128)()
        if rank == 0:
            _check(lib.wl_nccl_unique_id(uid))
        obj = [bytes(uid) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        _check(lib.wl_comm_create(world, rank, uid, device, ctypes.byref(h)))
        self.handle, self.rank, self.world, self.device = h, rank, world, device

    def close(self):
        if self.handle:
            load().wl_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """P ranks of the row-partitioned path in ONE process on one device (wl_loopback_create): each rank
    is driven by its own host thread and stream; halo exchanges are device copies and allreduces a
    fixed-order device sum.  Collective calls rendezvous across the ranks' threads (timeout seconds)."""

    def __init__(self, nranks: int, timeout: float = 600.0):
        h = ctypes.c_void_p()
        _check(load().wl_loopback_create(nranks, ctypes.byref(h)))
        self.handle, self.nranks = h, nranks
        _check(load().wl_loopback_set_timeout(h, float(timeout)))

    def close(self):
        if getattr(self, "handle", None):
            load().wl_loopback_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_loopback(nranks: int, fn, device: int = 0, timeout: float = 600.0):
    """Run fn(rank, comm, stream) for every rank of a loopback group, one host thread and one CUDA
    stream per rank on `device`; returns the per-rank results (the first exception is re-raised)."""
    import threading

    import torch
    group = LoopbackGroup(nranks, timeout)
    out, errs = [None] * nranks, [None] * nranks

    def body(r):
        comm = None
        try:
            torch.cuda.set_device(device)
            stream = torch.cuda.Stream(device)
            comm = Comm.loopback(group, r, device)
            with torch.cuda.stream(stream):
                out[r] = fn(r, comm, stream)
            stream.synchronize()
        except BaseException as e:  # noqa: BLE001 (re-raised in the caller's thread)
            errs[r] = e
        finally:
            if comm is not None:
                comm.close()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    group.close()
    for e in errs:
        if e is not None:
            raise e
    return out


class Workspace:
    def cg_iterations(self) -> int:
        """CG iterations executed by actions on this workspace so far (wl_workspace_stats)."""
        return self.stats()[0]

    def stats(self):
        """(cg_iterations, krylov_steps, krylov_batches) so far (wl_workspace_stats)."""
        v, k, b = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(load().wl_workspace_stats(self.handle, ctypes.byref(v), ctypes.byref(k), ctypes.byref(b)))
        return v.value, k.value, b.value

    def __init__(self, op: "Operator", max_b: int):
        self.op = op
        self.max_b = max_b
        h = ctypes.c_void_p()
        _check(load().wl_workspace_create(op.handle, max_b, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            load().wl_workspace_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Operator:
    """𝕃_θ(f) for one graph and n_theta downweighting values (wl_operator_create).

    rows [row_begin, row_end) of an n_global-node graph; row_ptr/col_idx are the HOST CSR arrays
    of those rows (global offsets and column ids).  f = ("exp", β) | ("resolvent", α) |
    ("series", [c0, c1, ...]).  solver="cg" (resolvent only) evaluates φ_θ = (1-μ²α²) 𝒜_θ(α)^{-1} by
    Jacobi-preconditioned conjugate gradients on the deformed Laplacian instead of Krylov on Z.
    lap_scale multiplies 𝕃 (wl_walkfun.scale; 1/(1+α) reproduces Fig. 4b's (1-α) normalisation).
    fp32=1: float storage of the Krylov batches' n-vectors, double sums (wl_opts.fp32; parity 1e-4).
    """

    def __init__(self, n_global, row_ptr, col_idx, thetas=(1.0,), f=("exp", 1.0), variant=None,
                 row_range=None, comm: Comm | None = None, krylov_dim=30, reorth=2, max_cols=32,
                 breakdown_tol=1e-12, rho_bound=0.0, relabel=1, solver="krylov", cg_tol=1e-9, cg_maxit=1000,
                 cg_check=8, lap_scale=1.0, krylov_tol=0.0, halo_overlap=1, lanczos=1, krylov_adaptive=0,
                 fp32=0, stream=None):
        lib = load()
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        rb, re = (0, n_global) if row_range is None else row_range
        thetas = [float(t) for t in np.atleast_1d(thetas)]
        if variant is None:
            variant = WL_BTDW
        elif isinstance(variant, str):
            variant = {"walk": WL_WALK, "nbt": WL_NBT, "btdw": WL_BTDW}[variant]
        th = (ctypes.c_double * len(thetas))(*thetas)
        kind, param = f
        coeffs = None
        wf = _WalkFun()
        if kind == "exp":
            wf.kind, wf.param = WL_F_EXP, float(param)
        elif kind == "resolvent":
            wf.kind, wf.param = WL_F_RESOLVENT, float(param)
        elif kind == "series":
            coeffs = (ctypes.c_double * len(param))(*[float(c) for c in param])
            wf.kind, wf.param, wf.coeffs, wf.ncoeffs = WL_F_SERIES, 0.0, coeffs, len(param)
        else:
            raise ValueError(kind)
        wf.scale = float(lap_scale)
        opts = _Opts()
        lib.wl_opts_default(ctypes.byref(opts))
        opts.krylov_dim, opts.reorth, opts.max_cols = krylov_dim, reorth, max_cols
        opts.breakdown_tol, opts.rho_bound, opts.relabel = breakdown_tol, rho_bound, relabel
        opts.solver = {"krylov": 0, "cg": 1}[solver]
        opts.cg_tol, opts.cg_maxit, opts.cg_check = cg_tol, cg_maxit, cg_check
        opts.tol = krylov_tol
        opts.halo_overlap = halo_overlap
        opts.lanczos = lanczos
        opts.krylov_adaptive = krylov_adaptive
        opts.fp32 = int(fp32)
        h = ctypes.c_void_p()
        _check(lib.wl_operator_create(comm.handle if comm else None, n_global, rb, re, rp.ctypes.data,
                                      ci.ctypes.data, variant, len(thetas) if variant == WL_BTDW else 1,
                                      th, ctypes.byref(wf), ctypes.byref(opts),
                                      _stream_handle(stream), ctypes.byref(h)))
        self.handle = h
        self.comm = comm
        self.reorth = reorth
        self.thetas = thetas if variant == WL_BTDW else [1.0 if variant == WL_WALK else 0.0]
        nl, nz, nh, nt = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        _check(lib.wl_operator_info(h, ctypes.byref(nl), ctypes.byref(nz), ctypes.byref(nh), ctypes.byref(nt)))
        self.n_local, self.nnz_local, self.n_halo, self.n_theta = nl.value, nz.value, nh.value, nt.value
        na = ctypes.c_int64()
        _check(lib.wl_operator_active_rows(h, ctypes.byref(na)))
        self.n_active = na.value  # rows carrying Krylov data (the isolated tail beyond: wl_operator_active_rows)
        self._ws = {}

    def workspace(self, max_b: int) -> Workspace:
        if max_b not in self._ws:
            self._ws[max_b] = Workspace(self, max_b)
        return self._ws[max_b]

    def diag_shift(self, stream=None):
        """t_θ = φ_θ 1 (n_local x n_theta)."""
        import torch
        out = torch.empty((self.n_local, self.n_theta), dtype=torch.float64, device="cuda")
        _check(load().wl_operator_diag_shift(self.handle, ctypes.c_void_p(out.data_ptr()), self.n_theta,
                                             _stream_handle(stream)))
        return out

    def _action(self, fn, V, out, ws, stream):
        import torch
        if V.dim() == 1:
            V = V.view(-1, 1)
        b = V.shape[1]
        V, ldv = _block(V, b, "V")
        cols = self.n_theta * b
        if out is None:
            out = torch.empty((self.n_local, cols), dtype=torch.float64, device=V.device)
        out2, ldo = _block(out, cols, "out")
        ws = ws or self.workspace(b)
        _check(fn(self.handle, b, ctypes.c_void_p(V.data_ptr()), ldv, ctypes.c_void_p(out2.data_ptr()), ldo,
                  ws.handle, _stream_handle(stream)))
        return out

    def apply(self, V, out=None, ws=None, stream=None):
        """𝕃_θ V for every θ: returns n_local x (n_theta * b), column i*b + c = 𝕃_{θ_i} V[:, c]."""
        return self._action(load().wl_apply, V, out, ws, stream)

    def phi_apply(self, V, out=None, ws=None, stream=None):
        """φ_θ V = Σ_k c_k q_k(A) V (same layout as apply)."""
        return self._action(load().wl_phi_apply, V, out, ws, stream)

    def apply_host(self, V: np.ndarray, out: np.ndarray | None = None, ws=None, stream=None) -> np.ndarray:
        """𝕃_θ V with host buffers (copies inside the C call)."""
        V = np.ascontiguousarray(V, dtype=np.float64)
        if V.ndim == 1:
            V = V[:, None]
        b = V.shape[1]
        cols = self.n_theta * b
        if out is None:
            out = np.empty((self.n_local, cols), dtype=np.float64)
        ws = ws or self.workspace(b)
        _check(load().wl_apply_host(self.handle, b, V.ctypes.data, b, out.ctypes.data, out.strides[0] // 8,
                                    ws.handle, _stream_handle(stream)))
        return out

    def diffuse(self, x0, taus, theta_index=0, k_out=80, out=None, ws=None, stream=None):
        """exp(-τ 𝕃_θ) x0 for every τ (columns)."""
        import torch
        taus = np.ascontiguousarray(np.atleast_1d(taus), dtype=np.float64)
        nt = len(taus)
        x0 = x0.reshape(-1)
        if not (x0.is_cuda and x0.dtype == torch.float64 and x0.is_contiguous()):
            raise TypeError("x0: expected a contiguous CUDA float64 vector")
        if out is None:
            out = torch.empty((self.n_local, nt), dtype=torch.float64, device=x0.device)
        out2, ldx = _block(out, nt, "out")
        ws = ws or self.workspace(1)
        _check(load().wl_diffuse(self.handle, theta_index, nt, taus.ctypes.data, ctypes.c_void_p(x0.data_ptr()),
                                 ctypes.c_void_p(out2.data_ptr()), ldx, k_out, ws.handle, _stream_handle(stream)))
        return out

    def spectral_radius(self, k: int = 60, stream=None) -> float:
        """ρ(A) of the operator's graph (wl_spectral_radius: Lanczos on A from the ones vector)."""
        rho = ctypes.c_double()
        _check(load().wl_spectral_radius(self.handle, k, ctypes.byref(rho), _stream_handle(stream)))
        return rho.value

    def markov(self, p0, nsteps, theta_index=0, out=None, ws=None, stream=None):
        """Markov chain P = I - diag(t)^{-1} 𝕃_θ (eq:let_there_be_markov): column k of the result is p_{k+1}."""
        import torch
        p0 = p0.reshape(-1)
        if not (p0.is_cuda and p0.dtype == torch.float64 and p0.is_contiguous()):
            raise TypeError("p0: expected a contiguous CUDA float64 vector")
        if out is None:
            out = torch.empty((self.n_local, nsteps), dtype=torch.float64, device=p0.device)
        out2, ldp = _block(out, nsteps, "out")
        ws = ws or self.workspace(1)
        _check(load().wl_markov(self.handle, theta_index, nsteps, ctypes.c_void_p(p0.data_ptr()),
                                ctypes.c_void_p(out2.data_ptr()), ldp, ws.handle, _stream_handle(stream)))
        return out

    def xnystrace_exp(self, omega, times, k, theta_index=0, ws=None, stream=None):
        """Average return probability p̂_0(t) ≈ (1/n) tr exp(-t 𝕃_θ) and its error estimate for every t
        (Alg. 1 XNysTrace-exp with poles at ∞; wl_xnystrace_exp).  omega: (n_local, M) CUDA float64 probes."""
        times = np.ascontiguousarray(np.atleast_1d(times), dtype=np.float64)
        M = omega.shape[1] if omega.dim() == 2 else 1
        om, ldo = _block(omega, M, "omega")
        p = np.empty(len(times))
        e = np.empty(len(times))
        ws = ws or self.workspace(M)
        _check(load().wl_xnystrace_exp(self.handle, theta_index, M, ctypes.c_void_p(om.data_ptr()), ldo, k,
                                       len(times), times.ctypes.data, p.ctypes.data, e.ctypes.data, ws.handle,
                                       _stream_handle(stream)))
        return p, e

    def laplacian_bound(self, theta_index: int = 0) -> float:
        """Gershgorin bound on ρ(𝕃_θ) (wl_laplacian_bound)."""
        v = ctypes.c_double()
        _check(load().wl_laplacian_bound(self.handle, theta_index, ctypes.byref(v)))
        return v.value

    def xnystrace_exp_rational(self, omega, times, poles="aaa", theta_index=0, inner_tol=1e-6, inner_maxit=500,
                               aaa_tol=1e-13, ws=None, stream=None):
        """Alg. 1 on the block RATIONAL Krylov space (wl_xnystrace_exp_rational).  poles: "aaa" (the AAA poles of
        exp(-x) on [0, t* ρ(𝕃)], with the library's Gershgorin bound for ρ) or an array of ξ (np.inf, real, or
        complex with Im > 0 for a conjugate pair).  Returns (p̂, ê, info) with info = {poles, inner_iters}."""
        times = np.ascontiguousarray(np.atleast_1d(times), dtype=np.float64)
        if isinstance(poles, str):
            poles = aaa_exp_poles(float(times.max()) * self.laplacian_bound(theta_index), aaa_tol)
        poles = np.asarray(poles, dtype=complex)
        re = np.ascontiguousarray(poles.real, dtype=np.float64)
        im = np.ascontiguousarray(np.abs(poles.imag), dtype=np.float64)
        M = omega.shape[1] if omega.dim() == 2 else 1
        om, ldo = _block(omega, M, "omega")
        p, e = np.empty(len(times)), np.empty(len(times))
        it = ctypes.c_int64()
        ws = ws or self.workspace(M)
        _check(load().wl_xnystrace_exp_rational(self.handle, theta_index, M, ctypes.c_void_p(om.data_ptr()), ldo,
                                                len(re), re.ctypes.data, im.ctypes.data, float(inner_tol),
                                                int(inner_maxit), len(times), times.ctypes.data, p.ctypes.data,
                                                e.ctypes.data, ctypes.byref(it), ws.handle, _stream_handle(stream)))
        return p, e, {"poles": poles, "inner_iters": it.value}

    def spectral_radius_z(self, theta_index: int = 0, k: int = 60, stream=None) -> float:
        """ρ(Z_θ) of the companion operator by k Arnoldi steps on Z (wl_spectral_radius_z)."""
        r = ctypes.c_double()
        _check(load().wl_spectral_radius_z(self.handle, theta_index, k, ctypes.byref(r), _stream_handle(stream)))
        return r.value

    def wait(self, stream=None):
        _check(load().wl_wait(self.handle, _stream_handle(stream)))

    def close(self):
        for ws in self._ws.values():
            ws.close()
        self._ws = {}
        if getattr(self, "handle", None):
            load().wl_operator_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
