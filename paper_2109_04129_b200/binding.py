"""ctypes binding of libps (include/ps.h). Marshalling only — no numerics here.

Vectors are passed as column-major N x nrhs complex128 buffers in the caller's
(RWG) order: torch CUDA tensors (device path, on_device=1) or numpy arrays /
pinned torch CPU tensors (host path, on_device=0).
"""
from __future__ import annotations

import ctypes
import os
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(HERE, "libps.so")

PS_OK, PS_EINVAL, PS_EIO, PS_EFORMAT, PS_ENOMEM, PS_ECUDA, PS_ENCCL, PS_ESINGULAR, PS_EDIVERGED, \
    PS_ESTATE = range(10)
STATUS_NAMES = ["PS_OK", "PS_EINVAL", "PS_EIO", "PS_EFORMAT", "PS_ENOMEM", "PS_ECUDA", "PS_ENCCL",
                "PS_ESINGULAR", "PS_EDIVERGED", "PS_ESTATE"]
PS_OP_RT, PS_OP_DINV, PS_OP_R, PS_OP_ZF, PS_OP_U = 1, 2, 3, 4, 5
INFO_KEYS = ["N", "n_leaves", "n_near", "n_far", "alpha_blocks", "nR", "nD", "nF", "height",
             "depth", "setup_madds", "setup_done", "nranks", "own_rows", "sep_rows", "chains",
             "chain_height", "T_entries", "op_bytes", "setup_bytes"]


class PsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 10 else status}: {msg}")
        self.status = status


class _Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("device", ctypes.c_int),
                ("nccl_unique_id", ctypes.c_void_p), ("partition", ctypes.c_int)]


class _Opts(ctypes.Structure):
    _fields_ = [("deterministic", ctypes.c_int), ("ordering", ctypes.c_int),
                ("amalgamate_separators", ctypes.c_int), ("ratio_threshold", ctypes.c_double)]


class _Report(ctypes.Structure):
    _fields_ = [("nrhs", ctypes.c_int64), ("it0_norm", ctypes.c_void_p), ("it1_norm", ctypes.c_void_p),
                ("n_diverged", ctypes.c_int), ("t_solve_ms", ctypes.c_double),
                ("bytes_moved", ctypes.c_double), ("flops", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64), ("ratio", ctypes.c_void_p)]


class _SeriesOpts(ctypes.Structure):
    _fields_ = [("max_terms", ctypes.c_int), ("tol", ctypes.c_double)]


class _SeriesReport(ctypes.Structure):
    _fields_ = [("nrhs", ctypes.c_int64), ("max_terms", ctypes.c_int64), ("it_norm", ctypes.c_void_p),
                ("n_terms", ctypes.c_int), ("n_diverged", ctypes.c_int), ("t_solve_ms", ctypes.c_double),
                ("bytes_moved", ctypes.c_double), ("flops", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64)]


_lib = None


def lib_path() -> str:
    return _SO


def load_library():
    """Load libps.so (building it first if the sources are newer and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    from .build import build, nvcc_available
    if nvcc_available():
        build(force=bool(os.environ.get("PS_REBUILD")))     # no-op unless sources are newer
    so = os.environ.get("PS_LIB", _SO)         # A/B experiments with alternative builds
    if not os.path.exists(so):
        raise ImportError(f"libps.so not found at {so}; run `python -m paper_2109_04129_b200.build`")
    L = ctypes.CDLL(so)
    P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    L.hm_load.restype = I
    L.hm_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(_Dist), ctypes.POINTER(ctypes.c_void_p)]
    L.ps_setup.restype = I
    L.ps_setup.argtypes = [P, ctypes.POINTER(_Opts)]
    L.ps_solve.restype = I
    L.ps_solve.argtypes = [P, I64, P, I64, P, I64, I, P, ctypes.POINTER(_Report)]
    L.ps_solve_async.restype = I
    L.ps_solve_async.argtypes = [P, I64, P, I64, P, I64, P]
    L.ps_solve_report.restype = I
    L.ps_solve_report.argtypes = [P, ctypes.POINTER(_Report)]
    L.ps_solve_series.restype = I
    L.ps_solve_series.argtypes = [P, ctypes.POINTER(_SeriesOpts), I64, P, I64, P, I64, I, P,
                                  ctypes.POINTER(_SeriesReport)]
    L.ps_farfield.restype = I
    L.ps_farfield.argtypes = [I64, P, I64, P, I64, P, P, P, P, D, D, P, I64, I64, I64, P, I, P, P, P]
    L.ps_apply.restype = I
    L.ps_apply.argtypes = [P, I, I64, P, P]
    L.ps_n.restype = I64
    L.ps_n.argtypes = [P]
    L.ps_last_error.restype = ctypes.c_char_p
    L.ps_last_error.argtypes = [P]
    L.ps_free.restype = None
    L.ps_free.argtypes = [P]
    L.ps_info.restype = I
    L.ps_info.argtypes = [P, ctypes.POINTER(D), I]
    L.ps_get_dinv.restype = I64
    L.ps_get_dinv.argtypes = [P, I64, P, I64]
    L.ps_profile.restype = I
    L.ps_profile.argtypes = [P, I]
    L.ps_profile_read.restype = I
    L.ps_profile_read.argtypes = [P, ctypes.POINTER(D), I]
    L.ps_analyze.restype = I
    L.ps_analyze.argtypes = [ctypes.c_char_p, ctypes.POINTER(D), I]
    L.ps_validate.restype = I64
    L.ps_validate.argtypes = [ctypes.c_char_p, I64, P, I]
    L.ps_analyze_rank.restype = I
    L.ps_analyze_rank.argtypes = [ctypes.c_char_p, I, I, ctypes.POINTER(D), I]
    L.ps_trace.restype = I
    L.ps_trace.argtypes = [P, I]
    L.ps_trace_read.restype = I64
    L.ps_trace_read.argtypes = [P, ctypes.POINTER(I64), I64]
    L.ps_elim_leaf.restype = I64
    L.ps_elim_leaf.argtypes = [P, I64]
    L.ps_setup_group.restype = I
    L.ps_setup_group.argtypes = [ctypes.POINTER(P), I, ctypes.POINTER(_Opts)]
    L.ps_solve_group.restype = I
    L.ps_solve_group.argtypes = [ctypes.POINTER(P), I, I64, P, I64, P, I64, P, ctypes.POINTER(_Report)]
    L.ps_nccl_unique_id.restype = I
    L.ps_nccl_unique_id.argtypes = [P, I64]
    L.ps_partition.restype = I64
    L.ps_partition.argtypes = [ctypes.c_char_p, I, P, P, I64]
    _lib = L
    return L


def _ptr_ld(X, N):
    """(pointer, leading dimension, on_device) of a column-major N x nrhs complex128 buffer."""
    try:
        import torch
        if isinstance(X, torch.Tensor):
            if X.dtype != torch.complex128:
                raise TypeError("expected complex128")
            if X.dim() == 1:
                X = X.unsqueeze(1)
            if X.shape[0] != N or X.stride(0) != 1:
                raise ValueError("expected a column-major (stride(0) == 1) N x nrhs tensor")
            ld = X.stride(1) if X.shape[1] > 1 else N
            return X.data_ptr(), ld, X.shape[1], (1 if X.is_cuda else 0)
    except ImportError:
        pass
    X = np.asarray(X)
    if X.dtype != np.complex128:
        raise TypeError("expected complex128")
    if X.ndim == 1:
        X = X[:, None]
    if X.shape[0] != N or not (X.flags.f_contiguous or X.shape[1] == 1):
        raise ValueError("expected a Fortran-ordered N x nrhs array")
    return X.ctypes.data, N, X.shape[1], 0


class PsHandle:
    """One loaded H-matrix on one GPU (hm_load / ps_setup / ps_solve)."""

    def __init__(self, path: str, device: int | None = None, rank: int = 0, nranks: int = 1,
                 partition: bool = False, nccl_id: bytes | None = None):
        """partition=False: replicated operator (the caller splits RHS columns).
        partition=True: row partition over nranks (include/ps.h ps_dist); with
        nccl_id (ps_nccl_unique_id() bytes shared by rank 0) ps_solve runs this
        rank's share with NCCL collectives, without it the handles of all ranks
        belong to one process and are solved together by solve_group()."""
        L = load_library()
        h = ctypes.c_void_p()
        dist = None
        self._idbuf = None
        if device is not None or nranks > 1:
            idp = None
            if nccl_id is not None:
                self._idbuf = ctypes.create_string_buffer(bytes(nccl_id), len(nccl_id))
                idp = ctypes.cast(self._idbuf, ctypes.c_void_p)
            dist = _Dist(rank, nranks, 0 if device is None else device, idp, 1 if partition else 0)
        st = L.hm_load(path.encode(), ctypes.byref(dist) if dist is not None else None, ctypes.byref(h))
        if st != PS_OK:
            raise PsError(st, L.ps_last_error(None).decode())
        self._h = h
        self.N = int(L.ps_n(h))
        self.last_report = None

    def _check(self, st: int):
        if st != PS_OK and st != PS_EDIVERGED:
            raise PsError(st, load_library().ps_last_error(self._h).decode())
        return st

    def close(self):
        if getattr(self, "_h", None):
            load_library().ps_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def setup(self, ratio_threshold: float = 0.1, ordering: int = 0):
        """ordering 0: the file's nested-dissection order; 2: reverse Cuthill-McKee."""
        o = _Opts(1, int(ordering), 0, float(ratio_threshold))
        self._check(load_library().ps_setup(self._h, ctypes.byref(o)))

    def solve(self, B, X, stream=None, want_norms: bool = True):
        """X <- two-term solution for B (both column-major N x nrhs complex128).
        Returns (status, report dict). PS_EDIVERGED becomes a warning."""
        bp, ldb, nrhs, bdev = _ptr_ld(B, self.N)
        xp, ldx, nrhs2, xdev = _ptr_ld(X, self.N)
        if nrhs != nrhs2 or bdev != xdev:
            raise ValueError("B and X must have the same shape and location")
        rep, it0, it1, ratio = _report(nrhs, want_norms)
        s = None
        if stream is not None:
            s = ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        st = self._check(load_library().ps_solve(self._h, nrhs, bp, ldb, xp, ldx, bdev, s,
                                                 ctypes.byref(rep)))
        r = dict(it0=it0, it1=it1, n_diverged=rep.n_diverged, t_solve_ms=rep.t_solve_ms,
                 bytes=rep.bytes_moved, flops=rep.flops, launches=rep.kernel_launches,
                 status=STATUS_NAMES[st])
        if want_norms:
            r["ratio"] = ratio
        if st == PS_EDIVERGED:
            warnings.warn(load_library().ps_last_error(self._h).decode(), RuntimeWarning, stacklevel=2)
        self.last_report = r
        return st, r

    def solve_async(self, B, X, stream=None):
        """Queue the two-term solve of DEVICE tensors on `stream` without synchronising
        (ps_solve_async); solve_report() later returns the last queued solve's report."""
        bp, ldb, nrhs, bdev = _ptr_ld(B, self.N)
        xp, ldx, nrhs2, xdev = _ptr_ld(X, self.N)
        if nrhs != nrhs2 or not (bdev and xdev):
            raise ValueError("solve_async takes device tensors of the same shape")
        s = None
        if stream is not None:
            s = ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        self._pend_nrhs = nrhs
        self._check(load_library().ps_solve_async(self._h, nrhs, bp, ldb, xp, ldx, s))

    def solve_report(self):
        """(status, report dict) of the last solve_async (ps_solve_report: synchronises its stream)."""
        nrhs = getattr(self, "_pend_nrhs", 0) or 1
        rep, it0, it1, ratio = _report(nrhs, True)
        st = self._check(load_library().ps_solve_report(self._h, ctypes.byref(rep)))
        r = dict(it0=it0, it1=it1, ratio=ratio, n_diverged=rep.n_diverged, t_solve_ms=rep.t_solve_ms,
                 bytes=rep.bytes_moved, flops=rep.flops, launches=rep.kernel_launches,
                 status=STATUS_NAMES[st])
        if st == PS_EDIVERGED:
            warnings.warn(load_library().ps_last_error(self._h).decode(), RuntimeWarning, stacklevel=2)
        self.last_report = r
        return st, r

    def solve_series(self, B, X, max_terms: int = 2, tol: float = 0.0, stream=None):
        """X <- n-term series solution (ps_solve_series): at most max_terms terms, stopping
        early once every column's newest term is <= tol x the partial sum (tol > 0).
        Returns (status, report dict with it_norm[n_terms, nrhs]). PS_EDIVERGED -> warning."""
        bp, ldb, nrhs, bdev = _ptr_ld(B, self.N)
        xp, ldx, nrhs2, xdev = _ptr_ld(X, self.N)
        if nrhs != nrhs2 or bdev != xdev:
            raise ValueError("B and X must have the same shape and location")
        itn = np.zeros((max(int(max_terms), 1), nrhs))
        rep = _SeriesReport(nrhs, itn.shape[0], itn.ctypes.data, 0, 0, 0.0, 0.0, 0.0, 0)
        o = _SeriesOpts(int(max_terms), float(tol))
        s = None
        if stream is not None:
            s = ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
        st = self._check(load_library().ps_solve_series(self._h, ctypes.byref(o), nrhs, bp, ldb, xp, ldx,
                                                        bdev, s, ctypes.byref(rep)))
        r = dict(n_terms=rep.n_terms, it_norm=itn[:rep.n_terms], n_diverged=rep.n_diverged,
                 t_solve_ms=rep.t_solve_ms, bytes=rep.bytes_moved, flops=rep.flops,
                 launches=rep.kernel_launches, status=STATUS_NAMES[st])
        if st == PS_EDIVERGED:
            warnings.warn(load_library().ps_last_error(self._h).decode(), RuntimeWarning, stacklevel=2)
        return st, r

    def apply(self, op: int, X, Y):
        """Y <- op X for DEVICE column-major tensors with ld = N (diagnostics)."""
        xp, ldx, nrhs, xdev = _ptr_ld(X, self.N)
        yp, ldy, nrhs2, ydev = _ptr_ld(Y, self.N)
        if not (xdev and ydev) or ldx != self.N or ldy != self.N or nrhs != nrhs2:
            raise ValueError("ps_apply takes device tensors with ld == N")
        self._check(load_library().ps_apply(self._h, op, nrhs, xp, yp))

    def info(self) -> dict:
        out = (ctypes.c_double * len(INFO_KEYS))()
        n = load_library().ps_info(self._h, out, len(INFO_KEYS))
        return {k: out[i] for i, k in enumerate(INFO_KEYS[:n])}

    def dinv(self, pos: int) -> np.ndarray:
        L = load_library()
        need = L.ps_get_dinv(self._h, pos, None, 0)      # -(n_k^2): the capacity to pass
        if need >= 0:
            raise PsError(PS_EINVAL, "ps_get_dinv failed")
        buf = np.zeros(-need, dtype=np.complex128)
        n = L.ps_get_dinv(self._h, pos, buf.ctypes.data, -need)
        if n <= 0:
            raise PsError(PS_EINVAL, "ps_get_dinv failed")
        return buf[:n * n].reshape(n, n, order="F")

    PROFILE_CLASSES = ["fwd_sweep", "bwd_sweep", "dinv", "far_stage1", "far_stage2", "aux", "solve_program", "far1p"]

    def profile(self, enable: bool = True):
        self._check(load_library().ps_profile(self._h, 1 if enable else 0))

    def profile_read(self) -> dict:
        n = 4 * len(self.PROFILE_CLASSES)
        out = (ctypes.c_double * n)()
        load_library().ps_profile_read(self._h, out, n)
        return {c: dict(ms=out[4 * i], launches=int(out[4 * i + 1]), flops=out[4 * i + 2],
                        bytes=out[4 * i + 3]) for i, c in enumerate(self.PROFILE_CLASSES)}

    def trace(self, cls: int):
        self._check(load_library().ps_trace(self._h, cls))

    def trace_read(self, cap: int = 2_000_000) -> np.ndarray:
        buf = np.zeros(14 * cap, dtype=np.int64)
        n = load_library().ps_trace_read(self._h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), cap)
        return buf[:14 * n].reshape(n, 14)

    def elim_leaf(self, pos: int) -> int:
        return int(load_library().ps_elim_leaf(self._h, pos))


def farfield(nodes, tris, tp, tm, vp, vm, k: float, eta: float, I, rhat, mono: bool = False,
             with_sigma: bool = True, stream=None):
    """ps_farfield: far-field vectors F and RCS sigma (m^2; theta, phi polarisation) of the RWG
    currents I (N x nrhs column-major complex128) in the directions rhat (ndir x 3). Host
    arrays are copied to the current CUDA device (marshalling); returns torch CUDA tensors
    F (ndir x nrhs x 3, or ndir x 3 with mono) and sigma (ndir x nrhs x 2, or ndir x 2)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())

    def d(a, dt):
        t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
        return t.to(device=dev, dtype=dt).contiguous()
    nodes_d, tris_d = d(nodes, torch.float64), d(tris, torch.int64)
    tp_d, tm_d, vp_d, vm_d = (d(a, torch.int64) for a in (tp, tm, vp, vm))
    rh = d(rhat, torch.float64).reshape(-1, 3)
    N = int(tp_d.numel())
    if isinstance(I, torch.Tensor):
        Id = I.to(device=dev, dtype=torch.complex128)
    else:
        Id = torch.from_numpy(np.ascontiguousarray(np.asfortranarray(I, dtype=np.complex128).T)).to(dev).T \
            if np.ndim(I) == 2 else torch.from_numpy(np.asarray(I, np.complex128)).to(dev)
    if Id.dim() == 1:
        Id = Id.unsqueeze(1)
    if Id.shape[0] != N or Id.stride(0) != 1:
        Id = Id.T.contiguous().T
    nrhs, ndir = Id.shape[1], rh.shape[0]
    ldi = Id.stride(1) if nrhs > 1 else N
    ncol = 1 if mono else nrhs
    F = torch.empty((ndir, ncol, 3), dtype=torch.complex128, device=dev)
    sig = torch.empty((ndir, ncol, 2), dtype=torch.float64, device=dev) if with_sigma else None
    s = None
    if stream is not None:
        s = ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    L = load_library()
    st = L.ps_farfield(nodes_d.shape[0] if nodes_d.dim() == 2 else nodes_d.numel() // 3, nodes_d.data_ptr(),
                       tris_d.numel() // 3, tris_d.data_ptr(), N, tp_d.data_ptr(), tm_d.data_ptr(),
                       vp_d.data_ptr(), vm_d.data_ptr(), float(k), float(eta), Id.data_ptr(), ldi, nrhs, ndir,
                       rh.data_ptr(), 1 if mono else 0, F.data_ptr(),
                       sig.data_ptr() if sig is not None else None, s)
    if st != PS_OK:
        raise PsError(st, L.ps_last_error(None).decode())
    if mono:
        F = F[:, 0]
        sig = sig[:, 0] if sig is not None else None
    return F, sig


def _report(nrhs, want_norms):
    it0 = np.zeros(nrhs) if want_norms else None
    it1 = np.zeros(nrhs) if want_norms else None
    ratio = np.zeros(nrhs) if want_norms else None
    rep = _Report(nrhs, it0.ctypes.data if want_norms else None, it1.ctypes.data if want_norms else None,
                  0, 0.0, 0.0, 0.0, 0, ratio.ctypes.data if want_norms else None)
    return rep, it0, it1, ratio


def solve_group(handles, B, X, stream=None, want_norms: bool = True):
    """ps_solve_group: one solve of an in-process row partition (handles =
    ranks 0..P-1, PsHandle(..., rank=g, nranks=P, partition=True)); B and X
    are device column-major N x nrhs complex128 tensors. Returns (status, report)."""
    L = load_library()
    N = handles[0].N
    bp, ldb, nrhs, bdev = _ptr_ld(B, N)
    xp, ldx, nrhs2, xdev = _ptr_ld(X, N)
    if nrhs != nrhs2 or not (bdev and xdev):
        raise ValueError("solve_group takes device tensors of equal shape")
    arr = (ctypes.c_void_p * len(handles))(*[h._h for h in handles])
    rep, it0, it1, ratio = _report(nrhs, want_norms)
    s = None
    if stream is not None:
        s = ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))
    st = L.ps_solve_group(arr, len(handles), nrhs, bp, ldb, xp, ldx, s, ctypes.byref(rep))
    if st != PS_OK and st != PS_EDIVERGED:
        raise PsError(st, L.ps_last_error(handles[0]._h).decode())
    r = dict(it0=it0, it1=it1, n_diverged=rep.n_diverged, t_solve_ms=rep.t_solve_ms,
             launches=rep.kernel_launches, status=STATUS_NAMES[st])
    if want_norms:
        r["ratio"] = ratio
    return st, r


def setup_group(handles, ratio_threshold: float = 0.1):
    """ps_setup_group: the sharded setup of an in-process row partition (handles =
    ranks 0..P-1, PsHandle(..., rank=g, nranks=P, partition=True))."""
    L = load_library()
    arr = (ctypes.c_void_p * len(handles))(*[h._h for h in handles])
    o = _Opts(1, 0, 0, float(ratio_threshold))
    st = L.ps_setup_group(arr, len(handles), ctypes.byref(o))
    if st != PS_OK:
        raise PsError(st, L.ps_last_error(handles[0]._h).decode())


def analyze(path: str, rank: int = 0, nranks: int = 1) -> dict:
    """Host-only ps_analyze_rank: structure and per-rank device bytes of a would-be handle."""
    L = load_library()
    out = (ctypes.c_double * len(INFO_KEYS))()
    n = L.ps_analyze_rank(path.encode(), rank, nranks, out, len(INFO_KEYS))
    if n < 0:
        raise PsError(-n, L.ps_last_error(None).decode())
    return {k: out[i] for i, k in enumerate(INFO_KEYS[:n])}


def validate(path: str, nrhs: int) -> dict:
    """Host-only ps_validate of the solve program for nrhs columns (raises on a violation)."""
    L = load_library()
    st = np.full(7, -1, dtype=np.int64)
    n = L.ps_validate(path.encode(), nrhs, st.ctypes.data, 7)
    if n < 0:
        raise PsError(-n, L.ps_last_error(None).decode())
    return dict(items=int(n), tasks=int(st[0]), segments=int(st[1]), work=int(st[2]), write_ranges=int(st[3]),
                read_ranges=int(st[4]), max_ticket_distance=int(st[5]),
                far1p_items=int(st[6]) if st[6] >= 0 else None)


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through libps (128 bytes; rank 0 creates, all ranks share)."""
    L = load_library()
    buf = ctypes.create_string_buffer(128)
    st = L.ps_nccl_unique_id(buf, 128)
    if st != PS_OK:
        raise PsError(st, L.ps_last_error(None).decode())
    return buf.raw


def partition(path: str, nranks: int):
    """Host-only: (owner, far_owner) per elimination position for nranks ranks
    (owner -1 = replicated separator node); see include/ps.h ps_partition."""
    L = load_library()
    cap = 1 << 22
    ow = np.zeros(cap, dtype=np.int32)
    fo = np.zeros(cap, dtype=np.int32)
    n = L.ps_partition(path.encode(), nranks, ow.ctypes.data, fo.ctypes.data, cap)
    if n < 0:
        raise PsError(-n, L.ps_last_error(None).decode())
    return ow[:n].copy(), fo[:n].copy()
