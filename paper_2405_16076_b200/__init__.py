"""Python binding of liboid.so (include/oid.h): argument marshalling only.

Every step of the ingest path runs in the library's CUDA kernels; PyTorch supplies device
memory (the workspace and the snapshot blocks), streams and, for row-sharded runs,
torch.distributed for the all-reduce of the exposed partial buffers.  There is no CPU
fallback: importing fails if liboid.so has not been built (``python
paper_2405_16076_b200/build.py`` or ``__graft_entry__.build()``).
"""

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboid.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python {_HERE}/build.py` "
                      "(the product path has no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

OID_OK, OID_EINVAL, OID_ESHAPE, OID_ENOMEM, OID_ECUDA, OID_ENCCL, OID_ENUMERIC, OID_ESTATE = 0, -1, -2, -3, -4, -5, -6, -7
_STATUS = {0: "OID_OK", -1: "OID_EINVAL", -2: "OID_ESHAPE", -3: "OID_ENOMEM", -4: "OID_ECUDA", -5: "OID_ENCCL",
           -6: "OID_ENUMERIC", -7: "OID_ESTATE"}
OID_F32, OID_F64 = 0, 1
K1_AUTO, K1_SIMT_F64, K1_TC_INT8, K1_TC_PAIR, K1_TC_FAST = 0, 1, 2, 3, 4
FLAG_NONFINITE_INPUT, FLAG_SJ_RANK_DEFICIENT, FLAG_E2_NEGATIVE, FLAG_K1_RECOMPUTED = 1, 2, 4, 8

EXPORTED = ["oid_workspace_query", "oid_init", "oid_ingest_block", "oid_ingest_sketch", "oid_ingest_commit",
            "oid_partials", "oid_estimate_begin", "oid_estimate_end", "oid_error_estimate", "oid_finalize", "oid_get",
            "oid_stats", "oid_stats_reset", "oid_sketch_table", "oid_destroy", "oid_last_error", "oid_version",
            "oid_gradient_gcv", "oid_gradient_coefficients", "oid_gradient_finalize", "oid_report",
            "oid_ingest_sketch_halo", "oid_grad_halo", "oid_gradient_ogo"]


class OidParams(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
                ("n_cap", ctypes.c_int64), ("k", ctypes.c_int32), ("ell", ctypes.c_int32), ("b_max", ctypes.c_int32),
                ("ell1", ctypes.c_int32), ("ell2", ctypes.c_int32), ("ell3", ctypes.c_int32),
                ("lam", ctypes.c_double), ("eps", ctypes.c_double), ("delta", ctypes.c_double), ("c", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("dtype", ctypes.c_int32), ("k1_mode", ctypes.c_int32),
                ("profile", ctypes.c_int32), ("device", ctypes.c_int32),
                ("grad_nfields", ctypes.c_int32), ("grad_nx", ctypes.c_int32), ("grad_ny", ctypes.c_int32),
                ("omega_cache", ctypes.c_int32), ("grad_hx", ctypes.c_double), ("grad_hy", ctypes.c_double),
                ("coeff_mode", ctypes.c_int32), ("epoch_mode", ctypes.c_int32),
                ("grad_nz", ctypes.c_int32), ("a9_mode", ctypes.c_int32), ("grad_hz", ctypes.c_double)]


class OidStats(ctypes.Structure):
    _fields_ = [("n_obs", ctypes.c_int64), ("epochs", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("k1_launches", ctypes.c_int64), ("k1_ms", ctypes.c_double), ("post_ms", ctypes.c_double),
                ("est_ms", ctypes.c_double), ("flags", ctypes.c_uint32), ("k1_mode_used", ctypes.c_int32),
                ("a9_ms", ctypes.c_double), ("a9_launches", ctypes.c_int64), ("admissions", ctypes.c_int64),
                ("dirty_slots", ctypes.c_int64), ("estimates", ctypes.c_int64), ("lat_min_ms", ctypes.c_double),
                ("lat_med_ms", ctypes.c_double), ("lat_max_ms", ctypes.c_double)]


_vp, _i64, _i32, _dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_double)
_sig = {
    "oid_workspace_query": [ctypes.POINTER(OidParams), ctypes.POINTER(ctypes.c_size_t)],
    "oid_init": [ctypes.POINTER(OidParams), _vp, ctypes.c_size_t, _vp, ctypes.POINTER(_vp)],
    "oid_ingest_block": [_vp, _vp, _i64, _i32, _vp],
    "oid_ingest_sketch": [_vp, _vp, _i64, _i32, _vp],
    "oid_ingest_commit": [_vp, _vp, _i64, _i32, _vp],
    "oid_ingest_sketch_halo": [_vp, _vp, _i64, _i32, _vp, _i64, _vp, _i64, _vp],
    "oid_grad_halo": [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
    "oid_gradient_ogo": [_vp, _vp],
    "oid_partials": [_vp, _i32, ctypes.POINTER(_dp), ctypes.POINTER(_i64)],
    "oid_estimate_begin": [_vp, _vp],
    "oid_estimate_end": [_vp, _vp, _vp],
    "oid_error_estimate": [_vp, _dp, _vp],
    "oid_finalize": [_vp, _vp, _vp, _i32, _vp, _vp],
    "oid_get": [_vp, _i32, _vp, ctypes.c_size_t, _vp],
    "oid_stats": [_vp, ctypes.POINTER(OidStats)],
    "oid_stats_reset": [_vp],
    "oid_sketch_table": [ctypes.POINTER(ctypes.c_int32), _dp],
    "oid_gradient_gcv": [_vp, ctypes.c_double, _dp, _vp],
    "oid_gradient_coefficients": [_vp, ctypes.c_double, _vp, _vp],
    "oid_gradient_finalize": [_vp, ctypes.c_double, ctypes.c_double, ctypes.c_double, _dp, _vp, _vp],
    "oid_report": [_vp, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t), _vp],
}
for _n, _a in _sig.items():
    getattr(_lib, _n).argtypes = _a
    getattr(_lib, _n).restype = ctypes.c_int
_lib.oid_destroy.argtypes = [_vp]
_lib.oid_destroy.restype = None
_lib.oid_last_error.argtypes = [_vp]
_lib.oid_last_error.restype = ctypes.c_char_p
_lib.oid_version.argtypes = []
_lib.oid_version.restype = ctypes.c_char_p


class OidError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


def lib():
    return _lib


def version():
    return _lib.oid_version().decode()


def sketch_table():
    """Host-only: (q[16] int32, scale) of the Gauss-16 sketch entries s * (q[n] + 1/2) (reading R2)."""
    q = (ctypes.c_int32 * 16)()
    s = ctypes.c_double()
    st = _lib.oid_sketch_table(q, ctypes.byref(s))
    if st != OID_OK:
        raise OidError(st, "oid_sketch_table")
    return np.frombuffer(q, dtype=np.int32).copy(), s.value


def hutch_split(ell):
    a, b = ell // 6, ell // 3
    return (a, b, ell - a - b)


def make_params(m, k, ell, b_max, n_cap, lam, split=None, eps=0.5, delta=0.05, c=1.0, seed=0, dtype="f64",
                row_begin=0, row_end=None, k1_mode=K1_AUTO, profile=False, device=0, grad=None,
                omega_cache=False, coeff="alg4", epochs="block", grad3=None, a9q=False):
    """grad: None, or (nfields, nx, ny[, hx, hy]) for the gradient-enhanced variant (A11) on a 2-D
    grid; grad3: (nfields, nx, ny, nz[, hx, hy, hz]) for the 3-D grid with three components (NEXT-4).
    coeff: "alg4" (Alg 4 every epoch, the hot path) or "argmin" (Algs 4-7 + NA-Hutch++ argmin, NEXT-1).
    epochs: "block" (one block = one epoch, R4) or "t" (the paper's t-column buffer, NEXT-2).
    a9q: the basis Gram on int8 tensor cores from a 31-bit quantised basis copy (a9_mode = 1,
    oid.h; with k1_mode = K1_TC_FAST)."""
    if coeff not in ("alg4", "argmin"):
        raise ValueError("coeff must be 'alg4' or 'argmin'")
    if epochs not in ("block", "t"):
        raise ValueError("epochs must be 'block' or 't'")
    split = hutch_split(ell) if split is None else split
    g = tuple(grad) + (0.0, 0.0)[len(grad) - 3:] if grad is not None else (0, 0, 0, 0.0, 0.0)
    nz, hz = 0, 0.0
    if grad3 is not None:
        g3 = tuple(grad3) + (0.0, 0.0, 0.0)[len(grad3) - 4:]
        g, nz, hz = (g3[0], g3[1], g3[2], g3[4], g3[5]), int(g3[3]), float(g3[6])
    return OidParams(m=m, row_begin=row_begin, row_end=m if row_end is None else row_end, n_cap=n_cap, k=k, ell=ell,
                     b_max=b_max, ell1=split[0], ell2=split[1], ell3=split[2], lam=lam, eps=eps, delta=delta, c=c,
                     seed=seed, dtype=OID_F64 if dtype in ("f64", "float64") else OID_F32, k1_mode=k1_mode,
                     profile=int(bool(profile)), device=device, grad_nfields=int(g[0]), grad_nx=int(g[1]),
                     grad_ny=int(g[2]), omega_cache=int(omega_cache), grad_hx=float(g[3]), grad_hy=float(g[4]),
                     coeff_mode=1 if coeff == "argmin" else 0, epoch_mode=1 if epochs == "t" else 0,
                     grad_nz=nz, grad_hz=hz, a9_mode=1 if a9q else 0)


def workspace_bytes(params):
    n = ctypes.c_size_t()
    st = _lib.oid_workspace_query(ctypes.byref(params), ctypes.byref(n))
    if st != OID_OK:
        raise OidError(st, "invalid parameters")
    return n.value


class Engine:
    """One oid context on one CUDA device (C ABI calls with torch-owned memory).

    stream: CUDA stream of the ingest calls (default: the current stream).  estimate_stream
    (optional): a second stream for the error-estimate calls, so that an estimate (basis Gram,
    Alg 8) overlaps the next block's ingest; the library orders the two internally.
    """

    def __init__(self, params, stream=None, estimate_stream=None):
        import torch
        self._torch = torch
        self.p = params
        self.device = torch.device("cuda", params.device)
        self.m_loc = params.row_end - params.row_begin
        self.ws_bytes = workspace_bytes(params)
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.estimate_stream = estimate_stream if estimate_stream is not None else self.stream
        h = ctypes.c_void_p()
        st = _lib.oid_init(ctypes.byref(params), ctypes.c_void_p(self.ws.data_ptr()), self.ws_bytes,
                           self._st(), ctypes.byref(h))
        if st != OID_OK:
            raise OidError(st, "oid_init failed: " + _lib.oid_last_error(None).decode())
        self.h = h
        self.dtype = torch.float64 if params.dtype == OID_F64 else torch.float32

    def _st(self):
        return ctypes.c_void_p(self.stream.cuda_stream)

    def _est(self):
        return ctypes.c_void_p(self.estimate_stream.cuda_stream)

    def _check(self, st, what):
        if st != OID_OK:
            raise OidError(st, f"{what}: {_lib.oid_last_error(self.h).decode()}")

    def _block(self, X):
        """X: device tensor (m_loc, ncols) with unit row stride (column-major) -> (ptr, ld, ncols)."""
        if X.device != self.device or X.dtype != self.dtype:
            raise ValueError(f"block must be a {self.dtype} tensor on {self.device}")
        if X.dim() != 2 or X.shape[0] != self.m_loc:
            raise ValueError(f"block must have shape (m_loc={self.m_loc}, ncols)")
        ncols = X.shape[1]
        if ncols > 0 and self.m_loc > 1 and X.stride(0) != 1:
            raise ValueError("block must be column-major (X.stride(0) == 1); pass Xt.T for a (ncols, m) tensor")
        ld = X.stride(1) if ncols > 1 else self.m_loc
        return ctypes.c_void_p(X.data_ptr()), ld, ncols

    def ingest_block(self, X):
        ptr, ld, nc = self._block(X)
        self._check(_lib.oid_ingest_block(self.h, ptr, ld, nc, self._st()), "oid_ingest_block")

    def ingest_sketch(self, X, halo_lo=None, halo_hi=None):
        """halo_lo / halo_hi: the block's stencil halos ((rows, ncols) device tensors, column-major)
        of a sharded gradient-variant context (grad_halo() rows below / above the slab)."""
        ptr, ld, nc = self._block(X)
        if halo_lo is None and halo_hi is None:
            self._check(_lib.oid_ingest_sketch(self.h, ptr, ld, nc, self._st()), "oid_ingest_sketch")
            return
        hp = []
        for H in (halo_lo, halo_hi):
            if H is None or H.shape[0] == 0:
                hp += [ctypes.c_void_p(), 0]
                continue
            if H.device != self.device or H.dtype != self.dtype or H.dim() != 2 or H.shape[1] != nc:
                raise ValueError(f"halo must be a (rows, {nc}) {self.dtype} tensor on {self.device}")
            if H.shape[0] > 1 and H.stride(0) != 1:
                raise ValueError("halo must be column-major (stride(0) == 1)")
            hp += [ctypes.c_void_p(H.data_ptr()), H.stride(1) if nc > 1 else H.shape[0]]
        self._check(_lib.oid_ingest_sketch_halo(self.h, ptr, ld, nc, hp[0], hp[1], hp[2], hp[3], self._st()),
                    "oid_ingest_sketch_halo")

    def grad_halo(self):
        """(rows below, rows above) of stencil halo this shard's blocks need (0, 0 when none)."""
        lo, hi = _i64(), _i64()
        self._check(_lib.oid_grad_halo(self.h, ctypes.byref(lo), ctypes.byref(hi)), "oid_grad_halo")
        return lo.value, hi.value

    def gradient_ogo(self):
        """This shard's part of Omega G^p Omega^T into partials(3) (sum over shards before the GCV)."""
        self._check(_lib.oid_gradient_ogo(self.h, self._st()), "oid_gradient_ogo")

    def ingest_commit(self, X):
        ptr, ld, nc = self._block(X)
        self._check(_lib.oid_ingest_commit(self.h, ptr, ld, nc, self._st()), "oid_ingest_commit")

    def partials(self, which=0):
        """fp64 torch view (aliasing the workspace) of the buffer to be summed over shards."""
        p = _dp()
        n = _i64()
        self._check(_lib.oid_partials(self.h, which, ctypes.byref(p), ctypes.byref(n)), "oid_partials")
        off = ctypes.cast(p, ctypes.c_void_p).value - self.ws.data_ptr()
        return self.ws[off:off + 8 * n.value].view(self._torch.float64)

    def estimate_begin(self):
        self._check(_lib.oid_estimate_begin(self.h, self._est()), "oid_estimate_begin")

    def estimate_end(self, out=None):
        ptr = ctypes.c_void_p(out.data_ptr()) if out is not None else ctypes.c_void_p()
        self._check(_lib.oid_estimate_end(self.h, ptr, self._est()), "oid_estimate_end")

    def error_estimate(self):
        out = (ctypes.c_double * 8)()
        self._check(_lib.oid_error_estimate(self.h, out, self._est()), "oid_error_estimate")
        v = list(out)
        return dict(e2=v[0], T=v[1], gpp=v[2], frob2=v[3], est_abs=v[4], est_rel=v[5], flags=int(v[6]), kappa=v[7])

    def gradient_gcv(self, mu):
        out = ctypes.c_double()
        self._check(_lib.oid_gradient_gcv(self.h, ctypes.c_double(mu), ctypes.byref(out), self._st()), "oid_gradient_gcv")
        return out.value

    def gradient_coefficients(self, mu):
        torch = self._torch
        n_obs = self.stats()["n_obs"]
        P = torch.empty((n_obs, self.p.k), dtype=torch.float64, device=self.device)   # column-major k x n_obs
        self._check(_lib.oid_gradient_coefficients(self.h, ctypes.c_double(mu), ctypes.c_void_p(P.data_ptr()), self._st()),
                    "oid_gradient_coefficients")
        self.stream.synchronize()
        return P.T

    def gradient_finalize(self, lo=-3.0, hi=3.0, tol=1e-3):
        torch = self._torch
        n_obs = self.stats()["n_obs"]
        P = torch.empty((n_obs, self.p.k), dtype=torch.float64, device=self.device)
        mu = ctypes.c_double()
        self._check(_lib.oid_gradient_finalize(self.h, ctypes.c_double(lo), ctypes.c_double(hi), ctypes.c_double(tol),
                                               ctypes.byref(mu), ctypes.c_void_p(P.data_ptr()), self._st()),
                    "oid_gradient_finalize")
        return mu.value, P.T

    def finalize(self, basis=False):
        torch = self._torch
        t = self.p.k
        J = np.empty(t, dtype=np.int64)
        n_obs = self.stats()["n_obs"]
        P = torch.empty((n_obs, t), dtype=torch.float64, device=self.device)   # column-major t x n_obs
        B = torch.empty((t, self.m_loc), dtype=self.dtype, device=self.device) if basis else None
        self._check(_lib.oid_finalize(self.h, ctypes.c_void_p(J.ctypes.data), ctypes.c_void_p(P.data_ptr()), 1,
                                      ctypes.c_void_p(B.data_ptr()) if basis else ctypes.c_void_p(), self._st()),
                    "oid_finalize")
        out = dict(J=J, P=P.T)
        if basis:
            out["basis"] = B.T
        return out

    def get(self, field):
        ell, t, bm = self.p.ell, self.p.k, self.p.b_max
        ga = (4 if self.p.grad_nz > 1 else 3) if self.p.grad_nfields > 0 else 1
        n_obs = self.stats()["n_obs"] if field == 2 else 0
        epochs = self.stats()["epochs"] if field == 14 else 0
        shapes = {0: ((t,), np.int64), 1: ((t,), np.float64), 2: ((n_obs, ell), np.float64),
                  3: ((ga * ell, ga * ell), np.float64), 4: ((8,), np.float64), 5: ((t + bm,), np.float64),
                  6: ((ga * ell,), np.float64), 7: (((ell + 1) * bm,), np.float64), 8: ((ell, t), np.float64),
                  9: ((3, 48), np.int32), 10: ((12, 4096), np.int64), 11: ((t, t), np.float64), 12: ((1024, 4), np.int64), 13: ((4096, 2), np.float64),
                  14: ((epochs, 6), np.float64), 15: ((256 * 32 + 8,), np.int32)}
        shape, dt = shapes[field]
        a = np.empty(shape, dtype=dt)
        self._check(_lib.oid_get(self.h, field, ctypes.c_void_p(a.ctypes.data), a.nbytes, self._st()), "oid_get")
        if field in (2, 3, 8):
            a = a.T   # stored column-major
        return a

    def J(self):
        return self.get(0)

    def scalars(self):
        v = self.get(4)
        return dict(frob2=v[0], lam=v[1], Ek=v[2], shift=v[3], trace=v[4], dmax=v[5], min_margin=v[6], kappa=v[7])

    def stats(self):
        s = OidStats()
        self._check(_lib.oid_stats(self.h, ctypes.byref(s)), "oid_stats")
        return {f: getattr(s, f) for f, _ in OidStats._fields_}

    def report(self):
        """Run report (include/oid.h oid_report): totals, per-epoch and per-estimate logs, as a dict."""
        import json
        need = ctypes.c_size_t()
        _lib.oid_report(self.h, None, 0, ctypes.byref(need), self._st())
        buf = ctypes.create_string_buffer(need.value)
        self._check(_lib.oid_report(self.h, buf, need.value, ctypes.byref(need), self._st()), "oid_report")
        return json.loads(buf.value.decode())

    def stats_reset(self):
        self._check(_lib.oid_stats_reset(self.h), "oid_stats_reset")

    def close(self):
        if getattr(self, "h", None):
            _lib.oid_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
