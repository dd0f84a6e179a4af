"""B200-native optimized-Schwarz gravimetry solver (arXiv 2112.03851) -- thin Python binding.

Argument marshalling only: every step of the solve runs in libosm's CUDA
kernels (``csrc/``), behind the C ABI declared in ``include/osm.h``.  The names
mirror the C entry points.  There is no CPU fallback: if ``libosm.so`` is
missing or cannot load, importing this package raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OSM_LIB") or os.path.join(_HERE, "libosm.so")  # OSM_LIB: experiment builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libosm.so not built ({LIB_PATH}); run `python paper_2112_03851_b200/build.py`")
_lib = C.CDLL(LIB_PATH)

OSM_OK, OSM_ERR_INVALID_ARG, OSM_ERR_GRID_TOO_SMALL, OSM_ERR_ILL_POSED, OSM_ERR_PRECOND = 0, 1, 2, 3, 4
OSM_NOT_CONVERGED, OSM_ERR_DIVERGED, OSM_ERR_CUDA, OSM_ERR_NCCL, OSM_ERR_STATE = 5, 6, 7, 8, 9
STATUS_NAMES = {0: "OK", 1: "INVALID_ARG", 2: "GRID_TOO_SMALL", 3: "ILL_POSED", 4: "PRECOND", 5: "NOT_CONVERGED",
                6: "DIVERGED", 7: "CUDA", 8: "NCCL", 9: "STATE"}

# symbols declared in include/osm.h (checked by tests/test_abi.py)
ABI_SYMBOLS = ["osm_abi_version", "osm_last_error", "osm_nccl_unique_id", "osm_create", "osm_destroy",
               "osm_decompose", "osm_set_robin", "osm_assemble", "osm_upload_density", "osm_upload_density_device",
               "osm_solve", "osm_get_history", "osm_get_inner_iters", "osm_get_solution", "osm_get_local_solution",
               "osm_get_trace", "osm_get_csr", "osm_get_interface_map", "osm_get_interface_mass",
               "osm_set_kernel_timing", "osm_get_kernel_timing", "osm_get_traffic_model", "osm_get_launch_count", "osm_solve_batch",
               "osm_get_batch_history", "osm_get_batch_inner_iters", "osm_get_batch_local_solution",
               "osm_plan", "osm_set_robin2", "osm_get_interface_stiffness", "osm_rate_max", "osm_rate_curve",
               "osm_cmaes_create", "osm_cmaes_destroy", "osm_cmaes_ask", "osm_cmaes_tell", "osm_cmaes_state",
               "osm_cmaes_should_stop", "osm_gravity_z", "osm_set_spmv_variant", "osm_upload_load_vector", "osm_solve_batch2",
               "osm_set_row_order", "osm_hub_create", "osm_hub_destroy", "osm_cmaes_dims",
               "osm_cmaes_batch_optimize"]


class MeshDesc(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64), ("lx", C.c_double), ("ly", C.c_double),
                ("lz", C.c_double), ("order", C.c_int)]


class DistDesc(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("device", C.c_int), ("nccl_uid", C.c_void_p),
                ("stream", C.c_void_p), ("hub", C.c_void_p)]


class SolveOpts(C.Structure):
    _fields_ = [("tol_outer", C.c_double), ("max_outer", C.c_int), ("tol_inner", C.c_double), ("max_inner", C.c_int),
                ("warm_start", C.c_int), ("diverge_window", C.c_int)]


class Report(C.Structure):
    _fields_ = [("outer_iters", C.c_int), ("converged", C.c_int), ("h_final", C.c_double), ("seconds", C.c_double),
                ("inner_total", C.c_int64), ("inner_maxed", C.c_int)]


class PlanSide(C.Structure):
    _fields_ = [("iface", C.c_int), ("side", C.c_int), ("sub", C.c_int), ("remote", C.c_int), ("peer", C.c_int)]


class BatchReport(C.Structure):
    _fields_ = [("B", C.c_int), ("outer_max", C.c_int), ("n_converged", C.c_int), ("inner_total", C.c_int64),
                ("seconds", C.c_double)]


class KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("total_ms", C.c_double)]


_P = C.c_void_p
_pd = C.POINTER(C.c_double)
_pi32 = C.POINTER(C.c_int32)
_pi64 = C.POINTER(C.c_int64)
_pint = C.POINTER(C.c_int)
_sigs = {
    "osm_abi_version": (C.c_int, []),
    "osm_last_error": (C.c_char_p, []),
    "osm_nccl_unique_id": (C.c_int, [_P]),
    "osm_create": (C.c_int, [C.POINTER(MeshDesc), C.POINTER(DistDesc), C.POINTER(_P)]),
    "osm_destroy": (None, [_P]),
    "osm_decompose": (C.c_int, [_P, C.c_int]),
    "osm_set_robin": (C.c_int, [_P, _pd, _pd]),
    "osm_assemble": (C.c_int, [_P]),
    "osm_upload_density": (C.c_int, [_P, _pd, C.c_double]),
    "osm_upload_density_device": (C.c_int, [_P, C.c_void_p, C.c_double]),
    "osm_solve": (C.c_int, [_P, C.POINTER(SolveOpts), C.POINTER(Report)]),
    "osm_get_history": (C.c_int, [_P, _pd, C.c_int, _pint]),
    "osm_get_inner_iters": (C.c_int, [_P, _pi32, C.c_int, _pint]),
    "osm_get_solution": (C.c_int, [_P, _pd, _pi64]),
    "osm_get_local_solution": (C.c_int, [_P, C.c_int, _pd, _pi64]),
    "osm_get_trace": (C.c_int, [_P, C.c_int, C.c_int, _pd, _pi64]),
    "osm_get_csr": (C.c_int, [_P, C.c_int, _pi64, _pi32, _pd, _pi64, _pi64]),
    "osm_get_interface_map": (C.c_int, [_P, C.c_int, C.c_int, _pi32, _pi64]),
    "osm_get_interface_mass": (C.c_int, [_P, _pi64, _pi32, _pd, _pi64, _pi64]),
    "osm_set_kernel_timing": (C.c_int, [_P, C.c_int]),
    "osm_get_kernel_timing": (C.c_int, [_P, C.POINTER(KernelTime), C.c_int, _pint]),
    "osm_get_traffic_model": (C.c_int, [_P, _pd, C.c_int]),
    "osm_get_launch_count": (C.c_int, [_P, _pi64]),
    "osm_solve_batch": (C.c_int, [_P, C.c_int, _pd, C.POINTER(SolveOpts), C.POINTER(BatchReport)]),
    "osm_get_batch_history": (C.c_int, [_P, C.c_int, _pd, C.c_int, _pint]),
    "osm_get_batch_inner_iters": (C.c_int, [_P, C.c_int, _pi32, C.c_int, _pint]),
    "osm_get_batch_local_solution": (C.c_int, [_P, C.c_int, C.c_int, _pd, _pi64]),
    "osm_set_robin2": (C.c_int, [_P, _pd, _pd, _pd, _pd]),
    "osm_get_interface_stiffness": (C.c_int, [_P, _pd, _pi64]),
    "osm_rate_max": (C.c_int, [C.c_double] * 6 + [C.c_int, _pd, _pd]),
    "osm_rate_curve": (C.c_int, [C.c_double] * 4 + [_pd, C.c_int, _pd]),
    "osm_cmaes_create": (C.c_int, [C.c_int, C.c_int, _pd, C.c_double, C.POINTER(_P)]),
    "osm_cmaes_destroy": (None, [_P]),
    "osm_cmaes_ask": (C.c_int, [_P, _pd, _pd]),
    "osm_cmaes_tell": (C.c_int, [_P, _pd]),
    "osm_cmaes_state": (C.c_int, [_P, _pd, _pd, _pd, _pd, _pd, _pint]),
    "osm_cmaes_should_stop": (C.c_int, [_P, C.c_int, C.c_double, _pint]),
    "osm_solve_batch2": (C.c_int, [_P, C.c_int, _pd, C.POINTER(SolveOpts), C.POINTER(BatchReport)]),
    "osm_upload_load_vector": (C.c_int, [_P, _pd, C.c_int64]),
    "osm_set_spmv_variant": (C.c_int, [_P, C.c_int, _pint]),
    "osm_set_row_order": (C.c_int, [_P, C.c_int]),
    "osm_gravity_z": (C.c_int, [_P, C.c_double, _pd, _pi64]),
    "osm_hub_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "osm_cmaes_dims": (None, [_P, _pint, _pint]),
    "osm_cmaes_batch_optimize": (C.c_int, [_P, _P, C.c_int, _pd, C.c_int, C.c_int, C.c_int, C.c_double, _pd, _pint]),
    "osm_hub_destroy": (None, [_P]),
    "osm_plan": (C.c_int, [C.c_int64, C.c_int, C.c_int, C.c_int, _pint, _pint, C.POINTER(PlanSide), C.c_int, _pint]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class OsmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(st, ok=(OSM_OK,)):
    if st not in ok:
        raise OsmError(st, _lib.osm_last_error().decode())
    return st


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def plan(nx, nsub, nranks, rank):
    """Host-only distribution plan: (s_begin, s_end, [dict(iface, side, sub, remote, peer), ...])."""
    sb, se, n = C.c_int(), C.c_int(), C.c_int()
    _check(_lib.osm_plan(nx, nsub, nranks, rank, C.byref(sb), C.byref(se), None, 0, C.byref(n)))
    arr = (PlanSide * max(1, n.value))()
    _check(_lib.osm_plan(nx, nsub, nranks, rank, C.byref(sb), C.byref(se), arr, n.value, C.byref(n)))
    return sb.value, se.value, [dict(iface=a.iface, side=a.side, sub=a.sub, remote=a.remote, peer=a.peer)
                                for a in arr[:n.value]]


def rate_max(p1, q1, p2, q2, kmin, kmax, nsamp=10000):
    """Fourier convergence-rate cost max_k rho(k) (osm_rate_max): (rho_max, argmax k)."""
    r, k = C.c_double(), C.c_double()
    _check(_lib.osm_rate_max(p1, q1, p2, q2, kmin, kmax, nsamp, C.byref(r), C.byref(k)))
    return r.value, k.value


def rate_curve(p1, q1, p2, q2, k):
    k = np.ascontiguousarray(k, dtype=np.float64)
    out = np.zeros_like(k)
    _check(_lib.osm_rate_curve(p1, q1, p2, q2, _ptr(k, C.c_double), k.size, _ptr(out, C.c_double)))
    return out


class CMAES:
    """Native CMA-ES (osm_cmaes_*): ask(z) with caller-supplied standard normals, tell(f)."""

    def __init__(self, mean, sigma0, lam=25):
        m = np.ascontiguousarray(mean, dtype=np.float64)
        self.n, self.lam = m.size, lam
        h = _P()
        _check(_lib.osm_cmaes_create(self.n, lam, _ptr(m, C.c_double), float(sigma0), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.osm_cmaes_destroy(self._h)
            self._h = None

    def ask(self, z):
        z = np.ascontiguousarray(z, dtype=np.float64).reshape(self.lam, self.n)
        x = np.zeros((self.lam, self.n))
        _check(_lib.osm_cmaes_ask(self._h, _ptr(z, C.c_double), _ptr(x, C.c_double)))
        return x

    def tell(self, f):
        f = np.ascontiguousarray(f, dtype=np.float64)
        _check(_lib.osm_cmaes_tell(self._h, _ptr(f, C.c_double)))

    def state(self):
        m, bx, cov = np.zeros(self.n), np.zeros(self.n), np.zeros((self.n, self.n))
        sig, bf, g = C.c_double(), C.c_double(), C.c_int()
        _check(_lib.osm_cmaes_state(self._h, _ptr(m, C.c_double), C.byref(sig), _ptr(cov, C.c_double),
                                    _ptr(bx, C.c_double), C.byref(bf), C.byref(g)))
        return dict(mean=m, sigma=sig.value, C=cov, best_x=bx, best_f=bf.value, generation=g.value)

    def optimize_batched(self, osm, z, n_outer=30, k0=5, max_iter=7200, ftol=5e-11):
        """CMA-ES over the batched-alpha solver of `osm` (osm_cmaes_batch_optimize): z is a (gens, lambda, n)
        array of standard normals; returns (costs [gens_done, lambda], gens_done)."""
        z = np.ascontiguousarray(z, dtype=np.float64).reshape(-1, self.lam, self.n)
        gens = z.shape[0]
        costs = np.zeros((gens, self.lam))
        done = C.c_int()
        _check(_lib.osm_cmaes_batch_optimize(osm._h, self._h, gens, _ptr(z, C.c_double), n_outer, k0, max_iter,
                                             float(ftol), _ptr(costs, C.c_double), C.byref(done)))
        return costs[: done.value], done.value

    def should_stop(self, max_iter=7200, ftol=5e-11):
        st = C.c_int()
        _check(_lib.osm_cmaes_should_stop(self._h, max_iter, ftol, C.byref(st)))
        return st.value


def cmaes_minimize(fun, mean, sigma0, z_stream, lam=25, max_iter=7200, ftol=5e-11):
    """ask/tell loop with the native CMA-ES; z_stream(g) -> lambda x n standard normals."""
    es = CMAES(mean, sigma0, lam)
    g = 0
    while True:
        X = es.ask(z_stream(g))
        es.tell([fun(x) for x in X])
        g += 1
        if es.should_stop(max_iter, ftol):
            break
    return es


def abi_version():
    return _lib.osm_abi_version()


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.osm_nccl_unique_id(buf))
    return buf.raw


class Hub:
    """In-process transport for `nranks` ranks that are threads of this process (osm_hub_create).

    Pass it as ``Osm(..., rank=r, nranks=n, hub=hub)`` from each rank's own thread; close it after
    every context attached to it is closed."""

    def __init__(self, nranks):
        h = _P()
        _check(_lib.osm_hub_create(nranks, C.byref(h)))
        self._h = h
        self.nranks = nranks

    def close(self):
        if getattr(self, "_h", None):
            _lib.osm_hub_destroy(self._h)
            self._h = None


class Osm:
    """One optimized-Schwarz context (one per process / GPU, or one per thread with a Hub).  Mirrors
    include/osm.h."""

    def __init__(self, nx, ny, nz, lx, ly, lz, order, rank=0, nranks=1, device=0, nccl_uid: bytes | None = None,
                 stream: int | None = None, hub: Hub | None = None):
        self.mesh = MeshDesc(nx, ny, nz, lx, ly, lz, order)
        self._uid = C.create_string_buffer(nccl_uid, 128) if nccl_uid else None
        dist = DistDesc(rank, nranks, device, C.cast(self._uid, C.c_void_p) if self._uid else None, stream,
                        hub._h if hub is not None else None)
        h = _P()
        _check(_lib.osm_create(C.byref(self.mesh), C.byref(dist), C.byref(h)))
        self._h = h
        self.order = order
        self.rank = rank
        self.nsub = 0
        self.lattice = (order * nx + 1, order * ny + 1, order * nz + 1)

    def close(self):
        if getattr(self, "_h", None):
            _lib.osm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- setup
    def decompose(self, nsub):
        _check(_lib.osm_decompose(self._h, int(nsub)))
        self.nsub = int(nsub)

    def set_robin(self, alpha_left, alpha_right):
        al = np.ascontiguousarray(alpha_left, dtype=np.float64)
        ar = np.ascontiguousarray(alpha_right, dtype=np.float64)
        if al.size != max(self.nsub - 1, 0) or ar.size != al.size:
            raise ValueError("need nsub-1 alphas per side")
        _check(_lib.osm_set_robin(self._h, _ptr(al, C.c_double), _ptr(ar, C.c_double)))

    def set_robin2(self, p_left, q_left, p_right, q_right):
        """OO2 transmission p M_Gamma + q S_Gamma per interface side (osm_set_robin2)."""
        n = max(self.nsub - 1, 0)
        arrs = [np.ascontiguousarray(np.broadcast_to(np.asarray(v, dtype=np.float64), (n,))) for v in
                (p_left, q_left, p_right, q_right)]
        _check(_lib.osm_set_robin2(self._h, *[_ptr(a, C.c_double) for a in arrs]))

    def interface_stiffness(self):
        nz = C.c_int64(0)
        _check(_lib.osm_get_interface_stiffness(self._h, None, C.byref(nz)))
        out = np.zeros(nz.value)
        _check(_lib.osm_get_interface_stiffness(self._h, _ptr(out, C.c_double), C.byref(nz)))
        return out

    def assemble(self):
        _check(_lib.osm_assemble(self._h))

    def upload_density(self, drho, G=6.672e-11):
        d = np.ascontiguousarray(drho, dtype=np.float64)
        if d.size != self.mesh.nx * self.mesh.ny * self.mesh.nz:
            raise ValueError("density must have nx*ny*nz cells")
        _check(_lib.osm_upload_density(self._h, _ptr(d, C.c_double), float(G)))

    def upload_load_vector(self, b_free):
        """Global free-DOF load vector (osm_upload_load_vector); interface rows split half/half."""
        b = np.ascontiguousarray(b_free, dtype=np.float64)
        _check(_lib.osm_upload_load_vector(self._h, _ptr(b, C.c_double), b.size))

    def upload_density_device(self, ptr: int, G=6.672e-11):
        _check(_lib.osm_upload_density_device(self._h, C.c_void_p(ptr), float(G)))

    # -- solve
    def solve(self, tol_outer=1e-8, max_outer=500, tol_inner=1e-10, max_inner=20000, warm_start=True,
              diverge_window=10):
        opts = SolveOpts(tol_outer, max_outer, tol_inner, max_inner, int(warm_start), diverge_window)
        rep = Report()
        st = _check(_lib.osm_solve(self._h, C.byref(opts), C.byref(rep)),
                    ok=(OSM_OK, OSM_NOT_CONVERGED, OSM_ERR_DIVERGED))
        return st, rep

    def solve_batch(self, alpha_left, alpha_right, tol_outer=1e-8, max_outer=500, tol_inner=1e-10, max_inner=20000,
                    warm_start=True):
        """Batched-alpha solve: alpha_left/right are (B, nsub-1) arrays.  Returns the report."""
        al = np.atleast_2d(np.asarray(alpha_left, dtype=np.float64))
        ar = np.atleast_2d(np.asarray(alpha_right, dtype=np.float64))
        B = al.shape[0]
        a = np.ascontiguousarray(np.stack([al, ar], axis=1))  # [b][side][iface]
        opts = SolveOpts(tol_outer, max_outer, tol_inner, max_inner, int(warm_start), 0)
        rep = BatchReport()
        _check(_lib.osm_solve_batch(self._h, B, _ptr(a, C.c_double), C.byref(opts), C.byref(rep)))
        return rep

    def solve_batch2(self, p_left, q_left, p_right, q_right, tol_outer=1e-8, max_outer=500, tol_inner=1e-10,
                     max_inner=20000, warm_start=True):
        """OO2 batched solve: each argument is a (B, nsub-1) array (osm_solve_batch2)."""
        arrs = [np.atleast_2d(np.asarray(v, dtype=np.float64)) for v in (p_left, q_left, p_right, q_right)]
        B = arrs[0].shape[0]
        pq = np.ascontiguousarray(np.stack(arrs, axis=1))  # [b][4][iface]
        opts = SolveOpts(tol_outer, max_outer, tol_inner, max_inner, int(warm_start), 0)
        rep = BatchReport()
        _check(_lib.osm_solve_batch2(self._h, B, _ptr(pq, C.c_double), C.byref(opts), C.byref(rep)))
        return rep

    def batch_history(self, b):
        n = C.c_int()
        _check(_lib.osm_get_batch_history(self._h, b, None, 0, C.byref(n)))
        out = np.zeros(n.value)
        _check(_lib.osm_get_batch_history(self._h, b, _ptr(out, C.c_double), n.value, C.byref(n)))
        return out

    def batch_inner_iters(self, b):
        n = C.c_int()
        _check(_lib.osm_get_batch_inner_iters(self._h, b, None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int32)
        _check(_lib.osm_get_batch_inner_iters(self._h, b, _ptr(out, C.c_int32), n.value, C.byref(n)))
        return out.reshape(-1, self.nsub)

    def batch_local_solution(self, b, s):
        n = C.c_int64(0)
        _check(_lib.osm_get_batch_local_solution(self._h, b, s, None, C.byref(n)))
        out = np.zeros(n.value)
        _check(_lib.osm_get_batch_local_solution(self._h, b, s, _ptr(out, C.c_double), C.byref(n)))
        return out

    # -- readback
    def history(self):
        n = C.c_int()
        _check(_lib.osm_get_history(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value)
        _check(_lib.osm_get_history(self._h, _ptr(out, C.c_double), n.value, C.byref(n)))
        return out

    def inner_iters(self):
        n = C.c_int()
        _check(_lib.osm_get_inner_iters(self._h, None, 0, C.byref(n)))
        out = np.zeros((n.value, self.nsub), dtype=np.int32)
        _check(_lib.osm_get_inner_iters(self._h, _ptr(out, C.c_int32), n.value, C.byref(n)))
        return out

    def solution(self, out=None):
        """[collective] Phi on the full lattice, gathered to rank 0 (other ranks get None)."""
        n = C.c_int64(int(np.prod(self.lattice)))
        if self.rank != 0:
            _check(_lib.osm_get_solution(self._h, None, C.byref(n)))
            return None
        if out is None:
            out = np.zeros(n.value)
        if out.dtype != np.float64 or not out.flags.c_contiguous or out.size < n.value:
            raise ValueError("out must be a contiguous float64 array of the lattice size")
        _check(_lib.osm_get_solution(self._h, _ptr(out, C.c_double), C.byref(n)))
        return out

    def gravity_z(self, z0):
        """[collective] g_z = -dPhi/dz on the plane z = z0 at the cell-centre columns (rank 0; else None)."""
        n = C.c_int64(self.mesh.nx * self.mesh.ny)
        if self.rank != 0:
            _check(_lib.osm_gravity_z(self._h, float(z0), None, C.byref(n)))
            return None
        out = np.zeros(n.value)
        _check(_lib.osm_gravity_z(self._h, float(z0), _ptr(out, C.c_double), C.byref(n)))
        return out

    def local_solution_size(self, s) -> int:
        n = C.c_int64(0)
        _check(_lib.osm_get_local_solution(self._h, s, None, C.byref(n)))
        return n.value

    def local_solution(self, s):
        n = C.c_int64(0)
        _check(_lib.osm_get_local_solution(self._h, s, None, C.byref(n)))
        out = np.zeros(n.value)
        _check(_lib.osm_get_local_solution(self._h, s, _ptr(out, C.c_double), C.byref(n)))
        return out

    def trace(self, iface, side):
        n = C.c_int64(0)
        _check(_lib.osm_get_trace(self._h, iface, side, None, C.byref(n)))
        out = np.zeros(n.value)
        _check(_lib.osm_get_trace(self._h, iface, side, _ptr(out, C.c_double), C.byref(n)))
        return out

    def csr(self, s):
        nr, nz = C.c_int64(0), C.c_int64(0)
        _check(_lib.osm_get_csr(self._h, s, None, None, None, C.byref(nr), C.byref(nz)))
        rp = np.zeros(nr.value + 1, dtype=np.int64)
        col = np.zeros(nz.value, dtype=np.int32)
        val = np.zeros(nz.value)
        _check(_lib.osm_get_csr(self._h, s, _ptr(rp, C.c_int64), _ptr(col, C.c_int32), _ptr(val, C.c_double),
                                C.byref(nr), C.byref(nz)))
        return rp, col, val

    def interface_map(self, iface, side):
        n = C.c_int64(0)
        _check(_lib.osm_get_interface_map(self._h, iface, side, None, C.byref(n)))
        out = np.zeros(n.value, dtype=np.int32)
        _check(_lib.osm_get_interface_map(self._h, iface, side, _ptr(out, C.c_int32), C.byref(n)))
        return out

    def interface_mass(self):
        nr, nz = C.c_int64(0), C.c_int64(0)
        _check(_lib.osm_get_interface_mass(self._h, None, None, None, C.byref(nr), C.byref(nz)))
        rp = np.zeros(nr.value + 1, dtype=np.int64)
        col = np.zeros(nz.value, dtype=np.int32)
        val = np.zeros(nz.value)
        _check(_lib.osm_get_interface_mass(self._h, _ptr(rp, C.c_int64), _ptr(col, C.c_int32), _ptr(val, C.c_double),
                                           C.byref(nr), C.byref(nz)))
        return rp, col, val

    # -- instrumentation
    def set_kernel_timing(self, enable: bool):
        _check(_lib.osm_set_kernel_timing(self._h, int(enable)))

    def kernel_timing(self):
        n = C.c_int()
        _check(_lib.osm_get_kernel_timing(self._h, None, 0, C.byref(n)))
        arr = (KernelTime * n.value)()
        _check(_lib.osm_get_kernel_timing(self._h, arr, n.value, C.byref(n)))
        return {a.name.decode(): (a.launches, a.total_ms) for a in arr}

    def set_spmv_variant(self, v: int) -> int:
        """Select the SpMV implementation (include/osm.h); returns the variant that will run."""
        a = C.c_int()
        _check(_lib.osm_set_spmv_variant(self._h, int(v), C.byref(a)))
        return a.value

    def set_row_order(self, order: int) -> None:
        """Internal row order of the GPU copy (include/osm.h); 4 enables the matrix-free SpMV (variant 5)."""
        _check(_lib.osm_set_row_order(self._h, int(order)))

    def launch_count(self) -> int:
        n = C.c_int64(0)
        _check(_lib.osm_get_launch_count(self._h, C.byref(n)))
        return n.value

    def traffic_model(self):
        out = np.zeros(8)
        _check(_lib.osm_get_traffic_model(self._h, _ptr(out, C.c_double), 8))
        return dict(spmv_bytes=out[0], update_bytes=out[1], dir_bytes=out[2], pad_entries=out[3], nnz=out[4],
                    rows=out[5], csr_equiv_bytes=out[6], exchange_bytes=out[7])


def setup(cfg: dict, drho, alpha=None, rank=0, nranks=1, device=0, nccl_uid=None, row_order=None,
          spmv=None, hub=None) -> Osm:
    """Create, decompose, assemble, set alpha (both sides) and upload the density of a config dict.
    row_order / spmv optionally select the internal row order and SpMV variant (row_order=4, spmv=5:
    the matrix-free Kuhn-stencil path)."""
    o = Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"], rank, nranks, device,
            nccl_uid, hub=hub)
    if row_order is not None:
        o.set_row_order(row_order)
    o.decompose(cfg["nsub"])
    if cfg["nsub"] > 1 and alpha is None and cfg.get("robin") is not None:
        n = cfg["nsub"] - 1
        p1, p2, q1, q2 = cfg["robin"]
        o.set_robin2(np.full(n, p1), np.full(n, q1), np.full(n, p2), np.full(n, q2))
    elif cfg["nsub"] > 1:
        a = cfg.get("alpha") if alpha is None else alpha
        n = cfg["nsub"] - 1
        if np.isscalar(a):
            al = ar = np.full(n, float(a))
        else:
            al = np.broadcast_to(np.asarray(a[0], dtype=np.float64), (n,))
            ar = np.broadcast_to(np.asarray(a[1], dtype=np.float64), (n,))
        o.set_robin(al, ar)
    o.assemble()
    if spmv is not None:
        o.set_spmv_variant(spmv)
    o.upload_density(drho)
    return o
