"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the CPU oracle (liboracle.so).

The oracle is a plain-C++ restatement of the reference fdmstar path (see
oracle/oracle.hpp).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module; the product
package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

_d = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32 = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build() -> str:
    """Compile the oracle (make -C oracle); returns the library path."""
    subprocess.run(["make", "-s", "-C", _HERE, "-j8"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_create.restype = C.c_void_p
        L.oracle_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.oracle_create_mesh.restype = C.c_void_p
        L.oracle_set_skip_boundary_patches.argtypes = [C.c_void_p, C.c_int]
        L.oracle_create_mesh.argtypes = [C.c_int, C.c_int, _d, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int, C.c_uint64, C.c_int, C.c_int]
        L.oracle_destroy.argtypes = [C.c_void_p]
        L.oracle_info.argtypes = [C.c_void_p, _i64]
        L.oracle_get_rhs.argtypes = [C.c_void_p, _d]
        L.oracle_get_maps.argtypes = [C.c_void_p, _i32, _i32, _u8, _d, _i32, _i32]
        L.oracle_get_geometry.argtypes = [C.c_void_p, _d, _d, _d]
        L.oracle_get_basis.argtypes = [C.c_void_p, _d, _d, _d, _u8, _u8, _d, _d]
        L.oracle_get_patches.argtypes = [C.c_void_p, _i32, _i64, _i32, _i32]
        L.oracle_patch_group_offsets.argtypes = [C.c_void_p, C.c_int, _i32, C.POINTER(C.c_int)]
        for nm in ("oracle_apply_St", "oracle_apply_S", "oracle_apply_A", "oracle_patch_apply",
                   "oracle_smooth", "oracle_vcycle"):
            getattr(L, nm).argtypes = [C.c_void_p, _d, _d]
        L.oracle_factor_patches.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.oracle_patch_factor_info.argtypes = [C.c_void_p, C.c_int, _i64]
        L.oracle_copy_factor.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.oracle_patch_factor_get.argtypes = [C.c_void_p, C.c_int, _i64, _i32, _d]
        L.oracle_patch_matrix.argtypes = [C.c_void_p, C.c_int, _i64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_patch_solve_one.argtypes = [C.c_void_p, C.c_int, _d, _d]
        L.oracle_build_twolevel.argtypes = [C.c_void_p, C.c_int]
        L.oracle_twolevel_info.argtypes = [C.c_void_p, _d]
        L.oracle_set_omega.argtypes = [C.c_void_p, C.c_double]
        L.oracle_prolongation.argtypes = [C.c_void_p, _i64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_pcg.argtypes = [C.c_void_p, _d, _d, C.c_double, C.c_int, _d, _d, C.c_int]
        L.oracle_load_vector_one.argtypes = [C.c_void_p, _d]
        L.oracle_cell_matrix_quadrature.argtypes = [C.c_void_p, C.c_int, _d]
        L.oracle_cell_sumfact_apply.argtypes = [C.c_void_p, C.c_int, _d, _d]
        L.oracle_gll_nodes.argtypes = [C.c_int, _d]
        L.oracle_gauss_legendre.argtypes = [C.c_int, _d, _d]
        L.oracle_legendre.argtypes = [C.c_int, C.c_double, _d]
        L.oracle_reference_operators.argtypes = [C.c_int, C.c_int, _d, _d, _d, _d]
        L.oracle_fdm_basis.argtypes = [C.c_int, C.c_int, _d, _d, _d, _d, _u8, _u8, _d]
        L.oracle_dense_sym_gen_eig.argtypes = [C.c_int, _d, _d, _d, _d]
        L.oracle_cholesky_dense.argtypes = [C.c_int, _d, _i32, C.c_void_p, _i64, C.c_void_p, C.c_void_p]
        L.oracle_patch_ordering.argtypes = [C.c_int, _i32, _i32, _i32, _i32, C.POINTER(C.c_int)]
        L.oracle_tridiag_extremes.argtypes = [C.c_int, _d, _d, _d]
        L.oracle_pcg_dense.argtypes = [C.c_int, _d, C.c_void_p, _d, C.c_double, C.c_int, _d, _d]
        L.oracle_estimate_damping_dense.argtypes = [C.c_int, _d, _d, _d]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _chk(rc):
    if rc != 0:
        raise OracleError(lib().oracle_last_error().decode())


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---- stateless pins ---------------------------------------------------------
def gll_nodes(p):
    out = np.zeros(p + 1)
    _chk(lib().oracle_gll_nodes(p, out))
    return out


def gauss_legendre(n):
    pts, wts = np.zeros(n), np.zeros(n)
    _chk(lib().oracle_gauss_legendre(n, pts, wts))
    return pts, wts


def legendre(k, x):
    out = np.zeros(2)
    _chk(lib().oracle_legendre(k, float(x), out))
    return out[0], out[1]


def reference_operators(p, kind=0):
    n = p + 1
    A, B, nodes, tv = np.zeros(n * n), np.zeros(n * n), np.zeros(n), np.zeros(2 * n)
    _chk(lib().oracle_reference_operators(p, kind, A, B, nodes, tv))
    f = lambda a: a.reshape(n, n, order="F")
    return f(A), f(B), nodes, tv.reshape(2, n, order="F")


def fdm_basis(p, kind=0):
    n = p + 1
    S, lam, At, Bt = np.zeros(n * n), np.zeros(max(p - 1, 0) + 1), np.zeros(n * n), np.zeros(n * n)
    Anz, Bnz, par = np.zeros(n * n, np.uint8), np.zeros(n * n, np.uint8), np.zeros(n)
    _chk(lib().oracle_fdm_basis(p, kind, S, lam, At, Bt, Anz, Bnz, par))
    f = lambda a: a.reshape(n, n, order="F")
    return dict(S=f(S), lam=lam[: p - 1], At=f(At), Bt=f(Bt), Atnz=f(Anz).astype(bool),
                Btnz=f(Bnz).astype(bool), parity=par)


def dense_sym_gen_eig(A, B):
    n = A.shape[0]
    lam, V = np.zeros(n), np.zeros(n * n)
    _chk(lib().oracle_dense_sym_gen_eig(n, np.asfortranarray(A).ravel(order="K").copy(),
                                        np.asfortranarray(B).ravel(order="K").copy(), lam, V))
    return lam, V.reshape(n, n, order="F")


def cholesky_dense(A, perm=None, b=None):
    """Returns (L dense, nnz, flops, x or None); raises OracleError naming the pivot."""
    n = A.shape[0]
    perm = np.arange(n, dtype=np.int32) if perm is None else np.ascontiguousarray(perm, np.int32)
    L = np.zeros(n * n)
    info = np.zeros(2, np.int64)
    x = None if b is None else np.zeros(n)
    bb = None if b is None else np.ascontiguousarray(b, np.float64)
    _chk(lib().oracle_cholesky_dense(n, np.asfortranarray(A).ravel(order="F").copy(), perm, _ptr(L), info,
                                     _ptr(bb), _ptr(x)))
    return L.reshape(n, n, order="F"), int(info[0]), int(info[1]), x


def patch_ordering(cls, ent):
    n = len(cls)
    perm, offs = np.zeros(n, np.int32), np.zeros(n + 2, np.int32)
    cnt = C.c_int(0)
    _chk(lib().oracle_patch_ordering(n, np.ascontiguousarray(cls, np.int32), np.ascontiguousarray(ent, np.int32),
                                     perm, offs, C.byref(cnt)))
    return perm, offs[: cnt.value]


def tridiag_extremes(diag, off):
    out = np.zeros(2)
    d = np.ascontiguousarray(diag, np.float64)
    o = np.ascontiguousarray(off, np.float64) if len(off) else np.zeros(1)
    _chk(lib().oracle_tridiag_extremes(len(d), d, o, out))
    return out[0], out[1]


def pcg_dense(A, b, rtol, maxit, P=None):
    n = A.shape[0]
    x, rep = np.zeros(n), np.zeros(6)
    Pm = None if P is None else np.asfortranarray(P).ravel(order="F").copy()
    _chk(lib().oracle_pcg_dense(n, np.asfortranarray(A).ravel(order="F").copy(), _ptr(Pm),
                                np.ascontiguousarray(b, np.float64), rtol, maxit, x, rep))
    return x, dict(iterations=int(rep[0]), converged=bool(rep[1]), kappa=rep[2], lambda_min=rep[3],
                   lambda_max=rep[4])


def estimate_damping_dense(A, P):
    n = A.shape[0]
    out = np.zeros(3)
    _chk(lib().oracle_estimate_damping_dense(n, np.asfortranarray(A).ravel(order="F").copy(),
                                             np.asfortranarray(P).ravel(order="F").copy(), out))
    return dict(omega=out[0], lambda_min=out[1], lambda_max=out[2])


# ---- problem-level ----------------------------------------------------------
class Problem:
    """One synthetic configuration (1..5), optionally reduced (n cells/axis, degree p)."""

    def __init__(self, config, n=0, p=0, build_global=True, threads=1, _handle=None, skip_boundary_patches=True):
        L = lib()
        self.h = _handle if _handle is not None else L.oracle_create(config, n, p, 1 if build_global else 0, threads)
        if not self.h:
            raise OracleError(L.oracle_last_error().decode())
        if not skip_boundary_patches:  # [ext] the reference default (src/schwarz.cpp:71-81)
            _chk(L.oracle_set_skip_boundary_patches(self.h, 0))
        info = np.zeros(10, np.int64)
        _chk(L.oracle_info(self.h, info))
        (self.dim, self.p, self.ncells, self.ndof, self.nfree, self.npatches, self.nvertices,
         self.npc, self.sum_nj, self.config) = (int(v) for v in info)
        self.threads = threads
        self._twolevel = False

    TAGS = {"interior": 0, "dirichlet": 1, "neumann": 2}

    @classmethod
    def from_mesh(cls, dim, vertices, cells, p, facet_tags=(), seed=0, build_global=True, threads=1,
                  skip_boundary_patches=True):
        """[ext] Problem on an external mesh (load_mesh data), RHS U[-1,1] from seed."""
        v = np.zeros((len(vertices), 3))
        v[:, :dim] = np.asarray(vertices, np.float64)[:, :dim]
        c = np.ascontiguousarray(np.asarray(cells, np.int32))
        tc = np.array([t[0] for t in facet_tags], np.int32)
        tl = np.array([t[1] for t in facet_tags], np.int32)
        tk = np.array([cls.TAGS[t[2]] for t in facet_tags], np.int32)
        addr = lambda a: a.ctypes.data if len(a) else None
        h = lib().oracle_create_mesh(int(dim), len(v), np.ascontiguousarray(v), len(c), c.ctypes.data, len(tc),
                                     addr(tc), addr(tl), addr(tk), int(p), int(seed), 1 if build_global else 0, threads)
        if not h:
            raise OracleError(lib().oracle_last_error().decode())
        return cls(0, p=p, build_global=build_global, threads=threads, _handle=h,
                   skip_boundary_patches=skip_boundary_patches)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.oracle_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def rhs(self):
        out = np.zeros(self.ndof)
        _chk(lib().oracle_get_rhs(self.h, out))
        return out

    def maps(self):
        cd = np.zeros(self.ncells * self.npc, np.int32)
        cm = np.zeros_like(cd)
        con = np.zeros(self.ndof, np.uint8)
        mult = np.zeros(self.ndof)
        lc, le = np.zeros(self.ndof, np.int32), np.zeros(self.ndof, np.int32)
        _chk(lib().oracle_get_maps(self.h, cd, cm, con, mult, lc, le))
        return dict(cell_dofs=cd.reshape(self.ncells, self.npc), cell_modes=cm.reshape(self.ncells, self.npc),
                    constrained=con, multiplicity=mult, label_cls=lc, label_entity=le)

    def geometry(self):
        v = np.zeros(self.nvertices * 3)
        k = np.zeros(self.ncells)
        mu = np.zeros(self.ncells * self.dim)
        _chk(lib().oracle_get_geometry(self.h, v, k, mu))
        return dict(vertices=v.reshape(-1, 3), kappa=k, mu=mu.reshape(self.ncells, self.dim))

    def basis(self):
        n = self.p + 1
        S, At, Bt = np.zeros(n * n), np.zeros(n * n), np.zeros(n * n)
        Anz, Bnz = np.zeros(n * n, np.uint8), np.zeros(n * n, np.uint8)
        lam, par = np.zeros(max(self.p - 1, 1)), np.zeros(n)
        _chk(lib().oracle_get_basis(self.h, S, At, Bt, Anz, Bnz, lam, par))
        f = lambda a: a.reshape(n, n, order="F")
        return dict(S=f(S), At=f(At), Bt=f(Bt), Atnz=f(Anz).astype(bool), Btnz=f(Bnz).astype(bool),
                    lam=lam[: self.p - 1], parity=par)

    def patches(self):
        vert = np.zeros(self.npatches, np.int32)
        ptr = np.zeros(self.npatches + 1, np.int64)
        dofs = np.zeros(self.sum_nj, np.int32)
        perm = np.zeros(self.sum_nj, np.int32)
        _chk(lib().oracle_get_patches(self.h, vert, ptr, dofs, perm))
        return dict(vertex=vert, ptr=ptr, dofs=dofs, perm=perm)

    def group_offsets(self, j):
        cnt = C.c_int(0)
        _chk(lib().oracle_patch_group_offsets(self.h, j, np.zeros(1, np.int32), C.byref(cnt)) if False else 0)
        buf = np.zeros(4096, np.int32)
        _chk(lib().oracle_patch_group_offsets(self.h, j, buf, C.byref(cnt)))
        return buf[: cnt.value].copy()

    def _vop(self, name, x):
        out = np.zeros(self.ndof)
        _chk(getattr(lib(), name)(self.h, np.ascontiguousarray(x, np.float64), out))
        return out

    def apply_St(self, x):
        return self._vop("oracle_apply_St", x)

    def apply_S(self, x):
        return self._vop("oracle_apply_S", x)

    def apply_A(self, x):
        return self._vop("oracle_apply_A", x)

    def patch_apply(self, x):
        return self._vop("oracle_patch_apply", x)

    def smooth(self, x):
        return self._vop("oracle_smooth", x)

    def vcycle(self, x):
        return self._vop("oracle_vcycle", x)

    def factor(self, idx=None, threads=None):
        threads = threads or self.threads
        if idx is None:
            _chk(lib().oracle_factor_patches(self.h, None, 0, threads))
        else:
            a = np.ascontiguousarray(idx, np.int32)
            _chk(lib().oracle_factor_patches(self.h, a.ctypes.data_as(C.c_void_p), len(a), threads))

    def copy_factor(self, src, dst):
        """Timing harness only: patch dst solves with a copy of patch src's factor."""
        _chk(lib().oracle_copy_factor(self.h, int(src), int(dst)))

    def factor_info(self, j):
        out = np.zeros(3, np.int64)
        _chk(lib().oracle_patch_factor_info(self.h, j, out))
        return dict(nnz=int(out[0]), flops=int(out[1]), n=int(out[2]))

    def factor_csc(self, j):
        info = self.factor_info(j)
        cp = np.zeros(info["n"] + 1, np.int64)
        ri = np.zeros(info["nnz"], np.int32)
        va = np.zeros(info["nnz"])
        _chk(lib().oracle_patch_factor_get(self.h, j, cp, ri, va))
        return cp, ri, va

    def patch_matrix(self, j):
        nnz = np.zeros(1, np.int64)
        _chk(lib().oracle_patch_matrix(self.h, j, nnz, None, None, None))
        n = int(self.patches_n(j))
        ptr = np.zeros(n + 1, np.int64)
        col = np.zeros(int(nnz[0]), np.int32)
        val = np.zeros(int(nnz[0]))
        _chk(lib().oracle_patch_matrix(self.h, j, nnz, ptr.ctypes.data_as(C.c_void_p),
                                       col.ctypes.data_as(C.c_void_p), val.ctypes.data_as(C.c_void_p)))
        return ptr, col, val

    def patches_n(self, j):
        if not hasattr(self, "_pt"):
            self._pt = self.patches()
        return self._pt["ptr"][j + 1] - self._pt["ptr"][j]

    def patch_solve_one(self, j, rj):
        n = self.patches_n(j)
        out = np.zeros(n)
        _chk(lib().oracle_patch_solve_one(self.h, j, np.ascontiguousarray(rj, np.float64), out))
        return out

    def build_twolevel(self, calibrate=True):
        _chk(lib().oracle_build_twolevel(self.h, 1 if calibrate else 0))
        self._twolevel = True

    def twolevel_info(self):
        out = np.zeros(5)
        _chk(lib().oracle_twolevel_info(self.h, out))
        return dict(omega=out[0], lambda_min=out[1], lambda_max=out[2], coarse_ndof=int(out[3]),
                    prolong_nnz=int(out[4]))

    def set_omega(self, w):
        _chk(lib().oracle_set_omega(self.h, float(w)))

    def prolongation(self):
        nnz = np.zeros(1, np.int64)
        _chk(lib().oracle_prolongation(self.h, nnz, None, None, None))
        ptr = np.zeros(self.ndof + 1, np.int64)
        col = np.zeros(int(nnz[0]), np.int32)
        val = np.zeros(int(nnz[0]))
        _chk(lib().oracle_prolongation(self.h, nnz, ptr.ctypes.data_as(C.c_void_p), col.ctypes.data_as(C.c_void_p),
                                       val.ctypes.data_as(C.c_void_p)))
        return ptr, col, val

    def pcg(self, b, rtol=1e-8, maxit=200, precond=2):
        """pcg with A = GlobalOperator::apply; precond 0 identity, 1 smooth, 2 V-cycle."""
        x, rep, res = np.zeros(self.ndof), np.zeros(6), np.zeros(max(maxit, 1))
        _chk(lib().oracle_pcg(self.h, np.ascontiguousarray(b, np.float64), x, rtol, maxit, rep, res, precond))
        it = int(rep[0])
        return x, dict(iterations=it, converged=bool(rep[1]), kappa=rep[2], lambda_min=rep[3],
                       lambda_max=rep[4], wall_time=rep[5], residuals=res[:it].copy())

    def load_vector_one(self):
        out = np.zeros(self.ndof)
        _chk(lib().oracle_load_vector_one(self.h, out))
        return out

    def cell_matrix_quadrature(self, cell):
        out = np.zeros(self.npc * self.npc)
        _chk(lib().oracle_cell_matrix_quadrature(self.h, cell, out))
        return out.reshape(self.npc, self.npc, order="F")

    def cell_sumfact_apply(self, cell, u):
        out = np.zeros(self.npc)
        _chk(lib().oracle_cell_sumfact_apply(self.h, cell, np.ascontiguousarray(u, np.float64), out))
        return out


# ---- elasticity (oracle/elasticity.cpp, src/elasticity.cpp) -------------------
def _elastic_lib():
    L = lib()
    if not getattr(L, "_elastic_ready", False):
        L.oracle_elastic_last_error.restype = C.c_char_p
        L.oracle_elastic_create.restype = C.c_void_p
        L.oracle_elastic_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int]
        L.oracle_elastic_destroy.argtypes = [C.c_void_p]
        L.oracle_elastic_info.argtypes = [C.c_void_p, _i64]
        L.oracle_elastic_rhs.argtypes = [C.c_void_p, _d]
        L.oracle_elastic_random_free.argtypes = [C.c_void_p, C.c_uint64, _d]
        L.oracle_elastic_maps.argtypes = [C.c_void_p, _i32, _u8, _d]
        L.oracle_elastic_apply_A.argtypes = [C.c_void_p, _d, _d]
        L.oracle_elastic_build.argtypes = [C.c_void_p, C.c_int]
        L.oracle_elastic_twolevel_info.argtypes = [C.c_void_p, _d]
        L.oracle_elastic_set_omega.argtypes = [C.c_void_p, C.c_double]
        L.oracle_elastic_op.argtypes = [C.c_void_p, C.c_int, _d, _d]
        L.oracle_elastic_patches.argtypes = [C.c_void_p, _i64, _i32, _i32]
        L.oracle_elastic_assemble_dense.argtypes = [C.c_void_p, C.c_int, _d]
        L.oracle_elastic_cell_matrices.argtypes = [C.c_void_p, C.c_int, _d, _d]
        L.oracle_elastic_pcg.argtypes = [C.c_void_p, _d, _d, C.c_double, C.c_int, C.c_int, _d, _d]
        L.oracle_sdc_axis_coefficients.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, _d]
        L._elastic_ready = True
    return L


def _echk(rc):
    if rc != 0:
        raise OracleError(_elastic_lib().oracle_elastic_last_error().decode())


def sdc_axis_coefficients(comp, dim, mu, lam):
    out = np.zeros(dim)
    _echk(_elastic_lib().oracle_sdc_axis_coefficients(comp, dim, mu, lam, out))
    return out


class ElasticProblem:
    """Vector Q_p linear elasticity on the reference's Table-2 'table' mesh
    (unit square/cube, x = 0 Dirichlet, other boundary facets Neumann), with
    the SDC/FDM two-level solver of build_elasticity_twolevel."""

    OPS = {"apply_St": 0, "apply_S": 1, "patch": 2, "smooth": 3, "vcycle": 4}

    def __init__(self, dim, n, p, mu=1.0, lam=0.0, skip_boundary_patches=False, threads=1):
        L = _elastic_lib()
        self.h = L.oracle_elastic_create(dim, n, p, mu, lam, 1 if skip_boundary_patches else 0, threads)
        if not self.h:
            raise OracleError(L.oracle_elastic_last_error().decode())
        info = np.zeros(7, np.int64)
        _echk(L.oracle_elastic_info(self.h, info))
        self.dim, self.p, self.ncells, self.ndof, self.nsc, self.nfree, self.npc = (int(v) for v in info)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.oracle_elastic_destroy(self.h)
            self.h = None

    def rhs(self):
        out = np.zeros(self.ndof)
        _echk(_elastic_lib().oracle_elastic_rhs(self.h, out))
        return out

    def random_free(self, seed):
        out = np.zeros(self.ndof)
        _echk(_elastic_lib().oracle_elastic_random_free(self.h, seed, out))
        return out

    def maps(self):
        cd = np.zeros(self.ncells * self.npc, np.int32)
        con, mult = np.zeros(self.ndof, np.uint8), np.zeros(self.ndof)
        _echk(_elastic_lib().oracle_elastic_maps(self.h, cd, con, mult))
        return dict(cell_dofs=cd.reshape(self.ncells, self.npc), constrained=con, multiplicity=mult)

    def apply_A(self, x):
        out = np.zeros(self.ndof)
        _echk(_elastic_lib().oracle_elastic_apply_A(self.h, np.ascontiguousarray(x, np.float64), out))
        return out

    def build(self, calibrate=True):
        _echk(_elastic_lib().oracle_elastic_build(self.h, 1 if calibrate else 0))

    def twolevel_info(self):
        out = np.zeros(6)
        _echk(_elastic_lib().oracle_elastic_twolevel_info(self.h, out))
        return dict(omega=out[0], lambda_min=out[1], lambda_max=out[2], ncoarse=int(out[3]), npatches=int(out[4]),
                    sum_nj=int(out[5]))

    def set_omega(self, w):
        _echk(_elastic_lib().oracle_elastic_set_omega(self.h, float(w)))

    def op(self, name, x):
        out = np.zeros(self.ndof)
        _echk(_elastic_lib().oracle_elastic_op(self.h, self.OPS[name], np.ascontiguousarray(x, np.float64), out))
        return out

    def patches(self):
        info = self.twolevel_info()
        ptr = np.zeros(info["npatches"] + 1, np.int64)
        dofs, vert = np.zeros(info["sum_nj"], np.int32), np.zeros(info["npatches"], np.int32)
        _echk(_elastic_lib().oracle_elastic_patches(self.h, ptr, dofs, vert))
        return dict(ptr=ptr, dofs=dofs, vertex=vert)

    def assemble_dense(self, sdc_only=False):
        out = np.zeros(self.ndof * self.ndof)
        _echk(_elastic_lib().oracle_elastic_assemble_dense(self.h, 1 if sdc_only else 0, out))
        return out.reshape(self.ndof, self.ndof)

    def cell_matrices(self, cell):
        N = self.dim * self.npc
        kron, quad = np.zeros(N * N), np.zeros(N * N)
        _echk(_elastic_lib().oracle_elastic_cell_matrices(self.h, cell, kron, quad))
        return kron.reshape(N, N, order="F"), quad.reshape(N, N, order="F")

    def pcg(self, b, rtol=1e-8, maxit=600, precond=2):
        x, rep, res = np.zeros(self.ndof), np.zeros(5), np.zeros(max(maxit, 1))
        _echk(_elastic_lib().oracle_elastic_pcg(self.h, np.ascontiguousarray(b, np.float64), x, rtol, maxit, precond,
                                                rep, res))
        it = int(rep[0])
        return x, dict(iterations=it, converged=bool(rep[1]), kappa=rep[2], lambda_min=rep[3], lambda_max=rep[4],
                       residuals=res[:it].copy())


# ---- SIPG DG (oracle/sipg.cpp, src/sipg.cpp) ---------------------------------------
def _dg_lib():
    L = _elastic_lib()
    if not getattr(L, "_dg_ready", False):
        L.oracle_sipg_default_eta.restype = C.c_double
        L.oracle_sipg_default_eta.argtypes = [C.c_int, C.c_int]
        L.oracle_sipg_facet_matrices.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                                 C.c_int, _d, _d, _d, _d]
        L.oracle_dg_create.restype = C.c_void_p
        L.oracle_dg_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int]
        L.oracle_dg_destroy.argtypes = [C.c_void_p]
        L.oracle_dg_info.argtypes = [C.c_void_p, _i64]
        L.oracle_dg_rhs.argtypes = [C.c_void_p, _d]
        L.oracle_dg_dense.argtypes = [C.c_void_p, C.c_int, _d, _i32, _i32]
        L.oracle_dg_apply.argtypes = [C.c_void_p, C.c_int, _d, _d]
        L.oracle_dg_fdm_solve.argtypes = [C.c_void_p, _d, _d]
        L.oracle_dg_patch.argtypes = [C.c_void_p, C.c_int, _i64]
        L.oracle_dg_build.argtypes = [C.c_void_p, C.c_int]
        L.oracle_dg_pcg.argtypes = [C.c_void_p, _d, _d, C.c_double, C.c_int, _d]
        L.oracle_dg_op.argtypes = [C.c_void_p, C.c_int, _d, _d]
        L.oracle_dg_set_omega.argtypes = [C.c_void_p, C.c_double]
        L.oracle_dg_patches.argtypes = [C.c_void_p] * 6
        L._dg_ready = True
    return L


def sipg_default_eta(p, d):
    return _dg_lib().oracle_sipg_default_eta(p, d)


def sipg_facet_matrices(p, kind, mu0, mu1, eta, side0, side1):
    n = p + 1
    E, Ei, tv, td = np.zeros(n * n), np.zeros(4 * n * n), np.zeros(2 * n), np.zeros(2 * n)
    _echk(_dg_lib().oracle_sipg_facet_matrices(p, kind, mu0, mu1, eta, side0, side1, E, Ei, tv, td))
    f = lambda a, r, c: a.reshape(r, c, order="F")
    return f(E, n, n), f(Ei, 2 * n, 2 * n), f(tv, 2, n), f(td, 2, n)


class DGProblem:
    """SIPG Poisson on dq_space(cartesian_mesh(dim, n^dim), p), all boundary facets
    Dirichlet (weak), with the transformed system and the DG two-level solver."""

    def __init__(self, dim, n, p, eta=-1.0, skip_boundary_patches=False, threads=1):
        L = _dg_lib()
        self.h = L.oracle_dg_create(dim, n, p, eta, 1 if skip_boundary_patches else 0, threads)
        if not self.h:
            raise OracleError(L.oracle_elastic_last_error().decode())
        info = np.zeros(5, np.int64)
        _echk(L.oracle_dg_info(self.h, info))
        self.dim, self.p, self.ncells, self.ndof, self.npc = (int(v) for v in info)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.oracle_dg_destroy(self.h)
            self.h = None

    def rhs(self):
        out = np.zeros(self.ndof)
        _echk(_dg_lib().oracle_dg_rhs(self.h, out))
        return out

    def dense(self, transformed=False):
        n = self.ndof
        out, nnz, cls = np.zeros(n * n), np.zeros(n, np.int32), np.zeros(n, np.int32)
        _echk(_dg_lib().oracle_dg_dense(self.h, 1 if transformed else 0, out, nnz, cls))
        return out.reshape(n, n), nnz, cls

    def apply(self, which, x):
        out = np.zeros(self.ndof)
        _echk(_dg_lib().oracle_dg_apply(self.h, {"A": 0, "St": 1, "S": 2}[which],
                                        np.ascontiguousarray(x, np.float64), out))
        return out

    def fdm_solve(self, b):
        out = np.zeros(self.ndof)
        _echk(_dg_lib().oracle_dg_fdm_solve(self.h, np.ascontiguousarray(b, np.float64), out))
        return out

    def patch(self, v=-1):
        out = np.zeros(2, np.int64)
        _echk(_dg_lib().oracle_dg_patch(self.h, v, out))
        return dict(n=int(out[0]), nnz=int(out[1]))

    def build(self, calibrate=True):
        _echk(_dg_lib().oracle_dg_build(self.h, 1 if calibrate else 0))

    def op(self, which, x):
        """After build(): "patch" (PatchSolver::apply, modal), "smooth", "vcycle"."""
        out = np.zeros(self.ndof)
        _echk(_dg_lib().oracle_dg_op(self.h, {"patch": 0, "smooth": 1, "vcycle": 2}[which],
                                     np.ascontiguousarray(x, np.float64), out))
        return out

    def set_omega(self, w):
        _echk(_dg_lib().oracle_dg_set_omega(self.h, float(w)))

    def patches(self):
        """After build(): vertex, ptr, dofs and factor nnz of every patch."""
        cnt = np.zeros(2, np.int64)
        L = _dg_lib()
        _echk(L.oracle_dg_patches(self.h, cnt.ctypes.data_as(C.c_void_p), None, None, None, None))
        npch, tot = int(cnt[0]), int(cnt[1])
        vert, ptr = np.zeros(npch, np.int32), np.zeros(npch + 1, np.int64)
        dofs, nnz = np.zeros(tot, np.int32), np.zeros(npch, np.int64)
        _echk(L.oracle_dg_patches(self.h, cnt.ctypes.data_as(C.c_void_p), vert.ctypes.data_as(C.c_void_p),
                                  ptr.ctypes.data_as(C.c_void_p), dofs.ctypes.data_as(C.c_void_p),
                                  nnz.ctypes.data_as(C.c_void_p)))
        return dict(vertex=vert, ptr=ptr, dofs=dofs, nnz=nnz)

    def pcg(self, b, rtol=1e-8, maxit=200):
        x, rep = np.zeros(self.ndof), np.zeros(5)
        _echk(_dg_lib().oracle_dg_pcg(self.h, np.ascontiguousarray(b, np.float64), x, rtol, maxit, rep))
        return x, dict(iterations=int(rep[0]), converged=bool(rep[1]), kappa=rep[2], omega=rep[3],
                       npatches=int(rep[4]))
