"""B200-native (sm_100a, FP64) vertex-star FDM Schwarz relaxation.

Python mirror of the reference's public entry points for the Poisson/PCG hot
path (/root/reference/proj/include/fdmstar): problem setup (cartesian_mesh,
q_space, make_bundle, star_dofs / patch_ordering), the batched patch
factorisation (build_patch_solver), the relaxation (TwoLevel::smooth), the
V(1,1) cycle (TwoLevel::apply), the matrix-free operator
(GlobalOperator::apply), damping calibration and PCG.  Everything goes
through the C ABI of lib/libfdmgpu.so (include/fdmgpu.h); torch is only used
for device memory and streams.  There is no CPU fallback: without the
library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FDMGPU_LIB") or os.path.join(_HERE, "lib", "libfdmgpu.so")  # override: A/B builds
_lib = None

OP_APPLY_ST, OP_APPLY_S, OP_PATCH, OP_SMOOTH, OP_A, OP_VCYCLE = range(6)
STATUS = {0: "ok", 1: "invalid argument", 2: "matrix not SPD", 3: "indefinite operator", 4: "out of memory",
          5: "CUDA error", 6: "unsupported"}


class FdmGpuError(RuntimeError):
    """Raised for every non-OK fdmgpu status; .status holds the code."""

    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


class NotSPDError(FdmGpuError):
    pass


class IndefiniteError(FdmGpuError):
    pass


class Layout(C.Structure):
    _fields_ = [("npatch", C.c_int32), ("n", C.c_int32), ("n_interior", C.c_int32), ("n_interface", C.c_int32),
                ("tile", C.c_int32), ("tile_cols", C.c_int32), ("tiles", C.c_int32), ("pad_", C.c_int32),
                ("nnz_L", C.c_int64), ("flops_ref", C.c_int64), ("factor_bytes", C.c_int64),
                ("tile_gemms", C.c_int64), ("nnz_L_reference", C.c_int64), ("flops_reference", C.c_int64),
                ("separator_order", C.c_int32), ("top_direct", C.c_int32), ("stream_bytes", C.c_int64),
                ("dmma_flops", C.c_int64), ("schur_split", C.c_int32), ("n_top", C.c_int32),
                ("solve_values", C.c_int64)]


class KrylovReport(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("kappa", C.c_double),
                ("lambda_min", C.c_double), ("lambda_max", C.c_double), ("final_residual", C.c_double),
                ("wall_time", C.c_double)]


_vp = C.c_void_p


def lib():
    """Load lib/libfdmgpu.so (built by __graft_entry__.build()); raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FdmGpuError(5, f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.fdmgpu_last_error.restype = C.c_char_p
        L.fdmgpu_last_error.argtypes = [_vp]
        L.fdmhost_last_error.restype = C.c_char_p
        L.fdmhost_problem_create.restype = _vp
        L.fdmhost_problem_create.argtypes = [C.c_int, C.c_int, C.c_int]
        L.fdmhost_problem_destroy.argtypes = [_vp]
        L.fdmhost_elastic_create.restype = _vp
        L.fdmhost_elastic_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int]
        L.fdmhost_dg_create.restype = _vp
        L.fdmhost_dg_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int]
        L.fdmhost_problem_from_mesh_file.restype = _vp
        L.fdmhost_problem_from_mesh_file.argtypes = [C.c_char_p, C.c_int, C.c_uint64]
        L.fdmhost_problem_from_mesh.restype = _vp
        L.fdmhost_problem_from_mesh.argtypes = [C.c_int, C.c_int, _vp, C.c_int, _vp, C.c_int, _vp, _vp, _vp, C.c_int,
                                                C.c_uint64]
        L.fdmhost_save_mesh.argtypes = [_vp, C.c_char_p]
        L.fdmhost_problem_set_skip_boundary_patches.argtypes = [_vp, C.c_int]
        L.fdmhost_write_matrix_market.argtypes = [C.c_char_p, C.c_int64, C.c_int64, _vp, _vp, _vp, C.c_int]
        L.fdmgpu_patch_schur.argtypes = [_vp, C.c_int32, _vp]
        L.fdmgpu_patch_solve_one.argtypes = [_vp, C.c_int32, _vp, _vp]
        L.fdmgpu_patch_factor.argtypes = [_vp, C.c_int32, _vp]
        L.fdmgpu_set_separator_order.argtypes = [_vp, C.c_int32]
        L.fdmgpu_set_patches.argtypes = [_vp, C.c_int32, _vp, _vp, _vp, _vp, _vp]
        L.fdmhost_problem_info.argtypes = [_vp, _vp]
        L.fdmhost_get_rhs.argtypes = [_vp, _vp]
        L.fdmhost_get_maps.argtypes = [_vp] * 7
        L.fdmhost_get_geometry.argtypes = [_vp] * 6
        L.fdmhost_get_basis.argtypes = [_vp] * 11
        L.fdmhost_get_patches.argtypes = [_vp] * 7
        L.fdmhost_get_coarse.argtypes = [_vp] * 5
        L.fdmhost_attach.argtypes = [_vp, C.c_int, C.c_int, C.POINTER(_vp)]
        L.fdmgpu_destroy.argtypes = [_vp]
        L.fdmgpu_set_stream.argtypes = [_vp, _vp]
        L.fdmgpu_synchronize.argtypes = [_vp]
        L.fdmgpu_factor.argtypes = [_vp]
        L.fdmgpu_get_layout.argtypes = [_vp, C.POINTER(Layout)]
        L.fdmgpu_get_patch_elimination_dofs.argtypes = [_vp, _vp]
        L.fdmgpu_apply.argtypes = [_vp, C.c_int32, C.c_double, _vp, _vp, C.c_int32]
        L.fdmgpu_apply_async.argtypes = [_vp, C.c_int32, C.c_double, _vp, _vp]
        L.fdmgpu_async_join.argtypes = [_vp]
        L.fdmgpu_pcg.argtypes = [_vp, _vp, _vp, C.c_double, C.c_int32, C.c_int32, C.POINTER(KrylovReport), _vp]
        L.fdmgpu_calibrate_damping.argtypes = [_vp, C.c_int32, C.c_uint32, C.c_int32, C.POINTER(C.c_double),
                                               C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.fdmgpu_set_omega.argtypes = [_vp, C.c_double]
        L.fdmgpu_get_omega.argtypes = [_vp, C.POINTER(C.c_double)]
        L.fdmgpu_launch_count.restype = C.c_int64
        L.fdmgpu_launch_count.argtypes = [_vp]
        L.fdmgpu_kernel_timing.argtypes = [_vp, C.c_int32]
        L.fdmgpu_set_cell_coeffs.argtypes = [_vp, _vp, _vp, _vp, _vp]
        L.fdmgpu_create.argtypes = [C.POINTER(_vp), C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_int32]
        L.fdmgpu_kernel_time.argtypes = [_vp, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        _lib = L
    return _lib


def _host_chk(rc):
    if rc != 0:
        raise FdmGpuError(1, lib().fdmhost_last_error().decode())


def _ptr(a):
    return None if a is None else _vp(a.ctypes.data)


def write_matrix_market(path, A, symmetric=False):
    """write_matrix_market (src/sparse.cpp:33-52): A is a dense array or a scipy
    sparse matrix; stored in column-major order (explicit entries of a sparse
    matrix, nonzeros of a dense one); `symmetric` writes the lower triangle."""
    if hasattr(A, "tocsc"):
        M = A.tocsc()
        M.sort_indices()
        rows, cols = M.shape
        colptr, rowidx, val = M.indptr, M.indices, M.data
    else:
        D = np.asarray(A, np.float64)
        rows, cols = D.shape
        nzr, nzc = np.nonzero(D.T)  # column-major: (column, row) pairs, rows ascending per column
        colptr = np.zeros(cols + 1, np.int64)
        np.add.at(colptr, nzr + 1, 1)
        colptr = np.cumsum(colptr)
        rowidx, val = nzc, D[nzc, nzr]
    colptr = np.ascontiguousarray(colptr, np.int64)
    rowidx = np.ascontiguousarray(rowidx, np.int32)
    val = np.ascontiguousarray(val, np.float64)
    _host_chk(lib().fdmhost_write_matrix_market(os.fsencode(path), rows, cols, _ptr(colptr),
                                                _ptr(rowidx) if len(rowidx) else None,
                                                _ptr(val) if len(val) else None, 1 if symmetric else 0))


class Problem:
    """One synthetic configuration (BASELINE.json configs 1..5), optionally
    reduced to n cells per axis / degree p, built by the host setup mirror."""

    def __init__(self, config: int, n: int = 0, p: int = 0, _handle=None, skip_boundary_patches=True):
        L = lib()
        self.h = _handle if _handle is not None else L.fdmhost_problem_create(config, n, p)
        if not self.h:
            raise FdmGpuError(1, L.fdmhost_last_error().decode())
        if skip_boundary_patches is False:
            _host_chk(L.fdmhost_problem_set_skip_boundary_patches(self.h, 0))
        self.skip_boundary_patches = skip_boundary_patches is not False
        info = np.zeros(16, np.int64)
        _host_chk(L.fdmhost_problem_info(self.h, _ptr(info)))
        (self.dim, self.p, self.ncells, self.ndof, self.nfree, self.npatches, self.nvertices, self.npc,
         self.sum_nj, self.ncoarse, self.P_nnz, self.q, self.config, self.n, cart, self.ncomp) = (int(v) for v in info)
        self.all_cartesian = bool(cart)

    @classmethod
    def elasticity(cls, dim, n, p, mu=1.0, lam=0.0, skip_boundary_patches=False):
        """Linear elasticity (src/elasticity.cpp) on the reference's Table-2 problem
        (tests/test_elasticity.cpp:24-30, 162-185) in dim = 2|3: unit square/cube
        with n cells per axis, x = 0 Dirichlet, other boundary facets Neumann,
        vector Q_p, Lame mu / lam, body force -0.02 e_{dim-1}.  The Solver then
        runs build_elasticity_twolevel's path: true-form operator, SDC/FDM
        relaxation per component, vector Q1 coarse space.  skip_boundary_patches
        defaults to the reference's SolverConfig default (False)."""
        h = lib().fdmhost_elastic_create(int(dim), int(n), int(p), float(mu), float(lam),
                                         1 if skip_boundary_patches else 0)
        if not h:
            raise FdmGpuError(1, lib().fdmhost_last_error().decode())
        return cls(0, _handle=h, skip_boundary_patches=True if skip_boundary_patches else None)

    @classmethod
    def sipg(cls, dim, n, p, eta=-1.0, skip_boundary_patches=False):
        """Symmetric interior-penalty DG Poisson (src/sipg.cpp) on dq_space of the
        unit square / cube with n cells per axis, every boundary facet weak
        Dirichlet, penalty eta (< 0: sipg_default_eta = (p+1)(p+d)), RHS
        load_vector(f = 1).  The Solver then runs the two-level DG solver of
        tests/test_sipg.cpp:184-197: dg_poisson_operator as A, vertex-star
        patches of transformed_dg_poisson ((2p+2)^d DOFs) as the relaxation,
        continuous Q1 coarse level.  skip_boundary_patches defaults to the
        reference's SolverConfig default (False)."""
        h = lib().fdmhost_dg_create(int(dim), int(n), int(p), float(eta), 1 if skip_boundary_patches else 0)
        if not h:
            raise FdmGpuError(1, lib().fdmhost_last_error().decode())
        pb = cls(0, _handle=h, skip_boundary_patches=True if skip_boundary_patches else None)
        pb.dg = True
        pb.skip_boundary_patches = bool(skip_boundary_patches)
        return pb

    dg = False

    # ---- external meshes (the reference's mesh file format, src/mesh.cpp:354-434) ----
    TAGS = {"interior": 0, "dirichlet": 1, "neumann": 2}

    @classmethod
    def from_mesh_file(cls, path, p, seed=0, skip_boundary_patches=True):
        """Q_p problem on a mesh file written by the reference's save_mesh (JSON:
        dim, vertices, cells, facet_tags); unit coefficient, RHS U[-1,1] from
        std::mt19937_64(seed), zero on Dirichlet DOFs.  Raises FdmGpuError with
        the reference's load_mesh messages.  skip_boundary_patches=False adds the
        boundary-vertex stars (SolverConfig's default, src/schwarz.cpp:71-81)."""
        h = lib().fdmhost_problem_from_mesh_file(os.fsencode(path), int(p), int(seed))
        if not h:
            raise FdmGpuError(1, lib().fdmhost_last_error().decode())
        return cls(0, _handle=h, skip_boundary_patches=skip_boundary_patches)

    @classmethod
    def from_mesh(cls, dim, vertices, cells, p, facet_tags=(), seed=0, skip_boundary_patches=True):
        """Same from arrays: vertices (nv x dim), cells (nc x 2^dim, the reference's
        corner order), facet_tags [(cell, local_facet, 'dirichlet'|'neumann'|'interior')]."""
        v = np.zeros((len(vertices), 3))
        v[:, :dim] = np.asarray(vertices, np.float64)[:, :dim]
        c = np.ascontiguousarray(np.asarray(cells, np.int32))
        tc = np.array([t[0] for t in facet_tags], np.int32)
        tl = np.array([t[1] for t in facet_tags], np.int32)
        tk = np.array([cls.TAGS[t[2]] for t in facet_tags], np.int32)
        h = lib().fdmhost_problem_from_mesh(int(dim), len(v), _ptr(np.ascontiguousarray(v)), len(c), _ptr(c), len(tc),
                                            _ptr(tc) if len(tc) else None, _ptr(tl) if len(tl) else None,
                                            _ptr(tk) if len(tk) else None, int(p), int(seed))
        if not h:
            raise FdmGpuError(1, lib().fdmhost_last_error().decode())
        return cls(0, _handle=h, skip_boundary_patches=skip_boundary_patches)

    def save_mesh(self, path):
        """Write the mesh in the reference's JSON format (save_mesh)."""
        _host_chk(lib().fdmhost_save_mesh(self.h, os.fsencode(path)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.fdmhost_problem_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def rhs(self):
        out = np.zeros(self.ndof)
        _host_chk(lib().fdmhost_get_rhs(self.h, _ptr(out)))
        return out

    def maps(self):
        cd = np.zeros(self.ncells * self.npc, np.int32)
        cm = np.zeros_like(cd)
        con = np.zeros(self.ndof, np.uint8)
        mult = np.zeros(self.ndof)
        lc, le = np.zeros(self.ndof, np.int32), np.zeros(self.ndof, np.int32)
        _host_chk(lib().fdmhost_get_maps(self.h, _ptr(cd), _ptr(cm), _ptr(con), _ptr(mult), _ptr(lc), _ptr(le)))
        return dict(cell_dofs=cd.reshape(self.ncells, self.npc), cell_modes=cm.reshape(self.ncells, self.npc),
                    constrained=con, multiplicity=mult, label_cls=lc, label_entity=le)

    def geometry(self):
        v = np.zeros(self.nvertices * 3)
        k = np.zeros(self.ncells)
        mu = np.zeros(self.ncells * self.dim)
        kind = np.zeros(self.ncells, np.uint8)
        xyz = np.zeros(self.ncells * (1 << self.dim) * 3)
        _host_chk(lib().fdmhost_get_geometry(self.h, _ptr(v), _ptr(k), _ptr(mu), _ptr(kind), _ptr(xyz)))
        return dict(vertices=v.reshape(-1, 3), kappa=k, mu=mu.reshape(self.ncells, self.dim), kind=kind,
                    corner_xyz=xyz.reshape(self.ncells, 1 << self.dim, 3))

    def basis(self):
        n = self.p + 1
        S, At, Bt, Ah, Bh = (np.zeros(n * n) for _ in range(5))
        Anz, Bnz = np.zeros(n * n, np.uint8), np.zeros(n * n, np.uint8)
        lam, par, nodes = np.zeros(max(self.p - 1, 1)), np.zeros(n), np.zeros(n)
        _host_chk(lib().fdmhost_get_basis(self.h, _ptr(S), _ptr(At), _ptr(Bt), _ptr(Anz), _ptr(Bnz), _ptr(lam),
                                          _ptr(par), _ptr(Ah), _ptr(Bh), _ptr(nodes)))
        f = lambda a: a.reshape(n, n, order="F")
        return dict(S=f(S), At=f(At), Bt=f(Bt), Atnz=f(Anz).astype(bool), Btnz=f(Bnz).astype(bool),
                    lam=lam[: self.p - 1], parity=par, A_hat=f(Ah), B_hat=f(Bh), nodes=nodes)

    def patches(self):
        vert = np.zeros(self.npatches, np.int32)
        ptr = np.zeros(self.npatches + 1, np.int64)
        dofs, perm = np.zeros(self.sum_nj, np.int32), np.zeros(self.sum_nj, np.int32)
        cells = np.zeros(self.npatches * (1 << self.dim), np.int32)
        colour = np.zeros(self.npatches, np.int32)
        _host_chk(lib().fdmhost_get_patches(self.h, _ptr(vert), _ptr(ptr), _ptr(dofs), _ptr(perm), _ptr(cells),
                                            _ptr(colour)))
        return dict(vertex=vert, ptr=ptr, dofs=dofs, perm=perm, cells=cells.reshape(self.npatches, -1),
                    colour=colour)

    def coarse(self):
        inv = np.zeros(self.ncoarse * self.ncoarse)
        ptr = np.zeros(self.ndof + 1, np.int64)
        col, val = np.zeros(self.P_nnz, np.int32), np.zeros(self.P_nnz)
        _host_chk(lib().fdmhost_get_coarse(self.h, _ptr(inv), _ptr(ptr), _ptr(col), _ptr(val)))
        return dict(inverse=inv.reshape(self.ncoarse, self.ncoarse), P_ptr=ptr, P_col=col, P_val=val)


class Solver:
    """GPU handle for one Problem: the device-side TwoLevel / PatchSolver.

    Vector arguments are either torch CUDA float64 tensors (device path) or
    numpy float64 arrays (host path: copied in and out inside the call, the
    LinOp drop-in of src/krylov.hpp:10)."""

    def __init__(self, problem: Problem, device: int = 0, stream=None, separator_order: str = "plane"):
        self.problem = problem
        self.ndof = problem.ndof
        h = _vp()
        order = {"plane": 0, "reference": 1}[separator_order]
        rc = lib().fdmhost_attach(problem.h, device, order, C.byref(h))
        if rc != 0:
            raise FdmGpuError(rc, lib().fdmhost_last_error().decode())
        self.h = h
        self._stream = None  # CUDA stream handle the library runs on (None: its own)
        if stream is not None:
            self.set_stream(stream)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            try:
                _lib.fdmgpu_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def _chk(self, rc):
        if rc != 0:
            msg = lib().fdmgpu_last_error(self.h).decode()
            cls = NotSPDError if rc == 2 else IndefiniteError if rc == 3 else FdmGpuError
            raise cls(rc, msg)

    def set_stream(self, stream):
        """Run on a caller's CUDA stream (e.g. torch.cuda.current_stream())."""
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self._chk(lib().fdmgpu_set_stream(self.h, _vp(handle)))
        self._stream = handle

    def _enter(self, t):
        """Order the library's stream after torch's producer of `t`; returns
        True when the call must be synchronised afterwards (different streams)."""
        import torch
        cur = torch.cuda.current_stream(t.device)
        if cur.cuda_stream == self._stream:
            return False
        cur.synchronize()
        return True

    def synchronize(self):
        self._chk(lib().fdmgpu_synchronize(self.h))

    def factor(self):
        """Batched numeric factorisation of all patches (build_patch_solver)."""
        self._chk(lib().fdmgpu_factor(self.h))

    def set_cell_coeffs(self, mu, kind=None, corner_xyz=None, kappa=None):
        """Replace the per-cell coefficients (ncells x dim kappa*mu^K; invalidates the factor)."""
        g = self.problem.geometry()
        kind = g["kind"] if kind is None else np.ascontiguousarray(kind, np.uint8)
        xyz = np.ascontiguousarray(g["corner_xyz"] if corner_xyz is None else corner_xyz, np.float64)
        kap = np.ascontiguousarray(g["kappa"] if kappa is None else kappa, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        self._chk(lib().fdmgpu_set_cell_coeffs(self.h, _ptr(kind), _ptr(mu), _ptr(xyz), _ptr(kap)))

    def set_patches(self, separator_order=None, patches=None):
        """Re-feed the patch lists (fdmgpu_set_patches; invalidates the factor),
        optionally under another separator order ("plane" | "reference") or
        from explicit lists (dict as Problem.patches() returns)."""
        if separator_order is not None:
            self._chk(lib().fdmgpu_set_separator_order(self.h, {"plane": 0, "reference": 1}[separator_order]))
        pt = self.problem.patches() if patches is None else patches
        arrs = [np.ascontiguousarray(pt["vertex"], np.int32), np.ascontiguousarray(pt["ptr"], np.int64),
                np.ascontiguousarray(pt["dofs"], np.int32), np.ascontiguousarray(pt["perm"], np.int32),
                np.ascontiguousarray(pt["cells"], np.int32)]
        self._chk(lib().fdmgpu_set_patches(self.h, len(arrs[0]), *(_ptr(a) for a in arrs)))

    def layout(self):
        L = Layout()
        self._chk(lib().fdmgpu_get_layout(self.h, C.byref(L)))
        return {k: getattr(L, k) for k, _ in Layout._fields_ if not k.startswith("pad")}

    def elimination_dofs(self):
        L = self.layout()
        out = np.zeros(L["npatch"] * L["n"], np.int32)
        self._chk(lib().fdmgpu_get_patch_elimination_dofs(self.h, _ptr(out)))
        return out.reshape(L["npatch"], L["n"])

    def patch_schur(self, j):
        """Separator Schur complement of patch j (dense m x m, this handle's separator order)."""
        m = self.layout()["n_interface"]
        out = np.zeros((m, m), order="F")
        self._chk(lib().fdmgpu_patch_schur(self.h, int(j), _ptr(out)))
        return out

    def patch_factor(self, j):
        """Separator Cholesky factor L of patch j (dense m x m lower; S_G = L L^T)."""
        m = self.layout()["n_interface"]
        out = np.zeros((m, m), order="F")
        self._chk(lib().fdmgpu_patch_factor(self.h, int(j), _ptr(out)))
        return out

    def patch_solve_one(self, j, rj):
        """x_j = A~_j^{-1} r_j for patch j alone (CholFactor::solve, src/cholesky.cpp:89-110);
        rj / x_j in the order of the patch's ascending star_dofs."""
        rj = np.ascontiguousarray(rj, np.float64)
        out = np.zeros_like(rj)
        self._chk(lib().fdmgpu_patch_solve_one(self.h, int(j), _ptr(rj), _ptr(out)))
        return out

    def export_patch_matrix(self, j, path):
        """Debug dump of patch j's separator Schur complement in MatrixMarket
        (symmetric, lower triangle), as write_matrix_market writes it."""
        write_matrix_market(path, self.patch_schur(j), symmetric=True)

    def launch_count(self):
        return int(lib().fdmgpu_launch_count(self.h))

    KERNEL_CLASSES = {"patch_solve": 0, "factor": 1, "transform": 2, "stiffness": 3, "top_block": 4}

    def kernel_timing(self, enable=True):
        """Start (and clear) or stop CUDA-event timing of the library's kernels."""
        self._chk(lib().fdmgpu_kernel_timing(self.h, 1 if enable else 0))

    def kernel_time(self, which):
        """(total ms, launches) recorded for a kernel class since kernel_timing(True)."""
        t, n = C.c_double(), C.c_int64()
        self._chk(lib().fdmgpu_kernel_time(self.h, self.KERNEL_CLASSES.get(which, which), C.byref(t), C.byref(n)))
        return t.value, n.value

    # ---- operators ---------------------------------------------------------
    def apply(self, op, x, out=None, omega=0.0):
        if isinstance(x, np.ndarray):
            x = np.ascontiguousarray(x, np.float64)
            out = np.zeros(self.ndof) if out is None else out
            self._chk(lib().fdmgpu_apply(self.h, op, omega, _ptr(x), _ptr(out), 1))
            return out
        import torch
        assert x.is_cuda and x.dtype == torch.float64 and x.is_contiguous()
        out = torch.empty_like(x) if out is None else out
        sync = self._enter(x)
        self._chk(lib().fdmgpu_apply(self.h, op, omega, _vp(x.data_ptr()), _vp(out.data_ptr()), 0))
        if sync:
            self.synchronize()
        return out

    def apply_async(self, op, host_in, host_out, omega=0.0):
        """fdmgpu_apply_async: host_in / host_out pinned float64 arrays (e.g.
        torch.empty(n, dtype=torch.float64).pin_memory().numpy()), left untouched
        until synchronize(); copies overlap the compute of neighbouring calls."""
        assert host_in.dtype == np.float64 and host_out.dtype == np.float64
        assert host_in.flags.c_contiguous and host_out.flags.c_contiguous
        assert host_in.size == self.ndof and host_out.size == self.ndof
        self._chk(lib().fdmgpu_apply_async(self.h, op, omega, _ptr(host_in), _ptr(host_out)))

    def async_join(self):
        """fdmgpu_async_join: the library stream waits for all apply_async copy-outs."""
        self._chk(lib().fdmgpu_async_join(self.h))

    def apply_St(self, x, out=None):
        return self.apply(OP_APPLY_ST, x, out)

    def apply_S(self, x, out=None):
        return self.apply(OP_APPLY_S, x, out)

    def patch_apply(self, x, out=None):
        return self.apply(OP_PATCH, x, out)

    def smooth(self, x, out=None):
        return self.apply(OP_SMOOTH, x, out)

    def apply_A(self, x, out=None):
        return self.apply(OP_A, x, out)

    def vcycle(self, x, out=None, omega=None):
        return self.apply(OP_VCYCLE, x, out, self.omega if omega is None else omega)

    @property
    def omega(self):
        w = C.c_double()
        self._chk(lib().fdmgpu_get_omega(self.h, C.byref(w)))
        return w.value

    @omega.setter
    def omega(self, w):
        self._chk(lib().fdmgpu_set_omega(self.h, float(w)))

    def calibrate_damping(self, lanczos_steps=10, seed=0x5EED, formula=0):
        w, lo, hi = C.c_double(), C.c_double(), C.c_double()
        self._chk(lib().fdmgpu_calibrate_damping(self.h, lanczos_steps, seed, formula, C.byref(w), C.byref(lo),
                                                 C.byref(hi)))
        return dict(omega=w.value, lambda_min=lo.value, lambda_max=hi.value)

    def pcg(self, b, x=None, rtol=1e-8, maxit=200, precond=2):
        """pcg (src/krylov.cpp:29-83): b, x torch CUDA tensors; precond 0/1/2 =
        identity / smooth / V(1,1) cycle.  Returns (x, report dict)."""
        import torch
        x = torch.empty_like(b) if x is None else x
        sync = self._enter(b)
        rep = KrylovReport()
        res = np.zeros(max(maxit, 1))
        self._chk(lib().fdmgpu_pcg(self.h, _vp(b.data_ptr()), _vp(x.data_ptr()), rtol, maxit, precond,
                                   C.byref(rep), _ptr(res)))
        if sync:
            self.synchronize()
        d = {k: getattr(rep, k) for k, _ in KrylovReport._fields_}
        d["converged"] = bool(d["converged"])
        d["residuals"] = res[: rep.iterations].copy()
        return x, d
