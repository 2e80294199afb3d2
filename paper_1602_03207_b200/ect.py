"""ctypes binding of the ectgpu C ABI (include/ectgpu.h).

This is the Python face of the drop-in boundary: the same entry points a
cgo/JNI/C++ caller would bind. It mirrors the reference's API names
(assemble_system/build_global -> Matrix, solve_iterative -> Matrix.solve,
ScanSession -> Session) and raises the reference's exception classes for the
ABI status codes (types.hpp:53-64). There is no CPU fallback: importing this
module on a host without the built library, or creating a Context without a
B200, fails loudly.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libectgpu.so"

D, I32, I64, U8 = C.c_double, C.c_int32, C.c_int64, C.c_uint8
VP = C.c_void_p


class EctError(RuntimeError):
    code = 1


class ConfigError(EctError):
    code = 2


class MeshError(EctError):
    code = 3


class SolverError(EctError):
    code = 4


class IoError(EctError):
    code = 5


class CudaError(EctError):
    code = 6


PRECOND = {"jacobi": 0, "amg": 1}

_ERRORS = {2: ConfigError, 3: MeshError, 4: SolverError, 5: IoError, 6: CudaError}


class Materials(C.Structure):
    """ect_materials == MaterialTable (materials.hpp:21-48)."""
    _fields_ = [("omega", D), ("sigma", D * 6), ("mu", D * 6), ("mu_tilde", D),
                ("delta_gauge", D), ("bc_penalty", D), ("sigma_eps", D),
                ("ibc_enabled", I32), ("l22_use_sigma_eps", I32), ("z_surface", D * 2)]


class Physics(C.Structure):
    """ect_physics == RunConfig [materials] (config.hpp:25-39); NaN = unset optional."""
    _fields_ = [("frequency", D), ("sigma_tube", D), ("mu_r_tube", D), ("sigma_defect", D),
                ("mu_r_defect", D), ("sigma_eps_ratio", D), ("delta_gauge", D),
                ("bc_penalty", D), ("mu_tilde_harmonic", I32), ("mu_tilde_fixed", D),
                ("sigma_tsp", D), ("mu_r_tsp", D), ("ibc_tsp", I32), ("l22_sigma_eps", I32)]

    @classmethod
    def defaults(cls) -> "Physics":
        """ect_physics_init: RunConfig's defaults."""
        ph = cls()
        lib().ect_physics_init(C.byref(ph))
        return ph


class Coil(C.Structure):
    _fields_ = [("r_inner", D), ("r_outer", D), ("height", D), ("gap", D)]


class IterOptions(C.Structure):
    _fields_ = [("tol", D), ("max_iter", I32), ("restart", I32)]


class IterResult(C.Structure):
    _fields_ = [("residual", D), ("iterations", I32), ("converged", I32)]


class SignalPoint(C.Structure):
    _fields_ = [("z", D), ("dz", D * 8), ("z_fa", D * 2), ("z_f3", D * 2), ("failed", I32),
                ("iterations", I32 * 4)]


class Timings(C.Structure):
    _fields_ = [("pattern_ms", D), ("assemble_ms", D), ("rhs_ms", D), ("solve_ms", D),
                ("spmv_ms_total", D), ("spmv_launches", I64), ("kernel_launches", I64),
                ("vec_ms_total", D), ("vec_launches", I64),
                ("spmv_partial_launches", I64), ("vec_partial_launches", I64),
                ("precond_ms_total", D), ("precond_launches", I64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"ectgpu library not built: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(str(LIB_PATH))
        L.ect_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().ect_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, EctError)(msg)


def _ptr(a):
    """Pointer of a numpy array (host) or a torch tensor (host or device)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _cvec(a, count, name, writable=False):
    """Validate a complex128 buffer of `count` elements, C-contiguous (numpy or
    torch, host or device); numpy inputs that are not are converted (inputs
    only). Buffers handed to the library as raw pointers must match exactly."""
    if hasattr(a, "data_ptr"):
        import torch
        if a.dtype != torch.complex128 or not a.is_contiguous() or a.numel() != count:
            raise ConfigError(f"{name}: need a contiguous complex128 tensor of {count} elements")
        return a
    if writable:
        if (not isinstance(a, np.ndarray) or a.dtype != np.complex128
                or not a.flags.c_contiguous or a.size != count or not a.flags.writeable):
            raise ConfigError(f"{name}: need a writable C-contiguous complex128 array of {count} elements")
        return a
    a = np.ascontiguousarray(a, np.complex128)
    if a.size != count:
        raise ConfigError(f"{name}: expected {count} complex values, got {a.size}")
    return a


def physics_struct(ph) -> Physics:
    """workloads.Physics -> ect_physics, starting from ect_physics_init's defaults.
    A negative / None optional (sigma_defect, mu_r_defect, sigma_tsp, mu_r_tsp)
    keeps the default (NaN = unset for the std::optional defect keys)."""
    if isinstance(ph, Physics):
        return ph
    out = Physics.defaults()
    for f, _ in Physics._fields_:
        if not hasattr(ph, f):
            continue
        v = getattr(ph, f)
        if f in ("sigma_defect", "mu_r_defect", "sigma_tsp", "mu_r_tsp") and (v is None or v < 0):
            continue
        setattr(out, f, int(v) if f in ("mu_tilde_harmonic", "ibc_tsp", "l22_sigma_eps") else v)
    return out


class Context:
    def __init__(self, device: int = 0):
        h = VP()
        _check(lib().ect_ctx_create(C.c_int(device), C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib().ect_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def timings(self, reset=False) -> dict:
        t = Timings()
        _check(lib().ect_ctx_timings(self.h, C.byref(t), C.c_int(int(reset))))
        return {f: getattr(t, f) for f, _ in Timings._fields_}

    def set_profiling(self, on: bool):
        _check(lib().ect_ctx_set_profiling(self.h, C.c_int(int(on))))

    def synchronize(self):
        _check(lib().ect_ctx_synchronize(self.h))

    def set_format(self, fmt: str):
        """SpMV storage of matrices assembled afterwards: 'nb' (default,
        sliced-ELL node blocks), 'sell' (SELL-32-sigma) or 'csr'."""
        _check(lib().ect_ctx_set_format(self.h, C.c_int({"nb": 0, "csr": 1, "sell": 3}[fmt])))

    def set_preconditioner(self, name: str):
        """Default preconditioner of matrices created afterwards: 'amg'
        (aggregation multigrid, the default) or 'jacobi'."""
        _check(lib().ect_ctx_set_preconditioner(self.h, I32(PRECOND[name])))

    def mark(self, slot: int):
        """Record event `slot` on the context stream (device-side timing)."""
        _check(lib().ect_ctx_mark(self.h, C.c_int(slot)))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = D()
        _check(lib().ect_ctx_elapsed_ms(self.h, C.c_int(a), C.c_int(b), C.byref(ms)))
        return ms.value


class Mesh:
    """Mesh + ConductorIndexMap + boundary pins, resident on the device."""

    def __init__(self, ctx: Context, xyz, tets, region):
        self.ctx = ctx
        xyz = np.ascontiguousarray(xyz, np.float64)
        tets = np.ascontiguousarray(tets, np.int32)
        region = np.ascontiguousarray(region, np.uint8)
        h = VP()
        _check(lib().ect_mesh_create(ctx.h, _ptr(xyz), I64(xyz.shape[0]), _ptr(tets),
                                     _ptr(region), I64(tets.shape[0]), C.byref(h)))
        self.h = h
        c = (I64 * 6)()
        _check(lib().ect_mesh_counts(h, c))
        (self.n_nodes, self.n_tets, self.n_cond, self.n_dofs, self.n_pins,
         self.n_defect) = list(c)

    @classmethod
    def from_gmsh(cls, ctx: Context, path):
        """load_mesh (mesh_io.cpp) + the GPU mesh: the file's validated boundary
        labels equal the geometric classification the device recomputes."""
        g = read_gmsh(path)
        return cls(ctx, g["xyz"], g["tets"], g["region"])

    def __del__(self, _lib=lib):
        if getattr(self, "h", None):
            _lib().ect_mesh_destroy(self.h)
            self.h = None

    def export(self):
        fwd = np.empty(self.n_nodes, np.int32)
        pins = np.empty(self.n_pins, np.int32)
        tets = np.empty((self.n_tets, 4), np.int32)
        _check(lib().ect_mesh_export(self.h, _ptr(fwd), _ptr(pins), _ptr(tets)))
        return {"cond_forward": fwd, "pinned_dofs": pins, "tets": tets}

    def materials(self, physics):
        p, r, two = Materials(), Materials(), I32()
        ph = physics_struct(physics)
        _check(lib().ect_materials_from_physics(self.h, C.byref(ph), C.byref(p), C.byref(r),
                                                C.byref(two)))
        return p, r, bool(two.value)

    def rhs(self, coil, z, which, amplitude, out=None):
        z = np.ascontiguousarray(np.atleast_1d(z), np.float64)
        which = np.ascontiguousarray(np.atleast_1d(which), np.int32)
        k = z.shape[0]
        if which.shape[0] != k:
            raise ConfigError(f"rhs: {k} probe positions but {which.shape[0]} coil indices")
        if out is None:
            out = np.empty((self.n_dofs, k), np.complex128)
        _cvec(out, self.n_dofs * k, "out", writable=True)
        cs = Coil(*coil)
        _check(lib().ect_rhs_coil(self.ctx.h, self.h, C.byref(cs), _ptr(z), _ptr(which), I32(k),
                                  D(amplitude), _ptr(out)))
        return out

    def rhs_support(self, support_tets, amplitude, out=None):
        """assemble_rhs(mesh, support_tets, amplitude, total_dofs) (assembly.cpp:335-378),
        not pinned (as the reference)."""
        sup = np.ascontiguousarray(np.atleast_1d(support_tets), np.int32)
        if out is None:
            out = np.empty(self.n_dofs, np.complex128)
        _cvec(out, self.n_dofs, "out", writable=True)
        _check(lib().ect_rhs_support(self.ctx.h, self.h, _ptr(sup), I64(sup.shape[0]),
                                     D(amplitude), _ptr(out)))
        return out

    def rhs_region(self, coil_tag, amplitude, out=None):
        """assemble_rhs(mesh, coil_tag, amplitude, total_dofs) (assembly.cpp:380-384)."""
        if out is None:
            out = np.empty(self.n_dofs, np.complex128)
        _cvec(out, self.n_dofs, "out", writable=True)
        _check(lib().ect_rhs_region(self.ctx.h, self.h, I32(coil_tag), D(amplitude), _ptr(out)))
        return out

    def apply_pins_to_rhs(self, rhs):
        """apply_pins_to_rhs (assembly.cpp:329-333) in place on [n] or [n, k]."""
        k = 1 if rhs.ndim == 1 else rhs.shape[1]
        _cvec(rhs, self.n_dofs * k, "rhs", writable=True)
        _check(lib().ect_apply_pins_to_rhs(self.ctx.h, self.h, _ptr(rhs), I32(k)))
        return rhs

    def delta_impedance(self, primary, reference, xk1, xk2, xl1, xl2):
        arrs = [np.ascontiguousarray(v, np.complex128) if not hasattr(v, "data_ptr") else v
                for v in (xk1, xk2, xl1, xl2)]
        dz = np.empty(8)
        _check(lib().ect_delta_impedance(self.ctx.h, self.h, C.byref(primary), C.byref(reference),
                                         *[_ptr(a) for a in arrs], _ptr(dz)))
        return dz.view(np.complex128)


class Matrix:
    """Global CSR system (pattern bit-identical to the reference CSC)."""

    def __init__(self, ctx: Context, mesh: Mesh | None = None, *, csr=None, csc=None):
        """From a mesh (K1 pattern; assemble() fills the values), or from
        external arrays: csr=(row_ptr, col_idx, values) or csc=(col_ptr,
        row_idx, values) = the reference's CscMatrix (sparse.hpp:56-66)."""
        self.ctx = ctx
        h = VP()
        ext = csr if csr is not None else csc
        if ext is not None:
            ptr, idx, val = (np.ascontiguousarray(ext[0], np.int32),
                             np.ascontiguousarray(ext[1], np.int32),
                             np.ascontiguousarray(ext[2], np.complex128))
            fn = lib().ect_matrix_from_csr if csr is not None else lib().ect_matrix_from_csc
            _check(fn(ctx.h, I64(ptr.shape[0] - 1), I64(idx.shape[0]), _ptr(ptr), _ptr(idx),
                      _ptr(val), C.byref(h)))
        else:
            _check(lib().ect_matrix_create(ctx.h, mesh.h, C.byref(h)))
        self.h = h
        self.mesh = mesh
        n, nnz = I64(), I64()
        _check(lib().ect_matrix_counts(h, C.byref(n), C.byref(nnz)))
        self.n, self.nnz = n.value, nnz.value

    def __del__(self, _lib=lib):
        if getattr(self, "h", None) and not getattr(self, "_borrowed", False):
            _lib().ect_matrix_destroy(self.h)
            self.h = None

    @property
    def symmetric(self) -> bool:
        v = I32()
        _check(lib().ect_matrix_symmetric(self.h, C.byref(v)))
        return bool(v.value)

    def set_preconditioner(self, name: str):
        _check(lib().ect_matrix_set_preconditioner(self.h, I32(PRECOND[name])))
        return self

    def precond_info(self) -> dict:
        """Multigrid hierarchy: levels, setup ms, operator complexity, coarsest n
        (builds it if needed; zeros for Jacobi)."""
        v = (D * 4)()
        _check(lib().ect_matrix_precond_info(self.h, v))
        return {"levels": int(v[0]), "setup_ms": v[1], "op_complexity": v[2],
                "coarsest_n": int(v[3])}

    def assemble(self, mats: Materials):
        _check(lib().ect_matrix_assemble(self.ctx.h, self.mesh.h, C.byref(mats), self.h))
        return self

    @property
    def format(self) -> str:
        nb = I32()
        _check(lib().ect_matrix_format(self.h, C.byref(nb)))
        return {0: "csr", 1: "nb", 3: "sell"}[nb.value]

    def nb_stats(self) -> dict:
        b, c = I64(), I64()
        _check(lib().ect_matrix_nb_counts(self.h, C.byref(b), C.byref(c)))
        return {"format": self.format, "blocks": b.value, "couplings": c.value}

    def export(self, values=True):
        rp = np.empty(self.n + 1, np.int32)
        ci = np.empty(self.nnz, np.int32)
        v = np.empty(self.nnz, np.complex128) if values else None
        _check(lib().ect_matrix_export(self.h, _ptr(rp), _ptr(ci), _ptr(v)))
        return rp, ci, v

    def export_csc(self):
        """The reference's CscMatrix arrays of build_global (col_ptr, row_idx, values)."""
        cp = np.empty(self.n + 1, np.int32)
        ri = np.empty(self.nnz, np.int32)
        v = np.empty(self.nnz, np.complex128)
        _check(lib().ect_matrix_export_csc(self.h, _ptr(cp), _ptr(ri), _ptr(v)))
        return cp, ri, v

    def multiply(self, x, out=None):
        """y = A x (CscMatrix::multiply); x is [n] or [n, k] interleaved."""
        k = 1 if x.ndim == 1 else x.shape[1]
        xs = _cvec(x, self.n * k, "x")
        if out is None:
            out = np.empty_like(xs) if not hasattr(xs, "data_ptr") else xs.new_empty(xs.shape)
        _cvec(out, self.n * k, "out", writable=True)
        _check(lib().ect_spmv(self.ctx.h, self.h, _ptr(xs), _ptr(out), I32(k)))
        return out

    def solve(self, b, tol=1e-8, max_iter=500, restart=80, out=None):
        """solve_iterative replacement: returns (x, [IterResult dicts])."""
        k = 1 if b.ndim == 1 else b.shape[1]
        bs = _cvec(b, self.n * k, "b")
        if out is None:
            out = np.empty_like(bs) if not hasattr(bs, "data_ptr") else bs.new_empty(bs.shape)
        _cvec(out, self.n * k, "out", writable=True)
        opts = IterOptions(tol, max_iter, restart)
        res = (IterResult * k)()
        _check(lib().ect_solve(self.ctx.h, self.h, _ptr(bs), _ptr(out), I32(k), C.byref(opts), res))
        return out, [{"iterations": r.iterations, "residual": r.residual,
                      "converged": bool(r.converged)} for r in res]


class Session:
    """ScanSession (scan.hpp:39-72) on the GPU."""

    def __init__(self, ctx: Context, mesh: Mesh, physics, coil, amplitude, tol=1e-8,
                 max_iter=20000, restart=80):
        self.ctx, self.mesh = ctx, mesh
        h = VP()
        ph = physics_struct(physics)
        cs = Coil(*coil)
        opts = IterOptions(tol, max_iter, restart)
        _check(lib().ect_session_create(ctx.h, mesh.h, C.byref(ph), C.byref(cs), D(amplitude),
                                        C.byref(opts), C.byref(h)))
        self.h = h

    def __del__(self, _lib=lib):
        if getattr(self, "h", None):
            _lib().ect_session_destroy(self.h)
            self.h = None

    def matrix(self, reference=False) -> Matrix:
        h = VP()
        _check(lib().ect_session_matrix(self.h, C.c_int(int(reference)), C.byref(h)))
        m = Matrix.__new__(Matrix)
        m.ctx, m.h, m.mesh, m._borrowed = self.ctx, h, self.mesh, True
        n, nnz = I64(), I64()
        _check(lib().ect_matrix_counts(h, C.byref(n), C.byref(nnz)))
        m.n, m.nnz = n.value, nnz.value
        return m

    def solve_positions(self, z, positions_per_batch=1, solutions=None):
        z = np.ascontiguousarray(np.atleast_1d(z), np.float64)
        pts = (SignalPoint * z.shape[0])()
        _check(lib().ect_session_solve_positions(self.h, _ptr(z), I32(z.shape[0]),
                                                 I32(positions_per_batch), pts, _ptr(solutions)))
        out = []
        for p in pts:
            dz = np.array(p.dz[:]).view(np.complex128)
            out.append({"z": p.z, "dz": dz, "z_fa": complex(p.z_fa[0], p.z_fa[1]),
                        "z_f3": complex(p.z_f3[0], p.z_f3[1]), "failed": bool(p.failed),
                        "iterations": list(p.iterations)})
        return out


# ---- Gmsh ASCII v2.2 files (load_mesh / write_mesh, mesh_io.hpp:30-38) -------------
def read_gmsh(path) -> dict:
    """Host-only reader: nodes, canonical tets, regions, labelled boundary faces
    (validated like the reference's load_mesh)."""
    h = VP()
    _check(lib().ect_gmsh_read(str(path).encode(), C.byref(h)))
    try:
        c = (I64 * 3)()
        _check(lib().ect_gmsh_counts(h, c))
        nn, nt, nf = list(c)
        out = {"xyz": np.empty((nn, 3), np.float64), "tets": np.empty((nt, 4), np.int32),
               "region": np.empty(nt, np.uint8), "faces": np.empty((nf, 3), np.int32),
               "labels": np.empty(nf, np.int32)}
        _check(lib().ect_gmsh_arrays(h, *[_ptr(out[k]) for k in
                                          ("xyz", "tets", "region", "faces", "labels")]))
        return out
    finally:
        lib().ect_gmsh_destroy(h)


def write_gmsh(path, xyz, tets, region, faces=None, labels=None):
    """write_mesh's format (%.17g coordinates, canonical tags)."""
    xyz = np.ascontiguousarray(xyz, np.float64)
    tets = np.ascontiguousarray(tets, np.int32)
    region = np.ascontiguousarray(region, np.uint8)
    faces = np.ascontiguousarray(np.zeros((0, 3)) if faces is None else faces, np.int32)
    labels = np.ascontiguousarray(np.zeros(0) if labels is None else labels, np.int32)
    _check(lib().ect_gmsh_write(str(path).encode(), _ptr(xyz), I64(xyz.shape[0]), _ptr(tets),
                                _ptr(region), I64(tets.shape[0]), _ptr(faces), _ptr(labels),
                                I64(labels.shape[0])))


# ---- distributed solve (row partition over GPUs) -------------------
class HaloPlan:
    """Host-only halo plan of one part (ect_halo_plan_*; no GPU needed)."""

    def __init__(self, n_nodes, nbr_off, nbr, cond_fwd, splits, part):
        nbr_off = np.ascontiguousarray(nbr_off, np.int32)
        nbr = np.ascontiguousarray(nbr, np.int32)
        cond_fwd = np.ascontiguousarray(cond_fwd, np.int32)
        splits = np.ascontiguousarray(splits, np.int64)
        h = VP()
        _check(lib().ect_halo_plan_create(I64(n_nodes), _ptr(nbr_off), _ptr(nbr), _ptr(cond_fwd),
                                          _ptr(splits), I32(len(splits) - 1), I32(part),
                                          C.byref(h)))
        self.h = h
        info = (I64 * 8)()
        _check(lib().ect_halo_plan_info(h, info))
        (self.n0, self.n1, self.L, self.G, self.c0, self.Vo, self.Vg, n_peers) = list(info)
        self.ghost_nodes = np.empty(self.G, np.int32)
        self.local_vdof = np.empty(self.L + self.G, np.int32)
        _check(lib().ect_halo_plan_arrays(h, _ptr(self.ghost_nodes), _ptr(self.local_vdof)))
        self.peers = []
        for i in range(n_peers):
            pi = (I64 * 7)()
            _check(lib().ect_halo_plan_peer(h, I32(i), pi, None, None))
            sn = np.empty(pi[5], np.int32)
            sc = np.empty(pi[6], np.int32)
            _check(lib().ect_halo_plan_peer(h, I32(i), pi, _ptr(sn), _ptr(sc)))
            self.peers.append({"part": pi[0], "recv_node_begin": pi[1], "recv_node_count": pi[2],
                               "recv_v_begin": pi[3], "recv_v_count": pi[4],
                               "send_nodes": sn, "send_cond_nodes": sc})

    def __del__(self, _lib=lib):
        if getattr(self, "h", None):
            _lib().ect_halo_plan_destroy(self.h)
            self.h = None


def comm_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().ect_comm_unique_id(buf))
    return bytes(buf)


class Comm:
    """NCCL communicator for one rank of the distributed solve."""

    def __init__(self, ctx: Context, rank: int, world: int, unique_id: bytes):
        h = VP()
        buf = (C.c_char * 128).from_buffer_copy(unique_id)
        _check(lib().ect_comm_create(ctx.h, I32(rank), I32(world), buf, C.byref(h)))
        self.h = h

    def __del__(self, _lib=lib):
        if getattr(self, "h", None):
            _lib().ect_comm_destroy(self.h)
            self.h = None


class Part:
    """Rows of nodes [splits[part], splits[part+1]) of an assembled matrix, or
    (matrix=None, mats=MaterialTable) assembled slab-locally without one."""

    def __init__(self, ctx: Context, mesh: Mesh, matrix: Matrix | None, splits, part: int,
                 mats: Materials | None = None):
        splits = np.ascontiguousarray(splits, np.int64)
        h = VP()
        if matrix is None:
            _check(lib().ect_part_create_assembled(ctx.h, mesh.h, C.byref(mats), _ptr(splits),
                                                   I32(len(splits) - 1), I32(part), C.byref(h)))
        else:
            _check(lib().ect_part_create(ctx.h, mesh.h, matrix.h, _ptr(splits),
                                         I32(len(splits) - 1), I32(part), C.byref(h)))
        self.h, self.ctx = h, ctx
        info = (I64 * 8)()
        _check(lib().ect_part_info(h, info))
        self.info = dict(zip(["n0", "n1", "L", "G", "Vo", "Vg", "n_peers", "n_blocks"], list(info)))

    def __del__(self, _lib=lib):
        if getattr(self, "h", None):
            _lib().ect_part_destroy(self.h)
            self.h = None


def dist_solve(parts, b, comm=None, tol=1e-8, max_iter=500, restart=80, out=None):
    """Partitioned Jacobi-COCG on global b ([n] or [n, k]); returns (x, results).
    comm=None runs every part in this process (one GPU); else one part/rank."""
    k = 1 if b.ndim == 1 else b.shape[1]
    bs = b if hasattr(b, "data_ptr") else np.ascontiguousarray(b, np.complex128)
    if out is None:
        out = np.zeros_like(bs) if not hasattr(b, "data_ptr") else b.new_zeros(b.shape)
    arr = (VP * len(parts))(*[p.h for p in parts])
    opts = IterOptions(tol, max_iter, restart)
    res = (IterResult * k)()
    _check(lib().ect_dist_solve(arr, I32(len(parts)), comm.h if comm else None, _ptr(bs), _ptr(out),
                                I32(k), C.byref(opts), res))
    return out, [{"iterations": r.iterations, "residual": r.residual,
                  "converged": bool(r.converged)} for r in res]
