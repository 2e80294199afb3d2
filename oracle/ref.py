"""ctypes binding of oracle/_ref/libectref.so — TEST INFRASTRUCTURE ONLY.

The library is the UNMODIFIED ectsim reference core (compiled by
oracle/Makefile from /root/reference/proj/core/src against our Eigen-subset
shim) plus oracle/ref_driver.cpp. Only tests/, __graft_entry__.smoke() and
bench.py's reference / cpu_baseline legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_ref" / "libectref.so"
# the reference with binding/iterative_gpu.cpp in place of iterative.cpp
GPU_LIB_PATH = HERE / "_ref" / "libectref_gpu.so"
REFERENCE_SRC = Path("/root/reference/proj/core/src")

_lib = None


class RefError(RuntimeError):
    pass


class Materials(C.Structure):
    """Packed MaterialTable (materials.hpp:21-48)."""
    _fields_ = [("omega", C.c_double), ("sigma", C.c_double * 6), ("mu", C.c_double * 6),
                ("mu_tilde", C.c_double), ("delta_gauge", C.c_double),
                ("bc_penalty", C.c_double), ("sigma_eps", C.c_double),
                ("ibc_enabled", C.c_int32), ("l22_use_sigma_eps", C.c_int32),
                ("z_surface", C.c_double * 2)]


class Physics(C.Structure):
    _fields_ = [("frequency", C.c_double), ("sigma_tube", C.c_double), ("mu_r_tube", C.c_double),
                ("sigma_defect", C.c_double), ("mu_r_defect", C.c_double),
                ("sigma_eps_ratio", C.c_double), ("delta_gauge", C.c_double),
                ("bc_penalty", C.c_double), ("mu_tilde_harmonic", C.c_int32),
                ("mu_tilde_fixed", C.c_double), ("sigma_tsp", C.c_double),
                ("mu_r_tsp", C.c_double), ("ibc_tsp", C.c_int32)]


def build_if_possible() -> bool:
    """Compile _ref from the reference sources (only where they exist)."""
    if LIB_PATH.exists():
        return True
    if not REFERENCE_SRC.exists():
        return False
    subprocess.run(["make", "-C", str(HERE), "-j", str(os.cpu_count() or 4)], check=True,
                   stdout=subprocess.DEVNULL)
    return LIB_PATH.exists()


def available() -> bool:
    return LIB_PATH.exists()


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RefError(f"{LIB_PATH} not built (run make -C oracle)")
        _lib = C.CDLL(str(LIB_PATH))
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_signal_modes.restype = None
        _lib.ref_mesh_destroy.restype = None
        _lib.ref_system_destroy.restype = None
        assert _lib.ref_sizeof_materials() == C.sizeof(Materials)
    return _lib


def _check(rc):
    if rc != 0:
        raise RefError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


D = C.c_double
I32 = C.c_int32
I64 = C.c_int64


def physics_struct(ph) -> Physics:
    return Physics(ph.frequency, ph.sigma_tube, ph.mu_r_tube, ph.sigma_defect, ph.mu_r_defect,
                   ph.sigma_eps_ratio, ph.delta_gauge, ph.bc_penalty, int(ph.mu_tilde_harmonic),
                   ph.mu_tilde_fixed, ph.sigma_tsp, ph.mu_r_tsp,
                   int(getattr(ph, "ibc_tsp", False)))


class RefMesh:
    def __init__(self, xyz, tets, region):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        tets = np.ascontiguousarray(tets, dtype=np.int32)
        region = np.ascontiguousarray(region, dtype=np.uint8)
        h = C.c_void_p()
        _check(lib().ref_mesh_create(I64(xyz.shape[0]), _p(xyz, D), I64(tets.shape[0]),
                                     _p(tets, I32), _p(region, C.c_uint8), C.byref(h)))
        self.h = h
        nn, nt, nc, nf = I64(), I64(), I64(), I64()
        _check(lib().ref_mesh_counts(h, C.byref(nn), C.byref(nt), C.byref(nc), C.byref(nf)))
        self.n_nodes, self.n_tets, self.n_cond, self.n_faces = nn.value, nt.value, nc.value, nf.value

    @classmethod
    def _from_handle(cls, h):
        self = cls.__new__(cls)
        self.h = h
        nn, nt, nc, nf = I64(), I64(), I64(), I64()
        _check(lib().ref_mesh_counts(h, C.byref(nn), C.byref(nt), C.byref(nc), C.byref(nf)))
        self.n_nodes, self.n_tets, self.n_cond, self.n_faces = nn.value, nt.value, nc.value, nf.value
        return self

    @classmethod
    def tube(cls, spec: dict):
        """generate_tube_mesh (tube_mesh.cpp:85-270) for a TubeMeshSpec given as a
        dict with the tube_mesh.hpp:35-57 field names (AnnularBox / CoilPair as
        4-tuples; absent optionals unset)."""
        nan = float("nan")
        box = lambda k: list(spec[k]) if spec.get(k) is not None else [nan] * 4
        p = np.array([spec["domain_radius"], spec["z_min"], spec["z_max"], spec["tube_r_inner"],
                      spec["tube_r_outer"], spec.get("tube_z_min", nan), spec.get("tube_z_max", nan),
                      *box("tsp"), *box("defect"), *spec["coil"], spec.get("coil_ref_z", 0.0),
                      spec.get("resolution", 8), spec.get("outer_radial_grading", 2.0)], np.float64)
        scan = np.ascontiguousarray(spec.get("scan_z", ()), np.float64)
        h = C.c_void_p()
        _check(lib().ref_tube_mesh_create(_p(p, D), _p(scan, D) if scan.size else None,
                                          I32(scan.size), C.byref(h)))
        return cls._from_handle(h)

    @classmethod
    def load(cls, path):
        """load_mesh (mesh_io.cpp): Gmsh ASCII 2.2, canonical tag map."""
        h = C.c_void_p()
        _check(lib().ref_mesh_load(str(path).encode(), C.byref(h)))
        return cls._from_handle(h)

    def write(self, path):
        """write_mesh (mesh_io.cpp)."""
        _check(lib().ref_mesh_write(self.h, str(path).encode()))

    def geometry(self):
        xyz = np.empty((self.n_nodes, 3), np.float64)
        region = np.empty(self.n_tets, np.uint8)
        _check(lib().ref_mesh_geometry(self.h, _p(xyz, D), _p(region, C.c_uint8)))
        return xyz, region

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_mesh_destroy(self.h)
            self.h = None

    def export(self):
        tets = np.empty((self.n_tets, 4), np.int32)
        fwd = np.empty(self.n_nodes, np.int32)
        faces = np.empty((self.n_faces, 3), np.int32)
        labels = np.empty(self.n_faces, np.int32)
        _check(lib().ref_mesh_export(self.h, _p(tets, I32), _p(fwd, I32), _p(faces, I32),
                                     _p(labels, I32)))
        return {"tets": tets, "cond_forward": fwd, "faces": faces, "face_labels": labels}

    def materials(self, physics):
        p, r, two = Materials(), Materials(), I32()
        ph = physics_struct(physics)
        _check(lib().ref_materials_from_physics(self.h, C.byref(ph), C.byref(p), C.byref(r),
                                                C.byref(two)))
        return p, r, bool(two.value)

    def coil_support(self, coil, z, which):
        coil = np.ascontiguousarray(coil, np.float64)
        out = np.empty(self.n_tets, np.int32)
        cnt = I64()
        _check(lib().ref_coil_support(self.h, _p(coil, D), D(z), I32(which), _p(out, I32),
                                      C.byref(cnt)))
        return out[:cnt.value].copy()

    def delta_impedance(self, primary, reference, x_k, x_l):
        out = np.empty(2)
        _check(lib().ref_delta_impedance(self.h, C.byref(primary), C.byref(reference),
                                         _p(np.ascontiguousarray(x_k, np.complex128), D),
                                         _p(np.ascontiguousarray(x_l, np.complex128), D),
                                         _p(out, D)))
        return complex(out[0], out[1])


class RefSystem:
    """assemble_system + apply_essential_bc + build_global (scan.cpp:52-59)."""

    def __init__(self, mesh: RefMesh, mats: Materials, parts=1, workers=1, seed=0):
        h = C.c_void_p()
        t = np.zeros(4)
        _check(lib().ref_assemble(mesh.h, C.byref(mats), I32(parts), I32(workers), C.c_uint32(seed),
                                  C.byref(h), _p(t, D)))
        self.h = h
        self.mesh = mesh
        self.timings = {"assemble": t[0], "reduce": t[1], "bc": t[2], "build_global": t[3]}
        n, nnz, npins = I64(), I64(), I64()
        _check(lib().ref_system_counts(h, C.byref(n), C.byref(nnz), C.byref(npins)))
        self.n, self.nnz, self.n_pins = n.value, nnz.value, npins.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_system_destroy(self.h)
            self.h = None

    def export(self):
        col_ptr = np.empty(self.n + 1, np.int32)
        row_idx = np.empty(self.nnz, np.int32)
        vals = np.empty(self.nnz, np.complex128)
        pins = np.empty(self.n_pins, np.int32)
        _check(lib().ref_system_export(self.h, _p(col_ptr, I32), _p(row_idx, I32), _p(vals, D),
                                       _p(pins, I32)))
        return col_ptr, row_idx, vals, pins

    def multiply(self, x, repeat=1):
        x = np.ascontiguousarray(x, np.complex128)
        y = np.empty_like(x)
        s = D()
        _check(lib().ref_multiply(self.h, _p(x, D), _p(y, D), I32(repeat), C.byref(s)))
        return y, s.value

    def position_rhs(self, coil, z, which, amplitude):
        coil = np.ascontiguousarray(coil, np.float64)
        b = np.empty(self.n, np.complex128)
        _check(lib().ref_position_rhs(self.mesh.h, self.h, _p(coil, D), D(z), I32(which),
                                      D(amplitude), _p(b, D)))
        return b

    def solve_iterative(self, b, tol=1e-8, max_iter=500, restart=80):
        b = np.ascontiguousarray(b, np.complex128)
        x = np.empty_like(b)
        it, res, conv, sec = I32(), D(), I32(), D()
        _check(lib().ref_solve_iterative(self.h, _p(b, D), D(tol), I32(max_iter), I32(restart),
                                         _p(x, D), C.byref(it), C.byref(res), C.byref(conv),
                                         C.byref(sec)))
        return {"x": x, "iterations": it.value, "residual": res.value,
                "converged": bool(conv.value), "seconds": sec.value}

    def solve_iterative_batch(self, bs, tol, max_iter, restart, threads, want_x=False):
        bs = np.ascontiguousarray(bs, np.complex128)
        k = bs.shape[0]
        x = np.empty_like(bs) if want_x else None
        it = np.empty(k, np.int32)
        res = np.empty(k)
        sec = D()
        _check(lib().ref_solve_iterative_batch(
            self.h, _p(bs, D), I32(k), D(tol), I32(max_iter), I32(restart), I32(threads),
            _p(x, D) if want_x else None, _p(it, I32), _p(res, D), C.byref(sec)))
        return {"x": x, "iterations": it, "residual": res, "seconds": sec.value}

    def solve_direct(self, bs):
        bs = np.ascontiguousarray(np.atleast_2d(bs), np.complex128)
        x = np.empty_like(bs)
        res = np.empty(bs.shape[0])
        _check(lib().ref_solve_direct(self.h, _p(bs, D), I32(bs.shape[0]), _p(x, D), _p(res, D)))
        return x, res

    def relative_residual(self, x, b):
        out = D()
        _check(lib().ref_relative_residual(self.h, _p(np.ascontiguousarray(x, np.complex128), D),
                                           _p(np.ascontiguousarray(b, np.complex128), D),
                                           C.byref(out)))
        return out.value


def signal_modes(dz):
    dz = np.ascontiguousarray(dz, np.complex128)
    out = np.empty(4)
    lib().ref_signal_modes(_p(dz, D), _p(out, D))
    return complex(out[0], out[1]), complex(out[2], out[3])


def tet_frame(p):
    p = np.ascontiguousarray(p, np.float64)
    g = np.empty(12)
    v = D()
    _check(lib().ref_tet_frame(_p(p, D), _p(g, D), C.byref(v)))
    return g.reshape(4, 3), v.value


def element_blocks(p, mu, mu_tilde, sigma, omega, delta_gauge):
    p = np.ascontiguousarray(p, np.float64)
    l11 = np.empty((12, 12), np.complex128)
    l12 = np.empty((12, 4), np.complex128)
    l21 = np.empty((4, 12), np.complex128)
    l22 = np.empty((4, 4), np.complex128)
    _check(lib().ref_element_blocks(_p(p, D), D(mu), D(mu_tilde), D(sigma), D(omega),
                                    D(delta_gauge), _p(l11, D), _p(l12, D), _p(l21, D),
                                    _p(l22, D)))
    return l11, l12, l21, l22


def system_from_csc(col_ptr, row_idx, values) -> "RefSystem":
    """RefSystem around CSC arrays (see ref_system_from_csc in ref_driver.cpp)."""
    col_ptr = np.ascontiguousarray(col_ptr, np.int32)
    row_idx = np.ascontiguousarray(row_idx, np.int32)
    values = np.ascontiguousarray(values, np.complex128)
    h = C.c_void_p()
    _check(lib().ref_system_from_csc(I64(len(col_ptr) - 1), I64(len(row_idx)), _p(col_ptr, I32),
                                     _p(row_idx, I32), _p(values, D), C.byref(h)))
    s = RefSystem.__new__(RefSystem)
    s.h, s.mesh, s.timings = h, None, {}
    s.n, s.nnz, s.n_pins = len(col_ptr) - 1, len(row_idx), 0
    return s


def trace_write(path, z, dz, modes, failed=None, config_hash=""):
    """The reference's write_trace_csv (scan.cpp:170-207)."""
    z = np.ascontiguousarray(z, np.float64)
    dz = np.ascontiguousarray(np.asarray(dz, np.complex128).reshape(len(z), 4))
    modes = np.ascontiguousarray(np.asarray(modes, np.complex128).reshape(len(z), 2))
    f = np.ascontiguousarray(np.zeros(len(z)) if failed is None else failed, np.int32)
    _check(lib().ref_trace_write(str(path).encode(), I32(len(z)), _p(z, D), _p(dz, D),
                                 _p(modes, D), _p(f, I32), config_hash.encode()))


def trace_max_relative_deviation(a, b):
    out = D()
    _check(lib().ref_trace_max_relative_deviation(str(a).encode(), str(b).encode(), C.byref(out)))
    return out.value


def _tube_params(spec: dict) -> np.ndarray:
    nan = float("nan")
    box = lambda k: list(spec[k]) if spec.get(k) is not None else [nan] * 4
    return np.array([spec["domain_radius"], spec["z_min"], spec["z_max"], spec["tube_r_inner"],
                     spec["tube_r_outer"], spec.get("tube_z_min", nan), spec.get("tube_z_max", nan),
                     *box("tsp"), *box("defect"), *spec["coil"], spec.get("coil_ref_z", 0.0),
                     spec.get("resolution", 8), spec.get("outer_radial_grading", 2.0)], np.float64)


def scan_session_tube(spec: dict, physics, amplitude, tol, max_iter, restart, gpu=False):
    """The reference's ScanSession (scan.cpp:27-143, solver.method = iterative)
    on generate_tube_mesh(spec), solve_position at every spec["scan_z"].
    gpu=False: the reference's own GMRES(restart)+ILU(0); gpu=True: the same
    reference code linked with the ectgpu drop-in solve_iterative
    (oracle/binding/iterative_gpu.cpp, _ref/libectref_gpu.so).
    Returns [n, 14]: z, dz (8), z_fa (2), z_f3 (2), failed."""
    L = lib() if not gpu else _gpu_lib()
    p = _tube_params(spec)
    zs = np.ascontiguousarray(spec["scan_z"], np.float64)
    out = np.empty((len(zs), 14))
    ph = physics_struct(physics)
    rc = L.ref_scan_session_tube(_p(p, D), _p(zs, D), I32(len(zs)), C.byref(ph), D(amplitude),
                                 D(tol), I32(max_iter), I32(restart), _p(out, D))
    if rc != 0:
        raise RefError(L.ref_last_error().decode())
    return out


_gpu_lib_h = None


def _gpu_lib():
    global _gpu_lib_h
    if _gpu_lib_h is None:
        if not GPU_LIB_PATH.exists():
            raise RefError(f"{GPU_LIB_PATH} not built (make -C oracle)")
        _gpu_lib_h = C.CDLL(str(GPU_LIB_PATH))
        _gpu_lib_h.ref_last_error.restype = C.c_char_p
    return _gpu_lib_h
