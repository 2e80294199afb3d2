"""numpy restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

A CPU port of ectsim's A–V assembly, right-hand side and impedance code,
vectorised with numpy, each function citing the reference it follows
(/root/reference/proj/core/...). Elementwise numpy ops are single IEEE
operations (no FMA contraction), and every accumulation below is a left fold
in the reference's insertion order, so the port reproduces the reference's
CscMatrix values bit for bit (pinned against oracle/_ref through the golden
fixtures in tests/test_oracle.py). Only tests/ and bench.py's CPU legs may
import this module; the product never does.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

KMU0 = 1.25663706212e-6            # types.hpp:18
TUBE, TSP, DEFECT, COIL1, COIL2, VACUUM = range(6)   # types.hpp:22-29
KFACE = ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2))  # mesh.cpp:107


def is_conductor(region):
    """is_conductor_region (types.hpp:46-48)."""
    return (region == TUBE) | (region == TSP) | (region == DEFECT)


def conductor_map(n_nodes, tets, region):
    """conductor_map (mesh.cpp:267-284): rank among conductor-incident nodes."""
    flag = np.zeros(n_nodes, bool)
    flag[tets[is_conductor(region)].ravel()] = True
    fwd = np.full(n_nodes, -1, np.int32)
    fwd[flag] = np.arange(int(flag.sum()), dtype=np.int32)
    if not flag.any():
        raise ValueError("mesh has no conductor region: scalar potential space is empty")
    return fwd


def exterior_faces(tets):
    """build_face_incidence (mesh.cpp:122-143): faces with one incident tet."""
    f = np.concatenate([tets[:, list(k)] for k in KFACE])
    f.sort(axis=1)
    _, idx, cnt = np.unique(f, axis=0, return_index=True, return_counts=True)
    return f[idx[cnt == 1]]


def pinned_dofs(xyz, tets):
    """classify_boundary + apply_essential_bc pins (mesh.cpp:145-182,
    assembly.cpp:285-312): z-dof on TOP/BOTTOM, x,y-dofs on LATERAL faces."""
    z = xyz[:, 2]
    z_lo, z_hi = z.min(), z.max()
    tol = 1e-9 * max(1.0, z_hi - z_lo)
    f = exterior_faces(tets)
    top = np.all(np.abs(z[f] - z_hi) <= tol, axis=1)
    bot = np.all(np.abs(z[f] - z_lo) <= tol, axis=1)
    tb = f[top | bot].ravel()
    lat = f[~(top | bot)].ravel()
    pins = np.unique(np.concatenate([3 * tb + 2, 3 * lat, 3 * lat + 1]))
    return pins.astype(np.int32)


def signed_volume(xyz, tets):
    """(b-a) x (c-a) . (d-a) / 6 (mesh.cpp:36-38)."""
    a, b, c, d = (xyz[tets[:, i]] for i in range(4))
    u, v, w = b - a, c - a, d - a
    cx = u[:, 1] * v[:, 2] - u[:, 2] * v[:, 1]
    cy = u[:, 2] * v[:, 0] - u[:, 0] * v[:, 2]
    cz = u[:, 0] * v[:, 1] - u[:, 1] * v[:, 0]
    return ((cx * w[:, 0] + cy * w[:, 1]) + cz * w[:, 2]) / 6.0


def tet_frames(xyz, tets):
    """TetFrame::from (element_forms.cpp:8-30) with Eigen's 3x3 determinant /
    cofactor inverse. Returns grads [T,4,3] and volumes [T]."""
    p = xyz[tets]                                   # [T,4,3]
    m = np.empty((len(tets), 3, 3))
    for c in range(3):
        m[:, :, c] = p[:, c + 1, :] - p[:, 0, :]    # jac.col(c)
    h0 = m[:, 0, 0] * (m[:, 1, 1] * m[:, 2, 2] - m[:, 1, 2] * m[:, 2, 1])
    h1 = m[:, 0, 1] * (m[:, 1, 0] * m[:, 2, 2] - m[:, 1, 2] * m[:, 2, 0])
    h2 = m[:, 0, 2] * (m[:, 1, 0] * m[:, 2, 1] - m[:, 1, 1] * m[:, 2, 0])
    det = (h0 - h1) + h2
    if np.any(~(det > 0.0)):
        raise ValueError("element frame on a degenerate or inverted tet")
    cof = np.empty_like(m)
    for i in range(3):
        for j in range(3):
            i1, i2, j1, j2 = (i + 1) % 3, (i + 2) % 3, (j + 1) % 3, (j + 2) % 3
            cof[:, i, j] = m[:, i1, j1] * m[:, i2, j2] - m[:, i1, j2] * m[:, i2, j1]
    det_inv = (cof[:, 0, 0] * m[:, 0, 0] + cof[:, 1, 0] * m[:, 1, 0]) + cof[:, 2, 0] * m[:, 2, 0]
    invdet = 1.0 / det_inv
    g = np.empty((len(tets), 4, 3))
    for k in range(3):
        for c in range(3):
            g[:, k + 1, c] = cof[:, c, k] * invdet
    g[:, 0, :] = -((g[:, 1, :] + g[:, 2, :]) + g[:, 3, :])
    return g, det / 6.0


def _dot(a, b):
    return (a[:, 0] * b[:, 0] + a[:, 1] * b[:, 1]) + a[:, 2] * b[:, 2]


def _fold(rows, cols, vals, n):
    """canonicalize + from_triplets (sparse.cpp:13-31, 83-113): stable sort by
    (row, col) and a LEFT FOLD of duplicates in insertion order. Returns CSR
    (== reference CSC read transposed, the pattern being symmetric)."""
    order = np.lexsort((np.arange(len(rows)), cols, rows))   # stable: insertion order last
    r, c, v = rows[order], cols[order], vals[order]
    key_change = np.ones(len(r), bool)
    key_change[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
    start = np.flatnonzero(key_change)
    seg = np.cumsum(key_change) - 1
    pos = np.arange(len(r)) - start[seg]
    acc = v[start].copy()
    for k in range(1, int(pos.max()) + 1 if len(pos) else 1):
        sel = pos == k
        np.add.at(acc, seg[sel], v[sel])          # one addend per segment per pass: exact fold
    ur, uc = r[start], c[start]
    row_ptr = np.zeros(n + 1, np.int64)
    np.add.at(row_ptr, ur + 1, 1)
    return np.cumsum(row_ptr).astype(np.int32), uc.astype(np.int32), acc


def assemble(xyz, tets, region, mats, cond_fwd=None, pins=None):
    """assemble_system (one partition) + apply_essential_bc + build_global
    (assembly.cpp:74-276, 285-327, 386-419). mats: dict with omega, sigma[6],
    mu[6], mu_tilde, delta_gauge, bc_penalty. Returns CSR (row_ptr, col, val)."""
    n_nodes = len(xyz)
    cond_fwd = conductor_map(n_nodes, tets, region) if cond_fwd is None else cond_fwd
    pins = pinned_dofs(xyz, tets) if pins is None else pins
    na = 3 * n_nodes
    n = na + int(cond_fwd.max()) + 1
    g, vol = tet_frames(xyz, tets)
    sigma = np.asarray(mats["sigma"])[region]
    mu = np.asarray(mats["mu"])[region]
    mu_inv = 1.0 / mu
    mt_inv = 1.0 / mats["mu_tilde"]
    mass_im = (-1.0 * mats["omega"]) * sigma
    T = len(tets)
    rows, cols, vals = [], [], []
    # element_l11 (element_forms.cpp:49-73), insertion order a, c, b, d (assembly.cpp:109-122)
    blocks = np.empty((T, 4, 3, 4, 3), np.complex128)
    for a in range(4):
        for b in range(4):
            ga, gb = g[:, a, :], g[:, b, :]
            dot = _dot(ga, gb)
            mass = (vol * (2.0 if a == b else 1.0)) / 20.0
            for c in range(3):
                for d in range(3):
                    curl = (dot if c == d else 0.0) - ga[:, d] * gb[:, c]
                    value = vol * (mu_inv * curl + (mt_inv * ga[:, c]) * gb[:, d])
                    if c == d:
                        blocks[:, a, c, b, d] = (value + 0.0) + 1j * (0.0 + mass_im * mass)
                    else:
                        blocks[:, a, c, b, d] = value
    node3 = 3 * tets.astype(np.int64)
    rr = (node3[:, :, None, None, None] + np.arange(3)[None, None, :, None, None])
    cc = (node3[:, None, None, :, None] + np.arange(3)[None, None, None, None, :])
    rr, cc = np.broadcast_to(rr, blocks.shape), np.broadcast_to(cc, blocks.shape)
    rows.append(rr.reshape(-1)); cols.append(cc.reshape(-1)); vals.append(blocks.reshape(-1))
    # conductor blocks (element_l12/l21/l22), conductor tets only
    ct = np.flatnonzero(is_conductor(region))
    if len(ct):
        gc, vc, sc, muc = g[ct], vol[ct], sigma[ct], mu[ct]
        w = vc / 4.0
        cf = cond_fwd[tets[ct]].astype(np.int64) + na
        n3 = node3[ct]
        l12 = np.empty((len(ct), 4, 3, 4))
        l21 = np.empty((len(ct), 4, 4, 3))
        for a in range(4):
            for c in range(3):
                for b in range(4):
                    l12[:, a, c, b] = ((-sc) * gc[:, b, c]) * w
                    l21[:, b, a, c] = ((-sc) * gc[:, b, c]) * w
        r12 = np.broadcast_to(n3[:, :, None, None] + np.arange(3)[None, None, :, None], l12.shape)
        c12 = np.broadcast_to(cf[:, None, None, :], l12.shape)
        r21 = np.broadcast_to(cf[:, :, None, None], l21.shape)
        c21 = np.broadcast_to(n3[:, None, :, None] + np.arange(3)[None, None, None, :], l21.shape)
        stiff = sc / mats["omega"]
        gauge = (mats["delta_gauge"] * muc) * sc
        l22 = np.empty((len(ct), 4, 4), np.complex128)
        for a in range(4):
            for b in range(4):
                s = vc * _dot(gc[:, a], gc[:, b])
                mass = (vc * (2.0 if a == b else 1.0)) / 20.0
                l22[:, a, b] = ((0.0 * s) + gauge * mass) + 1j * (stiff * s)
        r22 = np.broadcast_to(cf[:, :, None], l22.shape)
        c22 = np.broadcast_to(cf[:, None, :], l22.shape)
        for R, Cc, V in ((r12, c12, l12), (r21, c21, l21), (r22, c22, l22)):
            rows.append(R.reshape(-1)); cols.append(Cc.reshape(-1))
            vals.append(V.reshape(-1).astype(np.complex128))
    row_ptr, col, val = _fold(np.concatenate(rows), np.concatenate(cols), np.concatenate(vals), n)
    # apply_pins_to_matrix: pinned diagonals := (penalty, 0) (assembly.cpp:314-327)
    rws = np.repeat(np.arange(n), np.diff(row_ptr))
    diag = np.flatnonzero(rws == col)
    pin_diag = diag[np.isin(rws[diag], pins)]
    val[pin_diag] = mats["bc_penalty"] + 0j
    return row_ptr, col, val


def coil_support(xyz, tets, coil, z, which):
    """coil_support (tube_mesh.cpp:272-288)."""
    r_in, r_out, height, gap = coil
    lo = (z - 0.5 * gap) - height if which == 1 else z + 0.5 * gap
    hi = lo + height
    c = 0.25 * (((xyz[tets[:, 0]] + xyz[tets[:, 1]]) + xyz[tets[:, 2]]) + xyz[tets[:, 3]])
    r = np.hypot(c[:, 0], c[:, 1])
    return np.flatnonzero((r >= r_in) & (r <= r_out) & (c[:, 2] >= lo) & (c[:, 2] <= hi))


def assemble_rhs(xyz, tets, region, support, amplitude, n, pins):
    """assemble_rhs + apply_pins_to_rhs (assembly.cpp:329-378)."""
    if len(support) == 0:
        raise ValueError("coil support is empty")
    if np.any(is_conductor(region[support])):
        raise ValueError("coil support intersects a conductor region")
    n_nodes = len(xyz)
    flag = np.zeros(n_nodes, bool)
    flag[tets[support].ravel()] = True
    j = np.zeros((n_nodes, 3))
    x, y = xyz[flag, 0], xyz[flag, 1]
    r = np.hypot(x, y)
    ok = r > 0.0
    jj = np.zeros((flag.sum(), 3))
    jj[ok, 0] = amplitude * (-y[ok] / r[ok])
    jj[ok, 1] = amplitude * (x[ok] / r[ok])
    jj[ok, 2] = amplitude * 0.0
    j[flag] = jj
    touched = np.flatnonzero(flag[tets].any(axis=1))
    vol = signed_volume(xyz, tets[touched])
    rhs = np.zeros(n, np.complex128)
    k = tets[touched]
    contrib = np.empty((len(touched), 4, 3))
    for a in range(4):
        acc = np.zeros((len(touched), 3))
        for b in range(4):
            s = (vol * (2.0 if a == b else 1.0)) / 20.0
            acc = acc + s[:, None] * j[k[:, b]]
        contrib[:, a] = acc
    # fold per dof in tet order (rhs starts at 0)
    dof = (3 * k[:, :, None] + np.arange(3)).reshape(-1)
    v = contrib.reshape(-1)
    order = np.argsort(dof, kind="stable")
    d, vv = dof[order], v[order]
    change = np.ones(len(d), bool)
    change[1:] = d[1:] != d[:-1]
    start = np.flatnonzero(change)
    seg = np.cumsum(change) - 1
    pos = np.arange(len(d)) - start[seg]
    acc = np.zeros(len(start))
    for q in range(int(pos.max()) + 1):
        sel = pos == q
        acc[seg[sel]] = acc[seg[sel]] + vv[sel]
    rhs.real[d[start]] = acc
    rhs[pins] = 0.0
    return rhs


def solve_direct(row_ptr, col, val, b):
    """Direct solve (the reference's default solver role, solver.cpp:197-376),
    via SuperLU."""
    n = len(row_ptr) - 1
    A = sp.csc_matrix(sp.csr_matrix((val, col, row_ptr), shape=(n, n)))
    return spla.spsolve(A, b)


def delta_impedance(xyz, tets, region, cond_fwd, primary, reference, x_k, x_l):
    """delta_impedance (signals.cpp:67-99) over DEFECT tets, with curl_on_tet /
    electric_field_on_tet (signals.cpp:22-56)."""
    dt = np.flatnonzero(region == DEFECT)
    if len(dt) == 0:
        return 0j
    n_nodes = len(xyz)
    g, _ = tet_frames(xyz, tets[dt])
    vol = signed_volume(xyz, tets[dt])
    k = tets[dt]
    omega = primary["omega"]

    def fields(x):
        A = x[:3 * n_nodes].reshape(-1, 3)[k]               # [D,4,3]
        V = x[3 * n_nodes:][cond_fwd[k]]                    # [D,4]
        curl = np.zeros((len(dt), 3), np.complex128)
        for a in range(4):
            ga, Aa = g[:, a, :], A[:, a, :]
            curl[:, 0] += ga[:, 1] * Aa[:, 2] - ga[:, 2] * Aa[:, 1]
            curl[:, 1] += ga[:, 2] * Aa[:, 0] - ga[:, 0] * Aa[:, 2]
            curl[:, 2] += ga[:, 0] * Aa[:, 1] - ga[:, 1] * Aa[:, 0]
        e = 1j * omega * (0.25 * A.sum(axis=1)) + np.einsum("dac,da->dc", g, V)
        return curl, e

    ck, ek = fields(x_k)
    cl, el = fields(x_l)
    tag = region[dt]
    mu_d = np.asarray(primary["mu"])[tag]
    mu_e = np.asarray(reference["mu"])[tag]
    s_d = np.asarray(primary["sigma"])[tag]
    s_e = np.asarray(reference["sigma"])[tag]
    inv_iw = -1j / omega
    tot = inv_iw * ((mu_e - mu_d) / (mu_d * mu_e)) * vol * np.sum(ck * cl, axis=1)
    tot = tot + (s_d - s_e) * vol * np.sum(ek * el, axis=1)
    return complex(np.sum(tot))


def mats_dict(arr):
    """Packed MaterialTable array (oracle/make_golden.py layout) -> dict."""
    return {"omega": arr[0], "sigma": arr[1:7], "mu": arr[7:13], "mu_tilde": arr[13],
            "delta_gauge": arr[14], "bc_penalty": arr[15], "sigma_eps": arr[16]}
