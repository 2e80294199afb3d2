"""CPU experiment: COCG iteration counts with an aggregation-multigrid
preconditioner (V-cycle, damped-Jacobi smoothing, Galerkin coarse operators
with the plain transpose so M stays complex symmetric) against Jacobi, on
reference-assembled configs[1]-like meshes of growing size.

  python scripts/amg_probe.py nx ny nz [smooth]
"""
import sys
import time

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import ref
from paper_1602_03207_b200 import workloads
from paper_1602_03207_b200.workloads import Workload, _coil


def cocg(A, b, apply_m, tol=float(__import__("os").environ.get("TOL", 1e-8)), max_iter=int(__import__("os").environ.get("MAXIT", 5000))):
    x = np.zeros_like(b)
    r = b.copy()
    z = apply_m(r)
    p = z.copy()
    rho = r @ z
    bn = np.linalg.norm(b)
    for it in range(1, max_iter + 1):
        q = A @ p
        alpha = rho / (p @ q)
        x += alpha * p
        r -= alpha * q
        if np.linalg.norm(r) <= tol * bn:
            return x, it
        z = apply_m(r)
        rho_new = r @ z
        p = z + (rho_new / rho) * p
        rho = rho_new
    return x, max_iter


def aggregate(G):
    """Greedy 3-phase aggregation of the node graph G (CSR, no self loops)."""
    n = G.shape[0]
    agg = -np.ones(n, np.int64)
    ip, ix = G.indptr, G.indices
    na = 0
    for i in range(n):  # phase 1: node whose whole neighbourhood is free
        if agg[i] >= 0:
            continue
        nb = ix[ip[i]:ip[i + 1]]
        if np.all(agg[nb] < 0):
            agg[i] = na
            agg[nb] = na
            na += 1
    for i in range(n):  # phase 2: join a neighbouring aggregate
        if agg[i] >= 0:
            continue
        nb = ix[ip[i]:ip[i + 1]]
        a = agg[nb]
        a = a[a >= 0]
        if a.size:
            agg[i] = -2 - a[0]
    agg = np.where(agg <= -2, -2 - agg, agg)
    for i in range(n):  # phase 3: leftovers
        if agg[i] < 0:
            nb = ix[ip[i]:ip[i + 1]]
            agg[i] = na
            agg[nb[agg[nb] < 0]] = na
            na += 1
    return agg, na


def build_levels(A, n_nodes, cond, pinned, smooth=0, coarse_n=int(__import__("os").environ.get("COARSE_N", 2000)), omega_p=2 / 3):
    levels = []
    nodes = n_nodes
    # level description: dof_node (node index or -1), dof_kind (0..2 A comp, 3 V)
    na = 3 * n_nodes
    dof_node = np.concatenate([np.repeat(np.arange(n_nodes), 3), np.nonzero(cond >= 0)[0][np.argsort(cond[cond >= 0])]])
    dof_kind = np.concatenate([np.tile(np.arange(3), n_nodes), np.full(A.shape[0] - na, 3)])
    free = np.ones(A.shape[0], bool)
    free[pinned] = False
    while A.shape[0] > coarse_n:
        # node graph from the matrix pattern restricted to free dofs
        C = sp.csr_matrix((np.ones(A.nnz), A.indices, A.indptr), shape=A.shape)
        R = sp.csr_matrix((np.ones(A.shape[0]), (dof_node, np.arange(A.shape[0]))), shape=(nodes, A.shape[0]))
        G = (R @ C @ R.T).tocsr()
        G.setdiag(0)
        G.eliminate_zeros()
        agg, n_agg = aggregate(G)
        # coarse dofs: (aggregate, kind) for every kind present among free dofs
        key = agg[dof_node] * 4 + dof_kind
        vmode = __import__("os").environ.get("VAGG", "node")
        isv = dof_kind == 3
        if vmode == "none":
            free = free & ~isv
        elif vmode == "strength" and isv.any():
            th = float(__import__("os").environ.get("THETA", "0.05"))
            vi = np.nonzero(isv)[0]
            AV = A[vi][:, vi].tocsr()
            dv = np.abs(AV.diagonal())
            AV = AV.tocoo()
            strong = (np.abs(AV.data) >= th * np.sqrt(dv[AV.row] * dv[AV.col])) & (AV.row != AV.col)
            GV = sp.csr_matrix((np.ones(strong.sum()), (AV.row[strong], AV.col[strong])), shape=(len(vi), len(vi)))
            aggv, nv = aggregate(GV)
            key = key.copy()
            key[vi] = (n_agg + aggv) * 4 + 3
        ukeys, cidx = np.unique(key[free], return_inverse=True)
        P0 = sp.csr_matrix((np.ones(free.sum()), (np.nonzero(free)[0], cidx)), shape=(A.shape[0], len(ukeys)))
        if smooth:
            d = A.diagonal()
            Dinv = sp.diags(1.0 / d)
            DA = Dinv @ A
            lam = abs(spla.eigs(DA, k=1, which="LM", return_eigenvectors=False, tol=1e-2)[0])
            P = (P0 - (omega_p * 4 / 3 / lam) * (DA @ P0)).tocsr()
            P = P.multiply(free[:, None]).tocsr()
        else:
            P = P0
        Ac = (P.T @ A @ P).tocsr()
        levels.append({"A": A, "P": P, "d": A.diagonal()})
        print(f"  level {len(levels)-1}: n={A.shape[0]} nnz={A.nnz} -> {Ac.shape[0]} (nnz {Ac.nnz})", flush=True)
        A = Ac
        dof_node = ukeys // 4
        dof_kind = ukeys % 4
        nodes = int(dof_node.max()) + 1
        free = np.ones(A.shape[0], bool)
    import os
    if os.environ.get("INV"):
        reg = float(os.environ.get("REG", "0"))
        Ad = A.toarray()
        Ad = Ad + reg * np.diag(np.diag(Ad))
        Minv = np.linalg.inv(Ad)
        print(f"  coarsest n={A.shape[0]} dense inverse, reg={reg}, cond~{np.linalg.cond(Ad):.2e}", flush=True)
        class _Inv:
            def solve(self, b):
                return Minv @ b
        levels.append({"A": A, "lu": _Inv()})
    else:
        levels.append({"A": A, "lu": spla.splu(A.tocsc())})
    return levels


F32 = __import__("os").environ.get("F32") == "1"
ADD = __import__("os").environ.get("ADD") == "1"
ADD_W = float(__import__("os").environ.get("ADD_W", "0.6"))


def vcycle(levels, b, lvl=0, nu=1, w=0.7, gamma=1, oc=1.0):
    L = levels[lvl]
    if "lu" in L:
        return L["lu"].solve(b)
    A, P, d = L["A"], L["P"], L["d"]
    if ADD and lvl == 0:  # additive fine level: no fine-level SpMV in the cycle
        rc = P.T @ b
        e = vcycle(levels, rc, lvl + 1, nu, w, gamma, oc)
        if gamma == 2 and "lu" not in levels[lvl + 1]:
            Ac = levels[lvl + 1]["A"]
            e = e + vcycle(levels, rc - Ac @ e, lvl + 1, nu, w, gamma, oc)
        return ADD_W * b / d + oc * (P @ e)
    if F32 and lvl == 0:  # finest level smoothing in single precision
        if "A32" not in L:
            L["A32"] = A.astype(np.complex64)
        A32 = L["A32"]
        b32 = b.astype(np.complex64)
        x = (w * b / d).astype(np.complex64)
        r = (b32 - A32 @ x)
        rc = (P.T @ r.astype(np.complex128))
        e = vcycle(levels, rc, lvl + 1, nu, w, gamma, oc)
        if gamma == 2 and "lu" not in levels[lvl + 1]:
            Ac = levels[lvl + 1]["A"]
            e = e + vcycle(levels, rc - Ac @ e, lvl + 1, nu, w, gamma, oc)
        x = x + (oc * (P @ e)).astype(np.complex64)
        return x.astype(np.complex128) + w * (b - (A32 @ x).astype(np.complex128)) / d
    x = w * b / d
    for _ in range(nu - 1):
        x = x + w * (b - A @ x) / d
    r = b - A @ x
    rc = P.T @ r
    e = vcycle(levels, rc, lvl + 1, nu, w, gamma, oc)
    if gamma == 2 and "lu" not in levels[lvl + 1]:
        Ac = levels[lvl + 1]["A"]
        e = e + vcycle(levels, rc - Ac @ e, lvl + 1, nu, w, gamma, oc)
    x = x + oc * (P @ e)
    for _ in range(nu):
        x = x + w * (b - A @ x) / d
    return x


def main():
    dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (16, 16, 32)
    smooth = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    w = Workload("probe", dims, 1, ((0.9, 1.1),), workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0),
                 _coil(dims[2]), 1e6, (1.0 * workloads.SCALE,))
    mm = w.mesh()
    m = ref.RefMesh(mm.xyz, mm.tets, mm.region)
    p, rr, _ = m.materials(w.physics)
    if __import__("os").environ.get("CFG") == "ref":
        p = rr
    t = time.time()
    S = ref.RefSystem(m, p, parts=4, workers=4)
    cp, ri, v, pins = S.export()
    A = sp.csc_matrix((v, ri, cp), shape=(S.n, S.n)).tocsr()
    nn = len(mm.xyz)
    cond = m.export()["cond_forward"]
    print(f"dims {dims} N={S.n} nnz={S.nnz} assembled in {time.time()-t:.1f}s", flush=True)
    b = S.position_rhs(np.array(w.coil), w.positions[0], 1, w.amplitude)
    d = A.diagonal()
    t = time.time()
    x, it = cocg(A, b, lambda r: r / d) if not __import__("os").environ.get("NOJAC") else (b, 0)
    print(f"jacobi   iters={it:5d} true={np.linalg.norm(b - A @ x) / np.linalg.norm(b):.2e} {time.time()-t:.1f}s", flush=True)
    t = time.time()
    levels = build_levels(A, nn, cond, pins, smooth=smooth)
    print(f"setup {time.time()-t:.1f}s", flush=True)
    cfgs = ((1, 0.6, 1, 1.0), (1, 0.6, 2, 1.0), (1, 0.6, 1, 1.5), (1, 0.6, 2, 1.5), (1, 0.6, 1, 2.0))
    if __import__("os").environ.get("CFGS"):
        cfgs = [tuple(float(v) for v in c.split(":")) for c in __import__("os").environ["CFGS"].split(",")]
    for nu, wj, g, oc in cfgs:
        nu, g = int(nu), int(g)
        t = time.time()
        x, it = cocg(A, b, lambda r: vcycle(levels, r, nu=nu, w=wj, gamma=g, oc=oc))
        print(f"amg levels={len(levels)} nu={nu} w={wj} gamma={g} oc={oc} iters={it:5d} true={np.linalg.norm(b - A @ x) / np.linalg.norm(b):.2e} {time.time()-t:.1f}s", flush=True)


if __name__ == "__main__":
    main()
