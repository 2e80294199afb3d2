"""CPU experiment: COCG iteration counts under different symmetric
preconditioners on a reduced configs[1]-like mesh (reference-assembled matrix).

  python scripts/precond_probe.py [nx ny nz]
"""
import sys
import time

import numpy as np
import scipy.sparse as sp

from oracle import ref
from paper_1602_03207_b200 import workloads
from paper_1602_03207_b200.workloads import Workload, _coil


def cocg(A, b, apply_m, tol=1e-8, max_iter=20000):
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


def main():
    dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (24, 24, 48)
    w = Workload("probe", dims, 1, ((0.9, 1.1),), workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0),
                 _coil(dims[2]), 1e6, (1.0 * workloads.SCALE,))
    mm = w.mesh()
    m = ref.RefMesh(mm.xyz, mm.tets, mm.region)
    p, _, _ = m.materials(w.physics)
    t = time.time()
    S = ref.RefSystem(m, p, parts=8, workers=8)
    cp, ri, v, _ = S.export()
    A = sp.csc_matrix((v, ri, cp), shape=(S.n, S.n)).tocsr()
    nn = len(mm.xyz)
    print(f"dims {dims} N={S.n} nnz={S.nnz} assembled in {time.time()-t:.1f}s", flush=True)
    b = S.position_rhs(np.array(w.coil), w.positions[0], 1, w.amplitude)

    d = A.diagonal()
    jac = lambda r: r / d

    # node-block 3x3 (A-A) inverse, V diag
    na = 3 * nn
    rows = np.repeat(np.arange(na), 3)
    cols = (np.arange(na) // 3 * 3)[:, None] + np.arange(3)
    blk = np.asarray(A[rows, cols.ravel()]).reshape(nn, 3, 3)
    binv = np.linalg.inv(blk)
    def bj(r):
        out = np.empty_like(r)
        out[:na] = np.einsum("nij,nj->ni", binv, r[:na].reshape(nn, 3)).ravel()
        out[na:] = r[na:] / d[na:]
        return out

    # 4x4 blocks on conductor nodes (A of node + its V dof)
    import oracle.port as port
    cond = port.conductor_map(nn, mm.tets, mm.region)
    cn = np.nonzero(cond >= 0)[0]
    idx = np.concatenate([3 * cn[:, None] + np.arange(3), (na + cond[cn])[:, None]], axis=1)
    B4 = np.asarray(A[np.repeat(idx, 4, axis=1).ravel(), np.tile(idx, (1, 4)).ravel()]).reshape(-1, 4, 4)
    B4inv = np.linalg.inv(B4)
    def bj4(r):
        out = bj(r)
        out[idx.ravel()] = np.einsum("nij,nj->ni", B4inv, r[idx]).ravel()
        return out

    for name, M in (("jacobi", jac), ("block3", bj), ("block4", bj4)):
        t = time.time()
        x, it = cocg(A, b, M)
        rel = np.linalg.norm(b - A @ x) / np.linalg.norm(b)
        print(f"{name:8s} iters={it:6d} true_rel={rel:.2e} {time.time()-t:.1f}s", flush=True)


if __name__ == "__main__":
    main()
