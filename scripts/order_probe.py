"""Dev probe: does a tiled node numbering speed up the NB-E SpMV?  The configs[1]
mesh is renumbered (nodes sorted by a tile key) and the default kernel timed
at k = 2, 8 against the reference numbering.  python scripts/order_probe.py"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1602_03207_b200 import ect, workloads  # noqa: E402

w = workloads.config1()
m = w.mesh()
nx, ny, nz = 64, 64, 128
ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()  # node id order (i, j, k), k fastest


def run(name, perm):
    # perm[new] = old node id
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    xyz = m.xyz[perm]
    tets = inv[m.tets]
    ctx = ect.Context(0)
    mesh = ect.Mesh(ctx, xyz, tets, m.region)
    p, r, two = mesh.materials(w.physics)
    a = ect.Matrix(ctx, mesh).assemble(p)
    g = torch.Generator(device="cuda").manual_seed(2)
    for k in (2, 8):
        x = torch.complex(torch.rand(a.n, k, device="cuda", dtype=torch.float64, generator=g),
                          torch.rand(a.n, k, device="cuda", dtype=torch.float64, generator=g))
        y = torch.empty_like(x)
        for _ in range(3):
            a.multiply(x, out=y)
        ctx.synchronize()
        ctx.mark(0)
        for _ in range(20):
            a.multiply(x, out=y)
        ctx.mark(1)
        print(f"{name:28s} k={k}: {ctx.elapsed_ms(0, 1) / 20:.4f} ms", flush=True)
    del a, mesh
    ctx.close()


run("reference numbering", np.arange(ii.size))
for tj, tk in ((4, 8), (2, 16), (8, 4), (4, 32)):
    key = np.lexsort((kk % tk, jj % tj, kk // tk, jj // tj, ii))
    run(f"tiles j{tj} x k{tk} per plane", key)
# 3D tiles: 2 planes x 4 lines x 4 k
key = np.lexsort((kk % 4, jj % 4, ii % 2, kk // 4, jj // 4, ii // 2))
run("tiles i2 x j4 x k4", key)
