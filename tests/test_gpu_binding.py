"""The reference-side binding exercised:
the reference's own ScanSession::solve_position (scan.cpp:95-143,
solver.method = iterative) on its own tube geometry (generate_tube_mesh),
once with its GMRES(150)+ILU(0) (oracle/_ref/libectref.so) and once with the
ectgpu drop-in solve_iterative linked in place of iterative.cpp
(oracle/binding/iterative_gpu.cpp -> _ref/libectref_gpu.so). Everything but
the solver is the unmodified reference, so the signals must agree; the probe
position of the tube_r6 golden is also checked against the reference's direct
LU."""
import json

import numpy as np
import pytest

from paper_1602_03207_b200 import workloads
from tests.helpers import golden

pytestmark = pytest.mark.gpu


def _signals(rows):
    # dz (4 complex), z_fa, z_f3 per position
    v = rows[:, 1:13].reshape(len(rows), 6, 2)
    return v[..., 0] + 1j * v[..., 1]


def test_reference_scan_session_on_gpu_solver(ref_lib):
    ref = ref_lib
    if not ref.GPU_LIB_PATH.exists():
        pytest.skip("oracle/_ref/libectref_gpu.so not built")
    g = golden("tube_r6")
    spec = json.loads(str(g["tube_spec"]))
    phys = workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0)
    amp = float(g["amplitude"])
    gpu = ref.scan_session_tube(spec, phys, amp, 1e-11, 20000, 150, gpu=True)
    cpu = ref.scan_session_tube(spec, phys, amp, 1e-11, 20000, 150, gpu=False)
    assert not gpu[:, 13].any() and not cpu[:, 13].any()
    assert np.array_equal(gpu[:, 0], cpu[:, 0])
    a, b = _signals(gpu), _signals(cpu)
    # per signal over the curve, relative to the curve's largest value
    dev = np.max(np.abs(a - b), axis=0) / np.max(np.abs(b), axis=0)
    assert np.all(dev <= 1e-6), dev
    # the golden position against the reference's direct LU chain
    q = int(np.argmin(np.abs(gpu[:, 0] - float(g["z"]))))
    err = np.max(np.abs(a[q, :4] - g["dz"])) / np.max(np.abs(g["dz"]))
    assert err <= 1e-6, err
