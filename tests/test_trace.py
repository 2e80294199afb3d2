"""Impedance trace in the reference CSV format.

CPU: our writer reproduces the reference's write_trace_csv byte for byte.
GPU: a 5-position sweep through ect.Session matches the reference's own trace
(direct LU per material configuration) to max_relative_deviation <= 1e-6.
"""
import numpy as np
import pytest

from paper_1602_03207_b200 import ect, trace, workloads
from tests.helpers import GOLDEN, golden

GOLD = GOLDEN / "trace_small_6x6x12.csv"
TRACE_Z = (0.0085, 0.0095, 0.0100, 0.0105, 0.0115)


def _points_from(rows):
    return [{"z": z, "dz": v[:4], "z_fa": v[4], "z_f3": v[5], "failed": False} for z, v in rows]


def test_writer_matches_reference_bytes(tmp_path):
    rows = trace.read_trace_csv(GOLD)
    assert [z for z, _ in rows] == list(TRACE_Z)
    out = tmp_path / "t.csv"
    trace.write_trace_csv(out, _points_from(rows), config_hash="small_6x6x12")
    assert out.read_bytes() == GOLD.read_bytes()
    assert trace.max_relative_deviation(rows, trace.read_trace_csv(out)) == 0.0


def test_reference_reader_accepts_our_trace(tmp_path, ref_lib):
    out = tmp_path / "t.csv"
    pts = _points_from(trace.read_trace_csv(GOLD))
    pts[2]["dz"] = [d * (1 + 1e-9) for d in pts[2]["dz"]]
    trace.write_trace_csv(out, pts, config_hash="small_6x6x12")
    dev = ref_lib.trace_max_relative_deviation(GOLD, out)
    assert 0 < dev < 1e-8


@pytest.mark.gpu
def test_gpu_sweep_trace_matches_reference(ctx, tmp_path):
    g = golden("small_6x6x12")
    m = ect.Mesh(ctx, g["xyz"], g["tets"], g["region"])
    phys = workloads.Physics(sigma_defect=1e4, mu_r_defect=5.0)
    s = ect.Session(ctx, m, phys, tuple(g["coil"]), float(g["amplitude"]), tol=1e-11,
                    max_iter=20000)
    pts = s.solve_positions(list(TRACE_Z)[::-1], positions_per_batch=2)  # any order
    out = tmp_path / "gpu.csv"
    trace.write_trace_csv(out, pts, config_hash="small_6x6x12")
    dev = trace.max_relative_deviation(trace.read_trace_csv(GOLD), trace.read_trace_csv(out))
    assert dev <= 1e-6, dev
