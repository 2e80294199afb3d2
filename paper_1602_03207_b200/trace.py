"""Impedance trace I/O in the reference's CSV format.

Restates write_trace_csv / read_trace_csv / max_relative_deviation
(/root/reference/proj/core/src/scan.cpp:170-272) so a GPU sweep produces the
same file `ect scan` writes and can be diffed against it in one command
(`python -m paper_1602_03207_b200.trace a.csv b.csv`).
"""
from __future__ import annotations

import sys


def _g12(v: float) -> str:
    return "%.12g" % v


def write_trace_csv(path, points, config_hash="", workers=1, parts=1, factorizations=0,
                    timing=None):
    """points: dicts with z, dz (4 complex: Z11, Z12, Z21, Z22), z_fa, z_f3, failed
    (ect.Session.solve_positions output). Rows sorted by z (scan.cpp:188-190)."""
    t = {"mesh": 0.0, "partition": 0.0, "assemble": 0.0, "reduce": 0.0, "factorize": 0.0,
         "solve": 0.0, "total": 0.0}
    t.update(timing or {})
    with open(path, "w") as out:
        out.write("# ectsim impedance trace\n")
        out.write(f"# config {config_hash}\n")
        out.write(f"# workers {workers} parts {parts} factorizations {factorizations}\n")
        out.write("# timing mesh=%.3f partition=%.3f assemble=%.3f reduce=%.3f factorize=%.3f "
                  "solve=%.3f total=%.3f\n" % (t["mesh"], t["partition"], t["assemble"],
                                              t["reduce"], t["factorize"], t["solve"],
                                              t["total"]))
        out.write("z_m,re_Z11,im_Z11,re_Z12,im_Z12,re_Z21,im_Z21,re_Z22,im_Z22,"
                  "re_ZFA,im_ZFA,re_ZF3,im_ZF3\n")
        for p in sorted(points, key=lambda p: p["z"]):
            if p.get("failed"):
                out.write(f"# failed position z={p['z']:g}\n")
                continue
            dz = list(p["dz"])
            vals = [p["z"]]
            for c in dz + [p["z_fa"], p["z_f3"]]:
                vals += [complex(c).real, complex(c).imag]
            out.write(",".join(_g12(v) for v in vals) + "\n")


def read_trace_csv(path):
    """Rows of (z, [Z11, Z12, Z21, Z22, Z_FA, Z_F3]) (scan.cpp:209-250)."""
    rows, header = [], False
    with open(path) as f:
        for line in f:
            line = line.rstrip("\n")
            if not line or line.startswith("#"):
                continue
            if not header:
                if not line.startswith("z_m"):
                    raise ValueError(f"{path}: missing trace header row")
                header = True
                continue
            v = [float(c) for c in line.split(",")]
            if len(v) != 13:
                raise ValueError(f"{path}: malformed trace row")
            rows.append((v[0], [complex(v[1 + 2 * i], v[2 + 2 * i]) for i in range(6)]))
    if not header:
        raise ValueError(f"{path}: not a trace file")
    return rows


def max_relative_deviation(a, b) -> float:
    """scan.cpp:252-272: max over signals of |x - y| / max(|x|, |y|)."""
    if len(a) != len(b):
        raise ValueError("traces have different lengths and cannot be compared")
    worst = 0.0
    for (_, xa), (_, xb) in zip(a, b):
        for x, y in zip(xa, xb):
            scale = max(abs(x), abs(y))
            if scale:
                worst = max(worst, abs(x - y) / scale)
    return worst


if __name__ == "__main__":
    print(max_relative_deviation(read_trace_csv(sys.argv[1]), read_trace_csv(sys.argv[2])))
