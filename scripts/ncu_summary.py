"""Summarise an ncu capture of the SpMV kernel + a launch list into the JSON
bench.py reads for roofline.traffic (profiles/spmv_ncu_summary.json).

  python scripts/ncu_summary.py REPORT.ncu-rep|RAW.csv LAUNCHES.csv OUT.json \
      --command "..." --capture "..." --format-bytes B

REPORT may also be the `ncu -i REPORT --page raw --csv` export (made on the GPU
box, where the report itself is too large to bring back).
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

KEEP = ["sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size"]


def raw(report):
    if report.endswith(".csv"):
        out = open(report).read()
    else:
        out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def scale(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
    return float(v.replace(",", "")) * f.get(unit, 1)


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    per = defaultdict(list)
    for r in csv.DictReader(lines[start:]):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            per[r["Kernel Name"]].append(scale(r["Metric Value"], r["Metric Unit"]))
    tot = sum(sum(v) for v in per.values())
    return {k.split("(")[0].replace("(anonymous namespace)::", ""): {
        "launches": len(v), "mean_us": 1e6 * sum(v) / len(v), "share": sum(v) / tot}
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("launch_csv")
    ap.add_argument("out")
    ap.add_argument("--command", default="")
    ap.add_argument("--capture", default="")
    ap.add_argument("--format-bytes", type=int, default=0)
    a = ap.parse_args()
    h, units, rows = raw(a.report)

    def one(v):
        get = lambda n: scale(v[h.index(n)], units[h.index(n)])
        rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
        dur = get("gpu__time_duration.sum")
        return {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "",
                "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                "duration_s_cold": dur, "dram_GBps_cold": (rd + wr) / dur / 1e9,
                "metrics": {n: {"value": v[h.index(n)], "unit": units[h.index(n)]}
                            for n in KEEP if n in h}}

    kernels = [one(v) for v in rows if len(v) == len(h)]
    first = kernels[0]
    for k in kernels:  # bench.py reads the COCG SpMV's traffic
        if "k_nbe_spmv" in k["kernel"]:
            first = k
    summary = {**first, "command": a.command, "capture": a.capture,
               "nb_format_compulsory_bytes": a.format_bytes,
               "all_captured_kernels": kernels,
               "launch_list_shares": launches(a.launch_csv)}
    json.dump(summary, open(a.out, "w"), indent=1)
    print(json.dumps({k: summary[k] for k in ("kernel", "dram_bytes_per_launch", "duration_s_cold",
                                                "dram_GBps_cold")}))


if __name__ == "__main__":
    main()
