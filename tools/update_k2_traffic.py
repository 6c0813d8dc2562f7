"""Refresh profiles/k2_traffic.json from ncu --set full captures of K2.

Usage (in this container, after a GPU run brought the .ncu-rep files back):
    python tools/update_k2_traffic.py KEY REP [KEY REP ...]
KEY is bench.py's capture key (kernel_dist_N_leaf_tol, e.g.
laplace3d_cube_10000000_128_1e-06).  For each capture the record holds
dram__bytes_read.sum + dram__bytes_write.sum ('traffic', bytes per launch),
sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active as a fraction,
the kernel name, its duration and the sha256[:16] of the K2 sources the
capture was taken from (bench.py reports the figures only for those sources).
The raw page of each capture is also written next to the record as
profiles/r02/ncu_<tag>_raw.csv (the details page via --details).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def raw_metrics(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(m: dict, key: str) -> float:
    v, u = m[key]
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
             "GB": 1e9, "B": 1}.get(u, 1)
    return x * scale


def main(argv: list[str]) -> None:
    import bench  # the K2 source hash bench.py checks against

    path = os.path.join(ROOT, "profiles", "k2_traffic.json")
    pj = json.load(open(path))
    sha = bench.k2_source_sha()
    for key, rep in zip(argv[0::2], argv[1::2]):
        m = raw_metrics(rep)
        traffic = num(m, "dram__bytes_read.sum") + num(m, "dram__bytes_write.sum")
        pipe = num(m, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100.0
        dur, unit = m["gpu__time_duration.sum"]
        tag = os.path.basename(rep).replace(".ncu-rep", "")
        details = os.path.join(ROOT, "profiles", "r02", f"ncu_{tag}_final_details.csv")
        with open(details, "w") as fh:
            fh.write(subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], check=True,
                                    capture_output=True, text=True).stdout)
        pj["captures"][key] = {
            "traffic": traffic, "fp64_pipe_active": pipe, "k2_source_sha16": sha,
            "capture": os.path.relpath(details, ROOT),
            "kernel": m.get("Kernel Name", ("?", ""))[0], "duration": f"{dur} {unit}"}
        print(key, f"traffic {traffic / 1e9:.2f} GB, fp64 pipe {pipe:.3f}, {dur} {unit}")
    with open(path, "w") as fh:
        json.dump(pj, fh, indent=1)
        fh.write("\n")


if __name__ == "__main__":
    main(sys.argv[1:])
