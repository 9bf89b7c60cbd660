"""Per-kernel DRAM traffic of the bench workload from ncu (run on the GPU box).

    python scripts/ncu_traffic.py --n 7000000 [--mode auto]

Runs `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum`
over one bench step, maps the library kernels to bench.py's kernel names and writes
profiles/ncu_traffic.json with DRAM bytes per point per kernel (the `traffic` field of the
bench roofline).  ncu times are cold-cache and serialised: only the bytes are used.
"""

import argparse
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench_name(kernel: str):
    if "tc_fwd64_kernel" in kernel or "tc_fwd64w_kernel" in kernel:
        return "tc_forward"
    if "tc_dt64_kernel" in kernel:
        return "tc_dtheta"
    if "knn_grid_query_kernel" in kernel:
        return "knn_grid"
    m = re.search(r"tc_rev64w?_kernel<(?:\(bool\))?(\w+), (?:\(bool\))?(\w+)>", kernel)
    if m:
        return "tc_reverse_dloc" if m.group(2) in ("1", "true") else "tc_reverse"
    m = re.search(r"tc_gmc_kernel<\(?int\)?(\d+), \(?int\)?(\d+), \(?bool\)?(\d), \(?bool\)?(\d), \(?int\)?(\d+), \(?bool\)?(\d)>", kernel)
    if m:
        rev, dloc = m.group(4) == "1", m.group(6) == "1"
        return "tc_reverse_dloc" if dloc else ("tc_reverse" if rev else "tc_forward")
    m = re.search(r"tc_gmc_kernel<(\d+), (\d+), (\d), (\d), (\d+), (\d)>", kernel)
    if m:
        rev, dloc = m.group(4) == "1", m.group(6) == "1"
        return "tc_reverse_dloc" if dloc else ("tc_reverse" if rev else "tc_forward")
    if "tc_dtheta_kernel" in kernel:
        return "tc_dtheta"
    if "gmc_kernel" in kernel:
        return "simt_reverse" if re.search(r"gmc_kernel<[^,]+, \d+, (true|1)", kernel) else "simt_forward"
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=7_000_000)
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--csv", default=None, help="parse an existing ncu CSV instead of running ncu")
    args = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    log = args.csv or os.path.join(ROOT, "gpurun_out", "ncu_traffic.csv")
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:tc_|gmc|dtheta|fwd64|rev64|dt64", "--csv", "--log-file", log,
           sys.executable, os.path.join(ROOT, "bench.py"), "--n", str(args.n), "--steps", "1", "--warmup", "1",
           "--no-cpu", "--no-e2e", "--mode", args.mode]
    if not args.csv:
        subprocess.run(cmd, check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(open(log)))
    hdr = next(r for r in rows if r and r[0] == "ID")
    ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    per = {}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) != len(hdr):
            continue
        name = bench_name(r[ik])
        if not name:
            continue
        val = float(r[iv].replace(",", ""))
        unit = r[iu]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
        d = per.setdefault(name, {"launches": 0, "dram_read": 0.0, "dram_write": 0.0, "ns": 0.0})
        if r[im] == "dram__bytes_read.sum":
            d["dram_read"] += val * scale
        elif r[im] == "dram__bytes_write.sum":
            d["dram_write"] += val * scale
        elif r[im] == "gpu__time_duration.sum":
            d["ns"] += val * scale
            d["launches"] += 1
    out = {"n": args.n, "mode": args.mode, "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
           "(per launch, averaged over the bench step's launches)", "kernels": {}}
    for name, d in per.items():
        L = max(d["launches"], 1)
        out["kernels"][name] = {"launches": d["launches"],
                                "dram_bytes_per_point": (d["dram_read"] + d["dram_write"]) / L / args.n,
                                "dram_read_per_point": d["dram_read"] / L / args.n,
                                "dram_write_per_point": d["dram_write"] / L / args.n,
                                "ncu_ms_cold": d["ns"] / L / 1e6}
    dst = os.path.join(ROOT, "gpurun_out", "ncu_traffic.json")
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
