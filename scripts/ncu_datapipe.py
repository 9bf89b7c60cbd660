"""Per-kernel L1 data-pipe budget from an `ncu --set full` report of the bench workload.

    python scripts/ncu_datapipe.py gpurun_out/<report>.ncu-rep [more reports] [--n 7000000] [--out profiles/ncu_datapipe.json]

The warp-specialised kernels are bound by the SM's L1TEX data pipe (LSU wavefronts: global
gathers, own-row loads/stores and shared-memory traffic), not by HBM.  For each kernel this
writes the data-pipe utilisation (l1tex__data_pipe_lsu_wavefronts, % of peak) and the
wavefronts per point split into global/local (lgds) and shared, plus the tensor-core operand
reads from shared memory (l1tex__data_pipe_tc_wavefronts), issue utilisation and hit rates.
"""
import argparse
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def bench_name(kernel: str):
    from ncu_traffic import bench_name as bn  # same kernel -> bench-name mapping

    return bn(kernel)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="+")
    ap.add_argument("--n", type=int, default=7_000_000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_datapipe.json"))
    args = ap.parse_args()
    out = {"n": args.n, "report": ", ".join(os.path.basename(r) for r in args.report),
           "source": "ncu --set full --clock-control none (one launch per kernel); wavefronts per point = "
                     "SM-average x 148 SMs / n", "kernels": {}}
    for rep in args.report:
        one_report(rep, args, out)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


def one_report(report, args, out):
    raw = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}

    def val(r, k):
        try:
            return float(r[col[k]].replace(",", ""))
        except (KeyError, ValueError):
            return None

    for r in rows[2:]:
        name = bench_name(r[col["Kernel Name"]])
        if not name or name in out["kernels"]:
            continue
        sms = 148
        lg = val(r, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg")
        sh = val(r, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_shared.avg")
        tc = val(r, "l1tex__data_pipe_tc_wavefronts_mem_shared.sum")
        out["kernels"][name] = {
            "kernel": r[col["Kernel Name"]],
            "ncu_ms_cold": val(r, "gpu__time_duration.sum"),
            "l1_data_pipe_frac": round(val(r, "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed") / 100, 4),
            "lsu_wavefronts_per_point": {"global_local": round(lg * sms / args.n, 2) if lg else None,
                                         "shared": round(sh * sms / args.n, 2) if sh else None},
            "tc_smem_wavefronts_per_point": round(tc / args.n, 2) if tc else None,
            "issue_active_frac": round(val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active") / 100, 4),
            "l1_hit_rate": round(val(r, "l1tex__t_sector_hit_rate.pct") / 100, 4),
            "l2_hit_rate": round(val(r, "lts__t_sector_hit_rate.pct") / 100, 4),
            "dram_bytes_per_point": round((val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")) * 1e9 / args.n, 1),
            "registers_per_thread": val(r, "launch__registers_per_thread"),
            "tensor_pipe_frac": (round(val(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active") / 100, 4)
                                 if val(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active") is not None
                                 else None),
            "fp64_pipe_frac": (round(val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100, 4)
                               if val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") is not None
                               else None),
            "warps_active_per_smsp": val(r, "smsp__warps_active.avg.per_cycle_active"),
            "bank_conflict_wavefronts_per_point": (round(val(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum") / args.n, 2)
                                                   if val(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum") else None),
        }


if __name__ == "__main__":
    main()
