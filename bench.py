"""Benchmark: flex_conv forward + backward points/sec on B200 (BASELINE.json metric).

Workload (config C4 shape, with the backward the metric names): one flex-conv layer on a
single synthetic uniform-random cloud of N = 7,000,000 points, K = 8 (kNN, self
included), 64 -> 64 channels, Dp = 3, fp32 I/O.  A step = forward (out) + full backward
(d_features, d_theta, d_theta_b, d_locations) -- the reference harness's fwd and
bwd-with-locations pair (harness.py:520-527).  Neighbourhood (kNN) and reverse CSR are
built once before timing (as harness.py:516-517 does) and reported separately.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--mode M]

N > 1 (torchrun, one rank per GPU): weak scaling -- each rank runs its own 7M-point cloud
and the theta/theta_b gradients are all-reduced over NCCL every step (the data-parallel
training collective); value = all points / max-over-ranks time.
--impl reference: the reference's own CPU kernels (oracle/_ref, built from
/root/reference by oracle/build_ref.sh; else the C restatement in oracle/) on the host
cores, rank 0 only, a bounded sample per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "flex_conv fwd+bwd points/sec (1M-7M pts, K=8, 64->64)"
UNIT = "points/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--points", dest="n", type=int, default=7_000_000)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--c", type=int, default=64)
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--cpu-sample", type=int, default=131072)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp64", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: host-staged transport, only to exercise N ranks on one GPU")
    ap.add_argument("--shard", default=None, choices=["points", "clouds"],
                    help="N > 1: 'points' (default) = ONE n-point cloud point-chunk sharded with halos over "
                         "the ranks (strong scaling, the north_star's 7M cloud on 8 GPUs); 'clouds' = an "
                         "independent n-point cloud per rank (weak scaling)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1590.0)), "measured"
    return 6650.0, 1590.0, "fallback"


def algo_bytes_per_point(c_in, c_out, d, k, s=4):
    """compulsory bytes per point (fp32 I/O, int32 indices)."""
    fwd = s * c_in + 4 * d + 4 * k + s * c_out
    bwd = s * c_out + s * c_in + 4 * d + 4 * k + (4 + 4 * k) + s * c_in + 4 * d
    return fwd, bwd


def kernel_bytes_per_point(name, c_in, c_out, d, k, s=4):
    """Algorithmic bytes per centre point that each library kernel must move (every
    tensor it reads or writes once)."""
    table = {
        # features + positions + neighbour row in, output row out
        "tc_forward": s * c_in + 4 * d + 4 * k + s * c_out,
        "simt_forward": s * c_in + 4 * d + 4 * k + s * c_out,
        # + upstream row in, centre-role location term out
        "tc_dtheta": s * c_in + 4 * d + 4 * k + s * c_out + 4 * d,
        # upstream + positions + reverse CSR (offset + k entries on average) + own features
        # + centre term in; d_features + d_locations out
        "tc_reverse_dloc": s * c_out + 4 * d + (4 + 4 * k) + s * c_in + 4 * d + s * c_in + 4 * d,
        "tc_reverse": s * c_out + 4 * d + (4 + 4 * k) + s * c_in,
        "simt_reverse": s * c_out + 4 * d + (4 + 4 * k) + s * c_in + s * c_in + 4 * d + 4 * d,
    }
    return table.get(name)


def ncu_traffic(name):
    """DRAM bytes per point of kernel `name` from the committed ncu capture summary
    (profiles/ncu_traffic.json, written by scripts/ncu_traffic.py), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    return d.get("kernels", {}).get(name, {}).get("dram_bytes_per_point")


def ncu_datapipe(name):
    """The kernel's L1 data-pipe budget (profiles/ncu_datapipe.json, written by
    scripts/ncu_datapipe.py from an ncu --set full capture of this workload), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_datapipe.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    k = d.get("kernels", {}).get(name)
    if not k:
        return None
    return {"l1_data_pipe_frac": k["l1_data_pipe_frac"], "lsu_wavefronts_per_point": k["lsu_wavefronts_per_point"],
            "tc_smem_wavefronts_per_point": k["tc_smem_wavefronts_per_point"]}


def tensor_pipe(kern, c_in, c_out, d, n, bf16_peak):
    """Tensor-pipe side of the roofline for the contraction kernels: algorithmic contraction
    flops per point (2*Din*(Dp+1)*Dout for the forward / d_features, the same
    for d_theta) over the measured kernel time, against the measured dense bf16 peak, beside
    ncu's sm__pipe_tensor_cycles_active for the same kernel (profiles/ncu_datapipe.json)."""
    flops = 2 * c_in * (d + 1) * c_out
    per_kernel = {"tc_forward": flops, "tc_dtheta": flops, "tc_reverse_dloc": 2 * flops, "tc_reverse": flops,
                  "tc_reverse_dtheta": 2 * flops}
    out = {"unit": "TFLOP/s", "peak": bf16_peak, "peak_source": "MEASURED_PEAKS.json bf16_tflops (dense, burst)",
           "flops_per_point": "2*Din*(Dp+1)*Dout per contraction (d_features + d_theta in the reverse kernel)",
           "kernels": {}}
    p = os.path.join(ROOT, "profiles", "ncu_datapipe.json")
    ncu = {}
    if os.path.exists(p):
        with open(p) as fh:
            ncu = json.load(fh).get("kernels", {})
    for name, ms in kern.items():
        if name not in per_kernel:
            continue
        tf = per_kernel[name] * n / (ms / 1e3) / 1e12
        out["kernels"][name] = {"achieved": round(tf, 2), "frac": round(tf / bf16_peak, 4),
                                "ncu_pipe_tensor_active_frac": ncu.get(name, {}).get("tensor_pipe_frac")}
    return out


def knn_roofline(knn_ms, n, k, d, hbm):
    """The exact grid kNN (setup, timed with CUDA events around the whole builder: bbox, grid,
    bucket sort, query) against SURVEY.md §8(d)'s compulsory bytes (positions in, K int32
    indices out: 4*Dp + 4*K per point), beside what ncu says bounds its query kernel
    (profiles/ncu_datapipe.json: issue / fp64-pipe utilisation -- the query loop evaluates
    fp64 candidate distances, so it is latency/compute-bound, not HBM-bound)."""
    b = 4 * d + 4 * k
    gbs = b * n / (knn_ms / 1e3) / 1e9
    out = {"bound": "hbm", "ms": round(knn_ms, 3), "bytes_per_point": b, "achieved": round(gbs, 1),
           "unit": "GB/s", "peak": hbm, "frac": round(gbs / hbm, 4),
           "points_per_s": round(n / (knn_ms / 1e3), 1)}
    p = os.path.join(ROOT, "profiles", "ncu_datapipe.json")
    if os.path.exists(p):
        with open(p) as fh:
            kq = json.load(fh).get("kernels", {}).get("knn_grid")
        if kq:
            out["query_kernel_limiter"] = {x: kq.get(x) for x in ("ncu_ms_cold", "issue_active_frac", "fp64_pipe_frac",
                                                                    "l1_data_pipe_frac", "warps_active_per_smsp",
                                                                    "dram_bytes_per_point")}
            out["query_kernel_limiter"]["source"] = "profiles/ncu_datapipe.json"
    return out


def run_fp64(args, torch, _ops, feat, pos, nbr, csr, g, theta, theta_b, n, steps=2):
    f64 = [t.double() for t in (feat, pos, g, theta, theta_b)]
    torch.cuda.synchronize()

    def step():
        _ops.conv_forward(f64[0], f64[1], nbr, f64[3], f64[4], 1, n)
        _ops.conv_backward(f64[2], f64[0], f64[1], nbr, csr, f64[3], f64[4], 1, n, need=(True, True, True, True))

    step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    del f64
    return {"value": round(n / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 3), "steps": steps,
            "dtype": "f64", "note": "reported only: the reference's fp64 arithmetic on the GPU (SIMT fp64, forward "
                                    "bitwise equal to _native); the headline is the fp32-accurate engine"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        try:  # NVML (what nvidia-smi reads), sampled every 10 ms
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append([str(self.gpu), str(sm), str(mx), "", hex(rs)] +
                                 ["Active" if rs & b else "Not Active" for b in bits])
                self._stop.wait(0.01)
            return
        except Exception:  # noqa: BLE001 -- fall back to nvidia-smi
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._th.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU reference / baseline
def cpu_kernels():
    """The reference's own compiled kernels (oracle/_ref) if built, else the C restatement."""
    from oracle import oracle

    nat = oracle.ref_native()
    if nat is not None:
        return "reference", nat
    oracle.build()
    return "port", None


def cpu_sample(n_sample, k, c, seed=4):
    """A bounded sample of the workload: an n_sample-point cloud of the same construction.
    Nothing from the product package is loaded on this leg: the inputs come from numpy
    (paper_1803_07289_b200/core.py's generator is mirrored by oracle.synthetic_layer) and
    the neighbour table from the oracle's OpenMP brute-force kNN."""
    from oracle import oracle

    loc, feat, th, tb, up = oracle.synthetic_layer(seed, 0, n_sample, 3, c, c)
    nbr = oracle.knn_brute(loc, k)
    return loc, feat, th, tb, up, nbr


def time_cpu_step(kind, nat, sample):
    """One fwd + bwd(with locations) of the reference kernels on the sample; seconds."""
    from oracle import oracle

    loc, feat, th, tb, up, nbr = sample
    nthreads = os.cpu_count() or 1
    t0 = time.perf_counter()
    if kind == "reference":
        out = np.empty((feat.shape[0], th.shape[0]))
        nat.flex_conv_forward(feat, loc, nbr, th, tb, out, nthreads)
        t1 = time.perf_counter()
        bufs = [np.zeros_like(feat), np.zeros_like(loc), np.zeros_like(th), np.zeros_like(tb)]
        nat.flex_conv_backward(up, feat, loc, nbr, th, tb, bufs[0], bufs[1], bufs[2], bufs[3], True)
    else:
        oracle.conv_forward(feat, loc, nbr, th, tb, num_threads=nthreads)
        t1 = time.perf_counter()
        oracle.conv_backward(up, feat, loc, nbr, th, tb, True)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


# ------------------------------------------------------------------ workload
def make_cloud(n, c, seed, dev, d=3):
    """The synthetic layer inputs: positions on the 2^-24 lattice (exact in fp32), spatially
    ordered once; features / upstream N(0,1), theta / theta_b 0.1 N(0,1).  Returns the
    tensors and the spatial-order time (ms)."""
    import torch

    from paper_1803_07289_b200 import _ops

    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    pos = torch.floor(torch.rand(n, d, generator=gen, device=dev, dtype=torch.float64) * 2 ** 24) / 2 ** 24
    pos = pos.to(torch.float32)
    torch.cuda.synchronize()
    _ops.spatial_order(pos)  # first call: module load + memory-pool growth (not reported)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    order = _ops.spatial_order(pos)
    pos = pos[order.long()].contiguous()
    torch.cuda.synchronize()
    sort_ms = (time.perf_counter() - t0) * 1e3
    feat = torch.randn(n, c, generator=gen, device=dev)
    g = torch.randn(n, c, generator=gen, device=dev)
    theta = 0.1 * torch.randn(c, c, d, generator=gen, device=dev)
    theta_b = 0.1 * torch.randn(c, c, generator=gen, device=dev)
    return {"pos": pos, "feat": feat, "g": g, "theta": theta, "theta_b": theta_b, "sort_ms": sort_ms}


def make_workload(n, k, c, rank, dev, d=3):
    """The bench's synthetic layer on `dev` (tests/test_gpu_scale.py checks this exact
    workload against the oracle): make_cloud + the exact kNN table and reverse CSR, their
    setup costs timed with CUDA events."""
    import torch

    from paper_1803_07289_b200 import _ops

    w = make_cloud(n, c, 1234 + rank, dev, d)
    pos, feat, g, theta, theta_b, sort_ms = (w[x] for x in ("pos", "feat", "g", "theta", "theta_b", "sort_ms"))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nbr = _ops.knn(pos, 1, n, k)  # first call: scratch-pool growth, not reported
    knn_times = []
    for _ in range(3):  # the kNN builder (bbox, grid, bucket sort, query), median of 3 warm calls
        e0.record()
        nbr = _ops.knn(pos, 1, n, k)
        e1.record()
        torch.cuda.synchronize()
        knn_times.append(e0.elapsed_time(e1))
    knn_ms = statistics.median(knn_times)
    e0.record()
    csr = _ops.csr_build(nbr, 1, n)
    e1.record()
    torch.cuda.synchronize()
    csr_ms = e0.elapsed_time(e1)
    return {"pos": pos, "feat": feat, "g": g, "theta": theta, "theta_b": theta_b, "nbr": nbr, "csr": csr,
            "sort_ms": sort_ms, "knn_ms": knn_ms, "csr_ms": csr_ms}


# ------------------------------------------------------------------ distributed
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist

    local = local % torch.cuda.device_count()  # (ranks share a GPU only in --backend gloo tests)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    shard = args.shard or ("points" if world > 1 else "clouds")
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    if shard == "points":
        return run_sharded(args, world, rank, local, dev)

    from paper_1803_07289_b200 import _lib, _ops

    n, k, c, d = args.n, args.k, args.c, 3
    w = make_workload(n, k, c, rank, dev)
    pos, feat, g, theta, theta_b, nbr, csr = (w[x] for x in ("pos", "feat", "g", "theta", "theta_b", "nbr", "csr"))
    sort_ms, knn_ms, csr_ms = w["sort_ms"], w["knn_ms"], w["csr_ms"]

    def step(phase_events=None):
        if phase_events:
            phase_events[0].record()
        _ops.conv_forward(feat, pos, nbr, theta, theta_b, 1, n, args.mode)
        if phase_events:
            phase_events[1].record()
        _, dth, dtb, _ = _ops.conv_backward(g, feat, pos, nbr, csr, theta, theta_b, 1, n,
                                            need=(True, True, True, True), mode=args.mode)
        if phase_events:
            phase_events[2].record()
        if world > 1:
            flat = torch.cat([dth.reshape(-1), dtb.reshape(-1)])
            dist.all_reduce(flat)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    launches0 = _lib.launch_count()
    phases = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for s in range(args.steps):
            step(phases[s])
        stop.record()
        torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    ms_total = start.elapsed_time(stop)
    if world > 1:
        t = torch.tensor([ms_total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    fwd_ms = statistics.median(p[0].elapsed_time(p[1]) for p in phases)
    bwd_ms = statistics.median(p[1].elapsed_time(p[2]) for p in phases)
    value = world * n / (ms_step / 1e3)

    # ---------------- e2e: host buffers through the C ABI, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, torch, _ops, feat, pos, nbr, g, theta, theta_b, n, k, world, dist)

    # ---------------- per-kernel device times (library CUDA events on the launching stream),
    # taken in a separate pass after the timed region so the timed region stays clean
    with _lib.KernelTimer() as kt:
        for _ in range(max(1, min(args.steps, 5))):
            step()
    kern = {name: statistics.mean(v) for name, v in kt.times.items() if v and min(v) >= 0}

    # ---------------- the reference's own arithmetic (fp64 engine, bitwise forward), reported
    # only: the same workload cast to fp64, CUDA events, a few steps after the timed region
    fp64 = None
    if not args.no_fp64:
        fp64 = run_fp64(args, torch, _ops, feat, pos, nbr, csr, g, theta, theta_b, n)

    hbm, bf16, src = peaks()
    fwd_b, bwd_b = algo_bytes_per_point(c, c, d, k)
    kernels = {}
    for name, ms in kern.items():
        b = kernel_bytes_per_point(name, c, c, d, k)
        kernels[name] = {"ms": round(ms, 4), "bytes_per_point": b,
                         "GBps": round(b * n / ms / 1e6, 1) if b else None,
                         "frac": round(b * n / ms / 1e6 / hbm, 4) if b else None}
        # the gathered bytes (K neighbour rows + positions per point, read
        # through L1/L2) beside the compulsory ones -- the traffic the gathers actually move
        gb = k * (4 * c + 4 * d)
        kernels[name]["gathered_bytes_per_point"] = gb
        kernels[name]["gathered_GBps"] = round(gb * n / ms / 1e6, 1)
        dp = ncu_datapipe(name)
        if dp:  # the binding on-chip limit (ncu), beside the HBM roofline
            kernels[name]["limiter"] = dict(dp, source="profiles/ncu_datapipe.json")
    dom = max(kern, key=kern.get) if kern else None
    if dom is not None and kernel_bytes_per_point(dom, c, c, d, k):
        dom_b, dom_ms = kernel_bytes_per_point(dom, c, c, d, k), kern[dom]
    else:
        dom, dom_b, dom_ms = "conv_backward", bwd_b, bwd_ms
    achieved = dom_b * n / (dom_ms / 1e3) / 1e9
    traffic = ncu_traffic(dom)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4),
                "traffic": round(traffic * n) if traffic else None,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read+write)" if traffic else None,
                "peak_source": src + " (MEASURED_PEAKS.json hbm_gbs)" if src == "measured" else src,
                "algorithmic_bytes_per_point": dom_b, "kernels": kernels,
                "phases": {"forward": {"ms": round(fwd_ms, 4), "bytes_per_point": fwd_b,
                                       "GBps": round(fwd_b * n / fwd_ms / 1e6, 1)},
                           "backward": {"ms": round(bwd_ms, 4), "bytes_per_point": bwd_b,
                                        "GBps": round(bwd_b * n / bwd_ms / 1e6, 1)}}}

    roofline["tensor"] = tensor_pipe(kern, c, c, d, n, bf16)
    roofline["knn"] = knn_roofline(knn_ms, n, k, d, hbm)

    cpu = None
    if rank == 0 and not args.no_cpu:
        kind, nat = cpu_kernels()
        sample = cpu_sample(args.cpu_sample, k, c)
        tf, tb_ = time_cpu_step(kind, nat, sample)
        cpu = {"value": round(args.cpu_sample / (tf + tb_), 1), "unit": UNIT, "cores": os.cpu_count(),
               "kind": kind,
               "sample": f"{args.cpu_sample}-point cloud, K={k}, {c}->{c}, fwd {tf:.2f}s on "
                         f"{os.cpu_count()} threads + bwd {tb_:.2f}s (single-threaded by reference design, "
                         f"_native.pyx:77-78), fp64"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"flex_conv fwd+bwd (with d_locations), one {n}-point uniform cloud "
                                   f"per GPU, K={k}, {c}->{c}, Dp=3",
                       "points_per_gpu": n, "k": k, "c_in": c, "c_out": c, "dp": d, "mode": args.mode,
                       "parallelism": f"dp{world}" if world > 1 else "single",
                       "l2": "inputs (>= 1.8 GB) exceed the 126 MB L2; no flush needed",
                       "setup_ms": {"spatial_order": round(sort_ms, 2), "knn": round(knn_ms, 3),
                                    "reverse_csr": round(csr_ms, 3)}},
            "gpu_launches": launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "fp64_engine": fp64,
            "e2e": e2e,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline_line(args, k, c):
    kind, nat = cpu_kernels()
    sample = cpu_sample(args.cpu_sample, k, c)
    tf, tb_ = time_cpu_step(kind, nat, sample)
    return {"value": round(args.cpu_sample / (tf + tb_), 1), "unit": UNIT, "cores": os.cpu_count(), "kind": kind,
            "sample": f"{args.cpu_sample}-point cloud, K={k}, {c}->{c}, fwd {tf:.2f}s on {os.cpu_count()} threads + "
                      f"bwd {tb_:.2f}s (single-threaded by reference design, _native.pyx:77-78), fp64"}


def run_sharded(args, world, rank, local, dev):
    """ONE n-point cloud, point-chunk sharded with halos over the ranks (parallel.ShardedCloud):
    each rank keeps its block of the spatially ordered cloud, builds its exact kNN rows with
    the ghost-shell exchange (no global table anywhere), and a step is the sharded layer's
    forward (halo gather + kernels) and training backward (kernels, halo partials back to
    their owners, ordered d_theta sum).  value = n / max-over-ranks step time (strong)."""
    import torch
    import torch.distributed as dist

    from paper_1803_07289_b200 import _lib, parallel

    n, k, c, d = args.n, args.k, args.c, 3
    w = make_cloud(n, c, 1234, dev)  # the same cloud on every rank; each keeps its block
    lo, hi = parallel.shard_range(n, world, rank)
    pos, feat, g = (w[x][lo:hi].contiguous() for x in ("pos", "feat", "g"))
    theta, theta_b = w["theta"], w["theta_b"]
    del w
    torch.cuda.empty_cache()
    comm = parallel.Comm(device=dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cloud = parallel.ShardedCloud.build(pos, k, comm)
    torch.cuda.synchronize()
    build_ms = (time.perf_counter() - t0) * 1e3
    layer = parallel.ShardedFlexConv(cloud)
    # the layer's inputs live in [owned | halo] buffers (what a network's previous layer
    # would write into); the halo rows are exchanged inside every step
    feat_l, g_l = cloud.local_buffer(feat), cloud.local_buffer(g)

    def step():
        layer.forward(feat_l, theta, theta_b)
        layer.backward(g_l)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            step()
        b.record()
        torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    ms = a.elapsed_time(b)
    stats = torch.tensor([ms, cloud.halo_fraction, build_ms, cloud.n_ghost / max(cloud.n_own, 1)], device=dev,
                         dtype=torch.float64)
    gathered = comm.all_gather(stats) if world > 1 else [stats]
    ms = max(float(t[0]) for t in gathered)
    ms_step = ms / args.steps
    with _lib.KernelTimer() as kt:
        for _ in range(max(1, min(args.steps, 5))):
            step()
    kern = {name: statistics.mean(v) for name, v in kt.times.items() if v and min(v) >= 0}
    hbm, bf16, src = peaks()
    n_loc = cloud.n_local
    kernels = {}
    for name, kms in kern.items():
        bpp = kernel_bytes_per_point(name, c, c, d, k)
        kernels[name] = {"ms": round(kms, 4), "bytes_per_point": bpp, "rows": n_loc,
                         "GBps": round(bpp * n_loc / kms / 1e6, 1) if bpp else None,
                         "frac": round(bpp * n_loc / kms / 1e6 / hbm, 4) if bpp else None}
    dom = max((nm for nm in kern if kernel_bytes_per_point(nm, c, c, d, k)), key=kern.get, default=None)
    roofline = None
    if dom:
        ach = kernel_bytes_per_point(dom, c, c, d, k) * n_loc / (kern[dom] / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(ach / hbm, 4), "traffic": None, "peak_source": src,
                    "note": f"rank 0's shard ({n_loc} local rows incl. halo)", "kernels": kernels}
    # e2e: every step each rank copies its owned inputs in from pinned host buffers and its
    # results (forward output, d_features, d_locations, d_theta, d_theta_b) back out
    e2e = None
    if not args.no_e2e:
        host_in = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t) for t in (feat, g)]
        host_out = [torch.empty(s_, dtype=torch.float32, pin_memory=True)
                    for s_ in ((hi - lo, c), (hi - lo, c), (hi - lo, d), tuple(theta.shape), tuple(theta_b.shape))]

        def e2e_step():  # H2D straight into the owned rows of the layer's local buffers
            feat_l[: cloud.n_own].copy_(host_in[0], non_blocking=True)
            g_l[: cloud.n_own].copy_(host_in[1], non_blocking=True)
            out = layer.forward(feat_l, theta, theta_b)
            host_out[0].copy_(out, non_blocking=True)
            df, dth, dtb, dl = layer.backward(g_l)
            for h, t in zip(host_out[1:], (df, dl, dth, dtb)):
                h.copy_(t, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e_steps = max(1, min(args.steps, 10))
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record()
        for _ in range(e_steps):
            e2e_step()
        eb.record()
        torch.cuda.synchronize()
        ems = torch.tensor([ea.elapsed_time(eb) / e_steps], device=dev, dtype=torch.float64)
        ems = max(float(t[0]) for t in comm.all_gather(ems)) if world > 1 else float(ems[0])
        e2e = {"value": round(n / (ems / 1e3), 1), "unit": UNIT,
               "h2d_bytes_per_step": sum(t.numel() * t.element_size() for t in host_in) * world,
               "d2h_bytes_per_step": sum(t.numel() * t.element_size() for t in host_out) * world,
               "ms_per_step": round(ems, 3), "steps": e_steps,
               "path": "per rank: owned features / upstream H2D from pinned host buffers, sharded forward + "
                       "backward (halo exchanges over NCCL), owned results + theta gradients D2H (bytes summed "
                       "over ranks)"}
    cpu = cpu_baseline_line(args, k, c) if (rank == 0 and not args.no_cpu) else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(n / (ms_step / 1e3), 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"flex_conv fwd+bwd (with d_locations) on ONE {n}-point uniform cloud, K={k}, "
                                   f"{c}->{c}, Dp=3, point-chunk sharded with halos over {world} GPU(s)",
                       "points_total": n, "k": k, "c_in": c, "c_out": c, "dp": d, "parallelism": f"points{world}",
                       "halo_fraction_max": round(max(float(t[1]) for t in gathered), 4),
                       "ghost_fraction_max": round(max(float(t[3]) for t in gathered), 4),
                       "setup_ms": {"sharded_knn_and_plan_max": round(max(float(t[2]) for t in gathered), 2)},
                       "l2": "inputs exceed the 126 MB L2; no flush needed"},
            "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
            "e2e": e2e, "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, torch, _ops, feat, pos, nbr, g, theta, theta_b, n, k, world, dist):
    """Same metric through the C ABI with pinned HOST buffers: every step copies the inputs
    H2D, rebuilds the reverse neighbourhood, runs fwd + bwd and copies the results D2H."""
    dev = feat.device
    # pinned host buffers filled straight from the device (no pageable intermediate: at N
    # ranks per box this is N x 7.6 GB of page-locked memory, not 2x that transiently)
    outs_shape = [(n, theta.shape[0]), (n, feat.shape[1]), tuple(theta.shape), tuple(theta_b.shape), (n, 3)]
    ok, err = 1, ""
    try:
        host_in = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t)
                   for t in (feat, pos, nbr, g, theta, theta_b)]
        host_out = [torch.empty(s, dtype=torch.float32, pin_memory=True) for s in outs_shape]
    except (RuntimeError, MemoryError) as exc:  # e.g. page-locking failed on a small host
        ok, err = 0, f"{type(exc).__name__}: {str(exc)[:200]}"
    if world > 1:  # every rank takes the same branch (no rank left waiting in a collective)
        flag = torch.tensor([ok], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        ok = int(flag.item())
    if not ok:
        return {"value": None, "unit": UNIT, "error": err or "pinned host buffers unavailable on another rank"}
    h2d = sum(t.numel() * t.element_size() for t in host_in)
    d2h = sum(t.numel() * t.element_size() for t in host_out)
    steps = max(1, min(args.steps, 10))  # steady state: the pipeline fill / drain is amortised over the steps

    # Copies overlap where the data dependencies allow, on two copy streams that never wait
    # for each other: s_in carries every H2D back to back (the forward's inputs, then the
    # upstream gradient; the next step's inputs queue right behind), s_out every D2H (the
    # forward's output as soon as it exists, then the gradients).  The compute stream waits
    # only for its inputs -- not for the previous step's result copies -- so the H2D link
    # (3.9 GB per step) stays busy and the D2H (3.7 GB) runs underneath it.  The reverse-
    # neighbourhood build validates the indices (host-synchronising, like the reference's
    # range check) on its own stream: the host waits for this step's neighbour table only.
    main = torch.cuda.current_stream()
    s_in, s_out, s_csr = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

    def one():
        with torch.cuda.stream(s_in):
            f, p, nb, th, tb = (host_in[i].to(dev, non_blocking=True) for i in (0, 1, 2, 4, 5))
            ev_in = torch.cuda.Event()
            ev_in.record(s_in)
            gg = host_in[3].to(dev, non_blocking=True)
            ev_g = torch.cuda.Event()
            ev_g.record(s_in)
        for t in (f, p, nb, th, tb, gg):
            t.record_stream(main)
        nb.record_stream(s_csr)
        with torch.cuda.stream(s_csr):
            s_csr.wait_event(ev_in)
            csr = _ops.csr_build(nb, 1, n)
        for t in csr:
            t.record_stream(main)
        main.wait_stream(s_csr)
        main.wait_event(ev_in)
        out = _ops.conv_forward(f, p, nb, th, tb, 1, n, args.mode)
        ev_f = torch.cuda.Event()
        ev_f.record(main)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_f)
            host_out[0].copy_(out, non_blocking=True)
        out.record_stream(s_out)
        main.wait_event(ev_g)
        res = _ops.conv_backward(gg, f, p, nb, csr, th, tb, 1, n, mode=args.mode)
        ev_b = torch.cuda.Event()
        ev_b.record(main)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_b)
            for h, dv in zip(host_out[1:], res):
                h.copy_(dv, non_blocking=True)
        for dv in res:
            dv.record_stream(s_out)

    one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        one()
    main.wait_stream(s_out)  # the stop event covers the last step's result copies
    main.wait_stream(s_in)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": round(world * n / (ms / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 3), "steps": steps,
            "path": "C ABI (fc_csr_build + fc_conv_forward + fc_conv_backward), pinned host fp32 buffers; "
                    "all H2D back to back on one copy stream, all D2H on another (forward output as soon as it "
                    "exists, then the gradients), compute waiting only for its inputs; the index-validating "
                    "reverse-CSR build on a side stream"}


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU kernels on the host cores (rank 0 only)."""
    if rank != 0:
        return
    kind, nat = cpu_kernels()
    n_sample = min(args.cpu_sample, 65536)
    sample = cpu_sample(n_sample, args.k, args.c)
    for _ in range(args.warmup):
        time_cpu_step(kind, nat, sample)
    t0 = time.perf_counter()
    fw = bw = 0.0
    for _ in range(args.steps):
        a, b = time_cpu_step(kind, nat, sample)
        fw += a
        bw += b
    total = time.perf_counter() - t0
    ms_step = total / args.steps * 1e3
    value = n_sample / (total / args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"flex_conv fwd+bwd (with d_locations), K={args.k}, {args.c}->{args.c}, Dp=3; "
                               f"each step a {n_sample}-point sample of the {args.n}-point workload",
                   "points_per_step": n_sample, "parallelism": "cpu"},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": os.cpu_count(), "kind": kind,
                         "sample": f"{n_sample}-point cloud per step; fwd on {os.cpu_count()} threads "
                                   f"({fw / args.steps:.2f}s), bwd single-threaded by reference design "
                                   f"({bw / args.steps:.2f}s)"},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
