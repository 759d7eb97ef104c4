#!/usr/bin/env python3
"""Throughput benchmark of the B200-native ESDG shallow-water RHS (driver contract).

Workload (BASELINE.json configs[3], "C4"): modal (hybridized) ESDG, N = 4,
K1D = 1024 (K = 2,097,152 curved triangles, warp 0.1), periodic [-1,1]^2,
smooth-wave state (tests/test_solver.cpp:14-25 generator, seed 23) over the
lake bathymetry, g = 9.81, Lax-Friedrichs interface flux, LSRK45 in FP64.

A bench "step" is one LSRK45 time step = 5 RHS stages + register updates over
all K elements.  Metric: GDOF·RK-stages/s with DOF = K·Np·3.
`value` is measured on the device-resident state (CUDA events on the
handle's stream; max over ranks); `e2e` goes through the public C ABI with
pinned HOST buffers (H2D of the state, one step, D2H of the state per step).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = ("GDOF·RK-stages/sec (FP64) per B200 at N=4 and roofline fraction; "
          "1/2/4/8-GPU scaling")
UNIT = "GDOF*stages/s"
REF_BENCH = os.path.join(REPO, "oracle", "_ref", "swedg_refbench")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--N", type=int, default=4)
    p.add_argument("--k1d", type=int, default=1024)
    p.add_argument("--warp", type=float, default=0.1)
    p.add_argument("--mode", choices=["fast", "parity"], default="fast")
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--ref-k1d", type=int, default=128, help="reference CPU sample size")
    # functional check of the multi-rank orchestration on a single-GPU box (no timing
    # claims): every rank on device 0, halos exchanged over gloo through host memory
    p.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl")
    p.add_argument("--shared-device", action="store_true")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms; only samples whose
    timestamp falls inside the timed region (mark_start/mark_stop) are kept."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[tuple[float, str]] = []
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            deadline = time.time() + 5.0
            while not self.lines and time.time() < deadline:  # wait for the first sample
                time.sleep(0.02)
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark_start(self):
        self.t0 = time.time()

    def mark_stop(self):
        self.t1 = time.time()
        time.sleep(0.12)  # let the last in-window sample arrive

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, pw, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            if self.t0 is not None and not (self.t0 <= ts <= (self.t1 or ts) + 0.06):
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                pw.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------------------
def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU hot path (oracle/_ref build of the
    unmodified headers) on this box's host cores, bounded sample of the workload."""
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    if not os.path.exists(REF_BENCH):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/swedg_refbench not built "
                          "(needs /root/reference at build time)"}))
        return 0
    out = subprocess.run([REF_BENCH, str(args.N), str(args.ref_k1d), str(max(1, min(args.warmup, 2))),
                          str(max(1, min(args.steps, 10))), str(threads), str(args.warp)],
                         capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1]
    r = json.loads(out)
    sample = (f"K1D={r['K1D']} (K={r['K']}) of the C4 workload, {r['steps']} LSRK45 steps after "
              f"{r['warmup']} warm-up, reference rhs()+step_lsrk45 with ops.threads={threads}")
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world,
        "steps": r["steps"], "warmup": r["warmup"], "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args, args.ref_k1d, reference=True),
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def workload_config(args, k1d, world=1, reference=False):
    K = 2 * k1d * k1d
    cfg = {"workload": f"C4: modal ESDG N={args.N}, K1D={k1d} (K={K} curved tris, warp {args.warp}), "
                       "smooth wave + lake bathymetry, periodic [-1,1]^2, LF flux, LSRK45",
           "N": args.N, "K1D": k1d, "K": K, "warp": args.warp, "scheme": "hybridized",
           "mode": "reference CPU (IEEE, reference order)" if reference else args.mode,
           "step": "one LSRK45 step = 5 RHS stages",
           "l2": "inputs larger than L2 (device-resident state+geometry >> 126 MB)"}
    if world > 1:
        cfg["partition"] = (f"weak scaling: {world} y-strips of a K1D x (K1D*{world}) periodic mesh on "
                            f"[-1,1]x[-{world},{world}], {K} elements per GPU, per-stage NCCL halo "
                            "exchange of face traces")
        cfg["parallelism"] = f"element partition x{world}"
    return cfg


def cpu_baseline(args):
    threads = os.cpu_count() or 1
    if os.path.exists(REF_BENCH):
        out = subprocess.run([REF_BENCH, str(args.N), str(args.ref_k1d), "1", "3", str(threads), str(args.warp)],
                             capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1]
        r = json.loads(out)
        return {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"K1D={r['K1D']} (K={r['K']}) of the C4 workload, {r['steps']} LSRK45 steps, "
                          f"unmodified reference (oracle/_ref) with ops.threads={threads}"}
    # the C oracle port, single thread, on a small sample
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import numpy as np
    from oracle_py import Oracle

    from paper_2005_02516_b200 import capi

    c = capi.Case("smooth", N=args.N, nx=32, warp=args.warp)
    case = {"scheme": [0], "N": [c.N], "Np": [c.Np], "nq": [c.nq], "nf": [c.nf], "npf": [c.npf], "K": [c.K],
            "g": [c.g], "ref_Vq": c.array("Vq"), "ref_Vf": c.array("Vf"), "ref_Pq": c.array("Pq"),
            "ref_Qh_x": c.array("Qr"), "ref_Qh_y": c.array("Qs"), "Mh_inv": c.array("Mh_inv"),
            "surfq_w": c.array("surfq_w"), "gf": c.array("gf"), "sJ": c.array("sJ"), "nx": c.array("nx"),
            "ny": c.array("ny"), "nbr": c.iarray("nbr"), "perm": c.iarray("perm"), "b": c.b()}
    case = {k: np.asarray(v) for k, v in case.items()}
    orc = Oracle(case)
    u = c.u0()
    t0 = time.time()
    orc.step_lsrk45(u, np.zeros_like(u), c.dt, 2)
    sec = time.time() - t0
    val = c.K * c.Np * 3 * 10 / sec / 1e9
    return {"value": val, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"K1D=32 (K={c.K}), 2 LSRK45 steps, C oracle single thread"}


# ---------------------------------------------------------------------------
def flops_bytes_per_element(N):
    """Algorithmic FP64 flops and compulsory DRAM bytes per element per stage for
    the two kernels (SURVEY.md §8(d) accounting; divide = 1 flop)."""
    Np = (N + 1) * (N + 2) // 2
    nq = (N + 1) ** 2
    nf = 3 * (N + 1)
    nh = nq + nf
    U = nq * (nq - 1) // 2 + nq * nf
    f_proj = 6 * Np * (2 * nq + nh) + 9 * (nq + nh)
    f_vol = 55 * U + 7 * nh
    f_lift_v = 6 * Np * nq
    vol_flops = f_proj + f_vol + f_lift_v
    # volume kernel bytes: u, gf, b_stacked, src (volume rows) in; traces, acc_f, T1 out
    vol_bytes = 8 * (3 * Np + 4 * nh + nh + 2 * nq + 3 * nf + 3 * nf + 3 * Np)
    # surface+update kernel: traces (own + neighbour), acc_f, T1, surf (m,nx,ny), src_f,
    # nbr/perm, Mh_inv, u, res in; u, res out
    surf_flops = 71 * nf + 6 * Np * nf + 2 * Np * Np * 3 + 15 * Np
    # (M_h^{-1} stored symmetric-packed in FAST mode: Np(Np+1)/2 doubles)
    surf_bytes = 8 * (3 * nf * 2 + 3 * nf + 3 * Np + 3 * nf + 2 * nf + Np * (Np + 1) // 2 + 3 * Np * 2 + 3 * Np * 2) + 4 * (3 + nf)
    return {"vol_flops": vol_flops, "vol_bytes": vol_bytes, "surf_flops": surf_flops, "surf_bytes": surf_bytes,
            "U": U, "Np": Np, "nq": nq, "nf": nf, "nh": nh}


def load_traffic():
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


def run_ours(args, rank, world, local):
    import numpy as np
    import torch

    from paper_2005_02516_b200 import capi

    if args.shared_device:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    # weak scaling: rank r owns y-strip r (K1D x K1D quads) of a global
    # K1D x (K1D*world) periodic mesh; one halo exchange of face traces per stage
    # (paper_2005_02516_b200/partition.py, NCCL point-to-point over NVLink).
    t0 = time.time()
    if world > 1:
        case = capi.Case("smooth", N=args.N, nx=args.k1d, warp=args.warp, seed=23, strips=world, strip=rank)
    else:
        case = capi.Case("smooth", N=args.N, nx=args.k1d, warp=args.warp, seed=23)
    mode = capi.MODE_FAST if args.mode == "fast" else capi.MODE_PARITY
    h = case.handle(mode=mode, device=local)
    u0 = case.u0()
    setup_s = time.time() - t0
    K, Np = case.K, case.Np
    dof = K * Np * 3
    dt = case.dt
    stream = torch.cuda.Stream(device=local)
    h.set_stream(stream.cuda_stream)
    h.set_state(u0)
    plan = None
    if world > 1:
        from paper_2005_02516_b200.partition import StripHalo, stage_overlapped, trace_tensor

        t = torch.tensor([dt], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        dt = float(t.item())
        plan = StripHalo(world, rank, args.k1d, K)
        trace = trace_tensor(h)
        comm_stream = torch.cuda.Stream(device=local)

    def steps(n, sync):
        if plan is None:
            h.step(dt, n, sync=sync)
            return
        # per stage: boundary rows' volume kernel, NCCL halo exchange on the comm stream
        # overlapped with the interior volume kernel, then the surface kernel
        with torch.cuda.stream(stream):
            for _ in range(n):
                for s_ in range(5):
                    stage_overlapped(h, s_, dt, trace, plan, stream, comm_stream)
        if sync:
            h.check()

    # warm-up
    steps(args.warmup, True)
    torch.cuda.synchronize()
    # ---- timed region: device-resident LSRK45 steps
    h.enable_timers(True)
    h.read_timers()
    launches0 = h.launches
    clocks = ClockSampler(local)
    clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks.mark_start()
    e0.record(stream)
    steps(args.steps, False)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark_stop()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    h.check()
    ms = e0.elapsed_time(e1)
    kms, kn = h.read_timers()
    launches = h.launches - launches0
    h.enable_timers(False)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = dof * world * 5 * args.steps / (ms * 1e-3) / 1e9

    # ---- e2e through the public API with pinned host buffers
    uh_t = torch.empty((K, 3, Np), dtype=torch.float64, pin_memory=True)
    uh = uh_t.numpy()
    uh[...] = u0
    h.set_state(uh)
    stepper = None
    if plan is not None:
        from paper_2005_02516_b200.partition import HostStepper

        stepper = HostStepper(h, plan, stream, comm_stream)
    # untimed warm-up of the host-state path (copy streams, events, pinned pages)
    if plan is None:
        h.step_host(uh, dt, 1)
    else:
        stepper.step(uh_t, dt, 1)
        torch.cuda.synchronize()
        h.check()
    uh[...] = u0
    h.set_state(uh)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee0.record(stream)
    if plan is None:
        # swedg_step_lsrk45_host: every step reads its input state from the pinned host
        # buffer and writes its result back (H2D + D2H of the full state per step),
        # transfers pipelined with the compute in element chunks
        h.step_host(uh, dt, args.e2e_steps)
    else:
        # per rank: H2D of the strip's state, 5 stages with halo exchanges, D2H of the
        # result every step; chunked copies overlap the first and last stage
        stepper.step(uh_t, dt, args.e2e_steps)
    ee1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = ee0.elapsed_time(ee1)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = dof * world * 5 * args.e2e_steps / (e2e_ms * 1e-3) / 1e9
    state_bytes = K * 3 * Np * 8

    # ---- device diagnostics (outside the timed region): one exact-sum
    # compute_invariants sample of the resident state, as run() takes ~100 per run
    h.sample_invariants(0)
    torch.cuda.synchronize()
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record(stream)
    for _ in range(3):
        h.sample_invariants(0)
    d1.record(stream)
    torch.cuda.synchronize()
    inv_ms = d0.elapsed_time(d1) / 3
    inv = h.read_invariants(1)[0]

    # ---- roofline of the dominant kernel (volume: projection + flux differencing)
    fb = flops_bytes_per_element(args.N)
    vol_avg_ms = kms[0] / max(1, kn[0])
    surf_avg_ms = kms[1] / max(1, kn[1])
    fp64_peak = capi.probe_fp64_peak(local, 5)
    hbm_peak = None
    try:
        hbm_peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
        hbm_src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        hbm_peak, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    vol_tflops = fb["vol_flops"] * K / (vol_avg_ms * 1e-3) / 1e12
    surf_gbs = fb["surf_bytes"] * K / (surf_avg_ms * 1e-3) / 1e9
    traffic = load_traffic()
    def _tr(name):
        t = traffic.get(name)
        return None if not t else round(t["dram_bytes_per_element"] * K)

    vol_traffic = _tr("volume")
    surf_traffic = _tr("surface")
    roofline = {
        "kernel": "modal_volume_pair_n4_kernel (FAST: entropy projection + flux differencing + volume lift)",
        "bound": "fp64", "achieved": round(vol_tflops, 4), "peak": round(fp64_peak, 3), "unit": "TFLOP/s",
        "frac": round(vol_tflops / fp64_peak, 4), "traffic": vol_traffic,
        "traffic_note": "ncu --set full dram__bytes_read+write per element (profiles/ncu_traffic.json) x K",
        "peak_source": "measured in-run: DFMA chain probe (swedg_probe_fp64_peak); MEASURED_PEAKS.json has no FP64 entry",
        "algorithmic_flops_per_launch": fb["vol_flops"] * K, "avg_launch_ms": round(vol_avg_ms, 4),
        "share_of_step": round(kms[0] / ms if ms > 0 else 0.0, 4),
        "flops_per_element": fb["vol_flops"],
    }
    roofline_surface = {
        "kernel": "modal_surface_kernel<4,FAST> (interface flux + LF + lift + Mh_inv + LSRK update)",
        "bound": "hbm", "achieved": round(surf_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
        "frac": round(surf_gbs / hbm_peak, 4), "traffic": surf_traffic, "peak_source": hbm_src,
        "algorithmic_bytes_per_launch": fb["surf_bytes"] * K, "avg_launch_ms": round(surf_avg_ms, 4),
        "share_of_step": round(kms[1] / ms if ms > 0 else 0.0, 4),
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, args.k1d, world),
        "e2e": {"value": round(e2e_val, 4), "unit": UNIT, "h2d_bytes_per_step": state_bytes,
                "d2h_bytes_per_step": state_bytes,
                "steps": args.e2e_steps,
                "path": "swedg_step_lsrk45_host: per step H2D of the state from pinned host memory + 5 "
                        "stages + D2H of the result; 16 element chunks run through the stages as a "
                        "wavefront so copies overlap compute (N>1: partition.HostStepper, chunked "
                        "copies overlapping the first and last stage around the halo exchanges)"},
        "gpu_launches": launches,
        "roofline": roofline,
        "roofline_surface": roofline_surface,
        "cpu_baseline": cpu,
        "clocks": clk,
        "diagnostics": {"invariants_ms": round(inv_ms, 4), "mass": inv[1], "entropy": inv[4],
                        "note": "device compute_invariants (exact sums, fine rule degree 2N+2) of the "
                                "final state, outside the timed region"},
        "setup_s": round(setup_s, 2),
        "device_bytes": h.device_bytes,
    }
    if rank == 0:
        print(json.dumps(line))
    h.close()
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
