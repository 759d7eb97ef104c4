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
                    [--scaling weak|strong]

Multi-GPU (--gpus N > 1; launched by torchrun, or re-executed under it when
WORLD_SIZE is unset): the mesh is partitioned into N y-strips (setup.cpp
compact_strip), one rank per GPU; every RK stage exchanges only the cut-face
traces with ncclSend/ncclRecv on a library-owned NCCL communicator, overlapped
with the interior volume kernel, inside the captured step graph.  Weak scaling
(default): every rank owns a K1D x K1D strip of a K1D x (N K1D) mesh (the C4
workload per GPU).  Strong (--scaling strong, BASELINE configs[4]): the
K1D = 2048 mesh cut into N strips.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

# NCCL init logs (rank count per communicator) for the driver's multi-GPU checks
os.environ.setdefault("NCCL_DEBUG", "INFO")
os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

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
    p.add_argument("--k1d", type=int, default=None, help="default 1024 (weak), 2048 (strong)")
    p.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    p.add_argument("--no-extra", action="store_true", help="skip the C3 / N=3 secondary kernel lines")
    p.add_argument("--warp", type=float, default=0.1)
    p.add_argument("--mode", choices=["fast", "parity"], default="fast")
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--ref-k1d", type=int, default=256, help="reference CPU sample size (SURVEY §8(d))")
    # functional check of the multi-rank orchestration on a single-GPU box (no timing
    # claims): every rank on device 0, halos exchanged over gloo through host memory
    p.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl")
    # halo transport: peer-memory stores + stream flags (one node; default), NCCL, or the
    # host-staged gloo callback (default with --shared-device / --dist-backend gloo)
    p.add_argument("--transport", choices=["p2p", "nccl", "gloo"], default=None)
    p.add_argument("--shared-device", action="store_true")
    a = p.parse_args()
    if a.k1d is None:
        a.k1d = 2048 if a.scaling == "strong" else 1024
    if a.shared_device:  # NCCL refuses two ranks on one GPU: plumbing over gloo
        a.dist_backend = "gloo"
    if a.transport is None:
        a.transport = "gloo" if (a.shared_device or a.dist_backend == "gloo") else "p2p"
    return a


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args) -> int:
    """--gpus N without a torchrun environment: re-execute this script under
    torch.distributed.run with N ranks (the driver's own launch line)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
def host_info() -> dict:
    model, mem = None, None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                mem = round(int(ln.split()[1]) / 1024 ** 2, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "mem_gb": mem}


def ref_bench(N, k1d, warmup, steps, threads, warp):
    out = subprocess.run([REF_BENCH, str(N), str(k1d), str(warmup), str(steps), str(threads), str(warp)],
                         capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1]
    return json.loads(out)


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU hot path (oracle/_ref build of the
    unmodified headers: rhs() + step_lsrk45, ops.threads = all host cores) on this box,
    on a K1D = --ref-k1d sample of the workload (K1D = 256 and 512; the
    reference's dense per-element operators need ~36 KB/elem, so K1D = 1024 does not fit
    the host), --steps timed steps after --warmup.  Two extra legs describe the baseline:
    K1D = 512 (2 steps) and threads = 1 (K1D = 128, 2 steps)."""
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    if not os.path.exists(REF_BENCH):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/swedg_refbench not built "
                          "(needs /root/reference at build time)"}))
        return 0
    r = ref_bench(args.N, args.ref_k1d, args.warmup, args.steps, threads, args.warp)
    legs = {}
    if not args.no_extra:
        for name, (k1d, th) in {"k1d512": (512, threads), "threads1_k1d128": (128, 1)}.items():
            try:
                x = ref_bench(args.N, k1d, 1, 2, th, args.warp)
                legs[name] = {k: x[k] for k in ("value", "ms_per_step", "K", "K1D", "threads", "steps", "setup_s")}
            except Exception as e:  # reported, never fatal
                legs[name] = {"error": str(e)}
    sample = (f"K1D={r['K1D']} (K={r['K']}) of the C4 workload (per-DOF comparison: the GPU arm runs "
              f"K1D={args.k1d}), {r['steps']} LSRK45 steps after {r['warmup']} warm-up, unmodified reference "
              f"rhs()+step_lsrk45 (Eigen-subset shim, -O3) with ops.threads={threads}")
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world,
        "steps": r["steps"], "warmup": r["warmup"], "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args, args.ref_k1d, reference=True),
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample, **host_info(), "legs": legs},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, k1d, world=1, reference=False):
    K = 2 * k1d * k1d
    cfg = {"workload": f"C4: modal ESDG N={args.N}, K1D={k1d} (K={K} curved tris, warp {args.warp}), "
                       "smooth wave + lake bathymetry, periodic [-1,1]^2, LF flux, LSRK45",
           "N": args.N, "K1D": k1d, "K": K, "warp": args.warp, "scheme": "hybridized",
           "mode": "reference CPU (IEEE, reference order)" if reference else args.mode,
           "step": "one LSRK45 step = 5 RHS stages",
           "l2": "inputs larger than L2 (device-resident state+geometry >> 126 MB)"}
    if world > 1 or (not reference and args.scaling == "strong"):
        if args.scaling == "weak":
            cfg["workload"] = (f"C5 weak: modal ESDG N={args.N}, {world} y-strips of K1D x K1D = {k1d}x{k1d} quads "
                               f"({K} curved tris per GPU) of a {k1d} x {k1d * world} periodic mesh, LF, LSRK45")
            cfg["K"] = K * world
        else:
            cfg["workload"] = (f"C5 strong: modal ESDG N={args.N}, K1D={k1d} (K={K} curved tris) cut into {world} "
                               "y-strips, LF, LSRK45")
        cfg["partition"] = (f"{world} y-strips, one per GPU; per RK stage the cut-face traces (npf nodes x 3 "
                            "fields per face) go to the two neighbour ranks by ncclSend/ncclRecv on a comm "
                            "stream, overlapped with the interior volume kernel, inside the captured step graph")
        cfg["parallelism"] = f"element partition x{world}"
    return cfg


def cpu_baseline(args):
    threads = os.cpu_count() or 1
    if os.path.exists(REF_BENCH):
        r = ref_bench(args.N, args.ref_k1d, 1, 3, threads, args.warp)
        return {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": f"K1D={r['K1D']} (K={r['K']}) of the C4 workload, {r['steps']} LSRK45 steps, "
                          f"unmodified reference (oracle/_ref) with ops.threads={threads}", **host_info()}
    # the C oracle port, single thread, on a small sample
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import numpy as np
    from oracle_py import Oracle, case_dict

    from paper_2005_02516_b200 import capi

    c = capi.Case("smooth", N=args.N, nx=32, warp=args.warp)
    orc = Oracle(case_dict(c))
    u = c.u0()
    t0 = time.time()
    orc.step_lsrk45(u, np.zeros_like(u), c.dt, 2)
    sec = time.time() - t0
    val = c.K * c.Np * 3 * 10 / sec / 1e9
    return {"value": val, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"K1D=32 (K={c.K}), 2 LSRK45 steps, C oracle single thread", **host_info()}


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


SBP_FLOP_N4 = 55 * 666 + 33 * 15 + 7 * 37  # SURVEY §8(d) SBP N=4 (volume + surface + source), per element


def secondary_rooflines(args, fp64_peak, device=0):
    """Driver-visible fractions of the two other FP64-bound kernels:
    C3's SBP N=4 pair kernel (dam break, K1D=128, the config's own size) and the modal
    N=3 pair kernel (the C1/C2 degree) on the C4 generator at K1D=1024."""
    from paper_2005_02516_b200 import capi

    out = {}
    runs = [("roofline_c3", "sbp_rhs_pair_n4_kernel (C3: SBP N=4 dam break K1D=128, RHS + fused LSRK45 update)",
             lambda: capi.Case("dambreak", scheme=capi.SCHEME_SBP, N=4, nx=128, cfl=0.0625), SBP_FLOP_N4, 60),
            ("roofline_n3", "modal_volume_pair_n3_kernel (modal N=3, the C4 generator at K1D=1024: projection + "
             "flux differencing + volume lift)", lambda: capi.Case("smooth", N=3, nx=1024, warp=args.warp, seed=23),
             flops_bytes_per_element(3)["vol_flops"], 5)]
    for key, kname, mk, flop, steps in runs:
        try:
            c = mk()
            h = c.handle(mode=capi.MODE_FAST, diagnostics=False)
            h.set_state(c.u0())
            h.step(c.dt, 3)
            h.enable_timers(True)
            h.read_timers()
            h.step(c.dt, steps, sync=True)
            kms, kn = h.read_timers()
            serial_ms = kms[0] / max(1, kn[0])
            rec = {"kernel": kname, "bound": "fp64", "peak": round(fp64_peak, 3), "unit": "TFLOP/s",
                   "flops_per_element": flop, "K": c.K, "avg_launch_ms_serialised": round(serial_ms, 4),
                   "launches": kn[0]}
            ms = serial_ms
            if key == "roofline_c3":
                # the SBP step is five launches of this one kernel (LSRK45 update fused): the
                # production graph replay with programmatic dependent launch, timed with CUDA
                # events on the handle's stream over the whole region, / launches = the kernel's
                # average in-step launch duration (per-launch timers serialise the launches)
                import torch

                h.enable_timers(False)
                st = torch.cuda.ExternalStream(h.stream) if h.stream else torch.cuda.default_stream()
                h.step(c.dt, 3, sync=True)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                clk = ClockSampler(device)
                clk.start()
                torch.cuda.synchronize()
                clk.mark_start()
                e0.record(st)
                h.step(c.dt, steps, sync=False)
                e1.record(st)
                e1.synchronize()
                clk.mark_stop()
                rec["clocks"] = clk.stop()
                ms = e0.elapsed_time(e1) / (5 * steps)
                rec["avg_launch_ms_in_step"] = round(ms, 4)
                rec["timing"] = ("CUDA events over %d graph-replayed LSRK45 steps (5 launches of the kernel per "
                                 "step, PDL) / launches; avg_launch_ms_serialised: per-launch event timers" % steps)
            h.close()
            tf = flop * c.K / (ms * 1e-3) / 1e12
            rec.update({"achieved": round(tf, 4), "frac": round(tf / fp64_peak, 4), "avg_launch_ms": round(ms, 4)})
            out[key] = rec
            c.close()
        except Exception as e:  # reported, never fatal
            out[key] = {"error": str(e)}
    return out


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
    red_dev = "cuda" if (dist and args.dist_backend == "nccl") else "cpu"

    def allreduce(x, op):
        if not dist:
            return x
        t = torch.tensor([x], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    t0 = time.time()
    if world > 1:  # this rank's y-strip; halo map of its two cuts (setup.cpp compact_strip)
        case = capi.Case("smooth", N=args.N, nx=args.k1d, warp=args.warp, seed=23, strips=world, strip=rank,
                         scaling=args.scaling)
    else:
        case = capi.Case("smooth", N=args.N, nx=args.k1d, warp=args.warp, seed=23)
    mode = capi.MODE_FAST if args.mode == "fast" else capi.MODE_PARITY
    h = case.handle(mode=mode, device=local)
    u0 = case.u0()
    K, Np = case.K, case.Np
    dof = K * Np * 3
    dt = case.dt
    comm = None
    transport = "none (one rank)"
    if world > 1:
        from paper_2005_02516_b200.partition import attach_gloo, attach_nccl, attach_p2p

        halo = case.halo_desc()
        if args.transport == "gloo":
            attach_gloo(h, halo, case.nf)  # functional check only (ranks share a GPU)
            transport = "gloo (host-staged exchange callback; functional, not a performance path)"
        else:
            if args.transport == "p2p":
                ok = 1.0
                try:
                    attach_p2p(h, rank, world)
                except capi.SwedgError as e:  # e.g. no peer access between these GPUs
                    print(f"[bench] rank {rank}: peer-memory transport unavailable ({e})", file=sys.stderr)
                    ok = 0.0
                if allreduce(ok, dist.ReduceOp.MIN) == 1.0:  # every rank attached, or none uses it
                    transport = ("peer memory: cut-face traces stored into the peers' halo slots over NVLink "
                                 "(CUDA IPC), stream-ordered flags, in the step graph")
                else:
                    h.set_p2p(rank, None)
            if not transport.startswith("peer"):
                comm = attach_nccl(h, halo, world, rank, local)
                transport = "NCCL send/recv of packed cut-face traces (library-owned communicator)"
        dt = allreduce(dt, dist.ReduceOp.MIN)  # the global mesh's dt (owned minimum edges)
    dof_total = int(allreduce(float(dof), dist.ReduceOp.SUM)) if dist else dof
    setup_s = time.time() - t0
    stream = torch.cuda.Stream(device=local)
    h.set_stream(stream.cuda_stream)
    h.set_state(u0)

    # the other FP64 kernels' fractions first, on a GPU not yet heated by the C4 run (after
    # it the sustained-power clock cap slows the short C3 launches by up to 10 %); the
    # peak they are quoted against is probed right before them
    extra = {}
    if rank == 0 and world == 1 and not args.no_extra:
        extra = secondary_rooflines(args, capi.probe_fp64_peak(local, 5), local)
    # warm-up (the first multi-rank call captures the step graph)
    h.step(dt, args.warmup, sync=True)
    torch.cuda.synchronize()
    # ---- timed region: device-resident LSRK45 steps, per-kernel-class CUDA-event timers
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
    h.step(dt, args.steps, sync=False)
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
    ms = allreduce(ms, dist.ReduceOp.MAX) if dist else ms
    ms_per_step = ms / args.steps
    value = dof_total * 5 * args.steps / (ms * 1e-3) / 1e9

    # ---- e2e through the public API with pinned host buffers
    uh_t = torch.empty((K, 3, Np), dtype=torch.float64, pin_memory=True)
    uh = uh_t.numpy()
    uh[...] = u0
    h.set_state(uh)
    h.step_host(uh, dt, 1)  # untimed warm-up of the host-state path (copy streams, events, pinned pages)
    uh[...] = u0
    h.set_state(uh)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee0.record(stream)
    # swedg_step_lsrk45_host: every step reads its input state from the pinned host buffer
    # and writes its result back (H2D + D2H of the full state per step); one rank: the
    # transfers are pipelined with the compute in element chunks (wavefront)
    h.step_host(uh, dt, args.e2e_steps)
    ee1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = ee0.elapsed_time(ee1)
    e2e_ms = allreduce(e2e_ms, dist.ReduceOp.MAX) if dist else e2e_ms
    e2e_val = dof_total * 5 * args.e2e_steps / (e2e_ms * 1e-3) / 1e9
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

    # ---- roofline of the dominant kernel (volume: projection + flux differencing);
    # with a partition each stage's volume work is 2-3 range launches: per-stage totals
    fb = flops_bytes_per_element(args.N)
    nst = 5 * args.steps
    vol_stage_ms = kms[0] / nst
    surf_stage_ms = kms[1] / nst
    fp64_peak = capi.probe_fp64_peak(local, 5)
    hbm_peak = None
    try:
        hbm_peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"]
        hbm_src = "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        hbm_peak, hbm_src = 6650.0, "fallback (B200_PROFILING.md)"
    vol_tflops = fb["vol_flops"] * K / (vol_stage_ms * 1e-3) / 1e12
    surf_gbs = fb["surf_bytes"] * K / (surf_stage_ms * 1e-3) / 1e9
    traffic = load_traffic()

    def _tr(name):
        t = traffic.get(name)
        return None if not t else round(t["dram_bytes_per_element"] * K)

    roofline = {
        "kernel": "modal_volume_pair_n4_kernel (FAST: entropy projection + flux differencing + volume lift)",
        "bound": "fp64", "achieved": round(vol_tflops, 4), "peak": round(fp64_peak, 3), "unit": "TFLOP/s",
        "frac": round(vol_tflops / fp64_peak, 4), "traffic": _tr("volume"),
        "traffic_note": "ncu --set full dram__bytes_read+write per element (profiles/ncu_traffic.json) x K",
        "peak_source": "measured in-run: DFMA chain probe (swedg_probe_fp64_peak); MEASURED_PEAKS.json has no FP64 entry",
        "algorithmic_flops_per_launch": fb["vol_flops"] * K, "avg_launch_ms": round(vol_stage_ms, 4),
        "launches_per_stage": round(kn[0] / nst, 2),
        "share_of_step": round(kms[0] / ms if ms > 0 else 0.0, 4),
        "flops_per_element": fb["vol_flops"],
    }
    roofline_surface = {
        "kernel": "modal_surface_kernel<4,FAST> (interface flux + LF + lift + Mh_inv + LSRK update)",
        "bound": "hbm", "achieved": round(surf_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
        "frac": round(surf_gbs / hbm_peak, 4), "traffic": _tr("surface"), "peak_source": hbm_src,
        "algorithmic_bytes_per_launch": fb["surf_bytes"] * K, "avg_launch_ms": round(surf_stage_ms, 4),
        "share_of_step": round(kms[1] / ms if ms > 0 else 0.0, 4),
    }

    cpu = None
    if rank == 0 and world == 1:
        if not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline(args)
            except Exception as e:  # reported, never fatal
                cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                       "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, args.k1d, world),
        "e2e": {"value": round(e2e_val, 4), "unit": UNIT, "h2d_bytes_per_step": state_bytes,
                "d2h_bytes_per_step": state_bytes, "steps": args.e2e_steps,
                "path": "swedg_step_lsrk45_host: per step H2D of the state from pinned host memory + 5 "
                        "stages + D2H of the result" + ("; element chunks (24 at N=4 FAST) run through the "
                                                         "stages as a wavefront so copies overlap compute" if world == 1 else
                                                         " (per rank; bytes are per rank)")},
        "gpu_launches": launches,
        "roofline": roofline,
        "roofline_surface": roofline_surface,
        **extra,
        "cpu_baseline": cpu,
        "clocks": clk,
        "multi_gpu": {"world": world, "transport": transport, "dof_per_rank": dof, "dof_total": dof_total,
                      "n_halo_slots": case.n_halo, "dt": dt},
        "diagnostics": {"invariants_ms": round(inv_ms, 4), "mass": inv[1], "entropy": inv[4],
                        "note": "device compute_invariants (exact sums, fine rule degree 2N+2) of rank 0's "
                                "final state, outside the timed region"},
        "setup_s": round(setup_s, 2),
        "device_bytes": h.device_bytes,
    }
    if dist:  # every rank's streams drained before any rank unmaps (peer memory) or frees its buffers
        torch.cuda.synchronize()
        dist.barrier()
    h.close()
    if comm:
        capi.nccl_comm_destroy(comm)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return spawn_ranks(args)
    rank, world, local = dist_env()
    if args.impl == "ours" and "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
