#!/usr/bin/env python3
"""Summarise ncu artefacts from gpurun_out/ into profiles/ (tracked).

    python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/r1_launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep profiles/r1_volume_full.md [K]
    python tools/ncu_summary.py traffic profiles/ncu_traffic.json NAME gpurun_out/prof.ncu-rep K

`traffic` records dram__bytes_read.sum + dram__bytes_write.sum per launch (and
per element) for bench.py's roofline "traffic" field.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict


def read_launch_csv(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        if len(r) > vi:
            v = float(r[vi])
            unit = r[ui]
            ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit == "us" else v)
            out.append((r[ki], ms))
    return out


def launches(src, dst):
    ls = read_launch_csv(src)
    agg = OrderedDict()
    for k, ms in ls:
        agg.setdefault(k, []).append(ms)
    total = sum(ms for _, ms in ls)
    with open(dst, "w") as f:
        f.write(f"# ncu launch list summary\n\nsource: `{os.path.basename(src)}` "
                "(`--metrics gpu__time_duration.sum --clock-control none`, cold-cache, serialised)\n\n")
        f.write("| kernel | launches | mean ms | total ms | share |\n|---|---|---|---|---|\n")
        for k, v in agg.items():
            f.write(f"| `{k}` | {len(v)} | {sum(v) / len(v):.4f} | {sum(v):.3f} | {sum(v) / total:.1%} |\n")
    print(open(dst).read())


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        res.append({h: (u, v) for h, u, v in zip(hdr, units, vals)})
    return res


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/shared throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.per_cycle_active", "active warps / SM"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem / block"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs), blocks"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem), blocks"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall: MIO throttle"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall: math pipe throttle"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def to_bytes(u, v):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def full(rep, dst, K=None):
    recs = raw(rep)
    with open(dst, "w") as f:
        f.write(f"# ncu --set full summary: `{os.path.basename(rep)}`\n\n")
        for r in recs:
            name = r.get("Kernel Name", ("", "?"))[1]
            f.write(f"## `{name}`\n\n| metric | value | unit |\n|---|---|---|\n")
            for k, label in KEYS:
                if k in r:
                    u, v = r[k]
                    f.write(f"| {label} (`{k}`) | {v} | {u} |\n")
            if "dram__bytes_read.sum" in r:
                tot = to_bytes(*r["dram__bytes_read.sum"]) + to_bytes(*r["dram__bytes_write.sum"])
                f.write(f"| DRAM bytes read+write | {tot:.4g} | byte |\n")
                if K:
                    f.write(f"| DRAM bytes per element | {tot / K:.1f} | byte |\n")
            f.write("\n")
    print(open(dst).read())


def traffic(dst, name, rep, K):
    recs = raw(rep)
    r = recs[0]
    tot = to_bytes(*r["dram__bytes_read.sum"]) + to_bytes(*r["dram__bytes_write.sum"])
    d = json.load(open(dst)) if os.path.exists(dst) else {}
    d[name] = {"dram_bytes_per_launch_at_K": tot, "K_profiled": int(K), "dram_bytes_per_element": tot / int(K),
               "source": os.path.basename(rep)}
    json.dump(d, open(dst, "w"), indent=1)
    print(d[name])


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif cmd == "full":
        full(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else None)
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5])
