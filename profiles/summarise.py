"""Summarise ncu outputs into tracked files under profiles/.

  python profiles/summarise.py launches <launches.csv> <tag>      -> profiles/launches_<tag>.txt
  python profiles/summarise.py full <rep.ncu-rep> [...] <tag>      -> profiles/ncu_full_<tag>.md
                                                                     + profiles/ncu_kernels.json

`launches.csv` is the `ncu --metrics gpu__time_duration.sum --clock-control none --csv`
launch list of a bench command; the `.ncu-rep` files are `ncu --set full` captures. The JSON
keeps, per kernel, the DRAM bytes per launch that bench.py reports as `roofline.traffic`.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (warp inst/cycle/SM)"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs, CTAs/SM)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__thread_inst_executed.sum", "thread instructions"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def kernel_short(name: str) -> str:
    n = name.split("(")[0].strip()
    if n.startswith("void "):
        n = n[5:]
    return n.split("::")[-1].strip()


def launches(path: str, tag: str) -> str:
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    per = collections.defaultdict(list)
    order = []
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        k = kernel_short(d["Kernel Name"])
        per[k].append(v)
        order.append(k)
    tot = sum(sum(v) for v in per.values())
    lines = [f"# ncu launch list ({os.path.basename(path)}): {len(order)} launches, {tot:.2f} ms serialised, "
             "cold-cache (shares, not absolutes, are comparable with bench.py kernel_share)",
             f"{'kernel':22s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'mean ms':>9s}"]
    for k, v in sorted(per.items(), key=lambda x: -sum(x[1])):
        lines.append(f"{k:22s} {len(v):8d} {sum(v):10.3f} {100 * sum(v) / tot:6.1f}% {sum(v) / len(v):9.4f}")
    out = os.path.join(HERE, f"launches_{tag}.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    return out


def raw_rows(rep: str) -> list[dict]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            d[h] = (v, u)
        out.append(d)
    return out


def value(d: dict, key: str):
    if key not in d:
        return None
    v, u = d[key]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    if key.startswith("dram__bytes"):
        return x * SCALE.get(u, 1.0)
    if key == "gpu__time_duration.sum":
        return x * SCALE.get(u, 1.0)
    return x


def full(reps: list[str], tag: str) -> str:
    md = [f"# ncu --set full summaries ({tag})", "",
          "One launch per kernel, `ncu --set full --clock-control none --import-source on`, captured after the",
          "same bench command exited 0 without ncu. Durations are replayed (cold) single-launch times.", ""]
    js_path = os.path.join(HERE, "ncu_kernels.json")
    js = json.load(open(js_path)) if os.path.exists(js_path) else {"kernels": {}}
    picked = {}
    for rep in reps:  # per kernel, the longest captured launch
        for d in raw_rows(rep):
            name = kernel_short(d.get("Kernel Name", ("?", ""))[0])
            dur = value(d, "gpu__time_duration.sum") or 0.0
            if name not in picked or dur > picked[name][0]:
                picked[name] = (dur, d, rep)
    for name, (_, d, rep) in sorted(picked.items(), key=lambda x: -x[1][0]):
        if name:
            md.append(f"## {name}  ({os.path.basename(rep)})")
            md.append("| metric | value |")
            md.append("|---|---|")
            vals = {}
            for key, label in METRICS:
                v = value(d, key)
                if v is None:
                    continue
                vals[key] = v
                if key.startswith("dram__bytes"):
                    s = f"{v / 1e6:.2f} MB"
                elif key == "gpu__time_duration.sum":
                    s = f"{v:.4f} ms"
                elif isinstance(v, float):
                    s = f"{v:.4g}"
                else:
                    s = str(v)
                md.append(f"| {label} (`{key}`) | {s} |")
            md.append("")
            rd, wr = vals.get("dram__bytes_read.sum"), vals.get("dram__bytes_write.sum")
            js["kernels"][name] = {
                "dram_bytes_per_launch": (rd or 0) + (wr or 0) if rd is not None else None,
                "duration_ms": vals.get("gpu__time_duration.sum"),
                "ipc": vals.get("sm__inst_executed.avg.per_cycle_active"),
                "l2_hit_pct": vals.get("lts__t_sector_hit_rate.pct"),
                "source": f"{os.path.basename(rep)} ({tag})",
            }
    out = os.path.join(HERE, f"ncu_full_{tag}.md")
    open(out, "w").write("\n".join(md) + "\n")
    json.dump(js, open(js_path, "w"), indent=1, sort_keys=True)
    return out


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        print(launches(sys.argv[2], sys.argv[3]))
    elif mode == "full":
        print(full(sys.argv[2:-1], sys.argv[-1]))
    else:
        raise SystemExit(__doc__)
