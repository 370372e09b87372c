#!/usr/bin/env python3
"""Summaries of ncu output for profiles/ (no GPU needed).

  ncu_summarize.py launches LAUNCHES.csv > launches_summary.txt
      per-kernel launch count / total / mean of gpu__time_duration.sum from the
      `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list
  ncu_summarize.py kernel RAW.csv LANES N > summary.json
      selected metrics of one captured launch from `ncu -i X.ncu-rep --page raw
      --csv`; LANES x N (blind-rotation lanes x CMux iterations of that launch)
      scales the per-lane-and-CMux figures
"""
import csv
import json
import re
import sys
from collections import OrderedDict


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path, newline="") if l.startswith('"'))]
    head = rows[0]
    k, m, u, v = (head.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    acc = OrderedDict()
    for r in rows[1:]:
        if r[m] != "gpu__time_duration.sum":
            continue
        t = float(r[v].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}[r[u]]
        name = re.sub(r"\(.*$", "", r[k]).replace("<unnamed>::", "").strip()
        c = acc.setdefault(name, [0, 0.0])
        c[0] += 1
        c[1] += t
    total = sum(c[1] for c in acc.values())
    print("kernel, launches, total_ms, mean_ms, share")
    for name, (n, t) in acc.items():
        print(f"{name}, {n}, {t:.3f}, {t / n:.4f}, {t / total:.4f}")


def kernel(path, lanes, n):
    rows = list(csv.reader(l for l in open(path, newline="") if l.startswith('"')))
    head, units, vals = rows[0], rows[1], rows[2]
    raw = {}
    for h, u, v in zip(head, units, vals):
        try:
            raw[h] = float(v.replace(",", ""))
        except ValueError:
            raw[h] = v
    g = lambda key: raw.get(key)
    out = OrderedDict()
    out["kernel"] = raw.get("Kernel Name")
    out["grid"] = raw.get("Grid Size")
    dur = g("gpu__time_duration.sum")
    unit = units[head.index("gpu__time_duration.sum")] if "gpu__time_duration.sum" in head else "ns"
    if dur is not None:
        out["duration_ms"] = round(dur * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(unit, 1e-6), 3)
    pick = {
        "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "fp64_pipe_cycles_active_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1_wavefronts_pct_elapsed": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "registers_per_thread": "launch__registers_per_thread",
    }
    for k, m in pick.items():
        if g(m) is not None:
            out[k] = g(m)
    for k in head:
        if re.fullmatch(r"sm__(inst_executed_pipe|pipe)_fp64.*pct_of_peak_sustained_(active|elapsed)", k):
            out.setdefault("fp64_metrics", {})[k] = raw[k]
    work = lanes * n
    wf = g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    if wf is None:
        wf = g("memory_l1_wavefronts_shared")  # the SourceCounters roll-up
    if wf is not None:
        out["smem_wavefronts_per_launch"] = wf
        out["smem_wavefronts_per_lane_cmux"] = round(wf / work, 1)
    wi = g("smsp__inst_executed.sum")
    if wi is not None:
        out["warp_instructions_per_lane_cmux"] = round(wi / work, 1)
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    if rd is not None and wr is not None:
        scale = lambda key: {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[head.index(key)]]
        out["dram_bytes_per_launch"] = int(rd * scale("dram__bytes_read.sum") + wr * scale("dram__bytes_write.sum"))
    fp = [g(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum") for o in ("dadd", "dmul", "dfma")]
    if all(x is not None for x in fp):
        out["fp64_instr_per_cmux_lane_ncu"] = round(sum(fp) / work, 1)
    stalls = {}
    for k in head:
        mm = re.fullmatch(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", k)
        if mm and isinstance(raw[k], float) and raw[k] >= 0.02:
            stalls[mm.group(1)] = round(raw[k], 3)
    if stalls:
        out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    if len(sys.argv) >= 3 and sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif len(sys.argv) >= 5 and sys.argv[1] == "kernel":
        kernel(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
    else:
        sys.exit(__doc__)
