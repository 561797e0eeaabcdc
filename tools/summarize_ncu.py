#!/usr/bin/env python3
"""Summarize ncu evidence into profiles/ (run here, on the CPU box).

  python tools/summarize_ncu.py --rep gpurun_out/prof_r01c.ncu-rep \
      --launches gpurun_out/launches_r01c.csv --blocks 134217728 --tag r01c

Writes profiles/ncu_<tag>.md (key metrics of the top kernel + the launch-list
shares) and profiles/ncu_traffic.json (DRAM bytes per block, read by bench.py
for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.peak_sustained",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__thread_inst_executed_pipe_alu_pred_on.sum",
    "smsp__inst_executed_pipe_alu.sum", "smsp__inst_executed_pipe_fma.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_float(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += to_float(r[vi]) * scale.get(r[ui], 1.0)
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--blocks", type=int, required=True, help="blocks processed by the profiled launch")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--note", default="")
    ap.add_argument("--aux", action="store_true",
                    help="a side capture: write only the summary, not ncu_traffic.json / kernel_counters.json")
    a = ap.parse_args()
    m = raw_metrics(a.rep)
    lines = [f"# ncu summary {a.tag}", "", a.note, "",
             f"Source: `{os.path.basename(a.rep)}` (`ncu --set full --clock-control none --import-source on`,"
             f" one launch of {a.blocks} blocks = {a.blocks * 8 / 2**30:.3f} GiB, tools/profile_kernel.py)", "",
             "| metric | value | unit |", "|---|---|---|"]
    stalls = []
    for k in KEYS:
        if k in m:
            lines.append(f"| `{k}` | {m[k][0]} | {m[k][1]} |")
    for k, (v, u) in m.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            f = to_float(v)
            if f:
                stalls.append((f, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    tot = sum(f for f, _ in stalls) or 1
    lines += ["", "Warp-state samples (pc sampling):", "", "| reason | share |", "|---|---|"]
    for f, k in sorted(stalls, reverse=True)[:10]:
        lines.append(f"| {k} | {100 * f / tot:.1f}% |")
    rd = to_float(m.get("dram__bytes_read.sum", ("0", ""))[0])
    wr = to_float(m.get("dram__bytes_write.sum", ("0", ""))[0])
    unit = m.get("dram__bytes_read.sum", ("", "byte"))[1].lower()
    mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(unit, 1)
    per_block = (rd + wr) * mult / a.blocks
    lines += ["", f"DRAM traffic: {(rd + wr) * mult / 1e9:.3f} GB per launch = {per_block:.2f} B/block"
              f" (algorithmic: 16 B/block = 8 read + 8 write)."]
    if a.launches:
        agg = launch_shares(a.launches)
        total = sum(t for _, t in agg.values())
        lines += ["", f"Launch list (`{os.path.basename(a.launches)}`, `ncu --metrics gpu__time_duration.sum"
                  " --clock-control none`, cold and serialised -- compare shares, not absolutes):", "",
                  "| kernel | launches | total ms | share | avg ms |", "|---|---|---|---|---|"]
        for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{name[:70]}` | {c} | {t:.3f} | {100 * t / total:.1f}% | {t / c:.4f} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_{a.tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.aux:
        print("\n".join(lines))
        return
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump({"dram_bytes_per_block": per_block, "source": f"profiles/ncu_{a.tag}.md",
                   "blocks": a.blocks}, f, indent=1)
        f.write("\n")
    alu = to_float(m.get("smsp__inst_executed_pipe_alu.sum", (None, ""))[0])
    if alu:
        fma = to_float(m.get("smsp__inst_executed_pipe_fma.sum", ("0", ""))[0]) or 0.0
        allw = to_float(m.get("smsp__inst_executed.sum", ("0", ""))[0]) or 0.0
        pct = to_float(m.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", ("0", ""))[0])
        with open(os.path.join(ROOT, "profiles", "kernel_counters.json"), "w") as f:
            json.dump({"source": f"profiles/ncu_{a.tag}.md ({os.path.basename(a.rep)})", "blocks": a.blocks,
                       "alu_warp_inst": alu, "fma_warp_inst": fma, "all_warp_inst": allw,
                       "alu_thread_inst_per_block": alu * 32 / a.blocks,
                       "fma_thread_inst_per_block": fma * 32 / a.blocks,
                       "all_thread_inst_per_block": allw * 32 / a.blocks,
                       "alu_pipe_pct": pct,
                       "note": "alu_thread_inst_per_block counts every ALU-pipe instruction the kernel issues per "
                               "block (S-box gates and Feistel XORs = 48 (T + 32) / 32 algorithmic, the "
                               "load/store transposes ~20, loop and epilogue the rest); times blocks/s over "
                               "(148 SMs x 64 lanes x clock) it is the ALU pipe's busy fraction"}, f, indent=1)
            f.write("\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
