"""Summarise ncu captures of a gpurun session into profiles/.

  python tools/ncu_summary.py gpurun_out/<tag> <round-tag>

Reads prof_*.ncu-rep (ncu --set full) and launches.csv (gpu__time_duration
launch list) and writes profiles/<round-tag>_ncu_summary.{json,md} plus
profiles/ncu_v1_store.json (dram bytes per launch of the headline kernel,
read by bench.py for roofline.traffic)."""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict, defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "occ_limit_regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "pipe_alu_pct"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "pipe_fma_pct"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "pipe_lsu_pct"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "pipe_fmaheavy_cycles_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed", "pipe_alu_cycles_pct"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "lsu_data_pct"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "smem_atom_conflicts"),
    ("smsp__inst_executed.sum", "warp_insts"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "l2_write_sectors"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_long_sb"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall_short_sb"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall_math_throttle"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall_mio_throttle"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall_lg_throttle"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall_wait"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall_not_selected"),
    ("smsp__average_warps_issue_stalled_selected_per_issue_active.ratio", "stall_selected"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_barrier"),
    ("smsp__average_warps_issue_stalled_drain_per_issue_active.ratio", "stall_drain"),
]
SCALE = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0,
         "Ghz": 1e9, "Mhz": 1e6}


def read_rep(path):
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = OrderedDict(kernel=row[hdr.index("Kernel Name")])
        for m, key in METRICS:
            if m in hdr:
                v = row[hdr.index(m)].replace(",", "")
                try:
                    v = float(v) * SCALE.get(units[hdr.index(m)], 1.0)
                except ValueError:
                    pass
                d[key] = v
        out.append(d)
    return out


def read_launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        name = r[hdr.index("Kernel Name")]
        unit = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", "")) * SCALE.get(unit, 1e-9)
        agg[name][0] += 1
        agg[name][1] += v
    total = sum(v for _, v in agg.values())
    return [dict(kernel=k, launches=c, total_s=t, mean_us=t / c * 1e6, share=t / total) for k, (c, t) in agg.items()]


def main():
    src, tag = sys.argv[1], sys.argv[2]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    prof = os.path.join(root, "profiles")
    os.makedirs(prof, exist_ok=True)
    res = {"source": src, "captures": {}, "launch_list": None}
    for f in sorted(os.listdir(src)):
        if f.startswith("prof_") and f.endswith(".ncu-rep"):
            res["captures"][f[5:-8]] = read_rep(os.path.join(src, f))
    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        res["launch_list"] = read_launches(lp)
    with open(os.path.join(prof, f"{tag}_ncu_summary.json"), "w") as fh:
        json.dump(res, fh, indent=1)
    lines = [f"# ncu summary ({tag}) from {src}", ""]
    for name, caps in res["captures"].items():
        for c in caps:
            lines.append(f"## {name}: `{c['kernel']}`")
            for k, v in c.items():
                if k != "kernel":
                    lines.append(f"- {k}: {v:.6g}" if isinstance(v, float) else f"- {k}: {v}")
            lines.append("")
    if res["launch_list"]:
        lines += ["## launch list (gpu__time_duration, --clock-control none)", "",
                  "| kernel | launches | mean us | share |", "|---|---|---|---|"]
        for d in res["launch_list"]:
            lines.append(f"| `{d['kernel'][:90]}` | {d['launches']} | {d['mean_us']:.1f} | {d['share']:.3f} |")
    with open(os.path.join(prof, f"{tag}_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    v1 = res["captures"].get("v1")
    if v1:
        c = v1[0]
        with open(os.path.join(prof, "ncu_v1_store.json"), "w") as fh:
            json.dump({"kernel": c["kernel"], "source": f"profiles/{tag}_ncu_summary.json",
                       "dram_bytes_per_launch": c["dram_read"] + c["dram_write"],
                       "dram_read": c["dram_read"], "dram_write": c["dram_write"],
                       "duration_s": c["duration"]}, fh, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
