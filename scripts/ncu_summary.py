"""Summarise the ncu captures of scripts/profile.sh into profiles/.

    python scripts/ncu_summary.py TAG [workload ...]

Reads gpurun_out/launches_TAG_<w>.csv (per-launch gpu__time_duration) and
gpurun_out/prof_TAG_<w>.ncu-rep (one `--set full` capture of the step kernel)
and writes profiles/TAG_<w>_launches.csv, profiles/TAG_summary.md and merges
the per-launch DRAM traffic into profiles/ncu_traffic.json (read by bench.py
for roofline.traffic).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
NCU = "/usr/local/cuda/bin/ncu"

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "block limit (registers)"),
    ("launch__occupancy_limit_shared_mem", "block limit (smem)"),
    ("launch__shared_mem_per_block", "smem/block"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp instr"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__t_bytes_pipe_lsu_mem_global_op_st.sum", "L1 global store bytes"),
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "nsecond": 1e-9, "msecond": 1e-3, "ms": 1e-3}


def raw_page(rep):
    txt = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return []
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append({h: (v, u) for h, v, u in zip(head, r, units)})
    return out


def launches(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for d in csv.DictReader(io.StringIO("".join(lines))):
        if d.get("Metric Name") == "gpu__time_duration.sum":
            ns = float(d["Metric Value"].replace(",", "")) * (1e-3 if d["Metric Unit"] == "ps" else
                                                              1e3 if d["Metric Unit"] == "us" else 1)
            rows.append((d["Kernel Name"].split("(")[0].replace("marl_b200::<unnamed>::", ""), ns))
    return rows


def main():
    tag = sys.argv[1]
    wls = sys.argv[2:] or ["smax3m", "mpe_large", "overcooked", "smax27m"]
    os.makedirs(PROF, exist_ok=True)
    tpath = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    md = [f"# ncu summary {tag}", "",
          "Captured by `scripts/profile.sh` under gpurun on one B200: `ncu --set full --clock-control none "
          "--import-source on -k regex:step_kernel -s 4 -c 1` of `bench.py --workload W` (one step-kernel "
          "launch after warm-up), plus the launch list (`--metrics gpu__time_duration.sum`, cold-cache, "
          "serialised) of a 5-step run. Numbers measured under ncu are not bench values.", ""]
    for w in wls:
        lp = os.path.join(OUT, f"launches_{tag}_{w}.csv")
        if os.path.exists(lp):
            L = launches(lp)
            with open(os.path.join(PROF, f"{tag}_{w}_launches.csv"), "w") as f:
                f.write("kernel,ns\n")
                for k, ns in L:
                    f.write(f"{k},{ns:.0f}\n")
            tot = sum(ns for _, ns in L) or 1.0
            step = [ns for k, ns in L if "step_kernel" in k]
            md += [f"## {w}", "", f"Launch list: {len(L)} launches; step kernel {len(step)} launches, "
                   f"mean {sum(step) / max(len(step), 1) / 1e3:.1f} us, "
                   f"{100 * sum(step) / tot:.1f}% of all listed device time (the rest is reset / L2 flush fills).", ""]
        rp = os.path.join(OUT, f"prof_{tag}_{w}.ncu-rep")
        if not os.path.exists(rp):
            continue
        for d in raw_page(rp):
            name = d.get("Kernel Name", ("?", ""))[0].replace("marl_b200::<unnamed>::", "")
            md += [f"`{name[:150]}`", "", "| metric | value |", "|---|---|"]
            for key, label in METRICS:
                if key in d:
                    v, u = d[key]
                    md.append(f"| {label} (`{key}`) | {v} {u} |")
            smt = d.get("sm__throughput.avg.pct_of_peak_sustained_elapsed")
            if smt:
                mpath = os.path.join(PROF, "ncu_metrics.json")
                mm = json.load(open(mpath)) if os.path.exists(mpath) else {}
                mm[w] = {"sm_throughput_pct": float(smt[0].replace(",", "")),
                         "dram_throughput_pct": float(d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                                                            ("0", ""))[0].replace(",", "")),
                         "capture": f"profiles/{tag}_summary.md"}
                with open(mpath, "w") as f:
                    json.dump(mm, f, indent=1, sort_keys=True)
            rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
            if rd and wr:
                tb = float(rd[0].replace(",", "")) * SCALE.get(rd[1], 1) + \
                    float(wr[0].replace(",", "")) * SCALE.get(wr[1], 1)
                traffic[w] = tb
                md.append(f"| DRAM traffic per launch (read+write) | {tb / 1e6:.2f} MB |")
            md.append("")
    with open(os.path.join(PROF, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(md))


if __name__ == "__main__":
    main()
