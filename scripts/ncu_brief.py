"""Markdown brief of one `ncu --set full` capture: time, DRAM traffic, and the
compute-side utilisation (issue slots, FP64 / XU / tensor pipes) that bound
the non-HBM kernels.  python scripts/ncu_brief.py REP TITLE [algorithmic_bytes]"""
import csv
import io
import subprocess
import sys

M = [("gpu__time_duration.sum", "duration"),
     ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
     ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
     ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy % (compute roofline: 1 instr/cycle/SMSP)"),
     ("sm__inst_executed.avg.per_cycle_active", "IPC per SM (peak 4)"),
     ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
     ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
     ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
     ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads per warp instr"),
     ("launch__registers_per_thread", "registers/thread"), ("launch__shared_mem_per_block", "smem/block"),
     ("launch__grid_size", "grid"), ("launch__block_size", "block")]

rep, title = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, u, v = rows[0], rows[1], rows[2]
name = v[h.index("Kernel Name")] if "Kernel Name" in h else ""
print(f"## {title}\n\n`{name[:150]}`\n\n| metric | value |\n|---|---|")
vals = {}
for k, lab in M:
    if k in h:
        i = h.index(k)
        vals[k] = (v[i], u[i])
        print(f"| {lab} (`{k}`) | {v[i]} {u[i]} |")
if len(sys.argv) > 3:
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tr = sum(float(vals[k][0].replace(',', '')) * sc.get(vals[k][1], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    print(f"| DRAM traffic / algorithmic bytes | {tr / 1e6:.1f} MB / {float(sys.argv[3]) / 1e6:.1f} MB |")
print()
