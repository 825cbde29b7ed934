"""Copy a gpu_check.sh run (gpurun_out/<tag>) into profiles/: bench lines, timeline, launch lists, the
per-kernel ncu summary of the C5 step and the pass-1 traffic / issue figures bench.py reads.
    python tools/extract_profiles.py <tag> [round prefix, default r01]"""
import csv
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
rp = sys.argv[2] if len(sys.argv) > 2 else "r01"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "gpurun_out", tag)
dst = os.path.join(ROOT, "profiles")
for a, b in (("bench.json", f"{rp}_bench.json"), ("bench_ref.json", f"{rp}_bench_reference.json"),
             ("timeline.txt", f"{rp}_timeline_c5.txt"), ("launches_c5.csv", f"{rp}_launches_c5.csv"),
             ("launches_c4.csv", f"{rp}_launches_c4.csv")):
    if os.path.exists(os.path.join(src, a)):
        shutil.copy(os.path.join(src, a), os.path.join(dst, b))
metrics = ["gpu__time_duration.sum", "sm__inst_issued.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]
rep = os.path.join(src, "step_full.ncu-rep")
if os.path.exists(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True).stdout
else:   # summarised on the box (tools/gpu_final.sh): every raw metric of every kernel
    out = open(os.path.join(src, "step_full_raw.csv")).read()
for extra in os.listdir(src):   # per-line stall samples and raw CSVs written on the box
    if extra.startswith("lines_") or extra.endswith("_raw.csv"):
        shutil.copy(os.path.join(src, extra), os.path.join(dst, f"{rp}_{extra}"))
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
idx = [h.index("Kernel Name")] + [h.index(m) for m in metrics]
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
with open(os.path.join(dst, f"{rp}_step_ncu_summary.csv"), "w") as f:
    w = csv.writer(f)
    w.writerow(["kernel"] + [f"{m} [{units[h.index(m)]}]" for m in metrics])
    p1 = None
    for r in rows[2:]:
        name = r[idx[0]].split("(")[0]
        w.writerow([name] + [r[i] for i in idx[1:]])
        if name.startswith("void k_pass1_fast") and p1 is None:
            p1 = r
rd = float(p1[h.index("dram__bytes_read.sum")]) * mult[units[h.index("dram__bytes_read.sum")]]
wr = float(p1[h.index("dram__bytes_write.sum")]) * mult[units[h.index("dram__bytes_write.sum")]]
dur = float(p1[h.index("gpu__time_duration.sum")])
dur_ms = dur * {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "msecond": 1.0, "usecond": 1e-3}.get(units[h.index("gpu__time_duration.sum")], 1.0)
json.dump({"mixes": 4096, "bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
           "issue_active_pct": float(p1[h.index(metrics[1])]), "fma_pipe_pct": float(p1[h.index(metrics[3])]),
           "alu_pipe_pct": float(p1[h.index(metrics[4])]), "duration_ms_ncu": dur_ms,
           "source": f"ncu --set full --clock-control none of k_pass1_fast on the bench workload (C5, 4096 mixes), "
                     f"gpurun_out/{tag}/step_full.ncu-rep -> profiles/{rp}_step_ncu_summary.csv"},
          open(os.path.join(dst, "pass1_traffic.json"), "w"), indent=1)
print(open(os.path.join(dst, "pass1_traffic.json")).read())
