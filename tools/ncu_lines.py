"""Per-source-line warp-stall samples of one kernel from an ncu report (read here, not on the box).
    python tools/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[2]
i_s = h.index("Warp Stall Sampling (All Samples)")
i_e = h.index("Instructions Executed")
st = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot, recs = 0, []
fname = "?"
for r in rows[3:]:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) <= i_s or not r[0]:
        continue
    try:
        s = int(r[i_s])
    except ValueError:
        continue
    top = sorted(((int(r[i] or 0), h[i][6:]) for i in st), reverse=True)[:2]
    recs.append((s, int(r[i_e] or 0), f"{fname}:{r[0]}", r[1][:100], top))
    tot += s
recs.sort(reverse=True)
print("total samples", tot)
for s, e, l, src, top in recs[:n]:
    print(f"{s:7d} {100 * s / tot:5.1f}% ex={e:9d} {l}: {src}  {top}")
