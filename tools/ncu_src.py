"""Summarise an ncu source page: top CUDA lines by warp-stall samples for one kernel launch.
usage: ncu_src.py REPORT KERNEL_REGEX [SKIP] [TOP]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", "-k",
                      f"regex:{kre}", "-s", skip, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, res, hdr = None, [], None
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]; hdr = None; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr and r and r[0].isdigit():
        try:
            smp = int(r[4] or 0)
        except (ValueError, IndexError):
            continue
        if smp:
            res.append((smp, cur, r[0], r[1][:100].strip(), r[7] if len(r) > 7 else ""))
res.sort(reverse=True)
tot = sum(x[0] for x in res) or 1
for x in res[:top]:
    print(f"{100*x[0]/tot:5.1f}% {x[1]}:{x[2]} {x[3]}  [inst {x[4]}]")
