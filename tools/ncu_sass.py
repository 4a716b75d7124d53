"""Per-SASS-instruction view of one kernel launch in an ncu report: the
instructions executed at least MIN times (a hot loop), with warp-stall
samples and the dominant stall reason.
usage: ncu_sass.py REPORT KERNEL_REGEX MIN [PER]   (PER: divide counts, e.g. moves)"""
import csv, subprocess, sys
rep, kre, mn = sys.argv[1], sys.argv[2], float(sys.argv[3])
per = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      f"regex:{kre}", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ia, isrc, ismp, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stalls = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot_inst = tot_smp = 0
for r in rows[2:]:
    ex = float(r[iex] or 0)
    if ex < mn:
        continue
    smp = float(r[ismp] or 0)
    tot_inst += ex; tot_smp += smp
    st = max(stalls, key=lambda i: float(r[i] or 0))
    print(f"{r[ia][-5:]} {ex/per:7.2f} smp {smp:6.0f} {h[st][6:]:>16}  {r[isrc].strip()[:70]}")
print(f"instructions per unit {tot_inst/per:.1f}, samples {tot_smp:.0f}")
