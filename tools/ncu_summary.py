"""Summarise ncu reports + launch list into a markdown file under profiles/.
usage: ncu_summary.py ROUND  (reads gpurun_out/ROUND_*.ncu-rep, ROUND_launches.csv)"""
import csv, glob, json, subprocess, sys
from collections import defaultdict
R = sys.argv[1]
out = [f"# ncu summary, round {R}\n", "Captured on one B200 with `tools/profile_round.sh` (clock-control none).",
       "Launch-list times are cold-cache and serialised (compare shares, not absolutes); ",
       "per-kernel metrics come from one `ncu --set full` capture of the first launch of each kernel.\n"]
# launch list
rows = [r for r in csv.reader(open(f"gpurun_out/{R}_launches.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:]]
# one whole mp_order call: from the last-but-one fps_cluster_phase launch to the last
starts = [i for i, (k, _) in enumerate(data) if "fps_cluster_phase" in k]
half = data[starts[-2]:starts[-1]] if len(starts) >= 2 else data[len(data) // 2:]
tot = defaultdict(float); cnt = defaultdict(int)
for k, v in half:
    name = k.split("(")[0].replace("mp::<unnamed>::", "").replace("void ", "")[:60]
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
out.append("## Launch list (one mp_order call of the C2 bench; gpu__time_duration.sum)\n")
out.append("| kernel | launches | ms | share |\n|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:20]:
    out.append(f"| `{k}` | {cnt[k]} | {v/1e6:.3f} | {100*v/T:.1f}% |")
out.append(f"\nTotal kernel time {T/1e6:.1f} ms over {len(half)} launches.\n")
want = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Achieved Occupancy", "Registers Per Thread", "Block Size", "Grid Size", "Executed Ipc Active",
        "Warp Cycles Per Issued Instruction"]
import os
traffic = json.load(open("profiles/traffic.json")) if os.path.exists("profiles/traffic.json") else {}  # kernels not re-captured keep their entry
for rep in sorted(glob.glob(f"gpurun_out/{R}_ncu_*.ncu-rep")):
    kname = rep.split(f"{R}_ncu_")[1].replace(".ncu-rep", "")
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(det.splitlines()))
    if not r:
        continue
    hh = r[0]; mi = hh.index("Metric Name"); vv = hh.index("Metric Value"); uu = hh.index("Metric Unit")
    vals = {}
    for row in r[1:]:
        if row[mi] in want and row[mi] not in vals:
            vals[row[mi]] = f"{row[vv]} {row[uu]}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) >= 3:
        hdr, units, val = rr[0], rr[1], rr[2]
        d = dict(zip(hdr, val)); u = dict(zip(hdr, units))
        def num(key):
            x = d.get(key, "0").replace(",", "")
            try:
                f = float(x)
            except ValueError:
                return 0.0
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(key, "byte"), 1)
            return f * scale
        rb, wb = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        vals["DRAM read+write"] = f"{(rb + wb)/1e6:.2f} MB"
        traffic[kname.replace("_kernel", "").replace("fps_batched", "fps").replace("md_smem", "md")] = int(rb + wb)
        if kname in ("tri_scatter", "list_finish"):
            traffic["csr_build"] = traffic.get("csr_build", 0) + int(rb + wb)
    out.append(f"## `{kname}`\n")
    out.append("| metric | value |\n|---|---|")
    for k in want + ["DRAM read+write"]:
        if k in vals:
            out.append(f"| {k} | {vals[k]} |")
    src = subprocess.run([sys.executable, "tools/ncu_src.py", rep, kname, "0", "8"], capture_output=True, text=True).stdout
    out.append("\nTop source lines by warp-stall samples:\n```\n" + src.strip() + "\n```\n")
open(f"profiles/{R}_ncu_summary.md", "w").write("\n".join(out) + "\n")
json.dump(traffic, open("profiles/traffic.json", "w"), indent=1)
print("\n".join(out[:40]))
