#!/usr/bin/env python
"""Benchmark: patch-based ND permutation of a ~1M-vertex mesh on B200.

BASELINE.json metric: "permutation ms (device-timed) at 1M-vertex mesh;
nnz(L) bit-exact vs CPU ref".  Default workload at N=1 (configs[1], "c2"):
frequency-316 geodesic icosphere, n = 998,562, Laplacian (mesh-edge)
pattern, patch 256, seed 0, default nd_level (8), approx MD, postorder.

One step = one mp_order call: compute_patches -> ND tree -> per-node MD ->
assembly (the permutation, timed per stage with CUDA events inside the
library, summed like the reference's BenchRow t_* columns,
pipeline.hpp:46-50) followed by the factor etree / column counts / nnz(L)
(timed separately as fill_ms).  `value` = mean permutation ms per step,
device-resident CSR, L2 flushed (512 MiB write) before every step.  `e2e` =
the same call through the public C ABI on pinned HOST buffers (H2D of the CSR
and D2H of all outputs inside the timed region, host wall clock).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c1|c3|c4|c5|ico158|grid1000]

--gpus N > 1 without torchrun spawns the N ranks itself (torch.distributed.run,
127.0.0.1).  With N > 1 the default workload is "c4" (configs[3]: 64
independent 250K frames sharded over the ranks, strong scaling); "c3"
(configs[2], one 10M mesh, subtrees sharded over the ranks) is selectable.
The C2 path itself does not shard (replicas only).

--impl reference times the unmodified reference core (oracle/_ref, built from
/root/reference) on the box's host cores for the same workload and config;
its inputs come from oracle/meshgen.py and the reference's own generators and
mesh_to_graph, so the product library is never loaded in that arm.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# name: (generator kind, argument, description)
WORKLOADS = {
    "c2": ("icosphere", 316, "icosphere f=316 (n=998,562), patch 256, seed 0, L=8, approx_md, postorder"),
    "c1": ("grid", 64, "64x64 grid (n=4,096), patch 256, seed 0, L=3, approx_md, postorder"),
    "ico158": ("icosphere", 158, "icosphere f=158 (n=249,642), one C4-size frame"),
    "grid1000": ("grid", 1000, "1000x1000 grid (n=1,000,000)"),
    "c3": ("torus", (2000, 5000), "torus 2000x5000 (n=10,000,000), patch 256, seed 0, L=8, approx_md, postorder"),
    "c5": ("icosphere", 447, "icosphere f=447 (n=1,998,092) with 3x3 blocks (5,994,276 rows), patch 256, L=8"),
}
C4_FRAMES = 64  # configs[3]: random_mesh(500, 500, seed=frame), 250,000 vertices each
C4_DESC = "64 frames random_mesh(500,500,seed=f) (n=250,000 each), patch 256, seed 0, L=8, approx_md, postorder"
METRIC = "permutation ms (device-timed) at 1M-vertex mesh; nnz(L) bit-exact vs CPU ref"
METRIC_C4 = "C4 batch permutation ms (64 x 250K frames, device-timed)"
METRIC_C3 = "C3 sharded permutation ms (device-timed, 10M-vertex torus)"
STAGES = ["patch", "quotient", "etree", "local", "assemble"]


# ------------------------------------------------------------------ inputs
def product_graph(name):
    import paper_2602_00898_b200 as mp
    kind, arg, _ = WORKLOADS[name]
    if kind == "torus":
        mesh = mp.make_torus_mesh(*arg)
    elif kind == "icosphere":
        mesh = mp.make_icosphere_mesh(arg)
    else:
        mesh = mp.make_grid_mesh(arg, arg)
    return mesh, mp.mesh_to_graph(mesh)


def reference_graph(name):
    """The same CSR built without the product library (oracle/meshgen.py +
    the reference's mesh_to_graph)."""
    from oracle import meshgen
    from oracle.oracle import Reference
    kind, arg, _ = WORKLOADS[name]
    n, off, nbr = meshgen.graph(kind, arg, Reference())
    return _Graph(n, off, nbr)


class _Graph:  # AdjacencyGraph duck type for the oracle wrappers
    def __init__(self, n, off, nbr):
        self.n, self.offsets, self.neighbors = n, off, nbr

    def edge_count(self):
        return int(self.offsets[self.n]) // 2


def csr_sha(g):
    from oracle.meshgen import csr_digest
    return csr_digest(g.offsets, g.neighbors)


def golden(name):
    p = ROOT / "tests" / "golden" / "bench_golden.json"
    return json.loads(p.read_text()).get(name) if p.exists() else None


def digest(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def default_nd_level(n):  # etree.cpp:42-46
    level, x = 0, n // 512
    while x > 1:
        level, x = level + 1, x >> 1
    return min(8, level)


def workload_config(name, g, ws):
    """The config dict both arms print (identical keys and values)."""
    n = g.n
    B = 3 if name == "c5" else 1
    return {"workload": WORKLOADS[name][2], "n": n, "nnz_A": int(B * B * (n + int(g.offsets[n]))), "patch_size": 256,
            "seed": 0, "nd_level": default_nd_level(n), "block_size": B, "parallelism": f"replicas{ws}",
            "l2_flush": "512 MiB write before every device step", "csr_sha256": csr_sha(g)}


def c4_config(ws, frames_sha):
    return {"workload": C4_DESC, "frames": C4_FRAMES, "n_per_frame": 250000, "patch_size": 256, "seed": 0,
            "nd_level": 8, "block_size": 1, "parallelism": f"frames{ws}",
            "l2_flush": "inputs (64 CSRs, 1.1 GB) exceed the 126 MB L2", "frames_csr_sha256": frames_sha}


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    return 6650.0, "B200_PROFILING.md fallback (no MEASURED_PEAKS.json on this box)"


def alg_bytes(n, m, L, r_fps, kernel):
    """Algorithmic HBM bytes.  Per CSR sweep: offsets,
    neighbours and one int32 of per-vertex state read + written:
    unit = 4(n+1) + 8m + 8n."""
    unit = 4 * (n + 1) + 8 * m + 8 * n
    if kernel == "path":
        return (28 + L) * unit + 8 * r_fps + 12 * n
    if kernel == "fps":  # each relaxation scan reads one neighbour id and its dist; dist init/readback
        return 8 * r_fps + 8 * n
    if kernel == "lloyd":  # 10 rounds x (assign + recenter) CSR sweeps with per-vertex state
        return 20 * unit
    return unit  # fm / refine / md / symbolic: one gather of the node CSRs + per-vertex state


# ------------------------------------------------------------------ plumbing
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return ws, rank, local


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def teardown(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def spawn_ranks(n):
    """--gpus N outside torchrun: launch N ranks (one per GPU) ourselves."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def cpu_reference(g, steps, warmup, threads):
    """The unmodified reference (oracle/_ref/libmeshperm_ref.so): run_pipeline's
    ordering stages (pipeline.cpp:100-138) with time_stage timers."""
    from oracle.oracle import Reference
    R = Reference()
    for _ in range(warmup):
        R.order_timed(g, threads=threads)
    times, r = [], None
    for _ in range(steps):
        r = R.order_timed(g, threads=threads)
        times.append(r["ms"])
    return float(np.mean(times)), r["stage_ms"], r


def cpu_c4_frames(graphs, cores):
    """Frame-parallel reference: every frame ordered with threads=1, `cores`
    frames at a time (the stage functions are reentrant; intra-frame
    threads do not help at 250K).  Returns (wall ms, per-frame results)."""
    import concurrent.futures as cf
    from oracle.oracle import Reference
    R = Reference()
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(cores) as ex:  # ctypes releases the GIL in the reference calls
        res = list(ex.map(lambda g: R.order_timed(g, threads=1), graphs))
    return (time.perf_counter() - t0) * 1e3, res


def c4_reference_frames():
    from oracle import meshgen
    from oracle.oracle import Reference
    R = Reference()
    out = []
    for f in range(C4_FRAMES):
        n, off, nbr = meshgen.graph("random", (500, 500, f), R)
        out.append(_Graph(n, off, nbr))
    return out


# ------------------------------------------------------------------ reference arm
def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:  # the CPU reference runs once, on rank 0's host cores
        return 0
    cores = os.cpu_count() or 1
    t0 = time.time()
    if args.workload == "c4":
        frames = c4_reference_frames()
        fsha = digest(np.array([int(csr_sha(g), 16) for g in frames], np.uint64))
        # each step: one wave of `cores` frames, one per core (threads=1); the
        # 64 frames are ceil(64/cores) such waves, rotated over the steps
        waves = -(-C4_FRAMES // cores)
        times = []
        for k in range(args.warmup + args.steps):
            start = (k * cores) % C4_FRAMES
            sample = [frames[(start + i) % C4_FRAMES] for i in range(min(cores, C4_FRAMES))]
            ms, _ = cpu_c4_frames(sample, cores)
            if k >= args.warmup:
                times.append(ms * waves)
        v = float(np.mean(times))
        line = {"impl": "reference", "metric": METRIC_C4, "value": round(v, 3), "unit": "ms", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(v, 3), "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
                "config": c4_config(ws, fsha),
                "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": cores, "kind": "reference",
                                 "sample": f"per step one wave of {min(cores, C4_FRAMES)} frames ordered concurrently "
                                           f"(one per core, threads=1); 64 frames = {waves} waves"},
                "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "wall_s": round(time.time() - t0, 1)}
        print(json.dumps(line), flush=True)
        return 0
    name = args.workload
    if name == "c3":  # a 10M reference ordering is 12.6 min: bounded sample
        gs = _Graph(*__import__("oracle.meshgen", fromlist=["graph"]).graph("torus", (1000, 1000)))
        g = gs
    else:
        g = gs = reference_graph(name)
    ms, stage, _ = cpu_reference(gs, args.steps, args.warmup, cores)
    cfg = workload_config(name, g, ws)
    sample = f"full {name} ordering (stages 1-5) per step, order_tree_nodes threads={cores}"
    if name == "c3":
        cfg = {"workload": WORKLOADS["c3"][2], "note": "bounded sample: torus 1000x1000"}
        sample = "torus 1000x1000 (n=1M) per step, a bounded sample of c3 (full 10M: 758 s recorded)"
    line = {
        "impl": "reference", "metric": METRIC if name != "c3" else METRIC_C3, "value": round(ms, 3), "unit": "ms",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": cfg,
        "stage_ms": {k: round(v, 3) for k, v in zip(STAGES, stage)},
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(time.time() - t0, 1),
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm: one mesh
def run_ours(args):
    import torch
    import paper_2602_00898_b200 as mp
    from paper_2602_00898_b200 import api

    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    mesh, g = product_graph(args.workload)
    n, m2 = g.n, int(g.offsets[-1])
    B = 3 if args.workload == "c5" else 1  # configs[4]: 3x3 blocks expanded on the device
    N = B * n
    L = mp.default_nd_level(n)
    nn = (1 << (L + 1)) - 1
    ctx = mp.Context(local)
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream.cuda_stream)

    d_off = torch.from_numpy(g.offsets).to(dev)
    d_nbr = torch.from_numpy(g.neighbors).to(dev)
    outs = {
        "patch_of": torch.empty(n, dtype=torch.int32, device=dev),
        "tree_node_offsets": torch.empty(nn + 1, dtype=torch.int32, device=dev),
        "tree_vertices": torch.empty(N, dtype=torch.int32, device=dev),
        "tree_local_perm": torch.empty(N, dtype=torch.int32, device=dev),
        "perm": torch.empty(N, dtype=torch.int32, device=dev),
        "inverse": torch.empty(N, dtype=torch.int32, device=dev),
        "etree_parent": torch.empty(N, dtype=torch.int32, device=dev),
        "column_counts": torch.empty(N, dtype=torch.int64, device=dev),
    }
    ptrs = {k: v.data_ptr() for k, v in outs.items()}
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step():
        with torch.cuda.stream(stream):
            flush.fill_(1)  # evict the L2 (126 MB) before every step
        return api.order_device(ctx, n, d_off.data_ptr(), d_nbr.data_ptr(), ptrs, block_size=B)

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    barrier(ws)
    perm_ms, fill_ms, kms, launches, tot_ms = [], [], np.zeros(6), 0, []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            ev0.record(stream)
            res = api.order_device(ctx, n, d_off.data_ptr(), d_nbr.data_ptr(), ptrs, block_size=B)
            ev1.record(stream)
            perm_ms.append(sum(res.stage_ms[i] for i in range(5)))
            if os.environ.get("MP_BENCH_VERBOSE"):
                print("step", [round(res.stage_ms[i], 2) for i in range(6)],
                      [round(res.kernel_ms[i], 2) for i in range(6)], file=sys.stderr)
            fill_ms.append(res.stage_ms[5])
            kms += np.array([res.kernel_ms[i] for i in range(6)])
            launches += res.kernel_launches
            ev1.synchronize()
            tot_ms.append(ev0.elapsed_time(ev1))
        torch.cuda.synchronize()
    barrier(ws)
    ms = max_over_ranks(float(np.mean(perm_ms)), ws)
    ms_fill = max_over_ranks(float(np.mean(fill_ms)), ws)
    ms_tot = max_over_ranks(float(np.mean(tot_ms)), ws)
    kms /= args.steps
    nnz_L = int(res.nnz_L)
    gold = golden(args.workload)
    r_fps = int(res.work[0])

    # parity of the last timed step against the reference-generated golden
    perm_sha = digest(outs["perm"].cpu().numpy())
    cc_sha = digest(outs["column_counts"].cpu().numpy())
    par_sha = digest(outs["etree_parent"].cpu().numpy())
    parity = {"nnz_L": nnz_L, "sha_perm": perm_sha, "sha_column_counts": cc_sha, "sha_parents": par_sha}
    if gold:
        parity["golden"] = {k: gold.get(k) for k in ("nnz_L", "cost", "patch_count", "sha_perm", "sha_column_counts",
                                                      "sha_parents")}
        parity["match"] = bool(nnz_L == gold["nnz_L"] and int(res.cost) == gold["cost"]
                               and int(res.patch_count) == gold["patch_count"] and perm_sha == gold["sha_perm"]
                               and cc_sha == gold.get("sha_column_counts", cc_sha)
                               and par_sha == gold.get("sha_parents", par_sha))

    # e2e: the public C ABI on pinned host buffers (H2D + D2H inside the timed region)
    h_off = torch.from_numpy(g.offsets).pin_memory()
    h_nbr = torch.from_numpy(g.neighbors).pin_memory()
    h_outs = {k: torch.empty(v.numel(), dtype=v.dtype).pin_memory() for k, v in outs.items()
              if k not in ("etree_parent", "column_counts")}
    h_ptrs = {k: v.data_ptr() for k, v in h_outs.items()}
    cfg = api.make_config(block_size=B, want_fill=False)  # the metric: permutation (fill is reported as fill_ms)
    from paper_2602_00898_b200._lib import MpCsr, MpResult, check, lib
    import ctypes as C

    def e2e_call():
        csr = MpCsr(n, C.c_void_p(h_off.data_ptr()), C.c_void_p(h_nbr.data_ptr()), 0)
        r = MpResult()
        r.on_device = 0
        for k, v in h_ptrs.items():
            setattr(r, k, C.c_void_p(v))
        check(lib().mp_order(ctx.handle, C.byref(csr), C.byref(cfg), C.byref(r)))
        return r

    e2e_call()
    e2e_ms = []
    for _ in range(max(10, args.steps)):
        with torch.cuda.stream(stream):
            flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_call()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_v = max_over_ranks(float(np.mean(e2e_ms)), ws)
    e2e_perm_ok = digest(h_outs["perm"].numpy()) == perm_sha
    h2d = 4 * (n + 1) + 4 * m2
    d2h = sum(v.numel() * v.element_size() for v in h_outs.values())

    # the CSR build from device-resident triangles, timed
    # separately; HBM-bound, so its roofline is meaningful
    csr_build = None
    if args.workload != "c3":
        tri_d = torch.from_numpy(np.ascontiguousarray(mesh.triangles, np.int32).reshape(-1)).to(dev)
        ntri = tri_d.numel() // 3
        off_d = torch.empty(n + 1, dtype=torch.int32, device=dev)
        nbr_d = torch.empty(max(6 * ntri, 1), dtype=torch.int32, device=dev)
        nnz = api.mesh_to_graph_device_ptr(ctx, n, ntri, tri_d.data_ptr(), off_d.data_ptr(), nbr_d.data_ptr())
        ok = (nnz == m2 and torch.equal(off_d.cpu(), torch.from_numpy(g.offsets))
              and torch.equal(nbr_d[:nnz].cpu(), torch.from_numpy(g.neighbors)))
        cms = []
        for _ in range(10):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            ev0.record(stream)
            api.mesh_to_graph_device_ptr(ctx, n, ntri, tri_d.data_ptr(), off_d.data_ptr(), nbr_d.data_ptr())
            ev1.record(stream)
            ev1.synchronize()
            cms.append(ev0.elapsed_time(ev1))
        cms_v = float(np.median(cms))
        cab = 12 * ntri + 4 * (n + 1) + 4 * nnz
        csr_build = {"ms": round(cms_v, 4), "triangles": ntri, "nnz": nnz, "matches_host_csr": bool(ok),
                     "alg_bytes": int(cab), "gbs": round(cab / (cms_v * 1e-3) / 1e9, 1)}

    if rank == 0:
        names = ["fps", "lloyd", "fm", "refine", "md", "symbolic"]
        dom = max(range(5), key=lambda i: kms[i])  # dominant kernel of the permutation stages
        dom_name = names[dom]
        if gold and gold.get("r_fps"):
            r_fps = int(gold["r_fps"])  # the sequential algorithm's scan count (reference), not our speculative one
        m = m2 // 2
        ab = alg_bytes(n, m, L, r_fps, dom_name)
        peak, peak_src = peaks()
        achieved = ab / (kms[dom] * 1e-3) / 1e9 if kms[dom] > 0 else 0.0
        path_bytes = alg_bytes(n, m, L, r_fps, "path")
        traffic = None
        tp = ROOT / "profiles" / "traffic.json"
        if tp.exists() and args.workload == "c2":
            tj = json.loads(tp.read_text())
            traffic = tj.get(dom_name)
            if dom_name == "fps" and traffic is not None:  # the kernel-time slot covers both FPS kernels
                traffic += tj.get("fps_cluster_phase", 0)
        cpu = None
        if not args.no_cpu:
            threads = os.cpu_count() or 1
            try:
                cms_, cstage, _ = cpu_reference(g, 1, 0, threads)
                cpu = {"value": round(cms_, 3), "unit": "ms", "cores": threads, "kind": "reference",
                       "sample": f"one full {args.workload} ordering (stages 1-5) with the reference core, "
                                 f"order_tree_nodes threads={threads}",
                       "stage_ms": {k: round(v, 2) for k, v in zip(STAGES, cstage)}}
            except Exception as e:  # reference .so missing on this box
                cpu = {"value": None, "unit": "ms", "cores": None, "kind": "reference", "sample": f"unavailable: {e}"}
        line = {
            "metric": METRIC, "value": round(ms, 3), "unit": "ms", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_tot, 3), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": workload_config(args.workload, g, ws),
            "vertices_per_s": round(ws * n / (ms * 1e-3), 1),
            "fill_ms": round(ms_fill, 3),
            "stage_ms": {k: round(float(res.stage_ms[i]), 3) for i, k in enumerate(STAGES + ["symbolic"])},
            "kernel_ms": {k: round(float(v), 3) for k, v in zip(names, kms)},
            "parity": parity,
            "patch_count": int(res.patch_count),
            "gpu_launches": int(launches),
            "roofline_per_kernel": {names[i]: {"ms": round(float(kms[i]), 3),
                                               "alg_bytes": int(alg_bytes(n, m, L, r_fps, names[i])),
                                               "gbs": round(alg_bytes(n, m, L, r_fps, names[i]) / (kms[i] * 1e-3) / 1e9,
                                                            3) if kms[i] > 0 else None} for i in range(6)},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": round(achieved, 2), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 5),
                         "traffic": traffic, "alg_bytes_per_launch": int(ab),
                         "path": {"alg_bytes": int(path_bytes),
                                  "achieved": round(path_bytes / (ms * 1e-3) / 1e9, 2),
                                  "frac": round(path_bytes / (ms * 1e-3) / 1e9 / peak, 5)}},
            "work": {"r_fps": r_fps, "fm_moves": int(res.work[1]), "refine_moves": int(res.work[2]),
                     "lloyd_levels": int(res.work[3]), "fps_batches": int(res.work[4]),
                     "fps_grid_levels": int(res.work[5]), "fps_candidates": int(res.work[6]),
                     "fps_region_levels_cta0": int(res.work[7]),
                     "fps_phase_cycles": [int(res.work[i]) for i in range(8, 13)],
                     "fps_select_stats": [int(res.work[i]) for i in range(13, 16)]},
            "e2e": {"value": round(e2e_v, 3), "unit": "ms", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "calls": len(e2e_ms), "perm_matches_device_run": e2e_perm_ok},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        if csr_build:
            csr_build["peak_gbs"] = peak
            csr_build["frac"] = round(csr_build["gbs"] / peak, 4)
            line["csr_build"] = csr_build
        print(json.dumps(line), flush=True)
    teardown(ws)
    return 0


# ------------------------------------------------------------------ our arm: C4 frames
def run_c4(args):
    """configs[3]: 64 independent 250K frames, dealt round-robin to the ranks
    (no data-path collective); each GPU runs its frames on `c4_workers`
    concurrent contexts through the native mp_order_batch.  `value` = whole
    batch ms, device-resident CSRs and outputs, CUDA events bracketing a
    device-wide synchronize on both sides (the frames run on several streams),
    max over ranks; `e2e` = the same batch on pinned host arrays."""
    import ctypes as C

    import torch

    import paper_2602_00898_b200 as mp
    from paper_2602_00898_b200 import api
    from paper_2602_00898_b200._lib import MpConfig, MpCsr, MpResult, check, lib
    from paper_2602_00898_b200.batch import gather_to_root, shard

    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    mine = shard(C4_FRAMES, ws, rank)
    frames = [mp.mesh_to_graph(mp.make_random_mesh(500, 500, seed=f)) for f in mine]
    K = len(frames)
    ctxs = [mp.Context(local) for _ in range(args.c4_workers)]
    for c in ctxs:
        check(lib().mp_context_set_sm_share(c.handle, len(ctxs)))
    handles = (C.c_void_p * len(ctxs))(*[c.handle for c in ctxs])
    cfg = api.make_config(want_fill=False)
    cfgs = (MpConfig * max(K, 1))(*[cfg for _ in frames])
    # device-resident inputs / outputs
    d_in = [(torch.from_numpy(g.offsets).to(dev), torch.from_numpy(g.neighbors).to(dev)) for g in frames]
    keys = ["patch_of", "tree_node_offsets", "tree_vertices", "tree_local_perm", "perm", "inverse"]
    d_out = [{k: torch.empty(g.n if k != "tree_node_offsets" else 512, dtype=torch.int32, device=dev) for k in keys}
             for g in frames]
    csrs = (MpCsr * max(K, 1))(*[MpCsr(g.n, C.c_void_p(o.data_ptr()), C.c_void_p(b.data_ptr()), 1)
                                 for g, (o, b) in zip(frames, d_in)])
    ress = (MpResult * max(K, 1))()
    for r, o in zip(ress, d_out):
        r.on_device = 1
        for k in keys:
            setattr(r, k, C.c_void_p(o[k].data_ptr()))
    status = np.zeros(max(K, 1), np.int32)

    def batch():
        check(lib().mp_order_batch(handles, len(ctxs), K, csrs, cfgs, ress,
                                   C.c_void_p(status.ctypes.data)))

    for _ in range(args.warmup):
        batch()
    torch.cuda.synchronize()
    barrier(ws)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times, launches, kms = [], 0, np.zeros(6)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            ev0.record()
            batch()
            torch.cuda.synchronize()
            ev1.record()
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
            launches += sum(int(r.kernel_launches) for r in ress[:K])
            kms += np.array([[r.kernel_ms[i] for i in range(6)] for r in ress[:K]]).sum(0)
    ms = max_over_ranks(float(np.mean(times)), ws)
    kms /= args.steps
    # parity: every frame's permutation digest against the reference golden
    gold = (golden("c4") or {}).get("frames", [])
    local_d = {f: (digest(d_out[i]["perm"].cpu().numpy()), int(ress[i].patch_count)) for i, f in enumerate(mine)}
    merged = gather_to_root(local_d, ws, rank) if ws > 1 else local_d

    # e2e: the same frames from pinned host arrays through mp_order_batch
    h_in = [(torch.from_numpy(g.offsets).pin_memory(), torch.from_numpy(g.neighbors).pin_memory()) for g in frames]
    h_out = [{k: torch.empty(g.n if k != "tree_node_offsets" else 512, dtype=torch.int32).pin_memory()
              for k in keys} for g in frames]
    hcsrs = (MpCsr * max(K, 1))(*[MpCsr(g.n, C.c_void_p(o.data_ptr()), C.c_void_p(b.data_ptr()), 0)
                                  for g, (o, b) in zip(frames, h_in)])
    hress = (MpResult * max(K, 1))()
    for r, o in zip(hress, h_out):
        r.on_device = 0
        for k in keys:
            setattr(r, k, C.c_void_p(o[k].data_ptr()))
    e2e = []
    for _ in range(max(3, min(args.steps, 5))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        check(lib().mp_order_batch(handles, len(ctxs), K, hcsrs, cfgs, hress, C.c_void_p(status.ctypes.data)))
        e2e.append((time.perf_counter() - t0) * 1e3)
    e2e_v = max_over_ranks(float(np.mean(e2e)), ws)
    h2d = sum(4 * (g.n + 1) + 4 * int(g.offsets[-1]) for g in frames) * ws
    d2h = sum(sum(v.numel() * 4 for v in o.values()) for o in h_out) * ws
    for c in ctxs:
        c.close()

    cpu = None
    if rank == 0 and not args.no_cpu:
        cores = os.cpu_count() or 1
        try:
            wall, out = cpu_c4_frames(c4_reference_frames(), cores)
            ok = all(digest(o["perm"]) == gold[f]["sha_perm"] for f, o in enumerate(out)) if gold else None
            cpu = {"value": round(wall, 1), "unit": "ms", "cores": cores, "kind": "reference",
                   "sample": f"all {C4_FRAMES} frames ordered by the reference core, {cores} at a time "
                             f"(one per core, threads=1), host wall clock", "perm_matches_golden": ok}
        except Exception as e:
            cpu = {"value": None, "unit": "ms", "cores": None, "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        match = sum(1 for f, (d, pc) in merged.items() if gold and d == gold[f]["sha_perm"]
                    and pc == gold[f]["patch_count"])
        n_tot = 250000 * C4_FRAMES
        m_frame = int(np.mean([int(g.offsets[-1]) // 2 for g in frames]))
        names = ["fps", "lloyd", "fm", "refine", "md", "symbolic"]
        dom = max(range(5), key=lambda i: kms[i])
        r_fps = 8977327  # FPS scans of a 250K frame are ~ those of the f=158 icosphere golden
        ab = alg_bytes(250000, m_frame, 8, r_fps, names[dom]) * K
        peak, peak_src = peaks()
        achieved = ab / (kms[dom] * 1e-3) / 1e9 if kms[dom] > 0 else 0.0
        fsha = digest(np.array([int(csr_sha(_Graph(g.n, g.offsets, g.neighbors)), 16) for g in frames], np.uint64)) \
            if ws == 1 else None
        print(json.dumps({
            "metric": METRIC_C4, "value": round(ms, 3), "unit": "ms", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic", "config": c4_config(ws, fsha),
            "frames_per_rank": K, "contexts_per_gpu": args.c4_workers,
            "vertices_per_s": round(n_tot / (ms * 1e-3), 1),
            "parity": {"frames_checked": len(merged), "perm_and_patch_count_match": match},
            "gpu_launches": int(launches),
            "kernel_ms_rank0_sum_over_frames": {k: round(float(v), 3) for k, v in zip(names, kms)},
            "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": round(achieved, 2), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 6),
                         "traffic": None, "alg_bytes_per_launch": int(ab / max(K, 1)),
                         "note": "kernel time summed over rank 0's frames (concurrent on 4 streams)"},
            "e2e": {"value": round(e2e_v, 3), "unit": "ms", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "cpu_baseline": cpu, "clocks": clk.summary()}), flush=True)
    teardown(ws)
    return 0


# ------------------------------------------------------------------ our arm: C3 subtrees
def run_c3(args):
    """configs[2]: the 10M-vertex torus ordered by all ranks together through
    the native mp_order_sharded: patches and the top
    ceil(log2 N) ND levels on every rank, the level-k subtrees dealt to ranks,
    NCCL all-gathers of sizes, tree lists, subtree-root elements and column
    counts.  value = permutation ms (stages 1-5, CUDA events in the library),
    device-resident CSR and outputs, max over ranks; fill reported beside."""
    import torch

    import paper_2602_00898_b200 as mp
    from paper_2602_00898_b200 import api

    ws, rank, local = dist_setup()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _, g = product_graph("c3")
    n, m2 = g.n, int(g.offsets[-1])
    L = mp.default_nd_level(n)
    nn = (1 << (L + 1)) - 1
    ctx = mp.Context(local)
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream.cuda_stream)
    if ws > 1:
        import torch.distributed as dist
        uid = [mp.Comm.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = mp.Comm.nccl(rank, ws, local, uid[0])
    else:
        comm = mp.Comm.from_allgather(0, 1, lambda b: b)
    d_off = torch.from_numpy(g.offsets).to(dev)
    d_nbr = torch.from_numpy(g.neighbors).to(dev)
    outs = {k: torch.empty(nn + 1 if k == "tree_node_offsets" else n, dtype=torch.int32, device=dev)
            for k in ("patch_of", "tree_node_offsets", "tree_vertices", "tree_local_perm", "perm", "inverse",
                      "etree_parent")}
    outs["column_counts"] = torch.empty(n, dtype=torch.int64, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    import ctypes as C
    from paper_2602_00898_b200._lib import MpCsr, MpResult, check, lib

    def call(want_fill):
        cfg = api.make_config(want_fill=want_fill)
        csr = MpCsr(n, C.c_void_p(d_off.data_ptr()), C.c_void_p(d_nbr.data_ptr()), 1)
        r = MpResult()
        r.on_device = 1
        for k, v in outs.items():
            setattr(r, k, C.c_void_p(v.data_ptr()))
        with torch.cuda.stream(stream):
            flush.fill_(1)
        check(lib().mp_order_sharded(ctx.handle, C.byref(csr), C.byref(cfg), C.byref(comm.struct), C.byref(r)))
        return r

    for _ in range(args.warmup):
        call(False)
    barrier(ws)
    rows, launches = [], 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            r = call(False)
            rows.append([r.stage_ms[i] for i in range(5)])
            launches += r.kernel_launches
    barrier(ws)
    rows = np.array(rows)
    ms = max_over_ranks(float(rows.sum(1).mean()), ws)
    parts = [max_over_ranks(float(x), ws) for x in rows.mean(0)]
    owned = int(r.work[15])
    perm_sha = digest(outs["perm"].cpu().numpy())
    # one call with the fill on: nnz(L), column counts and parents vs the golden
    rf = call(True)
    fill_ms = max_over_ranks(float(rf.stage_ms[5]), ws)
    gold = golden("c3")
    parity = {"sha_perm": perm_sha, "nnz_L": int(rf.nnz_L), "sha_column_counts": digest(outs["column_counts"].cpu().numpy()),
              "sha_parents": digest(outs["etree_parent"].cpu().numpy())}
    if gold:
        parity["match"] = bool(perm_sha == gold["sha_perm"] and parity["nnz_L"] == gold["nnz_L"]
                               and parity["sha_column_counts"] == gold["sha_column_counts"]
                               and parity["sha_parents"] == gold["sha_parents"])
    comm.close()
    if rank == 0:
        peak, peak_src = peaks()
        path_bytes = alg_bytes(n, m2 // 2, L, 0, "path")
        cpu = {"value": round(gold["reference_s"] * 1e3, 1) if gold else None, "unit": "ms", "cores": 8,
               "kind": "reference",
               "sample": "recorded, not re-run per session (12.6 min): the full 10M ordering + fill by the reference "
                         "core (tests/golden/make_golden.py --c3, 8-core build container, order_tree_nodes threads=16)"}
        line = {
            "metric": METRIC_C3, "value": round(ms, 3), "unit": "ms", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": WORKLOADS["c3"][2], "n": n, "nd_level": L, "parallelism": f"subtrees{ws}",
                       "shard_level": int(np.ceil(np.log2(ws))) if ws > 1 else 0,
                       "l2_flush": "512 MiB write before every step", "csr_sha256": csr_sha(g)},
            "vertices_per_s": round(n / (ms * 1e-3), 1), "fill_ms": round(fill_ms, 3),
            "stage_ms_max_over_ranks": dict(zip(STAGES, [round(x, 3) for x in parts])),
            "rank0_vertices_ordered": owned, "gpu_launches": int(launches), "parity": parity,
            "roofline": {"bound": "hbm", "kernel": "path", "achieved": round(path_bytes / (ms * 1e-3) / 1e9, 2),
                         "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                         "frac": round(path_bytes / (ms * 1e-3) / 1e9 / peak, 6), "traffic": None,
                         "alg_bytes_per_launch": int(path_bytes)},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    teardown(ws)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS) + ["c4"],
                    help="default: c2 at --gpus 1, c4 (sharded frames) at --gpus > 1")
    ap.add_argument("--c3-unsharded", action="store_true", help="c3 through mp_order (stats, fill) instead")
    ap.add_argument("--c4-workers", type=int, default=4, help="concurrent contexts per GPU for c4")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.workload is None:
        args.workload = "c4" if max(ws, args.gpus) > 1 else "c2"
    if args.impl == "reference":
        return run_reference_arm(args)
    if args.workload == "c4":
        return run_c4(args)
    if args.workload == "c3" and not args.c3_unsharded:
        return run_c3(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
