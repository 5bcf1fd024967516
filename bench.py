#!/usr/bin/env python
"""Benchmark: DoFs/s per relaxation sweep (fp64) on B200 -- BASELINE.json metric.

One "step" = one rm_relax sweep (residual r = f - A u, all star-patch solves, scatter-add,
u_out = u_in + omega c) over the whole mesh of the workload.  Default workload: BASELINE.json
configs[4] (cfg5), the configuration the metric's 1/2/4/8-GPU weak scaling is quoted on: H(grad)
Q_15 on 16^3 perturbed trilinear hexes PER GPU, auxiliary operator with ICC-SC patches; at N > 1
the global mesh is 16 x 16 x 16N, z-slab partitioned with NCCL halos (scaling "weak").  The line
nests a "secondary" workload (default cfg2: Q_7 on 32^3 axis-aligned hexes, exact Cholesky; also
z-slabs at N > 1) measured the same way.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--secondary 2] [--impl ours|reference]

Timing: W untimed sweeps, then K sweeps between barrier + cuda.synchronize, CUDA events on the
library stream, max over ranks.  The patch factors and vectors (GBs) exceed the 126 MB L2, so no
L2 flush is needed ("l2": "inputs larger than L2").  value = free DoFs (all ranks) / s.

Extra keys: roofline (dominant kernel by measured time -- the persistent patch kernel, HBM-bound,
algorithmic bytes = 8 B x sum nnz(L) + 24 B/DoF; or the apply kernel: FP64-bound on
trilinear cells, HBM-bound on Cartesian ones), e2e (rm_relax_host with pinned host buffers,
copies inside the timed region), cpu_baseline (the oracle, on a bounded sample), clocks
(nvidia-smi during the timed region), gpu_launches (our kernels in the timed region).
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import rm_inputs as ri  # noqa: E402

# bounded oracle samples (same p, space, coefficient law, BCs; smaller mesh) -- DESIGN.md
# trilinear apply (apply_tri.cu, p = 15 tables padded to 16 x 24): per cell 2 x (196,608 + 442,368 +
# 884,736) FMA in the z / y / x contractions + ~97 flops at each of the 24^3 points
TRI_FLOPS_PER_CELL = 2 * 2 * (196608 + 442368 + 884736) + 97 * 24 ** 3
FP64_PEAK_TFLOPS = 36.9   # measured on this pool's B200 (scripts/fp64_bench.cu; DMMA and DFMA alike)
# cfg5 (p = 15, trilinear, ICC-SC): 2^3 cells (one full interior vertex star, 24,389 free DoFs);
# the oracle's auxiliary operator uses sparse Kronecker factors (setup ~25 s, one sweep ~20 s)
ORACLE_SAMPLE = {1: (4, 4, 4), 2: (3, 3, 3), 3: (2, 2, 2), 4: (2, 2, 2), 5: (2, 2, 2)}
ORACLE_UNAVAILABLE = {}
SPACE_NAME = {0: "H(grad) Q", 1: "H(curl) NCE", 2: "H(div) NCF"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(cfg, kernel="patch_solve"):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of the kernel (patch_solve: the
    persistent patch kernel; apply_tri: the trilinear apply) from the committed ncu --set full
    summary of the same workload, or None."""
    path = os.path.join(ROOT, "profiles", f"r02_ncu_{kernel}_cfg{cfg}.txt")
    if not os.path.exists(path):
        path = os.path.join(ROOT, "profiles", f"r01_ncu_{kernel}_cfg{cfg}.txt")
    try:
        vals = {}
        for line in open(path):
            parts = line.rstrip("\n").split("\t")
            if len(parts) >= 3 and parts[0].startswith("dram__"):
                vals[parts[0]] = (float(parts[1]), parts[2])
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
        return rd[0] * scale[rd[1]] + wr[0] * scale[wr[1]]
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, idx):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(idx), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.strip().split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1])); mx.append(float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if "Active" in v and "Not" not in v:
                        reasons.add(nm)
            except Exception:
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def oracle_sweep_rate(w, cfg):
    """The oracle as it stands, one sweep on a bounded sample mesh: free DoFs / s."""
    from oracle.solver import Problem
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    nx, ny, nz = ORACLE_SAMPLE[cfg]
    ws = w.with_mesh(nx, ny, nz)
    pb = Problem(ws.space, ws.p, nx, ny, nz, ri.vertex_coords(ws), ri.cell_alpha(ws), ri.cell_beta(ws), ws.gamma_d,
                 decomposition=ws.decomposition, factorization=ws.factorization, matfree=(ws.perturb > 0))
    f = ri.uniform_vector(ws.cfg, 0, pb.space.ndof); f[pb.constrained] = 0
    u = ri.uniform_vector(ws.cfg, 3, pb.space.ndof); u[pb.constrained] = 0
    t0 = time.perf_counter()
    pb.patch_solvers()
    if ws.decomposition == "ph":
        pb.potential()
    _ = pb.A if not pb.matfree else None
    setup = time.perf_counter() - t0
    times = []
    for _ in range(3):
        t = time.perf_counter()
        pb.relax(f, u)
        times.append(time.perf_counter() - t)
    sec = float(np.median(times))
    nfree = int(pb.free.sum())
    return nfree / sec, {"cores": cores, "sample": f"{nx}x{ny}x{nz} cells, p={ws.p}, {nfree} free DoFs, median of 3 "
                                                    f"sweeps (oracle setup {setup:.1f} s untimed)", "sec_per_sweep": sec}


def measure(w, cfg, args, world, rank, local, torch, dist, rmb, with_e2e=True):
    """Set up one workload (z-slabs over the ranks at N > 1), time
    args.steps sweeps after args.warmup, and return the bench-line fields of that workload."""
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    # N > 1: weak-scaled z-slabs of ONE global mesh (nz * N layers), each rank the N = 1 workload's
    # cells plus halos, exchanged by the library over NCCL inside rm_relax (row a3; every space)
    slab = world > 1
    wg = dataclasses.replace(w, nz=w.nz * world) if slab else w
    t0 = time.perf_counter()
    coords = None if wg.perturb == 0 else ri.vertex_coords(wg)
    kw = {}
    if slab:
        nid = [rmb.rm_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        kw = dict(rank=rank, nranks=world, z_begin=rank * w.nz, z_end=(rank + 1) * w.nz, nccl_id=nid[0])
    ctx = rmb.rm_setup(wg.nx, wg.ny, wg.nz, wg.p, wg.space, ri.cell_alpha(wg).ravel(), ri.cell_beta(wg).ravel(),
                       wg.gamma_d, coords=coords, decomposition=rmb.RM_PH if w.decomposition == "ph" else rmb.RM_PAFW,
                       factorization=rmb.RM_ICC_SC if w.factorization == "icc_sc" else rmb.RM_CHOL,
                       stream=stream.cuda_stream, device=torch.cuda.current_device(), **kw)
    setup_s = time.perf_counter() - t0
    info = ctx.info()
    if slab:
        print(f"[bench] rank {rank}: NCCL communicator of {info['comm_nranks']} ranks (z-slab halos + allreduce), "
              f"cells z [{rank * w.nz}, {(rank + 1) * w.nz})", file=sys.stderr, flush=True)
    n = ctx.n_local
    mask = ctx.constrained_mask()
    f = ri.uniform_vector(w.cfg, 0 + 7 * rank, n); f[mask] = 0
    u = ri.uniform_vector(w.cfg, 3 + 7 * rank, n); u[mask] = 0
    ft = torch.tensor(f, device=dev)
    ut = torch.tensor(u, device=dev)
    uo = torch.empty_like(ut)

    for _ in range(args.warmup):
        rmb.rm_relax(ctx, ft, ut, uo, 1.0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = Clocks(torch.cuda.current_device())
    time.sleep(0.3)
    rmb.rm_timing_enable(ctx, True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        rmb.rm_relax(ctx, ft, ut, uo, 1.0)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1) / args.steps
    phase_ms, launches = rmb.rm_timing_read(ctx)
    rmb.rm_timing_enable(ctx, False)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    nfree_all = info["n_free"] if slab else info["n_free"] * world   # slab: n_free is the global count
    value = nfree_all / (ms * 1e-3)

    # roofline of the dominant kernel, chosen by measured time: entry 4 = the persistent patch
    # kernel launches (HBM-bound factor stream), entry 5 = the apply kernel launches (Cartesian:
    # HBM-bound; trilinear: FP64-bound, DMMA + DFMA on one datapath).  Algorithmic bytes are
    # SURVEY 8(d)'s: one read of every factor entry -- nnz(L) of the exact Cholesky factor in the
    # pinned order, or of the ICC-SC mask (rm_info factor_nnz) -- plus 24 B per DoF (r in, c out);
    # not the product's stored format.
    hbm, peak_kind = peaks()
    phases = {"residual": phase_ms[0] / args.steps, "patch_stage": phase_ms[1] / args.steps,
              "potential_stage": phase_ms[2] / args.steps, "other": phase_ms[3] / args.steps,
              "patch_kernel": phase_ms[4] / args.steps, "apply_kernel": phase_ms[5] / args.steps}
    k_ms = phase_ms[4] / args.steps
    k_launch = max(launches[4] / args.steps, 1)
    prim_bytes = 8 * info["factor_nnz"] + 3 * 8 * n
    achieved = prim_bytes / (k_ms * 1e-3) / 1e9 if k_ms > 0 else 0.0
    pk_name = "patch_batch_kernel" if info.get("batched_families", 0) else "patch_stream_kernel"
    roof_patch = {"kernel": pk_name, "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                  "frac": achieved / hbm, "traffic": ncu_traffic(cfg), "peak_kind": peak_kind,
                  "bytes_per_launch": prim_bytes / k_launch, "launches_per_step": k_launch,
                  "launch_ms_avg": k_ms / k_launch, "share_of_step": k_ms / ms if ms > 0 else None,
                  "bytes_basis": "8 B x sum nnz(L) (SURVEY 8(d)) + 24 B/DoF",
                  "factor_unique_bytes": info["factor_unique_bytes"], "phase_ms_per_step": phases}
    a_ms = phase_ms[5] / args.steps
    a_launch = max(launches[5] / args.steps, 1)
    if wg.perturb > 0:
        ncell_loc = wg.nx * wg.ny * (n // ((wg.nx * wg.p + 1) * (wg.ny * wg.p + 1)) // wg.p)
        flops = ncell_loc * TRI_FLOPS_PER_CELL
        tf = flops / (a_ms * 1e-3) / 1e12 if a_ms > 0 else 0.0
        roof_apply = {"kernel": "apply_tri_kernel", "bound": "fp64", "achieved": tf, "peak": FP64_PEAK_TFLOPS,
                      "unit": "TFLOP/s", "frac": tf / FP64_PEAK_TFLOPS, "traffic": ncu_traffic(cfg, "apply_tri"),
                      "peak_kind": "measured DMMA m8n8k4 f64 throughput (scripts/fp64_bench.cu, profiles/r02_fp64_bench.txt)",
                      "flops_per_launch": flops / a_launch, "launches_per_step": a_launch, "launch_ms_avg": a_ms / a_launch,
                      "share_of_step": a_ms / ms if ms > 0 else None, "phase_ms_per_step": phases}
    else:
        ab = 3 * 8 * n
        gbs = ab / (a_ms * 1e-3) / 1e9 if a_ms > 0 else 0.0
        roof_apply = {"kernel": ("apply_q_kernel", "apply_nce_kernel", "apply_ncf_kernel")[w.space], "bound": "hbm",
                      "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "traffic": None,
                      "peak_kind": peak_kind, "bytes_per_launch": ab / a_launch, "launches_per_step": a_launch,
                      "launch_ms_avg": a_ms / a_launch, "share_of_step": a_ms / ms if ms > 0 else None,
                      "bytes_basis": "24 B/DoF (u, f in; r out)", "phase_ms_per_step": phases}
    sec_keys = ("kernel", "bound", "achieved", "peak", "unit", "frac", "launch_ms_avg", "share_of_step")
    if a_ms > k_ms:
        roof = roof_apply
        roof["secondary"] = {k: roof_patch[k] for k in sec_keys}
    else:
        roof = roof_patch
        roof["secondary"] = {k: roof_apply[k] for k in sec_keys}

    e2e = None
    if with_e2e:
        fh = torch.tensor(f).pin_memory()
        uh = torch.tensor(u).pin_memory()
        oh = torch.empty(n, dtype=torch.float64).pin_memory()
        rmb.rm_relax_host(ctx, fh, uh, oh, 1.0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(args.steps):
            rmb.rm_relax_host(ctx, fh, uh, oh, 1.0)
        dt = (time.perf_counter() - t) / args.steps
        if world > 1:
            tt = torch.tensor([dt], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        e2e = {"value": nfree_all / dt, "unit": "DoFs/s", "h2d_bytes_per_step": 2 * 8 * n,
               "d2h_bytes_per_step": 8 * n, "ms_per_step": dt * 1e3}
    workload = (f"cfg{cfg}: {SPACE_NAME[w.space]}_{w.p} on {w.nx}x{w.ny}x{w.nz} hexes, "
                f"{'perturbed trilinear' if w.perturb else 'axis-aligned'}, {w.decomposition.upper()} stars, "
                f"{'exact Cholesky' if w.factorization == 'chol' else 'ICC-SC'}")
    config = {"workload": workload + (f" per GPU, z-slabs of {wg.nx}x{wg.ny}x{wg.nz}" if slab else ""),
              "free_dofs_per_gpu": nfree_all // world, "dofs_per_gpu": n,
              "parallelism": (f"z-slab x{world} (NCCL halos, {info['comm_nranks']}-rank communicator)" if slab
                              else f"replicas x{world}") if world > 1 else "single",
              "l2": "inputs larger than L2 (patch factors %.1f GB streamed per sweep, %.2f GB distinct)"
                    % (8 * info["factor_nnz"] / 1e9, info["factor_unique_bytes"] / 1e9),
              "setup_s": setup_s,
              "setup": {"numeric_on_device": bool(info["setup_on_device"]),
                        "host_patch_families_s": info["setup_host_family_seconds"],
                        "device_numeric_s": info["setup_device_numeric_seconds"]},
              "patches": info["n_patches"] + info["n_patches_potential"],
              "factor_blocks": info["n_factor_blocks"]}
    # the whole sweep against its roofline, T_roof = sum over phases of
    # max(bytes / BW, flops / F64) with algorithmic bytes (u, f in, u_out out; one read of every
    # factor entry) and flops (trilinear apply: TRI_FLOPS_PER_CELL per cell; solves 4 per factor
    # entry; the Cartesian sum-factorised apply's O(p) flops per DoF are below its byte term)
    ncell_all = wg.nx * wg.ny * wg.nz
    t_apply = max(3 * 8 * n / (hbm * 1e9), (ncell_all * TRI_FLOPS_PER_CELL if wg.perturb > 0 else 0) / (FP64_PEAK_TFLOPS * 1e12))
    t_solve = max(8 * info["factor_nnz"] / (hbm * 1e9), 4 * info["factor_nnz"] / (FP64_PEAK_TFLOPS * 1e12))
    t_roof_ms = (t_apply + t_solve) * 1e3
    sweep_roof = {"t_roof_ms": t_roof_ms, "t_ms": ms, "frac": t_roof_ms / ms if ms > 0 else None,
                  "terms_ms": {"apply": t_apply * 1e3, "patch_solves": t_solve * 1e3},
                  "bw_GBs": hbm, "f64_TFs": FP64_PEAK_TFLOPS, "basis": "SURVEY 8(d) T_roof / T_measured"}
    res = {"value": value, "ms_per_step": ms, "config": config, "roofline": roof, "sweep_roofline": sweep_roof,
           "e2e": e2e, "clocks": clocks, "gpu_launches": int(sum(launches[:4]))}
    ctx.close()
    torch.cuda.empty_cache()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5,
                    help="BASELINE config (default 5: the weak-scaling workload the metric is quoted on)")
    ap.add_argument("--secondary", type=int, default=2, help="second workload nested in the line (0 = none)")
    ap.add_argument("--mesh", type=int, default=0, help="override cells per direction (testing only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    w = ri.CONFIGS[args.config]
    if args.mesh:
        w = w.with_mesh(args.mesh)
    metric = "DoFs/s per relaxation sweep (fp64)"
    workload = (f"cfg{args.config}: {SPACE_NAME[w.space]}_{w.p} on {w.nx}x{w.ny}x{w.nz} hexes, "
                f"{'perturbed trilinear' if w.perturb else 'axis-aligned'}, {w.decomposition.upper()} stars, "
                f"{'exact Cholesky' if w.factorization == 'chol' else 'ICC-SC'}")

    if args.impl == "reference":
        if rank != 0:
            return
        if ORACLE_SAMPLE.get(args.config) is None:
            print(json.dumps({"impl": "reference", "unavailable": ORACLE_UNAVAILABLE[args.config]}), flush=True)
            return
        rate, cb = oracle_sweep_rate(w, args.config)
        line = {"impl": "reference", "metric": metric, "value": rate, "unit": "DoFs/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["sec_per_sweep"] * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload + " (oracle on a bounded sample)", "sample": cb["sample"]},
                "cpu_baseline": {"value": rate, "unit": "DoFs/s", "cores": cb["cores"], "kind": "oracle",
                                 "sample": cb["sample"]},
                "e2e": {"value": rate, "unit": "DoFs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if world > 1:   # torchrun pins OMP_NUM_THREADS=1: give each rank's host setup its share of the cores
        os.environ.setdefault("RM_SETUP_THREADS", str(max(1, (os.cpu_count() or 8) // world)))
    import torch
    import torch.distributed as dist
    import paper_2211_14284_b200 as rmb

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")

    res = measure(w, args.config, args, world, rank, local, torch, dist, rmb, with_e2e=not args.no_e2e)
    sec = None
    # the nested secondary workload runs at N = 1 only (the scaling runs time the primary workload;
    # per-rank host setup at N = 8 gets 1/8 of the cores)
    if args.secondary and args.secondary != args.config and world == 1:
        ws = ri.CONFIGS[args.secondary]
        r2 = measure(ws, args.secondary, args, world, rank, local, torch, dist, rmb, with_e2e=not args.no_e2e)
        sec = {"value": r2["value"], "unit": "DoFs/s", "ms_per_step": r2["ms_per_step"], "config": r2["config"],
               "roofline": r2["roofline"], "sweep_roofline": r2["sweep_roofline"], "e2e": r2["e2e"], "clocks": r2["clocks"],
               "gpu_launches": r2["gpu_launches"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if ORACLE_SAMPLE.get(args.config) is None:
            cpu = {"value": None, "unit": "DoFs/s", "cores": os.cpu_count(), "kind": "oracle",
                   "sample": None, "unavailable": ORACLE_UNAVAILABLE[args.config]}
        else:
            rate, cb = oracle_sweep_rate(w, args.config)
            cpu = {"value": rate, "unit": "DoFs/s", "cores": cb["cores"], "kind": "oracle", "sample": cb["sample"]}

    if rank == 0:
        line = {"metric": metric, "value": res["value"], "unit": "DoFs/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (rm_inputs seeded recipe)",
                "config": res["config"], "roofline": res["roofline"], "sweep_roofline": res["sweep_roofline"],
                "cpu_baseline": cpu, "e2e": res["e2e"], "clocks": res["clocks"], "gpu_launches": res["gpu_launches"]}
        if sec is not None:
            line["secondary"] = sec
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
