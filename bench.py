"""Benchmark of the B200 Zolotarev filter path (BASELINE.json metric:
filtered vectors/s, all poles applied).

Workload (N=1): BASELINE config 2 -- 3D 7-point Laplacian on 32^3 (N=32768)
+ U[0,1] potential, SPD 7-point mass matrix B, real float64, p=8 poles
(r=4 factorizations), n_v=96, gmres_tol 1e-12, gmres_max 50, window of 64
interior eigenvalues near 6 (paper_1701_08935_b200/configs.py).

A step = one FilterOperator::apply_filter (filter_engine.hpp:86-155) of the
whole n_v-column block: 2r outer shifts by lock-step multi-shift GMRES on
G, every G application = r shifted LU solves (block-sparse nested-dissection
factors, DAG-scheduled DMMA sweeps) + B SpMM. The r factorizations are setup
(outside the timed region, reported separately as t_factor_ms).

  value : device-resident block, CUDA events on the library stream, K steps.
  e2e   : the public host API (zolo_apply_filter) from pinned host memory,
          H2D of V and D2H of Y inside the timed region.
Multi-GPU (torchrun), --shard columns (default): columns are independent (one
Krylov basis per column, filter_engine.hpp:109-111), so every rank filters its
own n_v-column block with no data-path collective -- weak scaling;
value = N * n_v / max-rank time. --shard poles: rank g factors poles
g, g + N, ... and every G application is all-reduced over NCCL inside the
library; all ranks filter the same block -- strong scaling, value = n_v / time.
--impl reference: the reference's own CPU FilterOperator (oracle/_ref,
compiled from /root/reference) on the host cores, bounded column sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "filtered vectors/s (all poles applied)"
UNIT = "vectors/s"


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    # the recipe's clocks line without power.draw (not reported; one query fewer per sample)
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        self.first = ""
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            # wait for its first sample: nvidia-smi's start-up (NVML init, device attach) stalls the
            # GPU for milliseconds and must not fall inside the timed steps
            self.first = self.proc.stdout.readline()
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        out = self.first + out
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_peaks():
    out = {}
    try:
        out.update(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))))
    except (OSError, ValueError):
        pass
    try:
        fp = json.load(open(os.path.join(REPO, "profiles", "fp64_peak_r01.json")))
        out["fp64_tflops"] = max(fp["dfma_tflops"], fp["dmma_m8n8k4_tflops"])
    except (OSError, ValueError, KeyError):
        pass
    return out


DESCR = {
    "cfg1": "2D 5-point Laplacian 64^2 (Dirichlet), B=I",
    "cfg2": "3D 7-point Laplacian 32^3 + U[0,1] potential, SPD mass B",
    "cfg3": "complex Hermitian 3D tight-binding 48^3 (Peierls phases, Anderson disorder 1.5), B=I+0.05 S",
    "cfg4": "chemistry-shaped block-sparse Hermitian pencil, 8000 atoms x 13x13 blocks, SPD overlap B",
    "cfg4s": "config 4's chemistry-shaped BSR pencil at 1000 atoms x 13x13 blocks (one-GPU size), SPD overlap B",
    "cfg5": "complex Hermitian 3D tight-binding 64^3 (disorder 2), B=I",
}


def workload(name):
    from paper_1701_08935_b200 import configs

    pen, cx, gaps, r, nv, nl = configs.config(name)
    return pen, cx, gaps, r, nv, nl


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU path (oracle/_ref)."""
    if rank != 0:
        return
    import oracle
    import paper_1701_08935_b200 as zb

    pen, cx, gaps, r, nv, nl = workload(args.config)
    cores = os.cpu_count() or 1
    if not oracle.Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libzoloref.so not built"}))
        return
    ref = oracle.Reference()
    op = ref.operator(pen, cx, gaps, r, threads=cores)
    k = min(nv, cores)
    v = zb.random_block(pen[0], nv, 1, cx=cx, orthonormalize=True)[:, :k]
    for _ in range(args.warmup):
        op.apply_filter(v)
    secs = []
    for _ in range(args.steps):
        _, it, s = op.apply_filter(v)
        secs.append(s)
    t = sum(secs) / len(secs)
    value = k / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} (reference CPU FilterOperator, {k}-column sample of n_v={nv})",
                   "N": int(pen[0]), "n_v": nv, "r": r, "gmres_tol": 1e-12},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"apply_filter on {k} of {nv} columns, {cores} threads; factorization "
                                   f"{op.t_factor:.1f} s excluded"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "t_factor_s": op.t_factor,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(pen, cx, gaps, r, nv):
    """Reference CPU path on a bounded sample (rank 0, N=1 only)."""
    import oracle
    import paper_1701_08935_b200 as zb

    cores = os.cpu_count() or 1
    if not oracle.Reference.available():
        return None
    op = oracle.Reference().operator(pen, cx, gaps, r, threads=cores)
    k = min(nv, cores)
    v = zb.random_block(pen[0], nv, 1, cx=cx, orthonormalize=True)[:, :k]
    _, it, s = op.apply_filter(v)
    return {"value": k / s, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": f"reference FilterOperator::apply_filter on {k} of {nv} columns ({cores} threads, "
                      f"{s:.1f} s); factorization {op.t_factor:.1f} s excluded"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", default="columns", choices=["columns", "poles"])
    args = ap.parse_args()
    ws, rank, local = dist_info()

    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import torch

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1701_08935_b200 as zb
    from paper_1701_08935_b200 import configs
    from paper_1701_08935_b200.design import build_filter_design

    pen, cx, gaps, r, nv, nl = workload(args.config)
    n = int(pen[0])
    design = build_filter_design(gaps, r)
    poles = args.shard == "poles" and ws > 1
    if poles:
        from paper_1701_08935_b200.sharding import pole_sharded_operator

        op = pole_sharded_operator(pen, design, r, cx, local)
    else:
        op = zb.FilterOperator(pen, design, r, is_complex=cx, device=local,
                               block_size=configs.BLOCK_SIZE.get(args.config, 1))
    t_factor_ms = op.last_timings()["factor_ms"]
    sp = op.sweep_profile()

    # each rank: its own n_v-column block (columns are independent units)
    v = zb.random_block(n, nv, 1 if poles else 1 + rank, cx=cx, orthonormalize=True)
    dt = torch.complex128 if cx else torch.float64
    dv = torch.from_numpy(np.ascontiguousarray(v.T)).to(device=f"cuda:{local}", dtype=dt)  # (nv, n) = column-major
    dy = torch.empty_like(dv)
    torch.cuda.synchronize()

    def step():
        return op.apply_filter_device(dv.data_ptr(), dy.data_ptr(), nv)

    for _ in range(args.warmup):
        step()
    units = nv if poles else ws * nv
    # e2e first, on a quiet host (the clock sampler below runs only around the device-timed loop):
    # public host API, pinned host buffers, H2D + D2H inside the timed region
    dtn = np.complex128 if cx else np.float64
    hv = torch.from_numpy(np.ascontiguousarray(v.T)).pin_memory()
    hy = torch.empty_like(hv).pin_memory()
    vh = hv.numpy().T  # column-major view over pinned memory
    yh = hy.numpy().T
    import ctypes as C

    def e2e_step():
        rep = zb._Report()
        cols = np.zeros(nv, dtype=np.int64)
        rep.column_iterations = cols.ctypes.data_as(C.POINTER(C.c_int64))
        st = zb.lib().zolo_apply_filter(op._h, C.c_void_p(hv.data_ptr()), C.c_void_p(hy.data_ptr()), nv, 1e-12, 50,
                                        C.byref(rep))
        zb._check(op._h, st)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    if ws > 1:
        torch.distributed.barrier()
    op.timer_start()
    e2e_wall = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        e2e_step()
        e2e_wall.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = op.timer_stop()
    print(f"[bench] e2e steps (wall ms): {[round(x, 2) for x in e2e_wall]}, device-timed {e2e_ms / args.steps:.2f} ms",
          file=sys.stderr, flush=True)
    if ws > 1:
        t = torch.tensor([e2e_ms], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = units / (e2e_ms / args.steps / 1e3)

    # timed region: inputs (factors 3.4 GB) are larger than L2, no flush needed
    clocks = ClockSampler(local)
    clocks.start()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    op.timer_start()
    trsm_ms = 0.0
    trsm_launches = 0
    kernel_launches = 0
    opapps = 0
    iters = []
    for _ in range(args.steps):
        rep = step()
        tm = op.last_timings()
        trsm_ms += tm["trsm_ms"]
        trsm_launches += tm["trsm_launches"]
        kernel_launches += tm["kernel_launches"]
        opapps += tm["operator_applications"]
        iters.append(rep.iterations)
    total_ms = op.timer_stop()
    torch.cuda.synchronize()
    clk = clocks.stop()
    time.sleep(0.5)  # let the host settle after the sampler exits (the eigensolver runs below)
    if ws > 1:
        t = torch.tensor([total_ms], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = units / (ms_per_step / 1e3)

    esize = 16 if cx else 8
    assert np.isfinite(yh).all()

    # roofline of the dominant kernel (the DAG-scheduled block-sparse triangular sweeps)
    peaks = load_peaks()
    # per G application, per column, per pole and per solve (P = 2 for complex pencils: solve + adjoint):
    # forward + backward sweep over the off-diagonal tiles plus the diagonal-block inverse
    # products = 2 (ntiles + nb) complex 32x32 tile-column products of 8 * 1024 flops
    chains_per_pole = 2 if cx else 1
    tile_products = 2 * (sp["offdiag_tiles"] + sp["block_rows"])
    trsm_flops = opapps * len(op.poles) * chains_per_pole * tile_products * 8.0 * 1024  # this rank, K steps
    achieved = trsm_flops / (trsm_ms * 1e-3) / 1e12 if trsm_ms > 0 else 0.0
    peak = peaks.get("fp64_tflops")
    traffic = None
    try:
        traffic = json.load(open(os.path.join(REPO, "profiles", "trsm_traffic.json"))).get("bytes_per_launch")
    except (OSError, ValueError):
        pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if poles else "weak",
        "vs_baseline": None,
        "dtype": "c128" if cx else "f64", "data": "synthetic (seeded generator, BASELINE config shape)",
        "config": {"workload": f"{args.config}: {DESCR.get(args.config, args.config)}, N={n}, "
                               f"r={r} (p={2 * r} poles), n_v={nv}, gmres_tol=1e-12, {nl}-eigenvalue window",
                   "N": n, "n_v": nv, "r": r, "ordering": "nested dissection (leaf 192), block-sparse 32x32 tiles",
                   "factor_tiles_per_pole": sp["offdiag_tiles"] + sp["block_rows"],
                   "l2": "factors > L2 (no flush needed)",
                   "parallelism": f"poles x{ws} (NCCL all-reduce per G application)" if poles
                   else f"columns x{ws} (weak)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": n * nv * esize,
                "d2h_bytes_per_step": n * nv * esize},
        "gpu_launches": int(kernel_launches),
        "roofline": {"bound": "tensor", "kernel": "dag2_kernel (warp-specialised DAG-scheduled block-sparse sweeps, DMMA f64)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": (achieved / peak) if peak else None, "traffic": traffic,
                     "peak_source": "measured FP64 tensor pipe (tools/fp64_peak.cu mma.sync.m8n8k4.f64, "
                                    "profiles/fp64_peak_r01.json; MEASURED_PEAKS.json has no FP64 figure)",
                     "algorithmic": "8 flops per complex MAC x stored factor entries (off-diagonal L and U "
                                    "tiles + diagonal-block inverses, 1024 per tile) per column per pole per "
                                    "solve per G application",
                     "trsm_share_of_step": trsm_ms / total_ms if total_ms else None,
                     "trsm_launches": trsm_launches},
        "clocks": clk,
        "t_factor_ms": t_factor_ms,
        "gmres_iterations": iters,
    }
    # the eigensolver below builds its own contexts: release this operator's factors first (config 5
    # holds 87 GB of them; two copies do not fit one GPU)
    del op
    import gc

    gc.collect()
    if ws == 1 and rank == 0:
        # BASELINE metric 2 on the same config: the whole eigensolver (factorization +
        # subspace iterations to tol 1e-10, eigensolver.hpp:154-217) through zolo_subspace_iteration
        from paper_1701_08935_b200.driver import SolveConfig, subspace_iteration

        # three independent solves (each builds its own context: ordering, symbolic analysis, factors); the
        # median is reported with all three (the first solve of a process pays one-time host/driver costs)
        runs = []
        for _ in range(3):
            res = subspace_iteration(pen, gaps, SolveConfig(n_lambda=nl, oversample_k=nv - nl, r=r, tol=1e-10,
                                                            seed=1), is_complex=cx, device=local)
            runs.append((res.time_to_all_eigenpairs, res))
        runs.sort(key=lambda x: x[0])
        res = runs[1][1]
        # the window's eigenvalue count by Sylvester inertia (BASELINE config 2: "counted by the oracle via
        # Sylvester inertia"), on the GPU
        ctr = zb.InertiaCounter(pen, is_complex=cx, device=local)
        inertia = ctr.count_in(0.5 * (gaps[0] + gaps[1]), 0.5 * (gaps[2] + gaps[3]))
        del ctr
        line["time_to_all_eigenpairs"] = {
            "value": res.time_to_all_eigenpairs, "unit": "s", "runs_s": [round(t, 4) for t, _ in runs],
            "statistic": "median of 3 solves", "t_factor_s": res.stats.factorization_time,
            "t_iter_s": res.stats.iteration_time, "found": int(len(res.lambdas)), "n_lambda": nl,
            "converged": bool(res.converged), "residual": res.residual, "n_iter": res.stats.n_iter,
            "n_gmres": res.stats.n_gmres, "inertia_count": inertia}
    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(pen, cx, gaps, r, nv)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
