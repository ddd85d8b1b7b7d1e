"""Benchmark of the B200 Zolotarev filter path (BASELINE.json metric: filtered
vectors/s, all poles applied; and time-to-all-eigenpairs in (a, b)).

Workload (N=1, default --config cfg3): BASELINE config 3, the largest one-GPU
config -- complex128 Hermitian 3D tight binding on a 48^3 periodic grid
(N = 110592, Peierls phases, Anderson disorder 1.5), B = I + 0.05 S, r = 8
factorizations (p = 16 poles), n_v = 192, gmres_tol 1e-12, window of 128
eigenvalues centred at 0 (paper_1701_08935_b200/configs.py). Inputs are
synthetic, seeded generators with the config's shapes (no dataset exists).

A step = one FilterOperator::apply_filter (filter_engine.hpp:86-155) of the
whole n_v-column block: 2r outer shifts by lock-step multi-shift GMRES on G,
every G application = 2r shifted solves (solve + adjoint on block-sparse
nested-dissection factors, DAG-scheduled DMMA sweeps) + B SpMM. The r
factorizations are setup (outside the timed region, t_factor_ms).

  value : device-resident block, CUDA events on the library stream, K steps.
  e2e   : the public host API (zolo_apply_filter) from pinned host memory,
          H2D of V and D2H of Y inside the timed region.
Multi-GPU (torchrun): --shard poles (default when r >= ranks): rank g factors
poles g, g + N, ... and every G application is all-reduced over NCCL inside
the library; all ranks filter the same block -- strong scaling, value = n_v /
max-rank time. --shard columns: every rank filters its own n_v block with all
r factors and no collective -- weak scaling, value = N n_v / max-rank time.

--impl reference: the reference's own CPU FilterOperator (oracle/_ref, compiled
from /root/reference) on the host cores; this process maps no product library
(its inputs come from the reference harness's RNG). Its RCM band LU cannot
factor config 3 within a bench step (8 x 12.4 GB, ~0.5-1 h: SURVEY.md §8(d)),
so for configs 3 / 5 the line carries value null with the reason, and its
cpu_baseline is measured on the same generator at 20^3 (configs.SMALL_SIBLING).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "filtered vectors/s (all poles applied)"
UNIT = "vectors/s"
HOST_RAM_FRACTION = 0.6  # the reference's band factors must fit in this share of host memory
REF_FACTOR_BUDGET_S = 300.0  # ... and factor within this (estimated) time to be timed at full size


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return None


def host_ram_gb():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2 ** 30
    except (ValueError, OSError):
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

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
            # wait for its first sample: nvidia-smi's start-up stalls the GPU for milliseconds and
            # must not fall inside the timed steps
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


def load_traffic(config):
    """DRAM bytes per sweep launch of this config from its committed ncu --set full capture
    (profiles/r02_traffic_<config>.json, written by tools/ncu_traffic.py), or None."""
    try:
        d = json.load(open(os.path.join(REPO, "profiles", f"r02_traffic_{config}.json")))
        return d.get("bytes_per_launch"), d.get("source")
    except (OSError, ValueError):
        return None, None


DESCR = {
    "cfg1": "2D 5-point Laplacian 64^2 (Dirichlet), B=I",
    "cfg2": "3D 7-point Laplacian 32^3 + U[0,1] potential, SPD mass B",
    "cfg3": "complex Hermitian 3D tight-binding 48^3 (Peierls phases, Anderson disorder 1.5), B=I+0.05 S",
    "cfg3s": "config 3's generator at 20^3 (N=8000), B=I+0.05 S",
    "cfg4": "chemistry-shaped block-sparse Hermitian pencil, 8000 atoms x 13x13 blocks, SPD overlap B",
    "cfg4s": "config 4's chemistry-shaped BSR pencil at 1000 atoms x 13x13 blocks (one-GPU size), SPD overlap B",
    "cfg5": "complex Hermitian 3D tight-binding 64^3 (disorder 2), B=I",
    "cfg5s": "config 5's generator at 20^3 (N=8000), B=I",
}


def reference_feasibility(ref, pen, cx, r, cores):
    """The reference's RCM band LU (band_factor.hpp:135-220) at this size: band bytes of the r
    factors and an estimated factorization time (8 N bw^2 flops per factor at ~6.5 GFlop/s per
    core, SURVEY.md §8(d) probe; r factors in parallel on min(r, cores) threads)."""
    import scipy.sparse as sp

    n, a, b = pen
    am = sp.csr_matrix((np.ones(len(a[1])), a[1], a[0]), shape=(n, n))
    bm = sp.identity(n) if b is None else sp.csr_matrix((np.ones(len(b[1])), b[1], b[0]), shape=(n, n))
    u = (am + bm).tocsr()
    u.sort_indices()
    _, bw, _ = ref.rcm(n, u.indptr.astype(np.int64), u.indices.astype(np.int64))
    band_gb = (2 * bw + 1) * n * 16 * r / 2 ** 30
    t_est = 8.0 * n * bw * bw / 6.5e9 * np.ceil(r / max(1, min(r, cores)))
    ram = host_ram_gb()
    ok = band_gb < HOST_RAM_FRACTION * (ram or 0) and t_est < REF_FACTOR_BUDGET_S
    why = (f"reference RCM band LU (band_factor.hpp:135-220) of {n} rows at half-bandwidth {bw}: "
           f"{band_gb:.0f} GB of band factors ({ram:.0f} GB host RAM), ~{t_est / 60:.0f} min of factorization "
           f"estimated -- beyond a bounded bench step")
    return ok, why, bw


def time_reference(ref, name, steps, warmup, cores):
    """The reference's FilterOperator::apply_filter on a column sample of `name` (host cores)."""
    from paper_1701_08935_b200 import configs

    pen, cx, gaps, r, nv, nl = configs.config(name)
    op = ref.operator(pen, cx, gaps, r, threads=cores)
    k = min(nv, cores)
    v = ref.random_block(pen[0], nv, 1, cx=cx, orthonormalize=True)[:, :k]
    for _ in range(warmup):
        op.apply_filter(v)
    secs = []
    for _ in range(steps):
        _, it, s = op.apply_filter(v)
        secs.append(s)
    t = sum(secs) / len(secs)
    return dict(value=k / t, seconds=t, k=k, nv=nv, t_factor=op.t_factor, n=int(pen[0]), r=r)


def reference_eigenpairs(ref, name, cores):
    """The reference's subspace_iteration (eigensolver.hpp:154-217): t_fact + t_iter."""
    from paper_1701_08935_b200 import configs

    pen, cx, gaps, r, nv, nl = configs.config(name)
    res = ref.subspace_iteration(pen, cx, gaps, nl, nv - nl, r, tol=1e-10, seed=1, threads=cores)
    return {"config": name, "value": res["t_fact"] + res["t_iter"], "unit": "s", "t_fact_s": res["t_fact"],
            "t_iter_s": res["t_iter"], "found": len(res["lambdas"]), "n_lambda": nl, "converged": res["converged"],
            "residual": res["residual"], "n_iter": res["n_iter"], "n_gmres": res["n_gmres"]}


def run_reference(args, ws, rank):
    """--impl reference: the reference's own CPU path (oracle/_ref) on this host's cores; no product
    library is mapped into this process."""
    if rank != 0:
        return
    import oracle
    from paper_1701_08935_b200 import configs

    cores = os.cpu_count() or 1
    if not oracle.Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libzoloref.so not built"}))
        return
    ref = oracle.Reference()
    configs.use_uniform_source(ref.uniform_stream)  # the seeded inputs without the product library
    pen, cx, gaps, r, nv, nl = configs.config(args.config)
    ok, why, bw = reference_feasibility(ref, pen, cx, r, cores)
    del pen
    line = {
        "impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128" if cx else "f64", "data": "synthetic (seeded generator, BASELINE config shape)",
        "config": {"workload": f"{args.config}: {DESCR.get(args.config, args.config)}", "r": r, "n_v": nv,
                   "gmres_tol": 1e-12, "reference_rcm_half_bandwidth": bw},
        "host": {"cpu_model": cpu_model(), "cores": cores, "ram_gb": host_ram_gb()},
    }
    if ok:
        t = time_reference(ref, args.config, args.steps, args.warmup, cores)
        line.update({"value": t["value"], "ms_per_step": t["seconds"] * 1e3, "t_factor_s": t["t_factor"]})
        line["config"]["workload"] += f" (reference CPU FilterOperator, {t['k']}-column sample of n_v={nv})"
        line["cpu_baseline"] = {"value": t["value"], "unit": UNIT, "cores": cores, "kind": "reference",
                                "sample": f"apply_filter on {t['k']} of {nv} columns, {cores} threads; factorization "
                                          f"{t['t_factor']:.1f} s excluded"}
        line["e2e"] = {"value": t["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    else:
        line.update({"value": None, "ms_per_step": None, "unavailable": why,
                     "e2e": {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
        sib = configs.SMALL_SIBLING.get(args.config)
        if sib:
            t = time_reference(ref, sib, max(1, min(args.steps, 2)), 0, cores)
            line["cpu_baseline"] = {
                "value": t["value"], "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"NOT the headline config: {sib} = {DESCR[sib]}, r={t['r']}, apply_filter on {t['k']} of "
                          f"{t['nv']} columns, {cores} threads; factorization {t['t_factor']:.1f} s excluded"}
            line["time_to_all_eigenpairs_sibling"] = reference_eigenpairs(ref, sib, cores)
    maps = open("/proc/self/maps").read()
    assert "libzolo_b200" not in maps, "the reference arm must not map the product library"
    line["product_library_mapped"] = False
    print(json.dumps(line), flush=True)


def cpu_baseline(name, cores):
    """Reference CPU path on a bounded sample (rank 0, N=1 only): the config itself when its band
    LU is feasible, else its small sibling (clearly labelled)."""
    import oracle
    from paper_1701_08935_b200 import configs

    if not oracle.Reference.available():
        return None, None
    ref = oracle.Reference()
    pen, cx, gaps, r, nv, nl = configs.config(name)
    ok, why, _ = reference_feasibility(ref, pen, cx, r, cores)
    target = name if ok else configs.SMALL_SIBLING.get(name)
    if target is None:
        return None, why
    t = time_reference(ref, target, 1, 0, cores)
    label = "" if ok else f"NOT the headline config ({why}): "
    return {"value": t["value"], "unit": UNIT, "cores": cores, "kind": "reference", "cpu_model": cpu_model(),
            "sample": f"{label}{target}, reference FilterOperator::apply_filter on {t['k']} of {t['nv']} columns "
                      f"({cores} threads, {t['seconds']:.1f} s); factorization {t['t_factor']:.1f} s excluded"}, \
        (None if ok else target)


def gpu_filter_rate(name, device, steps=3):
    """Our device-resident filtered vectors/s on another config (the same-instance comparison)."""
    import torch

    import paper_1701_08935_b200 as zb
    from paper_1701_08935_b200 import configs
    from paper_1701_08935_b200.design import build_filter_design

    pen, cx, gaps, r, nv, nl = configs.config(name)
    op = zb.FilterOperator(pen, build_filter_design(gaps, r), r, is_complex=cx, device=device,
                           block_size=configs.BLOCK_SIZE.get(name, 1))
    v = zb.random_block(pen[0], nv, 1, cx=cx, orthonormalize=True)
    dt = torch.complex128 if cx else torch.float64
    dv = torch.from_numpy(np.ascontiguousarray(v.T)).to(device=f"cuda:{device}", dtype=dt)
    dy = torch.empty_like(dv)
    op.apply_filter_device(dv.data_ptr(), dy.data_ptr(), nv)
    op.timer_start()
    for _ in range(steps):
        op.apply_filter_device(dv.data_ptr(), dy.data_ptr(), nv)
    ms = op.timer_stop() / steps
    return nv / (ms / 1e3)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-eigensolver", action="store_true")
    ap.add_argument("--shard", default="auto", choices=["auto", "columns", "poles"])
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

    pen, cx, gaps, r, nv, nl = configs.config(args.config)
    n = int(pen[0])
    design = build_filter_design(gaps, r)
    shard = args.shard
    if shard == "auto":  # north_star's mode: poles over the GPUs (columns only beyond r ranks)
        shard = "poles" if ws > 1 and r >= ws else "columns"
    poles = shard == "poles" and ws > 1
    if poles:
        from paper_1701_08935_b200.sharding import pole_sharded_operator

        op = pole_sharded_operator(pen, design, r, cx, local, block_size=configs.BLOCK_SIZE.get(args.config, 1))
    else:
        op = zb.FilterOperator(pen, design, r, is_complex=cx, device=local,
                               block_size=configs.BLOCK_SIZE.get(args.config, 1))
    t_factor_ms = op.last_timings()["factor_ms"]
    sp = op.sweep_profile()

    # each rank: its own n_v-column block (columns are independent units) or, pole-sharded, the same block
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
    hv = torch.from_numpy(np.ascontiguousarray(v.T)).pin_memory()
    hy = torch.empty_like(hv).pin_memory()
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

    # timed region: inputs (the factors, GBs) are larger than L2, no flush needed
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

    # roofline of the dominant kernel (the DAG-scheduled block-sparse triangular sweeps); per G
    # application, per column, per pole and per solve (P = 2 for complex pencils: solve + adjoint):
    # forward + backward sweep over the off-diagonal tiles plus the diagonal-block inverse products
    # = 2 (ntiles + nb) complex 32x32 tile-column products. ALGORITHMIC flops (SURVEY.md §8(d):
    # 8 flops per complex MAC x nnz of the factors x n_b) count the nonzero entries of those tiles
    # (sweep_profile nonzero_entries, the scalar fill); the kernel executes the entries of the
    # unmasked 8x4 blocks (executed_entries) with 3 real DMMAs per complex MAC (3M, mma.cuh).
    peaks = load_peaks()
    chains_per_pole = 2 if cx else 1
    tile_products = 2 * (sp["offdiag_tiles"] + sp["block_rows"])
    stored_entries = tile_products * 1024
    frac_nz = sp["nonzero_entries"] / stored_entries if stored_entries else None
    frac_exec = sp["executed_entries"] / stored_entries if stored_entries else None
    units_solved = opapps * len(op.poles) * chains_per_pole  # column solves, this rank, K steps
    stored_flops = units_solved * stored_entries * 8.0
    trsm_s = trsm_ms * 1e-3
    achieved = stored_flops * frac_nz / trsm_s / 1e12 if trsm_ms > 0 else 0.0  # algorithmic (scalar fill)
    # real flops the FP64 pipe executes: 3 DMMAs (6 flops) per complex MAC of the executed entries
    pipe_flops = units_solved * sp["executed_entries"] * 6.0
    peak = peaks.get("fp64_tflops")
    traffic, traffic_src = load_traffic(args.config)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if poles else "weak",
        "vs_baseline": None,
        "dtype": "c128" if cx else "f64", "data": "synthetic (seeded generator, BASELINE config shape)",
        "config": {"workload": f"{args.config}: {DESCR.get(args.config, args.config)}, N={n}, "
                               f"r={r} (p={2 * r} poles), n_v={nv}, gmres_tol=1e-12, {nl}-eigenvalue window, "
                               f"direct solves at every pole",
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
                     "traffic_source": traffic_src or "no ncu capture of this config committed (profiles/)",
                     "peak_source": "measured FP64 tensor pipe (tools/fp64_peak.cu mma.sync.m8n8k4.f64, "
                                    "profiles/fp64_peak_r01.json; MEASURED_PEAKS.json has no FP64 figure)",
                     "algorithmic": "8 flops per complex MAC x nonzero entries of the sweep tiles (off-diagonal "
                                    "L and U tiles + diagonal-block inverses: the scalar fill of the factors) per "
                                    "column per pole per solve per G application (SURVEY.md §8(d) flops_G)",
                     "stored_entries_per_pole_solve": stored_entries,
                     "executed_fraction": frac_exec, "scalar_fill_fraction": frac_nz,
                     "achieved_stored_tiles": stored_flops / trsm_s / 1e12 if trsm_ms > 0 else None,
                     "fp64_pipe_tflops_executed": pipe_flops / trsm_s / 1e12 if trsm_ms > 0 else None,
                     "trsm_share_of_step": trsm_ms / total_ms if total_ms else None,
                     "trsm_launches": trsm_launches},
        "clocks": clk,
        "t_factor_ms": t_factor_ms,
        "gmres_iterations": iters,
    }
    # the eigensolver below builds its own contexts: release this operator's factors first
    del op
    import gc

    gc.collect()
    zb.pool_trim(local)
    if ws == 1 and rank == 0 and not args.no_eigensolver:
        # BASELINE metric 2 on the same config: the whole eigensolver (design + factorization +
        # subspace iterations to tol 1e-10, eigensolver.hpp:154-217) through zolo_subspace_iteration
        from paper_1701_08935_b200.driver import SolveConfig, subspace_iteration

        runs = []
        for _ in range(3):
            res = subspace_iteration(pen, gaps, SolveConfig(n_lambda=nl, oversample_k=nv - nl, r=r, tol=1e-10,
                                                            seed=1), is_complex=cx, device=local)
            runs.append((res.time_to_all_eigenpairs, res))
        runs.sort(key=lambda x: x[0])
        res = runs[1][1]
        zb.pool_trim(local)
        ctr = zb.InertiaCounter(pen, is_complex=cx, device=local)
        inertia = ctr.count_in(0.5 * (gaps[0] + gaps[1]), 0.5 * (gaps[2] + gaps[3]))
        del ctr
        line["time_to_all_eigenpairs"] = {
            "value": res.time_to_all_eigenpairs, "unit": "s", "runs_s": [round(t, 4) for t, _ in runs],
            "statistic": "median of 3 solves", "t_factor_s": res.stats.factorization_time,
            "t_iter_s": res.stats.iteration_time, "found": int(len(res.lambdas)), "n_lambda": nl,
            "converged": bool(res.converged), "residual": res.residual,
            "residual_rel_lambda": res.residual_rel_lambda, "n_iter": res.stats.n_iter,
            "n_gmres": res.stats.n_gmres, "refined_from_iteration": res.stats.refined_from,
            "first_iteration_residual": res.stats.first_residual, "inertia_count": inertia}
    if ws == 1 and rank == 0 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        cb, sib = cpu_baseline(args.config, cores)
        line["cpu_baseline"] = cb
        if sib:  # the same-instance comparison on the sibling the reference can run
            ours = gpu_filter_rate(sib, local)
            line["sibling_comparison"] = {"config": sib, "ours": ours, "reference": cb["value"], "unit": UNIT,
                                          "ratio": ours / cb["value"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
