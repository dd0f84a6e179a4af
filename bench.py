#!/usr/bin/env python
"""Benchmark of the B200 optimized-Schwarz gravimetry solve (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

One "step" = one full Schwarz solve to h <= 1e-8 (every row of SURVEY 8(a): load
update from the resident density, warm-start residuals, batched PCG to 1e-10,
Robin traces, exchange, glued residual) on the BASELINE config C3 (P2, 64^3
cells on the paper's 250 x 250 x 15 km box, Chicxulub-like density, 8 x-slab
subdomains, two-sided OO2 transmission).  value = DOF x PCG iterations / second
summed over subdomains (SURVEY 8(d) DOF.iter/s form (ii): the throughput of the
hot loop, whole job); time_to_tol_s and DOF x outer-iterations / s (form (i)) are
reported beside it.
For N > 1 launch with torchrun (one rank per GPU, NCCL); the 8 subdomains are
split over the ranks (strong scaling at fixed S).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "DOF*CG-iter/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel="k_cg_spmv"):
    """dram bytes per launch of a kernel from the committed ncu --set full capture (or None), and the
    capture it came from (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p))
    return d.get(kernel), d.get("_source")


class ClockSampler(threading.Thread):
    """NVML clocks / throttle reasons sampled every 100 ms during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index):
        super().__init__(daemon=True)
        self.index, self.samples, self.reasons, self.stop_ev, self.max_mhz = index, [], 0, threading.Event(), None
        self.ok = False

    def run(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            while not self.stop_ev.is_set():
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                try:
                    self.reasons |= pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                except AttributeError:
                    self.reasons |= pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                time.sleep(0.1)
        except Exception as e:  # NVML missing: report, do not fail the bench
            self.err = str(e)

    def summary(self):
        self.stop_ev.set()
        self.join(timeout=2)
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b], "samples": len(self.samples)}


# ----------------------------------------------------------------------------- oracle sample (CPU)
def oracle_sample(cfg, drho, iters):
    """Times the CPU oracle (oracle/, as it stands) on a bounded sample of the workload.

    Sample: `iters` Jacobi-PCG iterations of the oracle on interior subdomain 1 (Robin-augmented
    K_1 of the config's transmission, cold start, rhs = b_1), single thread.  Returns (seconds per
    CG iteration, rows of the slab, threads used).  Assembly of the sample is not timed.
    """
    from threadpoolctl import threadpool_limits

    from oracle import linalg, mesh, schwarz

    box = mesh.Box(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
    s = 1 if cfg["nsub"] > 2 else 0
    prob = schwarz.build_problem(box, cfg["nsub"], drho=drho, only=[s], monolithic=False)
    pl, ql, pr, qr = synth.robin(cfg)
    A = schwarz.robin_operators(prob, pl, pr, ql, qr)
    Ks = schwarz.subdomain_operator(prob, s, A)
    b = prob.subs[s].b
    with threadpool_limits(limits=1):
        t = time.perf_counter()
        linalg.pcg(Ks, b, tol=1e-300, maxit=iters)
        dt = time.perf_counter() - t
    return dt / iters, Ks.shape[0], 1


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, cfg, drho, rank):
    """Reference arm: the CPU oracle as it stands, one host core, bounded sample per step."""
    if rank != 0:
        return
    vals = []
    for k in range(args.warmup + args.steps):
        t_iter, n_s, cores = oracle_sample(cfg, drho, args.ref_iters)
        if k >= args.warmup:
            vals.append((n_s / t_iter, t_iter))
    v = statistics.median([a for a, _ in vals])
    t = statistics.median([b for _, b in vals])
    sample = (f"{args.ref_iters} oracle Jacobi-PCG iterations on subdomain 1 of {args.config} (scipy CSR, 1 thread) "
              f"per step; DOF x CG-iterations / s measured directly")
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * args.ref_iters * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, cfg),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_block(args, cfg):
    return {"workload": f"{args.config}: P{cfg['order']} {cfg['nx']}x{cfg['ny']}x{cfg['nz']} Kuhn box "
                        f"{cfg['lx']/1e3:g}x{cfg['ly']/1e3:g}x{cfg['lz']/1e3:g} km, {cfg['field']} density, "
                        f"{cfg['nsub']} x-slab subdomains",
            "dof": cfg["dof"], "nsub": cfg["nsub"],
            "transmission": ({"kind": "OO2 two-sided", "p1_p2_q1_q2": cfg["robin"]} if cfg.get("robin") is not None
                             else {"kind": "OO0", "alpha": cfg["alpha"]}),
            "tol_outer": 1e-8, "tol_inner": 1e-10,
            "l2": "no flush: CG working set >> 126 MB L2 (939 MB per CG iteration at C3 on 1 GPU)",
            "parallelism": f"{cfg['nsub']} subdomains over {args.gpus} GPU(s)"}


# ----------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--alpha", default=None, help="alpha or alpha_1:alpha_2 (two-sided)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-iters", type=int, default=200)
    ap.add_argument("--e2e-steps", type=int, default=None, help="default: --steps")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (192^3, 56 M DOF) block")
    ap.add_argument("--no-alt-spmv", action="store_true",
                    help="skip the block timing the 3-byte value-indexed SELL (variant 10, row order 3)")
    ap.add_argument("--no-cpu-full", action="store_true", help="skip the oracle's measured time-to-tolerance")
    ap.add_argument("--timing-steps", type=int, default=1)
    args = ap.parse_args()
    if args.e2e_steps is None:
        args.e2e_steps = args.steps

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = dict(synth.CONFIGS[args.config])
    if args.alpha is not None:  # p | p1:p2 (OO0) | p1:p2:q1:q2 (OO2)
        v = [float(t) for t in args.alpha.split(":")]
        cfg["robin"] = tuple(v) if len(v) == 4 else None
        if len(v) < 4:
            cfg["alpha"] = v[0] if len(v) == 1 else tuple(v)
    o_ = cfg["order"]
    cfg["dof"] = (o_ * cfg["nx"] - 1) * (o_ * cfg["ny"] - 1) * (o_ * cfg["nz"] - 1)
    drho = synth.density(cfg)

    if args.impl == "reference":
        if world > 1:
            import torch.distributed as dist

            dist.init_process_group("gloo")
        run_reference(args, cfg, drho, rank)
        if world > 1:
            dist.destroy_process_group()
        return

    import torch

    import paper_2112_03851_b200 as P

    torch.cuda.set_device(local_rank)
    dist = None
    uid = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        obj = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    stream = torch.cuda.Stream()
    osm = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"], rank=rank,
                nranks=world, device=local_rank, nccl_uid=uid, stream=stream.cuda_stream)
    osm.decompose(cfg["nsub"])
    S = cfg["nsub"]
    osm.set_robin2(*synth.robin(cfg))
    t_setup = time.perf_counter()
    osm.assemble()
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    d_drho = torch.from_numpy(drho).to(f"cuda:{local_rank}")  # inputs resident in HBM
    torch.cuda.synchronize()

    def step():
        osm.upload_density_device(d_drho.data_ptr())
        return osm.solve(tol_outer=1e-8, max_outer=1000)

    for _ in range(args.warmup):
        st, rep = step()
    if st != 0:
        raise SystemExit(f"warm-up solve did not converge: status {st}, h = {rep.h_final}")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local_rank)
    clocks.start()
    launches0 = osm.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    outer, inner, cg_work = 0, 0, 0.0
    barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        st, rep = step()
        outer += rep.outer_iters
        inner += rep.inner_total
        cg_work += local_cg_work(osm, S, rank, world)
    ev1.record(stream)
    barrier()
    clk = clocks.summary()
    launches = osm.launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    if dist is not None:
        t = torch.tensor([ms], device=f"cuda:{local_rank}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        w = torch.tensor([cg_work], device=f"cuda:{local_rank}", dtype=torch.float64)
        dist.all_reduce(w)
        cg_work = float(w.item())
    ms_step = ms / args.steps
    value = cg_work / (ms / 1e3)  # DOF x CG-iterations per second, whole job

    # Dominant kernel roofline (k_cg_spmv): CUDA events around every launch on the library
    # stream, recorded during instrumented solves run right after the timed region (per-launch
    # events cost ~1 us of GPU time each, so they stay out of the timed steps).
    osm.set_kernel_timing(True)
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    traffic = dict(spmv_bytes=0.0, update_bytes=0.0, dir_bytes=0.0)
    traffic_csr = 0.0
    ev2.record(stream)
    for _ in range(args.timing_steps):
        step()
        tm = osm.traffic_model()
        for k in traffic:
            traffic[k] += tm[k]
        traffic_csr += tm["csr_equiv_bytes"]
    ev3.record(stream)
    torch.cuda.synchronize()
    ms_instr = ev2.elapsed_time(ev3)
    kt = osm.kernel_timing()
    # the same instrumented solve with the fp64 SELL kernel (variant 2): the HBM-bound reference
    # implementation of the same SpMV (bitwise-identical iterations), for the HBM roofline
    active = osm.set_spmv_variant(2)
    osm.set_kernel_timing(True)
    step()
    kt2 = osm.kernel_timing()
    tm2 = osm.traffic_model()
    default_variant = osm.set_spmv_variant(HOT_VARIANT)
    osm.set_kernel_timing(False)
    peak, peak_src = hbm_peak()
    spmv_launches, spmv_ms = kt["cg_spmv"]
    achieved = traffic["spmv_bytes"] / (spmv_ms / 1e3) / 1e9 if spmv_ms > 0 else None
    tr, tr_src = ncu_traffic()
    per_launch_alg = traffic["spmv_bytes"] / max(1, spmv_launches)
    fp64_ach = tm2["spmv_bytes"] / (kt2["cg_spmv"][1] / 1e3) / 1e9 if kt2["cg_spmv"][1] > 0 else None
    roofline_fp64 = {"bound": "hbm", "kernel": "k_cg_spmv<2> (fp64 SELL-256)", "achieved": fp64_ach, "peak": peak,
                     "unit": "GB/s", "frac": fp64_ach / peak if fp64_ach else None,
                     "traffic": ncu_traffic("fp64_sell_variant2_k_cg_spmv_r01b")[0],
                     "us_per_launch": 1e3 * kt2["cg_spmv"][1] / max(1, kt2["cg_spmv"][0]), "variant": active}
    brick = default_variant == 11
    # the Kuhn SpMV carries the direction update (k_cg_dir then runs only as the per-solve flush)
    fused = brick and kt["cg_dir"][0] < kt["cg_spmv"][0] // 2
    kname = (f"k_cg_spmv_kuhn{'_fused' if fused else ''}<{brick_bi(cfg)}>" if brick
             else f"k_cg_spmv<{default_variant}>")
    if brick:
        tr, tr_src = ncu_traffic("k_cg_spmv_kuhn_fused" if fused else "k_cg_spmv_kuhn")
    roofline = {"bound": "hbm", "kernel": kname, "variant": default_variant, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak if achieved else None,
                "traffic": tr, "traffic_source": tr_src, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": per_launch_alg,
                "share_of_cg_time": spmv_ms / sum(kt[k][1] for k in ("cg_spmv", "cg_update", "cg_dir")),
                "share_of_step": spmv_ms / ms_instr if ms_instr > 0 else None,
                "instrumented_steps": args.timing_steps,
                "cg_kernels_gbs": {k: (traffic[b] / (kt[k][1] / 1e3) / 1e9 if kt[k][1] > 0 else None)
                                   for k, b in (("cg_update", "update_bytes"), ("cg_dir", "dir_bytes"))},
                "kernel_ms": {k: v[1] for k, v in kt.items()}, "kernel_launches": {k: v[0] for k, v in kt.items()},
                "us_per_launch": 1e3 * spmv_ms / max(1, spmv_launches),
                "format": ("brick copy (row order 6): per (row, stencil slot) one u8 dictionary index, slots "
                           "in column order, 16 x BI x 2-point bricks of each parity class; + 16 B per row (p "
                           "read, q write); the p boxes are TMA-staged in shared memory (their halo re-reads "
                           "come from L2 and are not counted); dictionary (<= 256 slots) in the constant bank"
                           + ("; fused direction update: + 33 B per row (r and the 1-byte D^-1 code read, x "
                              "read and written, p_{k+1} written)" if fused else "")
                           if brick else
                           "value-indexed SELL-256, 3-byte entries: per 8 entries one 16-B load of int16 column "
                           "offsets and one 8-B load of u8 dictionary indices, + 16 B per row (p, q); dictionary "
                           "(<= 256 slots) in the constant bank (kernel parameter)" if default_variant == 10 else
                           "SELL-256 (variant %d) + 16 B per row (p, q)" % default_variant),
                "csr_equivalent_gbs": traffic_csr / (spmv_ms / 1e3) / 1e9 if spmv_ms > 0 else None,
                "frac_vs_spec_8000": achieved / SPEC_HBM_GBS if achieved else None,
                "dram_gbs_from_ncu_traffic": (tr / (1e-3 * spmv_ms / max(1, spmv_launches)) / 1e9
                                              if tr and spmv_ms > 0 and default_variant == HOT_VARIANT else None),
                "exchange": exchange_block(kt, tm, world),
                "limiter": ("instruction issue and latency at ~27 resident warps per SM (shared-memory loads, "
                            "dictionary LDCs and the FMA chain per row), not HBM: DESIGN.md 'Brick SpMV'"
                            if brick else "latency of the dependent load chains (packed entry -> x gather -> FMA)"),
                "fused_direction": fused,
                "limiter_metrics": ncu_traffic("k_cg_spmv_kuhn_fused_pipes" if fused else "k_cg_spmv_kuhn_pipes")[0]
                if brick else None}

    # Whole PCG hot loop against the HBM roofline: algorithmic bytes of the three CG kernels (SpMV in
    # its own format + update + direction) of one solve, over the timed step (everything included).
    cg_bytes = (traffic["spmv_bytes"] + traffic["update_bytes"] + traffic["dir_bytes"]) / max(1, args.timing_steps)
    cg_gbs = cg_bytes / (ms_step / 1e3) / 1e9
    cg_roofline = {"bound": "hbm", "achieved": cg_gbs, "peak": peak, "unit": "GB/s", "frac": cg_gbs / peak,
                   "frac_vs_spec_8000": cg_gbs / SPEC_HBM_GBS,
                   "bytes_per_step": cg_bytes,
                   "note": "algorithmic bytes of k_cg_spmv + k_cg_update + k_cg_dir per solve / ms_per_step "
                           "(the step also holds the outer-iteration kernels and host polling)"}

    # SURVEY 8(f) NEXT-4, reported separately: the matrix-free Kuhn-stencil SpMV (variant 5, row
    # order 4) on the same workload, timed the same way (it deviates from the paper's CSR)
    matrix_free = None
    if world == 1:
        matrix_free = run_matrix_free(P, args, cfg, d_drho, stream, peak, torch)

    # the 3-byte value-indexed SELL (variant 10, row order 3: the round-1 default), timed the same way:
    # the same CSR product in a row-wise SELL format, reported beside the default brick copy
    sell = None
    if world == 1 and not args.no_alt_spmv:
        sell = run_alt_spmv(P, args, cfg, d_drho, stream, peak, torch, row_order=3, variant=10)

    # C4 (BASELINE configs[3]), reported alongside: one batched-alpha evaluation of a CMA-ES population
    # (lambda = 25) on the C2 problem, 30 outer iterations per candidate (the cost window)
    batched = None
    if world == 1:
        batched = run_batched_alpha(P, stream, torch)

    # C5 (BASELINE configs[4], the north_star's >= 50 M-DOF target): S = 8 fixed at every N (strong
    # scaling); one instrumented warm-up solve (per-kernel events) + one timed solve
    c5 = None
    if not args.no_c5:
        c5 = run_c5(P, args, stream, torch, rank, world, dist, local_rank)

    # e2e through the C ABI with host buffers: pinned drho H2D + solve + Phi D2H, every step
    h_drho = torch.from_numpy(drho).pin_memory()
    phi = torch.empty(int(np.prod(osm.lattice)), dtype=torch.float64).pin_memory() if rank == 0 else None
    # one untimed e2e step: the instrumented solves above switched SpMV variants and kernel timing,
    # which drops the captured CUDA graphs; their re-capture is setup, not a step
    osm.upload_density(h_drho.numpy())
    osm.solve(tol_outer=1e-8, max_outer=1000)
    osm.solution(out=phi.numpy() if phi is not None else None)
    barrier()
    t0 = time.perf_counter()
    e2e_cg_work = 0.0
    for _ in range(args.e2e_steps):
        osm.upload_density(h_drho.numpy())
        st2, rep2 = osm.solve(tol_outer=1e-8, max_outer=1000)
        e2e_cg_work += local_cg_work(osm, S, rank, world)
        osm.solution(out=phi.numpy() if phi is not None else None)
    barrier()
    t_e2e = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([t_e2e], device=f"cuda:{local_rank}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_e2e = float(t.item())
        w = torch.tensor([e2e_cg_work], device=f"cuda:{local_rank}", dtype=torch.float64)
        dist.all_reduce(w)
        e2e_cg_work = float(w.item())
    e2e = {"value": e2e_cg_work / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(drho.nbytes),
           "d2h_bytes_per_step": int(np.prod(osm.lattice)) * 8, "steps": args.e2e_steps,
           "path": "osm_upload_density(host pinned) + osm_solve + osm_get_solution(host pinned)"}

    if rank != 0:
        osm.close()
        if dist is not None:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        t_iter, n_s, cores = oracle_sample(cfg, drho, args.ref_iters)
        cpu = {"value": n_s / t_iter, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"{args.ref_iters} oracle Jacobi-PCG iterations on subdomain 1 of {args.config} "
                         f"(scipy CSR, 1 thread)", "seconds_per_cg_iteration": t_iter, "sample_rows": n_s,
               "time_to_tol_s_extrapolated": t_iter / n_s * (cg_work / args.steps), "host": host_info()}
        if not args.no_cpu_full:
            cpu["measured"] = oracle_time_to_tol(args.config)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_block(args, cfg),
            "time_to_tol_s": ms_step / 1e3, "outer_iters": outer / args.steps, "inner_total": inner / args.steps,
            "dof_outer_iter_per_s": cfg["dof"] * outer / (ms / 1e3), "setup_s": t_setup,
            "roofline": roofline, "roofline_cg_step": cg_roofline, "roofline_fp64_sell": roofline_fp64,
            "matrix_free": matrix_free, "sell_spmv": sell, "batched_alpha": batched, "c5": c5,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
            "status": int(st)}
    print(json.dumps(line), flush=True)
    osm.close()
    if dist is not None:
        dist.destroy_process_group()


def exchange_block(kt, tm, world):
    """NCCL trace exchange of the instrumented solve: bytes this rank sent, time of the
    exchange calls on the stream, and the resulting rate (latency-bound at these message sizes)."""
    if world == 1:
        return None
    n, ms = kt.get("exchange", (0, 0.0))
    b = tm.get("exchange_bytes", 0.0)
    return {"calls": n, "ms": ms, "bytes_sent": b, "us_per_call": 1e3 * ms / max(1, n),
            "gbs": b / (ms / 1e3) / 1e9 if ms > 0 else None,
            "note": "per outer iteration: [g|u] to each neighbour and the interface-row residual; NVLink "
                    "fraction = gbs / 900 GB/s per direction"}


_rows = {}
HOT_VARIANT = 11  # library default SpMV: the brick copy (row order 6; falls back to 10, 6, 7 or 2)
SPEC_HBM_GBS = 8000.0  # B200 HBM3e specification (SURVEY 8(d) reports against both)


def run_batched_alpha(P, stream, torch, B=25, N=30, reps=2):
    """C4 workload: B candidate Robin parameters alpha_b = alpha0 exp(0.5 z_b) on C2 (synth), one batched
    solve of N outer iterations each, device-timed (CUDA events on the library stream)."""
    cfg = dict(synth.CONFIGS["C2"])
    o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"], stream=stream.cuda_stream)
    o.decompose(cfg["nsub"])
    o.set_robin(np.full(cfg["nsub"] - 1, cfg["alpha"]), np.full(cfg["nsub"] - 1, cfg["alpha"]))
    o.assemble()
    o.upload_density(synth.density(cfg))
    al = np.repeat(synth.alpha_candidates(cfg["alpha"], B=B)[:, None], cfg["nsub"] - 1, axis=1)
    o.solve_batch(al, al, tol_outer=1e-300, max_outer=2)  # warm-up (buffers, first launches)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(reps):
        rep = o.solve_batch(al, al, tol_outer=1e-300, max_outer=N)
    ev1.record(stream)
    torch.cuda.synchronize()
    s = ev0.elapsed_time(ev1) / 1e3 / reps
    rows = sum(o.local_solution_size(k) for k in range(cfg["nsub"]))
    o.close()
    return {"workload": f"C4: {B} candidates x {N} outer iterations on C2 (P2 32^3, 2 subdomains)",
            "seconds": s, "candidate_outer_iters_per_s": B * N / s,
            "dof_cg_iter_per_s": rows / cfg["nsub"] * rep.inner_total / s,  # equal slabs: mean n_s x inner
            "inner_total": rep.inner_total}


def brick_bi(cfg):
    """x extent (class-local planes) of the brick kernel's bricks, as brick.cu's brick_build picks it:
    the widest slab's class-local x extent (cells + 1 for P2 interface planes) in chunks of <= 12."""
    S = cfg["nsub"]
    cells = -(-cfg["nx"] // S)
    iext = cells + 1 if cfg["order"] == 2 else cells
    nchunk = -(-iext // 12)
    return -(-iext // nchunk)


def run_alt_spmv(P, args, cfg, d_drho, stream, peak, torch, row_order, variant):
    """Time an alternative SpMV (row order / variant) on the headline workload: K timed steps after W
    warm-ups (CUDA events on the library stream), then one instrumented solve for the per-launch time
    and the roofline in its own bytes (osm traffic model)."""
    S = cfg["nsub"]
    o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"], stream=stream.cuda_stream)
    o.set_row_order(row_order)
    o.decompose(S)
    o.set_robin2(*synth.robin(cfg))
    o.assemble()
    active = o.set_spmv_variant(variant)

    def step():
        o.upload_density_device(d_drho.data_ptr())
        return o.solve(tol_outer=1e-8, max_outer=1000)

    for _ in range(args.warmup):
        st, rep = step()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    work, outer = 0.0, 0
    ev0.record(stream)
    for _ in range(args.steps):
        st, rep = step()
        work += local_cg_work(o, S, 0, 1)
        outer += rep.outer_iters
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    o.set_kernel_timing(True)
    step()
    kt, tm = o.kernel_timing(), o.traffic_model()
    o.set_kernel_timing(False)
    o.close()
    n, t = kt["cg_spmv"]
    gbs = tm["spmv_bytes"] / (t / 1e3) / 1e9 if t > 0 else None
    return {"variant": active, "row_order": row_order, "status": int(st), "value": work / (ms / 1e3), "unit": UNIT,
            "time_to_tol_s": ms / args.steps / 1e3, "outer_iters": outer / args.steps,
            "spmv_us_per_launch": 1e3 * t / max(1, n), "spmv_bytes_per_launch": tm["spmv_bytes"] / max(1, n),
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak if gbs else None,
                         "note": ("bytes = the u8 index stream (1 B per brick point and stencil slot, padding "
                                  "included) + p read + q write" if active == 11 else
                                  "bytes = 3 B per kept entry (int16 offset + u8 index) + p read + q write"
                                  if active == 10 else "bytes: osm traffic model of variant %d" % active)},
            "cg_kernels_us": {k: 1e3 * v[1] / max(1, v[0]) for k, v in kt.items()}}


def run_matrix_free(P, args, cfg, d_drho, stream, peak, torch):
    """Time the matrix-free SpMV path (variant 5 in row order 4) on the headline workload: K timed
    steps after W warm-ups (CUDA events on the library stream), then one instrumented solve for the
    per-launch SpMV time.  Its algorithmic SpMV bytes are p (read), q (written) and the 1-byte row
    table code: 17 B/row."""
    S = cfg["nsub"]
    mf = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"],
               stream=stream.cuda_stream)
    mf.set_row_order(4)
    mf.decompose(S)
    mf.set_robin2(*synth.robin(cfg))
    mf.assemble()
    active = mf.set_spmv_variant(5)

    def step():
        mf.upload_density_device(d_drho.data_ptr())
        return mf.solve(tol_outer=1e-8, max_outer=1000)

    for _ in range(args.warmup):
        st, rep = step()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    work, outer = 0.0, 0
    ev0.record(stream)
    for _ in range(args.steps):
        st, rep = step()
        work += local_cg_work(mf, S, 0, 1)
        outer += rep.outer_iters
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    mf.set_kernel_timing(True)
    step()
    kt = mf.kernel_timing()
    tm = mf.traffic_model()
    mf.set_kernel_timing(False)
    mf.close()
    n, t = kt["cg_spmv"]
    gbs = tm["spmv_bytes"] / (t / 1e3) / 1e9 if t > 0 else None
    return {"variant": active, "row_order": 4, "status": int(st), "value": work / (ms / 1e3), "unit": UNIT,
            "time_to_tol_s": ms / args.steps / 1e3, "outer_iters": outer / args.steps,
            "spmv_us_per_launch": 1e3 * t / max(1, n),
            "spmv_share_of_cg_time": t / sum(kt[k][1] for k in ("cg_spmv", "cg_update", "cg_dir")),
            "roofline": {"bound": "latency", "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak if gbs else None,
                         "note": "algorithmic bytes = 17 B/row (p read, q write, 1-byte row code): no matrix "
                                 "bytes, so the kernel is bound by the latency of its gather chains, not HBM"},
            "csr_equivalent_gbs": tm["csr_equiv_bytes"] / (t / 1e3) / 1e9 if t > 0 else None,
            "cg_kernels_us": {k: 1e3 * v[1] / max(1, v[0]) for k, v in kt.items()}}


def host_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def oracle_time_to_tol(config):
    """The oracle, as it stands, solved to h <= 1e-8 on the host cores in the paper's shape (one
    process per subdomain; oracle.slabwise = oracle.schwarz distributed):
    C1 single-thread, and the bench workload with min(S, nproc) single-threaded processes.  Measured
    wall seconds of the iteration (||f|| and every outer iteration; the workers' assembly excluded)."""
    from oracle import mesh, slabwise

    out = {}
    for name in ("C1", config):
        cfg = dict(synth.CONFIGS[name])
        box = mesh.Box(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], cfg["order"])
        S = cfg["nsub"]
        nproc = 1 if name == "C1" else min(S, os.cpu_count() or 1)
        tstart = time.perf_counter()
        rep = slabwise.schwarz_slabwise(box, S, synth.density(cfg), synth.robin(cfg), tol_outer=1e-8, max_outer=1000,
                                        nproc=nproc)
        out[name] = {"time_to_tol_s": rep.seconds, "wall_incl_assembly_s": time.perf_counter() - tstart,
                     "outer_iters": rep.outer_iters, "inner_total": int(sum(map(sum, rep.inner))),
                     "converged": rep.converged, "processes": nproc, "threads_per_process": 1}
    return out


def run_c5(P, args, stream, torch, rank, world, dist, local_rank):
    """C5: 192^3 P2 cells on the paper box (56,181,887 DOF), S = 8 x-slabs split over the N ranks, OO2
    (synth.C5_ROBIN), solved to h <= 1e-8.  Warm-up = one instrumented solve (kernel events on the
    library stream: per-kernel times and the SpMV roofline in its own bytes); then one timed solve
    (CUDA events on the library stream, max over ranks)."""
    cfg = dict(synth.CONFIGS["C5"])
    uid = None
    if world > 1:
        obj = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    t0 = time.perf_counter()
    o = P.Osm(cfg["nx"], cfg["ny"], cfg["nz"], cfg["lx"], cfg["ly"], cfg["lz"], 2, rank=rank, nranks=world,
              device=local_rank, nccl_uid=uid, stream=stream.cuda_stream)
    o.decompose(cfg["nsub"])
    o.set_robin2(*synth.robin(cfg))
    o.assemble()
    d = torch.from_numpy(synth.density(cfg)).to(f"cuda:{local_rank}")
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    S = cfg["nsub"]
    o.set_kernel_timing(True)
    o.upload_density_device(d.data_ptr())
    st, rep = o.solve(tol_outer=1e-8, max_outer=200)
    kt, tm = o.kernel_timing(), o.traffic_model()
    o.set_kernel_timing(False)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    o.upload_density_device(d.data_ptr())
    st, rep = o.solve(tol_outer=1e-8, max_outer=200)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    work = local_cg_work(o, S, rank, world)
    if dist is not None:
        t = torch.tensor([ms, work], device=f"cuda:{local_rank}", dtype=torch.float64)
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:])
        ms, work = float(t[0].item()), float(t[1].item())
    peak, _ = hbm_peak()
    n, spmv_ms = kt["cg_spmv"]
    cg_ms = sum(kt[k][1] for k in ("cg_spmv", "cg_update", "cg_dir"))
    gbs = tm["spmv_bytes"] / (spmv_ms / 1e3) / 1e9 if spmv_ms > 0 else None
    out = {"workload": "C5: P2 192x192x192 Kuhn box 250x250x15 km, chicxulub density, 8 x-slab subdomains "
                       f"over {world} GPU(s), OO2 {synth.C5_ROBIN}",
           "dof": 56181887, "status": int(st), "time_to_tol_s": ms / 1e3, "outer_iters": rep.outer_iters,
           "inner_total": rep.inner_total, "value": work / (ms / 1e3), "unit": UNIT, "setup_s": setup,
           "spmv_variant": o.set_spmv_variant(HOT_VARIANT),
           "roofline": {"bound": "hbm", "kernel": "k_cg_spmv (rank 0, instrumented warm-up solve)",
                        "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak if gbs else None,
                        "us_per_launch": 1e3 * spmv_ms / max(1, n)},
           "cg_kernels_gbs": {k: (tm[b] / (kt[k][1] / 1e3) / 1e9 if kt[k][1] > 0 else None)
                              for k, b in (("cg_update", "update_bytes"), ("cg_dir", "dir_bytes"))},
           "kernel_share_of_cg": {k: kt[k][1] / cg_ms for k in ("cg_spmv", "cg_update", "cg_dir")},
           "timing": "one timed solve after one instrumented warm-up solve; CUDA events, max over ranks"}
    o.close()
    del d
    torch.cuda.empty_cache()
    return out


def local_cg_work(osm, S, rank, world):
    """sum over local subdomains s and outer iterations n of n_s x PCG iterations (DOF x CG-iter)."""
    lo, hi = rank * S // world, (rank + 1) * S // world
    its = osm.inner_iters().astype(np.int64)
    w = 0
    for s in range(lo, hi):
        key = (id(osm), osm.lattice, s)  # per context: C3, C5 and the matrix-free contexts differ
        if key not in _rows:
            _rows[key] = osm.local_solution_size(s)
        w += _rows[key] * int(np.clip(its[:, s], 0, None).sum())
    return float(w)


if __name__ == "__main__":
    main()
