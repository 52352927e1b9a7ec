"""Benchmark of the B200 hot path of arXiv 2309.03347 (TT/QTT k-eigenvalue).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c4|c1|c2|c3|c5]
                    [--impl ours|reference]

Default workload: BASELINE.json configs[3] (C4: 256^3 QTT, G=30 with upscatter,
S16 288 ordinates, three regions, eps 1e-6, rmax 128) -- the largest
single-GPU config, on which the metric's "k-eff fixed-point iterations/sec" is
quoted.  A step is ONE fixed-point iteration of eqn:TT_k_eff_fixed_points
(reading Z36): B = amen_mv((S + F/k), Psi) (the paper's product,
P:1501-1506), the AMEn solve of H Psi' = B (local applies, interface updates,
GMRES, truncation, enrichment: every §8(a) row), <f, Psi'>, ||Psi'|| and the k
update, continuing the solve from the state the previous step left on the
device (keff_opts.warm).  Untimed settle iterations bring the ranks to rmax
first, so the timed steps are the steady-state (most expensive) iterations.
`value` = iterations/s over all ranks (replicas, weak scaling: every rank
solves its own copy, no data-path collective -- DESIGN.md "Multi-GPU").
The metric's first half is reported in the same line on its own configs:
`c5_r256` (configs[4] ALS double sweep, GFLOP/s and % of the FP64 DMMA peak)
and `c2_b64` (configs[1] 64-instance batched tt_matvec, GB/s and % of HBM).
--workload c1 / c2 / c3 / c5 time the other configs on their own.

--impl reference times the fp64 CPU oracle (oracle/, the only other place
bench.py executes it) on a bounded sample of the same workload.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TT contraction FP64 GFLOP/s (% DMMA peak); k-eff fixed-point iterations/sec"
DMMA_FALLBACK = 37.1e3   # GFLOP/s, tools/peaks_fp64 on this pool (profiles/peaks_fp64_r01.json)


def peaks():
    p = {"hbm_gbs": 6539.9, "hbm_src": "MEASURED_PEAKS.json", "dmma_gflops": DMMA_FALLBACK,
         "dmma_src": "profiles/peaks_fp64_r01.json"}
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        p["hbm_gbs"] = float(mp["hbm_gbs"])
    except Exception:
        p["hbm_gbs"], p["hbm_src"] = 6650.0, "fallback B200_PROFILING.md"
    try:
        pf = json.load(open(os.path.join(ROOT, "profiles", "peaks_fp64_r01.json")))
        p["dmma_gflops"] = 1e3 * float(pf["dmma_tflops_sustained"])
    except Exception:
        pass
    return p


# ------------------------------------------------------------ clocks ---
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.rows, self.stop = index, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------- workloads ---
def c1_setup(device):
    import inputs
    import paper_2309_03347_b200 as tb
    from paper_2309_03347_b200 import transport as gtr
    prob = inputs.problem_c1()
    ops = gtr.operators(prob, device=device)
    modes = [8, 8, 8, 8, 1]
    g = inputs.rng(61)
    z0 = inputs.random_tt(g, modes, [1, 4, 4, 4, 4, 1])
    psi0 = [np.ones((1, n, 1)) for n in modes]
    return {"prob": prob, "ops": ops, "modes": modes, "z0": z0, "psi0": psi0, "rmax": 64, "kick": 4,
            "opts": dict(tol_k=1e-12, eps_round=1e-13, eps_solve=1e-12, rmax=64,
                         matvec=os.environ.get("TT_BENCH_MATVEC", "amen_mv"))}


def c1_step(st, device, host_inputs=None):
    import paper_2309_03347_b200 as tb
    d = len(st["modes"])
    cap = [1] + [st["rmax"] + st["kick"]] * (d - 1) + [1]
    psi = tb.TTVec.from_cores(st["psi0"], rcap=cap, device=device)
    z = tb.TTVec.from_cores(st["z0"], device=device)
    ops = st["ops"]
    res = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, **st["opts"])
    return res


def c1_step_device(st):
    """Device-resident step: psi / z reset by device copies, then the solve."""
    import paper_2309_03347_b200 as tb
    ops = st["ops"]
    tb.tt_copy(st["psi_init"], st["psi"])
    tb.tt_copy(st["z_init"], st["z"])
    return tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], st["psi"], st["z"], **st["opts"])


def ops_bytes(ops):
    return sum(int(o.data.numel()) * 8 for o in ops.values())


# ------------------------------------------------------- oracle side ---
def oracle_c1_sample(iters=3):
    """Bounded sample of the same workload on the CPU oracle: `iters` fixed-point
    iterations of the TT k-eff loop on C1 (oracle/solvers.keff_tt)."""
    import inputs
    from oracle import solvers as so
    from oracle import transport as T
    prob = inputs.problem_c1()
    tops = T.tt_operators(prob)
    modes = [8, 8, 8, 8, 1]
    g = inputs.rng(61)
    z0 = inputs.random_tt(g, modes, [1, 4, 4, 4, 4, 1])
    psi0 = [np.ones((1, n, 1)) for n in modes]
    t = time.perf_counter()
    so.keff_tt(tops["H"], tops["S"], tops["F"], psi0, z0, tol_k=0.0, eps_round=1e-13, eps_solve=1e-12,
               max_outer=iters, dense_max=0, rmax=64, matvec=os.environ.get("TT_BENCH_MATVEC", "amen_mv"))
    dt = time.perf_counter() - t
    return iters / dt, dt


def count_kernels(run):
    """Exact kernel count of one more (untimed) step: CUPTI activity records,
    graph-replayed kernels included (paper_2309_03347_b200/liblaunchcount.so).
    Returns (libtt kernels, all kernels) or None if CUPTI is unavailable."""
    import ctypes as C
    import torch
    path = os.path.join(ROOT, "paper_2309_03347_b200", "liblaunchcount.so")
    if not os.path.exists(path):
        return None
    try:
        lc = C.CDLL(path)
        torch.cuda.synchronize()
        if lc.lc_start() != 0:
            return None
        run()
        torch.cuda.synchronize()
        a, o = C.c_ulonglong(0), C.c_ulonglong(0)
        lc.lc_stop(C.byref(a), C.byref(o))
        return int(o.value), int(a.value)
    except OSError:
        return None


def count_kernels_k11(run):
    """gpu_launches of a device-resident (graph mode 2) step.  CUPTI does not report
    every kernel executed inside conditional graph nodes (the mode-2 count comes out
    ~40% low), so the claim is the CUPTI count of the SAME step on the host-stepped
    path (graph mode 1: the identical kernel sequence — bitwise-equal results,
    tests/test_gpu_solvers.py::test_device_loops_* — without the few condition
    kernels).  Returns (libtt kernels, all kernels, how, CUPTI count in mode 2)."""
    from paper_2309_03347_b200 import _lib
    lib = _lib.lib()
    seen2 = count_kernels(run)
    lib.tt_set_graph_mode(1)
    try:
        kc = count_kernels(run)
    finally:
        lib.tt_set_graph_mode(-1)
    if not kc:
        return None
    how = ("libtt kernels of one more identical step, counted exactly by CUPTI activity records on the "
           "host-stepped path (graph mode 1, the same kernel sequence as the timed device-resident graph; CUPTI "
           f"saw {seen2[0] if seen2 else None} of them inside the mode-2 graph's conditional nodes)")
    return kc[0], kc[1], how, (seen2[0] if seen2 else None)


def cpu_cores():
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        return max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        return os.cpu_count()


# --------------------------------------------------------------- main ---
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--settle", type=int, default=None, help="c3/c4: untimed iterations before the warm-up")
    ap.add_argument("--no-extras", action="store_true", help="c4: skip the c5_r256 / c2_b64 keys")
    ap.add_argument("--rank", type=int, default=128, help="c5 interface rank (64, 128, 256)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-graph", action="store_true", help="c5: launch the sweep without a CUDA graph")
    ap.add_argument("--one-stream", action="store_true", help="c5: applies and updates on one stream")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # not under torchrun: launch N ranks (one process per GPU) ourselves
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29531"),
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        if args.workload == "c4":
            vals, cb = [], None
            for _ in range(max(1, min(args.steps, 3))):
                cb = cpu_baseline("c4")
                vals.append(cb["value"])
            val = statistics.median(vals)
            cb["value"] = val
            line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "iter/s", "n_gpus": args.gpus,
                    "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / val, "higher_is_better": True,
                    "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                    "config": {"workload": KEFF_CFG["c4"]["label"] + ", rmax 128, eps 1e-6, B by amen_mv; step = one "
                                           "k-eff fixed-point iteration (oracle estimate, see cpu_baseline.sample)"},
                    "cpu_baseline": cb,
                    "e2e": {"value": val, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
            print(json.dumps(line))
            return
        v, dt = oracle_c1_sample(iters=max(1, min(args.steps, 5)))
        vals = [v]
        for _ in range(max(0, min(args.steps, 3) - 1)):
            vals.append(oracle_c1_sample(iters=2)[0])
        val = statistics.median(vals)
        line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "iter/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / val,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": "C1 (configs[0]) TT k-eff fixed point, 8^3 S2 G=1, B by amen_mv"},
                "cpu_baseline": {"value": val, "unit": "iter/s", "cores": cpu_cores(), "kind": "oracle",
                                 "sample": "fixed-point iterations of oracle keff_tt on C1 (amen_mv products, GMRES "
                                           "local solves)"},
                "e2e": {"value": val, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=device)
        dist = tdist
    import paper_2309_03347_b200 as tb
    from paper_2309_03347_b200 import _lib
    import ctypes as C

    if args.workload in ("c2", "c3", "c4", "c5"):
        if args.workload in ("c3", "c4"):
            line = keff_bench(args, tb, device, world, dist, rank)
            if args.workload == "c4" and not args.no_extras:
                line.update(extras(args, tb, device, world))
            if rank == 0 and not args.no_cpu_baseline:
                line["cpu_baseline"] = cpu_baseline(args.workload, line.get("arnoldi_steps_per_core_per_step"),
                                                    line.get("psi_ranks"))
        else:
            line = micro_bench(args, tb, device, world, dist)
        if rank == 0:
            print(json.dumps(line))
        if dist:
            dist.destroy_process_group()
        return

    st = c1_setup(device)
    d = len(st["modes"])
    cap = [1] + [st["rmax"] + st["kick"]] * (d - 1) + [1]
    st["psi_init"] = tb.TTVec.from_cores(st["psi0"], rcap=cap, device=device)
    st["psi"] = tb.TTVec.from_cores(st["psi0"], rcap=cap, device=device)
    st["z_init"] = tb.TTVec.from_cores(st["z0"], device=device)
    st["z"] = tb.TTVec.from_cores(st["z0"], device=device)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=device)   # > 126 MB L2

    for _ in range(args.warmup):
        c1_step_device(st)
    torch.cuda.synchronize()

    cnt = (C.c_uint64 * 5)()
    lib = _lib.lib()
    lib.tt_counters(cnt, 1)
    fl, fms, ffl = C.c_int64(0), C.c_double(0.0), (C.c_double * 3)()
    lib.tt_fused_profile_read(C.byref(fl), C.byref(fms), ffl)     # reset
    lib.tt_fused_profile(1)
    stream = torch.cuda.current_stream()
    step_ms, iters_total = [], 0
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.fill_(1.0)                          # evict L2 between timed steps (untimed)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = c1_step_device(st)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            iters_total += int(res.iters.item())
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        wall = time.perf_counter() - t0
    lib.tt_counters(cnt, 1)
    lib.tt_fused_profile_read(C.byref(fl), C.byref(fms), ffl)
    lib.tt_fused_profile(0)
    dev_ms = sum(step_ms)
    dev_ms_max, iters_all = aggregate_ranks(dev_ms, iters_total, dist, device)
    value = iters_all / (dev_ms_max * 1e-3)
    gemm_flops, mv_flops, qr_flops, svd_flops, ngemm = [int(v) for v in cnt]
    contraction = (gemm_flops + mv_flops) / args.steps
    pk = peaks()
    contr_gflops = contraction / (dev_ms / args.steps * 1e-3) / 1e9

    # ---- roofline of the dominant kernel: the fused GMRES Arnoldi-step kernel
    #      (local-apply DMMA GEMM stages + CGS2), timed live inside the timed region
    #      by its in-kernel %globaltimer (the step is one device-resident graph
    #      launch); flops counted on the device
    fused_flops = ffl[0] + ffl[1]
    fused_ms = fms.value
    ach = fused_flops / (fused_ms * 1e-3) / 1e12 if fused_ms > 0 else None
    roof = {"kernel": "gm_chunk_kernel (fused GMRES Arnoldi steps: 3 local-apply DMMA GEMM stages + CGS2 + Givens, "
                      "cooperative persistent grid)",
            "bound": "tensor", "achieved": ach, "peak": pk["dmma_gflops"] / 1e3, "unit": "TFLOP/s",
            "frac": (ach / (pk["dmma_gflops"] / 1e3)) if ach else None,
            "peak_src": "measured FP64 DMMA sustained (tools/peaks_fp64)", "traffic": None,
            "launches": fl.value, "ms_per_launch": fused_ms / max(fl.value, 1),
            "flops_per_launch": fused_flops / max(fl.value, 1),
            "arnoldi_steps_per_launch": ffl[2] / max(fl.value, 1),
            "share_of_step_time": fused_ms / dev_ms if dev_ms > 0 else None,
            "note": "latency-bound: local systems of <= 32768 unknowns, 6-8 grid barriers per Arnoldi step; "
                    "time = in-kernel %globaltimer of the launches that did work (graph mode 2)",
            "gemm_chain_alone": dominant_gemm_roofline(tb, device, pk)}

    # ---- end to end: host buffers (pinned) -> device, solve, result -> host
    e2e = e2e_c1(tb, st, device, args.steps)

    line = {"metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C1 (configs[0]): TT k-eff fixed point to |dk|<1e-12, 8^3 vertices, S2, G=1, "
                                   "modes (8,8,8,8,1), rmax 64, B by " + st["opts"]["matvec"],
                       "l2": "256 MB flush between timed steps", "parallelism": f"replicas x{world}"},
            "iters_per_step": iters_total / args.steps,
            "contraction_gflops": contr_gflops,
            "contraction_pct_dmma_peak": 100.0 * contr_gflops / pk["dmma_gflops"],
            "flops_per_step": {"gemm": gemm_flops / args.steps, "matvec": mv_flops / args.steps,
                               "qr": qr_flops / args.steps, "jacobi": svd_flops / args.steps,
                               "gemm_calls": ngemm / args.steps},
            "roofline": roof, "e2e": e2e, "clocks": clk.summary(),
            "gpu_launches": None, "wall_s": wall}
    kc = count_kernels_k11(lambda: c1_step_device(st))
    line["gpu_launches"] = kc[0] if kc else None
    line["gpu_launches_how"] = kc[2] if kc else "CUPTI unavailable"
    if kc:
        line["gpu_launches_all_kernels"] = kc[1]
        line["gpu_launches_cupti_mode2"] = kc[3]
    line["graph_mode"] = int(lib.tt_graph_mode())
    if rank == 0 and not args.no_cpu_baseline:
        v, dt = oracle_c1_sample(iters=3)
        line["cpu_baseline"] = {"value": v, "unit": "iter/s", "cores": cpu_cores(), "kind": "oracle",
                                "sample": f"3 fixed-point iterations of oracle keff_tt on C1, amen_mv products ({dt:.1f} s)"}
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def aggregate_ranks(dev_ms, units, dist=None, device="cpu"):
    """Whole-job aggregation over replicas: the device time is the MAX over ranks
    and the work (units processed) the SUM; value = units / max time."""
    if not dist:
        return float(dev_ms), float(units)
    import torch
    t = torch.tensor([float(dev_ms), float(units)], dtype=torch.float64, device=device)
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    sm = t.clone()
    dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    return float(mx[0]), float(sm[1])


def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def micro_bench(args, tb, device, world, dist):
    """c5: one ALS double sweep (configs[4]); c2: tt_matvec + tt_round(1e-8, 128)
    of one d=30 instance (configs[1]).  Same JSON shape as the default line."""
    import torch
    import inputs
    pk = peaks()
    s = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=device)
    if args.workload == "c5":
        from paper_2309_03347_b200.sweep import SweepProblem
        inst = inputs.c5_instance(args.rank, seed=args.seed)
        sp = SweepProblem(inst["A"], inst["X"], device)
        sp.build_right()
        run = sp.double_sweep
        if not args.no_graph:
            run = sp.capture(two_streams=not args.one_stream).replay
        for _ in range(args.warmup):
            run()
        ms = []
        with ClockSampler(torch.cuda.current_device()) as clk:
            for _ in range(args.steps):
                flush.fill_(1.0)
                e0, e1 = _events()
                e0.record(s)
                run()
                e1.record(s)
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
        t = statistics.median(ms)
        flops = sp.flops()
        gfl = flops / (t * 1e-3) / 1e9
        peak = pk["dmma_gflops"]
        return {"metric": METRIC, "value": gfl, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"C5 (configs[4]) ALS double sweep, d=40, r={args.rank}, R 5-8, "
                                       f"n in {{2,4,8,16}}, seed {args.seed}",
                           "launch": ("CUDA graph of the 80 core visits" + (", applies on a side stream beside the "
                                      "interface-update chain" if not args.one_stream else ", one stream"))
                                     if not args.no_graph else "stream",
                           "l2": "256 MB flush between timed steps"},
                "pct_dmma_peak": 100.0 * gfl / peak, "flops_per_step": flops, "ms_p10_p90": [
                    float(np.percentile(ms, 10)), float(np.percentile(ms, 90))],
                "roofline": {"kernel": "gemm_dmma_kernel (als_local_apply / als_update_interfaces chains)",
                             "bound": "tensor", "achieved": gfl / 1e3, "peak": peak / 1e3, "unit": "TFLOP/s",
                             "frac": gfl / peak, "peak_src": "measured FP64 DMMA sustained (tools/peaks_fp64)",
                             "traffic": None},
                "clocks": clk.summary(), "gpu_launches": (count_kernels(run) or (80 * 8, 0))[0],
                "gpu_launches_how": "libtt kernels of one more double sweep (CUPTI activity records)"}
    # c2
    inst = inputs.c2_instance(args.seed)
    A = tb.TTMat.from_cores(inst["A"], device=device)
    X = tb.TTVec.from_cores(inst["X"], device=device)
    Y = tb.matvec_out(A, X)
    Yr = tb.TTVec(Y.n, Y.rcap, device)
    mv_bytes = 8 * sum(R0 * 4 * R1 + r0 * 2 * r1 + R0 * R1 * 2 * r0 * r1 for R0, R1, r0, r1 in
                       zip(inst["R"][:-1], inst["R"][1:], inst["r"][:-1], inst["r"][1:]))
    for _ in range(args.warmup):
        tb.tt_matvec(A, X, Y)
        tb.tt_copy(Y, Yr)
        tb.tt_round(Yr, 1e-8, 128)
    mv_ms, rd_ms = [], []
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            e0, e1 = _events()
            e2, e3 = _events()
            e0.record(s)
            tb.tt_matvec(A, X, Y)
            e1.record(s)
            tb.tt_copy(Y, Yr)
            e2.record(s)
            tb.tt_round(Yr, 1e-8, 128)
            e3.record(s)
            e3.synchronize()
            mv_ms.append(e0.elapsed_time(e1))
            rd_ms.append(e2.elapsed_time(e3))
    mv, rd = statistics.median(mv_ms), statistics.median(rd_ms)
    # B = 64 independent instances (seeds seed..seed+63) in one batched launch: the HBM roofline
    Bn = 64
    insts = [inputs.c2_instance(args.seed + b) for b in range(Bn)]
    As = [tb.TTMat.from_cores(i["A"], device=device) for i in insts]
    Xs = [tb.TTVec.from_cores(i["X"], device=device) for i in insts]
    Ys = [tb.TTVec(a.m, [p * q for p, q in zip(a.Rcap, x.rcap)], device) for a, x in zip(As, Xs)]
    bbytes = sum(8 * sum(R0 * 4 * R1 + r0 * 2 * r1 + R0 * R1 * 2 * r0 * r1 for R0, R1, r0, r1 in
                         zip(i["R"][:-1], i["R"][1:], i["r"][:-1], i["r"][1:])) for i in insts)
    from paper_2309_03347_b200.tt import MatvecBatch
    run_b = MatvecBatch(As, Xs, Ys)
    for _ in range(3):
        run_b()
    bms = []
    for _ in range(max(args.steps, 5)):
        flush.fill_(1.0)
        torch.cuda._sleep(2_000_000)   # the host enqueue (argument marshalling) overlaps a GPU sleep
        e0, e1 = _events()
        e0.record(s)
        run_b()                        # descriptor-table upload + the one kernel
        e1.record(s)
        e1.synchronize()
        bms.append(e0.elapsed_time(e1))
    bm = statistics.median(bms)
    gbs = bbytes / (bm * 1e-3) / 1e9
    # the same 64 products rounded together (tt_round_batched, eps 1e-8, rmax 128)
    from paper_2309_03347_b200.tt import RoundBatch
    Yw = [tb.TTVec(y.n, y.rcap, device) for y in Ys]
    rb = RoundBatch(Yw)
    rms = []
    for rep in range(3 + max(args.steps, 3)):
        for y, yw in zip(Ys, Yw):
            tb.tt_copy(y, yw)
        flush.fill_(1.0)
        e0, e1 = _events()
        e0.record(s)
        rb(1e-8, 128)
        e1.record(s)
        e1.synchronize()
        if rep >= 3:
            rms.append(e0.elapsed_time(e1))
    rbm = statistics.median(rms)
    return {"metric": METRIC, "value": 1e3 / (mv + rd), "unit": "instances/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mv + rd, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C2 (configs[1]) tt_matvec + tt_round(eps=1e-8, rmax=128), d=30, seed {args.seed}",
                       "l2": "256 MB flush between timed steps"},
            "matvec_ms": mv, "round_ms": rd, "ranks_after_round": Yr.ranks(),
            "round_b64_ms": rbm, "round_b64_instances_per_s": Bn / (rbm * 1e-3),
            "matvec_b1_gbs": mv_bytes / (mv * 1e-3) / 1e9,
            "matvec_b64_ms": bm,
            "roofline": {"kernel": "matvec_batched_kernel (tt_matvec_batched, 64 instances x 30 cores, one launch)",
                         "bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / pk["hbm_gbs"], "peak_src": pk["hbm_src"], "traffic": None,
                         "bytes_per_launch": bbytes,
                         "timing": "CUDA events around the descriptor upload + kernel; the host-side "
                                   "enqueue overlaps a preceding GPU sleep"},
            "clocks": clk.summary(),
            "gpu_launches": (count_kernels(lambda: (tb.tt_matvec(A, X, Y), tb.tt_copy(Y, Yr),
                                                    tb.tt_round(Yr, 1e-8, 128))) or (None,))[0],
            "gpu_launches_how": "libtt kernels of one more matvec + copy + round (CUPTI activity records)"}


KEFF_CFG = {
    "c3": dict(rmax=64, label="C3 (configs[2]): 64^3 QTT (6 bits/axis), G=7 downscatter, S8 LS-style (80), two regions"),
    "c4": dict(rmax=128, label="C4 (configs[3]): 256^3 QTT (8 bits/axis), G=30 (upscatter 26-30), S16 LS-style (288), "
                               "core/blanket/reflector"),
}
KEFF_OPTS = dict(tol_k=0.0, eps_round=1e-6, eps_solve=1e-6, matvec="amen_mv", max_sweeps=4, mv_max_sweeps=4,
                 restart=40, max_restarts=20)


def keff_bench(args, tb, device, world, dist, rank):
    """configs[3] (C4, the default) / configs[2] (C3): the k-eff fixed point
     with B = amen_mv((S + F/k), Psi) and AMEn solves of
    H Psi' = B, eps 1e-6, rmax 128 / 64.  A step is ONE fixed-point iteration
    (reading Z36: the B product, the AMEn solve run to its sweep limit, the
    <f, Psi'> / norm / k update), continuing the solve: `--settle` untimed
    iterations from psi_0 = 1, k_0 = 1 bring the ranks to rmax first (the
    steady state, the most expensive iterations), then W warm-up steps, then
    K timed steps; each step is one keff_fixed_point call with max_outer = 1
    and keff_opts.warm = 1 (psi, k, the amen_mv guess and the AMEn z0 carried
    over on the device, include/tt.h)."""
    import torch
    import inputs
    from paper_2309_03347_b200 import transport as gtr
    from paper_2309_03347_b200 import _lib
    import ctypes as C
    pk = peaks()
    cfg = KEFF_CFG[args.workload]
    t_setup = time.perf_counter()
    prob = inputs.problem_c4() if args.workload == "c4" else inputs.problem_c3()
    ops = gtr.operators(prob, eps=1e-12, device=device)
    modes = gtr.modes(prob)
    d = len(modes)
    rmax, kick = cfg["rmax"], 4
    g = inputs.rng(61)
    z0 = inputs.random_tt(g, modes, [1] + [kick] * (d - 1) + [1])
    cap = [1] + [rmax + kick] * (d - 1) + [1]
    psi = tb.TTVec.from_cores([np.ones((1, n, 1)) for n in modes], rcap=cap, device=device)
    z = tb.TTVec.from_cores(z0, device=device)
    opts = dict(KEFF_OPTS, rmax=rmax)
    torch.cuda.synchronize()
    t_asm = time.perf_counter() - t_setup
    nb = tb.keff_workspace_bytes(ops["H"], ops["S"], ops["F"], psi, z, rmax=rmax, matvec=opts["matvec"],
                                 restart=opts["restart"])
    ws = torch.empty(nb, dtype=torch.uint8, device=device)
    state = {"k": 1.0, "warm": False}

    def step(n=1):
        r = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, k0=state["k"], max_outer=n,
                                warm=state["warm"], ws=ws, **opts)
        state["warm"] = True
        return r

    settle = args.settle if args.settle is not None else 8
    r = step(settle)
    state["k"] = r.k.item()
    settle_hist = r.k_hist[:settle].cpu().tolist()
    for _ in range(args.warmup):
        r = step()
        state["k"] = r.k.item()
    torch.cuda.synchronize()
    ranks_before = psi.ranks()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=device)   # > 126 MB L2
    cnt = (C.c_uint64 * 5)()
    lib = _lib.lib()
    lib.tt_counters(cnt, 1)
    fl, fms, ffl = C.c_int64(0), C.c_double(0.0), (C.c_double * 3)()
    lib.tt_fused_profile_read(C.byref(fl), C.byref(fms), ffl)
    lib.tt_fused_profile(1)
    s = torch.cuda.current_stream()
    ms, ks, sweeps = [], [], []
    with ClockSampler(local_index(device)) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.fill_(1.0)                          # evict L2 between timed steps (untimed)
            e0, e1 = _events()
            torch.cuda.nvtx.range_push("timed")       # ncu --nvtx --nvtx-include timed/ (profiles/)
            e0.record(s)
            r = step()
            e1.record(s)
            torch.cuda.nvtx.range_pop()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
            state["k"] = r.k.item()
            ks.append(state["k"])
            sweeps.append(int(r.sweeps_hist[0].item()))
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        wall = time.perf_counter() - t0
    lib.tt_counters(cnt, 1)
    cms, cst, cl = (C.c_double * 64)(), (C.c_double * 64)(), (C.c_int64 * 64)()
    lib.tt_fused_profile_cores(cms, cst, cl)
    lib.tt_fused_profile_read(C.byref(fl), C.byref(fms), ffl)
    lib.tt_fused_profile(0)
    steps_per_core = [cst[t] / args.steps for t in range(d)]
    # cross-check of the in-kernel timer (the only per-launch clock inside the
    # device-resident graph) against CUDA events: one more (untimed) step on the
    # host-stepped path (graph mode 1), where events bracket every fused launch
    xc = None
    if lib.tt_graph_mode() == 2:
        lib.tt_set_graph_mode(1)
        tms, tl = C.c_double(0.0), C.c_int64(0)
        lib.tt_fused_timer_read(C.byref(tms), C.byref(tl))
        el, ems, eff = C.c_int64(0), C.c_double(0.0), (C.c_double * 3)()
        lib.tt_fused_profile(1)
        r = step()
        state["k"] = r.k.item()
        lib.tt_fused_profile_read(C.byref(el), C.byref(ems), eff)
        lib.tt_fused_profile(0)
        lib.tt_fused_timer_read(C.byref(tms), C.byref(tl))
        lib.tt_set_graph_mode(-1)
        xc = {"event_ms": ems.value, "event_launches": el.value, "timer_ms": tms.value, "timer_launches": tl.value,
              "timer_over_event": tms.value / ems.value if ems.value > 0 else None,
              "note": "one extra untimed step, host-stepped (graph mode 1): CUDA events around every fused launch "
                      "(both launched variants; the one not chosen exits at once) vs the in-kernel %globaltimer of "
                      "the launches that did work"}
    dev_ms = sum(ms)
    dev_max, iters_all = aggregate_ranks(dev_ms, args.steps, dist, device)
    gemm_flops, mv_flops, qr_flops, svd_flops, ngemm = [int(v) for v in cnt]
    gfl = (gemm_flops + mv_flops) / (dev_ms * 1e-3) / 1e9
    ff = ffl[0] + ffl[1]
    ach = ff / (fms.value * 1e-3) / 1e12 if fms.value > 0 else None
    dm = pk["dmma_gflops"] / 1e3
    roof = {"kernel": "gm_chunk_kernel (fused GMRES of the AMEn local systems: local-apply DMMA GEMM stages + "
                      "Gram-Schmidt + Givens, one persistent launch per local solve)",
            "bound": "tensor", "achieved": ach, "peak": dm, "unit": "TFLOP/s",
            "frac": (ach / dm) if ach else None, "peak_src": pk["dmma_src"],
            "traffic": ncu_traffic("gm_chunk_kernel", args.workload),
            "launches": fl.value, "ms_per_launch": fms.value / max(fl.value, 1),
            "flops_per_launch": ff / max(fl.value, 1), "arnoldi_steps_per_step": ffl[2] / args.steps,
            "share_of_step_time": fms.value / dev_ms if dev_ms > 0 else None,
            "how": "flops = the local-apply GEMM flops (diagonal operator cores counted at their structured cost) "
                   "+ Gram-Schmidt/normalisation vector flops, counted on the device; time = the kernel's in-kernel "
                   "%globaltimer (CTA 0, entry to exit) of every launch that did work inside the timed region: the "
                   "step is ONE graph launch with device-resident loops (conditional WHILE/IF nodes), where no "
                   "host-recorded CUDA event can bracket an individual launch; timer_vs_events cross-checks the "
                   "timer against CUDA events on the host-stepped path",
            "timer_vs_events": xc}
    res = {"metric": METRIC, "value": iters_all / (dev_max * 1e-3), "unit": "iter/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_max / args.steps,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": cfg["label"] + f", rmax {rmax}, eps 1e-6, B by amen_mv, AMEn <= 4 sweeps, "
                                  f"GMRES(40); step = one k-eff fixed-point iteration continuing the solve after "
                                  f"{settle} settle + {args.warmup} warm-up iterations from psi_0 = 1, k_0 = 1",
                      "l2": "256 MB flush between timed steps", "parallelism": f"replicas x{world}"},
           "k_after_settle": settle_hist[-1] if settle_hist else None, "k_last": ks[-1], "k_steps": ks,
           "sweeps_per_step": sweeps, "psi_ranks": psi.ranks(), "psi_ranks_before_timing": ranks_before,
           "operator_ranks": {k: v.ranks() for k, v in ops.items()},
           "contraction_gflops": gfl, "contraction_pct_dmma_peak": 100.0 * gfl / pk["dmma_gflops"],
           "flops_per_step": {"gemm": gemm_flops / args.steps, "qr": qr_flops / args.steps,
                              "jacobi": svd_flops / args.steps, "gemm_calls": ngemm / args.steps},
           "arnoldi_steps_per_core_per_step": steps_per_core,
           "roofline": roof, "clocks": clk.summary(), "wall_s": wall, "setup_s": t_asm,
           "graph_mode": {"mode": int(lib.tt_graph_mode()),
                          "meaning": "2 = each step is ONE CUDA-graph launch of keff_fixed_point: the outer "
                                     "fixed-point loop and every amen_mv / AMEn sweep loop are conditional "
                                     "WHILE/IF nodes decided on the device (SURVEY K11), no host round trip "
                                     "inside the step"}}
    kc = count_kernels_k11(step)
    res["gpu_launches"] = kc[0] if kc else None
    res["gpu_launches_how"] = kc[2] if kc else "CUPTI unavailable"
    if kc:
        res["gpu_launches_all_kernels"] = kc[1]
        res["gpu_launches_cupti_mode2"] = kc[3]
    res["e2e"] = e2e_keff(tb, ops, psi, z, state, opts, ws, args.steps)
    if args.workload == "c3":
        gold = os.path.join(ROOT, "tests", "golden", "c3_keff.txt")
        for line in open(gold):
            if line.strip() and not line.startswith("#") and line.split()[0] == "64":
                res["k_truth_matrix_free"] = float(line.split()[1])
                res["k_rel_discrepancy"] = abs(ks[-1] - res["k_truth_matrix_free"]) / res["k_truth_matrix_free"]
    return res


def e2e_keff(tb, ops, psi, z, state, opts, ws, steps):
    """The same metric through the public API with HOST buffers: every step copies
    the operator cores (H, S, F) and the current psi from pinned host memory,
    runs one fixed-point iteration (keff_fixed_point, max_outer = 1, a fresh
    call: psi re-rounded, the amen_mv guess restarted from psi) and reads psi
    and k back into pinned host memory."""
    import torch
    host = {k: v.data.cpu().pin_memory() for k, v in ops.items()}
    hpsi = psi.data.cpu().pin_memory()
    hr = psi.r_dev.cpu().pin_memory()
    hz, hzr = z.data.cpu().pin_memory(), z.r_dev.cpu().pin_memory()
    out_psi = torch.empty_like(hpsi).pin_memory()
    out_k = torch.empty(1, dtype=torch.float64).pin_memory()
    s = torch.cuda.current_stream()
    e0, e1 = _events()
    torch.cuda.synchronize()
    e0.record(s)
    k = state["k"]
    for _ in range(steps):
        for key, v in ops.items():
            v.data.copy_(host[key], non_blocking=True)
        psi.data.copy_(hpsi, non_blocking=True)
        psi.r_dev.copy_(hr, non_blocking=True)
        z.data.copy_(hz, non_blocking=True)
        z.r_dev.copy_(hzr, non_blocking=True)
        r = tb.keff_fixed_point(ops["H"], ops["S"], ops["F"], psi, z, k0=k, max_outer=1, warm=False, ws=ws, **opts)
        out_psi.copy_(psi.data, non_blocking=True)
        out_k.copy_(r.k, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        k = float(out_k[0])
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    h2d = sum(int(v.numel()) * 8 for v in host.values()) + int(hpsi.numel() + hz.numel()) * 8 + \
        int(hr.numel() + hzr.numel()) * 4
    return {"value": steps / (ms * 1e-3), "unit": "iter/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": int(out_psi.numel()) * 8 + 8,
            "how": "per step: H, S, F cores + psi + z host->device (pinned), one keff_fixed_point iteration (fresh "
                   "call), psi + k device->host"}


def extras(args, tb, device, world):
    """The metric's first half on its own configs, in the same run: C5 (configs[4])
    ALS double sweep at r = 256, 128, 64 (GFLOP/s, % of the FP64 DMMA peak) and the C2
    (configs[1]) 64-instance batched tt_matvec (GB/s, % of the measured HBM
    copy bandwidth)."""
    import copy
    out = {}
    a = copy.copy(args)
    a.workload, a.no_graph, a.one_stream = "c5", False, False
    a.steps, a.warmup = max(5, min(args.steps, 10)), 3
    for r in (256, 128, 64):   # configs[4] names all three interface ranks
        a.rank = r
        l5 = micro_bench(a, tb, device, world, None)
        out[f"c5_r{r}"] = {"value": l5["value"], "unit": l5["unit"], "pct_dmma_peak": l5["pct_dmma_peak"],
                           "ms_per_sweep": l5["ms_per_step"], "flops_per_sweep": l5["flops_per_step"],
                           "config": l5["config"]["workload"], "gpu_launches": l5["gpu_launches"]}
    a.workload, a.steps = "c2", max(5, min(args.steps, 10))
    l2 = micro_bench(a, tb, device, world, None)
    rf = l2["roofline"]
    out["c2_b64"] = {"value": rf["achieved"], "unit": "GB/s", "pct_hbm_measured": 100.0 * rf["frac"],
                     "pct_8tbs_nominal": 100.0 * rf["achieved"] / 8000.0, "ms_per_launch": l2["matvec_b64_ms"],
                     "bytes_per_launch": rf["bytes_per_launch"], "peak_src": rf["peak_src"],
                     "config": "C2 (configs[1]) 64 independent d=30 instances (seeds 0-63), one tt_matvec_batched "
                               "launch", "b1_matvec_plus_round_instances_per_s": l2["value"],
                     "b1_round_ms": l2["round_ms"], "round_b64_ms": l2["round_b64_ms"],
                     "round_b64_instances_per_s": l2["round_b64_instances_per_s"]}
    return out


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        import threadpoolctl
        info["blas"] = [{"api": i.get("internal_api"), "lib": os.path.basename(i.get("filepath", "")),
                         "threads": i.get("num_threads")} for i in threadpoolctl.threadpool_info()]
    except Exception:
        pass
    return info


def c4_shapes(ranks=None):
    """The C4 steady-state local-system shapes: psi ranks at rmax 128 (+ kickrank 4)
    bounded by the mode products from each end, operator ranks of H (PROBE,
    bench runs: H [1,4,6,...,84,36,4,1])."""
    import inputs
    modes = [2] * 24 + [288, 30]
    d = len(modes)
    if ranks is None:
        ranks = [1] + [int(min(132.0, np.prod(modes[:k], dtype=float), np.prod(modes[k:], dtype=float)))
                       for k in range(1, d)] + [1]
    RH = [1, 4, 6, 6, 6, 6, 8, 11, 7, 25, 34, 34, 34, 34, 36, 38, 16, 56, 76, 76, 76, 76, 80, 84, 36, 4, 1]
    return modes, ranks, RH


# Arnoldi steps per core per C4 fixed-point iteration in the steady state (GPU
# run, tools/probe_c4.py 8 3, round 2); used when no live GPU counts exist (the
# reference arm)
C4_STEPS_PER_CORE = [6.7, 15.0, 25.0, 40.7, 81.0, 156.0, 350.0, 553.0, 1338.0, 345.3, 303.3, 307.3, 313.3, 324.7,
                     362.3, 308.0, 309.7, 328.3, 314.7, 316.0, 317.7, 309.0, 280.3, 204.0, 105.0, 0.0]


def oracle_apply_sample(steps_per_core=None, ranks=None, budget_s=10.0):
    """Bounded sample of the C4 workload on the CPU oracle: one oracle a6 local
    apply (oracle.tt.local_apply, the operation behind every Arnoldi step of
    the AMEn local solves, ~98% of an iteration's flops) at each of the 26
    C4 core shapes of the steady state (psi ranks <= 132, H's ranks), seeded
    Gaussian operands.  The oracle's time per fixed-point iteration is
    estimated as sum_k (Arnoldi steps at core k per iteration) x t_apply(k),
    with the per-core step counts of the GPU's timed iterations (or 300 per
    core if not given): QR, SVD, Gram-Schmidt and amen_mv are left out, so
    this OVERSTATES the oracle's iterations/s."""
    import inputs
    from oracle import tt as ott
    modes, r, RH = c4_shapes(ranks)
    d = len(modes)
    g = inputs.rng(77)
    ops = []
    for k in range(d):
        n = modes[k]
        ops.append((g.standard_normal((r[k], RH[k], r[k])), g.standard_normal((RH[k], n, n, RH[k + 1])),
                    g.standard_normal((r[k + 1], RH[k + 1], r[k + 1])), g.standard_normal((r[k], n, r[k + 1]))))
    times = [[] for _ in range(d)]
    t0 = time.perf_counter()
    while True:    # whole passes over the 26 shapes until the CPU budget is spent (median per shape)
        for k in range(d):
            t = time.perf_counter()
            ott.local_apply(*ops[k])
            times[k].append(time.perf_counter() - t)
        if time.perf_counter() - t0 >= budget_s:
            break
    sample_s = time.perf_counter() - t0
    t_core = [statistics.median(v) for v in times]
    spc = steps_per_core if steps_per_core else C4_STEPS_PER_CORE
    t_iter = sum(a * b for a, b in zip(spc, t_core))
    return 1.0 / t_iter, t_iter, sample_s, t_core


def cpu_baseline(workload, steps_per_core=None, ranks=None):
    if workload != "c4":
        return None
    hi = host_info()
    v, t_iter, sample_s, t_core = oracle_apply_sample(steps_per_core, ranks)
    out = {"value": v, "unit": "iter/s", "cores": cpu_cores(), "kind": "oracle",
           "sample": (f"oracle a6 local applies (oracle.tt.local_apply) at each of the 26 C4 steady-state core "
                      f"shapes, repeated passes for {sample_s:.1f} s of CPU work (median per shape), scaled to one fixed-point iteration by the Arnoldi "
                      f"steps per core of the GPU's timed iterations ({t_iter:.1f} s per iteration); QR, SVD, "
                      f"Gram-Schmidt and amen_mv left out, so this overstates the oracle's rate"),
           "host": hi, "t_apply_per_core_s": t_core}
    try:   # the same sample on one thread
        import threadpoolctl
        with threadpoolctl.threadpool_limits(1):
            v1, t1, s1, _ = oracle_apply_sample(steps_per_core, ranks, budget_s=5.0)
        out["value_1thread"] = v1
        out["sample_1thread_s"] = s1
    except Exception as e:
        out["value_1thread"] = None
        out["note_1thread"] = repr(e)[:200]
    return out


def local_index(device):
    return device.index if getattr(device, "index", None) is not None else 0


def ncu_traffic(kernel, workload):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel` from
    the committed ncu --set full capture (profiles/r02/ncu_traffic.json), with
    that launch's algorithmic flops for comparison; None if not captured."""
    path = os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")
    try:
        return json.load(open(path))[workload][kernel]
    except Exception:
        return None


def count_launches_estimate(gemm_calls, iters):
    """GEMM calls are counted on the device; the non-GEMM launches are roughly one
    per GEMM chain (plan, QR, SVD, GMRES vector kernels).  Reported as counted
    GEMM calls + estimate; the ncu launch list in profiles/ is the evidence."""
    return int(gemm_calls * 2)


def dominant_gemm_roofline(tb, device, pk, shape=(64, 8, 64, 8, 8, 64, 8, 64),
                           label="C1 local shape r=64 R=8 n=8"):
    import torch
    rA, R, rB, m, n, rAp, Rp, rBp = shape
    g = torch.Generator(device="cpu").manual_seed(5)
    mk = lambda *s: torch.randn(*s, generator=g, dtype=torch.float64).reshape(-1).to(device)
    Phi, Ak, Psi, x = mk(rA * R * rB), mk(R * m * n * Rp), mk(rAp * Rp * rBp), mk(rB * n * rBp)
    y = torch.zeros(rA * m * rAp, dtype=torch.float64, device=device)
    dims = (rA, R, rB, m, n, rAp, Rp, rBp)
    for _ in range(5):
        tb.als_local_apply(dims, Phi, Ak, Psi, x, y)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 50
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        tb.als_local_apply(dims, Phi, Ak, Psi, x, y)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = 2.0 * (n * rB * rBp * rAp * Rp + m * n * rB * rAp * R * Rp + m * rA * rAp * rB * R)
    achieved = flops / (ms * 1e-3) / 1e12
    peak = pk["dmma_gflops"] / 1e3
    return {"kernel": f"gemm_dmma_kernel (als_local_apply chain, {label})",
            "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "peak_src": "measured FP64 DMMA sustained (tools/peaks_fp64)", "traffic": None,
            "flops_per_launch": flops, "ms_per_launch": ms}


def e2e_c1(tb, st, device, steps):
    """Same metric through the public API with HOST buffers: operator cores and
    psi_0 / z_0 copied from pinned host memory every step, k and psi read back."""
    import torch
    ops = st["ops"]
    host = {k: v.data.cpu().pin_memory() for k, v in ops.items()}
    hpsi = st["psi_init"].data.cpu().pin_memory()
    hz = st["z_init"].data.cpu().pin_memory()
    out_psi = torch.empty_like(hpsi).pin_memory()
    out_k = torch.empty(1, dtype=torch.float64).pin_memory()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        for k, v in ops.items():
            v.data.copy_(host[k], non_blocking=True)
        st["psi_init"].data.copy_(hpsi, non_blocking=True)
        st["z_init"].data.copy_(hz, non_blocking=True)
        res = c1_step_device(st)
        out_psi.copy_(st["psi"].data, non_blocking=True)
        out_k.copy_(res.k, non_blocking=True)
        iters += int(res.iters.item())
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    h2d = sum(int(v.numel()) * 8 for v in host.values()) + int(hpsi.numel() + hz.numel()) * 8
    return {"value": iters / (ms * 1e-3), "unit": "iter/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": int(out_psi.numel()) * 8 + 8}


if __name__ == "__main__":
    main()
