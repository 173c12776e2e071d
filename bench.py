"""Benchmark: DD/TD/QD LU + solve on B200 (BASELINE.json metric: effective
(2/3)n^3 flop/s and the fraction of the FP64 roofline).

Default workload = BASELINE config 2, TD LU with partial pivoting +
forward/back substitution at n = 2048 (seeded synthetic system; x_true from
the same recipe, b = A*x_true in TD on the device).  A step = restore A
(device-to-device copy of the pristine matrix, which also evicts L2:
2 x 100 MB > 126 MB L2) + LU + solve.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--k 3] [--dim 2048]
    python bench.py --impl reference ...   (CPU oracle port, all host threads)

    python bench.py --config {1,3,4}       (GEMM, TD-mpmath IR, distributed)

Multi-GPU (torchrun, one rank per GPU): without --config, BASELINE config 4
-- ONE DD n = 32768 system, column-block-cyclic over the ranks through the
native distributed driver (strong scaling; under torchrun at N = 1, or with
`--config 4`, the same code with a one-rank world is the curve's first
point).  Configs 1-3
are single-GPU workloads ("replicas only" under torchrun).  Barrier + max
over ranks of the device time.
"""

import argparse
import ctypes
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

NAMES = {2: "DD", 3: "TD", 4: "QD"}
# FP64 instructions the device executes per op: the reference op counts
# (madd 29/264/376) minus the residuals of the final cascade
# sweep, which the reference computes and discards (dead code on the GPU).
MADD_INSTR = {2: 29, 3: 214, 4: 326}
REF_MADD_INSTR = {2: 29, 3: 264, 4: 376}
MUL_INSTR = {2: 9, 3: 133, 4: 181}
DIV_INSTR = {2: 113, 3: 491, 4: 1165}
# DFMA per op (one per two_prod; each DFMA is 2 flops): flop-weighted rates
MADD_DFMA = {2: 1, 3: 6, 4: 6}
MUL_DFMA = {2: 1, 3: 6, 4: 6}
SEED = 210712550 + 2                      # config index 2


def work_counts(n, k):
    """FP64 instruction counts of LU + solve."""
    lu_madds = (n - 1) * n * (2 * n - 1) // 6
    lu_muls = n * (n - 1) // 2
    lu_divs = n - 1
    sv_madds = n * (n - 1)
    sv_divs = n
    instr = ((lu_madds + sv_madds) * MADD_INSTR[k] + lu_muls * MUL_INSTR[k]
             + (lu_divs + sv_divs) * DIV_INSTR[k])
    flops = instr + (lu_madds + sv_madds) * MADD_DFMA[k] + lu_muls * MUL_DFMA[k]
    return dict(lu_madds=lu_madds, sv_madds=sv_madds, instr=instr,
                flops=flops)


def update_madds(n, nb):
    """madds of the wide trailing-update launches over one LU (profile slot
    "update"; the look-ahead's next-panel columns are slot "update_next")."""
    t = 0
    for J in range(0, n, nb):
        w = min(nb, n - J)
        rest = n - J - w
        w2 = min(nb, rest)
        t += rest * (rest - w2) * w
    return t


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        # one nvidia-smi in loop mode (50 ms) for the whole timed region
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the first sample land before timing
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.1)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=10)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.splitlines():
            if line.strip():
                self.samples.append([s.strip() for s in line.split(",")])

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace('.', '').isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace('.', '').isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for i, nm in enumerate(names):
                if len(s) > 4 + i and s[4 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


class stdout_to_stderr:
    """Route file descriptor 1 to 2 for a block (native libraries' prints)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        pg = dist
    return world, rank, local, pg


def barrier(pg):
    if pg is not None:
        pg.barrier()


def max_over_ranks(pg, v):
    if pg is None:
        return v
    import torch
    t = torch.tensor([float(v)], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline(k, n_sample, threads=None, seed=SEED):
    """Oracle port (C++/AVX2/OpenMP restatement of the reference lane
    path) on a bounded sample: LU + solve of the same recipe at n_sample."""
    import oracle
    from oracle import gen
    # every host thread this process may run on (torchrun sets
    # OMP_NUM_THREADS=1 per rank; the baseline runs on rank 0 alone)
    if not threads:
        try:
            threads = len(os.sched_getaffinity(0))
        except AttributeError:
            threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    cores = oracle.num_threads()
    A = gen.planes(k, (n_sample, n_sample), 0, n_sample, seed)
    x = gen.planes(k, (n_sample,), 2, n_sample, seed)
    b = oracle.matvec(A, x)
    t0 = time.perf_counter()
    lu, sw = oracle.lu(A)
    oracle.solve(lu, sw, b)
    dt = time.perf_counter() - t0
    gf = (2.0 / 3.0) * n_sample ** 3 / dt / 1e9
    return dict(value=gf, unit="GFLOP/s", cores=cores, kind="port",
                seconds=dt,
                sample="%s LU+solve n=%d (same seeded recipe; %.2f s); "
                       "C++ restatement of the reference lane path, "
                       "AVX2 + OpenMP over rows" % (NAMES[k], n_sample, dt))


def config_dict(args, world):
    """The workload's config object -- the same dict on both arms."""
    k, n = args.k, args.n
    if args.config == 1:
        return {"workload": "config1: %s GEMM n=%d" % (NAMES[k], n),
                "n": n, "k": k, "parallelism": "replicas x%d" % world,
                "l2": "A, B, C = 3 x %d MB (> L2)" % (k * n * n * 8 >> 20)}
    if args.config == 3:
        return {"workload": "config3: TD-mpmath IR n=%d kappa=1e30" % n,
                "n": n, "long_bits": 512, "rtol": "1e-100", "atol": "0",
                "maxtimes": 20, "parallelism": "replicas x%d" % world}
    if args.config == 4:
        return {"workload": "config4: distributed %s LU+PP+solve n=%d"
                % (NAMES[k], n), "n": n, "k": k, "nb": args.dist_nb,
                "parallelism": "column-block-cyclic x%d (one process per "
                "GPU), NCCL panel + pivot broadcast, column-cyclic back "
                "substitution" % world,
                "l2": "A restored from a pristine copy each step (>> L2)"}
    return {"workload": "config2: %s LU+PP+solve n=%d" % (NAMES[k], n),
            "n": n, "k": k, "nb": args.nb or 32,
            "l2": "A restored by a 2x%d MB D2D copy each step (> L2)"
                  % (k * n * n * 8 // 2 ** 20),
            "parallelism": "replicas x%d" % world}


def run_reference(args):
    """The reference arm: the reference's CPU path for the same workload,
    timed on this box's host cores -- the oracle port (C++ restatement of
    the reference lane path, AVX2 + OpenMP over rows; the pure-Python
    reference does not exist on the GPU box and takes ~25 min per config-2
    solve).  Each step is a bounded sample of the workload: the full
    config-2 LU + solve; for config 1 an n = 1024 GEMM; for config 3 the
    short side (TD LU + the solves) of the refinement; for config 4 a DD
    n = 4096 LU + solve whose rate stands for n = 32768 (time x 512).
    Rank 0 only under torchrun."""
    world, rank, local, pg = dist_setup(args)
    if rank != 0:
        return
    import oracle
    from oracle import gen
    k, n = args.k, args.n
    try:
        threads = len(os.sched_getaffinity(0))
    except AttributeError:
        threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    res = []
    for i in range(args.warmup + args.steps):
        if args.config == 1:
            ns = args.cpu_n or 1024
            A = gen.planes(k, (ns, ns), 0, ns, 210712551)
            B = gen.planes(k, (ns, ns), 1, ns, 210712551)
            t0 = time.perf_counter()
            oracle.gemm(A, B)
            dt = time.perf_counter() - t0
            r = dict(value=2.0 * ns ** 3 / dt / 1e9, seconds=dt,
                     sample="%s GEMM n=%d of the config-1 recipe" %
                            (NAMES[k], ns))
        elif args.config == 3:
            from paper_2107_12550_b200.refine import CONFIG3_SEED  # noqa
            A = gen.planes(3, (n, n), 0, n, CONFIG3_SEED)
            b = gen.planes(3, (n,), 2, n, CONFIG3_SEED)
            t0 = time.perf_counter()
            lu, sw = oracle.lu(A)
            for _ in range(4):       # the first solve + 3 corrections
                oracle.solve(lu, sw, b)
            dt = time.perf_counter() - t0
            r = dict(value=dt, seconds=dt,
                     sample="short side of the config-3 refinement only "
                            "(TD LU n=%d + 4 solves; the reference's "
                            "512-bit residual loop is pure Python and not "
                            "ported): a lower bound of its CPU time" % n)
        else:
            ns = args.cpu_n or (4096 if args.config == 4 else n)
            seed = 210712550 + (4 if args.config == 4 else 2)
            r = cpu_baseline(k, ns, threads, seed=seed)
            if args.config == 4:
                r["sample"] += ("; rate at n=%d stands for n=%d "
                                "(time x (n/%d)^3)" % (ns, n, ns))
        if i >= args.warmup:
            res.append(r)
    v = statistics.median([r["value"] for r in res])
    sec = statistics.median([r["seconds"] for r in res])
    if args.config == 3:
        metric, unit, hib = "TD-mpmath IR time-to-rtol (s)", "s", False
        ms = sec * 1e3
    elif args.config == 1:
        metric, unit, hib = "%s GEMM eff. GFLOP/s (2n^3/s)" % NAMES[k], \
            "GFLOP/s", True
        ms = sec * 1e3
    else:
        metric, unit, hib = ("%s LU+solve eff. GFLOP/s ((2/3)n^3/s)"
                             % NAMES[k]), "GFLOP/s", True
        ms = (2.0 / 3.0) * n ** 3 / (v * 1e9) * 1e3
    line = {
        "impl": "reference", "metric": metric, "value": v, "unit": unit,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": hib,
        "scaling": "strong" if args.config == 4 else "weak",
        "vs_baseline": None, "dtype": "f64x%d" % k,
        "data": "synthetic (the same seeded recipe)",
        "config": config_dict(args, world),
        "cpu_baseline": {"value": v, "unit": unit, "cores": threads,
                         "kind": "port", "seconds": sec,
                         "sample": res[-1]["sample"] + " (median of %d)"
                         % len(res)},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_ours(args):
    world, rank, local, pg = dist_setup(args)
    os.environ.setdefault("MPCORE_DEVICE", str(local))
    from paper_2107_12550_b200 import _native as nat
    from paper_2107_12550_b200.linalg import (DeviceMatrix, DeviceVector,
                                              device_solve_system)
    L = nat.lib()
    k, n, nb = args.k, args.n, args.nb
    seed = SEED
    # inputs resident in HBM: pristine A, work copy, x_true, b = A x_true
    A0 = DeviceMatrix(k, n, n)
    A0.generate(0, n, seed)
    xt = DeviceVector(k, n)
    xt.generate(2, n, seed)
    b = DeviceVector(k, n)
    nat.check(L.mpcore_mat_vec(A0.handle, xt.handle, b.handle), "mat_vec")
    # one step: restore [A | b] (augmented n x (n+1) work matrix) from the
    # pristine copies, then the one-call solve -- LU with b riding along as
    # an extra column (its forward substitution), back substitution after
    W = DeviceMatrix(k, n, n + 1)
    x = DeviceVector(k, n)
    a0p, bp, wp, xp = (A0.device_ptr(), b.device_ptr(), W.device_ptr(),
                       x.device_ptr())
    sw = np.zeros(n, dtype=np.int32)
    sstep = ctypes.c_int32()

    def step():
        nat.check(L.mpcore_dev_copy2d(k, n, n, wp, n + 1, n * (n + 1), a0p, n,
                                      n * n), "restore A")
        nat.check(L.mpcore_dev_copy2d(k, n, 1, wp + n * 8, n + 1, n * (n + 1),
                                      bp, 1, n), "restore b")
        nat.check(L.mpcore_dev_solve_system(
            k, n, wp, n + 1, n * (n + 1), nb, xp,
            sw.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            ctypes.byref(sstep)), "solve_system")

    for _ in range(args.warmup):
        step()
    nat.sync()
    peak_add, peak_fma = nat.fp64_peak() if rank == 0 else (0.0, 0.0)
    barrier(pg)
    nat.sync()
    # timed region: CUDA events on the library stream (all of a step's
    # kernels and copies run there), synchronised on both sides
    timer = nat.StreamTimer()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        timer.start()
        for _ in range(args.steps):
            step()
        dev_total = timer.stop()
        nat.sync()
        wall = time.perf_counter() - t0
    wall_ms = wall * 1e3 / args.steps
    ms = max_over_ranks(pg, dev_total / args.steps)
    barrier(pg)
    # kernel breakdown: the same K steps again with CUDA events around every
    # kernel family on the library stream (direct launches instead of the
    # captured LU graph, so the events can bracket each launch)
    nat.prof_reset()
    nat.prof_enable(True)
    for _ in range(args.steps):
        step()
    nat.sync()
    nat.prof_enable(False)
    prof = nat.prof_read()
    dev_ms = sum(v[0] for v in prof.values()) / args.steps
    barrier(pg)

    # end-to-end through the C ABI with host buffers (pinned), per step:
    # H2D A + b, LU, solve, D2H x
    hA = nat.PinnedBuffer((k, n, n))
    A0.download(hA.array)
    hb = nat.PinnedBuffer((k, n))
    b.download(hb.array)
    hx = nat.PinnedBuffer((k, n))
    # double-buffered: while step i solves on one [A, b] pair, step i+1's
    # inputs upload into the other (mpcore_set_planes_async; its own copy
    # stream), so every step still moves its A and b across the link and
    # reads x back, inside the timed region
    Es = [DeviceMatrix(k, n, n), DeviceMatrix(k, n, n)]
    ebs = [DeviceVector(k, n), DeviceVector(k, n)]
    ex = DeviceVector(k, n)

    def upload(slot):
        nat.set_planes_async(Es[slot].handle, hA.array)
        nat.set_planes_async(ebs[slot].handle, hb.array)

    # warm-up pass, then K timed steps: the first timed step's upload is
    # inside the timed region too, the last step queues none, so the
    # region holds exactly K uploads, K solves and K downloads
    upload(0)
    device_solve_system(Es[0], ebs[0], ex, nb)
    ex.download(hx.array)
    barrier(pg)
    nat.sync()
    e_steps = args.steps
    timer.start()
    upload(1)
    for i in range(1, e_steps + 1):
        if i < e_steps:
            upload((i + 1) % 2)                   # the next step's inputs
        device_solve_system(Es[i % 2], ebs[i % 2], ex, nb)
        ex.download(hx.array)                     # synchronous D2H of x
    nat.sync()
    e2e_ms = max_over_ranks(pg, timer.stop() / e_steps)
    assert hx.array.tobytes() == x.download().tobytes()

    # the drop-in Python API on host containers (planes page-locked by the
    # container constructors): lu_factor_pp uploads A, factors, downloads
    # the factors; lu_solve uploads factors + b, solves, downloads x.  Host
    # timed (the calls are synchronous); restoring A between steps is not.
    from paper_2107_12550_b200.linalg import (DenseMatrix, McDomain, Vector,
                                              lu_factor_pp, lu_solve)
    dom = McDomain({2: "dd", 3: "td", 4: "qd"}[k])
    Ah = DenseMatrix.zeros(dom, n, n)
    A0.download(Ah.data)
    Aw = Ah.copy()
    bv = Vector.zeros(dom, n)
    b.download(bv.data)
    api_t = []
    for i in range(args.warmup + args.steps):
        Aw.data[...] = Ah.data
        t0 = time.perf_counter()
        piv = lu_factor_pp(Aw)
        xs_api = lu_solve(Aw, piv, bv)
        if i >= args.warmup:
            api_t.append(time.perf_counter() - t0)
    assert xs_api.data.tobytes() == x.download().tobytes()
    api_ms = max_over_ranks(pg, statistics.median(api_t) * 1e3)
    bwd = None
    if rank == 0 and k < 4:
        import torch
        dev = torch.device("cuda", local)
        bwd = qd_backward_error(
            k, n, torch.from_numpy(A0.download()).to(dev),
            torch.from_numpy(b.download()).to(dev),
            torch.from_numpy(x.download()).to(dev))
    if rank != 0:
        return
    flops = (2.0 / 3.0) * n ** 3
    value = world * flops / (ms * 1e-3) / 1e9
    wc = work_counts(n, k)
    # dominant kernel: trailing update; algorithmic FP64 instructions
    upd_ms, upd_launches = prof["update"]
    upd_ms /= args.steps
    upd_instr = update_madds(n, nb or 32) * MADD_INSTR[k]
    upd_rate = upd_instr / (upd_ms * 1e-3) if upd_ms > 0 else 0.0
    peak = peak_add
    overall_rate = wc["instr"] / (ms * 1e-3)
    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_baseline(k, args.cpu_n or n)
    clocks = clk.summary()
    line = {
        "metric": "%s LU+solve eff. GFLOP/s ((2/3)n^3/s)" % NAMES[k],
        "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "timing": "CUDA events on the library stream around the K steps; "
                  "host wall clock %.3f ms/step" % wall_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64x%d (%s, bit-exact EFT arithmetic)" % (k, NAMES[k]),
        "data": "synthetic (seeded splitmix64 recipe, SURVEY 8d; seed %d)"
                % seed,
        "config": config_dict(args, world),
        "e2e": {"value": world * flops / (e2e_ms * 1e-3) / 1e9,
                "unit": "GFLOP/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": (k * n * n + k * n) * 8,
                "d2h_bytes_per_step": k * n * 8,
                "path": "C ABI, pinned host buffers, double-buffered: "
                        "set_planes_async(A, b) of the next step (own copy "
                        "stream, overlapping this step's solve) + "
                        "solve_system (LU with b as an extra column + back "
                        "substitution; = lu_factor + lu_solve bit for bit) + "
                        "get_planes(x); K uploads, K solves, K downloads "
                        "between the events"},
        "check": bwd,
        "api_e2e": {"value": world * flops / (api_ms * 1e-3) / 1e9,
                    "unit": "GFLOP/s", "ms_per_step": api_ms,
                    "h2d_bytes_per_step": (2 * k * n * n + k * n) * 8,
                    "d2h_bytes_per_step": (k * n * n + k * n) * 8,
                    "path": "drop-in Python API: lu_factor_pp(DenseMatrix) "
                            "+ lu_solve(.., PivotRecord, Vector) on host "
                            "containers (page-locked planes); median of K, "
                            "host clock"},
        "roofline": {
            "bound": "fp64",
            "kernel": "trailing update, wide launches (gemm_kernel NEG_A; "
                      "main stream)",
            "achieved": upd_rate / 1e12, "peak": peak / 1e12,
            "unit": "T FP64 instr/s", "frac": upd_rate / peak if peak else None,
            "peak_source": "measured DADD issue rate (mpcore_fp64_peak) on "
                           "this GPU; nominal 148*64*1.965e9 = 18.6e12",
            "per_launch_avg_ms": upd_ms * args.steps / max(1, upd_launches),
            "update_share_of_step": upd_ms / ms if ms else None,
            "traffic": traffic_bytes(k, n),
            "traffic_note": "DRAM bytes of one captured update launch "
                            "(profiles/r02_traffic.json; its algorithmic "
                            "bytes are listed there)",
            "whole_step_frac": overall_rate / peak if peak else None,
            # flop-weighted (DFMA = 2 flops) against the DFMA issue peak
            # (the datasheet's FP64 TFLOP/s figure is 2 x the DFMA rate)
            "fp64_tflops": wc["flops"] / (ms * 1e-3) / 1e12,
            "fp64_tflops_peak": 2 * peak_fma / 1e12,
            "flop_frac": (wc["flops"] / (ms * 1e-3)) / (2 * peak_fma)
                         if peak_fma else None,
            # the latency-bound kernels against HBM
            "solve_hbm_gbs": (k * 8 * n * n / 2 + 4 * k * 8 * n)
                             / (prof["solve"][0] / args.steps * 1e-3) / 1e9
                             if prof["solve"][1] else None,
            "panel_hbm_gbs": (2 * k * 8 * n * (n + 32) / 2)
                             / (prof["panel"][0] / args.steps * 1e-3) / 1e9
                             if prof["panel"][1] else None,
            "hbm_peak_gbs": 6553.3,
        },
        "kernels_ms_per_step": {s: v[0] / args.steps for s, v in prof.items()
                                if v[1]},
        "device_ms_per_step": dev_ms,
        "gpu_launches": int(sum(v[1] for v in prof.values())),
        "clocks": clocks,
        "fp64_peak": {"dadd_per_s": peak_add, "dfma_per_s": peak_fma},
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line))


def traffic_bytes(k, n):
    """dram__bytes_read + dram__bytes_write of the captured trailing-update
    launch (ncu --set full), when the capture matches this workload."""
    try:
        d = json.load(open(os.path.join(os.path.dirname(os.path.abspath(
            __file__)), "profiles", "r02_traffic.json")))
    except (OSError, ValueError):
        return None
    return d["dram_bytes"] if (d.get("k"), d.get("n")) == (k, n) else None


U_P = {2: 2.0 ** -104, 3: 2.0 ** -156, 4: 2.0 ** -208}


def qd_backward_error(k, n, A, b, x):
    """Normwise backward error ||b - A x||_inf / (||A||_inf ||x||_inf) with
    the residual formed in QD on the GPU (k-component inputs lift to QD
    exactly; mat_vec and the subtraction are the library's kernels).  A: a
    CUDA tensor (k, n, ld >= n), b and x: (k, n).  The north star's bound
    is n * u_p (DD 2^-104, TD 2^-156)."""
    import torch
    from paper_2107_12550_b200 import _native as nat
    from paper_2107_12550_b200.linalg import DeviceVector
    ld = A.shape[2]
    Aq = torch.zeros((4, n, ld), dtype=torch.float64, device=A.device)
    Aq[:k] = A
    xq = torch.zeros((4, n), dtype=torch.float64, device=A.device)
    xq[:k] = x
    y = torch.zeros_like(xq)
    torch.cuda.synchronize()
    nat.check(nat.lib().mpcore_dev_matvec(4, n, n, Aq.data_ptr(), ld, n * ld,
                                          xq.data_ptr(), y.data_ptr()),
              "QD mat_vec")
    bq = torch.zeros_like(xq)
    bq[:k] = b
    B = DeviceVector.from_planes(bq.cpu().numpy())
    Y = DeviceVector.from_planes((-y).cpu().numpy())
    R = DeviceVector(4, n)
    nat.check(nat.lib().mpcore_elementwise(0, B.handle, Y.handle, R.handle),
              "QD subtract")
    r = float(np.max(np.abs(R.download()[0])))
    norm_a = float(A[0, :, :n].abs().sum(dim=1).max())
    norm_x = float(x[0].abs().max())
    del Aq
    torch.cuda.empty_cache()
    return {"backward_error": r / (norm_a * norm_x),
            "bound_n_u": n * U_P[k],
            "residual": "b - A x in QD on the GPU (mat_vec + subtraction "
                        "kernels), norms from the heads"}


def config4_work(n, nb):
    """madds of config 4's trailing updates (K = nb) and the FP64
    instructions of the whole LU + solve."""
    upd = 0
    for J in range(0, n, nb):
        w = min(nb, n - J)
        rest = n - J - w
        upd += rest * rest * w
    return upd


def run_dist(args):
    """BASELINE config 4: distributed DD LU + solve of ONE n x n system
    (n = 32768, ~17 GB in DD), column-block-cyclic over the ranks (nb =
    256), through the native driver (libmpcore dist.cu: one C-ABI call per
    solve; NCCL panel + pivot broadcasts of the live rows, look-ahead,
    column-cyclic back substitution; b rides along as a replicated column).
    One process per GPU; N = 1 runs the same code with a one-rank world.
    Strong scaling: value = (2/3) n^3 / (max-over-ranks device time)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ.setdefault("MPCORE_DEVICE", str(local))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        # host plumbing only (id exchange, timing max): the data path is
        # libmpcore's own NCCL communicator
        dist.init_process_group("gloo", rank=rank, world_size=world)
    pg = dist if world > 1 else None
    from paper_2107_12550_b200 import _native as nat
    from paper_2107_12550_b200.dist import (DeviceBackend, Layout, NcclComm,
                                            dist_lu_solve)
    k, n, nb = args.k, args.n, args.dist_nb
    seed = 210712550 + 4
    layout = Layout(n, nb, world)
    be = DeviceBackend(k)
    L = nat.lib()
    lc = layout.local_cols(rank)
    # b = A x_true (x_true = ones, DD mat_vec in the reference's order) on
    # rank 0 from the full matrix, shared with every rank (setup, untimed)
    bh = torch.zeros((k, n), dtype=torch.float64)
    if rank == 0:
        full = be.alloc(n, n)
        be.generate(full, Layout(n, nb, 1), 0, 0, seed)
        xt = torch.zeros((k, n), dtype=torch.float64, device="cuda")
        xt[0] = 1.0
        bd = torch.zeros_like(xt)
        torch.cuda.synchronize()
        nat.check(L.mpcore_dev_matvec(k, n, n, full.data_ptr(), n, n * n,
                                      xt.data_ptr(), bd.data_ptr()), "matvec")
        bh = bd.cpu()
        del full, xt, bd
        torch.cuda.empty_cache()
    if pg is not None:
        pg.broadcast(bh, src=0)
    M0 = be.alloc(n, lc + 1)
    base, ld, plane = be.view(M0)
    torch.cuda.synchronize()      # (torch's zero fill before the generator)
    if lc > 0:
        nat.check(L.mpcore_dev_generate_cyclic(
            k, base, ld, plane, n, lc, nb, world, rank, 0, n, seed),
            "generate_cyclic")
    M0[:, :, lc] = bh.to(M0.device)
    M = M0.clone()
    torch.cuda.synchronize()
    x = torch.zeros((k, n), dtype=torch.float64, device=M.device)
    with stdout_to_stderr():      # (NCCL's version banner goes to stdout)
        comm = NcclComm(world, rank)
    try:
        ncclv = ".".join(str(v) for v in torch.cuda.nccl.version())
    except Exception:
        ncclv = "?"
    print("[bench config4] rank %d/%d: libmpcore NCCL communicator up on "
          "cuda:%d (%s), NCCL %s, local columns %d of %d"
          % (rank, world, local, torch.cuda.get_device_name(local), ncclv,
             lc, n), file=sys.stderr, flush=True)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def step(phases=False):
        M.copy_(M0)
        return dist_lu_solve(layout, {rank: M}, {rank: x}, k, comm=comm,
                             stream=sp, phases=phases)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    peak_add, peak_fma = nat.fp64_peak()
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), \
        torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        launches = 0
        for _ in range(args.steps):
            launches += step()[2]
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = max_over_ranks(pg, ev0.elapsed_time(ev1) / args.steps)
    # per-panel critical-path breakdown: one more step with phase events
    # (--dist-trace PATH: every phase of every panel, start / end ms)
    if args.dist_trace and rank == 0:
        os.environ["MPCORE_DIST_TRACE"] = args.dist_trace
    _, phases, _ = step(phases=True)
    os.environ.pop("MPCORE_DIST_TRACE", None)
    torch.cuda.synchronize()
    xs = x.cpu().numpy()
    # end to end: this rank's columns from page-locked host memory each
    # step (H2D inside the timed region), solve, x back to the host
    e2e = None
    if not args.no_e2e:
        try:
            import psutil
            room = psutil.virtual_memory().available > 3 * M0.numel() * 8
        except Exception:
            room = False
        # one decision for every rank (each one's host memory check runs
        # while the others pin theirs): all run the e2e leg or none
        room = max_over_ranks(pg, 0.0 if room else 1.0) == 0.0
        if room:
            hM = torch.empty(M0.shape, dtype=torch.float64, pin_memory=True)
            hM.copy_(M0.cpu())
            hx = torch.empty((k, n), dtype=torch.float64, pin_memory=True)
            if pg is not None:
                pg.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            e_steps = max(1, min(args.steps, 2))
            for _ in range(e_steps):
                M.copy_(hM, non_blocking=True)
                dist_lu_solve(layout, {rank: M}, {rank: x}, k, comm=comm,
                              stream=sp)
                hx.copy_(x, non_blocking=True)
            ev1.record(stream)
            torch.cuda.synchronize()
            e_ms = max_over_ranks(pg, ev0.elapsed_time(ev1) / e_steps)
            assert hx.numpy().tobytes() == xs.tobytes()
            e2e = {"value": (2.0 / 3.0) * n ** 3 / (e_ms * 1e-3) / 1e9,
                   "unit": "GFLOP/s", "ms_per_step": e_ms,
                   "h2d_bytes_per_step": M0.numel() * 8,
                   "d2h_bytes_per_step": k * n * 8,
                   "path": "torch pinned host tensor -> this rank's local "
                           "columns + b (H2D, every step), mpcore_dist_lu_"
                           "solve (C ABI), x -> pinned host"}
    comm.close()
    if rank != 0:
        if pg is not None:
            pg.barrier()
        return
    err = float(np.max(np.abs((xs[0] - 1.0) + xs[1])))
    bwd = qd_backward_error(k, n, M0, M0[:, :, lc], x) if world == 1 \
        else None
    flops = (2.0 / 3.0) * n ** 3
    wc = work_counts(n, k)
    upd_instr = config4_work(n, nb) * MADD_INSTR[k]
    cpu = None
    if not args.no_cpu and world == 1:
        cpu = cpu_baseline(k, args.cpu_n or 4096, seed=seed)
        cpu["sample"] += ("; rate at n=%d stands for n=%d (time x (n/%d)^3)"
                          % (args.cpu_n or 4096, n, args.cpu_n or 4096))
    line = {
        "metric": "%s LU+solve eff. GFLOP/s ((2/3)n^3/s)" % NAMES[k],
        "value": flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64x%d (%s, bit-exact EFT arithmetic)" % (k, NAMES[k]),
        "data": "synthetic (seeded recipe, SURVEY 8d; seed %d)" % seed,
        "config": config_dict(args, world),
        "check": {"max_abs_err_x_vs_ones": err, **(bwd or {})},
        "roofline": {
            "bound": "fp64",
            "kernel": "trailing update (gemm_kernel NEG_A, K = %d), rank 0"
                      % nb,
            "achieved": upd_instr / world / (phases["update"] * 1e-3) / 1e12
            if phases["update"] > 0 else None,
            "peak": peak_add / 1e12, "unit": "T FP64 instr/s per GPU",
            "frac": upd_instr / world / (phases["update"] * 1e-3) / peak_add
            if phases["update"] > 0 and peak_add else None,
            "peak_source": "measured DADD issue rate (mpcore_fp64_peak)",
            "whole_step_frac": wc["instr"] / (ms * 1e-3) / world / peak_add
            if peak_add else None,
            "traffic": None},
        "phases_ms_rank0": phases,
        "phases_note": "one extra step with CUDA events around every phase "
                       "of every panel on its own stream (factor + pack: "
                       "side stream; bcast: comm stream incl. waiting for "
                       "the root; exch_trsm, update, back: main stream); "
                       "overlapping streams, so the parts exceed the total",
        "e2e": e2e,
        "gpu_launches": int(launches / max(1, args.steps)),
        "clocks": clk.summary(),
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line))
    if pg is not None:
        pg.barrier()


def run_config1(args):
    """BASELINE config 1: DD/TD/QD dense GEMM C = A*B, n = 2048 (the
    reference's mat_mul_blocked, linalg.py:577-617; every output's chain
    ascending in p from exact +0).  value = 2 n^3 / t; replicas for N > 1."""
    world, rank, local, pg = dist_setup(args)
    os.environ.setdefault("MPCORE_DEVICE", str(local))
    from paper_2107_12550_b200 import _native as nat
    from paper_2107_12550_b200.linalg import DeviceMatrix
    L = nat.lib()
    k, n = args.k, args.n
    seed = 210712550 + 1
    A = DeviceMatrix(k, n, n)
    A.generate(0, n, seed)
    B = DeviceMatrix(k, n, n)
    B.generate(1, n, seed)
    C = DeviceMatrix(k, n, n)

    def step():
        nat.check(L.mpcore_mat_mul(A.handle, B.handle, C.handle), "mat_mul")

    for _ in range(args.warmup):
        step()
    nat.sync()
    peak_add, peak_fma = nat.fp64_peak() if rank == 0 else (0.0, 0.0)
    barrier(pg)
    timer = nat.StreamTimer()   # CUDA events on the library stream
    with ClockSampler(local) as clk:
        timer.start()
        for _ in range(args.steps):
            step()
        dev_total = timer.stop()
        nat.sync()
    ms = max_over_ranks(pg, dev_total / args.steps)
    nat.prof_reset()
    nat.prof_enable(True)
    step()
    nat.sync()
    nat.prof_enable(False)
    prof = nat.prof_read()
    # e2e: host A, B (pinned) -> product -> host C
    hA, hB, hC = (nat.PinnedBuffer((k, n, n)) for _ in range(3))
    A.download(hA.array)
    B.download(hB.array)
    # double-buffered: the next step's A and B upload and the previous
    # step's C downloads (own copy stream) while this step multiplies;
    # every step moves A, B in and C out inside the timed region
    EA = [DeviceMatrix(k, n, n), DeviceMatrix(k, n, n)]
    EB = [DeviceMatrix(k, n, n), DeviceMatrix(k, n, n)]
    EC = [DeviceMatrix(k, n, n), DeviceMatrix(k, n, n)]
    hC2 = nat.PinnedBuffer((k, n, n))
    hCs = [hC, hC2]

    def upload(slot):
        nat.set_planes_async(EA[slot].handle, hA.array)
        nat.set_planes_async(EB[slot].handle, hB.array)

    def e2e_step(i, last=False):
        if not last:
            upload((i + 1) % 2)
        nat.check(L.mpcore_mat_mul(EA[i % 2].handle, EB[i % 2].handle,
                                   EC[i % 2].handle), "mm")
        nat.get_planes_async(EC[i % 2].handle, hCs[i % 2].array)

    upload(0)
    e2e_step(0, last=True)                        # warm-up
    nat.sync()
    e_steps = args.steps
    timer.start()
    upload(1)             # every timed step's A and B cross inside the region
    for i in range(1, e_steps + 1):
        e2e_step(i, last=i == e_steps)
    nat.sync()                                    # the last C is on the host
    e2e_ms = max_over_ranks(pg, timer.stop() / e_steps)
    hC = hCs[e_steps % 2]
    assert hC.array.tobytes() == C.download().tobytes()
    if rank != 0:
        return
    flops = 2.0 * n ** 3
    instr = n ** 3 * MADD_INSTR[k]
    gemm_ms = prof["gemm"][0] / max(1, prof["gemm"][1])
    line = {
        "metric": "%s GEMM eff. GFLOP/s (2n^3/s)" % NAMES[k],
        "value": world * flops / (ms * 1e-3) / 1e9, "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64x%d (%s, bit-exact EFT arithmetic)" % (k, NAMES[k]),
        "data": "synthetic (seeded splitmix64 recipe, SURVEY 8d; seed %d)"
                % seed,
        "config": config_dict(args, world),
        "e2e": {"value": world * flops / (e2e_ms * 1e-3) / 1e9,
                "unit": "GFLOP/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 2 * k * n * n * 8,
                "d2h_bytes_per_step": k * n * n * 8,
                "path": "C ABI, pinned host buffers, double-buffered: "
                        "set_planes_async(A, B) of the next step + mat_mul + "
                        "get_planes_async(C) (own copy stream, overlapping "
                        "the next product; all copies done before the stop "
                        "event)"},
        "roofline": {"bound": "fp64", "kernel": "gemm_kernel",
                     "achieved": instr / (gemm_ms * 1e-3) / 1e12,
                     "peak": peak_add / 1e12, "unit": "T FP64 instr/s",
                     "frac": instr / (gemm_ms * 1e-3) / peak_add
                     if peak_add else None, "traffic": None},
        "gpu_launches": int(sum(v[1] for v in prof.values())),
        "clocks": clk.summary(),
    }
    print(json.dumps(line))


def run_config3(args):
    """BASELINE config 3: TD-mpmath mixed-precision IR, n = 1024, A =
    U diag(sigma) W with kappa = 1e30 at 512 bits, rtol 1e-100, atol 0,
    maxtimes 20.  One step = the refinement driver from the long-precision
    system in host memory to the converged x (conversion to TD, TD LU on the
    GPU, residual loop on the host cores with the correction solves on the
    GPU); the system build is reported separately.  Replicas only."""
    world, rank, local, pg = dist_setup(args)
    os.environ.setdefault("MPCORE_DEVICE", str(local))
    from paper_2107_12550_b200 import _native as nat
    from paper_2107_12550_b200.refine import refine_config3, CONFIG3_SEED
    n = args.n
    kw = dict(n=n, seed=CONFIG3_SEED, kappa_exp10=30, short_k=3,
              long_bits=512, rtol="1e-100", atol="0", max_iter=20)
    for _ in range(max(1, args.warmup)):
        refine_config3(**kw)
    # kernel launches of one step (profiled pass, outside the timed steps)
    nat.prof_enable(True)
    nat.prof_reset()
    refine_config3(**kw)
    launches = sum(c for _, c in nat.prof_read().values())
    nat.prof_enable(False)
    runs = []
    barrier(pg)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            runs.append(refine_config3(**kw))
    t_step = [r["timings"]["convert"] + r["timings"]["factor"] +
              r["timings"]["loop"] for r in runs]
    sec = max_over_ranks(pg, statistics.median(t_step))
    if rank != 0:
        return
    r = runs[-1]
    tm = {a: statistics.median([q["timings"][a] for q in runs])
          for a in r["timings"]}
    line = {
        "metric": "TD-mpmath IR time-to-rtol (s)", "value": sec, "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f64x3 short side (TD) / 512-bit long side",
        "data": "synthetic: A = U diag(sigma) W, sigma geometric 1..1e-30, "
                "U, W seeded butterfly-orthogonal at 576-bit fixed point "
                "(stands in for QR of a Gaussian, SURVEY 7); b = A*ones",
        "config": config_dict(args, world),
        "result": {"iterations": r["iterations"],
                   "stop_reason": r["stop_reason"],
                   "residuals": r["residuals"],
                   "max_abs_err_vs_ones": r["max_abs_err_vs_ones"]},
        "timings_s": tm,
        # (bytes: the exact long A (96 B per element, flat), b as TD
        # planes and as a long vector, x (long) for every residual and the
        # TD right-hand side of every correction solve in; the long
        # residual of every iteration and the TD solution of every solve
        # out)
        "e2e": {"value": sec, "unit": "s", "h2d_bytes_per_step":
                96 * n * n + 3 * n * 8 + 96 * n
                + len(r["residuals"]) * 96 * n
                + r["iterations"] * 3 * n * 8,
                "d2h_bytes_per_step": len(r["residuals"]) * 96 * n
                + (r["iterations"] + 1) * 3 * n * 8,
                "path": "C ABI mpcore_refine_config3: host long system -> "
                        "flat exact values -> GPU (round to 512 bits, TD "
                        "heads, LU + first solve) -> residual loop: GPU "
                        "long residuals, host norms / checks, GPU "
                        "correction solves"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if not args.no_cpu and world == 1:
        # the same driver with the short side on the CPU: the oracle port's
        # TD LU + the solves, plus this run's host (long-side) time
        import oracle
        from oracle import gen
        A = gen.planes(3, (n, n), 0, n, CONFIG3_SEED)
        b = gen.planes(3, (n,), 2, n, CONFIG3_SEED)
        t0 = time.perf_counter()
        lu, sw = oracle.lu(A)
        t_lu = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.solve(lu, sw, b)
        t_sv = time.perf_counter() - t0
        host = tm["convert"] + tm["loop"] - tm["short_solves"]
        cpu_s = host + t_lu + (r["iterations"] + 1) * t_sv
        line["cpu_baseline"] = {
            "value": cpu_s, "unit": "s", "cores": oracle.num_threads(),
            "kind": "port",
            "sample": "TD LU (%.2f s) + solve (%.3f s) of a seeded n=%d TD "
                      "matrix by the oracle port (C++ restatement, OpenMP), "
                      "x%d solves, + this run's host long-side time (%.2f s)"
                      % (t_lu, t_sv, n, r["iterations"] + 1, host)}
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=None, choices=[1, 2, 3, 4],
                    help="BASELINE config (default: 2 on one GPU; 4 -- the "
                         "distributed n=32768 DD LU, strong scaling -- when "
                         "launched on several GPUs)")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--dim", dest="n", type=int, default=None)
    ap.add_argument("--nb", type=int, default=0)
    ap.add_argument("--dist-nb", type=int, default=256)
    ap.add_argument("--cpu-n", type=int, default=0,
                    help="CPU baseline sample size (0: per config)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-trace", default="",
                    help="config 4: write the per-panel phase timeline here")
    ap.add_argument("--no-extras", action="store_true",
                    help="default run: skip the other single-GPU configs "
                         "measured after the headline (the 'extras' key)")
    args = ap.parse_args()
    explicit = args.config is not None or args.k is not None or \
        args.n is not None
    if args.config is None:
        # the multi-GPU launch (torchrun, any world size, or --gpus > 1)
        # measures the north star's strong-scaling curve: config 4; a plain
        # single-process run measures config 2 (the BASELINE metric's)
        multi = (int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.gpus > 1
                 or "TORCHELASTIC_RUN_ID" in os.environ)
        args.config = 4 if multi else 2
    if args.config == 4:
        args.k = args.k or 2
        args.n = args.n or 32768
    elif args.config == 3:
        args.k = 3
        args.n = args.n or 1024
    elif args.config == 1:
        args.k = args.k or 2
        args.n = args.n or 2048
    else:
        args.k = args.k or 3
        args.n = args.n or 2048
    if args.impl == "reference":
        run_reference(args)
    elif args.config == 4:
        run_dist(args)
    elif args.config == 3:
        run_config3(args)
    elif args.config == 1:
        run_config1(args)
    elif explicit or args.no_extras or args.gpus > 1 or \
            int(os.environ.get("WORLD_SIZE", "1")) > 1:
        run_ours(args)
    else:
        line = captured(run_ours, args)
        line["extras"] = run_extras(args)
        print(json.dumps(line))


def captured(fn, args):
    """Run one bench leg in this process and return its JSON line."""
    import contextlib
    import io
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        fn(args)
    return json.loads(buf.getvalue().strip().splitlines()[-1])


def run_extras(args):
    """The default run's supplementary legs, AFTER the headline's timed
    region (so they cannot disturb it): the other single-GPU BASELINE
    workloads -- config 2 in QD, the DD LU + solve at n = 2048, the config-1
    GEMMs in DD/TD/QD and config 3 -- each with its own warm-up, CUDA-event
    timing on the library stream and clock sampling, summarised to its
    value, per-step time, e2e and roofline fractions, so every config's
    number comes out of the driver's own run.  --no-extras skips them."""
    legs = [("config2_qd_lu_solve_n2048", run_ours,
             dict(config=2, k=4, n=2048, steps=5, warmup=3)),
            ("dd_lu_solve_n2048", run_ours,
             dict(config=2, k=2, n=2048, steps=10, warmup=3)),
            ("config1_dd_gemm_n2048", run_config1,
             dict(config=1, k=2, n=2048, steps=5, warmup=2)),
            ("config1_td_gemm_n2048", run_config1,
             dict(config=1, k=3, n=2048, steps=3, warmup=2)),
            ("config1_qd_gemm_n2048", run_config1,
             dict(config=1, k=4, n=2048, steps=3, warmup=2)),
            ("config3_td_mpmath_ir_n1024", run_config3,
             dict(config=3, k=3, n=1024, steps=5, warmup=2))]
    out = {}
    for name, fn, kw in legs:
        a = argparse.Namespace(**vars(args))
        a.no_cpu = True
        for key, v in kw.items():
            setattr(a, key, v)
        try:
            d = captured(fn, a)
        except Exception as e:  # a leg's failure must not void the headline
            out[name] = {"error": "%s: %s" % (type(e).__name__, e)}
            continue
        rf = d.get("roofline") or {}
        e2e = d.get("e2e") or {}
        out[name] = {
            "metric": d["metric"], "value": d["value"], "unit": d["unit"],
            "ms_per_step": d["ms_per_step"], "steps": d["steps"],
            "warmup": d["warmup"], "higher_is_better": d["higher_is_better"],
            "e2e": e2e.get("value"),
            "dominant_kernel_frac": rf.get("frac"),
            "whole_step_frac": rf.get("whole_step_frac"),
            "clocks": d.get("clocks"),
            **({"result": d["result"]} if "result" in d else {})}
    return out


if __name__ == "__main__":
    main()
