#!/usr/bin/env python
"""FLIP timestep benchmark (BASELINE.json: particle-steps/s and ms per step
at 256^3, dam-break, 8 particles/cell, PCG + MIC(0)).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One JSON line on rank 0.  A "step" is one full flipsim.sim.step() (all ten
stages) of the dam-break scene at --res (default 256).  The scene comes from
the reference's own scene builder restated on the device (synthetic, seed 0).

* value     particle-steps/s = sum over timed steps of the particle count
            entering the step / device time (CUDA events on the library's
            stream, warm state resident in HBM; max over ranks).
* e2e       the same metric through the C ABI with HOST buffers: every step
            uploads particles + labels from pinned host memory, steps, and
            downloads the particles.
* roofline  dominant kernel = the MIC(0) substitution sweeps (k_mic_quad,
            forward + backward, ~52% of the step): algorithmic bytes (3 x 8 B
            per row) over the measured per-launch time of every launch in
            the timed region.  The per-launch time comes from %globaltimer
            stamps the kernel writes itself (first CTA past its programmatic
            launch wait, last CTA exit): CUDA events recorded between the
            launches would break the programmatic-dependent-launch overlap
            of the PCG loop (measured: +3 ms per step).  The round-1
            kernels (FLIPB200_QUAD=0) are still bracketed by CUDA events.
* clocks    nvidia-smi every 50 ms from before the warm-up; only samples
            inside the timed region's wall-clock window are kept.
* cpu_baseline  the oracle (C restatement of the reference step, all host
            threads) on a bounded sample of the same workload.
* --impl reference  times the oracle port as the reference arm (the Python
            reference cannot travel to the GPU box; oracle/ is its bit-exact
            C restatement, pinned by tests/).

Multi-GPU (torchrun, one process per GPU, NCCL): the z-slab decomposition
(csrc/slab.cu, driven from inside flip_step through paper_2404_01931_b200/
dist.py's transport): every stage runs on the rank's planes / rows /
particles with 1-plane halos, particle migration and ghost planes, MAX
allreduces and the bit-exact distributed pairwise dot; the MIC(0) sweeps are
one global recurrence, replicated on the all-gathered vector.
The total workload stays the 256^3 scene ("scaling": "strong"); results are
bit-identical to one GPU.
"""

from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

BASE_METRIC = "particle-steps/sec and ms/FLIP step at 256^3 (1/2/4/8 B200) + HBM roofline %"
UNIT = "particle-steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--res", type=int, default=256)
    ap.add_argument("--scene", default="dam-break")
    ap.add_argument("--solver", default="pcg")
    ap.add_argument("--precond", default="mic0",
                    help="mic0 (the reference's, default) or mg (extension: multigrid, "
                         "converged, tolerance-validated)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def workload(args) -> dict:
    if args.solver == "pcg":
        prec = ("MIC(0)-PCG, cap 100" if getattr(args, "precond", "mic0") == "mic0"
                else f"{args.precond}-PCG (extension), cap 100")
    else:
        prec = f"{args.solver}, cap 2000"
    return {"workload": f"{args.scene} {args.res}^3, density 2 (8 particles/cell), {prec}, "
                        f"tol 1e-6, flip 0.95, seed 0",
            "res": args.res, "scene": args.scene, "solver": args.solver,
            "l2_policy": "inputs larger than L2 (particle state >= 1.2 GB per step)"}


# ------------------------------------------------------------- clocks -----
class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = f"/tmp/flipb200_clocks_{os.getpid()}.csv"
        self.window = None

    def start(self):
        """Started before the warm-up (nvidia-smi takes a while to begin
        sampling); mark() brackets the timed region and only samples inside
        it are kept."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "50"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def mark(self, t0: float, t1: float):
        self.window = (t0, t1)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8 or f[1] != str(self.idx):
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[2]), float(f[3]), f[4:8]))
            except ValueError:
                continue
        if self.window is not None:
            inside = [r for r in rows if self.window[0] <= r[0] <= self.window[1]]
            rows = inside or sorted(rows, key=lambda r: abs(r[0] - self.window[1]))[:1]
        sm, mx, reasons = [r[1] for r in rows], [r[2] for r in rows], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[3]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------- oracle -----
def oracle_sample(args, steps: int, warm: int, threads: int):
    """Oracle (C restatement of flipsim.sim.step) on the same scene: returns
    (particle-steps/s, seconds per step, detail)."""
    sys.path.insert(0, os.path.join(HERE, "oracle"))
    import oracle as O
    O.build()
    O.set_threads(threads)
    spec = O.Spec(name=args.scene, res=args.res, solver=args.solver)
    t0 = time.perf_counter()
    st = O.make_scene(spec, rng_seed=0)
    setup = time.perf_counter() - t0
    n0 = st.n
    for _ in range(warm):
        O.step(st, spec)
    tot_n, tot_t, iters = 0, 0.0, []
    for _ in range(steps):
        n_in = st.n
        t0 = time.perf_counter()
        r = O.step(st, spec)
        tot_t += time.perf_counter() - t0
        tot_n += n_in
        iters.append(r["solver_iterations"])
    return tot_n / tot_t, tot_t / max(steps, 1), {"setup_s": round(setup, 2), "n0": n0,
                                                  "iters": iters, "n_final": st.n}


def run_reference(args):
    """The reference arm: the oracle port of flipsim.sim.step (bit-identical
    to the reference, 2.7x faster than it) on all host threads, timing the
    SAME step indices as our arm: max(3, W) untimed steps from make_scene,
    then K timed steps (steps W+1 .. W+K), same scene/solver/config keys."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    steps = max(1, args.steps)
    warm = max(3, args.warmup)
    v, sps, det = oracle_sample(args, steps, warm, threads)
    sample = (f"steps {warm + 1}..{warm + steps} of the {args.res}^3 scene (the step indices "
              f"our arm times) after {warm} untimed steps, {threads} OpenMP threads, "
              f"make_scene ({det['setup_s']} s) excluded")
    line = {"metric": BASE_METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": sps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference scene builder, seed 0)",
            "config": dict(workload(args), particles_initial=det["n0"],
                           parallelism="single"),
            "impl": "reference",
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "detail": {"solver_iterations": det["iters"], "particles_final": det["n_final"]}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- ours -----
def load_traffic():
    p = os.path.join(HERE, "profiles", "roofline_traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return None


def measured_peak():
    try:
        return float(json.load(open(os.path.join(HERE, "MEASURED_PEAKS.json")))["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def run_ours(args):
    import ctypes as C

    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hooks: ranks sharing one GPU over gloo (no NCCL with duplicate GPUs)
    if os.environ.get("FLIPB200_SAME_GPU"):
        local = 0
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group(os.environ.get("FLIPB200_DIST_BACKEND", "nccl"))
    torch.cuda.set_device(local)

    import paper_2404_01931_b200 as P
    from paper_2404_01931_b200 import _lib
    from paper_2404_01931_b200._lib import LIB, check

    spec = P.SceneSpec(name=args.scene, res=args.res, solver=args.solver, precond=args.precond)
    if world > 1:
        from paper_2404_01931_b200 import dist as D
        st = D.make_scene(spec, rng_seed=0, device=local)
        do_step = D.step
    else:
        st = P.make_scene(spec, rng_seed=0, device=local)
        do_step = P.step
    dev = st.device
    n0 = st.particles.count
    clocks = ClockSampler(local)
    clocks.start()
    warm = max(3, args.warmup)
    for _ in range(warm):
        do_step(st, spec)
    stream = torch.cuda.ExternalStream(dev.stream_ptr(), device=local)

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---------------- device-resident timed region ----------------
    check(LIB.flip_set_probe(dev.ctx, 1))
    barrier()
    torch.cuda.synchronize()
    wall0 = time.time()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    parts = 0
    launches = 0
    stage = {}
    iters = []
    rows_acc = []
    for _ in range(args.steps):
        parts += st.particles.count
        rep = do_step(st, spec)
        launches += rep.gpu_launches
        iters.append(rep.solver_iterations)
        rows_acc.append(rep.nrows)
        for k, v in rep.timings.as_dict().items():
            stage[k] = stage.get(k, 0.0) + v
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    barrier()
    clocks.mark(wall0, time.time())
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    pms, plaunch, pbytes = C.c_double(0), C.c_int64(0), C.c_double(0)
    check(LIB.flip_get_probe(dev.ctx, C.byref(pms), C.byref(plaunch), C.byref(pbytes)))
    check(LIB.flip_set_probe(dev.ctx, 0))
    total_parts = parts
    ms_max = ms
    if dist is not None:
        t = torch.tensor([ms, float(parts), float(launches)], device=f"cuda:{local}",
                         dtype=torch.float64)
        tm = t.clone()
        dist.all_reduce(tm[0:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:3], op=dist.ReduceOp.SUM)
        ms_max, total_parts, launches = float(tm[0]), float(t[1]), int(t[2])
        n0 = int(st.slab.tr.allreduce_sum_int(n0))
    value = total_parts / (ms_max / 1e3)

    # ---------------- end to end through the C ABI (host buffers) ----------
    e2e = None
    if not args.no_e2e:
        # pinned host buffers with headroom for the per-step reseed growth
        cap = min(int(dev.count() * 1.25) + 4096, 12 * dev.dims.ncells)
        host = [torch.empty(cap, dtype=torch.float64, pin_memory=True) for _ in range(6)]
        hv = [h.numpy() for h in host]
        lab = torch.empty(dev.dims.ncells, dtype=torch.uint8, pin_memory=True).numpy()
        lab[:] = st.grid.label
        n = dev.count()
        check(LIB.flip_get_particles(dev.ctx, *[a.ctypes.data_as(_lib._d) for a in hv]))
        params = P.sim._params(spec, dev.dims.dtau, 0)
        repc = _lib.StepReportC()
        h2d = d2h = 0
        e2e_steps = args.steps
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_parts = 0
        for k in range(e2e_steps):
            # step inputs from pinned host memory
            check(LIB.flip_set_particles(dev.ctx, n, *[a.ctypes.data_as(_lib._d) for a in hv]))
            check(LIB.flip_set_grid(dev.ctx, None, None, None, None,
                                    lab.ctypes.data_as(_lib._u8)))
            h2d += 48 * n + lab.size
            if world > 1:
                dev.bump()
                do_step(st, spec)   # the slab step through the public API
                e2e_parts += n
                n = dev.count()
            else:
                params.reseed_seed = P.rng.derive_seed(st.rng_seed, st.step_count + 1)
                rc = LIB.flip_step(dev.ctx, C.byref(params), C.byref(repc))
                check(rc)
                st.step_count += 1
                e2e_parts += n
                n = int(repc.particle_count)
            if n > cap:
                raise RuntimeError("e2e host buffers too small")
            # result back to pinned host memory
            check(LIB.flip_get_particles(dev.ctx, *[a.ctypes.data_as(_lib._d) for a in hv]))
            d2h += 48 * n
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        dev.bump()
        w = torch.tensor([wall, float(e2e_parts), float(h2d), float(d2h)], dtype=torch.float64,
                         device=f"cuda:{local}")
        if dist is not None:
            wm = w.clone()
            dist.all_reduce(wm[0:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(w[1:4], op=dist.ReduceOp.SUM)
            w[0] = wm[0]
            h2d, d2h = int(w[2]), int(w[3])
        e2e = {"value": float(w[1]) / float(w[0]), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d // e2e_steps), "d2h_bytes_per_step": int(d2h // e2e_steps),
               "timing": "wall clock around K synchronous C-ABI steps incl. pinned H2D/D2H"}

    n_final = dev.count()
    if dist is not None:
        n_final = int(st.slab.tr.allreduce_sum_int(n_final))
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    mean_rows = sum(rows_acc) / max(len(rows_acc), 1)
    # ---------------- roofline of the dominant kernel ----------------
    peak, peak_kind = measured_peak()
    roof = None
    if plaunch.value > 0:
        avg_ms = pms.value / plaunch.value
        alg = pbytes.value / plaunch.value
        achieved = alg / (avg_ms / 1e3) / 1e9
        tr = load_traffic()
        quad = os.environ.get("FLIPB200_QUAD", "1") != "0"
        kname = ("k_mic_quad (MIC(0) substitution wavefront, 2x2 pencils per thread, DSMEM "
                 "clusters, fwd+bwd)" if quad else
                 "k_mic_cl (MIC(0) substitution wavefront, DSMEM clusters, fwd+bwd)")
        roof = {"bound": "hbm", "kernel": kname,
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_kind": peak_kind, "alg_bytes_per_launch": alg,
                "avg_launch_ms": avg_ms, "launches_timed": int(plaunch.value),
                "share_of_step": pms.value / ms,
                # the ncu capture is of the 256^3 dam-break sweep
                "traffic": ((tr or {}).get("k_mic_quad_dram_bytes_per_launch" if quad else
                                           "k_mic_cl_dram_bytes_per_launch")
                            if (args.res, args.scene) == (256, "dam-break") else None),
                "timing": ("in-kernel %globaltimer stamps per launch (first CTA start after "
                           "the PDL wait, last CTA end), every launch of the timed region"
                           if quad else "CUDA events bracketing each launch"),
                "note": "latency-bound dependency wavefront (see DESIGN.md); "
                        "frac is of the HBM copy peak"}

    cpu = None
    if not args.no_cpu and world == 1:
        try:
            threads = os.cpu_count() or 1
            v, sps, det = oracle_sample(args, 1, 1, threads)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": f"1 full {args.res}^3 oracle step after 1 warm-up step, "
                             f"{threads} OpenMP threads (setup {det['setup_s']} s excluded)"}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                   "sample": f"failed: {exc}"}

    # whole-step HBM roofline: algorithmic bytes of every
    # stage, with this run's particle count, rows and solver iterations
    res = args.res
    C_ = float(res ** 3)
    F_ = 3.0 * (res + 1) * res * res
    N_ = float(total_parts) / args.steps     # global particles entering a step
    R_ = float(mean_rows) if mean_rows else 0.0
    its = sum(iters) / max(len(iters), 1)
    per_it = 147.0 * R_ if args.solver == "pcg" else 25.0 * R_
    step_bytes = (24 * N_ + 72 * N_ + (96 * N_ + 8 * C_) + 6 * C_ + (48 * N_ + 8 * C_ + 17 * F_)
                  + (16 * F_ + C_) + (8 * F_ + C_ + 9 * R_) + its * per_it + 17 * R_
                  + (18 * C_ + 66 * F_) + (72 * N_ + 16 * F_) + (96 * N_ + 8 * C_))
    step_gbs = step_bytes / (ms_max / args.steps / 1e3) / 1e9
    roof_step = {"alg_bytes_per_step": step_bytes, "achieved": step_gbs, "unit": "GB/s",
                 "peak": peak, "frac": step_gbs / peak,
                 "formula": "SURVEY 8(d) per-stage algorithmic bytes, N/R/iterations measured"}

    line = {"metric": BASE_METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": warm, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference dam-break scene builder on the device, seed 0)",
            "config": dict(workload(args), particles_initial=n0,
                           parallelism=(f"slab-z{world}" if world > 1 else "single")),
            "clocks": clk, "e2e": e2e, "gpu_launches": launches, "roofline": roof,
            "roofline_step": roof_step,
            "cpu_baseline": cpu,
            "detail": {"stage_ms_mean": {k: v / args.steps for k, v in stage.items()},
                       "solver_iterations": iters,
                       "particles_final": n_final}}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
