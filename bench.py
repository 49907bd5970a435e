#!/usr/bin/env python
"""Benchmark: batched branch-MPC solves/sec (BASELINE.json configs[4]).

Workload (one "step"): 4096 independent instances of the paper's
intersection case (cfg0: build_intersection_case(intersection_spec(63, 10.0,
0.1), 2, 2), 250 nodes) PER GPU, instance i's measured state perturbed with
std::mt19937_64(42 + global index) — solved to convergence with the default
pmsilqr options by ONE kernel launch per GPU (one thread block per instance).
`value` = solves/sec of the whole job (all ranks; weak scaling), inputs
resident in HBM. `e2e` = the same through the public batch API with host
buffers: H2D of every instance's problem data, solve, D2H of trajectories and
reports inside the timed region. For N > 1 ranks the step ends with the
north star's final gather of all trajectories to rank 0 over NVLink (NCCL).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the reference's own CPU solver (oracle/_ref, the
unmodified headers compiled against the Eigen shim) on all host threads over
a bounded sample of the same instances (rank 0 only).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "BMPC solve latency (ms) vs horizon×scenarios; batched solves/sec at 1/2/4/8 GPU"
UNIT = "solves/s"
WORKLOAD = "cfg4: batched intersection_spec(63,10,0.1) 2x2 (250 nodes) x 4096 instances per GPU, perturbed x0"
PER_GPU = 4096
# Algorithmic FP64 work per non-leaf node per inner pass, MEASURED on the
# reference path (oracle/flop_count.cpp: the unmodified reference compiled
# against the Eigen shim with its opt-in flop counter, cfg0;
# profiles/r2_flop_count.json): linearize 1543.4, evaluate 117.4 (x2),
# backward 3451.8 (tree scan: init_bwd_element + combine_bwd) or 803.7
# (sequential Riccati — what the GPU's team sweep executes), forward 463.8,
# expected change 84.8, and 129.6 per line-search trial. The line search stops
# at the first round holding an accepted step size (same result), so its share
# is counted per step size actually evaluated: F_PASS per pass + F_ALPHA per
# evaluated alpha. roofline.achieved uses the work-efficient count (the
# algorithm the GPU runs); the reference-arithmetic count is reported beside it.
F_ALPHA = 129.6
F_PASS = 1543.4 + 2 * 117.4 + 803.7 + 463.8 + 84.8          # work-efficient (sequential Riccati backward)
F_PASS_REF = 1543.4 + 2 * 117.4 + 3451.8 + 463.8 + 84.8      # reference arithmetic (tree-scan backward)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--instances", type=int, default=PER_GPU)
    ap.add_argument("--no-latency", action="store_true", help="skip the single-solve latency table")
    ap.add_argument("--ref-sample", type=int, default=0, help="reference sample size (0 = auto)")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if len(s) > 2 + k and "Active" in s[2 + k]
                          and "Not" not in s[2 + k]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def host_info():
    """Cores this process may run on (affinity / cgroup aware) and the CPU model."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return cores, model


def ref_single_ms(family, horizon, branchings=(), parallel=1, caps=None, repeats=1):
    """The reference's own single-solve time (SolveReport::times.total_s,
    solver.hpp:563-570) of one scenario on this host; caps = (inner, outer)
    bounds the run for per-pass timing of the largest trees."""
    import _refbind as R

    sc = R.scenario(family, horizon, total_time=10.0, shared=(0.1, 0.0), v=(2, 2), branchings=branchings)
    o = R.default_options()
    o.parallel = parallel
    if caps:
        o.max_inner_iterations, o.max_outer_iterations = caps
    best, rep = None, None
    for _ in range(repeats):
        _, _, rep, _ = R.solve(sc, o, max_records=4000)
        t = rep["times"][5]
        best = t if best is None else min(best, t)
    return 1e3 * best, rep["n_records"] + rep["outer_iterations"], rep


def cpu_reference(sample, threads, seed0=42):
    """Reference CPU solver (oracle/_ref) over `sample` perturbed cfg0
    instances on `threads` host threads; returns (solves/s, seconds)."""
    import ctypes as C

    import _refbind as R

    sc = R.scenario(0, 63, perturb_seed=seed0)
    o = R.default_options()
    o.parallel = 0  # one solve per thread (bench.cpp:259-269 parallel_sweep pattern)
    secs, conv, inner = C.c_double(), C.c_int(), C.c_longlong()
    rc = R.lib().ref_batch_solve(C.byref(sc), C.byref(o), int(sample), int(threads), C.byref(secs),
                                 C.byref(conv), C.byref(inner))
    if rc != 0:
        raise RuntimeError(R.lib().ref_last_error().decode())
    return sample / secs.value, secs.value, conv.value


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads, model = host_info()
    # Each step: a work-stealing pool of `threads` std::threads over `sample`
    # distinct cfg4 instances (8 per thread, so one long solve does not decide
    # the wall time); successive steps take successive slices of the 4096 seeds.
    sample = args.ref_sample or 8 * threads
    for w in range(args.warmup):
        cpu_reference(threads, threads, seed0=42 + (w * threads) % PER_GPU)
    vals = []
    t0 = time.perf_counter()
    for k in range(args.steps):
        v, _, _ = cpu_reference(sample, threads, seed0=42 + (k * sample) % PER_GPU)
        vals.append(v)
    wall = time.perf_counter() - t0
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference scenario builders, seeded perturbations)",
            "config": {"workload": WORKLOAD, "sample_instances_per_step": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference", "cpu": model,
                             "sample": f"{sample} distinct perturbed cfg0 instances per step (successive slices of "
                                       f"the 4096 bench seeds), reference solve() with parallel=false on a "
                                       f"{threads}-thread work-stealing pool"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2506_13624_b200 as B

    # A dedicated (non-default) stream shared by torch events and the solver.
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = B.Context(local, stream=stream.cuda_stream)
    from paper_2506_13624_b200.sharding import ShardedBatch

    count = args.instances
    spec = B.intersection_spec(63, 10.0, 0.1)
    # This rank's contiguous shard of the job's world * count instances
    # (bmpc_shard_range): seeds 42 + global index.
    sharded = ShardedBatch(ctx, lambda b, k: [B.build_intersection_case(spec, 2, 2, perturb_seed=42 + b + i)
                                              for i in range(k)], world * count, world, rank)
    batch, probs = sharded.batch, sharded.problems
    n, nx, nu = batch.n, batch.nx, batch.nu
    h2d_setup = batch.set_models()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        batch.solve()
        if world > 1:  # final gather of every trajectory to rank 0 over NVLink
            sharded.gather(device="cuda")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for s in range(args.steps):
            kev[s][0].record(stream)
            batch.solve()
            kev[s][1].record(stream)
            if world > 1:
                sharded.gather(device="cuda")
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = ctx.launches - launches0
    elapsed = ev0.elapsed_time(ev1) / 1e3
    kernel_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    t = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = float(t.item())
    value = world * count * args.steps / elapsed

    reps, _ = batch.results(want_reports=True)
    status = np.array([r.status for r in reps])
    passes = np.array([r.n_records + r.outer_iterations for r in reps])
    nl = int((probs[0].tree.child_count > 0).sum())
    alpha_evals = float(sum(r.alpha_evals for r in reps))
    flops_per_launch = nl * (F_PASS * float(passes.sum()) + F_ALPHA * alpha_evals)
    flops_ref_arith = nl * (F_PASS_REF * float(passes.sum()) + F_ALPHA * alpha_evals)

    # e2e: public API with host buffers, copies inside the timed region. cfg4
    # instances share the scenario (references, predictions) and differ in the
    # measured initial state, so each call uploads the 4096 x0 (the receding-
    # horizon call, bmpc_batch_set_initial_states) and reads back every
    # trajectory and report. The variant that re-uploads every instance's full
    # node data each step is reported beside it (e2e_full_upload).
    xh = np.empty((count, n, nx))
    uh = np.empty((count, n, nu))
    x0_host = np.array([p.initial_state for p in probs])
    e2e_steps = max(1, min(args.steps, 3))

    def e2e_run(full_upload, scene=False):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h2d = d2h = 0
        for _ in range(e2e_steps):
            if scene:  # device-side scene generation from the spec, then the measured states
                h2d = batch.set_scenes(spec) + batch.set_initial_states(x0_host)
            else:
                h2d = batch.set_models() if full_upload else batch.set_initial_states(x0_host)
            batch.solve()
            _, d2h = batch.results(xh, uh, want_reports=True, as_array=True)
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return world * count * e2e_steps / float(te.item()), h2d, d2h

    e2e_scene, h2d_scene, _ = e2e_run(False, scene=True)
    e2e_full, h2d_full, _ = e2e_run(True)
    e2e_value, h2d, d2h = e2e_run(False)

    if rank == 0:
        peak = B.fp64_peak_tflops(ctx)
        achieved = flops_per_launch / (kernel_ms * 1e-3) / 1e12
        traffic = None
        prof = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("dram_bytes_per_step")
            except Exception:
                traffic = None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (in-library scenario builders, bit-identical to the reference's; seeded x0 "
                    "perturbations)",
            "config": {"workload": WORKLOAD, "instances_per_gpu": count, "nodes_per_instance": n,
                       "nonleaf_nodes": nl, "parallelism": f"dp{world} (independent instances, final NCCL gather)",
                       "l2": "per-step working set %.0f MB > 126 MB L2 (no flush needed)" %
                             (count * batch_bytes(n, nx, nu) / 1e6),
                       "converged": int((status == 0).sum()), "mean_inner_passes": float(passes.mean())},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "call": "set_initial_states(x0 of every instance) + solve + results(x, u, reports)"},
            "e2e_full_upload": {"value": e2e_full, "unit": UNIT, "h2d_bytes_per_step": int(h2d_full),
                                "d2h_bytes_per_step": int(d2h),
                                "call": "set_models(every instance's node data) + solve + results"},
            "e2e_scene": {"value": e2e_scene, "unit": UNIT, "h2d_bytes_per_step": int(h2d_scene),
                          "d2h_bytes_per_step": int(d2h),
                          "call": "set_scenes(scene spec: references and predictions generated on the GPU) + "
                                  "set_initial_states + solve + results"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "peak_source": "measured DFMA microbenchmark (bmpc_fp64_peak_tflops)",
                         "traffic_source": "DRAM bytes read+written by every launch of one step, one ncu session "
                                           "(profiles/traffic.json, tools/traffic.py)",
                         "kernel_ms": kernel_ms,
                         "algorithmic_flops_per_launch": flops_per_launch,
                         "flops_source": "per-phase FP64 flops of the reference path measured with the Eigen-shim "
                                         "flop counter (oracle/flop_count.cpp, profiles/r2_flop_count.json); "
                                         "work-efficient count (sequential Riccati backward, as the GPU runs it)",
                         "achieved_reference_arithmetic": flops_ref_arith / (kernel_ms * 1e-3) / 1e12},
            "clocks": clocks.summary(),
        }
        if world == 1:
            threads, model = host_info()
            sample = 256
            try:
                v, secs, _ = cpu_reference(sample, threads)
                serial_ms, _, _ = ref_single_ms(0, 63, parallel=0, repeats=3)
                line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference",
                                        "cpu": model, "serial_single_solve_ms": serial_ms,
                                        "sample": f"{sample} perturbed cfg0 instances (seeds 42..{41 + sample}), "
                                                  f"reference solve() (parallel=false) on a {threads}-thread "
                                                  f"work-stealing pool, {secs:.1f} s wall"}
            except Exception as e:  # reference library absent
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                        "sample": f"unavailable: {e}"}
            if not args.no_latency:
                line["latency_ms"] = latency_table(B, ctx, peak)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def batch_bytes(n, nx, nu):
    # state + scratch per instance, approximate (doubles)
    return 8 * n * (nx + nu + 8 + 58 + nx + 12 + 2 * 56 + 2 * 20 + nx + nu + 20) * 1.0


def latency_table(B, ctx, peak):
    """Single-solve latency of configs 0-3 on the GPU (kernel time of the one
    solve launch, inputs resident) next to the reference's own solve() on this
    host (SolveReport total time, default options = its own std::async
    parallelism), with each config's FP64 roofline fraction. The two cfg3
    trees take the reference minutes per solve, so the reference runs a capped
    solve there (3 inner passes, one outer) and the comparison is per pass."""
    import torch
    cases = [("cfg0 N=63 4 leaves", "int", 63, ()),
             ("cfg1 N=500 4 leaves", "int", 500, ()),
             ("cfg1 N=1000 4 leaves", "int", 1000, ()),
             ("cfg2 N=100 2 leaves {1}", "ms", 100, ((1, 2),)),
             ("cfg2 N=100 64 leaves {1,26,51}", "ms", 100, ((1, 4), (26, 4), (51, 4))),
             ("cfg3 N=500 256 leaves {1,100,200,300}", "ms", 500, ((1, 4), (100, 4), (200, 4), (300, 4))),
             ("cfg3 N=500 256 leaves {1,2,3,4}", "ms", 500, ((1, 4), (2, 4), (3, 4), (4, 4)))]
    out = {}
    for name, kind, N, br in cases:
        if kind == "int":
            p = B.build_intersection_case(B.intersection_spec(N, 10.0, 0.1), 2, 2)
        else:
            p = B.build_multistage_case(B.multistage_spec(N, list(br)))
        bt = B.Batch(ctx, [p])
        bt.set_models()
        bt.solve()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = torch.cuda.current_stream()
        e0.record(s)
        bt.solve()
        e1.record(s)
        torch.cuda.synchronize()
        rep, _ = bt.results(want_reports=True)
        r = rep[0]
        ms = e0.elapsed_time(e1)
        passes = r.n_records + r.outer_iterations
        nl = int((p.tree.child_count > 0).sum())
        row = {"ms": ms, "nodes": p.tree.node_count, "status": r.status_name, "inner": r.inner_iterations,
               "outer": r.outer_iterations, "passes": passes, "us_per_pass": 1e3 * ms / passes}
        # FP64 roofline: algorithmic flops per pass (SURVEY §8d constants, per evaluated step size).
        flops = nl * (F_PASS * passes + F_ALPHA * r.alpha_evals)
        row["roofline_frac"] = flops / (ms * 1e-3) / (peak * 1e12) if peak else None
        try:
            if name.startswith("cfg3"):
                ref_ms, ref_passes, _ = ref_single_ms(2, N, br, caps=(3, 1))
                row["reference_ms_per_pass"] = ref_ms / ref_passes
                row["speedup_per_pass"] = (ref_ms / ref_passes) / row["us_per_pass"] * 1e3
            else:
                ref_ms, ref_passes, rr = ref_single_ms(0 if kind == "int" else 2, N, br)
                row["reference_ms"] = ref_ms
                row["reference_inner"] = rr["inner_iterations"]
                row["speedup"] = ref_ms / ms
        except Exception as e:  # reference library absent
            row["reference_ms"] = f"unavailable: {e}"
        out[name] = row
    return out


if __name__ == "__main__":
    main()
