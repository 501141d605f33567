#!/usr/bin/env python
"""Benchmark: random-forest fit trees/s (+ predict rows/s) on B200 vs the host CPU reference.

Workload (BASELINE.json configs[3], "C4"): synthetic AIWC table 1,000,036 rows x 64
predictors (synthesize(6757 kernels, 37 devices) + make_dataset), mtry 8, min.node.size 5,
1000 trees per GPU (weak scaling: rank r grows trees [1000r, 1000(r+1)) of the
1000*N-tree forest keyed by derive_seed(1, "forest")), OOB statistics included (a fit
step is `fit()` exactly as forest.hpp:480 defines it: grow + compute_oob).
Secondary (reported in "predict"): configs[4] "C5", a 1000-tree forest on the C1 table
(m=6, mns=5) scoring 100M device-selection query rows.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One JSON line on rank 0.  Timing: CUDA events, barrier + synchronize around the K timed
steps, max over ranks.  Inputs (512 MB column store + ranks) exceed the 126 MB L2.
"""
from __future__ import annotations

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

C4_KERNELS, C4_DEVICES, C4_MTRY, C4_MNS = 6757, 37, 8, 5
C5_TREES, C5_MTRY, C5_MNS = 1000, 6, 5
METRIC = "RF fit trees/s + predict rows/s at 1/2/4/8 B200 (% HBM roofline) vs host CPU"


def traffic_per_launch(trees: int, launches: int):
    """Measured DRAM bytes of the grow phase per launch (a launch = one fit's grow phase):
    the committed ncu capture's bytes per tree times the trees each launch grew."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_grow_traffic.json")) as fh:
            d = json.load(fh)
        return d["dram_bytes_per_tree"] * trees / max(1, launches)
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.samples, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,utilization.gpu,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        util = [int(s[2]) if s[2].isdigit() else 0 for s in self.samples]
        loaded = [s for s, u in zip(self.samples, util) if u > 0] or self.samples
        sm = sorted(int(s[0]) for s in loaded if s[0].isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in loaded for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": int(self.samples[0][1]) if self.samples[0][1].isdigit() else None,
                "reasons": reasons, "samples": len(loaded)}


# ----------------------------------------------------------------------------------------
# CPU arms (reference compiled from /root/reference by oracle/Makefile -> oracle/_ref)
# ----------------------------------------------------------------------------------------
def cpu_worker(args) -> dict:
    """Times the reference's own fit (forest.hpp:480) on a bounded tree sample of C4.
    Runs in a subprocess: the reference's multi-threaded fit reads freed memory
    (oracle/REFERENCE_DEFECT.md), so a crash must not take the bench down."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Ref, RefData

    L = Ref.lib()
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    d = RefData(C4_KERNELS, C4_DEVICES)
    t1 = time.perf_counter()
    prep = d.prepared()
    t2 = time.perf_counter()
    seed = Ref.derive_seed(1, "forest")
    # distinct trees every step (step i: trees [i*sample, (i+1)*sample) of the 1000-tree
    # forest), OOB included: the reference's fit body over the range (ref_fit_range)
    sample = args.cpu_trees or cores
    rates, times = [], []
    import ctypes as C

    L.ref_fit_range.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                C.c_uint32, C.c_uint32, C.c_uint, C.POINTER(C.c_double)]
    out6 = (C.c_double * 6)()
    for step in range(max(1, args.cpu_steps)):
        t_lo = (step * sample) % max(1, 1000 - sample)
        s = time.perf_counter()
        Ref.check(L.ref_fit_range(prep, 1000, C4_MTRY, C4_MNS, seed, t_lo, t_lo + sample, cores,
                                  out6))
        times.append(time.perf_counter() - s)
        rates.append(sample / times[-1])
    # the other configurations, each a bounded sample, same cores
    from oracle_lib import RefForest, ref_evaluate

    extra = {}
    try:
        d1 = RefData()
        rows1 = d1.rows_rowmajor()
        s = time.perf_counter()
        f1 = RefForest.fit(d1, 500, 6, 5, seed, jobs=cores)  # C1: fit (OOB included)
        f1.predict(rows1, jobs=cores)
        extra["c1_trees_per_s"] = 500 / (time.perf_counter() - s)
        f5 = RefForest.fit(d1, 1000, 6, 5, seed, jobs=cores)  # C5 forest
        q = 50_000
        idx = np.array([Ref.bounded_draws(Ref.derive_seed(7, "query", i), 2220, 1)[0]
                        for i in range(q)])
        qrows = np.ascontiguousarray(rows1[idx])
        s = time.perf_counter()
        f5.predict(qrows, jobs=cores)
        extra["c5_rows_per_s"] = q / (time.perf_counter() - s)
        extra["c5_sample_rows"] = q
        s = time.perf_counter()
        ref_evaluate(d1, 505, 30, 9, seed, jobs=cores)  # C3: 37 folds
        extra["c3_folds_per_s"] = 37 / (time.perf_counter() - s)
    except Exception as e:  # noqa: BLE001
        extra["extra_error"] = str(e)[-200:]
    return {"value": sample * len(times) / float(np.sum(times)), "unit": "trees/s", "cores": cores,
            "kind": "reference", "rates": rates, **extra,
            "sample": f"{max(1, args.cpu_steps)} step(s) of {sample} distinct C4 trees each "
                      f"(step i: trees [i*{sample}, (i+1)*{sample}) of the 1000-tree m=8 mns=5 "
                      f"forest), the reference's fit body: TreeGrower::grow via "
                      f"parallel_for_with_state (forest.hpp:500-505) + compute_oob over the "
                      f"step's trees (forest.hpp:393-454), jobs={cores}; synth+join "
                      f"{t1 - t0:.1f}s and PreparedDataset {t2 - t1:.1f}s excluded "
                      f"(reported separately)",
            "prepare_s": t2 - t1, "synth_s": t1 - t0}


def run_cpu_subprocess(trees: int, steps: int, timeout: int | None = None) -> dict:
    timeout = timeout or 300 + 90 * steps
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-worker", "--cpu-trees", str(trees),
           "--cpu-steps", str(steps)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        for line in r.stdout.splitlines()[::-1]:
            if line.startswith("{"):
                return json.loads(line)
        return {"value": None, "error": (r.stderr or r.stdout)[-400:], "kind": "reference"}
    except Exception as e:  # noqa: BLE001
        return {"value": None, "error": str(e), "kind": "reference"}


# ----------------------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--trees-per-gpu", type=int, default=1000)
    ap.add_argument("--predict-rows", type=int, default=100_000_000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--skip-predict", action="store_true")
    ap.add_argument("--skip-grid", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="headline: weak = --trees-per-gpu trees on every GPU; strong = "
                         "--trees-per-gpu trees in total split by tree range (N > 1 also "
                         "measures the other mode and gathers the strong-mode forest)")
    ap.add_argument("--strong-steps", type=int, default=3,
                    help="timed steps of the secondary (non-headline) scaling mode at N > 1")
    ap.add_argument("--grid-cells", type=int, default=34,
                    help="cells of the C2 warm-up sample (and of the timed runs with "
                         "--grid-sample-only)")
    ap.add_argument("--grid-sample-only", action="store_true",
                    help="time the sample instead of the full 1,700-cell grid")
    ap.add_argument("--grid-runs", type=int, default=1)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--cpu-worker", action="store_true")
    ap.add_argument("--cpu-trees", type=int, default=0)
    ap.add_argument("--cpu-steps", type=int, default=1)
    args = ap.parse_args()
    global ARGS
    ARGS = args

    if args.cpu_worker:
        print(json.dumps(cpu_worker(args)))
        return

    world, rank, local = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return
        steps = max(1, args.steps)
        res = run_cpu_subprocess(args.cpu_trees, steps)
        v = res.get("value")
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "trees/s",
                "n_gpus": world, "steps": steps, "warmup": args.warmup,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": "C4 fit: synthetic AIWC 1,000,036 x 64, mtry 8, "
                                       "min.node.size 5, seed derive_seed(1,'forest')",
                           "parallelism": "host threads"},
                "cpu_baseline": {k: res.get(k) for k in ("value", "unit", "cores", "kind",
                                                         "sample")},
                "e2e": {"value": v, "unit": "trees/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        if v is None:
            line["error"] = res.get("error")
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    import paper_1811_00156_b200 as pkg

    backend = os.environ.get("AIWC_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())  # functional check: ranks share GPUs
    torch.cuda.set_device(local)
    # AIWC_BENCH_BACKEND=gloo: the N > 1 code path on ONE GPU (ranks share cuda:0, host-
    # staged collectives) -- a functional check only, its timings mean nothing
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    cdev = "cuda" if backend == "nccl" else "cpu"  # where the small reductions live

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t)
        return float(t.item())

    # CPU baseline on rank 0 (bounded sample, own subprocess), run after the GPU legs
    cpu_res = {}
    cpu_thread = None
    if rank == 0 and not args.skip_cpu:
        def _cpu():  # 4 steps of `cores` distinct trees (4 per thread), OOB included
            cpu_res.update(run_cpu_subprocess(args.cpu_trees, 4))
        cpu_thread = threading.Thread(target=_cpu, daemon=True)

    # ---------------- C4 fit ----------------
    t_setup = time.perf_counter()
    table = pkg.Table(C4_KERNELS, C4_DEVICES)
    prep = pkg.PreparedDataset.from_table(table, device=local)
    setup_s = time.perf_counter() - t_setup
    seed = pkg.derive_seed(1, "forest")
    from paper_1811_00156_b200 import shard

    dev = torch.device("cuda", local)
    dsend, drecv = shard.torch_device_transport(host_staging=backend != "nccl")

    def measure(mode: str, steps: int, warmup: int, keep_last: bool = False):
        """Timed C4 fits.  weak: rank r grows trees [T r, T (r+1)) of a T*N-tree forest;
        strong: the T-tree forest split by tree_range.  OOB (forest.hpp:393-454) is part of
        every step: one GPU finalises its own; N GPUs chain the per-row sums in tree order
        over NCCL on the devices (shard.chained_oob_device)."""
        T = args.trees_per_gpu
        total = T * world if mode == "weak" else T
        tb, te = (rank * T, (rank + 1) * T) if mode == "weak" else shard.tree_range(rank, world, T)
        params = pkg.ForestParams(total, C4_MTRY, C4_MNS, seed)

        def step():
            if world == 1:
                f = pkg.fit(prep, params)
                return f, f.oob
            f = pkg.fit(prep, params, tb, te, compute_oob_stats=False)
            res = shard.chained_oob_device(
                table.n, rank, world, dev,
                lambda ps, pc: pkg.oob_accumulate_device(f, prep, ps, pc), dsend, drecv)
            if res is None:
                return f, None
            rs, rc = res
            return f, pkg.oob_finalize(table.y, rs.cpu().numpy(),
                                       rc.cpu().numpy().view(np.uint32))

        for _ in range(warmup):
            f, _ = step()
            del f
        barrier()
        l0 = pkg.launch_count()
        stream = torch.cuda.current_stream()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r = {"grow_ms": 0.0, "split_rows": 0, "grow_launches": 0, "oob": None, "nodes": 0,
             "trees_total": total, "trees_rank": te - tb, "step_ms": [], "step_grow_ms": []}
        last = None
        with ClockSampler(local) as clk:
            barrier()
            ev0.record(stream)
            for i in range(steps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                f, o = step()
                e1.record(stream)
                e1.synchronize()
                r["step_ms"].append(e0.elapsed_time(e1))
                prof = f.profile()
                r["step_grow_ms"].append(prof["grow_ms"])
                r["grow_ms"] += prof["grow_ms"]
                r["split_rows"] += prof["split_rows"]
                r["grow_launches"] += prof["grow_launches"]
                r["oob"] = o if o is not None else r["oob"]
                r["nodes"] = f.total_nodes
                if keep_last and i == steps - 1:
                    last = f
                del f
            ev1.record(stream)
            barrier()
        r["launches"] = pkg.launch_count() - l0
        r["ms"] = max_over_ranks(ev0.elapsed_time(ev1))
        r["clocks"] = clk.summary()
        r["value"] = total * steps / (r["ms"] / 1e3)
        # the OOB statistic lives on the chain's last rank: hand it to rank 0
        err = r["oob"].error_pct if r["oob"] is not None else -1.0
        r["oob_error_pct"] = max_over_ranks(err)
        return r, last

    head, _ = measure(args.scaling, args.steps, args.warmup)
    per = head["trees_rank"]
    total_trees = head["trees_total"]
    ms, value, launches = head["ms"], head["value"], head["launches"]
    grow_ms, split_rows, grow_launch = head["grow_ms"], head["split_rows"], head["grow_launches"]
    nodes_last = head["nodes"]
    oob = head["oob_error_pct"]
    clk_summary = head["clocks"]
    tb, te = ((rank * args.trees_per_gpu, (rank + 1) * args.trees_per_gpu) if args.scaling == "weak"
              else shard.tree_range(rank, world, args.trees_per_gpu))
    params = pkg.ForestParams(total_trees, C4_MTRY, C4_MNS, seed)
    # roofline of the grow kernel: SURVEY 8d algorithmic bytes
    #   B_tree = 4n + sum_split_nodes rows(N) * (24*mtry + 16)
    n = table.n
    alg_bytes = args.steps * per * 4 * n + split_rows * (24 * C4_MTRY + 16)
    achieved = alg_bytes / (grow_ms / 1e3) / 1e9
    peak, peak_kind = peaks()

    # ---------------- e2e through the C-ABI with host buffers ----------------
    # one untimed warm-up step (the first new context grows the memory pool), then
    # --e2e-steps timed steps; every step is reported, the headline is their median
    e2e_times, e2e_parts, h2d, d2h = [], [], 0, 0
    barrier()
    for it in range(1 + max(1, args.e2e_steps)):
        s = time.perf_counter()
        p2 = pkg.PreparedDataset(table.col, table.y, table.n, table.p, device=local,
                                 host_mirror=True)
        s1 = time.perf_counter()
        if world == 1:
            f2 = pkg.fit(p2, params)
            _ = f2.oob
        else:
            f2 = pkg.fit(p2, params, int(tb), int(te), compute_oob_stats=False)
        s2 = time.perf_counter()
        arrs = f2.export(view=True)  # DMA into the forest's pinned host mirror
        s3 = time.perf_counter()
        ib = f2.inbag(view=True)
        s4 = time.perf_counter()
        if it > 0:
            e2e_times.append(s4 - s)
            e2e_parts.append([round(x, 4) for x in (s1 - s, s2 - s1, s3 - s2, s4 - s3)])
        h2d = table.col.nbytes + table.y.nbytes
        d2h = sum(a.nbytes for a in arrs) + ib.nbytes
        del f2, p2, arrs, ib
    e2e_s = max_over_ranks(float(np.median(e2e_times)))
    e2e_value = total_trees / e2e_s

    # ---------------- the other scaling mode + whole-forest gather (N > 1) ----
    other = None
    if world > 1:
        mode = "strong" if args.scaling == "weak" else "weak"
        r2, last = measure(mode, max(1, args.strong_steps), 1, keep_last=(mode == "strong"))
        other = {"scaling": mode, "value": r2["value"], "unit": "trees/s",
                 "ms_per_step": r2["ms"] / max(1, args.strong_steps),
                 "steps": max(1, args.strong_steps), "trees_total": r2["trees_total"],
                 "oob_error_pct": r2["oob_error_pct"], "clocks": r2["clocks"]}
        if mode == "strong" or args.scaling == "strong":
            if last is None:  # headline strong: refit the strong shard once for the gather
                T = args.trees_per_gpu
                a0, a1 = shard.tree_range(rank, world, T)
                last = pkg.fit(prep, pkg.ForestParams(T, C4_MTRY, C4_MNS, seed), a0, a1,
                               compute_oob_stats=False)
            pkg.release_cached(local)  # room for the gathered forest's torch buffers
            other["forest_gather"] = bench_forest_gather(pkg, torch, shard, last, rank, world,
                                                         local, barrier, max_over_ranks,
                                                         sum_over_ranks)
            del last

    del prep
    pkg.release_cached(local)
    torch.cuda.empty_cache()

    # ---------------- C5 predict ----------------
    predict = None
    if not args.skip_predict:
        predict = bench_predict(pkg, torch, args, local, barrier, max_over_ranks, world, peak)

    # ---------------- C2 grid + C3 hold-one-kernel-out (sharded by cell / fold) -----------
    grid = loko = c1 = None
    if not args.skip_grid:
        grid, loko, c1 = bench_grid_loko(pkg, torch, local, rank, world, barrier, max_over_ranks)

    if cpu_thread:
        # after every GPU-side measurement: the reference's jobs=nproc threads and our
        # host threads (grower lanes, copy threads, fold workers) must not share cores
        cpu_thread.start()
        cpu_thread.join(timeout=1200)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": value, "unit": "trees/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference synthesize()+make_dataset() restated bit-exactly; "
                "random forest trained from scratch each step)",
        "config": {"workload": "C4 fit: synthetic AIWC 1,000,036 x 64 (6757 kernels x 4 "
                               "sizes x 37 devices), mtry 8, min.node.size 5, "
                               + (f"{per} trees/GPU" if args.scaling == "weak" else
                                  f"{total_trees} trees split over {world} GPU(s)")
                               + ", OOB included",
                   "trees_total": total_trees, "rows": table.n, "predictors": table.p,
                   "parallelism": f"tree-seed shards x{world}, chained OOB on the devices",
                   "l2": "inputs (512 MB f64 column store + 128 MB ranks) exceed L2"},
        "oob_error_pct": None if oob < 0 else oob,
        "step_ms": head["step_ms"],
        "step_outside_grow_ms": [a - b for a, b in zip(head["step_ms"], head["step_grow_ms"])],
        "nodes_per_tree": nodes_last / per,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_per_launch(per * args.steps,
                                                                            grow_launch),
                     "traffic_source": "profiles/r2_grow_traffic.json (ncu dram__bytes of every "
                                       "grow kernel, 148-tree fit, per tree x trees per launch)",
                     "peak_kind": peak_kind,
                     "kernel": "wide grower: the level kernels w_* of one fit (grow phase)",
                     "algorithmic_bytes_per_launch": alg_bytes / max(1, grow_launch),
                     "kernel_ms_per_launch": grow_ms / max(1, grow_launch),
                     "kernel_share_of_step": grow_ms / max(1e-9, ms)},
        "e2e": {"value": e2e_value, "unit": "trees/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": len(e2e_times), "warmup": 1,
                "step_s": [round(x, 4) for x in e2e_times],
                "step_parts_s": {"ctx_create,fit,export,inbag": e2e_parts},
                "path": "aiwc_ctx_create(host col,y; host mirror on)+aiwc_fit (in-bag draws "
                        "DMA'd to pinned host memory as tree batches finish)+"
                        "aiwc_forest_host_view (nodes DMA'd into the forest's pinned mirror)"},
        "gpu_launches": launches,
        "clocks": clk_summary,
        "setup_s": setup_s,
        "cpu_baseline": ({k: cpu_res.get(k) for k in ("value", "unit", "cores", "kind", "sample")}
                         if cpu_res else None),
        "cpu_baseline_other": ({k: cpu_res.get(k) for k in ("c1_trees_per_s", "c5_rows_per_s",
                                                            "c5_sample_rows", "c3_folds_per_s",
                                                            "extra_error") if k in cpu_res}
                               if cpu_res else None),
        "predict": predict,
        "other_scaling": other,
        "c1": c1,
        "grid": grid,
        "loko": loko,
    }
    if cpu_res.get("error"):
        line["cpu_baseline_error"] = cpu_res["error"]
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_forest_gather(pkg, torch, shard, f, rank, world, local, barrier, max_over_ranks,
                        sum_over_ranks):
    """The strong-mode forest (every rank's tree range of the 1000-tree C4 forest) is
    all-gathered device to device over NCCL (shard.allgather_forest: export -> all_gather
    -> import, in-bag draws included), so every rank ends with the whole forest that was
    fit (~8.9 GB of nodes + 4 GB of in-bag draws)."""
    total_nodes = int(sum_over_ranks(float(f.total_nodes)))
    total_trees = int(sum_over_ranks(float(f.num_trees)))
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    import torch.distributed as dist

    ag = (dist.all_gather if os.environ.get("AIWC_BENCH_BACKEND", "nccl") == "nccl"
          else shard.host_staged_all_gather(dist.all_gather))
    g = shard.allgather_forest(f, world, local, ag, with_inbag=True)
    ev1.record(stream)
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    ok = g.num_trees == total_trees and g.total_nodes == total_nodes
    gathered = total_nodes * 24 + total_trees * f.n * 4  # node SoA + in-bag draws
    del g
    torch.cuda.empty_cache()
    return {"trees": total_trees, "nodes": total_nodes, "ms": ms,
            "bytes_per_rank": gathered, "GB_per_s_per_rank": gathered / ms / 1e6,
            "complete": bool(ok),
            "path": "aiwc_forest_export_device -> NCCL all_gather -> aiwc_forest_import_device"}


def bench_predict(pkg, torch, args, local, barrier, max_over_ranks, world, peak):
    """C5: 1000-tree forest on the C1 table; 100M queries per GPU resident in HBM."""
    t = pkg.Table()
    prep = pkg.PreparedDataset.from_table(t, device=local)
    seed = pkg.derive_seed(1, "forest")
    forest = pkg.fit(prep, pkg.ForestParams(C5_TREES, C5_MTRY, C5_MNS, seed))
    rows = torch.from_numpy(t.predictor_rows()).cuda()
    q = args.predict_rows
    qbuf = torch.empty((q, t.p), dtype=torch.float64, device="cuda")
    out = torch.empty(q, dtype=torch.float64, device="cuda")
    pkg.make_queries(rows.data_ptr(), t.n, t.p, q, 7, local, qbuf.data_ptr())
    for _ in range(max(1, args.warmup)):
        forest.predict_device(qbuf.data_ptr(), q, t.p, out.data_ptr())
    barrier()
    steps = max(1, args.steps)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(steps):
        forest.predict_device(qbuf.data_ptr(), q, t.p, out.data_ptr())
    ev1.record()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1)) / steps
    rate = q * world / (ms / 1e3)
    alg = q * (8 * t.p + 8)
    # e2e: host rows through aiwc_predict (H2D + kernel + D2H), bounded host buffer
    qe = min(q, 10_000_000)
    host = qbuf[:qe].cpu().numpy()
    _ = forest.predict_response(host[:1_000_000])  # warm: pinned staging, pool
    ts = []
    for _ in range(3):
        s = time.perf_counter()
        _ = forest.predict_response(host)
        ts.append(time.perf_counter() - s)
    e2e = qe / float(np.median(ts))
    # device selection (cmd_rank, tools/main.cpp:338-349): 1M feature rows x every device
    nfeat = 27
    ndev = t.p - nfeat
    feats = np.ascontiguousarray(host[:1_000_000, :nfeat])
    forest.rank(feats[:1000], ndev)
    ts = []
    for _ in range(3):
        s = time.perf_counter()
        _ = forest.rank(feats, ndev)
        ts.append(time.perf_counter() - s)
    rank_s = float(np.median(ts))
    del qbuf, out
    torch.cuda.empty_cache()
    return {"workload": "C5: 1000-tree C1 forest (m=6, mns=5), 100M device-selection queries "
                        "(row q = C1 row Rng(derive_seed(7,'query',q)).bounded(2220))",
            "rows_per_s": rate, "unit": "rows/s", "ms_per_pass": ms, "rows": q * world,
            "roofline": {"bound": "hbm", "achieved": alg / (ms / 1e3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": alg / (ms / 1e3) / 1e9 / peak,
                         "note": "B_row = 8p+8 = 344 B; node visits (~12K/row) bind on-chip"},
            "e2e": {"value": e2e, "unit": "rows/s", "rows": qe,
                    "h2d_bytes": qe * t.p * 8, "d2h_bytes": qe * 8},
            "rank": {"workload": f"cmd_rank over {len(feats)} feature rows x {ndev} devices "
                                 "(aiwc_rank, host buffers, best device + responses)",
                     "queries_per_s": len(feats) / rank_s,
                     "device_rows_per_s": len(feats) * ndev / rank_s}}


def bench_grid_loko(pkg, torch, local, rank, world, barrier, max_over_ranks):
    """C2: the num.trees x mtry x min.node.size OOB grid on the C1 table -- a bounded
    sample of (mtry, mns) cells, each one 1000-tree fit whose 20 tree prefixes
    (50..1000) give the 20 num.trees points (tree-prefix property); cell i on rank
    i mod N.  C3: evaluate at the paper's 505/30/9, folds split over the ranks."""
    from paper_1811_00156_b200 import shard

    t = pkg.Table()
    prep = pkg.PreparedDataset.from_table(t, device=local)
    seed = pkg.derive_seed(1, "forest")
    counts = list(range(50, 1001, 50))
    ncell = max(1, ARGS.grid_cells)
    sample = [(m, 1 + (7 * m) % 50) for m in range(1, 35)][:ncell]
    # the paper's full grid: mtry 1..34 x min.node.size 1..50 (x 20 num.trees prefixes)
    full = [(m, mns) for m in range(1, 35) for mns in range(1, 51)]
    cells = sample if ARGS.grid_sample_only else full
    nccl = os.environ.get("AIWC_BENCH_BACKEND", "nccl") == "nccl"
    allreduce = (shard.torch_allreduce_sum(torch.device("cuda", local) if nccl else None)
                 if world > 1 else (lambda a: a))
    # warm-up: the sample plus the grid's largest batch (mtry 34, min.node.size 1..34)
    _ = pkg.grid_oob(prep, sample + [(34, k) for k in range(1, 35)], counts, seed)
    grid_runs = []
    for _ in range(ARGS.grid_runs):  # every run reported; the headline is their mean
        barrier()
        s = time.perf_counter()
        err = shard.grid_sharded(cells, counts, rank, world,
                                 lambda cs: pkg.grid_oob(prep, cs, counts, seed), allreduce)
        barrier()
        grid_runs.append(max_over_ranks(time.perf_counter() - s))
    gs = float(np.mean(grid_runs))
    # C1: the paper-shaped table itself -- 500-tree fit (OOB included) + predict of its
    # 2220 rows, the reference's configs[0]
    c1p = pkg.ForestParams(500, 6, 5, seed)
    rows = t.predictor_rows()
    _ = pkg.fit(prep, c1p).predict_response(rows)
    ts = []
    for _ in range(5):
        s = time.perf_counter()
        f1 = pkg.fit(prep, c1p)
        _ = f1.oob
        _ = f1.predict_response(rows)
        ts.append(time.perf_counter() - s)
    c1 = {"workload": "C1: 2220 x 42 paper-shaped table, 500 trees m=6 mns=5, fit (OOB "
                      "included) + predict_response of all 2220 rows, host buffers",
          "trees_per_s": 500 / float(np.median(ts)), "s": float(np.median(ts)),
          "oob_error_pct": f1.oob.error_pct}
    what = "sample of" if ARGS.grid_sample_only else "full grid:"
    grid = {"workload": f"C2 {what} {len(cells)} (mtry, min.node.size) cells x {len(counts)} "
                        "num.trees values (50..1000) on the C1 table = "
                        f"{len(cells) * len(counts)} grid points, one 1000-tree fit per cell "
                        "(tree-prefix OOB), OOB error_pct of every point",
            "cells": len(cells), "points": len(cells) * len(counts),
            "cells_per_s": len(cells) / gs, "grid_points_per_s": len(cells) * len(counts) / gs,
            "s": gs, "runs_s": grid_runs,
            "best": {"error_pct": float(err.min()),
                     "cell": cells[int(err.argmin() // len(counts))],
                     "num_trees": counts[int(err.argmin() % len(counts))]}}
    prm = pkg.ForestParams(505, 30, 9, 0)
    _ = pkg.evaluate(t, prm, seed, device=local,  # warm-up: this rank's whole fold share
                     folds=shard.fold_range(rank, world, t.kernels))
    loko_runs = []
    for _ in range(3):  # every run reported; the headline is their mean
        barrier()
        s = time.perf_counter()
        part = pkg.evaluate(t, prm, seed, device=local,
                            folds=shard.fold_range(rank, world, t.kernels))
        pred = allreduce(part)
        barrier()
        loko_runs.append(max_over_ranks(time.perf_counter() - s))
    ls = float(np.mean(loko_runs))
    err_row = 100.0 * np.abs(pred - t.seconds) / t.seconds
    loko = {"workload": "C3: evaluate(C1, 505/30/9): 37 folds x 60 held-out rows",
            "folds_per_s": t.kernels / ls, "s": ls, "runs_s": loko_runs, "mape_pct": float(err_row.mean())}
    del prep
    return grid, loko, c1


ARGS = None

if __name__ == "__main__":
    main()
