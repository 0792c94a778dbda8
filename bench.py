#!/usr/bin/env python
"""Headline benchmark: full-graph GraphSAGE training epoch on the synthetic
Reddit-shape graph (BASELINE.json configs[1]), B200 engine vs the CPU oracle.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

A step is one epoch: forward over 3 layers (602 -> 64 -> 64 -> 41), softmax
cross-entropy over all 232,965 vertices, backward, weight all-reduce and SGD.
Rows are split into N contiguous blocks (strong scaling: the graph is fixed).
Timing: W untimed epochs, then K epochs bracketed by barrier + synchronize,
CUDA events on the compute stream, max over ranks.  Every epoch streams the
458 MB column array and the 567 MB input-feature operand through HBM, so the
per-step working set exceeds the 126 MB L2 (no explicit flush).

Prints ONE JSON line on rank 0.
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

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

REDDIT = dict(n=232965, degree=491.99, seed=11, dims=[602, 64, 64, 41])
METRIC = "GCN epoch ms & aggregation edges/s, synthetic Reddit-shape graph, 1/2/4/8 B200"
MODEL = "sage"
# BASELINE.json configs beyond the headline (configs[1]); selected with --config
CONFIGS = {
    "reddit-sage": dict(n=232965, degree=491.99, seed=11, kind="sage", dims=[602, 64, 64, 41],
                        mode="full", lr=0.1,
                        workload="reddit-shape full-graph 3-layer GraphSAGE-mean training epoch "
                                 "(BASELINE configs[1])"),
    "reddit-gcn56-eas": dict(n=232965, degree=491.99, seed=11, kind="gcn", dims=[602] + [64] * 55 + [41],
                             mode="eas", eas=(1, 15, 3), lr=0.01,
                             workload="reddit-shape 56-layer normalised GCN, expansion-aware sampling "
                                      "EAS(m=1,k=15,seed=3), one emulated server per GPU (random "
                                      "partition), loss on inner vertices (BASELINE configs[2])"),
    "products-gcn": dict(n=2449029, degree=25.26, seed=13, kind="gcn", dims=[100, 64, 64, 47],
                         mode="full", lr=0.1,
                         workload="ogbn-products-shape full-graph 3-layer normalised GCN, features "
                                  "resident on every GPU (shared preload with one server) "
                                  "(BASELINE configs[3])"),
    "papers-cobatch": dict(n=111059956, degree=14.55, seed=17, kind="sage", dims=[128, 64, 64, 172],
                           mode="cobatch", eas=(1, 15, 3), batches=256, lr=0.1,
                           workload="ogbn-papers100M-shape cooperative-batching mini-batch 3-layer "
                                    "GraphSAGE-mean: one server, its GPUs share every batch "
                                    "(split_batch), sampled closure EAS(m=1,k=15,seed=3), R batches "
                                    "= R SGD steps per epoch (BASELINE configs[4])"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--eager", action="store_true", help="launch kernels eagerly (no CUDA graph)")
    ap.add_argument("--cpu-sample-rows", type=int, default=0)
    ap.add_argument("--config", default="reddit-sage", choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=0, help="override the vertex count (0: config's)")
    ap.add_argument("--degree", type=float, default=0.0)
    ap.add_argument("--batches", type=int, default=0, help="cobatch R (0: config's)")
    return ap.parse_args()


def bind_numa(local: int) -> list:
    """Pin this rank to the CPUs of its GPU's NUMA node (NVML affinity), so the pinned
    host buffers of the end-to-end feature stream are allocated (first touch) next to
    the GPU's PCIe root.  Returns the CPU list (empty if NVML is unavailable)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(local)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = [64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1]
        if cpus and os.environ.get("GDX_NUMA_BIND", "1") != "0":
            os.sched_setaffinity(0, cpus)
        return cpus
    except Exception:
        return []


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------------
def cpu_baseline_record(args, steps=1, warmup=0):
    """The oracle port's fp64 SAGE epoch (forward, loss, backward, SGD) on all host
    threads, restricted to destination rows < rows (default: all rows), timed and
    extrapolated linearly to the whole epoch."""
    import oracle as O

    threads = os.cpu_count() or 1
    rows = min(args.n, args.cpu_sample_rows or args.n)
    dims = REDDIT["dims"]
    g = O.gen_random_graph(args.n, args.degree, REDDIT["seed"])
    x = O.make_features(args.n, dims[0], 1)
    labels = O.make_labels(args.n, dims[-1], 2)
    model = O.Model(O.SAGE, dims)
    w = np.random.default_rng(0).uniform(-0.5, 0.5, model.weight_count())
    times = []
    for i in range(warmup + steps):
        t = time.perf_counter()
        O.train_epoch(g, x, labels, model, w, 0.1, row_limit=rows, nthreads=threads)
        if i >= warmup:
            times.append(time.perf_counter() - t)
    sec = statistics.median(times)
    epoch_ms = sec * 1e3 * args.n / rows
    return {
        "value": round(epoch_ms, 1), "unit": "ms", "cores": threads, "kind": "port",
        "sample": (f"oracle port (fp64 C restatement of the reference loops, OpenMP {threads} "
                   f"threads): one SAGE epoch over {rows} of {args.n} destination rows, median of "
                   f"{steps} ({sec:.2f} s), x{args.n / rows:.2f} to a full epoch; the reference has "
                   f"no training path (SPEC.md:9), so its own code cannot run this epoch"),
    }


# ---------------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clock and throttle reasons every 5 ms on a thread (NVML) while the
    timed region runs; falls back to nvidia-smi polling when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.max_mhz = None
        self._stop = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis else self.gpu
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return self
        self._stop = threading.Event()

        def loop():
            while not self._stop.is_set():
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.samples.append((sm, rs))
                except Exception:
                    pass
                self._stop.wait(0.005)

        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        sm = [s for s, _ in self.samples]
        reasons = sorted({k for _, r in self.samples for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "nvml 5 ms polling during the timed region"}


def load_peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


def launches_per_epoch(tr) -> int:
    """libgdx kernel launches in one eager epoch (graph replays issue the same kernels)."""
    import torch
    from paper_2311_06837_b200 import _lib
    torch.cuda.synchronize()
    a = _lib.launch_count()
    tr.train_epoch(sync_loss=False)
    torch.cuda.synchronize()
    return _lib.launch_count() - a


def probe_l2_peak(torch, dev):
    """Live L2 read ceiling: the library's coalesced-stream probe over a 60 MB
    (L2-resident) buffer, best of 3, GB/s."""
    from paper_2311_06837_b200._lib import call
    from paper_2311_06837_b200.device import stream_handle
    buf = torch.randn(60 * 262144, device=dev)
    sink = torch.zeros(4, device=dev)
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call("gdx_probe_bandwidth", buf.data_ptr(), buf.numel() * 4, 40, 0, sink.data_ptr(), stream_handle())
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 40 * buf.numel() * 4 / e0.elapsed_time(e1) / 1e6)
    return best


def load_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    try:
        with open(os.path.join(HERE, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get("aggregate_dram_bytes_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------------------------
def run_reference(args, world, rank):
    if rank != 0:
        return
    steps, warmup = max(1, args.steps), max(0, args.warmup)
    # keep the whole reference run within a few minutes: 1 warm-up sample at most
    rec = cpu_baseline_record(args, steps=min(steps, 3), warmup=min(warmup, 1))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": rec["value"], "unit": "ms",
        "n_gpus": args.gpus, "steps": min(steps, 3), "warmup": min(warmup, 1),
        "ms_per_step": rec["value"], "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "reddit-shape full-graph 3-layer GraphSAGE epoch (configs[1])",
                   "vertices": args.n, "avg_degree": args.degree, "dims": REDDIT["dims"],
                   "parallelism": "cpu"},
        "cpu_baseline": rec,
        "e2e": {"value": rec["value"], "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cobatch_cpu_baseline(tr, plan) -> dict:
    """The oracle port's fp64 masked epoch on batch 0's local graph (the same rows,
    levels and loss rows as the GPU step), timed once and scaled by the batch count."""
    import torch
    import oracle as O

    geo = tr.geoms[0]
    threads = os.cpu_count() or 1
    lp = geo.csr.row_ptr.cpu().numpy().astype(np.uint64)
    lc = geo.csr.col[:max(geo.nnz, 1)].cpu().numpy().view(np.uint32)[:geo.nnz]
    csr = O.CSR(geo.nloc, lp, lc)
    idx = geo.l2g.long()
    ld = tr.Xall.ld

    def plane(t):
        return (t.view(-1, ld)[idx, :tr.F].to(torch.int32).bitwise_left_shift(16).view(torch.float32))
    x = (plane(tr.Xall.hi) + plane(tr.Xall.lo)).double().cpu().numpy()
    lab = tr.labels_all[idx].cpu().numpy()
    model = O.Model({"sage": O.SAGE, "gcn": O.GCN, "sum": O.SUM}[tr.cfg.kind], tr.cfg.dims)
    w = np.random.default_rng(0).uniform(-0.5, 0.5, model.weight_count())
    t = time.perf_counter()
    O.train_epoch_masked(csr, x, lab, model, w, 0.1, geo.loss_rows, float(geo.loss_count),
                         nthreads=threads, layer_rows=list(geo.rows_out))
    sec = time.perf_counter() - t
    R = len(plan.batches)
    return {"value": round(sec * 1e3 * R, 1), "unit": "ms", "cores": threads, "kind": "port",
            "sample": (f"oracle port (fp64, OpenMP {threads} threads): the SGD step of batch 0 "
                       f"({geo.nloc} rows, {geo.nnz} local edges) in {sec:.2f} s, x{R} batches "
                       f"to an epoch")}


def run_cobatch(args, C, world, rank, local, dev, pg):
    """configs[4]: cooperative-batching epochs (R batches, one SGD step each)."""
    import torch
    import torch.distributed as dist

    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200 import _lib
    from paper_2311_06837_b200.cobatch import CobatchTrainer
    from paper_2311_06837_b200.graph import Partition
    from paper_2311_06837_b200.train import ModelConfig

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    R = args.batches or C["batches"]
    dims = list(C["dims"])
    L = len(dims) - 1
    t0 = time.perf_counter()
    g = G.gen_random_graph(args.n, args.degree, C["seed"])
    n = g.num_vertices()
    t_gen = time.perf_counter() - t0
    # one server holding every vertex; its GPUs by partition_random with the
    # hierarchical_partition(g, 1, world, "random", 4) seed (partition.cpp:226-259)
    sp = Partition(np.zeros(n, np.uint32), 1)
    ga = np.zeros(n, np.uint32)
    _lib.call("gdx_host_partition_random", n, world, G.mix64(4 ^ 1), ga.ctypes.data)
    gp = Partition(ga, world)
    m, k, sseed = C["eas"]
    scfg = G.SamplingConfig(m, k, sseed)
    t0 = time.perf_counter()
    sub = G.extract_sampled(g, sp, 0, scfg)
    plan = G.plan_cobatch_fixed_r(sub, g, L, scfg, R, G.ModelSpec(L, dims[1], dims[0]),
                                  target_split="random")
    t_plan = time.perf_counter() - t0
    cfg = ModelConfig(C["kind"], dims, lr=C["lr"])
    t0 = time.perf_counter()
    tr = CobatchTrainer(g, cfg, plan, sp, gp, 0, rank=rank, world=world, pg=pg)
    t_geo = time.perf_counter() - t0
    del sub
    for _ in range(max(args.warmup, 3)):
        tr.train_epoch(sync_loss=False)
    barrier()
    tr.enable_kernel_events(True)
    tr.train_epoch(sync_loss=False)
    barrier()
    agg_ms_epoch, agg_launches, agg_bytes = tr.kernel_event_summary()
    tr.enable_kernel_events(False)
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            tr.train_epoch(sync_loss=False)
        e1.record()
        barrier()
    launches = _lib.launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    loss = tr.train_epoch(sync_loss=True)
    t_ms = torch.tensor([ms, agg_ms_epoch], dtype=torch.float64, device=dev)
    ed = torch.tensor([float(sum(geo.edges_per_step for geo in tr.geoms))], dtype=torch.float64,
                      device=dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(ed)
    ms, agg_ms = float(t_ms[0]), float(t_ms[1])
    edges_epoch = float(ed[0])
    peak, peak_kind = load_peaks()
    agg_avg_ms = agg_ms_epoch / agg_launches if agg_launches else None
    achieved = (agg_bytes / agg_launches) / (agg_avg_ms * 1e-3) / 1e9 if agg_launches else None
    rows = [geo.nloc for geo in tr.geoms]
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cobatch_cpu_baseline(tr, plan)
        out = {
            "metric": METRIC, "value": round(ms, 3), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 3),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 (tcgen05 GEMMs: bf16x3 split, fp32 accumulate)",
            "data": f"synthetic: gen_random_graph({n}, {args.degree}, {C['seed']}) papers-shape "
                    f"G(n,p), features/labels from the reference keyed RNG streams",
            "config": {"workload": C["workload"], "name": args.config,
                       "model": f"{cfg.kind} {'-'.join(map(str, dims))} ({L} layers), no bias, "
                                f"SGD lr {cfg.lr}, one step per batch",
                       "vertices": n, "directed_edges": g.num_edges(), "batches": R,
                       "target_split": "split_targets_random (host min-cut of 111 M vertices "
                                       "replaced; structure-free graph)",
                       "batch_rows_per_rank": {"max": max(rows), "mean": int(np.mean(rows))},
                       "global_batch": int(n / R),
                       "parallelism": f"cooperative batch split x{world} (split_batch), "
                                      f"per-layer NVLink row push inside the batch",
                       "l2": "no flush: every batch streams its CSR and > 1 GB of rows"},
            "epoch_ms": round(ms, 3),
            "aggregation_edges_per_s": round(edges_epoch / (agg_ms * 1e-3), 1) if agg_ms else None,
            "epoch_edges_per_s": round(edges_epoch / (ms * 1e-3), 1),
            "loss_after": round(loss, 6),
            "roofline": {
                "bound": "hbm", "kernel": "gdx aggregate_vec4 (K1/K3 gather-reduce)",
                "achieved": round(achieved, 1) if achieved else None, "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4) if achieved else None, "traffic": None,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "algorithmic_bytes_per_launch": int(agg_bytes / agg_launches) if agg_launches else None,
                "avg_launch_ms": round(agg_avg_ms, 4) if agg_avg_ms else None,
                "share_of_step": round(agg_ms / ms, 3) if ms else None},
            "gpu_launches": int(launches / max(args.steps, 1)),
            "cuda_graph": False,
            "clocks": clk.summary(),
            "e2e": None,
            "e2e_note": "not measured for this config: host-side features would be 57 GB",
            "cpu_baseline": cpu,
            "setup_s": {"graph_generation": round(t_gen, 2), "plan": round(t_plan, 2),
                        "batch_geometry": round(t_geo, 2)},
        }
        print(json.dumps(out), flush=True)
    barrier()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    C = CONFIGS[args.config]
    args.n = args.n or C["n"]
    args.degree = args.degree or C["degree"]
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        bind_numa(local)
    pg = None
    if world > 1:
        opts = dist.ProcessGroupNCCL.Options()
        opts.is_high_priority_stream = True  # collectives get SMs ahead of the aggregation
        dist.init_process_group("nccl", device_id=dev, pg_options=opts)
        pg = dist.group.WORLD

    if C["mode"] == "cobatch":
        run_cobatch(args, C, world, rank, local, dev, pg)
        return

    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200 import _lib
    from paper_2311_06837_b200.train import FullGraphTrainer, ModelConfig

    t0 = time.perf_counter()
    g = G.gen_random_graph(args.n, args.degree, C["seed"])
    t_gen = time.perf_counter() - t0
    cfg = ModelConfig(C["kind"], list(C["dims"]), lr=C["lr"])
    sub = None
    if C["mode"] == "eas":
        m, k, sseed = C["eas"]
        part = G.partition_random(g, world, 1)
        sub = G.extract_sampled(g, part, rank, G.SamplingConfig(m, k, sseed))
    tr = FullGraphTrainer(g, cfg, rank=rank, world=world, pg=pg, subgraph=sub)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        tr.train_epoch(sync_loss=False)
    barrier()

    # ---- kernel-level roofline: the aggregation launches of K eager epochs, timed
    # with CUDA events on the launching stream ----
    tr.enable_kernel_events(True)
    barrier()
    for _ in range(args.steps):
        tr.train_epoch(sync_loss=False)
    barrier()
    agg_ms_total, agg_launches, agg_bytes = tr.kernel_event_summary()
    tr.enable_kernel_events(False)
    eager_epoch_events = None

    # ---- timed region: K epochs (CUDA-graph replays unless --eager) ----
    use_graph = not args.eager
    if use_graph:
        tr.capture(warmup=1)
        for _ in range(2):
            tr.replay()
    step = tr.replay if use_graph else (lambda: tr.train_epoch(sync_loss=False))
    barrier()
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        barrier()
    launches = _lib.launch_count() - launches0
    if use_graph:
        launches = launches_per_epoch(tr) * args.steps
    ms = e0.elapsed_time(e1) / args.steps
    loss = tr.train_epoch(sync_loss=True)

    t_ms = torch.tensor([ms, agg_ms_total / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms, agg_ms_step = float(t_ms[0]), float(t_ms[1])

    # ---- e2e through the public API: every step copies its feature block and labels
    # host -> device (pinned) and reads its loss back; the copy of step i+1 overlaps the
    # compute of step i (FeatureStream double buffering) ----
    e2e = None
    if not args.no_e2e:
        from paper_2311_06837_b200.train import FeatureStream
        xh = torch.empty((tr.nloc, tr.F), dtype=torch.float32).pin_memory()
        xh.copy_(tr.X[:tr.nloc, :tr.F].cpu())
        lh = tr.labels[:tr.nloc].cpu().pin_memory()
        loss_h = torch.zeros(1, dtype=torch.float64).pin_memory()
        fs = FeatureStream(tr)
        barrier()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        fs.prefetch(xh, lh)
        for i in range(args.steps):
            if i + 1 < args.steps:
                fs.prefetch(xh, lh)
            fs.consume()
            if use_graph:
                tr.replay()
            else:
                tr.train_epoch(sync_loss=False)
            loss_h.copy_(tr.loss_acc, non_blocking=True)
            done = torch.cuda.Event()
            done.record()
            done.synchronize()  # the step's loss is on the host before the next step
        s1.record()
        barrier()
        e2e_ms = torch.tensor([s0.elapsed_time(s1) / args.steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e = {"value": round(float(e2e_ms[0]), 3), "unit": "ms",
               "h2d_bytes_per_step": int(xh.numel() * 4 + lh.numel() * 4) * world,
               "d2h_bytes_per_step": 8 * world,
               "pipelining": "step i+1's feature H2D overlaps step i's compute (double buffer)",
               "h2d_ms_per_step": round(fs.copy_ms(), 3)}

    l2_peak = probe_l2_peak(torch, dev)
    edges_total = g.num_edges()
    # edges aggregated per epoch over all ranks (forward + backward passes)
    ed = torch.tensor([float(tr.nnz_local)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ed)
    agg_edges_epoch = 2 * cfg.layers * float(ed[0])
    peak, peak_kind = load_peaks()
    agg_avg_ms = (agg_ms_total / agg_launches) if agg_launches else None
    achieved = (agg_bytes / agg_launches) / (agg_avg_ms * 1e-3) / 1e9 if agg_launches else None

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline and args.config == "reddit-sage":
            cpu = cpu_baseline_record(args)
        clocks = clk.summary()
        out = {
            "metric": METRIC,
            "value": round(ms, 3),
            "unit": "ms",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms, 3),
            "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32 (tcgen05 GEMMs: bf16x3 split, fp32 accumulate)",
            "data": "synthetic: gen_random_graph(232965, 491.99, 11) Reddit-shape G(n,p), "
                    "features/weights/labels from the reference keyed RNG streams",
            "config": {"workload": C["workload"], "name": args.config,
                       "model": f"{cfg.kind} {'-'.join(map(str, cfg.dims[:3]))}...{cfg.dims[-1]} "
                                f"({cfg.layers} layers), no bias, SGD lr {cfg.lr}",
                       "vertices": args.n, "directed_edges": edges_total, "global_batch": args.n,
                       "parallelism": f"row-partition x{world} (all-gather per layer, NCCL)",
                       "l2": "no flush: each epoch streams >1 GB (CSR cols 458 MB + features 567 MB) "
                             "through a 126 MB L2"},
            "epoch_ms": round(ms, 3),
            "aggregation_edges_per_s": round(agg_edges_epoch / (agg_ms_step * 1e-3), 1) if agg_ms_step else None,
            "epoch_edges_per_s": round(agg_edges_epoch / (ms * 1e-3), 1),
            "loss_after": round(loss, 6),
            "roofline": {
                "bound": "hbm",
                "kernel": "gdx aggregate_vec4 (K1/K3 gather-reduce, 64/44-wide rows)",
                "achieved": round(achieved, 1) if achieved else None,
                "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4) if achieved else None,
                "traffic": load_traffic(),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                "algorithmic_bytes_per_launch": int(agg_bytes / agg_launches) if agg_launches else None,
                "avg_launch_ms": round(agg_avg_ms, 4) if agg_avg_ms else None,
                "share_of_step": round(agg_ms_step / ms, 3) if ms else None,
                "note": "bytes = 4 nnz + 8 (rows+1) + 4 F nnz + 4 F rows per launch (SURVEY §8d); "
                        "the gathered 64-wide rows (60 MB) are L2-resident, so achieved exceeds HBM: "
                        "see l2 for the binding roofline",
                "l2": {"achieved": round(achieved, 1) if achieved else None,
                       "peak": round(l2_peak, 1), "unit": "GB/s",
                       "frac": round(achieved / l2_peak, 4) if achieved else None,
                       "peak_source": "live probe: gdx_probe_bandwidth coalesced stream over a "
                                      "60 MB L2-resident buffer (best of 4)"},
            },
            "gpu_launches": int(launches),
            "cuda_graph": use_graph,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "setup_s": {"graph_generation": round(t_gen, 2)},
        }
        print(json.dumps(out), flush=True)
    # release the captured graph (it references the NCCL communicator) before teardown
    tr.graph = None
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
