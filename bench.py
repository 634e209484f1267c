#!/usr/bin/env python
"""Bench: candidate schedules rounded + evaluated per second (BASELINE.json metric).

A step = one pass of the whole hot path (a1-a7 of SURVEY §8(a), plus the a8 MIN all-reduce
of the keys at N>1) over one batch of synthetic, device-resident S*.
Default workload: the ResNet-50-shaped training DAG (n=353, |E|=560), G1 LP-like S*,
theta = 0.5, 16 budgets, 125,000 S* per GPU per step (the 10^6-candidate config sharded
over 8 GPUs; weak scaling).  Default S* layout: blocked strict lower triangle (CM_LAYOUT_BLK,
250.6 KB per S*, 0.85 % over the triangle: 31.3 GB per GPU; --layout dense: 128-byte rows,
67.8 GB), far above L2 (126 MB), so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

At N>1 each rank evaluates its own contiguous S* range (global index_base) and step i's keys
are MIN-reduced on a side stream that waits for call i through the library's device-side
completion word (cm_stream_wait_call), so the reduction never stalls call i+1's overlap with
call i.  CM_DIST_BACKEND=gloo (default nccl) and ranks sharing a GPU (LOCAL_RANK modulo the
device count) exercise that path on one GPU.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate schedules rounded+evaluated/sec at n≈350, 1/2/4/8 B200; % HBM roofline"
UNIT = "candidates/s"
BENCH_SEED = 20250101

CONFIGS = {
    # name: (graph builder, family, thetas, budget rule, S* per GPU per step)
    "resnet50": ("resnet50", "g1", [0.5], "grid16", 125000),
    "vgg16": ("vgg16", "g1", [0.5], "grid16", 100000),
    "unet": ("unet", "g1", [0.5], "unet", 125000),
    "mobilenet": ("mobilenet", "g1", [0.5], "grid16", 125000),
    "fcn8": ("fcn8", "g1", [0.5], "grid16", 62500),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="resnet50", choices=sorted(CONFIGS))
    ap.add_argument("--family", default=None)
    ap.add_argument("--thetas", default=None,
                    help="comma-separated thresholds (deterministic rounding, N_theta <= 4 per pass) "
                         "instead of the config's")
    ap.add_argument("--max-batch", action="store_true",
                    help="also run the max-batch epilogue (Eq. 13) per budget in the timed step")
    ap.add_argument("--samples", type=int, default=None,
                    help="randomized rounding (DESIGN.md R1) with this many samples per S* instead of the thresholds")
    ap.add_argument("--batch", type=int, default=None, help="S* per GPU per step")
    ap.add_argument("--layout", default="blk", choices=["tri4", "dense", "blk"])
    ap.add_argument("--ld", type=int, default=None,
                    help="dense row stride in floats (default: n rounded up to 32, i.e. 128-byte rows)")
    ap.add_argument("--overlap", default="on", choices=["on", "off"],
                    help="consecutive steps' calls with CM_EVAL_OVERLAP | CM_EVAL_INIT_KEYS on two "
                         "alternating output sets (a call starts while the previous one drains)")
    ap.add_argument("--step-events", action="store_true",
                    help="with --overlap on: also record CUDA events around every call")
    ap.add_argument("--keys", default="nccl", choices=["nccl", "nvls"],
                    help="a8 at N>1: NCCL MIN all-reduce of each call's keys on a side stream (default), "
                         "or nvls: multimem.red.min into an NVLink multicast buffer inside the reduce step "
                         "(dist.MulticastKeys; also runs at N=1 on a one-device multicast object)")
    ap.add_argument("--e2e-batch", type=int, default=16384)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def build_workload(cfg, family=None):
    from workloads import budgets as B
    from workloads import graphs as G
    gname, fam, thetas, rule, batch = CONFIGS[cfg]
    g = G.NETWORKS[gname]()
    if rule == "unet":
        budgets = B.unet_grid(g)
        g = g.scaled(5)
    else:
        budgets = B.geometric_grid(g, 16)
    return g, (family or fam), thetas, budgets, batch


def tri_bytes(n):
    return 4 * n * (n - 1) // 2


def load_peaks():
    """HBM peak (GB/s) from the driver-written MEASURED_PEAKS.json: the sustained copy figure
    when the file has one (the fused kernel runs ~7 ms inside a step), else its plain / burst
    HBM figure; the profiling guide's fallback 6650 GB/s when the file is absent."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
        except Exception:
            d = {}
        flat = {}

        def walk(prefix, v):
            if isinstance(v, dict):
                for k, x in v.items():
                    walk(f"{prefix}.{k}" if prefix else str(k), x)
            elif isinstance(v, (int, float)):
                flat[prefix.lower()] = float(v)
        walk("", d)
        hbm = {k: v for k, v in flat.items() if "hbm" in k and ("gb" in k or "tb" in k or k.endswith("hbm"))}
        for pref in ("sustained", "sust", ""):
            for k, v in sorted(hbm.items()):
                if pref in k and "burst" not in k or (pref == "" and k == "hbm_gbs"):
                    val = v * 1000.0 if "tb" in k else v
                    return val, f"measured ({k})"
        if "hbm_gbs" in flat:
            return flat["hbm_gbs"], "measured (hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(cfg, layout, batch):
    """DRAM bytes (read + write) of one launch, from the committed ncu --set full capture
    (profiles/traffic.json[cfg]["layouts"][layout]: bytes per S* of the fused kernel, written by
    tools/traffic_from_ncu.py), scaled to the batch; None when that layout was not captured."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p)).get(cfg, {}).get("layouts", {}).get(layout)
        if d:
            return d["dram_bytes_per_sstar"] * batch, d["source"]
    return None, None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons DURING the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for nm, v in zip(names, r[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle legs

def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _oracle_worker(args):
    fam, seed, s_list, thetas, cfg = args
    from oracle import Instance, evaluate
    from workloads.sstar import gen_sstar
    g, _, _, _, _ = build_workload(cfg, fam)
    inst = Instance.from_graph(g)
    xs = [gen_sstar(g, fam, seed, s, 1)[0] for s in s_list]
    counters = []
    t0 = time.perf_counter()
    for x in xs:
        for th in thetas:
            counters.append(evaluate(inst, x, th)["counters"])
    return time.perf_counter() - t0, len(xs) * len(thetas), counters


def ops_alg_of(n, counters):
    """SURVEY §8(d) algorithmic integer ops per candidate: tri + n W + V + F + sum R + sum S,
    from the oracle's A8 counters (mean over the sample)."""
    tri, W = n * (n - 1) // 2, (n + 63) // 64
    per = [tri + n * W + c["closure_visits"] + c["free_events"] + c["sum_R"] + c["sum_S"] for c in counters]
    return float(np.mean(per))


def cpu_oracle_rate(cfg, fam, seed, thetas, seconds):
    """The oracle as it stands on this host's cores (multiprocessing), bounded sample; also the
    1-core rate and the A8 counters of the sampled candidates (the INT roofline's Ops_alg)."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    dt, cnt, c0 = _oracle_worker((fam, seed, [0], thetas, cfg))          # calibrate one S* on one core
    per = dt / cnt
    per_core = max(1, int(seconds / per / len(thetas)))
    jobs = [(fam, seed, list(range(1 + c * per_core, 1 + (c + 1) * per_core)), thetas, cfg) for c in range(cores)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_oracle_worker, jobs)
    wall = time.perf_counter() - t0
    total = sum(r[1] for r in res)
    busy = max(r[0] for r in res)
    one = sum(r[1] for r in res) / sum(r[0] for r in res)               # per-process rate, averaged
    counters = c0 + [c for r in res for c in r[2]]
    return {"value": total / busy, "unit": UNIT, "cores": cores, "kind": "oracle",
            "one_core_value": one, "cpu_model": cpu_model(),
            "sample": f"{total} candidates (S* #1..{cores * per_core}, {fam}, theta={thetas}) of the "
                      f"{cfg} workload on {cores} processes; {wall:.1f}s wall incl. pool start"}, counters


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    g, fam, thetas, budgets, batch = build_workload(a.config, a.family)
    if a.thetas:
        thetas = [float(t) for t in a.thetas.split(",")]
    from oracle import Instance, evaluate
    from workloads.sstar import gen_sstar
    inst = Instance.from_graph(g)
    per_step = 8
    xs = [gen_sstar(g, fam, 7, s, 1)[0] for s in range(per_step)]
    for _ in range(a.warmup):
        evaluate(inst, xs[0], thetas[0])
    t0 = time.perf_counter()
    cnt = 0
    for _ in range(a.steps):
        for x in xs:
            for th in thetas:
                evaluate(inst, x, th)
                cnt += 1
    dt = time.perf_counter() - t0
    v = cnt / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1000 * dt / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": f"{a.config} n={g.n} |E|={len(g.edges)} {fam} S*, theta={thetas}, "
                                   f"{len(budgets)} budgets", "global_batch": per_step * len(thetas)},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"{per_step} S* x {len(thetas)} theta per step, 1 process"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def load_ops_alg(cfg, fam):
    """Committed fallback for Ops_alg (profiles/ops_alg.json, written by tools/ops_alg.py from
    the oracle's counters) when the CPU leg is skipped."""
    p = os.path.join(ROOT, "profiles", "ops_alg.json")
    if os.path.exists(p):
        d = json.load(open(p)).get(cfg, {}).get(fam)
        if d:
            return d["ops_alg_per_candidate"], "profiles/ops_alg.json (" + d["sample"] + ")"
    return None, None


# ----------------------------------------------------------------------------- GPU leg

def main():
    a = parse()
    if a.impl == "reference":
        return run_reference(a)
    import torch
    import torch.distributed as dist

    import paper_1910_02653_b200 as cm
    from workloads.device_gen import DeviceGenerator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = max(1, torch.cuda.device_count())
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    backend = os.environ.get("CM_DIST_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    g, fam, thetas, budgets, batch = build_workload(a.config, a.family)
    if a.thetas:
        thetas = [float(t) for t in a.thetas.split(",")]
    if a.batch:
        batch = a.batch
    seed = BENCH_SEED
    n_theta = a.samples if a.samples else len(thetas)
    graph = cm.Graph.from_workload(g)
    ld = a.ld if a.ld else (-(-g.n // 32) * 32 if a.layout == "dense" else None)
    gen = DeviceGenerator(g, fam, seed, layout=a.layout, ld=ld)
    sstar = torch.empty(gen.shape(batch), dtype=torch.float32, device=dev)
    s_base = rank * batch
    gen.fill(sstar, s_base)
    th = torch.tensor(thetas, dtype=torch.float32, device=dev)
    bu = torch.tensor(budgets, dtype=torch.int64, device=dev)
    overlap = a.overlap == "on"
    n_sets = 2 if overlap else 1                     # overlapped calls alternate two output sets
    n_calls = max(a.warmup, 3) + a.steps + 8
    # one key vector per call (tiny): call i's keys may still be in the MIN all-reduce on the side
    # stream while calls i+1, i+2 run, so no call reuses another's keys
    nvls = a.keys == "nvls"
    mkeys = mbkeys = None
    if nvls:
        # a8 inside the kernel: every call has its own slot of a multicast buffer, set to
        # CM_KEY_NONE once on every rank before any call (no per-call init, no all-reduce)
        from paper_1910_02653_b200.dist import MulticastKeys
        mkeys = MulticastKeys(n_calls * len(budgets))
        keys = mkeys.local.view(n_calls, len(budgets))
        mkeys.reset()
        if a.max_batch:
            mbkeys = MulticastKeys(n_calls * len(budgets))
            mbkeys.reset()
        bkeys = mbkeys.local.view(n_calls, len(budgets)) if mbkeys else None
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    else:
        keys = torch.empty((n_calls, len(budgets)), dtype=torch.int64, device=dev)
        bkeys = torch.empty((n_calls, len(budgets)), dtype=torch.int64, device=dev) if a.max_batch else None
    from workloads.budgets import eq13_cost_limit
    limit = eq13_cost_limit(g) if a.max_batch else None
    peaks = [torch.empty(batch * n_theta, dtype=torch.int64, device=dev) for _ in range(n_sets)]
    costs = [torch.empty(batch * n_theta, dtype=torch.int64, device=dev) for _ in range(n_sets)]
    calls = [0]
    events = not overlap or a.step_events
    total = world * batch * n_theta
    stream = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)
    works = []
    k_start = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    k_end = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]

    def step(i=None, ovl=overlap):
        c = calls[0]
        calls[0] += 1
        h = c % n_sets
        key, bkey = keys[c % n_calls], (bkeys[c % n_calls] if bkeys is not None else None)
        if not ovl and not nvls:
            key.fill_(cm.CM_KEY_NONE)
            if bkey is not None:
                bkey.fill_(cm.CM_KEY_NONE)
        if i is not None and events:
            k_start[i].record(stream)
        slot = 8 * len(budgets) * (c % n_calls)
        cm.round_and_evaluate(graph, sstar, None if a.samples else th, bu, layout=a.layout,
                              index_base=s_base * n_theta, total_candidates=total, best_key=key,
                              peak=peaks[h], cost=costs[h], stream=stream.cuda_stream, samples=a.samples,
                              seed=seed, cost_limit=limit, best_batch_key=bkey,
                              init_keys=ovl and not nvls, overlap=ovl,
                              best_key_mc=mkeys.mc + slot if nvls else None,
                              best_batch_key_mc=mbkeys.mc + slot if mbkeys else None)
        if i is not None and events:
            k_end[i].record(stream)
        if world > 1 and not nvls:
            # a8: MIN all-reduce of this call's keys on the side stream, which waits for the call
            # through the library's device-side completion word -- nothing is enqueued on `stream`
            cm.stream_wait_call(graph, cm.last_call_seq(graph), side.cuda_stream)
            with torch.cuda.stream(side):
                works.append(dist.all_reduce(key, op=dist.ReduceOp.MIN, async_op=True))
                if bkey is not None:
                    works.append(dist.all_reduce(bkey, op=dist.ReduceOp.MIN, async_op=True))
        return key

    def drain():
        while works:
            works.pop(0).wait()                      # `stream` waits for the reductions

    for _ in range(max(a.warmup, 3)):
        step()
    drain()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(dev.index) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0.record(stream)
    for i in range(a.steps):
        last_key = step(i)
    drain()
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    elapsed_ms = t0.elapsed_time(t1)
    # per-call device time; overlapped calls (no events between them) -> the per-step time
    kern_ms = (float(np.mean([s.elapsed_time(e) for s, e in zip(k_start, k_end)])) if events
               else elapsed_ms / a.steps)
    # isolated launch: serial calls (keys filled first, no overlap), CUDA events on `stream`
    iso = []
    iso_key = torch.empty(len(budgets), dtype=torch.int64, device=dev)
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iso_key.fill_(cm.CM_KEY_NONE)
        e0.record(stream)
        cm.round_and_evaluate(graph, sstar, None if a.samples else th, bu, layout=a.layout,
                              index_base=s_base * n_theta, total_candidates=total, best_key=iso_key,
                              peak=peaks[0], cost=costs[0], stream=stream.cuda_stream, samples=a.samples, seed=seed)
        e1.record(stream)
        torch.cuda.synchronize()
        iso.append(e0.elapsed_time(e1))
    iso_ms = float(np.median(iso))
    if world > 1:
        t = torch.tensor([elapsed_ms, kern_ms, iso_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, kern_ms, iso_ms = float(t[0]), float(t[1]), float(t[2])
    best = last_key.cpu().tolist()

    # one extra traced step (untimed, every rank: it joins the collective): the fused path
    # records its single launch; the two-kernel pipeline records per chunk K1 and K2+K3
    kernels = None
    launches = None
    try:
        os.environ["CM_TRACE"] = "1"
        step()
        drain()
        torch.cuda.synchronize()
        tr = cm.debug_trace()
        per_step = cm.debug_last_launches()
        os.environ["CM_TRACE"] = "0"
        launches = a.steps * per_step
        span = max(t[3] for t in tr) - min(t[0] for t in tr)
        if per_step == 1:
            kernels = {"path": "fused persistent kernel (K1 rounding warps + K2 scan warps per CTA, "
                               "L2 ring handoff, K3 reduce in the K2 warps)", "fused_ms": span}
        else:
            k1 = sum(t[1] - t[0] for t in tr)
            k2 = sum(t[3] - t[2] for t in tr)
            kernels = {"path": "two-kernel pipeline", "chunks": len(tr), "k1_round_ms": k1,
                       "k2_scan_reduce_ms": k2, "span_ms": span,
                       "overlap": "K1(chunk c+1) runs on an internal stream concurrently with K2(chunk c)"}
    except Exception as ex:  # pragma: no cover
        kernels = {"error": str(ex)}

    # ---- e2e through the public API with HOST buffers (rank-local, then the same MIN) ----
    e2e = None
    if not a.no_e2e and not a.samples:
        # e2e through the public API: pinned HOST buffers in a packed triangle layout (the
        # timed run's blocked layout, or tri4 when that one is dense: half the PCIe bytes of
        # dense); H2D copies, kernels and D2H of peak/cost/keys all timed.
        eb = min(a.e2e_batch, batch)
        elay = a.layout if a.layout in ("blk", "tri4") else "tri4"
        egen = DeviceGenerator(g, fam, seed, layout=elay)
        staging = torch.empty(egen.shape(eb), dtype=torch.float32, device=dev)
        egen.fill(staging, s_base)
        host = torch.empty((eb, egen.stride), dtype=torch.float32, pin_memory=True)
        host.copy_(staging.view(eb, -1))
        del staging
        pipe = cm.HostPipeline(graph, egen.stride, chunk=2048, n_theta=n_theta, n_budget=len(budgets),
                               layout=elay, device=dev)
        pipe.run(host, th, bu, index_base=rank * eb * n_theta, total_candidates=world * eb * n_theta)
        torch.cuda.synchronize()
        e_steps = max(1, min(a.steps, 5))
        if world > 1:
            dist.barrier()
        te = time.perf_counter()
        for _ in range(e_steps):
            _, _, kk = pipe.run(host, th, bu, index_base=rank * eb * n_theta,
                                total_candidates=world * eb * n_theta)
            if world > 1:
                kd = kk.to(dev)
                dist.all_reduce(kd, op=dist.ReduceOp.MIN)
                kk = kd.cpu()
        e_dt = time.perf_counter() - te
        if world > 1:
            t = torch.tensor([e_dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_dt = float(t[0])
        e2e = {"value": world * eb * n_theta * e_steps / e_dt, "unit": UNIT,
               "h2d_bytes_per_step": eb * egen.stride * 4,
               "d2h_bytes_per_step": eb * n_theta * 16 + 8 * len(budgets),
               "batch_per_gpu": eb, "host_memory": "pinned", "layout": elay,
               "h2d_gb_per_s": eb * egen.stride * 4 * e_steps / e_dt / 1e9,
               "note": "PCIe-bound: the S* bytes cross the host link every step"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    cand_per_step = world * batch * n_theta
    value = cand_per_step * a.steps / (elapsed_ms / 1000.0)
    peak_gbs, peak_src = load_peaks()
    alg_bytes = batch * tri_bytes(g.n) + batch * n_theta * 16 + 8 * len(budgets)
    path_ms = kern_ms                     # per-call device time (events around each launch, or the
                                          # per-step time when consecutive calls overlap)
    achieved = alg_bytes / (path_ms / 1000.0) / 1e9
    traffic, traffic_src = load_traffic(a.config, a.layout, batch)
    # ---- integer-pipe term (K-mu): measured INT peak, Ops_alg from the oracle's A8 counters ----
    ipk = None
    try:
        from tools.int_peak import measure as int_peak_measure
        ipk = int_peak_measure()
    except Exception as ex:  # pragma: no cover
        ipk = {"error": str(ex)}
    cpu, counters = None, None
    if not a.no_cpu_baseline and world == 1 and not a.samples:
        cpu, counters = cpu_oracle_rate(a.config, fam, seed, thetas, a.cpu_seconds)
    if counters:
        ops_pc, ops_src = ops_alg_of(g.n, counters), f"oracle A8 counters of the cpu_baseline sample ({len(counters)} candidates)"
    elif a.samples:
        # the randomized candidates' own phase-2 counters (their S differ from the rounded ones:
        # about twice the closure, frees and recomputes of G1 at theta 0.5)
        ops_pc, ops_src = load_ops_alg(a.config, "rand_" + fam)
        if ops_pc is None:
            ops_pc, ops_src = load_ops_alg(a.config, fam)
    else:
        ops_pc, ops_src = load_ops_alg(a.config, fam)
    if a.samples:
        # randomized rounding adds the generator's integer work per stored element and sample:
        # 10 rounds x (4 multiplies, 4 xors, 2 key adds) per Philox block = 100, one block per
        # four (node, sample) uniforms (R1), plus scale / convert / compare (4): 29
        ops_pc = (ops_pc or 0.0) + 29.0 * (g.n * (g.n - 1) // 2)
    int_term = None
    if ops_pc and ipk and "int_peak_tops" in ipk:
        ops_rate = ops_pc * batch * n_theta / (path_ms / 1000.0)
        int_term = {"achieved": ops_rate / 1e12, "peak": ipk["int_peak_tops"], "unit": "T int lane-ops/s",
                    "frac": ops_rate / 1e12 / ipk["int_peak_tops"], "ops_alg_per_candidate": ops_pc,
                    "ops_alg_source": ops_src,
                    "peak_source": "measured live: tools/int_peak.py lop3+imad (alu + fma pipes) at %.0f MHz; "
                                   "alu pipe alone %.2f T/s" % (ipk["classes"]["lop3+imad"]["sm_mhz"], ipk["alu_tops"])}
    hbm_term = {"achieved": achieved, "peak": peak_gbs, "unit": "GB/s", "frac": achieved / peak_gbs}
    binds = "int" if int_term and int_term["frac"] > hbm_term["frac"] else "hbm"
    roof = {"bound": "alu" if binds == "int" else "hbm",
            "achieved": int_term["achieved"] if binds == "int" else achieved,
            "peak": int_term["peak"] if binds == "int" else peak_gbs,
            "unit": int_term["unit"] if binds == "int" else "GB/s",
            "frac": int_term["frac"] if binds == "int" else achieved / peak_gbs,
            "traffic": traffic,
            "traffic_source": ("profiles/traffic.json (DRAM bytes read + write per S* x batch; " + traffic_src +
                               "); not measured in this run") if traffic_src else "no capture of this layout",
            "terms": {"hbm": hbm_term, "int": int_term},
            "binds": binds,
            "kernel": "cm2::fused_kernel: the whole a1-a7 path in one launch per step (" +
                      ("CUDA events around each call on the launching stream" if events else
                       "consecutive launches overlap (CM_EVAL_OVERLAP): timed region / steps") + ")",
            "alg_bytes_per_launch": alg_bytes, "ms_per_launch": path_ms,
            "isolated_launch_ms": iso_ms,
            "isolated_frac": alg_bytes / (iso_ms / 1000.0) / 1e9 / peak_gbs,
            "kernels": kernels, "peak_source": peak_src, "int_peak": ipk}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": max(a.warmup, 3), "ms_per_step": elapsed_ms / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": f"{a.config}: n={g.n}, |E|={len(g.edges)}, {fam} LP-like S* "
                                   f"({a.layout} fp32), "
                                   + (f"randomized rounding, {a.samples} samples per S*" if a.samples
                                      else f"theta={thetas}") + f", {len(budgets)} budgets",
                       "global_batch": cand_per_step, "per_gpu_sstar": batch, "layout": a.layout,
                       "parallelism": (f"candidates sharded over {world} GPU(s) (a8: multimem.red.min of each "
                                       "call's keys into an NVLink multicast buffer inside the reduce step)"
                                       if nvls else
                                       f"candidates sharded over {world} GPU(s) ({backend if world > 1 else 'no'} "
                                       "MIN all-reduce of each step's keys on a side stream)"),
                       "l2": f"inputs {batch * gen.stride * 4 / 1e9:.1f} GB per GPU > 126 MB L2; no flush",
                       "calls": ("overlapped: CM_EVAL_OVERLAP" + ("" if nvls else " | CM_EVAL_INIT_KEYS")
                                 + ", two alternating output sets" if overlap
                                 else "serial: keys filled by the caller before each call")},
            "gpu_launches": launches, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks,
            "best": [cm.decode_key(k, cm.key_idx_bits(total)) for k in best]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
