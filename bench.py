#!/usr/bin/env python
"""bench.py -- malloc+free throughput of the B200 device allocator.

Metric (BASELINE.json): malloc+free ops/sec vs size (16 B-8 KiB, 1M threads);
% of L2-atomic roofline.

Default workload = BASELINE configs[1]: page allocator, standard (Array)
queues, 1 GiB heap, 2^20 device threads, size sweep 4 B ... 8 KiB (powers of
two plus the paper's 1000 B).  One *step* = one pass over the sweep: for each
size, 2^20 threads malloc (timed kernel), write + verify the pattern (checked,
not in the metric), free (timed kernel).  L2 is flushed (256 MiB write) before
every timed kernel.  value = successful malloc+free pairs / (sum of alloc +
free kernel time), device-timed with CUDA events, max over ranks for N>1
(weak scaling: every GPU owns an independent heap and the same per-GPU work).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config pq1g|cq64m|va8g|...]
  python bench.py --impl reference ...   # the reference CPU allocator (oracle port)
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

SWEEP = [4, 8, 16, 32, 64, 128, 256, 512, 1000, 1024, 2048, 4096, 8192]
CONFIGS = {
    # name: (description, kind, flavor, heap, threads, sizes)
    "cq64m": ("configs[0]: chunk allocator, Array queues, 64 MiB heap, 65536 threads x malloc(16)",
              1, 0, 64 << 20, 65536, [16]),
    "pq1g": ("configs[1]: page allocator (PQ), Array queues, 1 GiB heap, 1M threads, size sweep 4 B-8 KiB",
             0, 0, 1 << 30, 1 << 20, SWEEP),
    "vapq8g": ("configs[2]: VAPQ, 8 GiB heap, 1M threads, 16 B-8 KiB", 0, 1, 8 << 30, 1 << 20, SWEEP[2:]),
    "vacq8g": ("configs[2]: VACQ, 8 GiB heap, 1M threads, 16 B-8 KiB", 1, 1, 8 << 30, 1 << 20, SWEEP[2:]),
    "vlpq8g": ("configs[2]: VLPQ, 8 GiB heap, 1M threads, 16 B-8 KiB", 0, 2, 8 << 30, 1 << 20, SWEEP[2:]),
    "vlcq8g": ("configs[2]: VLCQ, 8 GiB heap, 1M threads, 16 B-8 KiB", 1, 2, 8 << 30, 1 << 20, SWEEP[2:]),
    "cq1g": ("chunk allocator (CQ), Array queues, 1 GiB heap, 1M threads, 16 B-8 KiB", 1, 0, 1 << 30, 1 << 20, SWEEP[2:]),
    "pq16g4m": ("configs[4] per GPU: PQ, 16 GiB heap, 4M threads, 16 B-1 KiB", 0, 0, 16 << 30, 1 << 22,
                [16, 32, 64, 128, 256, 512, 1000, 1024]),
    "cq16g4m": ("configs[4] per GPU: CQ, 16 GiB heap, 4M threads, 16 B-1 KiB", 1, 0, 16 << 30, 1 << 22,
                [16, 32, 64, 128, 256, 512, 1000, 1024]),
    # configs[3]: mixed churn; a step = 10 rounds, sizes 8 B-4 KiB drawn per (thread, round)
    "churn": ("configs[3]: mixed churn, CQ, 16 GiB heap, 4M threads, sizes 8 B-4 KiB, 10 rounds per step",
              1, 0, 16 << 30, 1 << 22, None),
    "churn-pq": ("configs[3]: mixed churn, PQ, 16 GiB heap, 4M threads, sizes 8 B-4 KiB, 10 rounds per step",
                 0, 0, 16 << 30, 1 << 22, None),
}
CHURN_ROUNDS_PER_STEP = 10
HEADLINE_RANGE = (16, 1024)  # BASELINE target band


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="pq1g", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-threads", type=int, default=0)
    ap.add_argument("--sizes", default="", help="comma list overriding the config's sweep (experiments)")
    ap.add_argument("--block", type=int, default=256, help="threads per block of the malloc/free launches")
    ap.add_argument("--waves", type=int, default=0,
                    help="persistent grid of WAVES x resident blocks (0: one thread per request)")
    return ap.parse_args()


# --------------------------------------------------------------- clocks ----
REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    """nvidia-smi sampled every 100 ms during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,utilization.gpu",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, busy = [], 0, set(), []
        for ln in self.lines:
            try:
                a, b, r, u = [x.strip() for x in ln.split(",")]
                sm.append(float(a))
                mx = max(mx, float(b))
                code = int(r, 16)
                for bit, name in REASONS.items():
                    if code & bit:
                        reasons.add(name)
                busy.append(float(u))
            except Exception:
                continue
        loaded = [s for s, u in zip(sm, busy) if u > 0] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons - {"gpu_idle"}), "samples": len(sm)}


# ------------------------------------------------------------ reference ----
def _metric():
    """BASELINE.json's metric string, identical in both arms."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return "malloc+free ops/sec vs size (16 B\u20138 KiB, 1M threads); % of L2-atomic roofline"


def config_dict(cfgname, hc_variant=None):
    """The `config` object both arms print for a sweep configuration."""
    desc, kind, flavor, heap, n, sizes = CONFIGS[cfgname]
    from paper_2504_18211_b200._abi import variant_name_of
    return {"workload": desc, "variant": variant_name_of(kind, flavor), "heap_bytes": heap, "threads": n,
            "sizes": sizes, "unit_of_work": "one successful malloc+free pair",
            "value_formula": "sum over sizes of successful pairs / sum over sizes of (alloc + free time)",
            "backoff": "FenceRetry, fence.sc.cta between rounds (SPEC.md:279 asks seq-cst; CTA scope is the "
                       "documented deviation, DESIGN.md section 3), max_retries 64"}


def cpu_sweep(cfgname, passes, warmup, threads):
    """The reference CPU allocator (the SPEC restatement oracle/ouro_oracle.cpp on
    std::thread workers behind a start barrier) on the SAME
    workload as the GPU arm: 2^20 slots per size, the same sizes, one persistent
    heap.  A pass = one size's trial of 2 iterations (alloc all / write / verify /
    free all); its timed figure is iteration 2 (mean_subsequent).
    Passes cycle through the sizes; every size gets >= 1 timed pass.  Returns the
    per-size means and value = sum of per-size pairs / sum of per-size times, the
    GPU arm's composition."""
    from oracle_lib import OHeap, TrialOut, oracle
    from paper_2504_18211_b200._abi import Config
    desc, kind, flavor, heap, n, sizes = CONFIGS[cfgname]
    cfg = Config(heap, 64 << 10, 16, 8192, flavor, kind, 0, 0, 64, 100, 100000)
    L = oracle()
    oh = OHeap(cfg)
    per = {s: {"ok": [], "ms": []} for s in sizes}
    timed = max(passes, len(sizes))
    verified = True
    pass_ms = []
    for i in range(warmup + timed):
        s = sizes[i % len(sizes)]
        out = TrialOut()
        assert L.orc_bench_trial(oh.h, n, s, None, 2, threads, 7, C.byref(out)) == 0
        verified = verified and bool(out.verified)
        if i >= warmup:
            per[s]["ok"].append(out.ok_allocs // 2)
            per[s]["ms"].append(out.alloc_ms[1] + out.free_ms[1])
            pass_ms.append(out.alloc_ms[1] + out.free_ms[1])
    oh.close()
    ok = sum(statistics.mean(p["ok"]) for p in per.values())
    ms = sum(statistics.mean(p["ms"]) for p in per.values())
    per_size = {str(s): {"ok": int(statistics.mean(p["ok"])), "alloc_free_ms": round(statistics.mean(p["ms"]), 3),
                         "passes": len(p["ms"])} for s, p in per.items()}
    return {"value": ok / (ms / 1e3), "per_size": per_size, "ms_per_step": statistics.mean(pass_ms),
            "timed_passes": timed, "verified": verified, "threads": threads, "slots": n}


def run_reference(args, cfgname):
    """--impl reference: the reference CPU allocator on all host threads, same
    metric / unit / config as the GPU arm (the reference tree has no runnable
    allocator, so its CPU restatement is the reference)."""
    desc, kind, flavor, heap, n, sizes = CONFIGS[cfgname]
    threads = args.ref_threads or os.cpu_count() or 1
    if sizes is None:  # churn: ops = mallocs + frees per second
        from oracle_lib import OHeap, oracle
        from paper_2504_18211_b200._abi import ChurnResult, Config
        sample = min(n, 1 << 20)
        cfg = Config(heap, 64 << 10, 16, 8192, flavor, kind, 0, 0, 64, 100, 100000)
        L = oracle()
        oh = OHeap(cfg)
        slots = (C.c_uint64 * sample)(*([2 ** 64 - 1] * sample))
        tot_ops, tot_s, r0 = 0, 0.0, 0
        for step in range(args.warmup + args.steps):
            res, ms = ChurnResult(), C.c_double()
            assert L.orc_churn(oh.h, sample, r0, CHURN_ROUNDS_PER_STEP, 1, threads, slots, C.byref(res),
                               C.byref(ms)) == 0
            r0 += CHURN_ROUNDS_PER_STEP
            if step >= args.warmup:
                tot_ops += res.mallocs_ok + res.mallocs_failed + res.frees
                tot_s += ms.value / 1e3
        value = tot_ops / tot_s
        print(json.dumps({
            "metric": "churn malloc+free ops/s", "impl": "reference", "value": value, "unit": "ops/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_s / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32/u64", "data": "synthetic",
            "config": {"workload": desc, "sample_threads": sample},
            "cpu_baseline": {"value": value, "unit": "ops/s", "cores": threads, "kind": "port",
                             "sample": f"{sample} slots x {CHURN_ROUNDS_PER_STEP} rounds per step"},
            "e2e": {"value": value, "unit": "ops/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return
    r = cpu_sweep(cfgname, args.steps, args.warmup, threads)
    sample = (f"{n} slots per size (the GPU arm's thread count), sizes {sizes}; a step = one size's trial "
              f"of 2 iterations timed on iteration 2 (mean_subsequent), sizes cycled, {r['timed_passes']} timed "
              f"steps after {args.warmup} warm-up steps; oracle/ouro_oracle.cpp on std::thread x {threads}")
    line = {
        "metric": _metric(), "impl": "reference", "value": r["value"], "unit": "pairs/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32/u64",
        "data": "synthetic", "same_config": True,
        "config": dict(config_dict(cfgname), per_size=r["per_size"], verified=r["verified"]),
        "cpu_baseline": {"value": r["value"], "unit": "pairs/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": r["value"], "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def cpu_baseline(cfgname):
    """The reference CPU allocator timed beside the GPU arm (rank 0, N=1): the same
    sweep as the reference arm, one timed pass per size after no warm-up step (each
    pass is itself a 2-iteration trial timed on iteration 2)."""
    threads = os.cpu_count() or 1
    r = cpu_sweep(cfgname, 0, 0, threads)
    desc, kind, flavor, heap, n, sizes = CONFIGS[cfgname]
    return {"value": r["value"], "unit": "pairs/s", "cores": threads, "kind": "port",
            "sample": f"{n} slots x each of {sizes}, one 2-iteration trial per size timed on iteration 2, "
                      f"oracle/ouro_oracle.cpp on std::thread x {threads}",
            "per_size": r["per_size"], "verified": r["verified"]}


# ------------------------------------------------------------------ GPU ----
def page_bytes(size, min_page=16):
    """Class page size for a request: next power of two >= max(size, 16)."""
    return max(min_page, 1 << (max(size, 1) - 1).bit_length())


def rmw_per_pair(kind, flavor, size, chunk=64 << 10):
    """SURVEY.md 8(d) algorithmic work: L2 RMW element-ops per malloc+free pair with
    32-lane warp aggregation.  PQ: (2 + 32 + 2 + 32) / 32 (count + ticket per warp,
    per-lane slot tag on each side); virtual flavours + per-warp segment refcount;
    CQ: class-queue visit + bitmap + free_count per warp, chunk assign/return per chunk."""
    ppc = chunk // page_bytes(size)
    if kind == 0:
        return 2.125 if flavor == 0 else 2.25
    if ppc >= 32:
        a, v = (10 + 9 * 32 / ppc) / 32, 1
    else:
        v = 32 / ppc
        a = 7 * v / 32 + 9 / ppc
    return a if flavor == 0 else a + 4 * v / 32


def _traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    capture of the current tree (profiles/r2_traffic.json): the 16 B alloc launch,
    where every thread is served (8.6 MB against 8.4 MB of algorithmic slot reads)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            return json.load(f)["per_launch_dram_bytes"]["16"]
    except Exception:
        return None


def storm_roofline(per_size, n, max_retries, hot_lat_s, block, resident_per_sm=6, sms=148):
    """Latency roofline of the OOM-heavy alloc launches (> half the requests OOM): a warp
    that fails declares OutOfMemory only after max_retries - 1 further rounds, each needing
    an observation of the queue made after the previous one, i.e. one
    dependent hot-word load per round at best; blocks run in n / (block x resident) waves.
    floor = waves x (max_retries - 1) x measured hot-word load latency (ouro_atomic_peak
    mode 4: 888 concurrent pollers of one word, the storm's contention)."""
    waves = n / (block * resident_per_sm * sms)
    floor_us = waves * (max_retries - 1) * hot_lat_s * 1e6
    out = {}
    for s, p in per_size.items():
        if p["oom"] * 2 > n:
            out[s] = {"alloc_us": p["alloc_us"], "floor_us": round(floor_us, 1),
                      "frac": round(floor_us / p["alloc_us"], 3)}
    return {"bound": "latency", "resource": "one dependent L2 load of the class-queue count per retry round",
            "hot_load_ns": round(hot_lat_s * 1e9, 1), "waves": round(waves, 2),
            "rounds": max_retries - 1, "per_size": out}


def sweep_floor(per_size, n, max_retries, hot_lat_s, block, p_same):
    """The alloc kernel's floor over the whole sweep: per size, the same-address chain
    floor (ceil(ok/32) RMWs per chain address at the measured same-address peak) or,
    for OOM-heavy sizes, the retry-round latency floor (storm_roofline); summed and
    compared with the summed measured alloc time."""
    storm = storm_roofline(per_size, n, max_retries, hot_lat_s, block)["per_size"]
    floor = actual = 0.0
    for s, p in per_size.items():
        chain_us = (p["ok"] + 31) // 32 / p_same * 1e6
        floor += max(chain_us, storm[s]["floor_us"]) if s in storm else chain_us
        actual += p["alloc_us"]
    return {"floor_us": round(floor, 1), "alloc_us": round(actual, 1),
            "frac": round(floor / actual, 3) if actual else None,
            "model": "sum over sizes of max(chain floor, OOM-round latency floor) / sum of alloc times"}


def job_totals(tot_ms, tot_ok, world, device="cpu"):
    """Whole-job totals for weak scaling: time = MAX over ranks of the device
    time, work = SUM over ranks of successful pairs (independent heaps, no
    collective on the data path; this reduction is bookkeeping only)."""
    if world <= 1:
        return float(tot_ms), float(tot_ok)
    import torch
    import torch.distributed as dist
    tmax = torch.tensor([float(tot_ms)], dtype=torch.float64, device=device)
    tsum = torch.tensor([float(tot_ok)], dtype=torch.float64, device=device)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    return float(tmax[0]), float(tsum[0])


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, args.config)
        return
    import torch
    import torch.distributed as dist

    import paper_2504_18211_b200 as ob
    if args.gpus > 1 and world == 1 and CONFIGS[args.config][5] is not None:
        return run_threads_driver(args)
    torch.cuda.set_device(local)
    if world > 1:
        # host-side bookkeeping only (start barrier, max-over-ranks time): every GPU owns
        # an independent heap and no data crosses GPUs, so no NCCL communicator is made
        dist.init_process_group("gloo")
    desc, kind, flavor, heap_bytes, n, sizes = CONFIGS[args.config]
    if sizes is None:
        return run_churn(args, world, rank, local, desc, kind, flavor, heap_bytes, n)
    if args.sizes:
        sizes = [int(x) for x in args.sizes.split(",")]
    hc = ob.HeapConfig(heap_bytes, allocator_kind=ob.AllocatorKind(kind), queue_flavor=ob.QueueFlavor(flavor))
    heap = ob.Heap(hc, local)
    heap.set_launch_shape(args.block, args.waves)
    ptrs = torch.zeros(n, dtype=torch.int64, device="cuda")
    res = torch.zeros(4, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # roofline denominators measured on this device
    p_same = ob.atomic_peak(local, 2)      # same-address RMW, one per warp
    p_dist = ob.atomic_peak(local, 0)      # distinct-address 32-bit RMW, one per sector
    hot_lat_s = 1.0 / ob.atomic_peak(local, 4)  # hot-word dependent load latency, 888 pollers

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    per = {s: {"alloc_ms": [], "free_ms": [], "write_ms": [], "verify_ms": [], "ok": [], "verify_bad": 0}
           for s in sizes}
    launches = 0

    def one_step(record):
        nonlocal launches
        for s in sizes:
            res.zero_()
            res[1] = -1
            flush.fill_(1)
            ev[0].record()
            heap.launch_alloc(n, ptrs, size=s)
            ev[1].record()
            heap.launch_count(n, ptrs, res[2:3])
            ev[6].record()
            heap.launch_write(n, ptrs, 99, 0)
            ev[4].record()
            heap.launch_verify(n, ptrs, 99, 0, res)
            ev[5].record()
            flush.fill_(2)
            ev[2].record()
            heap.launch_free(n, ptrs)
            ev[3].record()
            ev[3].synchronize()
            if record:
                launches += 5  # ours per size: alloc, count, write, verify, free
                p = per[s]
                p["alloc_ms"].append(ev[0].elapsed_time(ev[1]))
                p["free_ms"].append(ev[2].elapsed_time(ev[3]))
                p["write_ms"].append(ev[6].elapsed_time(ev[4]))
                p["verify_ms"].append(ev[4].elapsed_time(ev[5]))
                p["ok"].append(int(res[2]))
                p["verify_bad"] += int(res[0])

    with ClockSampler(local) as clk:
        deadline = time.time() + 3.0
        while not clk.lines and time.time() < deadline:   # sampler running before any timing
            time.sleep(0.05)
        for _ in range(args.warmup):
            one_step(False)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            one_step(True)
        barrier()
        wall = time.perf_counter() - t0
        while time.perf_counter() - t0 < 0.3:              # at least a few samples under load
            one_step(False)
        barrier()
    err = heap.last_error()
    tot_ms = sum(sum(p["alloc_ms"]) + sum(p["free_ms"]) for p in per.values())
    tot_ok = sum(sum(p["ok"]) for p in per.values())
    ms_job, ok_job = job_totals(tot_ms, tot_ok, world)
    value = ok_job / (ms_job / 1e3)

    # ---------------- e2e through the public C-ABI with host buffers ----------------
    # Every size's request array (4 B per thread, pinned host memory) is copied
    # H2D on a copy stream while the previous size's alloc/count/free run on the
    # compute stream (double-buffered); each success count comes back D2H.  All
    # copies are inside the timed region.
    e2e_ms, e2e_ok = 0.0, 0
    e2e_reps = []
    # 16-bit request sizes (ouro_launch_alloc_u16): every valid request is <= 8 KiB
    h_sizes = [torch.full((n,), s, dtype=torch.int16).pin_memory() for s in sizes]
    h_res = torch.zeros(len(sizes), dtype=torch.int64).pin_memory()
    d_sizes = [torch.empty(n, dtype=torch.int16, device="cuda") for _ in range(2)]
    d_res = torch.zeros(len(sizes), dtype=torch.int64, device="cuda")
    s_copy, s_comp = torch.cuda.Stream(), torch.cuda.Stream()
    for rep in range(args.warmup + args.steps):  # warm-up passes, then K timed passes
        copied = [torch.cuda.Event() for _ in sizes]
        done = [torch.cuda.Event() for _ in sizes]
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d_res.zero_()
        torch.cuda.synchronize()
        t_start.record(s_comp)
        s_copy.wait_event(t_start)
        for i, s in enumerate(sizes):
            with torch.cuda.stream(s_copy):
                if i >= 2:
                    s_copy.wait_event(done[i - 2])      # buffer i%2 free again
                d_sizes[i % 2].copy_(h_sizes[i], non_blocking=True)
                copied[i].record(s_copy)
            s_comp.wait_event(copied[i])
            heap.launch_alloc(n, ptrs, sizes=d_sizes[i % 2], stream=s_comp)
            heap.launch_count(n, ptrs, d_res[i:i + 1], stream=s_comp)
            heap.launch_free(n, ptrs, stream=s_comp)
            done[i].record(s_comp)
        with torch.cuda.stream(s_comp):
            h_res.copy_(d_res, non_blocking=True)        # D2H: the step's results
        t_end.record(s_comp)
        t_end.synchronize()
        if rep >= args.warmup:
            e2e_reps.append(t_start.elapsed_time(t_end))
            e2e_ms += e2e_reps[-1]
            e2e_ok += int(h_res.sum())

    # e2e job totals: max over ranks of the e2e time, sum of the successes
    e2e_ms_job, e2e_ok_job = job_totals(e2e_ms, e2e_ok, world)
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---------------- roofline of the dominant kernel ----------------
    a_ms = sum(sum(p["alloc_ms"]) for p in per.values())
    f_ms = sum(sum(p["free_ms"]) for p in per.values())
    dom = "alloc" if a_ms >= f_ms else "free"
    dom_ms = max(a_ms, f_ms)
    # binding resource: the per-class queue counters (count + head for alloc,
    # count + tail for free), each one serial RMW per warp group = ceil(ok/32)
    chain_ops = sum(sum((o + 31) // 32 for o in p["ok"]) for p in per.values())
    achieved = chain_ops / (dom_ms / 1e3)
    per_size = {}
    elem_ops = 0.0
    for s, p in per.items():
        am, fm = statistics.mean(p["alloc_ms"]), statistics.mean(p["free_ms"])
        ok = statistics.mean(p["ok"])
        chain = (int(ok) + 31) // 32  # RMWs per chain address per launch (warp aggregation)
        pb = page_bytes(s)
        a_pair = rmw_per_pair(kind, flavor, s)
        elem_ops += a_pair * sum(p["ok"])
        per_size[str(s)] = {"ok": int(ok), "oom": n - int(ok), "alloc_us": round(am * 1e3, 2),
                            "free_us": round(fm * 1e3, 2),
                            "alloc_us_median": round(statistics.median(p["alloc_ms"]) * 1e3, 2),
                            "free_us_median": round(statistics.median(p["free_ms"]) * 1e3, 2),
                            "pairs_per_s": ok / ((am + fm) / 1e3),
                            "alloc_roofline_frac": round(chain / (am / 1e3) / p_same, 3),
                            "free_roofline_frac": round(chain / (fm / 1e3) / p_same, 3),
                            "rmw_elem_ops_per_pair": round(a_pair, 4),
                            "write_gbs": round(ok * pb / (statistics.median(p["write_ms"]) / 1e3) / 1e9, 1),
                            "verify_gbs": round(ok * pb / (statistics.median(p["verify_ms"]) / 1e3) / 1e9, 1)}
    band = [s for s in sizes if HEADLINE_RANGE[0] <= s <= HEADLINE_RANGE[1]]
    band_ok = sum(sum(per[s]["ok"]) for s in band)
    band_ms = sum(sum(per[s]["alloc_ms"]) + sum(per[s]["free_ms"]) for s in band)
    full = [s for s in sizes if per_size[str(s)]["oom"] == 0]
    full_ok = sum(sum(per[s]["ok"]) for s in full)
    full_ms = sum(sum(per[s]["alloc_ms"]) + sum(per[s]["free_ms"]) for s in full)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args.config)
        except Exception as e:  # reported, not fatal
            cpu = {"error": str(e)}
    line = {
        "metric": _metric(),
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_job / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32/u64 (integer allocator; no floating point)",
        "data": "synthetic",
        "config": dict(config_dict(args.config),
                       l2="flushed (256 MiB write) before every timed kernel",
                       timed="alloc kernel + free kernel per size, CUDA events, default stream",
                       per_size=per_size,
                       pairs_per_s_16B_1KiB=band_ok / (band_ms / 1e3) if band_ms else None,
                       pairs_per_s_sizes_without_oom=full_ok / (full_ms / 1e3) if full_ms else None,
                       sizes_without_oom=full,
                       verify_mismatched_words=sum(p["verify_bad"] for p in per.values()),
                       sticky_error=err[0], wall_s_timed=wall, sizes=sizes),
        "roofline": {"bound": "l2_atomic", "kernel": dom,
                     "resource": "same-address RMW chain on the class-queue counters (1 per warp group)",
                     "achieved": achieved / 1e9, "peak": p_same / 1e9, "unit": "Gop/s",
                     "frac": achieved / p_same, "traffic": _traffic(),
                     "peak_source": "measured in-run: ouro_atomic_peak mode 2 (same-address atomicAdd, one per warp)",
                     "distinct_address_peak_gops": p_dist / 1e9,
                     "element_ops": {"what": "SURVEY.md 8(d): A RMW element-ops per successful pair "
                                             "(per size: rmw_elem_ops_per_pair) x pairs / (alloc + free time), "
                                             "against the distinct-address atomic peak",
                                     "achieved_gops": elem_ops / ((a_ms + f_ms) / 1e3) / 1e9,
                                     "peak_gops": p_dist / 1e9,
                                     "frac": elem_ops / ((a_ms + f_ms) / 1e3) / p_dist},
                     "dominant_kernel_share": dom_ms / (a_ms + f_ms),
                     "oom_storm": storm_roofline(per_size, n, hc.max_retries, hot_lat_s, args.block),
                     "sweep_floor": sweep_floor(per_size, n, hc.max_retries, hot_lat_s, args.block, p_same),
                     "note": "sweep-level: the OOM-heavy sizes spend their alloc time in the SPEC's "
                             "max_retries rounds, not on the RMW chain; per_size[*].alloc_roofline_frac "
                             "gives the fraction where all threads are served"},
        "e2e": {"value": e2e_ok_job / (e2e_ms_job / 1e3), "unit": "pairs/s",
                "h2d_bytes_per_step": 2 * n * len(sizes), "d2h_bytes_per_step": 8 * len(sizes),
                "ms_per_step_median": statistics.median(e2e_reps), "steps": len(e2e_reps),
                "path": "ouro_launch_alloc_u16/count/free (C-ABI) per size; per-thread 16-bit request sizes copied H2D "
                        "from pinned host memory on a copy stream (overlapping the previous size's kernels), "
                        "success counts copied D2H, all inside the timed region"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_threads_driver(args):
    """--gpus N without torchrun: one process, one host thread and one heap per GPU
    (ouro_multi_sweep, paper_2504_18211_b200/csrc/ouro_multi.cpp): a host barrier
    before every step, CUDA events per device, no collective.  value = pairs summed
    over GPUs / the slowest GPU's summed alloc + free kernel time (weak scaling)."""
    import paper_2504_18211_b200 as ob
    desc, kind, flavor, heap_bytes, n, sizes = CONFIGS[args.config]
    if args.sizes:
        sizes = [int(x) for x in args.sizes.split(",")]
    hc = ob.HeapConfig(heap_bytes, allocator_kind=ob.AllocatorKind(kind), queue_flavor=ob.QueueFlavor(flavor))
    with ClockSampler(0) as clk:
        r = ob.multi_sweep(hc, list(range(args.gpus)), n, sizes, warmup=args.warmup, steps=args.steps)
    print(json.dumps({
        "metric": _metric(), "value": r.pairs_per_s, "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r.max_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32/u64 (integer allocator; no floating point)", "data": "synthetic",
        "config": dict(config_dict(args.config), sizes=sizes,
                       driver="one process, one host thread + heap per GPU (ouro_multi_sweep), no collective",
                       per_gpu_ms=[r.dev_ms[d] for d in range(r.ndev)],
                       per_gpu_pairs=[r.dev_pairs[d] for d in range(r.ndev)], verified=bool(r.verified)),
        "e2e": None, "gpu_launches": args.gpus * (args.warmup + args.steps) * len(sizes) * 3,
        "clocks": clk.summary(), "cpu_baseline": None}))


def run_churn(args, world, rank, local, desc, kind, flavor, heap_bytes, n):
    """BASELINE configs[3]: 4M threads, interleaved alloc/free rounds (one kernel
    per round: each thread frees its slot on odd hash, else mallocs 8 B-4 KiB and
    stamps it; occupied even-hash slots check their stamp).  ops = mallocs
    (successful or not) + frees; fragmentation = live bytes / bytes of assigned
    chunks; reuse = mallocs served from pages handed out before."""
    import torch
    import torch.distributed as dist

    import paper_2504_18211_b200 as ob
    hc = ob.HeapConfig(heap_bytes, allocator_kind=ob.AllocatorKind(kind), queue_flavor=ob.QueueFlavor(flavor))
    heap = ob.Heap(hc, local)
    slots = torch.zeros(n, dtype=torch.int64, device="cuda")
    res = torch.zeros(5, dtype=torch.int64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    r0 = 0
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            heap.launch_churn(n, r0, CHURN_ROUNDS_PER_STEP, 1, slots, res)
            r0 += CHURN_ROUNDS_PER_STEP
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        res.zero_()
        ms = 0.0
        for _ in range(args.steps):
            ev[0].record()
            heap.launch_churn(n, r0, CHURN_ROUNDS_PER_STEP, 1, slots, res)
            ev[1].record()
            ev[1].synchronize()
            ms += ev[0].elapsed_time(ev[1])
            r0 += CHURN_ROUNDS_PER_STEP
    ok, failed, frees, reused, bad = [int(x) for x in res]
    ops = ok + failed + frees
    ms_job, ops_job = job_totals(ms, ops, world)
    a = heap.audit(n, slots)
    st = heap.stats()
    assigned = sum(st.cls[k].chunks for k in range(st.num_classes))
    frag = a.bytes / (assigned * hc.chunk_bytes) if assigned else None
    if rank == 0:
        print(json.dumps({
            "metric": "churn malloc+free ops/s", "value": ops_job / (ms_job / 1e3), "unit": "ops/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_job / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32/u64",
            "data": "synthetic",
            "config": {"workload": desc, "variant": ob.variant_name(hc.variant), "threads": n,
                       "rounds_timed": args.steps * CHURN_ROUNDS_PER_STEP,
                       "mallocs_ok": ok, "mallocs_failed": failed, "frees": frees,
                       "reuse_fraction": reused / ok if ok else None, "stamp_check_failures": bad,
                       "live_allocations": a.live, "live_bytes": a.bytes, "assigned_chunks": assigned,
                       "fragmentation_live_over_assigned": frag,
                       "audit_overlaps": a.overlaps, "sticky_error": heap.last_error()[0]},
            "gpu_launches": args.steps * CHURN_ROUNDS_PER_STEP, "clocks": clk.summary()}))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
