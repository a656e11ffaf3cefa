#!/usr/bin/env python
"""Throughput of the sliding super point detector hot path on B200.

One step = one time slice (slot) of BASELINE.json's config C2: scan the slot's
pairs into the RSEA grid (stamps and window ring updated in place), find hot
estimators, reconstruct the super points (levels 2..r-1 + finalize, reports
back on the host), advance the slot.  Slots pipeline: a slot's
reconstruction is collected after the next slot's scan is queued.  At N GPUs
each GPU is one edge router scanning its own shard of the slot (weak scaling)
and the routers merge by union-min before reconstruction (default: cells
sharded among the routers, pairs relayed over NVLink; see
paper_1803_11036_b200/dist.py and --merge).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c1] [--no-cpu-baseline] [--no-e2e] [--merge ...]
                  [--stamp-width 8|16|32] [--window k] [--q/--eta/--theta ...]

Prints ONE JSON line (rank 0).  `--impl reference` times the reference's own
CPU implementation (oracle/_ref, compiled from /root/reference/proj) on the
same workload on this host's cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]: single router, 1B-packet Zipf trace with injected
    # scanner / DDoS super points, full-HBM estimator table.
    "c2": dict(workload="C2: 1 router/GPU, 1e9-pair Zipf(1.1) trace (10 slots x 1e8 pairs) with "
                        "100 scanners + 10 DDoS victims at 4*theta injected, full-HBM table "
                        "q16 r5 delta6 eta65536 (80 GiB u32 stamps)",
               q=16, r=5, delta=6, eta=1 << 16, seed=0x5eed, k=5, theta=1024.0,
               pairs_per_slot=100_000_000, trace_slots=10, hosts=1 << 21, pool=16, zipf=1.1,
               n_super=110, fanout=4096),
    # C2 with SURVEY §8(d)'s upper pool bound: 64 distinct opposites per
    # background host (~4x the distinct pairs per slot).  theta and the
    # injected fanout scale 4x so the window's background stays below the hot
    # cutoff (distinct pairs per window << theta * 2^q); the pair set doubles.
    "c2p64": dict(workload="C2 with 64-entry opposite pools: 1 router/GPU, 1e9-pair Zipf(1.1) trace (10 "
                           "slots x 1e8 pairs), 100 scanners + 10 DDoS victims at 4*theta injected, "
                           "theta 4096, full-HBM table q16 r5 delta6 eta65536 (80 GiB u32 stamps)",
                  q=16, r=5, delta=6, eta=1 << 16, seed=0x5eed, k=5, theta=4096.0,
                  pairs_per_slot=100_000_000, trace_slots=10, hosts=1 << 21, pool=64, zipf=1.1,
                  n_super=110, fanout=16384, pairset_log2=26),
    # configs[0]: the reference's CPU-runnable case (reference default geometry).
    "c1": dict(workload="C1: 1 router/GPU, 10 slots x 1e6 (cip,oip) pairs: 20 planted supers x "
                        "2048 distinct oips, the rest uniform; reference default table q14 r5 "
                        "delta6 eta2048", q=14, r=5, delta=6, eta=2048, seed=0x5eed, k=5, theta=1024.0,
               pairs_per_slot=1_000_000, trace_slots=10, hosts=1, pool=0, zipf=1.1,
               n_super=20, fanout=2048),
}

PKT_BYTES = 800  # the paper's Gb/s convention


def env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v not in (None, "") else default


class SynthParams(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("hosts", C.c_uint32), ("pool", C.c_uint32),
                ("n_super", C.c_uint32), ("super_fanout", C.c_uint32),
                ("pairs_per_slot", C.c_uint64), ("shard", C.c_uint32), ("n_shards", C.c_uint32)]


def synth_params(cfg, rank, world):
    return SynthParams(cfg["seed"] ^ 0xC2C2, cfg["hosts"], cfg["pool"], cfg["n_super"],
                       cfg["fanout"], cfg["pairs_per_slot"] * world, rank, world)


B200_L2_BYTES = 126 << 20  # what torch reports for a B200 (L2_cache_size)


def l2_policy(cfg):
    """(flush?, note): the timing rule's L2 statement for this workload.  C2's
    800 MB slot is larger than L2; C1's 8 MB slot is not, so every GPU step
    starts with a 2xL2 write inside the timed region."""
    slot_bytes = cfg["pairs_per_slot"] * 8
    if slot_bytes < 2 * B200_L2_BYTES:
        return True, (f"GPU L2 ({B200_L2_BYTES >> 20} MiB) flushed before every step by a "
                      f"{2 * B200_L2_BYTES >> 20} MiB write inside the timed region; slot input "
                      f"{slot_bytes / 1e6:g} MB")
    return False, (f"inputs larger than L2: {slot_bytes / 1e6:g} MB per slot vs "
                   f"{B200_L2_BYTES >> 20} MiB GPU L2, no flush")


def config_of(cfg):
    """The `config` object both arms print, identical for the same workload
    (implementation details go under `setup`)."""
    return {"workload": cfg["workload"], "pairs_per_step_per_gpu": cfg["pairs_per_slot"],
            "window_k": cfg["k"], "theta": cfg["theta"], "l2": l2_policy(cfg)[1]}


def zipf_cdf(L, cfg):
    cdf = np.empty(cfg["hosts"], dtype=np.uint64)
    assert L.sspd_synth_zipf_cdf(cfg["hosts"], cfg["zipf"], cdf.ctypes.data) == 0
    return cdf


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML from a
    thread every 2 ms (the timed region of a default run is tens of ms), else
    `nvidia-smi -lms 100` as a fallback."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.nvml = None
        self.samples = []  # (sm_mhz, reasons bitmask) taken while `active`
        self.active = False   # set by the timed loops between their synchronizes
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_dev{device}.csv")

    def _nvml_index(self):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x.strip() for x in vis.split(",") if x.strip()]
        if ids and all(x.isdigit() for x in ids) and self.device < len(ids):
            return int(ids[self.device])
        return self.device

    def __enter__(self):
        try:
            import threading

            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self._nvml_index())
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            self.bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                         "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                         "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                         "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
            self.stop = threading.Event()

            def run():
                while not self.stop.is_set():
                    if self.active:
                        sample = (N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM),
                                  N.nvmlDeviceGetCurrentClocksEventReasons(h))
                        if self.active:
                            self.samples.append(sample)
                    time.sleep(0.002)

            self.nvml = N
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.nvml:
            self.stop.set()
            self.thread.join()
            try:
                self.nvml.nvmlShutdown()
            except Exception:
                pass
        elif self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if self.nvml:
            sm = [c for c, _ in self.samples]
            reasons = sorted({nm for _, m in self.samples for nm, b in self.bits.items() if m & b})
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(sm),
                    "source": "nvml every 2 ms inside the timed regions (device + e2e loops)"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(self.NAMES, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 100"}


# ---------------------------------------------------------------------------
# Reference arm / cpu baseline: the compiled reference on host cores.

def run_reference(cfg, steps, warmup, pairs_cap, time_budget_s, workers=None):
    """Reference Rsea at the same geometry: per step one slot of the same
    trace through scan_batch (alpha=32768 batches, pipeline.cpp:58-63),
    reconstruct_leveled and advance_slot, workers = all host cores (or
    $SSPD_REF_WORKERS, or `workers`)."""
    from oracle import oracle as O

    # the workload comes from the host-only generator (no CUDA runtime in
    # this process): the same traces the device generator makes
    S = C.CDLL(os.path.join(ROOT, "oracle", "libsynth_host.so"))
    if workers is None:
        workers = env_int("SSPD_REF_WORKERS", os.cpu_count() or 1)
    t0 = time.time()
    g = O.RefGrid(cfg["q"], cfg["r"], cfg["delta"], cfg["seed"], cfg["eta"])
    t_init = time.time() - t0
    cdf = np.empty(cfg["hosts"], dtype=np.uint64)
    assert S.sspd_synth_zipf_cdf_host(C.c_uint32(cfg["hosts"]), C.c_double(cfg["zipf"]),
                                      C.c_void_p(cdf.ctypes.data)) == 0
    sp = synth_params(cfg, 0, 1)
    n = min(cfg["pairs_per_slot"], pairs_cap)
    buf = np.empty((n, 2), dtype=np.uint32)
    times, scan_t, rec_t, adv_t, n_rep = [], [], [], [], []
    budget_hit = False
    for i in range(warmup + steps):
        assert S.sspd_synth_pairs_host(C.byref(sp), C.c_void_p(cdf.ctypes.data),
                                       C.c_uint64(i % cfg["trace_slots"]), C.c_uint64(0),
                                       C.c_uint64(n), C.c_void_p(buf.ctypes.data)) == 0
        a = time.perf_counter()
        g.scan_alpha(buf, workers)
        b = time.perf_counter()
        rep = g.reconstruct(cfg["k"], cfg["theta"], workers=workers)
        c = time.perf_counter()
        g.advance(workers)
        d = time.perf_counter()
        if i >= warmup:
            times.append(d - a)
            scan_t.append(b - a)
            rec_t.append(c - b)
            adv_t.append(d - c)
            n_rep.append(len(rep))
        if time.time() - t0 > time_budget_s and len(times) >= 1:
            budget_hit = True
            break
    mean = sum(times) / len(times)
    return {
        "value": n / mean / 1e6, "steps_timed": len(times), "pairs_per_step": n,
        "workers": workers, "init_s": t_init, "scan_ms": 1e3 * statistics.mean(scan_t),
        "reconstruct_ms": 1e3 * statistics.mean(rec_t), "advance_ms": 1e3 * statistics.mean(adv_t),
        "step_ms": 1e3 * mean, "reports": n_rep[-1] if n_rep else 0, "budget_hit": budget_hit,
    }


# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--window", type=int, default=0, help="override the window k (C4 sweeps)")
    ap.add_argument("--theta", type=float, default=0.0, help="override theta (C5 sweeps)")
    ap.add_argument("--eta", type=int, default=0, help="override eta, buckets per estimator (C5 sweeps)")
    ap.add_argument("--q", type=int, default=0, help="override q, log2 columns per row (C5 sweeps)")
    ap.add_argument("--merge", default="auto", choices=["auto", "pairs", "push", "bitmap", "stamps", "shard"],
                    help="router exchange at N>1 (auto = shard, else pairs if symmetric memory is "
                         "unavailable): distinct pairs pushed over NVLink during the scan (push), the "
                         "same lists all-gathered after the scan (pairs), OR of touched bitmaps, "
                         "the literal all-reduce(max) of the full stamp grid, or cells sharded among "
                         "routers with pairs relayed to their owners through pair owners (shard)")
    ap.add_argument("--stamp-width", type=int, default=32, choices=[8, 16, 32],
                    help="bits per recorder stamp (C4): 8/16 keep R_k (k <= window) and the reports "
                         "exact, 32 also the full distances")
    ap.add_argument("--scan-mode", default="auto", choices=["auto", "bitmap", "direct", "dedup", "binned"])
    ap.add_argument("--filter", type=int, default=-1, help="L1 duplicate probe 0/1 (-1 = default)")
    ap.add_argument("--ref-pairs", type=int, default=100_000_000,
                    help="pairs per reference step (bounded sample of the slot)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.window:
        cfg["k"] = args.window
    for key in ("theta", "eta", "q"):
        if getattr(args, key):
            cfg[key] = getattr(args, key)
            cfg["workload"] += f"; {key} overridden to {getattr(args, key):g}"
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    if world > 1 and args.stamp_width != 32 and args.impl == "ours":
        ap.error("--stamp-width 8/16 is single-router only: the router exchanges need full stamps")
    local = env_int("LOCAL_RANK", 0)
    unit = "Mpackets/s"
    metric = "scan+reconstruct throughput, Mpackets/s (Gb/s at 800 B/pkt in gbps_800B)"

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_reference(cfg, args.steps, args.warmup, args.ref_pairs, time_budget_s=240)
        line = {
            "impl": "reference", "metric": metric, "value": round(r["value"], 3), "unit": unit,
            "n_gpus": args.gpus, "steps": r["steps_timed"], "warmup": args.warmup,
            "ms_per_step": round(r["step_ms"], 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32/u16 integer", "data": "synthetic",
            "config": config_of(cfg),
            "setup": {"sample": f"{r['pairs_per_step']} pairs per step", "parallelism": "host OpenMP",
                      "recorders": "u16 distances (the reference's Recorder)"},
            "gbps_800B": round(r["value"] * 1e6 * PKT_BYTES * 8 / 1e9, 3),
            "reconstruct_ms": round(r["reconstruct_ms"], 3),
            "phases_ms": {"scan": round(r["scan_ms"], 3), "reconstruct": round(r["reconstruct_ms"], 3),
                          "advance": round(r["advance_ms"], 3)},
            "cpu_baseline": {"value": round(r["value"], 3), "unit": unit, "cores": r["workers"],
                             "kind": "reference",
                             "sample": f"{r['steps_timed']} slots x {r['pairs_per_step']} pairs of "
                                       f"the {args.config} trace, reference grid at full geometry"},
            "e2e": {"value": round(r["value"], 3), "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    import paper_1803_11036_b200 as P
    from paper_1803_11036_b200 import dist as PD

    if world > 1:
        import datetime

        # a wedged collective fails the run after 5 minutes instead of NCCL's 10
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"),
                                timeout=datetime.timedelta(seconds=int(os.environ.get("SSPD_DIST_TIMEOUT", "300"))))
    torch.cuda.set_device(local)
    dev = local
    L = P.load()
    # One non-default stream carries every kernel of the grid, the NCCL
    # collectives and the timing events (torch's default stream is the legacy
    # NULL stream, which the grid's stream would not be ordered with).
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    # --- setup (untimed): grid, trace resident in HBM, pinned host copy ------
    if cfg.get("pairset_log2"):
        os.environ.setdefault("SSPD_PAIRSET_LOG2", str(cfg["pairset_log2"]))
    def new_grid(shard=None):
        gr = P.Grid(cfg["q"], cfg["r"], cfg["delta"], cfg["seed"], cfg["eta"], device=dev,
                    width=args.stamp_width, k_max=cfg["k"], shard=shard)
        gr.set_stream(stream.cuda_stream)
        gr.scan_mode({"auto": -1, "bitmap": 0, "direct": 1, "dedup": 2, "binned": 3}[args.scan_mode], args.filter)
        return gr

    merge_used = args.merge
    if world > 1 and args.merge in ("auto", "shard"):
        # cells sharded among the routers: each router's grid
        # holds only the cells it owns (sspd_grid_create_sharded), so N routers
        # hold an N-times larger table; pair lists if symmetric memory is missing
        # a router pushes each of its new pairs at most once per owner, plus the
        # padding of its warps' last list blocks (kernels.cuh list_pad) per launch
        shard_cap = cfg["pairs_per_slot"] + 40 * torch.cuda.get_device_properties(local).multi_processor_count * 4 * 8 * 64
        try:
            g = new_grid(shard=(world, rank))
            PD.prepare(g, PD.SHARD, region_cap=shard_cap)
            merge_used = "shard"
        except Exception as e:
            if args.merge == "shard":
                raise
            print(f"[bench] shard exchange unavailable ({type(e).__name__}: {e}); using pairs", file=sys.stderr)
            g = new_grid()
            PD.prepare(g, PD.PAIRS)
            merge_used = "pairs"
    else:
        g = new_grid()
        if world > 1 and args.merge != "stamps":
            cap = min(cfg["pairs_per_slot"], 32 << 20)
            PD.prepare(g, {"pairs": PD.PAIRS, "push": PD.PUSH, "bitmap": PD.BITMAP}[args.merge], region_cap=cap)
    cdf = torch.from_numpy(zipf_cdf(L, cfg).view(np.int64)).to(f"cuda:{dev}")
    sp = synth_params(cfg, rank, world)
    n_local = cfg["pairs_per_slot"]
    S = cfg["trace_slots"]
    trace = torch.empty((S, n_local, 2), dtype=torch.int32, device=f"cuda:{dev}")
    for s in range(S):
        P._cabi.check(L.sspd_synth_device(dev, C.byref(sp), C.c_void_p(cdf.data_ptr()), s, 0,
                                          n_local, C.c_void_p(trace[s].data_ptr()),
                                          C.c_void_p(stream.cuda_stream)))
    torch.cuda.synchronize()
    host_trace = None
    if not args.no_e2e:
        host_trace = torch.empty((S, n_local, 2), dtype=torch.int32, pin_memory=True)
        host_trace.copy_(trace)
        torch.cuda.synchronize()

    k, theta = cfg["k"], cfg["theta"]
    # Timing rule: inputs larger than L2, else flush L2 between steps.  C2's
    # slot is 800 MB; C1's is 8 MB, so C1 steps start by writing a 2x-L2
    # buffer (inside the timed region: it is charged to the step).
    l2_bytes = max(torch.cuda.get_device_properties(dev).L2_cache_size, B200_L2_BYTES)
    flush = None
    if l2_policy(cfg)[0]:
        flush = torch.empty(2 * l2_bytes // 4, dtype=torch.int32, device=f"cuda:{dev}")

    # Slots pipeline: slot i's reconstruction is queued (sspd_reconstruct_async)
    # and its reports collected after slot i+1's scan is queued, so the GPU
    # never waits for the host between slots.  Sharded routers reconstruct
    # through collectives and stay synchronous.
    pipelined = not (world > 1 and merge_used == "shard")
    queued = [False]

    def collect():
        queued[0] = False
        return g.reconstruct_collect()

    def step(i, from_host=False):
        s = i % S
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        if flush is not None:
            flush.fill_(i)
        e0.record(stream)
        if from_host:
            g.scan_host_ptr(host_trace[s].data_ptr(), n_local)
        else:
            g.scan_device(trace[s].data_ptr(), n_local)
        if world > 1:
            if args.merge == "stamps":
                PD.merge_stamps_max(g)
            else:
                PD.merge(g)
        e1.record(stream)
        rep = None
        if pipelined:
            if queued[0]:
                rep = collect()  # the previous slot's reports
            g.reconstruct_async(k, theta)
            queued[0] = True
        else:
            rep = PD.reconstruct(g, k, theta)
        e2.record(stream)
        g.advance_slot()
        return rep, (e1, e2)

    def timed_loop(n_steps, start, from_host, clk=None):
        marks = []
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if clk is not None:
            clk.active = True
        ev_a = torch.cuda.Event(enable_timing=True)
        ev_b = torch.cuda.Event(enable_timing=True)
        ev_a.record(stream)
        reps = None
        for i in range(n_steps):
            reps, m = step(start + i, from_host)
            marks.append(m)
        if queued[0]:
            reps = collect()  # the last slot's reports, inside the timed region
        ev_b.record(stream)
        torch.cuda.synchronize()
        if clk is not None:
            clk.active = False
        if world > 1:
            dist.barrier()
        ms = ev_a.elapsed_time(ev_b)
        recon = [a.elapsed_time(b) for a, b in marks]
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{dev}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, recon, reps

    for i in range(args.warmup):
        step(i)
    slot = args.warmup

    # --- device-resident timed region --------------------------------------
    g.profile(True)
    g.profile_reset()
    launches0 = P.launch_count()
    fresh0 = g.fresh_pairs()
    clk = ClockSampler(dev).__enter__()
    ms, recon, reps = timed_loop(args.steps, slot, False, clk)
    launches = P.launch_count() - launches0
    fresh = g.fresh_pairs() - fresh0  # pairs new to their slot (pipelined dedup scan's device counter)
    slot += args.steps
    prof = {}
    for name in ("bin", "scan", "commit", "hist_counts", "count", "reconstruct", "hot_compact", "level2",
                 "level_ext", "finalize", "merge", "rebase"):
        t, n, u = g.profile_read(name)
        if n:
            prof[name] = {"ms": t, "launches": n, "units": u}
    g.profile(False)
    g.profile_reset()
    total_pairs = n_local * args.steps * world
    value = total_pairs / (ms / 1e3) / 1e6

    # --- e2e through the public API with host buffers ----------------------
    e2e = None
    if host_trace is not None:
        for i in range(2):
            step(slot + i, True)
        slot += 2
        g.io_bytes(reset=True)
        ms_e, _, _ = timed_loop(args.steps, slot, True, clk)
        h2d, d2h = g.io_bytes(reset=True)
        slot += args.steps
        e2e = {"value": round(total_pairs / (ms_e / 1e3) / 1e6, 3), "unit": unit,
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
               "ms_per_step": round(ms_e / args.steps, 3)}

    clk.__exit__(None, None, None)

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # --- roofline of the dominant kernel --------------------------------------
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm = peaks.get("hbm_gbs", 6650.0)
    dom = max(prof, key=lambda x: prof[x]["ms"]) if prof else None
    r = cfg["r"]
    roof = None
    if dom:
        d = prof[dom]
        per_launch_ms = d["ms"] / d["launches"]
        units_per_launch = d["units"] / d["launches"]
        bytes_per_unit = {"scan": 8 + r * 32,                       # 168 B/pkt at r=5
                          "count": cfg["eta"] * 4,                  # one estimator of u32 stamps
                          "commit": 8 / 32 * 32,                    # bitmap word read+clear per 32 rec
                          "merge": 4 * 2}.get(dom)
        if bytes_per_unit is not None:
            achieved = bytes_per_unit * units_per_launch / (per_launch_ms / 1e3) / 1e9
            # DRAM bytes per launch of the same kernel at the same config, from
            # the committed ncu --set full capture (bench cannot run ncu itself)
            traffic, tsrc = None, None
            for rnd in ("r02", "r01"):  # the newest capture of this kernel at this config
                try:
                    with open(os.path.join(ROOT, "profiles", f"{rnd}_traffic.json")) as f:
                        t = json.load(f).get(args.config, {}).get(dom)
                except Exception:
                    t = None
                if t and t["units_per_launch"] == units_per_launch and (
                        rnd != "r01" or args.config != "c2"):  # r01's C2 capture is the replaced kernel
                    traffic, tsrc = t, f"profiles/{rnd}_traffic.json"
                    break
            tb = traffic["dram_bytes_per_launch"] if traffic else None
            roof = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                    "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": tb,
                    # what DRAM actually moved per launch at this launch time (the dedup scan
                    # skips the repeated pairs' work, so traffic < algorithmic bytes)
                    "traffic_gbs": round(tb / (per_launch_ms / 1e3) / 1e9, 1) if tb else None,
                    "dram_frac": round(tb / (per_launch_ms / 1e3) / 1e9 / hbm, 4) if tb else None,
                    "traffic_source": tsrc,
                    "bytes_per_unit": bytes_per_unit, "units_per_launch": units_per_launch,
                    "launch_ms": round(per_launch_ms, 4),
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}
            if dom == "scan" and cfg["pool"] == 0:
                # uniform pairs (C1): every pair does r random touches, the pattern of the
                # random-access probe (tools/fetch_probe.cu, profiles/r01_access_probe.txt:
                # red.max / atom.max / ld+atom into 640 MB, at most 5.06 Gpkt/s at r = 5) -- the
                # scan's ceiling is that, not the streaming copy peak
                ceiling = 5060.0
                scan_mpkts = units_per_launch / (per_launch_ms / 1e3) / 1e6
                roof["random_access"] = {"ceiling_mpkts": ceiling, "scan_mpkts": round(scan_mpkts, 1),
                                         "frac": round(scan_mpkts / ceiling, 3),
                                         "source": "tools/fetch_probe.cu best of red, atom and ld+atom into 640 MB, r=5 (profiles/r01_access_probe.txt)"}
            elif dom == "scan" and prof[dom]["launches"] and fresh:
                # Zipf traffic (C2): only the pairs new to their slot stamp their r recorders
                # (random sector read-modify-writes); the rest cost one pair-set probe, whose L2
                # misses are the other random DRAM accesses.  The kernel's DRAM accesses come
                # from the ncu capture of the same kernel (64 B per read fill, 32 B per written
                # sector) at this launch time; the ceiling is the best random-access rate
                # tools/fetch_probe.cu measured on a B200 (profiles/r01_access_probe.txt:
                # 4-byte loads into a 40 GB table at 16 CTAs/SM, 8.94 Gpkt/s x 5 = 44.7 G/s;
                # returning atomics reach 20 G/s at any table size).
                launch_s = per_launch_ms / 1e3
                fresh_pl = fresh / prof[dom]["launches"]
                roof["fresh_pairs_per_launch"] = int(fresh_pl)
                roof["dram_bytes_per_fresh_pair"] = round(tb / fresh_pl, 1) if tb else None
                ra = {"stamp_rmw_per_s": round(fresh_pl * r / launch_s / 1e9, 3), "unit": "G accesses/s",
                      "ceiling_per_s": 44.7,
                      "source": "fresh pairs: device counter of the pipelined dedup scan (sspd_grid_fresh_pairs); "
                                "DRAM accesses: ncu dram__bytes_read/64 + dram__bytes_write/32 of the same kernel "
                                f"({tsrc}); ceiling: tools/fetch_probe.cu best random-load rate "
                                "(profiles/r01_access_probe.txt); stamp atomic ceiling: tools/tlb_probe.cu random "
                                "atom.max into 80 GiB (profiles/r02_tlb_probe.txt)"}
                # the stamps are returning atomics: tools/tlb_probe.cu (profiles/r02_tlb_probe.txt)
                # measured random atom.max on an 80 GiB table at 21.0 G/s (best CTAs/SM; 20-21 G/s
                # at any footprint), so 47M stamps per slot cannot take less than ~2.2 ms
                ra["stamp_atomic_ceiling_per_s"] = 21.0
                ra["stamp_atomic_frac"] = round(fresh_pl * r / launch_s / 21.0e9, 3)
                if traffic:
                    acc = traffic["dram_read"] / 64 + traffic["dram_write"] / 32
                    ra["dram_accesses_per_s"] = round(acc / launch_s / 1e9, 3)
                    ra["frac"] = round(acc / launch_s / 44.7e9, 3)
                    if traffic.get("l2_read_miss_sectors") is not None:
                        # read misses (32 B sectors) minus the streamed pairs' own: the probes'
                        ra["probe_miss_sectors_per_launch"] = int(
                            max(0.0, traffic["l2_read_miss_sectors"] - units_per_launch * 8 / 32))
                roof["random_access"] = ra
    kernels_share = {k2: round(v["ms"] / ms, 4) for k2, v in prof.items()}

    # Detection accuracy of the last timed slot against the generator's
    # truth: the injected super points are the only hosts at or above theta
    # (background hosts draw from 16-entry pools; C1's uniform pairs spread
    # 5e6 pairs over 2^32 hosts).  evaluate() semantics (workload.cpp:360-385).
    truth = {int(L.sspd_synth_super_cip(C.byref(sp), i)) for i in range(cfg["n_super"])}
    got = {d.cip for d in reps} if reps is not None else set()
    accuracy = {"true_supers": len(truth), "reported": len(got),
                "fpr": round(len(got - truth) / max(len(truth), 1), 6),
                "fnr": round(len(truth - got) / max(len(truth), 1), 6),
                "truth": "generator"}
    if world == 1:
        # and against exact distinct counts of the same window, on the device
        # (sspd_exact_counts): the union of the last k slots' pairs
        last = args.warmup + args.steps - 1
        segs = [trace[(last - j) % S] for j in range(min(k, last + 1))]
        try:
            exact = P.exact_counts(segs, min_count=int(np.ceil(theta)), distinct_hint=32 << 20,
                                   device=dev, stream_ptr=stream.cuda_stream)
            ex = set(exact)
            accuracy.update({"exact_true_supers": len(ex),
                             "exact_fpr": round(len(got - ex) / max(len(ex), 1), 6),
                             "exact_fnr": round(len(ex - got) / max(len(ex), 1), 6),
                             "truth": "generator + exact device counts of the window"})
        except Exception as e:
            accuracy["exact"] = f"unavailable: {type(e).__name__}: {e}"

    # --- CPU baseline: the compiled reference on this host ---------------------
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            rr = run_reference(cfg, steps=1, warmup=1, pairs_cap=args.ref_pairs, time_budget_s=150)
            cpu = {"value": round(rr["value"], 3), "unit": unit, "cores": rr["workers"],
                   "kind": "reference",
                   "sample": f"{rr['steps_timed']} slot(s) x {rr['pairs_per_step']} pairs of the "
                             f"same trace after 1 warm-up slot; scan_batch alpha=32768 + "
                             f"reconstruct_leveled + advance_slot, full-size grid in host RAM",
                   "step_ms": round(rr["step_ms"], 1), "reconstruct_ms": round(rr["reconstruct_ms"], 1)}
        except Exception as e:  # report, do not hide
            cpu = {"value": None, "unit": unit, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {type(e).__name__}: {e}"}
        if cpu and cpu["value"] and cfg["pairs_per_slot"] <= 10_000_000:
            # BASELINE.md section 3 also asks for a 1-core row (cheap at the C1
            # geometry): the reference arm in a child process with one OpenMP
            # thread, since hot_sets uses every OpenMP thread whatever `workers` says
            try:
                env = dict(os.environ, OMP_NUM_THREADS="1", SSPD_REF_WORKERS="1")
                out = subprocess.run([sys.executable, os.path.abspath(__file__), "--impl", "reference",
                                      "--config", args.config, "--steps", "1", "--warmup", "1"],
                                     env=env, capture_output=True, text=True, timeout=300)
                r1 = json.loads(out.stdout.strip().splitlines()[-1])
                cpu["one_core"] = {"value": r1["value"], "step_ms": r1["ms_per_step"],
                                   "reconstruct_ms": r1["reconstruct_ms"], "cores": r1["cpu_baseline"]["cores"]}
            except Exception as e:
                cpu["one_core"] = f"failed: {type(e).__name__}: {e}"

    line = {
        "metric": metric, "value": round(value, 3), "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
        "higher_is_better": True, "scaling": "weak",
        # BASELINE.md's only published packets/s is the paper's GSSD 109 Mpkt/s on a
        # GTX 950 at the paper parameters -- the C1 geometry
        "vs_baseline": round(value / 109.0, 2) if args.config == "c1" else None,
        "dtype": {8: "u8 stamps", 16: "u16 stamps", 32: "u32"}[args.stamp_width], "data": "synthetic",
        "config": config_of(cfg),
        "setup": {"stamp_bits": args.stamp_width,
                   "merge": {"pairs": "union-min: all-gather of each router's distinct pairs per slot",
                             "push": "union-min: distinct pairs pushed to peers over NVLink during the scan",
                             "bitmap": "union-min: OR all-reduce of the slot's touched bitmaps",
                             "stamps": "union-min: NCCL all-reduce(max) of the full stamp grid",
                             "shard": "union-min over cells sharded among routers: new pairs relayed over "
                                      "NVLink through pair owners to their cells' owners, hot bits OR- and "
                                      "survivor masks AND-reduced",
                             "auto": "none (single router)"}[merge_used],
                   "parallelism": f"{world} routers, one per GPU"},
        "gbps_800B": round(value * 1e6 * PKT_BYTES * 8 / 1e9, 1),
        # the paper's form: Mpkt/s * 800 * 8 / 1024, i.e. 109 Mpkt/s -> 681.25
        "gbps_800B_paper": round(value * PKT_BYTES * 8 / 1024, 1),
        "reconstruct_ms": round(statistics.mean(recon), 3),
        "reports_last_step": len(reps) if reps is not None else None,
        "accuracy": accuracy,
        "kernels_share": kernels_share,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
