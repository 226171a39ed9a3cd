#!/usr/bin/env python
"""bench.py — samples dispatched/sec of the embedding-sample dispatch path.

One bench step = one dispatch iteration of the reference's run() loop
(sim.hpp:421-441) on the next batch of the reference's Zipf input stream:
expected-cost matrix build -> EcoMix decision (exact Hungarian block +
capacity-bounded greedy) -> per-worker cache update (SimState::step).  The
batches are sequential because each dispatch changes the cache state.

Default workload = BASELINE.json configs[2] ("C3"), the largest configuration
that runs on one GPU (configs[3], C4, is declared 8-GPU sharded): Criteo-shaped,
16 heterogeneous workers (8 x 5 Gbps + 8 x 0.5 Gbps), batch 8192 (m=512), 26
Zipf(1.05) ids per sample over a 10M-id vocabulary, 800K-entry caches, hybrid
dispatcher alpha=0.125 (an exact block of k = 1024 rows).  `prefill`
untimed iterations precede the timed ones.  --config C1/C2/C4/C5 select the
other BASELINE configs (parity-test cases, not the headline).

  value : samples/s with the batches already resident in HBM
  e2e   : samples/s through the C ABI (edx_engine_iterate) from pinned host
          buffers, H2D of the ids and D2H of decision + report inside the
          timed region
  --impl reference : the reference's own CPU dispatcher (oracle/_ref, the
          unmodified headers compiled in place) on this host's cores.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HET = lambda n: [5e9] * (n // 2) + [5e8] * (n - n // 2)
WORKLOADS = {
    "C1": dict(n=4, m=256, L=26, V=100_000, cap=10_000, bw=[5e9] * 4, alpha=0.0, prefill=20,
               desc="C1: Zipf(1.05), 26 fields, batch 1024, 4 uniform workers, 10% cache, greedy only"),
    "C2": dict(n=8, m=128, L=26, V=100_000, cap=10_000, bw=HET(8), alpha=0.5, prefill=20,
               desc="C2: Zipf(1.05), 26 fields, batch 1024, 8 heterogeneous workers "
                    "(4x5Gbps+4x0.5Gbps), 10% cache, hybrid EcoMix alpha=0.5"),
    "C3": dict(n=16, m=512, L=26, V=10_000_000, cap=800_000, bw=HET(16), alpha=0.125, prefill=3,
               desc="C3: Criteo-shaped, 10M ids, batch 8192, 16 heterogeneous workers, alpha=0.125"),
    "C4": dict(n=32, m=512, L=100, V=10_000_000, cap=800_000, bw=HET(32), alpha=0.0625, prefill=2,
               desc="C4: Avazu-shaped, 100 ids/sample, batch 16384, 32 workers, alpha=1/16"),
    # BASELINE configs[4], the scaling sweep (batch 4K-64K x workers 8-64; n=128 has no
    # oracle, the reference rejects n > 64): default = the corner, override with
    # --batch / --workers.
    "C5": dict(n=64, m=1024, L=26, V=10_000_000, cap=800_000, bw=HET(64), alpha=0.0, prefill=1,
               desc="C5: scaling sweep, 26 Zipf ids, 10M-id vocabulary, greedy (alpha 0)"),
}
METRIC = "samples dispatched/sec (cost matrix + hybrid decision + cache update)"
ZIPF_S, SEED = 1.05, 42


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--prefill", type=int, default=None)
    ap.add_argument("--cpu-sample", type=int, default=10, help="timed iterations of cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="do not flush L2 between iterations")
    ap.add_argument("--batch", type=int, default=None, help="C5 sweep: samples per iteration")
    ap.add_argument("--workers", type=int, default=None, help="C5 sweep: workers (<= 64)")
    ap.add_argument("--debug-times", action="store_true", help="per-iteration times in the line")
    ap.add_argument("--no-ncu", action="store_true",
                    help="skip the ncu DRAM-traffic capture of the cost build")
    ap.add_argument("--ncu-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--spread-ids", action="store_true",
                    help="map every id through a bijection onto [0, 2^32) and run the engine "
                         "without an id bound (the device id table; SimState(cfg) semantics)")
    return ap.parse_args()


def workload(args):
    w = dict(WORKLOADS[args.config])
    if args.alpha is not None:
        w["alpha"] = args.alpha
    if args.prefill is not None:
        w["prefill"] = args.prefill
    if args.workers is not None or args.batch is not None:
        if args.config != "C5":
            raise SystemExit("--batch/--workers apply to the C5 sweep only")
        n = args.workers or w["n"]
        if not 1 <= n <= 64:
            raise SystemExit("--workers must lie in [1, 64] (the reference rejects n > 64)")
        R = args.batch or w["n"] * w["m"]
        if R % n:
            raise SystemExit("--batch must be a multiple of --workers")
        w.update(n=n, m=R // n, bw=HET(n))
    w["R"] = w["n"] * w["m"]
    w["spread"] = bool(getattr(args, "spread_ids", False))
    if w["spread"]:
        w["desc"] += "; ids spread over [0, 2^32) (bijection), engine without an id bound"
    if args.config == "C5":
        w["desc"] = f"{w['desc']}: batch {w['R']}, {w['n']} workers"
    return w


def spread(ids):
    """uint32 bijection (odd multiplier mod 2^32): the Zipf ids spread over the
    whole 32-bit range, as hashed feature ids are (tests/scale_state.py)."""
    x = ids.astype(np.uint64)
    return ((x * np.uint64(0x9E3779B1) + np.uint64(0x7F4A7C15)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def batches(w, count):
    """The reference's ZipfStream (workload.hpp:94-133) through the product's
    own host generator (bit-identical; tests/test_host.py pins it)."""
    import paper_2512_21615_b200 as edx
    z = edx.ZipfStream(w["V"], w["L"], ZIPF_S, count, SEED, w["R"])
    out = [ids for ids in z]
    return [spread(b) for b in out] if w.get("spread") else out


def reference_batches(w, count):
    """The same stream from the reference's own ZipfStream (oracle/_ref), so
    the reference arm maps no product library."""
    orc, _ = reference_oracle()
    out = list(orc.zipf_batches(w["V"], w["L"], ZIPF_S, count, SEED, w["R"]))
    return [spread(b) for b in out] if w.get("spread") else out


def parallelism(world):
    return (f"row-sharded cost build x{world}, NCCL gather to rank 0, rank-0 solve, decision "
            "broadcast, replicated cache update" if world > 1 else "1 GPU")


def config_json(w, args, extra=None):
    c = {"workload": w["desc"], "n_workers": w["n"], "m": w["m"], "batch": w["R"],
         "ids_per_sample": w["L"], "id_space": w["V"], "cache_per_worker": w["cap"],
         "alpha": w["alpha"], "zipf_s": ZIPF_S, "seed": SEED,
         "prefill_iterations": w["prefill"],
         "l2": "flushed between timed iterations (256 MiB write)" if not args.no_flush
         else "not flushed"}
    if extra:
        c.update(extra)
    return c


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.gpu_idle,"
              "clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        names = ["gpu_idle", "sw_power_cap", "hw_slowdown", "hw_thermal_slowdown",
                 "sw_thermal_slowdown"]
        sm, mx, reasons = [], 0, set()
        for l in getattr(self, "lines", []):
            p = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, p[3:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- product arm
def fp64_adds(w, ids, glob):
    """F_alg = sum over (cell, id) with the latest copy not on the
    cell's worker of (1 + popcount(owners)) -- per id occurrence,
    (n - popcount(latest)) * (1 + popcount(owners)) -- from the state the build reads."""
    gid, ow, la, _ = glob
    order = np.argsort(gid)
    sid = gid[order]
    pos = np.minimum(np.searchsorted(sid, ids), max(len(sid) - 1, 0))
    hit = (sid[pos] == ids) if len(sid) else np.zeros(len(ids), bool)
    o = np.where(hit, ow[order][pos], 0).astype(np.uint64)
    l = np.where(hit, la[order][pos], 0).astype(np.uint64)
    nl = w["n"] - np.bitwise_count(l).astype(np.int64)
    return int(np.sum(nl * (1 + np.bitwise_count(o).astype(np.int64))))


def algorithmic_build_bytes(w, ids):
    """B_alg = 4 R L (ids) + 16 U (owners+latest per unique id)
    + 8 n (unit costs) + 8 R n (matrix write)."""
    U = len(np.unique(ids))
    return 4 * w["R"] * w["L"] + 16 * U + 8 * w["n"] + 8 * w["R"] * w["n"], U


def product(args, w, rank, world, local_rank):
    import torch
    import paper_2512_21615_b200 as edx

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n, m, L, R = w["n"], w["m"], w["L"], w["R"]
    K, W, P = args.steps, args.warmup, w["prefill"]
    total = P + 2 * (W + K) + 1  # +1: the batch the last timed e2e step prefetches
    host = batches(w, total)
    offs = np.arange(R + 1, dtype=np.uint64) * np.uint64(L)
    cfg = edx.ClusterConfig(n=n, m=m, bandwidths_bps=w["bw"], d_tran_bytes=2048,
                            cache_capacity=w["cap"], alpha=w["alpha"])
    nccl_id = None
    if world > 1:  # rank 0's ncclUniqueId, shared over the torch process group
        import torch.distributed as dist
        buf = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(edx.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())
    eng = edx.SimState(cfg, id_space=0 if w["spread"] else w["V"], max_batch_ids=R * L,
                       device=local_rank, rank=rank,
                       world_size=world, nccl_id=nccl_id)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=dev)
    flush = None if args.no_flush else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # prefill to steady state (untimed)
    for b in host[:P]:
        eng.iterate(b, offs, want_decision=False)

    # ---- value: inputs resident in HBM
    seg = host[P:P + W + K]
    d_ids = torch.from_numpy(np.stack(seg).view(np.int32)).to(dev)
    d_offs = torch.from_numpy(offs.view(np.int64)).to(dev)
    torch.cuda.synchronize()

    def one_resident(i):  # the reference's run() body as one fused call (a CUDA-graph replay)
        return eng.iterate_device(d_ids[i].data_ptr(), d_offs.data_ptr(), R, R * L,
                                  want_decision=False, want_expected=False)

    def one_profiled(i):  # the same iteration phase by phase, CUDA events per phase
        eng.load(None, on_device=True, ids_ptr=d_ids[i].data_ptr(), offsets_ptr=d_offs.data_ptr(),
                 rows=R, total_ids=R * L)
        eng.build(None)
        eng.dispatch(want_decision=False, want_expected=False)
        return eng.step()

    def timed(fn, idx):
        starts = [torch.cuda.Event(enable_timing=True) for _ in idx]
        ends = [torch.cuda.Event(enable_timing=True) for _ in idx]
        for t, i in enumerate(idx):
            if flush is not None:
                with torch.cuda.stream(stream):
                    flush.fill_(t & 0xFF)
            starts[t].record(stream)
            fn(i)
            ends[t].record(stream)
        torch.cuda.synchronize()
        return [s.elapsed_time(e) for s, e in zip(starts, ends)]

    for i in range(W):
        one_resident(i)
    # FP64 adds of the first timed build, from the state it reads (untimed)
    f_alg = fp64_adds(w, seg[W], eng.global_masks()) if world == 1 else None
    eng.phase_times(reset=True)
    with ClockSampler(local_rank) as clk:
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ms = timed(one_resident, range(W, W + K))
        torch.cuda.synchronize()
    _, counts = eng.phase_times(reset=True)
    launches = int(counts[0])
    # phase breakdown (not part of `value`): the next iterations, phase by phase
    eng.set_profiling(True)
    eng.phase_times(reset=True)
    timed(one_profiled, range(W, W + K))
    phase_ms, counts = eng.phase_times(reset=True)
    eng.set_profiling(False)
    solver_steps = int(counts[1])
    step_ms = sum(ms) / K

    # ---- K8 baseline_hitgreedy latency on the same resident batches (reported
    # beside the metric), on a copy of the state's clock
    hg_ms = None
    if world == 1:
        def one_hitgreedy(i):
            eng.load(None, on_device=True, ids_ptr=d_ids[i].data_ptr(),
                     offsets_ptr=d_offs.data_ptr(), rows=R, total_ids=R * L)
            eng.dispatch_hitgreedy(want_decision=False)
        one_hitgreedy(W)
        hg = timed(one_hitgreedy, range(W, W + K))
        hg_ms = sum(hg) / K

    # ---- e2e: through edx_engine_iterate from pinned host buffers
    seg2 = host[P + W + K:]
    pinned = torch.from_numpy(np.stack(seg2).view(np.int32)).pin_memory()
    pinned_offs = torch.from_numpy(offs.view(np.int64)).pin_memory()
    pin_np = pinned.numpy().view(np.uint32)
    poffs_np = pinned_offs.numpy().view(np.uint64)
    # batch i+1's host->device copy is issued (edx_engine_prefetch, copy stream,
    # double-buffered) before iteration i runs -- the paper's pipelined input
    # loading; every step still copies its own batch inside the timed region
    def one_e2e(i):
        nxt = (pin_np[i + 1], poffs_np) if i + 1 < len(pin_np) else None
        return eng.iterate(pin_np[i], poffs_np, prefetch_next=nxt)

    eng.prefetch(pin_np[0], poffs_np)
    for i in range(W):
        one_e2e(i)
    e2e_ms = timed(one_e2e, range(W, W + K))
    e2e_step_ms = sum(e2e_ms) / K

    # ---- roofline of the cost build (K1), per launch
    b_alg, uniq = zip(*(algorithmic_build_bytes(w, host[P + W + i]) for i in range(K)))
    t_build_ms = phase_ms[0] / K
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    achieved = (sum(b_alg) / K) / (t_build_ms * 1e-3) / 1e9 if t_build_ms > 0 else None
    dadd_peak = None
    try:
        dadd_peak = json.load(open(os.path.join(ROOT, "profiles", "r01_dadd_peak.json")))["dadd_per_s"]
    except (OSError, ValueError, KeyError):
        pass
    fp64_rate = f_alg / (t_build_ms * 1e-3) if (f_alg and t_build_ms > 0) else None
    kernels = eng.last_kernels()
    traffic = None if (args.no_ncu or world > 1) else ncu_build_traffic(args, kernels["build"])

    out = {
        "metric": METRIC, "value": R / (step_ms * 1e-3), "unit": "samples/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": step_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference ZipfStream (s=1.05, seed 42), state warmed by prefill",
        "config": config_json(w, args, {"parallelism": parallelism(world)}),
        "e2e": {"value": R / (e2e_step_ms * 1e-3), "unit": "samples/s",
                "ms_per_step": e2e_step_ms,
                "note": "edx_engine_iterate from pinned host buffers; the next batch's H2D is "
                        "prefetched on the engine's copy stream during each iteration",
                "h2d_bytes_per_step": R * L * 4 + (R + 1) * 8,
                "d2h_bytes_per_step": R * 4 + 8 + (3 * n + 4) * 8},
        "roofline": {"kernel": kernels["build"] + " (K1, cost.hpp:81-125)",
                     "bound": "hbm",
                     "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": (achieved / hbm_peak) if achieved else None,
                     "traffic": traffic["dram_bytes"] if traffic else None,
                     "traffic_source": traffic["source"] if traffic else
                     "not captured (--no-ncu, N > 1, or ncu unavailable)",
                     "traffic_launch_ns_ncu": traffic["ncu_ns"] if traffic else None,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else
                     "fallback 6.65 TB/s",
                     "algorithmic_bytes_per_launch": sum(b_alg) / K,
                     "unique_ids_per_batch": sum(uniq) / K, "launch_ms": t_build_ms,
                     "fp64": {"adds_per_launch": f_alg, "achieved_adds_per_s": fp64_rate,
                              "peak_adds_per_s": dadd_peak,
                              "frac": (fp64_rate / dadd_peak) if (fp64_rate and dadd_peak) else None,
                              "peak_source": "profiles/r01_dadd_peak.json (tools/dadd_peak.cu)",
                              "note": "second roof of the build (sequential fp64 add chains, "
                                      "SURVEY 8d); adds counted on the first timed batch"}},
        "dominant_kernel": dominant_kernel(kernels, phase_ms),
        "kernels": kernels,
        "solver": {"exact_rows": n * int(np.floor(m * w["alpha"] + 1e-9)),
                   "latency_ms_per_batch": phase_ms[2] / K,
                   "dijkstra_steps_last_batch": solver_steps,
                   "ns_per_step": (phase_ms[2] / K) * 1e6 / solver_steps if solver_steps else None},
        "phases_note": "per-phase CUDA events on a separate profiled pass (phase-by-phase calls); "
                       "the timed value runs each iteration as one CUDA-graph replay",
        "phases_ms_per_step": {"build": phase_ms[0] / K, "gap_sort": phase_ms[1] / K,
                               "exact_solve": phase_ms[2] / K, "greedy": phase_ms[3] / K,
                               "cache_update": phase_ms[4] / K, "dispatch_total": phase_ms[5] / K},
        "build_decide": {"value": R / ((phase_ms[0] + phase_ms[5]) / K * 1e-3),
                         "unit": "samples/s",
                         "note": "reference timing regions only (matrix_s + decision_s, "
                                 "sim.hpp:423-432)"},
        "hitgreedy": {"ms_per_batch": hg_ms, "note": "baseline_hitgreedy (assign.hpp:346-392) "
                      "on the resident batches after the timed region: scores, order, assignment"},
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    if args.debug_times:
        out["debug_times"] = {"value_ms": ms, "e2e_ms": e2e_ms}
    return out, host[:P + W + K], offs


# ------------------------------------------------------------ reference arm
def reference_oracle():
    from oracle import pyoracle
    if os.path.exists(pyoracle.REF_SO):
        return pyoracle.Oracle("reference"), "reference"
    if not os.path.exists(pyoracle.PORT_SO):
        pyoracle.build(ref=False)
    return pyoracle.Oracle("port"), "port"


def cpu_run(w, host, offs, prefill, warmup, steps, threads):
    """Reference iterations (orc_ref_iteration: snapshot, build, ecomix, step)
    on host cores; returns per-iteration seconds of the timed ones."""
    from oracle import pyoracle
    orc, kind = reference_oracle()
    sim = orc.sim(pyoracle.Cfg(w["n"], w["m"], w["bw"], cap=w["cap"], alpha=w["alpha"]))
    times, bd = [], []
    for i, ids in enumerate(host[:prefill + warmup + steps]):
        t0 = time.perf_counter()
        _, _, _, ph = sim.iteration(ids, offs, threads=threads)
        dt = time.perf_counter() - t0
        if i >= prefill + warmup:
            times.append(dt)
            bd.append(ph[1] + ph[2])
    return times, bd, kind


def cpu_baseline(w, host, offs, sample):
    import platform
    P = w["prefill"]
    times, bd, kind = cpu_run(w, host, offs, P, 0, sample, threads=1)
    cpu = platform.processor() or ""
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                cpu = l.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    mean = sum(times) / len(times)
    return {"value": w["R"] / mean, "unit": "samples/s", "cores": 1, "kind": kind,
            "sample": f"{w['desc'].split(':')[0]} iterations {P}..{P + sample - 1} after {P} "
                      f"untimed prefill iterations, reference run() body "
                      f"(snapshot+build_matrix+ecomix+step), 1 thread as shipped",
            "ms_per_step": mean * 1e3,
            "build_decide_samples_per_s": w["R"] / (sum(bd) / len(bd)),
            "host_cpu": cpu, "host_nproc": os.cpu_count()}


def reference_arm(args, w, rank, world):
    if rank != 0:
        return None
    threads = os.cpu_count() or 1
    K, W, P = args.steps, args.warmup, w["prefill"]
    host = reference_batches(w, P + W + K)
    offs = np.arange(w["R"] + 1, dtype=np.uint64) * np.uint64(w["L"])
    times, bd, kind = cpu_run(w, host, offs, P, W, K, threads=threads)
    mean = sum(times) / len(times)
    value = w["R"] / mean
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": mean * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference ZipfStream (s=1.05, seed 42), state warmed by prefill",
        "config": config_json(w, args, {"parallelism": parallelism(world)}),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": kind,
                         "sample": f"iterations {P + W}..{P + W + K - 1}; build_matrix rows "
                                   f"split over {threads} threads (bit-identical), ecomix and "
                                   f"step single-threaded as in the reference"},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "build_decide": {"value": w["R"] / (sum(bd) / len(bd)), "unit": "samples/s"},
    }


def dominant_kernel(kernels, phase_ms):
    """The phase with the largest device time (profiled pass) and the kernel
    the engine launched for it (edx_engine_last_kernels)."""
    names = {
        0: f"{kernels['build']} (K1 cost build, cost.hpp:81-125)",
        2: f"{kernels['solver']} (K6 exact EcoMix block, assign.hpp:80-157; latency-bound)",
        3: f"{kernels['greedy']} (K4 EcoMix greedy, assign.hpp:162-192)",
        4: "K7 step kernels (cache update, sim.hpp:87-218)",
    }
    return names[max(names, key=lambda i: phase_ms[i])]


# ------------------------------------------------- K1 DRAM traffic (ncu)
def ncu_child(args, w):
    """Run under ncu by ncu_build_traffic: the product engine, eagerly (no
    CUDA graph), over the same prefill + warm-up batches as the timed run,
    then ONE cost build of the first timed batch -- the launch ncu captures."""
    import paper_2512_21615_b200 as edx
    n, m, L, R = w["n"], w["m"], w["L"], w["R"]
    P, W = w["prefill"], args.warmup
    host = batches(w, P + W + 1)
    offs = np.arange(R + 1, dtype=np.uint64) * np.uint64(L)
    cfg = edx.ClusterConfig(n=n, m=m, bandwidths_bps=w["bw"], d_tran_bytes=2048,
                            cache_capacity=w["cap"], alpha=w["alpha"])
    eng = edx.SimState(cfg, id_space=0 if w["spread"] else w["V"], max_batch_ids=R * L)
    for b in host[:P + W]:
        eng.iterate(b, offs, want_decision=False)
    eng.load((host[P + W], offs))
    eng.build(None)
    eng.dispatch(want_decision=False, want_expected=False)


def ncu_build_traffic(args, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum of the first timed batch's
    cost-build launch, captured by ncu in a child process of this run (cold L2,
    as the timed loop's flush makes it)."""
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None
    w = workload(args)
    skip = w["prefill"] + args.warmup
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--print-units", "base", "--csv",
           "-k", "regex:^k_cost_build", "--launch-skip", str(skip), "--launch-count", "1",
           sys.executable, os.path.abspath(__file__), "--ncu-child", "--config", args.config,
           "--warmup", str(args.warmup)]
    for flag, val in (("--alpha", args.alpha), ("--prefill", args.prefill),
                      ("--batch", args.batch), ("--workers", args.workers)):
        if val is not None:
            cmd += [flag, str(val)]
    if args.spread_ids:
        cmd.append("--spread-ids")
    env = dict(os.environ, EDX_GRAPH="0")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    except (OSError, subprocess.TimeoutExpired):
        return None
    vals = {}
    import csv
    rows = [l for l in r.stdout.splitlines() if l.startswith('"')]
    for rec in csv.DictReader(rows):
        name, val = rec.get("Metric Name"), rec.get("Metric Value", "").replace(",", "")
        if name and val:
            try:
                vals[name] = float(val)
            except ValueError:
                pass
    if "dram__bytes_read.sum" not in vals:
        return None
    return {"dram_bytes": vals["dram__bytes_read.sum"] + vals.get("dram__bytes_write.sum", 0.0),
            "ncu_ns": vals.get("gpu__time_duration.sum"),
            "source": f"ncu in this run: {kernel}, launch {skip} (first timed batch), "
                      "dram__bytes_read.sum + dram__bytes_write.sum, cold L2"}


def emit(out, fd):
    os.write(fd, (json.dumps(out) + "\n").encode())


def main():
    args = parse()
    # native libraries write to fd 1 (NCCL's version banner at communicator
    # init): route everything else to stderr, keep stdout for the one JSON line
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    w = workload(args)
    if args.ncu_child:
        ncu_child(args, w)
        return
    if args.impl == "reference":
        out = reference_arm(args, w, rank, world)
        if out is not None:
            emit(out, json_fd)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out, host, offs = product(args, w, rank, world, local_rank)
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([out["ms_per_step"], out["e2e"]["ms_per_step"]], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["ms_per_step"], out["e2e"]["ms_per_step"] = float(t[0]), float(t[1])
        out["value"] = w["R"] / (out["ms_per_step"] * 1e-3)
        out["e2e"]["value"] = w["R"] / (out["e2e"]["ms_per_step"] * 1e-3)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(w, host, offs, args.cpu_sample)
        emit(out, json_fd)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
