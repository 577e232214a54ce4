"""bench.py -- WAH index build throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

Workload (BASELINE.json configs[3], the north-star size): per GPU 2^28 uint32
values, Zipf(s=1) over 65,536 keys, generated with the reference's own
libstdc++ distributions (mt19937_64(42 + rank)).  A "step" is one full index
build (plan -> sort -> emit -> table) over that column.

  value  whole-job values/s with the keys already resident in HBM, device
         time from CUDA events on the launch stream, max over ranks.
  e2e    the same metric through the public host API per step: pinned keys
         H2D, the four stages, counts + words + table D2H.
  roofline  the dominant stage's algorithmic bytes / its live event time,
         against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  the reference's reference_index (1 thread, oracle/_ref) on a
         bounded sample of the same stream, rank 0 at N=1.

--impl reference runs the reference's own data-parallel CPU build
(wah::build_index on its simulated device, all host threads) on a bounded
sample per step (rank 0 only; other ranks exit 0).
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

METRIC = "WAH index build values/sec"
UNIT = "values/s"

CONFIGS = {
    "C4": dict(desc="WAH index build, 2^28 uint32 values per GPU, Zipf(s=1) over 65536 keys",
               n=1 << 28, kind="zipf", k=65536, seed=42),
    "C3": dict(desc="WAH index build, 2^26 uint32 values per GPU, 1024 uniform keys (4-stage chain)",
               n=1 << 26, kind="uniform", k=1024, seed=1),
    "C5": dict(desc="WAH index build, 2^30 uint32 values, 65536 uniform keys",
               n=1 << 30, kind="uniform", k=65536, seed=1),
}


def gen_values(cfg, n, rank, out=None):
    from paper_1709_07781_b200 import gen

    if cfg["kind"] == "zipf":
        return gen.zipf(cfg["seed"] + rank, n, cfg["k"], 1.0, out)
    return gen.uniform(cfg["seed"] + rank, n, cfg["k"], out)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def b_alg(n, W, D, passes):
    """algorithmic bytes of a build, (8 + 16 P) N + 4 W + 12 D."""
    return (8 + 16 * passes) * n + 4 * W + 12 * D


def b_min(n, W, D):
    """The compulsory floor: read the keys, write words + table."""
    return 4 * n + 4 * W + 12 * D


def golden_digest(cfg, n):
    """The reference's digest of this workload (tests/golden/digests.json,
    generated from oracle/_ref), or None when no fixture covers it."""
    p = os.path.join(ROOT, "tests", "golden", "digests.json")
    try:
        with open(p) as f:
            d = json.load(f)
    except OSError:
        return None
    for w in d.get("workloads", []) + d.get("gpu_workloads", []):
        if (w["kind"], w["seed"], w["n"], w["k"]) == (cfg["kind"], cfg["seed"], n, cfg["k"]):
            return w["digest"]
    return None


def device_result_digest(n, d_counts, d_words, d_entries):
    """Digest of an index left in HBM by the actor chain: counts, words and
    table copied to the host, FNV-1a-64 of the WAH1 bytes in native code."""
    from paper_1709_07781_b200 import ndx
    from paper_1709_07781_b200.runtime import index_digest

    L = ndx.load()
    c = np.zeros(4, np.uint64)
    ndx.check(L.ndx_memcpy_d2h_async(c.ctypes.data, d_counts, 24, None), "d2h counts")
    ndx.check(L.ndx_device_synchronize(), "sync")
    W, D = int(c[0]), int(c[1])
    w = np.empty(max(W, 1), np.uint32)
    e = np.empty(max(3 * D, 1), np.uint32)
    if W:
        ndx.check(L.ndx_memcpy_d2h_async(w.ctypes.data, d_words, 4 * W, None), "d2h words")
    if D:
        ndx.check(L.ndx_memcpy_d2h_async(e.ctypes.data, d_entries, 12 * D, None), "d2h entries")
    ndx.check(L.ndx_device_synchronize(), "sync")
    return "%016x" % index_digest(n, e[: 3 * D], w[:W]), W, D


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the
    timed region (nvidia-smi -lms in the background)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the first sample land before the timed region
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        rows = [[x.strip() for x in ln.split(",")] for ln in out.strip().splitlines() if ln.strip()]
        sm = [float(r[0]) for r in rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        busy = [s for s in sm if s > 0.5 * (max(mx) if mx else 0)] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 4 + i and
                          r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or getattr(args, "force_sharded", False):
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        # NCCL runs inside the C++ runtime (libndactor dlopens it); its
        # communicator lines go to stderr (stdout carries one JSON line).
        # torch.distributed (gloo, CPU) only bootstraps: the NCCL id, host
        # barriers, the max over ranks.
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        if args.impl == "ours":
            torch.cuda.set_device(local)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


def ref_values(cfg, n, rank=0):
    """The same synthetic stream from the reference's own generators
    (oracle/_ref: libstdc++ distributions), so the CPU legs never load the
    product libraries; the C restatement's stream when oracle/_ref is absent."""
    import oracle

    seed = cfg["seed"] + rank
    if oracle.Reference.available():
        r = oracle.Reference()
        return r.gen_zipf(seed, n, cfg["k"], 1.0) if cfg["kind"] == "zipf" else r.gen_uniform(seed, n, cfg["k"])
    raise RuntimeError("oracle/_ref/libndref.so missing: build it with make -C oracle")


def cpu_baseline(cfg):
    """reference_index (the reference's CPU path, 1 thread) on a bounded sample."""
    import oracle

    n = 1 << 25
    v = ref_values(cfg, n)
    if oracle.Reference.available():
        impl, kind = oracle.Reference(), "reference"
    else:
        impl, kind = oracle.Port(), "port"
    t0 = time.perf_counter()
    impl.digest_of(v)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"wah::reference_index, 1 thread, first 2^25 values of the same stream "
                      f"({dt:.1f} s)"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, cfg):
    """The reference's own data-parallel CPU build, wah::build_index on its
    simulated device (p/core/src/wah_builder.cpp:38-307), compiled from the
    reference sources into oracle/_ref.  Inputs come from the reference's
    generators; nothing of the product package is imported or loaded."""
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return 0
    import oracle

    n = args.ref_sample
    v = ref_values(cfg, n)
    cores = os.cpu_count() or 1
    if not oracle.Reference.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libndref.so was not built"}))
        return 0
    ref = oracle.Reference()
    # all host threads as compute units, 8-bit digits
    # at N >= 2^26 (16-bit digits need 4N-entry histograms per pass)
    build = lambda: ref.build_index_sim(v, cores, 8)  # noqa: E731
    what = f"wah::build_index on the reference's simulated device, {cores} compute units, 8-bit digits"
    for _ in range(args.warmup):
        build()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        build()
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    value = n / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": cfg["desc"], "sample_values_per_step": n,
                   "sample": f"first {n} values of the config's stream (reference generator)",
                   "cpu": cpu_model(), "nproc": cores},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{what}; the first {n} values of the same stream per step, median of {args.steps}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def json_stdout():
    """The one JSON line goes to the real stdout; anything native code prints
    there (NCCL's banner) is sent to stderr instead."""
    out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    return out


def run_sharded(args, cfg, world, rank, local):
    """N > 1 (or --force-sharded): one process per GPU.  The column is split
    into 31-aligned row shards; each step, on every rank and stream-ordered
    on its GPU with no host round trip (include/ndactor/wah_dist.hpp):
      1. the shard's build through the shard chain of compute actors
         (plan * sort * emit * table * meta, global row ids);
      2. one NCCL group (from the C++ runtime): all-gather of every shard's
         counts and per-value metadata;
      3. the boundary merge plan on the GPU, replicated;
      4. the word exchange as one kernel: each rank copies its owned value
         range of the merged words straight out of the other GPUs' word
         buffers over NVLink.
    `value` times steps 1-4.  The gather of the whole index to rank 0 (the
    same step with rank 0 pulling every word) is timed beside it.
    Scaling: strong by default (the config's column split over the ranks:
    C4 = 2^28 values in total); --scaling weak gives every rank the config's
    size (total rows must stay below 2^31: the index format's u32 offsets)."""
    import torch
    import torch.distributed as dist

    from paper_1709_07781_b200 import shard
    from paper_1709_07781_b200.runtime import DistBuild, Runtime

    jout = json_stdout()
    strong = args.scaling == "strong"
    n_total = (args.n or cfg["n"]) * (1 if strong else world)
    if n_total >= 1 << 31:
        raise SystemExit(f"{n_total} rows: a build takes fewer than 2^31 (use --scaling strong)")
    bounds = shard.shard_bounds(n_total, world).astype(np.int64)
    base, n_r = int(bounds[rank]), int(bounds[rank + 1] - bounds[rank])
    local_cap = int(np.max(np.diff(bounds)))
    dev = torch.device("cuda", local)
    host_keys = torch.empty(max(n_r, 1), dtype=torch.int32, pin_memory=True)
    if strong:  # one global column: every rank makes the stream and keeps its shard
        col = gen_values(cfg, n_total, 0)
        host_keys.numpy().view(np.uint32)[:n_r] = col[base:base + n_r]
        del col
    else:
        gen_values(cfg, n_r, rank, host_keys.numpy().view(np.uint32))
    keys = host_keys.to(dev)

    rt = Runtime(device=local)
    obj = [DistBuild.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    meta_cap = 1 << 16 if cfg["k"] <= 1 << 16 else max(1 << 16, local_cap)
    d = DistBuild(rt, rank, world, obj[0], local_cap, meta_cap, 2 * n_total + 64)
    rts = torch.cuda.ExternalStream(rt.stream, device=dev)

    def barrier():
        rt.synchronize()
        torch.cuda.synchronize(dev)
        dist.barrier()

    def max_over_ranks(x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(steps, gather):
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(rts)
        for _ in range(steps):
            d.step(keys.data_ptr(), n_r, base, gather_all=gather and rank == 0)
        rt.synchronize()  # every stage issued (actor hops) and done
        a1.record(rts)
        a1.synchronize()
        t = a0.elapsed_time(a1) / steps
        barrier()
        return max_over_ranks(t)

    W_ = max(args.warmup, 3)
    K = args.steps
    for _ in range(W_):
        d.step(keys.data_ptr(), n_r, base)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ms = timed(K, False)
    clk = clocks.stop()
    value = n_total / (ms * 1e-3)

    # results of the last owned-slice step: totals, bounds; then the gather
    from paper_1709_07781_b200 import ndx
    L = ndx.load()

    def read_totals():
        o = d.outputs()
        tot = np.zeros(4, np.uint64)
        bnd = np.zeros(world + 1, np.uint64)
        ndx.check(L.ndx_memcpy_d2h_async(tot.ctypes.data, o["totals"], 32, None), "d2h")
        ndx.check(L.ndx_memcpy_d2h_async(bnd.ctypes.data, o["bounds"], 8 * (world + 1), None), "d2h")
        ndx.check(L.ndx_device_synchronize(), "sync")
        return o, tot, bnd

    _, tot, bnd = read_totals()
    owned_ok = int(tot[2]) == 0
    gather_ms = timed(max(1, min(K, 5)), True)
    o, tot_g, _ = read_totals()
    D, W = int(tot_g[0]), int(tot_g[1])
    check = {"error_flags": int(tot_g[2]), "words": W, "distinct": D}
    if rank == 0:
        from paper_1709_07781_b200.runtime import index_digest

        ent = np.zeros(3 * D, np.uint32)
        words = np.zeros(W, np.uint32)
        ndx.check(L.ndx_memcpy_d2h_async(ent.ctypes.data, o["entries"], 12 * D, None), "d2h")
        ndx.check(L.ndx_memcpy_d2h_async(words.ctypes.data, o["slice"], 4 * W, None), "d2h")
        ndx.check(L.ndx_device_synchronize(), "sync")
        dg = "%016x" % index_digest(n_total, ent, words)
        want = golden_digest(cfg, n_total) if strong else None
        check.update({"digest": dg, "golden": want, "ok": int(tot_g[2]) == 0 and owned_ok and
                      (want is None or dg == want)})

    # end to end: every step uploads this rank's pinned keys; rank 0 reads the
    # merged table back, every rank its owned slice
    e2e_steps = max(1, min(K, args.e2e_steps))
    slice_words = int(bnd[rank + 1] - bnd[rank])
    hw = torch.empty(max(slice_words, 1), dtype=torch.int32, pin_memory=True)
    he = torch.empty(max(3 * D, 1), dtype=torch.int32, pin_memory=True)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        kk = host_keys.to(dev, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        d.step(kk.data_ptr(), n_r, base)
        rt.synchronize()
        oo = d.outputs()
        ndx.check(L.ndx_memcpy_d2h_async(hw.data_ptr(), oo["slice"], 4 * slice_words, None), "d2h")
        if rank == 0:
            ndx.check(L.ndx_memcpy_d2h_async(he.data_ptr(), oo["entries"], 12 * D, None), "d2h")
        ndx.check(L.ndx_device_synchronize(), "sync")
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / e2e_steps)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W_, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": cfg["desc"] + (f" -- {n_total} values split over {world} GPUs" if strong else
                                               f" -- {n_r} values per GPU"),
                   "values_total": n_total, "values_per_gpu": n_r, "keys": cfg["k"],
                   "distribution": "zipf s=1" if cfg["kind"] == "zipf" else "uniform",
                   "l2": "inputs larger than L2" if n_r * 4 > 126 << 20 else "inputs may fit L2 (strong scaling)",
                   "parallelism": f"row shards x{world} (31-aligned), NCCL all-gather of the shard metadata, "
                                  f"merge plan on the GPU, owned-slice word exchange over NVLink peer memory",
                   "words": W, "distinct": D,
                   "path": "per rank: shard chain of compute actors (plan*sort*emit*table*meta) -> NCCL group "
                           "all-gather (C++ runtime) -> ndx_dist_plan -> ndx_dist_pull (one kernel reading the "
                           "other GPUs' words); no host round trip inside a step"},
        "gather_to_rank0_ms": gather_ms,
        "result_check": check,
        "e2e": {"value": n_total / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 4 * n_r,
                "d2h_bytes_per_step": 4 * slice_words + (12 * D if rank == 0 else 0), "ms_per_step": e2e_ms},
        # per step: the shard chain's 13 kernels (plan 2, sort 5, emit 4, table 1,
        # meta 1), the merge plan's 7 (5 + two scans) and the pull (N > 1)
        "gpu_launches": (13 + 7 + (1 if world > 1 else 0)) * K,
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), file=jout, flush=True)
    d.close()
    rt.close()
    dist.destroy_process_group()
    return 0


def extra_config(rt, raw, dev, K, W_, name="C3"):
    """BASELINE config 3 beside the headline: 2^26 uniform values over 1024
    keys through the same 4-stage actor chain (device-resident keys, CUDA
    events on the runtime stream) plus its per-stage times."""
    import torch

    c = CONFIGS[name]
    n = c["n"]
    keys = torch.from_numpy(gen_values(c, n, 0).view(np.int32)).to(dev)
    rts = torch.cuda.ExternalStream(rt.stream, device=dev)
    for _ in range(W_):
        rt.build_index_device(keys.data_ptr(), n)
    rt.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(rts)
    for _ in range(K):
        ptrs = rt.build_index_device(keys.data_ptr(), n)
    rt.synchronize()  # every stage issued (actor hops, launcher ring) and done
    a1.record(rts)
    a1.synchronize()
    ms = a0.elapsed_time(a1) / K
    dg, _, _ = device_result_digest(n, *ptrs)
    want = golden_digest(c, n)
    stream = torch.cuda.current_stream()
    calls = raw.stage_calls(keys, n, row_base=0, stream=stream)
    for _, cl in calls:
        cl()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(calls) + 1)] for _ in range(K)]
    for k in range(K):
        ev[k][0].record(stream)
        for i, (_, cl) in enumerate(calls):
            cl()
            ev[k][i + 1].record(stream)
    torch.cuda.synchronize(dev)
    stage_ms = {nm: sum(ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(K)) / K
                for i, (nm, _) in enumerate(calls)}
    W, D = raw.counts()
    raw_ms = sum(stage_ms.values())
    return {"workload": c["desc"], "value": n / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "stage_ms": stage_ms, "raw_launch_ms": raw_ms, "chain_overhead_vs_raw": ms / raw_ms - 1.0,
            "gbs_alg": b_alg(n, W, D, 1) / (ms * 1e-3) / 1e9,
            "words": W, "distinct": D, "data": "synthetic (mt19937(1), uniform)",
            "result_digest": dg, "golden_digest": want, "result_check_ok": want is not None and dg == want}


def run_ours(args, cfg):
    import torch

    from paper_1709_07781_b200 import ndx
    from paper_1709_07781_b200.runtime import Runtime

    world, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    if world > 1 or args.force_sharded:
        return run_sharded(args, cfg, world, rank, local)
    dev = torch.device("cuda", local)
    n = args.n or cfg["n"]

    host_keys = torch.empty(n, dtype=torch.int32, pin_memory=True)
    gen_values(cfg, n, rank, host_keys.numpy().view(np.uint32))
    keys = host_keys.to(dev)
    torch.cuda.synchronize(dev)

    rt = Runtime(device=local)                   # actor chain: table*emit*sort*plan
    rts = torch.cuda.ExternalStream(rt.stream, device=dev)
    raw = ndx.WahBuilder(n, device=local)        # the same kernels launched raw
    stream = torch.cuda.current_stream()
    calls = raw.stage_calls(keys, n, row_base=0, stream=stream)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    W_ = max(args.warmup, 3)
    K = args.steps
    for _ in range(W_):
        rt.build_index_device(keys.data_ptr(), n)
        for _, c in calls:
            c()
    rt.synchronize()
    barrier()

    # ---- headline: the actor chain on HBM-resident keys (1 GiB/GPU > 126 MB L2)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    a0 = torch.cuda.Event(enable_timing=True)
    a1 = torch.cuda.Event(enable_timing=True)
    a0.record(rts)
    for _ in range(K):
        ptrs = rt.build_index_device(keys.data_ptr(), n)
    # the requests return once queued: the stages reach the stream through
    # the actor hops and the launcher thread, so the end event is recorded
    # only after everything was issued and has finished
    rt.synchronize()
    a1.record(rts)
    barrier()
    a1.synchronize()
    ms = max_over_ranks(a0.elapsed_time(a1) / K)

    # ---- content check of the headline result (the actor chain's index in
    #      HBM) against the reference's digest of this workload
    chain_digest, _, _ = device_result_digest(n, *ptrs)
    want_digest = golden_digest(cfg, n)

    # ---- the same four stages launched raw through the C ABI (per-stage events)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(calls) + 1)] for _ in range(K)]
    barrier()
    for k in range(K):
        ev[k][0].record(stream)
        for i, (_, c) in enumerate(calls):
            c()
            ev[k][i + 1].record(stream)
    barrier()
    clk = clocks.stop()
    stage_ms = {name: sum(ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(K)) / K
                for i, (name, _) in enumerate(calls)}
    raw_ms = max_over_ranks(sum(stage_ms.values()))
    W, D = raw.counts()
    value = world * n / (ms * 1e-3)

    # ---- end to end through the public host API (runtime C ABI): every step
    #      uploads its pinned keys, builds through the actor chain and writes
    #      counts + words + table back to pinned host memory.  Steps are
    #      pipelined two deep (ndactor_wah_build_index_async): step i+1's
    #      upload and build overlap step i's result copy (opposite PCIe
    #      directions, copy engines).  The fully synchronous call is timed
    #      once beside it.
    hk = host_keys.numpy().view(np.uint32)
    ecap = 3 * max(65536, cfg["k"]) * 4
    hw = [torch.empty(2 * n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in range(2)]
    he = [torch.empty(ecap, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32) for _ in range(2)]
    hc = [torch.zeros(3, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64) for _ in range(2)]
    e2e_steps = max(2, min(K, args.e2e_steps))
    # warm both pipeline slots with two builds in flight: the first use
    # allocates the slots' key buffers and a second set of result buffers
    warm = [rt.build_index_async(hk, hw[i], he[i], hc[i]) for i in range(2)]
    for tk in warm:
        rt.wait(tk)
    barrier()
    t0 = time.perf_counter()
    pend = []
    trace = os.environ.get("NDX_E2E_TRACE")
    for i in range(e2e_steps):
        ta = time.perf_counter()
        if len(pend) == 2:
            rt.wait(pend.pop(0))
        tb = time.perf_counter()
        pend.append(rt.build_index_async(hk, hw[i % 2], he[i % 2], hc[i % 2]))
        if trace:
            print(f"e2e step {i}: wait {1e3 * (tb - ta):.1f} ms issue {1e3 * (time.perf_counter() - tb):.1f} ms",
                  file=sys.stderr, flush=True)
    for tk in pend:
        rt.wait(tk)
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / e2e_steps)
    last = (e2e_steps - 1) % 2
    W_e2e, D_e2e = int(hc[last][0]), int(hc[last][1])
    d2h = 24 + 4 * W_e2e + 12 * D_e2e
    from paper_1709_07781_b200.runtime import index_digest

    e2e_digest = "%016x" % index_digest(n, he[last][: 3 * D_e2e], hw[last][:W_e2e])
    e2e_ok = 3 * D_e2e <= ecap and (e2e_digest == want_digest if want_digest else
                                    (W_e2e == W and D_e2e == D and e2e_digest == chain_digest))
    t0 = time.perf_counter()
    rt.build_index(hk, hw[0], he[0])
    e2e_sync_ms = (time.perf_counter() - t0) * 1e3

    # ---- BASELINE config 2: one-warp kernels raw vs through a compute actor
    iters = 10000 if not args.no_probe else 10
    for _ in range(3 if not args.no_probe else 0):  # threads and clocks settle over the first few rounds
        rt.dispatch_probe_ex(iters)
    probes = [rt.dispatch_probe_ex(iters) for _ in range(5)]
    pr = sorted(probes, key=lambda x: x["actor_ms"] / x["raw_ms"])[2]  # median of 5 by overhead
    p_raw, p_act, chk = pr["raw_ms"], pr["actor_ms"], pr["counter"]

    # ---- roofline of the dominant stage (algorithmic bytes)
    peak, peak_kind = measured_peaks()
    # the sort's passes follow the plan the device made from the key range
    # (wah_sort.cu k_plan): range < 2^11 -> one wide pass (keys in, row ids
    # out: 8N); top 16 bits constant -> the compact passes A (keys in,
    # packed u32 out: 8N) and B (u32 in, row ids out: 8N) -- both write the
    # sorted stream in rows form, the emit reads 4 B per value; otherwise one
    # legacy byte pass per varying byte (12N, then 16N each) and (key, row)
    # pairs (8 B per value) into the emit
    kmin, kmax = raw.key_range()
    stream_b = 4
    if kmax - kmin < 2048:
        sort_alg, sort_what = 8 * n, "wide pass: 4 B keys in, 4 B row ids out"
    elif (kmin >> 16) == (kmax >> 16):
        sort_alg, sort_what = 16 * n, "pass A: 4 B keys in, 4 B packed out; pass B: 4 B in, 4 B row ids out"
    else:
        nb = sum(1 for b in range(4) if (kmin >> (8 * b)) != (kmax >> (8 * b)))
        sort_alg, sort_what = 12 * n + 16 * n * (nb - 1), f"{nb} byte passes (u64 ping-pong)"
        stream_b = 8
    alg = {
        "plan": 4 * n,                                # one read of the keys (+ per-chunk counts, KB)
        "sort": sort_alg,
        "emit": stream_b * n + 4 * W + 8 * D,        # stream in, words + (start, value) out
        "table": 20 * D,
    }
    dom = max(stage_ms, key=stage_ms.get)
    achieved = alg[dom] / (stage_ms[dom] * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(args.config, {}).get(dom)

    ba, bm = b_alg(n, W, D, 2), b_min(n, W, D)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W_, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": cfg["desc"], "values_per_gpu": n, "keys": cfg["k"],
                   "distribution": "zipf s=1" if cfg["kind"] == "zipf" else "uniform",
                   "l2": "inputs larger than L2 (4 B keys x values per GPU > 126 MB)",
                   "parallelism": f"row shards x{world}", "words": W, "distinct": D,
                   "path": "compute-actor chain table*emit*sort*plan over device MemRefs"},
        "result_check": {"what": "FNV-1a-64 of the WAH1 bytes of the actor chain's index (HBM, last timed "
                                 "step) against the reference's digest (tests/golden/digests.json)",
                         "digest": chain_digest, "golden": want_digest,
                         "ok": want_digest is not None and chain_digest == want_digest},
        "build_gbs": {"b_alg_bytes": ba, "gbs_alg": ba / (ms * 1e-3) / 1e9,
                      "frac_alg": ba / (ms * 1e-3) / 1e9 / peak, "frac_alg_spec_8tbs": ba / (ms * 1e-3) / 8e12,
                      "b_min_bytes": bm, "gbs_effective": bm / (ms * 1e-3) / 1e9,
                      "model": "SURVEY 8(d): B_alg = 40N + 4W + 12D (2-pass LSD model), B_min = 4N + 4W + 12D"},
        "stage_ms": stage_ms,
        "dispatch": {"chain_ms": ms, "raw_launch_ms": raw_ms,
                     "chain_overhead_vs_raw": ms / raw_ms - 1.0,
                     "probe_iters": iters, "probe_raw_us_per_kernel": p_raw * 1e3 / iters,
                     "probe_actor_us_per_request": p_act * 1e3 / iters,
                     "probe_raw_enqueue_us": pr["raw_enqueue_ms"] * 1e3 / iters,
                     "probe_actor_host_only_us": pr["actor_host_only_ms"] * 1e3 / iters,
                     "probe_overhead": p_act / p_raw - 1.0, "probe_check_ok": chk == 2 * iters,
                     "probe_runs": 5, "probe_overheads": [x["actor_ms"] / x["raw_ms"] - 1.0 for x in probes]},
        "roofline": {"bound": "hbm", "kernel_stage": dom, "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "algorithmic_bytes": alg[dom],
                     "model": sort_what if dom == "sort" else "SURVEY 8(d) per-stage bytes",
                     "timing": "CUDA events around the stage's launches on the launch stream, mean of the "
                               "timed builds; per-kernel split in profiles/ (ncu)"},
        "e2e": {"value": world * n / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 4 * n,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "steps": e2e_steps,
                "pipelined": "2 deep: step i+1 upload (H2D) and build overlap step i result copy (D2H on the copy engines)",
                "result_check_ok": e2e_ok, "result_digest": e2e_digest, "sync_call_ms": e2e_sync_ms},
        # per build: plan 2 (k_hist, k_plan_scan), sort 5 (three TMA pass kinds,
        # k_pass_bytes, k_vs), emit 4 (k_tile_prep, k_tile_heads, k_emit_rows,
        # k_emit), table 1 -- the launches that return at once included
        "gpu_launches": 12 * K,
        "clocks": clk,
    }
    if world == 1 and args.config == "C4" and not args.no_extra:
        line["other_configs"] = {"C3": extra_config(rt, raw, dev, K, W_)}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    rt.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C4")
    ap.add_argument("--n", type=int, default=0, help="values per GPU (default: the config's)")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--ref-sample", type=int, default=1 << 26)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the C3 line inside the C4 report")
    ap.add_argument("--no-probe", action="store_true",
                    help="skip the 5 x 10^4-launch dispatch probe (for ncu launch lists, which profile every launch)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the multi-GPU step (shard meta, all-gather, merge) even at N=1")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="N > 1: the config's column split over the GPUs (strong) or per GPU (weak)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
