"""Benchmark of the CacheOPT per-iteration hot path on B200.

Workload (BASELINE.json config 2): ShareGPT-shaped trace of 65,536 requests
arriving within ~65 ms (rate 1e6/s), Llama-2-13B KV layout (16-token blocks),
KV pool capacity 166,400 tokens, SLO baselines 2 s / 200 ms, CacheOPT policy.
One "step" is one engine iteration (engine.py:606-641) over the whole live set.
The run is pre-rolled to step 40 (all requests live, steady state; SURVEY.md
section 6), then W untimed warm-up steps, then exactly K timed steps.

  python bench.py [--gpus N] [--steps K] [--warmup W]          # device arm
  python bench.py --impl reference [...]                         # CPU reference arm

Multi-GPU (torchrun): one independent instance per rank, each with its own
65,536-request shard of one 65,536*N trace (weak scaling, no data-path
collective); time = max over ranks, value = sum of decisions / that time.
"""
from __future__ import annotations

import argparse
import gc
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

METRIC = "sched decisions/s @64K live reqs"
UNIT = "decisions/s"
N_PER_GPU = 65_536
CAPACITY = 166_400
WINDOW_START = 40
L2_FLUSH_BYTES = 256 << 20
STAGE_KERNEL = {"plan": "k_serial", "apply": "k_serial", "plan+apply": "k_serial", "classify": "k_classify",
                "begin+admit": "k_begin", "decode": "k_decode_tc05", "data": "k_data"}


E2E_REPS = 5
_RESULT_FD = None  # the real stdout while native libraries' banners are routed to stderr


def emit(line: dict) -> None:
    """The ONE JSON line on stdout (NCCL and driver banners go to stderr)."""
    data = (json.dumps(line) + "\n").encode()
    if _RESULT_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_RESULT_FD, data)


def route_native_stdout_to_stderr() -> None:
    """fd 1 -> fd 2 for everything native code prints (NCCL prints its version
    banner on stdout at communicator init); the result goes to the saved fd."""
    global _RESULT_FD
    if _RESULT_FD is None:
        sys.stdout.flush()
        _RESULT_FD = os.dup(1)
        os.dup2(2, 1)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def make_trace(rank: int, world: int, device=None):
    """Shard `rank` of a ShareGPT trace of 65,536*world requests (ids are
    arrival-ordered, so a contiguous id slice is a contiguous time slice).
    With a device, the whole trace and its SLOs are drawn on that GPU
    (devrng, bit-identical to numpy's) and only the shard is materialised."""
    import paper_2503_13773_b200 as P
    spec = P.PRESETS["sharegpt"].sized(N_PER_GPU * world, 1e6 * world)
    lo, hi = rank * N_PER_GPU, (rank + 1) * N_PER_GPU
    if device is not None:
        from paper_2503_13773_b200 import devrng
        cols = devrng.trace_arrays_device(spec, 0, device)
        ttft, tbt = devrng.assign_slos_device(cols["prompt_len"], 2_000_000, 200_000, P.SloPolicy(), 0)
        a, p, o = (cols[k][lo:hi].cpu().tolist() for k in ("arrival_us", "prompt_len", "true_output_len"))
        t, b = ttft[lo:hi].cpu().tolist(), tbt[lo:hi].cpu().tolist()
        shard = [P.Request(id=lo + i, arrival_us=a[i], prompt_len=p[i], true_output_len=o[i], slo_ttft_us=t[i],
                           slo_tbt_us=b[i]) for i in range(len(a))]
    else:
        reqs = P.generate(spec, 0)
        P.assign_slos(reqs, 2_000_000, 200_000, P.SloPolicy(), 0)
        shard = reqs[lo:hi]
    cfg = P.EngineConfig(capacity_tokens=CAPACITY, reserved_blocks=8,
                         sched=P.SchedulerConfig(small_block_b=16), seed=0)
    return shard, cfg


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML (the library behind
    nvidia-smi) every ~0.5 ms while the timed region runs, so even a few-ms
    region gets samples; falls back to nvidia-smi polling without NVML."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.how = "nvml"
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.rows.append((float(sm), float(mx), int(rs)))
                self._stop.wait(0.0005)
            pynvml.nvmlShutdown()
            return
        except Exception:
            self.how = "nvidia-smi"
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.active"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                a, b, r = [x.strip() for x in out.split(",")]
                self.rows.append((float(a), float(b), int(r, 16)))
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        mx = max(r[1] for r in self.rows)
        reasons = sorted({n for r in self.rows for n, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows), "how": f"{self.how}, sampled only while the K timed steps run"}


def stage_bytes(n: int, live: int, stage: str, running: int = 0) -> int:
    """Algorithmic HBM bytes of one launch of a stage."""
    if stage == "plan":
        # the running set's and the N'_w head's 64-byte views, the sorted
        # segment indices it walks, and the plan lists it writes
        return running * (64 + 4) + 64 * (64 + 4) + running * 8 * 4
    if stage == "apply":
        return running * (64 + 8 * 4)
    if stage == "plan+apply":  # k_serial: both in one single-CTA launch
        return stage_bytes(n, live, "plan", running) + stage_bytes(n, live, "apply", running)
    if stage == "classify":
        # every live slot: state (1 B) + fixed waiting key (8 B) read; the
        # 64-byte views written for the running set and the N'_w head only
        return live * 9 + (running + 64) * 64
    return 0


def ncu_traffic(kernel: str):
    """DRAM bytes (read + write) of one launch of `kernel` from the committed
    ncu --set full summary (profiles/r02/ncu_full_summary.csv, else r01; cold
    cache), or None when the kernel was not captured."""
    path = os.path.join(ROOT, "profiles", "r02", "ncu_full_summary.csv")
    if not os.path.exists(path):
        path = os.path.join(ROOT, "profiles", "r01", "ncu_full_summary.csv")
    try:
        with open(path) as fh:
            for line in fh:
                f = line.strip().split(",")
                if len(f) > 3 and f[0].split("<")[0].strip().lstrip("void ").strip() == kernel:
                    return int(float(f[2])) + int(float(f[3]))
    except OSError:
        pass
    return None


def host_cpu():
    """The host's CPU model and core counts (reported beside every CPU number)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"model": model, "total_cores": os.cpu_count(), "usable_cores": usable}


def run_cpu_baseline(reqs, cfg, k: int, warmup: int, budget_s: float = 10.0, max_reps: int = 200):
    """The oracle port timed on this host over EXACTLY the device arm's window:
    pre-rolled (untimed) to step WINDOW_START - warmup, `warmup` untimed steps,
    then steps WINDOW_START .. WINDOW_START+k-1 timed one by one.  The window is
    replayed from a snapshot until ~budget_s of CPU work has been timed, so the
    sample is bounded and repeatable; only the timed steps' time counts.
    Returns (decisions/s, ms/step, reps, timed seconds)."""
    import copy
    from oracle.cacheopt_oracle import CacheOptOracle
    orc = CacheOptOracle(reqs, cfg)
    for _ in range(WINDOW_START):
        orc.step()
    orc.events.clear()  # drained before the window, as the device arm drains
    snap = copy.deepcopy(orc)
    dec = 0
    t_sum = 0.0
    steps = 0
    reps = 0
    while reps < max_reps and (reps == 0 or t_sum < budget_s):
        o = copy.deepcopy(snap)
        gc.collect()  # as the device arm's e2e: no collection of earlier garbage inside the window
        for _ in range(k):
            live0, pend0 = o.n_live, o.next_pending
            t0 = time.perf_counter()
            ok = o.step()
            t_sum += time.perf_counter() - t0
            if not ok:
                break
            dec += live0 + (o.next_pending - pend0)  # live set after admission
            steps += 1
        reps += 1
    return dec / t_sum, 1e3 * t_sum / max(steps, 1), reps, t_sum


def _cpu_shard_worker(args):
    rank, world, k, warmup, budget_s, core = args
    try:
        saved = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {core})
    except (AttributeError, OSError):
        saved = None
    try:
        reqs, cfg = make_trace(rank, world)
        return run_cpu_baseline(reqs, cfg, k, warmup, budget_s)
    finally:
        if saved is not None:
            os.sched_setaffinity(0, saved)


def cpu_aggregate(world: int, k: int, warmup: int, budget_s: float = 10.0):
    """one pinned CPU process per instance, each on its
    own shard, running concurrently; aggregate = sum of per-process
    decisions/s (each process's rate over its own timed steps)."""
    import multiprocessing as mp
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count()))
    jobs = [(r, world, k, warmup, budget_s, cores[r % len(cores)]) for r in range(world)]
    if world == 1:
        res = [_cpu_shard_worker(jobs[0])]
    else:
        with mp.get_context("fork").Pool(world) as pool:
            res = pool.map(_cpu_shard_worker, jobs)
    val = sum(r[0] for r in res)
    ms = max(r[1] for r in res)
    reps = min(r[2] for r in res)
    return val, ms, reps, len({j[5] for j in jobs}), res


def reference_arm(args, rank, world):
    if rank != 0:
        return
    cpu = host_cpu()
    val, ms, reps, cores, _ = cpu_aggregate(world, args.steps, args.warmup)
    sample = (f"oracle port, {world} process(es) x 1 thread pinned to {cores} core(s), each on its own config-2 "
              f"shard: steps {WINDOW_START}..{WINDOW_START + args.steps - 1} (the device arm's timed window) "
              f"replayed {reps}x from a snapshot")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": workload_config(world),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "host_cpu": cpu},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def workload_config(world):
    return {"workload": "BASELINE config 2: ShareGPT 65,536 reqs/instance @1e6 req/s, KV pool 166,400 tok "
                        "(Llama-2-13B layout, 16-tok blocks), SLO baselines 2 s/200 ms, CacheOPT",
            "requests_per_instance": N_PER_GPU, "instances": world, "window_start_step": WINDOW_START,
            "l2": "flushed (256 MiB memset) before every timed step", "parallelism": f"{world} independent instances"}


def long_output_trace(n=200, rate=1.0, seed=0):
    """BASELINE config 5 trace: prompt 512 [16, 4096], output 4096 [1024, 8192], cv 0.5."""
    import paper_2503_13773_b200 as P
    spec = P.TraceSpec(arrival_rate=rate, num_requests=n, input_mean=512, input_min=16, input_max=4096,
                       output_mean=4096, output_min=1024, output_max=8192, length_cv=0.5)
    reqs = P.generate(spec, seed)
    P.assign_slos(reqs, 2_000_000, 100_000, P.SloPolicy(), seed)
    return reqs


def swap_leg(dev):
    """N2: swap-out/in of the mean swapped sequence of the long-output trace
    (4,731 tokens, Llama-2-70B layout: 1.55 GB) through the engine's own data
    kernel, against the pinned cudaMemcpyAsync peak of this host link."""
    import ctypes as C
    import paper_2503_13773_b200 as P
    from paper_2503_13773_b200 import _native as N
    lib = N.load()
    d2h, h2d = C.c_double(), C.c_double()
    N.check(lib.co_host_link_gbs(1 << 30, C.byref(d2h), C.byref(h2d)), "host link")
    kv = P.KVLayout.llama2_70b(host_swap_pages=320, decode=False)
    cfg = P.EngineConfig(capacity_tokens=65_536, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=16))
    eng = P.Engine(long_output_trace(n=8), cfg, device=dev, kv=kv)
    ntok = 4731
    out_ms, in_ms = eng.swap_bench(ntok, iters=5)
    eng.close()
    nbytes = ntok * kv.bytes_per_token
    out_gbs, in_gbs = nbytes / out_ms / 1e6, nbytes / in_ms / 1e6
    return {"metric": "KV swap GB/s", "tokens": ntok, "bytes": nbytes,
            "swap_out_gbs": out_gbs, "swap_in_gbs": in_gbs,
            "host_link_peak_gbs": {"d2h": d2h.value, "h2d": h2d.value, "how": "pinned cudaMemcpyAsync 1 GiB, best of 5"},
            "roofline": {"bound": "host-link", "frac_out": out_gbs / d2h.value, "frac_in": in_gbs / h2d.value},
            "kernel": "k_data (SM copy through mapped pinned host pages)"}


def decode_leg(dev, warm_steps=6000, k=10, split=512):
    """N3: paged decode over the engine's block tables, Llama-2-70B layout,
    long-output trace; decode enabled only for the k timed steps."""
    import ctypes as C
    import paper_2503_13773_b200 as P
    from paper_2503_13773_b200 import _native as N
    kv = P.KVLayout.llama2_70b(host_swap_pages=4096, decode=True, decode_split=split)
    cfg = P.EngineConfig(capacity_tokens=65_536, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=16),
                         record_events=False)
    eng = P.Engine(long_output_trace(), cfg, device=dev, kv=kv)
    eng.set_decode(False)
    eng.run_steps(warm_steps)
    eng.set_decode(True)
    st0 = eng.data_stats()
    step_ms = (C.c_double * k)()
    stage_ms = (C.c_double * N.NSTAGES)()
    eng._dirty()
    N.check(eng._lib.co_time_steps(eng._h, k, L2_FLUSH_BYTES, step_ms, stage_ms), "co_time_steps")
    st1 = eng.data_stats()
    # correctness of what was timed: every member of the last timed step, then
    # of two more steps, against the fp64 reference (tests/kv_reference.py)
    from tests.kv_reference import decode_reference_torch
    worst, n_checked, per_step = 0.0, 0, []
    for extra in range(3):
        if extra:
            eng.step()
        rids, ctxs, out, step_id = eng.last_decode()
        per_step.append(len(rids))
        for j in range(len(rids)):
            ref = decode_reference_torch(rids[j], int(ctxs[j]), step_id, kv.layers, kv.q_heads, kv.kv_heads,
                                         device=f"cuda:{dev}")
            worst = max(worst, float(np.abs(out[j] - ref).max() / max(np.abs(ref).max(), 1e-6)))
            n_checked += 1
    bad, checked = eng.kv_verify()
    eng.close()
    members = st1["decode_member_steps"] - st0["decode_member_steps"]
    ctx = st1["decode_ctx_tokens"] - st0["decode_ctx_tokens"]
    dec_ms = stage_ms[7]
    nbytes = ctx * kv.bytes_per_token
    peak, kind = load_peaks()
    gbs = nbytes / (dec_ms * 1e-3) / 1e9 if dec_ms else 0.0
    return {"metric": "paged-decode tokens/s", "value": members / (dec_ms * 1e-3) if dec_ms else 0.0,
            "unit": "tokens/s", "steps": k, "members_per_step": members / k, "mean_ctx": ctx / max(members, 1),
            "decode_ms_per_step": dec_ms / k,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak, "peak_kind": peak_kind_label(kind),
                         "algorithmic_bytes_per_launch": nbytes // k},
            "kv_integrity": {"mismatches": bad, "checked": checked},
            "parity": {"max_rel_err": worst, "tolerance": 1e-2, "members_checked": n_checked,
                       "members_per_checked_step": per_step,
                       "how": "every decode member of the last timed step and of 2 further steps vs the fp64 "
                              "torch reference of tests/kv_reference.py (all 80 layers x 64 q heads)"},
            "config": "BASELINE config 5: Llama-2-70B KV layout (80 layers, 64 q / 8 kv heads), long-output trace "
                      "200 reqs @1 req/s, pool 65,536 tokens (21.5 GB), decode on for the timed steps after "
                      f"{warm_steps} warm steps"}


def costmodel_leg(dev):
    """swap and recompute latencies measured on this B200
    (Llama-2-70B layout; swap = the engine's k_data round trip, recompute = a
    bf16 prefill proxy), fitted with the reference's estimators; then BASELINE
    config 3 (2x-rate heavy preemption) runs with those hardware-true costs and
    the Llama-2-70B KV data plane, so its preemptions move real bytes."""
    import dataclasses
    import paper_2503_13773_b200 as P
    from paper_2503_13773_b200 import costprofile as cp
    from tests.cases import config3
    t0 = time.perf_counter()
    res = cp.hardware_truth(kv_layout=P.KVLayout.llama2_70b(decode=False), dims=cp.ModelDims.llama2_70b(),
                            device=dev)
    t_prof = time.perf_counter() - t0
    reqs, cfg = config3()
    cfg = dataclasses.replace(cfg, truth=res["truth"])
    kv = P.KVLayout.llama2_70b(host_swap_pages=2048, decode=False)
    eng = P.Engine(reqs, cfg, device=dev, kv=kv)
    wall, bad, checked = 0.0, 0, 0
    while True:
        # the KV of every live holder is verified every 1,000 steps while the
        # trace runs (only the run_steps calls are timed)
        t0 = time.perf_counter()
        done = eng.run_steps(1000)
        wall += time.perf_counter() - t0
        b, c = eng.kv_verify()
        bad, checked = bad + b, checked + c
        if done < 1000:
            break
    evs = eng.events
    st = eng.data_stats()
    io = eng.swap_io_stats()
    iters = sum(1 for e in evs if e["ev"] == "iter")
    pre = [e for e in evs if e["ev"] == "preempt"]
    n_swap = sum(1 for e in pre if e["strategy"] == "swap")
    eng.close()
    return {"metric": "B200-fitted swap/recompute cost models",
            "model": "Llama-2-70B KV (327,680 B/token)",
            "swap_ms": res["swap"], "recompute_ms": res["recompute"], "sweet_spot_tokens": res["sweet_spot"],
            "crossover": res["crossover_note"] or "crossover inside the range",
            "profile_s": t_prof,
            "config3_with_fitted_costs": {
                "iterations": iters, "preemptions": len(pre), "swaps": n_swap, "recomputes": len(pre) - n_swap,
                "swap_out_gb": st["swap_out_bytes"] / 1e9, "swap_in_gb": st["swap_in_bytes"] / 1e9,
                "wall_s": wall, "iterations_per_s": iters / wall,
                "kv_integrity": {"mismatches": bad, "checked": checked},
                "in_run_swap_io": in_run_io(io, dev)}}


def in_run_io(io, dev):
    """k_swapio's device-timed totals over a run vs the measured host link:
    link-time fraction = (bytes out / D2H peak + bytes in / H2D peak) / time."""
    import ctypes as C
    from paper_2503_13773_b200 import _native as N
    d2h, h2d = C.c_double(), C.c_double()
    N.check(N.load().co_host_link_gbs(1 << 30, C.byref(d2h), C.byref(h2d)), "host link")
    t = io["device_s"]
    ideal = io["bytes_out"] / (d2h.value * 1e9) + io["bytes_in"] / (h2d.value * 1e9)
    return {"bytes_out": io["bytes_out"], "bytes_in": io["bytes_in"], "device_s": t,
            "gbs": io["gbs"], "launches": io["launches"], "ctas": io["ctas"],
            "link_peak_gbs": {"d2h": d2h.value, "h2d": h2d.value},
            "frac_of_link": ideal / t if t else None,
            "how": "k_swapio (split swap I/O on a side stream, overlapping the decode), %globaltimer from its "
                   "first CTA in to its last CTA out, summed over the run's launches that moved data"}


def tracegen_leg(dev, n=524_288, reps=3):
    """the config-4 trace (512K requests) with its SLOs and
    predictor noise drawn on the GPU (csrc/trace_gen.cuh) vs numpy on the host
    (the reference's own generators), and checked bit-exact against it."""
    import paper_2503_13773_b200 as P
    from paper_2503_13773_b200 import devrng, hostprep
    from paper_2503_13773_b200.config import EngineConfig, PredictorConfig
    spec = P.PRESETS["sharegpt"].sized(n, 1e6)
    pol = P.SloPolicy()
    pc = PredictorConfig(error_dist="uniform", error_scale=24, direction_accuracy=0.9)

    def device_once():
        cols = devrng.trace_arrays_device(spec, 0, dev)
        t, b = devrng.assign_slos_device(cols["prompt_len"], 2_000_000, 200_000, pol, 0)
        e, f = devrng.predictor_draws_device(pc, 0, n, dev)
        return cols, t, b, e, f

    device_once()  # module load / first-touch
    ms = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = device_once()
        ms.append((time.perf_counter() - t0) * 1e3)
    cols, t, b, e, f = out
    t0 = time.perf_counter()
    h = P.trace_arrays(spec, 0)
    ht, hb = P.workload.slo_arrays(h["prompt_len"], 2_000_000, 200_000, pol, 0)
    t_host_trace = time.perf_counter() - t0
    cfg = EngineConfig(predictor=pc)
    t0 = time.perf_counter()
    he, hf = hostprep.noise_draws(cfg, n)
    t_host_pred = time.perf_counter() - t0
    exact = bool((cols["arrival_us"].cpu().numpy() == h["arrival_us"]).all()
                 and (cols["prompt_len"].cpu().numpy() == h["prompt_len"]).all()
                 and (cols["true_output_len"].cpu().numpy() == h["true_output_len"]).all()
                 and (t.cpu().numpy() == ht).all() and (b.cpu().numpy() == hb).all()
                 and (e.cpu().numpy() == he).all() and (f.cpu().numpy() == hf).all())
    dev_ms = min(ms)
    host_ms = (t_host_trace + t_host_pred) * 1e3
    return {"metric": "trace generation requests/s", "requests": n,
            "workload": "BASELINE config 4 trace: sharegpt x 524,288 @1e6 req/s + assign_slos(2 s, 200 ms) + "
                        "uniform(24) / 90%-direction predictor draws, seed 0",
            "device_ms": dev_ms, "device_ms_all": ms, "value": n / (dev_ms * 1e-3),
            "host_numpy_ms": host_ms, "host_numpy_value": n / (host_ms * 1e-3),
            "host_breakdown_ms": {"trace+slos": t_host_trace * 1e3, "predictor": t_host_pred * 1e3},
            "bit_exact_vs_numpy": exact,
            "how": "wall clock around the synchronous C-ABI calls (outputs allocated by torch), best of "
                   f"{reps} after one warm call; host = numpy Generator + the reference's per-request loops"}


def peak_kind_label(kind):
    return f"{kind} (MEASURED_PEAKS.json hbm_gbs)" if kind == "measured" else kind


def device_arm(args, rank, world, dist):
    import ctypes as C
    import torch
    from paper_2503_13773_b200 import Engine
    from paper_2503_13773_b200 import _native as N

    torch.cuda.set_device(rank % max(1, torch.cuda.device_count()))
    dev = torch.cuda.current_device()
    reqs, cfg = make_trace(rank, world, dev)
    cfg.record_events = True
    eng = Engine(reqs, cfg, device=dev)
    if dist:
        # N4: per-iteration global-reserve all-reduce inside the step graph
        from paper_2503_13773_b200.multi import attach_global_reserve
        attach_global_reserve(eng, rank, world)
    pre = max(0, WINDOW_START - args.warmup)
    eng.run_steps(pre)
    eng.run_steps(args.warmup)
    eng.events  # drain the arrival burst outside the timed region
    s0 = eng._scalars()
    d0, it0 = s0.decisions, s0.iterations
    step_ms = (C.c_double * args.steps)()
    stage_ms = (C.c_double * N.NSTAGES)()
    with ClockSampler(dev) as clocks:
        t_wait = time.perf_counter()
        while not clocks.rows and time.perf_counter() - t_wait < 2.0:
            time.sleep(0.001)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        eng._dirty()
        # events only at the step boundaries: stage event nodes would split the
        # step graph (and cost ~25 us/step); the breakdown is a separate pass
        N.check(eng._lib.co_time_steps(eng._h, args.steps, L2_FLUSH_BYTES, step_ms, None), "co_time_steps")
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    eng._dirty()
    s1 = eng._scalars()
    dev_ms = float(sum(step_ms))
    decisions = s1.decisions - d0
    coll = None
    if dist:
        gfree, grsv, calls = eng.global_reserve()
        coll = {"op": "ncclAllReduce(sum, int64[2]={free_tokens, reserved_blocks}) per iteration, side stream",
                "calls": calls, "global_free_tokens": gfree, "global_reserved_blocks": grsv}
    live = s1.n_live
    running = int((eng._field("STATE") == 2).sum())
    kps = C.c_int32()
    N.check(eng._lib.co_kernels_per_step(eng._h, C.byref(kps)), "co_kernels_per_step")
    kernels_per_step = kps.value
    eng.close()

    def fresh():
        """A new instance pre-rolled to the same window (steps 40.. timed)."""
        e = Engine(reqs, cfg, device=dev)
        if dist:
            from paper_2503_13773_b200.multi import attach_global_reserve
            attach_global_reserve(e, rank, world)
        e.run_steps(pre + args.warmup - 1)
        e.events  # drain the arrival burst outside the timed region
        return e

    def e2e_run(drain_events: bool):
        """The public per-step API on the SAME window as the device timing
        (steps 40..40+K-1): Engine.step_result() returns the iteration's
        members every step; with drain_events the step's event log is also
        materialised as host dicts every step (what the CPU arm builds)."""
        e = fresh()
        e.prepare_step()  # instantiate the single-step graph outside the timed loop
        e.step_result()   # (one untimed step builds the host-side result buffers)
        e.events
        gc.collect()  # the harness's own garbage (traces, earlier instances) collected before, not inside, the window
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        dd0 = e._scalars().decisions
        nev0 = len(e._events)
        d2h = 0
        t0 = time.perf_counter()
        for _ in range(args.steps):
            _, members, _ = e.step_result(drain=drain_events)
            d2h += members.size * 4 + 16
            if drain_events:
                e.events
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        e._dirty()
        dec = e._scalars().decisions - dd0
        nev = len(e.events) - nev0
        e.close()
        return el, dec, d2h, nev

    # the window is only K steps of ~70 us of host wall clock each: E2E_REPS
    # fresh repetitions per variant, the median one reported
    def median_run(drain):
        runs = sorted((e2e_run(drain) for _ in range(E2E_REPS)), key=lambda r: r[0] / max(r[1], 1))
        return runs[len(runs) // 2]

    e2e_s, e2e_dec, d2h, e2e_nev = median_run(True)
    e2e_s_nd, e2e_dec_nd, _, _ = median_run(False)
    if dist:
        t = torch.tensor([dev_ms, e2e_s * 1e3, e2e_s_nd * 1e3], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        s = torch.tensor([decisions, e2e_dec, e2e_dec_nd], dtype=torch.float64, device="cuda")
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        dev_ms, e2e_ms, e2e_ms_nd = float(t[0]), float(t[1]), float(t[2])
        decisions, e2e_dec, e2e_dec_nd = float(s[0]), float(s[1]), float(s[2])
    else:
        e2e_ms, e2e_ms_nd = e2e_s * 1e3, e2e_s_nd * 1e3
    if rank != 0:
        return
    # stage breakdown: a second instance replays the same window with an
    # event node at every stage boundary
    eng2 = Engine(reqs, cfg, device=dev)
    eng2.run_steps(pre + args.warmup)
    eng2.events
    step2 = (C.c_double * args.steps)()
    eng2._dirty()
    N.check(eng2._lib.co_time_steps(eng2._h, args.steps, L2_FLUSH_BYTES, step2, stage_ms), "co_time_steps")
    eng2._dirty()
    staged_step_ms = float(sum(step2)) / args.steps
    eng2.close()
    stages = {N.STAGES[q]: stage_ms[q] / args.steps for q in range(N.NSTAGES)}
    stages.pop("bucket", None)  # (round 1's deadline bucketing; k_classify collects the N'_w head now)
    # plan and apply are ONE launch (k_serial) in the headline step; the replay
    # splits them only to attribute time
    kstage = dict(stages)
    kstage["plan+apply"] = kstage.pop("plan") + kstage.pop("apply")
    dom = max(kstage, key=kstage.get)
    peak, peak_kind = load_peaks()
    n = len(reqs)
    algo = stage_bytes(n, live, dom, running)
    ach = algo / (kstage[dom] * 1e-3) / 1e9 if algo else 0.0
    cpu_val, cpu_ms, cpu_reps, cpu_cores, _ = cpu_aggregate(1, args.steps, args.warmup)
    extra = {}
    if not args.skip_legs and world == 1:
        try:
            extra["swap"] = swap_leg(dev)
        except Exception as exc:  # reported, never silently replaced
            extra["swap"] = {"error": repr(exc)}
        try:
            extra["decode"] = decode_leg(dev)
        except Exception as exc:
            extra["decode"] = {"error": repr(exc)}
        try:
            extra["costmodel"] = costmodel_leg(dev)
        except Exception as exc:
            extra["costmodel"] = {"error": repr(exc)}
        try:
            extra["tracegen"] = tracegen_leg(dev)
        except Exception as exc:
            extra["tracegen"] = {"error": repr(exc)}
    line = {
        "metric": METRIC, "value": decisions / (dev_ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (seeded ShareGPT-shaped trace)", "config": workload_config(world),
        "stage_ms_per_step": stages,
        "stage_breakdown_how": "same window replayed on a second instance with a CUDA event node at every stage "
                               f"boundary (its step: {staged_step_ms * 1e3:.1f} us; the event nodes split the "
                               "step graph, so the headline ms_per_step is timed with boundary events only)",
        "live_requests": live,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak if peak else None, "traffic": ncu_traffic(STAGE_KERNEL.get(dom, dom)),
                     "traffic_source": "profiles/r02/ncu_full_summary.csv (one ncu --set full launch, cold cache)",
                     "peak_kind": peak_kind, "algorithmic_bytes_per_launch": algo,
                     "note": "the step's dominant kernel is the single-CTA plan+apply (k_serial: the ordered greedy "
                             "loops of scheduler.py and engine.py): latency-bound on instruction fetch (ncu: "
                             "stall_no_instruction ~46%, ~54 KB of SASS executed per step), so its HBM fraction "
                             "is ~0 by construction; the decode leg carries the bandwidth roofline"},
        "cpu_baseline": {"value": cpu_val, "unit": UNIT, "cores": cpu_cores, "kind": "port",
                         "ms_per_step": cpu_ms, "host_cpu": host_cpu(),
                         "sample": f"oracle port, 1 thread pinned to 1 core, config-2 steps {WINDOW_START}.."
                                   f"{WINDOW_START + args.steps - 1} (the same window as the device timing) "
                                   f"replayed {cpu_reps}x from a snapshot"},
        "e2e": {"value": e2e_dec / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 256 + d2h // max(args.steps, 1),
                "events_per_step": e2e_nev / max(args.steps, 1),
                "how": "Engine.step_result() per step through the public API (control block + the iteration's "
                       "members read back every step) AND the step's event log materialised as host dicts "
                       "(Engine.events) every step, on the same window as the device timing (steps "
                       f"{WINDOW_START}..{WINDOW_START + args.steps - 1}) of a fresh instance, median of "
                       f"{E2E_REPS} repetitions; trace uploaded once at construction (no per-step inputs: no "
                       "arrivals in the window)",
                "without_event_drain": e2e_dec_nd / (e2e_ms_nd * 1e-3)},
        "gpu_launches": args.steps * kernels_per_step,
        "gpu_launches_note": f"{kernels_per_step} own kernels per step (k_classify: begin + admission + "
                             "the planner's views; k_serial: plan + apply + invariant check + log mirror); no library kernels",
        "clocks": clocks.summary(),
        "collective": coll,
        **extra,
    }
    emit(line)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--skip-legs", action="store_true", help="only the scheduler leg")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    route_native_stdout_to_stderr()
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if world > 1 or "LOCAL_RANK" in os.environ:
        # under torchrun (any N, so the 1-GPU box exercises the same path):
        # NCCL process group + the per-iteration global-reserve all-reduce
        import torch
        import torch.distributed as td
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        td.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
        dist = td
    device_arm(args, rank, world, dist)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
