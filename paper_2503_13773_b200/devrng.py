"""The run's random streams generated on the GPU.

Device twins of the reference's numpy draws, bit-identical for the same
seeds (``csrc/trace_gen.cuh``):

* ``trace_arrays_device(spec, seed)``  -- workload.py:85-109 ``generate``;
* ``assign_slos_device(prompt, ...)``  -- workload.py:181-194 ``assign_slos``;
* ``predictor_draws_device(cfg, n)``   -- estimation.py:76-99 noise draws
  from ``default_rng([cfg.seed, 3])`` in admission order (engine.py:267/348);
* ``standard_device`` / ``raw_device`` -- the underlying samplers.

Outputs are torch tensors on the device (torch is only the allocator here);
``generate_device`` returns the reference's ``List[Request]``.  There is no
host fallback: without the CUDA library these raise.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Tuple

from . import _native as N
from .core import Request
from .workload import HOUR_US, SloPolicy, TraceSpec, _lognormal


def _torch():
    import torch
    return torch


def _dev(device: int):
    torch = _torch()
    d = torch.cuda.current_device() if device is None or device < 0 else device
    return d, torch.device("cuda", d)


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def raw_device(seed: int, stream: int, count: int, device: int = -1):
    """First ``count`` raw outputs of default_rng([seed, stream]) (as int64 bits)."""
    torch = _torch()
    lib = N.load()
    d, dev = _dev(device)
    out = torch.empty(count, dtype=torch.int64, device=dev)
    N.check(lib.co_gen_raw(seed, stream, count, d, _ptr(out)), "co_gen_raw")
    return out


def standard_device(kind: str, seed: int, stream: int, n: int, device: int = -1):
    """default_rng([seed, stream]).standard_exponential(n) / .standard_normal(n)."""
    torch = _torch()
    lib = N.load()
    d, dev = _dev(device)
    code = {"exponential": 0, "normal": 1}[kind]
    out = torch.empty(n, dtype=torch.float64, device=dev)
    N.check(lib.co_gen_std(code, seed, stream, n, d, _ptr(out)), "co_gen_std")
    return out


def trace_arrays_device(spec: TraceSpec, seed: int, device: int = -1) -> Dict[str, object]:
    """workload.generate's columns on the device: arrival_us (int64),
    prompt_len, true_output_len (int32)."""
    torch = _torch()
    lib = N.load()
    d, dev = _dev(device)
    n = spec.num_requests
    sp = N.CoTraceSpec()
    sp.n = n
    sp.gap_scale = 1.0 / spec.arrival_rate
    sp.mu_in, sp.sigma_in = _lognormal(spec.input_mean, spec.length_cv)
    sp.mu_out, sp.sigma_out = _lognormal(spec.output_mean, spec.length_cv)
    sp.input_min, sp.input_max = spec.input_min, spec.input_max
    sp.output_min, sp.output_max = spec.output_min, spec.output_max
    arr = torch.empty(n, dtype=torch.int64, device=dev)
    pr = torch.empty(n, dtype=torch.int32, device=dev)
    ou = torch.empty(n, dtype=torch.int32, device=dev)
    N.check(lib.co_gen_trace(C.byref(sp), seed, d, _ptr(arr), _ptr(pr), _ptr(ou)), "co_gen_trace")
    return {"arrival_us": arr, "prompt_len": pr, "true_output_len": ou}


def assign_slos_device(prompt_len, baseline_ttft_us: int, baseline_tbt_us: int, policy: SloPolicy,
                       seed: int) -> Tuple[object, object]:
    """SLO columns (int64) for the device prompt lengths (int32 tensor)."""
    torch = _torch()
    lib = N.load()
    if prompt_len.dtype != torch.int32 or not prompt_len.is_cuda:
        raise ValueError("prompt_len must be an int32 CUDA tensor")
    prompt_len = prompt_len.contiguous()
    n = prompt_len.numel()
    sp = N.CoSloSpec()
    sp.base_ttft_us, sp.base_tbt_us = int(baseline_ttft_us), int(baseline_tbt_us)
    sp.scale_lo, sp.scale_hi, sp.chunk_budget = policy.scale_lo, policy.scale_hi, policy.chunk_budget
    ttft = torch.empty(n, dtype=torch.int64, device=prompt_len.device)
    tbt = torch.empty(n, dtype=torch.int64, device=prompt_len.device)
    N.check(lib.co_gen_slos(n, _ptr(prompt_len), C.byref(sp), seed, prompt_len.device.index, _ptr(ttft),
                            _ptr(tbt)), "co_gen_slos")
    return ttft, tbt


def predictor_draws_device(predictor, seed: int, n: int, device: int = -1):
    """(err int32, flip uint8) for n arrivals from default_rng([seed, 3])."""
    torch = _torch()
    lib = N.load()
    d, dev = _dev(device)
    sp = N.CoPredictorSpec()
    sp.error_dist = N.ERR_DIST[predictor.error_dist]
    sp.error_scale = float(predictor.error_scale)
    sp.direction_accuracy = float(predictor.direction_accuracy)
    err = torch.empty(n, dtype=torch.int32, device=dev)
    flip = torch.empty(n, dtype=torch.uint8, device=dev)
    N.check(lib.co_gen_predictor(n, C.byref(sp), seed, d, _ptr(err), _ptr(flip)), "co_gen_predictor")
    return err, flip


def generate_device(spec: TraceSpec, seed: int, device: int = -1) -> List[Request]:
    """workload.py:85-109 generate() with the draws made on the GPU."""
    cols = {k: v.cpu().numpy() for k, v in trace_arrays_device(spec, seed, device).items()}
    return [Request(id=i, arrival_us=int(a), prompt_len=int(p), true_output_len=int(o),
                    slo_ttft_us=HOUR_US, slo_tbt_us=HOUR_US)
            for i, (a, p, o) in enumerate(zip(cols["arrival_us"], cols["prompt_len"], cols["true_output_len"]))]
