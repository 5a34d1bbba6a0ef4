"""the run's random streams on the device.

CPU tests pin the restatement (oracle/rng_oracle.py) against numpy's own
Generator and, when /root/reference is present, against the reference's
generate / assign_slos / predictor consumption.  GPU tests compare the
device streams (csrc/trace_gen.cuh through the C ABI) with numpy bit for bit:
raw PCG64 words, ziggurat doubles, and the integer trace / SLO / noise
columns at BASELINE sizes (config 2: 65,536 requests; config 4: 524,288).
"""
import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import rng_oracle as R  # noqa: E402

REF_SRC = "/root/reference/pkg/src"


# -- CPU: the oracle against numpy ------------------------------------------------

@pytest.mark.parametrize("ent", [[0, 0], [0, 3], [12345, 2], [2 ** 40 + 7, 11], [1, 1], [0, 10]])
def test_seed_and_raw_stream(ent):
    g = np.random.default_rng(ent)
    st = g.bit_generator.state["state"]
    s, inc = R.pcg64_seed(ent)
    assert (s, inc) == (st["state"], st["inc"])
    mine, _ = R.pcg64_raw(s, inc, 256)
    assert (g.bit_generator.random_raw(256) == mine).all()


def test_advance_matches_stepping():
    s, inc = R.pcg64_seed([5, 0])
    a, _ = R.pcg64_raw(s, inc, 1000)
    b, _ = R.pcg64_raw(R.pcg64_advance(s, inc, 700), inc, 300)
    assert (a[700:] == b).all()


@pytest.mark.parametrize("seed", [0, 1, 7])
def test_ziggurat_against_numpy(seed):
    n = 20000
    ref = np.random.default_rng([seed, 0]).standard_exponential(n)
    st = R.Stream([seed, 0])
    assert (ref == np.array([st.std_exponential() for _ in range(n)])).all()
    ref = np.random.default_rng([seed, 1]).standard_normal(n)
    st = R.Stream([seed, 1])
    assert (ref == np.array([st.std_normal() for _ in range(n)])).all()


@pytest.mark.parametrize("dist,scale,acc", [("uniform", 24, 1.0), ("uniform", 24, 0.8), ("normal", 30.0, 0.9),
                                            ("zero", 0, 0.7), ("uniform", 3, 0.5), ("uniform", 2 ** 30, 0.6)])
def test_predictor_consumption(dist, scale, acc):
    """estimation.py:76-99 consumed per arrival, including Lemire rejections
    (scale 2**30: about half the 32-bit draws reject)."""
    g = np.random.default_rng([9, 3])
    e, f = [], []
    for _ in range(3000):
        if dist == "uniform":
            e.append(int(g.integers(-int(scale), int(scale) + 1)) if int(scale) > 0 else 0)
        elif dist == "normal":
            e.append(math.floor(float(g.normal(0.0, scale)) + 0.5))
        else:
            e.append(0)
        f.append(1 if acc < 1.0 and g.random() < 1.0 - acc else 0)
    me, mf = R.gen_predictor(3000, dist, scale, acc, 9)
    assert list(me) == e and list(mf) == f


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present")
def test_trace_and_slos_against_reference():
    sys.path.insert(0, REF_SRC)
    from kvcsim import workload as W
    spec = W.PRESETS["sharegpt"].sized(3000, 50.0)
    reqs = W.generate(spec, 4)
    W.assign_slos(reqs, 2_000_000, 200_000, W.SloPolicy(), 4)
    mi, si = W._lognormal_params(spec.input_mean, spec.length_cv)
    mo, so = W._lognormal_params(spec.output_mean, spec.length_cv)
    a, p, o = R.gen_trace(3000, spec.arrival_rate, mi, si, spec.input_min, spec.input_max, mo, so,
                          spec.output_min, spec.output_max, 4)
    assert list(a) == [r.arrival_us for r in reqs]
    assert list(p) == [r.prompt_len for r in reqs]
    assert list(o) == [r.true_output_len for r in reqs]
    t, b = R.gen_slos(p, 2_000_000, 200_000, 0.5, 2.5, 2048, 4)
    assert list(t) == [r.slo_ttft_us for r in reqs] and list(b) == [r.slo_tbt_us for r in reqs]


def test_table_header_matches_numpy_layers():
    """The committed tables are numpy's: the layer recursion agrees to 1e-12."""
    t = R.tables()
    r = R.ZIG_NOR_R
    assert abs(t["fi"][255] - math.exp(-0.5 * r * r)) < 1e-15
    assert abs(t["wi"][255] * 2.0 ** 52 - r) < 1e-12
    assert t["ki"][1] == 0 and t["ke"][1] == 0
    assert abs(t["fe"][255] - math.exp(-R.ZIG_EXP_R)) < 1e-15


# -- GPU: the device streams ------------------------------------------------------

def _pkg():
    import paper_2503_13773_b200 as P
    from paper_2503_13773_b200 import devrng
    return P, devrng


@pytest.mark.gpu
@pytest.mark.parametrize("ent", [[0, 0], [12345, 3], [2 ** 40 + 7, 11]])
def test_device_seed(ent):
    import ctypes as C
    from paper_2503_13773_b200 import _native as N
    lib = N.load()
    out = (C.c_uint64 * 4)()
    arr = (C.c_uint64 * len(ent))(*ent)
    N.check(lib.co_pcg64_seed(arr, len(ent), out), "seed")
    st = np.random.default_rng(ent).bit_generator.state["state"]
    assert (out[0] << 64 | out[1]) == st["state"] and (out[2] << 64 | out[3]) == st["inc"]


@pytest.mark.gpu
@pytest.mark.parametrize("seed,stream,count", [(0, 0, 1), (0, 3, 1000), (7, 1, 1_000_003), (2 ** 33 + 1, 10, 77777)])
def test_device_raw(seed, stream, count):
    _, devrng = _pkg()
    d = devrng.raw_device(seed, stream, count).cpu().numpy().view(np.uint64)
    ref = np.random.default_rng([seed, stream]).bit_generator.random_raw(count)
    assert (d == ref).all()


def _ulp_diff(a, b):
    ai = a.view(np.int64)
    bi = b.view(np.int64)
    return np.abs(ai - bi)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["exponential", "normal"])
@pytest.mark.parametrize("seed", [0, 5])
def test_device_ziggurat(kind, seed):
    """2M samples: positions resolved exactly (orbit), values bit-identical
    except possibly an ulp on the log1p / exp tail paths."""
    _, devrng = _pkg()
    n = 2_000_000
    d = devrng.standard_device(kind, seed, 1, n).cpu().numpy()
    g = np.random.default_rng([seed, 1])
    ref = g.standard_exponential(n) if kind == "exponential" else g.standard_normal(n)
    ul = _ulp_diff(d, ref)
    assert ul.max() <= 1, (kind, int(ul.max()))
    assert (ul > 0).sum() <= n // 10000, int((ul > 0).sum())


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed,preset,rate", [(1, 0, "sharegpt", 4.0), (1000, 0, "sharegpt", 4.0),
                                               (65536, 0, "sharegpt", 1e6), (524288, 0, "sharegpt", 1e6),
                                               (50000, 3, "alpaca", 32.0), (20000, 9, "bookcorpus", 1.2)])
def test_device_trace(n, seed, preset, rate):
    """workload.generate columns, bit-exact (configs 1, 2 and 4 sizes)."""
    P, devrng = _pkg()
    spec = P.PRESETS[preset].sized(n, rate)
    d = {k: v.cpu().numpy() for k, v in devrng.trace_arrays_device(spec, seed).items()}
    h = P.trace_arrays(spec, seed)
    for k in ("arrival_us", "prompt_len", "true_output_len"):
        assert (d[k].astype(np.int64) == h[k]).all(), k


@pytest.mark.gpu
def test_device_slos():
    import torch
    P, devrng = _pkg()
    spec = P.PRESETS["sharegpt"].sized(65536, 1e6)
    cols = devrng.trace_arrays_device(spec, 2)
    pol = P.SloPolicy()
    t, b = devrng.assign_slos_device(cols["prompt_len"], 2_000_000, 200_000, pol, 2)
    from paper_2503_13773_b200.workload import slo_arrays
    ht, hb = slo_arrays(cols["prompt_len"].cpu().numpy(), 2_000_000, 200_000, pol, 2)
    assert (t.cpu().numpy() == ht).all() and (b.cpu().numpy() == hb).all()
    # long prompts: chunk factor > 1
    pr = torch.tensor([1, 2048, 2049, 4096, 4097, 8192, 100000], dtype=torch.int32, device="cuda")
    t, b = devrng.assign_slos_device(pr, 1_000_003, 77_777, P.SloPolicy(0.3, 3.1, 2048), 11)
    ht, hb = slo_arrays(pr.cpu().numpy(), 1_000_003, 77_777, P.SloPolicy(0.3, 3.1, 2048), 11)
    assert (t.cpu().numpy() == ht).all() and (b.cpu().numpy() == hb).all()


@pytest.mark.gpu
@pytest.mark.parametrize("dist,scale,acc,n", [("zero", 0, 1.0, 1000), ("zero", 0, 0.8, 20000),
                                              ("uniform", 24, 1.0, 20001), ("uniform", 24, 0.7, 20000),
                                              ("normal", 30.0, 1.0, 20000), ("normal", 12.5, 0.9, 20001),
                                              ("uniform", 2 ** 30, 0.6, 5000), ("uniform", 2 ** 30, 1.0, 5001)])
def test_device_predictor(dist, scale, acc, n):
    """estimation.py:76-99 draws; scale 2**30 forces Lemire rejections
    (the sequential re-run path)."""
    P, devrng = _pkg()
    from paper_2503_13773_b200.config import PredictorConfig
    pc = PredictorConfig(error_dist=dist, error_scale=scale, direction_accuracy=acc)
    e, f = devrng.predictor_draws_device(pc, 17, n)
    he, hf = R.gen_predictor(n, dist, scale, acc, 17)
    assert (e.cpu().numpy() == he).all() and (f.cpu().numpy() == hf).all()
