"""The _hostlog extension (csrc/hostlog.c) builds exactly the reference's
event dicts (engine.py:353, :520, :630-633, :383-384, :401-402, :412) from
co_event records -- checked against a plain-Python restatement on CPU."""
import ctypes as C

import numpy as np
import pytest

from paper_2503_13773_b200 import _native as N
from paper_2503_13773_b200 import engine as E
from paper_2503_13773_b200.build import build_hostlog


@pytest.fixture(autouse=True, scope="module")
def _built():
    build_hostlog()  # gcc, about a second; a no-op when up to date


def py_convert(evs, n, mem, rid):
    out = []
    for k in range(n):
        e = evs[k]
        if e.kind == N.EV_ITER:
            m = mem[2 * e.c: 2 * (e.c + e.idx)].tolist()
            out.append({"ev": "iter", "t": e.t, "end": e.a, "tokens": e.b,
                        "members": [[rid[m[j]], m[j + 1]] for j in range(0, len(m), 2)]})
        elif e.kind == N.EV_ARRIVE:
            out.append({"ev": "arrive", "t": e.t, "req": rid[e.idx]})
        elif e.kind == N.EV_ADMIT:
            out.append({"ev": "admit", "t": e.t, "req": rid[e.idx]})
        elif e.kind == N.EV_PREEMPT:
            out.append({"ev": "preempt", "t": e.t, "req": rid[e.idx], "strategy": E._STRATEGY_NAMES[e.b],
                        "kv": e.a, "cause": E._CAUSE_NAMES[e.c]})
        elif e.kind == N.EV_READMIT:
            out.append({"ev": "readmit", "t": e.t, "req": rid[e.idx], "ready_at": e.a})
        else:
            out.append({"ev": "complete", "t": e.t, "req": rid[e.idx]})
    return out


def test_hostlog_matches_python_restatement():
    rng = np.random.default_rng(1)
    n, nm = 400, 3000
    evs = (N.CoEvent * n)()
    mem = np.zeros(2 * nm, dtype=np.int32)
    rid = [int(x) for x in rng.permutation(10_000)[:500]]
    mem[0::2] = rng.integers(0, len(rid), nm)
    mem[1::2] = rng.integers(1, 2048, nm)
    off = 0
    for k in range(n):
        kind = int(rng.integers(0, 6))
        evs[k].kind = kind
        evs[k].t = int(rng.integers(0, 1 << 40))
        evs[k].a = int(rng.integers(0, 1 << 40))
        if kind == N.EV_ITER:
            cnt = int(rng.integers(0, 12))
            evs[k].idx, evs[k].c, evs[k].b = cnt, off, int(rng.integers(0, 4096))
            off += cnt
        else:
            evs[k].idx = int(rng.integers(0, len(rid)))
            evs[k].b = int(rng.integers(0, 2))
            evs[k].c = int(rng.integers(0, len(N.CAUSES)))
    got = E._load_hostlog().convert(C.addressof(evs), n, mem.ctypes.data, rid, E._STRATEGY_NAMES, E._CAUSE_NAMES)
    assert got == py_convert(evs, n, mem, rid)


def test_hostlog_rejects_bad_records():
    evs = (N.CoEvent * 1)()
    evs[0].kind, evs[0].idx = N.EV_ARRIVE, 7
    mem = np.zeros(2, dtype=np.int32)
    with pytest.raises(ValueError):
        E._load_hostlog().convert(C.addressof(evs), 1, mem.ctypes.data, [1, 2], E._STRATEGY_NAMES, E._CAUSE_NAMES)
