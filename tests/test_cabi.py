"""The drop-in boundary: libcacheopt.so loads, exports exactly what
include/cacheopt.h declares, and the ctypes mirrors have the header's layout.
No compute calls (this runs without a GPU)."""
import os
import re
import subprocess
import sys
import tempfile

import pytest

from paper_2503_13773_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cacheopt.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(co_\w+)\s*\(", src, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    names = declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(N.EXPORTS) == names


def test_version_string():
    assert b"sm_100a" in N.load().co_version()


def test_struct_layouts_match_header():
    import ctypes as C
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "cacheopt.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(co_config), sizeof(co_trace), sizeof(co_luts),
         sizeof(co_scalars), sizeof(co_event), offsetof(co_config, s_star), offsetof(co_scalars, n_live),
         sizeof(co_step_args), offsetof(co_step_args, counts), offsetof(co_step_args, drain));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    want = [C.sizeof(N.CoConfig), C.sizeof(N.CoTrace), C.sizeof(N.CoLuts), C.sizeof(N.CoScalars),
            C.sizeof(N.CoEvent), N.CoConfig.s_star.offset, N.CoScalars.n_live.offset,
            C.sizeof(N.CoStepArgs), N.CoStepArgs.counts.offset, N.CoStepArgs.drain.offset]
    assert got == want


def test_engine_fails_loudly_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("this check is for CPU-only machines")
    import paper_2503_13773_b200 as P
    reqs = [P.Request(0, 0, 10, 3, 10**9, 10**9)]
    with pytest.raises(Exception):
        P.Engine(reqs, P.EngineConfig())


def test_unsupported_modes_are_rejected_not_emulated():
    import paper_2503_13773_b200 as P
    reqs = [P.Request(0, 0, 10, 3, 10**9, 10**9)]
    with pytest.raises(ValueError):
        P.Engine(reqs, P.EngineConfig(sched=P.SchedulerConfig(policy="fifo")))  # not a reference policy


def test_loading_the_library_before_torch_keeps_torch_importable():
    # libcacheopt must not pin an NCCL older than torch's (N4 resolves NCCL lazily)
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_2503_13773_b200 import _native as N; N.load()\n"
            "import torch; print('ok')\n") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_no_link_time_nccl_dependency():
    out = subprocess.run(["ldd", str(N.LIB_PATH)], capture_output=True, text=True)
    assert "nccl" not in out.stdout
