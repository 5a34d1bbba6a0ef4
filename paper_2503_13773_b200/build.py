"""Builds libcacheopt.so in-tree for sm_100a with nvcc (no JIT cache)."""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
SRC = PKG / "csrc" / "cacheopt.cu"
OUT = PKG / "_lib" / "libcacheopt.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted((PKG / "csrc").glob("*.cu*")) + [PKG.parent / "include" / "cacheopt.h"]



HOSTLOG_SRC = PKG / "csrc" / "hostlog.c"


def hostlog_path() -> Path:
    import sysconfig
    return PKG / ("_hostlog" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_hostlog(force: bool = False) -> Path:
    """The CPython extension that turns drained device events into the
    reference's dicts (csrc/hostlog.c), built in-tree with the system C
    compiler against this interpreter's headers."""
    import sysconfig
    out = hostlog_path()
    if out.exists() and not force and out.stat().st_mtime >= HOSTLOG_SRC.stat().st_mtime:
        return out
    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc:
        raise RuntimeError("no C compiler for csrc/hostlog.c")
    tmp = out.with_suffix(".tmp")
    subprocess.run([cc, "-O2", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"], "-o", str(tmp),
                    str(HOSTLOG_SRC)], check=True)
    tmp.replace(out)
    return out


def build(force: bool = False, verbose: bool = False) -> Path:
    build_hostlog(force)
    if OUT.exists() and not force:
        newest = max(p.stat().st_mtime for p in sources())
        if OUT.stat().st_mtime >= newest:
            return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = OUT.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-I", str(PKG.parent / "include"), "-o", str(tmp), str(SRC), "-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    # development builds only (e.g. -DCO_MBAR_WATCHDOG); never set for the product
    cmd[1:1] = os.environ.get("CACHEOPT_NVCC_EXTRA", "").split()
    subprocess.run(cmd, check=True)
    tmp.replace(OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
