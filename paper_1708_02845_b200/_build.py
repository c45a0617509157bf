"""In-tree build of libpathfield_b200.so (sm_100a) with nvcc.

Each ``csrc/*.cu`` is compiled to an object with its own flags (the tracer
needs ``-fmad=false`` so FP64 rounding follows the reference's numpy
arithmetic exactly; every other file uses default contraction), then linked
into one shared library next to this file.  Static cudart; the library only
ever sees raw device pointers and a cudaStream_t, so it coexists with
torch's own runtime in the same process.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB = PKG / "libpathfield_b200.so"
BUILD = PKG.parent / "build"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INCLUDE}",
          "--expt-relaxed-constexpr"]
HOST = ["-O2", "-g", "-std=c++17", "-fPIC", f"-I{INCLUDE}"]
# Per-file extra flags.
EXTRA = {
    "trace.cu": ["-fmad=false"],
}


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; cannot build libpathfield_b200.so")


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _fingerprint() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh"))
                    + list(CSRC.glob("*.cpp"))
                    + list(INCLUDE.glob("*.h"))):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(repr((ARCH, COMMON, EXTRA, HOST)).encode())
    return h.hexdigest()


def _obj_fingerprint(src: Path, cmd: list) -> str:
    """Source + every shared header + the command line (headers are few)."""
    h = hashlib.sha256(" ".join(cmd).encode())
    for p in [src] + sorted(list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every CUDA source for sm_100a and link the shared library.

    Objects are rebuilt only when their source, a shared header or the
    flags changed, in parallel."""
    from concurrent.futures import ThreadPoolExecutor
    stamp = PKG / ".libpathfield_b200.stamp"
    fp = _fingerprint()
    if not force and LIB.exists() and stamp.exists() and stamp.read_text() == fp:
        return LIB
    nvcc = nvcc_path()
    BUILD.mkdir(exist_ok=True)
    jobs = []
    for src in _sources():
        obj = BUILD / (src.stem + ".o")
        if src.suffix == ".cpp":  # host-only runtime (symbolic plans): plain g++
            cmd = [shutil.which("g++") or "g++", *HOST, "-c", str(src), "-o", str(obj)]
        else:
            cmd = [nvcc, *ARCH, *COMMON, *EXTRA.get(src.name, []), "-c", str(src), "-o",
                   str(obj)]
        ofp = _obj_fingerprint(src, cmd)
        ostamp = obj.with_suffix(".stamp")
        fresh = (not force and obj.exists() and ostamp.exists()
                 and ostamp.read_text() == ofp)
        jobs.append((cmd, obj, ostamp, ofp, fresh))

    def run(job):
        cmd, obj, ostamp, ofp, fresh = job
        if fresh:
            return
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        ostamp.write_text(ofp)

    with ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1))) as ex:
        list(ex.map(run, jobs))
    objs = [str(j[1]) for j in jobs]
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *objs, "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    stamp.write_text(fp)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
