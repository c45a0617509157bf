"""Host build of csrc/wire_core.cuh (the exact digit generators the device
formatter runs) checked against CPython: f"{v:.17g}" and repr(v).

python tools/wire_host_check.py [n_random]
"""
import ctypes
import subprocess
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
import proto_wire as P  # noqa: E402

SRC = r'''
#include "wire_core.cuh"
extern "C" int pf_host_format(double v, int kind, char *out) {
  return pf::wire::format_double(v, kind, out);
}
'''


def build():
    d = Path(tempfile.mkdtemp())
    (d / "h.cpp").write_text(SRC)
    so = d / "libwirehost.so"
    subprocess.run(["g++", "-O2", "-shared", "-fPIC", "-std=c++17",
                    f"-I{ROOT / 'paper_1708_02845_b200' / 'csrc'}", str(d / "h.cpp"), "-o", str(so)],
                   check=True)
    lib = ctypes.CDLL(str(so))
    lib.pf_host_format.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_char_p]
    return lib


def main(n):
    lib = build()
    buf = ctypes.create_string_buffer(64)
    vals = P.test_values(n)
    bad = 0
    for v in vals:
        v = float(v)
        for kind, ref in ((0, format(v, ".17g")), (1, repr(v))):
            k = lib.pf_host_format(v, kind, buf)
            got = buf.raw[:k].decode("ascii", "replace")
            if got != ref:
                bad += 1
                if bad < 15:
                    print("MISMATCH kind", kind, repr(v), got, ref)
    print("values", len(vals), "mismatches", bad)
    return bad


if __name__ == "__main__":
    sys.exit(1 if main(int(sys.argv[1]) if len(sys.argv) > 1 else 20000) else 0)
