// wire.cu — the field / path wire formats of the reference rendered on the
// GPU, byte for byte (pathfield/fileio.py:37-79; service/app.py:95-114).
//
//   field CSV   "vertex,value\n" + f"{i},{v:.17g}\n" per vertex   (fileio.py:37-40)
//   path CSV    "x,y\n" + f"{x:.17g},{y:.17g}\n" per point          (fileio.py:73-76)
//   field JSON  json.dumps(payload, indent=2): each value float.__repr__
//               (NaN / Infinity / -Infinity), ",\n    " between  (fileio.py:43-53)
//   compact     the service's JSON list "[v,v,...]" (starlette JSONResponse:
//               separators (",", ":"), repr, NaN/inf rejected)
//
// Both digit generators are exact (a per-thread fixed-capacity big integer,
// 42 x 32-bit limbs: every double's ratio R/S fits):
//   .17g   dtoa mode 2: 17 significant digits of the exact binary value,
//          round half even, trailing zeros dropped;
//   repr   dtoa mode 0: the shortest digit string that reads back to v, ties
//          broken exactly as CPython's _Py_dg_dtoa;
// and the layout is CPython's format_float_short ('g': exponent when decpt
// <= -4 or > 17; 'r': <= -4 or > 16, ".0" on integers, exponent "e+XX").
// tools/proto_wire.py is the same algorithm in Python integers, checked
// against CPython on ~400K values; tests/test_wire_gpu.py checks this port.
//
// Lines are formatted into fixed 64-byte slots with their lengths, then
// packed at their exclusive-scan offsets (pf_pack_lines).
#include <stdint.h>

#include "pf_common.cuh"
#include "wire_core.cuh"

namespace pf {
namespace wire {

// Line kinds of pf_format_lines.
enum { kFieldCsv = 0, kPathCsv = 1, kJsonIndent = 2, kJsonCompact = 3, kRepr = 4, kG17 = 5 };

__global__ void __launch_bounds__(128) format_lines_kernel(const double *__restrict__ vals,
                                                            int64_t n, int kind, int64_t index0,
                                                            char *__restrict__ slots,
                                                            int32_t *__restrict__ lens,
                                                            uint32_t *__restrict__ nonfinite) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    char *s = slots + i * kSlot;
    int o = 0;
    switch (kind) {
      case kFieldCsv:
        o = format_u64(static_cast<uint64_t>(index0 + i), s);
        s[o++] = ',';
        o += format_double(vals[i], 0, s + o);
        s[o++] = '\n';
        break;
      case kPathCsv:
        o = format_double(vals[2 * i], 0, s);
        s[o++] = ',';
        o += format_double(vals[2 * i + 1], 0, s + o);
        s[o++] = '\n';
        break;
      case kJsonIndent:
        o = format_double(vals[i], 2, s);
        if (i + 1 < n) {
          const char sep[] = ",\n    ";
          for (int u = 0; u < 6; ++u) s[o++] = sep[u];
        }
        break;
      case kJsonCompact:
        if (!isfinite(vals[i]) && nonfinite) atomicOr(nonfinite, 1u);
        o = format_double(vals[i], 1, s);
        if (i + 1 < n) s[o++] = ',';
        break;
      case kRepr:
        o = format_double(vals[i], 1, s);
        break;
      default:
        o = format_double(vals[i], 0, s);
        break;
    }
    lens[i] = o;
  }
}

// out[offs[i] .. offs[i] + lens[i]) = slot i; warp per 32 slots, lanes copy
// 2-byte pieces so neighbouring lanes write neighbouring bytes.
__global__ void __launch_bounds__(256) pack_lines_kernel(const char *__restrict__ slots,
                                                         const int32_t *__restrict__ lens,
                                                         const int64_t *__restrict__ offs,
                                                         int64_t n, char *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    const int len = lens[i];
    const char *src = slots + i * kSlot;
    char *dst = out + offs[i];
    for (int u = lane; u < len; u += 32) dst[u] = src[u];
  }
}

}  // namespace wire
}  // namespace pf

using namespace pf;

extern "C" {

int pf_format_lines(const double *vals, int64_t n, int kind, int64_t index0, char *slots,
                    int32_t *lens, uint32_t *nonfinite, pf_stream_t stream) {
  if (n <= 0) return 0;
  if (!vals || !slots || !lens) return fail(PF_E_ARG, "format_lines: null");
  if (kind < 0 || kind > wire::kG17) return fail(PF_E_ARG, "format_lines: kind %d", kind);
  int64_t blocks = (n + 127) / 128;
  if (blocks > static_cast<int64_t>(sm_count()) * 64) blocks = static_cast<int64_t>(sm_count()) * 64;
  wire::format_lines_kernel<<<static_cast<unsigned>(blocks), 128, 0, as_stream(stream)>>>(
      vals, n, kind, index0, slots, lens, nonfinite);
  return check_launch("format_lines");
}

int pf_pack_lines(const char *slots, const int32_t *lens, const int64_t *offs, int64_t n,
                  char *out, pf_stream_t stream) {
  if (n <= 0) return 0;
  if (!slots || !lens || !offs || !out) return fail(PF_E_ARG, "pack_lines: null");
  int64_t blocks = (n + 7) / 8;
  if (blocks > static_cast<int64_t>(sm_count()) * 16) blocks = static_cast<int64_t>(sm_count()) * 16;
  wire::pack_lines_kernel<<<static_cast<unsigned>(blocks), 256, 0, as_stream(stream)>>>(
      slots, lens, offs, n, out);
  return check_launch("pack_lines");
}

}  // extern "C"
