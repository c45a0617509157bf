// wire_core.cuh — exact double -> text digit generation shared by the device
// formatter (wire.cu) and its host build (tools/wire_host_check.py): a
// fixed-capacity big integer, dtoa modes 2 (17 digits) and 0 (shortest
// round trip, CPython's tie rules), and CPython's format_float_short layout.
#pragma once

#include <stdint.h>
#include <string.h>

#include <cmath>

#ifdef __CUDACC__
#define PF_HD __host__ __device__
#else
#define PF_HD
#endif

namespace pf {
namespace wire {

PF_HD inline int clz32(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __clz(x);
#else
  return x ? __builtin_clz(x) : 32;
#endif
}
PF_HD inline int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __clzll(x);
#else
  return x ? __builtin_clzll(x) : 64;
#endif
}
PF_HD inline uint64_t dbits(double v) {
  uint64_t b;
  memcpy(&b, &v, 8);
  return b;
}

constexpr int kLimbs = 42;   // 1344 bits; the largest ratio met needs 38 limbs
constexpr int kSlot = 64;    // bytes per formatted line slot

struct Big {
  uint32_t w[kLimbs];
  int n;  // used limbs (no leading zero limb; 0 for zero)
};

PF_HD inline void set_u64(Big &a, uint64_t x) {
  a.w[0] = static_cast<uint32_t>(x);
  a.w[1] = static_cast<uint32_t>(x >> 32);
  a.n = a.w[1] ? 2 : (a.w[0] ? 1 : 0);
}

PF_HD inline void trim(Big &a) {
  while (a.n > 0 && a.w[a.n - 1] == 0) --a.n;
}

PF_HD void shl(Big &a, int k) {
  if (a.n == 0 || k == 0) return;
  const int lw = k >> 5, b = k & 31;
  if (b == 0) {
    for (int i = a.n - 1; i >= 0; --i) a.w[i + lw] = a.w[i];
    a.w[a.n + lw] = 0;
  } else {
    a.w[a.n + lw] = 0;
    for (int i = a.n - 1; i >= 0; --i) {
      a.w[i + lw + 1] |= a.w[i] >> (32 - b);
      a.w[i + lw] = a.w[i] << b;
    }
  }
  for (int i = 0; i < lw; ++i) a.w[i] = 0;
  a.n += lw + 1;
  trim(a);
}

PF_HD void mul_small(Big &a, uint32_t f) {
  uint64_t c = 0;
  for (int i = 0; i < a.n; ++i) {
    c += static_cast<uint64_t>(a.w[i]) * f;
    a.w[i] = static_cast<uint32_t>(c);
    c >>= 32;
  }
  if (c) a.w[a.n++] = static_cast<uint32_t>(c);
}

PF_HD void mul_pow10(Big &a, int q) {
  constexpr uint32_t p10[10] = {1u,      10u,      100u,      1000u,      10000u,
                                100000u, 1000000u, 10000000u, 100000000u, 1000000000u};
  while (q >= 9) {
    mul_small(a, 1000000000u);
    q -= 9;
  }
  if (q > 0) mul_small(a, p10[q]);
}

PF_HD int cmp(const Big &a, const Big &b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
  return 0;
}

PF_HD void sub(Big &a, const Big &b) {  // a -= b, a >= b
  int64_t br = 0;
  for (int i = 0; i < a.n; ++i) {
    int64_t d = static_cast<int64_t>(a.w[i]) - (i < b.n ? b.w[i] : 0u) - br;
    br = d < 0;
    a.w[i] = static_cast<uint32_t>(d + (br << 32));
  }
  trim(a);
}

PF_HD void add_to(Big &dst, const Big &a, const Big &b) {  // dst = a + b
  const int n = a.n > b.n ? a.n : b.n;
  uint64_t c = 0;
  for (int i = 0; i < n; ++i) {
    c += static_cast<uint64_t>(i < a.n ? a.w[i] : 0u) + (i < b.n ? b.w[i] : 0u);
    dst.w[i] = static_cast<uint32_t>(c);
    c >>= 32;
  }
  dst.n = n;
  if (c) dst.w[dst.n++] = static_cast<uint32_t>(c);
}

PF_HD int bitlen(const Big &a) {
  return a.n == 0 ? 0 : 32 * (a.n - 1) + (32 - clz32(a.w[a.n - 1]));
}

// bits [sh, sh + 128) of a
PF_HD unsigned __int128 bits_from(const Big &a, int sh) {
  const int lw = sh >> 5, b = sh & 31;
  unsigned __int128 lo = 0;
  for (int i = 3; i >= 0; --i) {
    const int j = lw + i;
    lo = (lo << 32) | (j < a.n ? a.w[j] : 0u);
  }
  if (b == 0) return lo;
  const uint32_t top = (lw + 4) < a.n ? a.w[lw + 4] : 0u;
  return (lo >> b) | (static_cast<unsigned __int128>(top) << (128 - b));
}

// q = floor(R / S) (< 2^64), R -= q S.  T is scratch.
PF_HD uint64_t quot(Big &R, const Big &S, Big &T) {
  const int bs = bitlen(S);
  uint64_t q;
  if (bs <= 64) {
    const unsigned __int128 r128 = bits_from(R, 0);
    const uint64_t s64 = static_cast<uint64_t>(bits_from(S, 0));
    q = static_cast<uint64_t>(r128 / s64);
  } else {
    const int sh = bs - 64;
    const unsigned __int128 rt = bits_from(R, sh);
    const uint64_t st = static_cast<uint64_t>(bits_from(S, sh));
    q = st == ~uint64_t{0} ? static_cast<uint64_t>(rt >> 64)
                           : static_cast<uint64_t>(rt / (static_cast<unsigned __int128>(st) + 1));
  }
  if (q) {  // T = S * q
    unsigned __int128 c = 0;
    for (int i = 0; i < S.n; ++i) {
      c += static_cast<unsigned __int128>(S.w[i]) * q;
      T.w[i] = static_cast<uint32_t>(c);
      c >>= 32;
    }
    T.n = S.n;
    while (c) {
      T.w[T.n++] = static_cast<uint32_t>(c);
      c >>= 32;
    }
    trim(T);
    sub(R, T);
  }
  while (cmp(R, S) >= 0) {
    sub(R, S);
    ++q;
  }
  return q;
}

// The same operations on one 128-bit word: the fast path for values whose
// digit-generation ratios provably fit (1e-5 <= v < 1e20, see fast_ok).
struct W128 {
  unsigned __int128 v;
};
PF_HD inline void set_u64(W128 &a, uint64_t x) { a.v = x; }
PF_HD inline void shl(W128 &a, int k) { a.v <<= k; }
PF_HD inline void mul_small(W128 &a, uint32_t f) { a.v *= f; }
PF_HD inline void mul_pow10(W128 &a, int q) {
  while (q >= 9) {
    a.v *= 1000000000u;
    q -= 9;
  }
  while (q-- > 0) a.v *= 10u;
}
PF_HD inline int cmp(const W128 &a, const W128 &b) { return a.v < b.v ? -1 : (a.v > b.v ? 1 : 0); }
PF_HD inline void sub(W128 &a, const W128 &b) { a.v -= b.v; }
PF_HD inline void add_to(W128 &d, const W128 &a, const W128 &b) { d.v = a.v + b.v; }
PF_HD inline bool is_zero(const W128 &a) { return a.v == 0; }
PF_HD inline bool is_zero(const Big &a) { return a.n == 0; }
PF_HD inline uint64_t quot(W128 &R, const W128 &S, W128 &) {
  const uint64_t q = static_cast<uint64_t>(R.v / S.v);
  R.v -= static_cast<unsigned __int128>(q) * S.v;
  return q;
}

struct Parts {
  uint64_t m;
  int e;
  bool frac0;
  int be;
};

PF_HD inline Parts decompose(double v) {  // v > 0 finite
  const uint64_t bits = dbits(v);
  Parts p;
  p.be = static_cast<int>((bits >> 52) & 0x7ff);
  const uint64_t frac = bits & ((uint64_t{1} << 52) - 1);
  p.frac0 = frac == 0;
  if (p.be == 0) {
    p.m = frac;
    p.e = -1074;
  } else {
    p.m = frac | (uint64_t{1} << 52);
    p.e = p.be - 1075;
  }
  return p;
}

PF_HD inline int est_k(const Parts &p) {  // floor(log10 v), may be 1 low
  const int l2 = 63 - clz64(p.m) + p.e;
  return static_cast<int>(std::floor(static_cast<double>(l2) * 0.30102999566398114));
}

// 17 significant digits (dtoa mode 2): writes digits (trailing zeros dropped),
// returns their count; *decpt = decimal exponent of the first digit + 1.
template <class N>
PF_HD int digits_g17_t(double v, char *dig, int *decpt) {
  const Parts p = decompose(v);
  N R0, S0, R, S, T;
  set_u64(R0, p.m);
  set_u64(S0, 1);
  if (p.e >= 0) shl(R0, p.e); else shl(S0, -p.e);
  int E = est_k(p);
  uint64_t D;
  constexpr uint64_t k16 = 10000000000000000ull, k17 = 100000000000000000ull;
  for (;;) {
    R = R0;
    S = S0;
    const int q = 16 - E;
    if (q >= 0) mul_pow10(R, q); else mul_pow10(S, -q);
    D = quot(R, S, T);
    if (D < k16) { --E; continue; }
    if (D >= k17) { ++E; continue; }
    break;
  }
  // round half even on the exact remainder: compare 2R with S
  shl(R, 1);
  const int c = cmp(R, S);
  if (c > 0 || (c == 0 && (D & 1))) {
    ++D;
    if (D == k17) {
      D = k16;
      ++E;
    }
  }
  char buf[17];
  for (int i = 16; i >= 0; --i) {
    buf[i] = static_cast<char>('0' + D % 10);
    D /= 10;
  }
  int nd = 17;
  while (nd > 1 && buf[nd - 1] == '0') --nd;
  for (int i = 0; i < nd; ++i) dig[i] = buf[i];
  *decpt = E + 1;
  return nd;
}

// Shortest round-trip digits (dtoa mode 0, CPython's tie rules).
template <class N>
PF_HD int digits_shortest_t(double v, char *dig, int *decpt) {
  const Parts p = decompose(v);
  const bool even = (p.m & 1) == 0;
  const bool spec = p.frac0 && p.be > 1;  // gap below is half the gap above
  N R, S, Mm, Mp, T;
  set_u64(R, p.m);
  if (p.e >= 0) {
    set_u64(S, spec ? 4 : 2);
    shl(R, p.e + (spec ? 2 : 1));
    set_u64(Mm, 1);
    shl(Mm, p.e);
    set_u64(Mp, 1);
    shl(Mp, p.e + (spec ? 1 : 0));
  } else {
    shl(R, spec ? 2 : 1);
    set_u64(S, 1);
    shl(S, -p.e + (spec ? 2 : 1));
    set_u64(Mm, 1);
    set_u64(Mp, spec ? 2 : 1);
  }
  int k = est_k(p) + 1;
  if (k >= 0) {
    mul_pow10(S, k);
  } else {
    mul_pow10(R, -k);
    mul_pow10(Mm, -k);
    mul_pow10(Mp, -k);
  }
  add_to(T, R, Mp);
  const int ct = cmp(T, S);
  if (even ? ct >= 0 : ct > 0) {
    ++k;
    mul_small(S, 10);
  }
  // Digits accumulate in an integer (at most 17 < 20 decimal digits) and are
  // written once at the end: nvcc's optimiser mishandled per-digit stores into
  // the caller's array in this loop (wrong bytes with -O3, right with -G).
  uint64_t acc = 0;
  int nd = 0;
  for (;;) {
    mul_small(R, 10);
    mul_small(Mm, 10);
    mul_small(Mp, 10);
    int d = static_cast<int>(quot(R, S, T));
    const int j = cmp(R, Mm);
    int j1;
    if (cmp(Mp, S) > 0) {
      j1 = 1;
    } else {
      T = S;
      sub(T, Mp);
      j1 = cmp(R, T);
    }
    int last = -1;  // >= 0: final digit; 10: emit 9 and round the string up
    if (j1 == 0 && even) {
      last = d == 9 ? 10 : (j > 0 ? d + 1 : d);
    } else if (j < 0 || (j == 0 && even)) {
      if (is_zero(R)) {
        last = d;
      } else {
        last = d;
        if (j1 > 0) {
          shl(R, 1);
          const int c = cmp(R, S);
          if (c > 0 || (c == 0 && (d & 1))) last = d == 9 ? 10 : d + 1;
        }
      }
    } else if (j1 > 0) {
      last = d == 9 ? 10 : d + 1;
    }
    if (last < 0) {
      acc = acc * 10 + static_cast<uint64_t>(d);
      ++nd;
      continue;
    }
    if (last == 10) {  // ...d9 -> round up: ...(d+1), carries through trailing 9s
      acc = acc * 10 + 9 + 1;
      ++nd;
      uint64_t p10 = 1;
      for (int i = 0; i < nd; ++i) p10 *= 10;
      if (acc == p10) {
        acc = 1;
        nd = 1;
        ++k;
      }
    } else {
      acc = acc * 10 + static_cast<uint64_t>(last);
      ++nd;
    }
    break;
  }
  char buf[20];
  for (int i = nd - 1; i >= 0; --i) {
    buf[i] = static_cast<char>('0' + acc % 10);
    acc /= 10;
  }
  while (nd > 1 && buf[nd - 1] == '0') --nd;
  for (int i = 0; i < nd; ++i) dig[i] = buf[i];
  *decpt = k;
  return nd;
}

// 1e-5 <= v < 1e20: every ratio of both generators stays below 2^127 (mode 2:
// m 10^22 < 2^127; mode 0: S <= 2^72, M+ <= 2 10^5 10^17), so one 128-bit
// word replaces the big integer; outside that range the 42-limb integer runs.
PF_HD inline bool fast_ok(double v) { return v >= 1e-5 && v < 1e20; }

PF_HD inline int digits_g17(double v, char *dig, int *decpt) {
  return fast_ok(v) ? digits_g17_t<W128>(v, dig, decpt) : digits_g17_t<Big>(v, dig, decpt);
}
PF_HD inline int digits_shortest(double v, char *dig, int *decpt) {
  return fast_ok(v) ? digits_shortest_t<W128>(v, dig, decpt)
                    : digits_shortest_t<Big>(v, dig, decpt);
}

// CPython format_float_short layout; returns the length written to out.
PF_HD int layout(const char *dig, int nd, int decpt, bool repr_mode, char *out) {
  int o = 0;
  const bool use_exp = repr_mode ? (decpt <= -4 || decpt > 16) : (decpt <= -4 || decpt > 17);
  int ex = 0;
  if (use_exp) {
    ex = decpt - 1;
    decpt = 1;
  }
  const int vstart = decpt <= 0 ? decpt - 1 : 0;
  int vend = nd;
  const int need = (!use_exp && repr_mode) ? decpt + 1 : decpt;
  if (vend < need) vend = need;
  if (decpt <= 0) {
    for (int i = 0; i < decpt - vstart; ++i) out[o++] = '0';
    out[o++] = '.';
    for (int i = 0; i < -decpt; ++i) out[o++] = '0';
  }
  if (0 < decpt && decpt <= nd) {
    for (int i = 0; i < decpt; ++i) out[o++] = dig[i];
    out[o++] = '.';
    for (int i = decpt; i < nd; ++i) out[o++] = dig[i];
  } else {
    for (int i = 0; i < nd; ++i) out[o++] = dig[i];
  }
  if (nd < decpt) {
    for (int i = 0; i < decpt - nd; ++i) out[o++] = '0';
    out[o++] = '.';
    for (int i = 0; i < vend - decpt; ++i) out[o++] = '0';
  } else {
    for (int i = 0; i < vend - nd; ++i) out[o++] = '0';
  }
  if (out[o - 1] == '.') --o;
  if (use_exp) {
    out[o++] = 'e';
    out[o++] = ex < 0 ? '-' : '+';
    int a = ex < 0 ? -ex : ex;
    char t[4];
    int nt = 0;
    do {
      t[nt++] = static_cast<char>('0' + a % 10);
      a /= 10;
    } while (a);
    if (nt < 2) t[nt++] = '0';
    while (nt) out[o++] = t[--nt];
  }
  return o;
}

// kind: 0 = .17g (Python f"{v:.17g}"), 1 = repr, 2 = json.dumps float
// (repr; NaN / Infinity / -Infinity).  Returns the length.
PF_HD int format_double(double v, int kind, char *out) {
  int o = 0;
  if (std::isnan(v)) {
    const char *s = kind == 2 ? "NaN" : "nan";
    for (int i = 0; s[i]; ++i) out[o++] = s[i];
    return o;
  }
  const bool neg = std::signbit(v);
  if (std::isinf(v)) {
    const char *s = kind == 2 ? (neg ? "-Infinity" : "Infinity") : (neg ? "-inf" : "inf");
    for (int i = 0; s[i]; ++i) out[o++] = s[i];
    return o;
  }
  if (neg) out[o++] = '-';
  const double a = std::fabs(v);
  if (a == 0.0) {
    out[o++] = '0';
    if (kind != 0) {
      out[o++] = '.';
      out[o++] = '0';
    }
    return o;
  }
  char dig[20];
  int decpt, nd;
  if (kind == 0) nd = digits_g17(a, dig, &decpt);
  else nd = digits_shortest(a, dig, &decpt);
  return o + layout(dig, nd, decpt, kind != 0, out + o);
}

PF_HD int format_u64(uint64_t x, char *out) {
  char t[20];
  int n = 0;
  do {
    t[n++] = static_cast<char>('0' + x % 10);
    x /= 10;
  } while (x);
  for (int i = 0; i < n; ++i) out[i] = t[n - 1 - i];
  return n;
}

}  // namespace wire
}  // namespace pf
