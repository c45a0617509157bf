"""Prototype (Python integers) of the device float formatters in csrc/wire.cu,
structured exactly like the CUDA port, validated against Python's own
formatting: f"{v:.17g}" (fileio.py field/path CSV) and repr(v) (json.dumps in
fileio.field_to_json and the service's JSON responses).

python scripts/proto_wire.py [n_random]
"""
import math
import struct
import sys

import numpy as np


def decompose(v):
    """v > 0 finite -> (m, e, mantissa_bits_zero, biased_exp) with v = m * 2**e."""
    bits = struct.unpack("<Q", struct.pack("<d", v))[0]
    be = (bits >> 52) & 0x7FF
    frac = bits & ((1 << 52) - 1)
    if be == 0:
        return frac, -1074, frac == 0, be
    return frac | (1 << 52), be - 1075, frac == 0, be


def est_k(v):
    """floor(log10(v)) estimate (may be off by one; fixed by the callers)."""
    m, e, _, _ = decompose(v)
    return math.floor((m.bit_length() - 1 + e) * 0.30102999566398114)


def quot(R, S):
    """floor(R / S) for a quotient < 2**64 via a top-bits estimate + fixup
    (what the CUDA bignum does), returns (q, R - q*S)."""
    bs = S.bit_length()
    if bs <= 64:
        q = R // S
    else:
        sh = bs - 64
        q = (R >> sh) // ((S >> sh) + 1)
    r = R - q * S
    while r >= S:
        r -= S
        q += 1
    return q, r


def digits_g17(v):
    """(digits, decpt): 17 significant digits correctly rounded (half even on
    the exact value), trailing zeros stripped — dtoa mode 2, ndigits 17."""
    m, e, _, _ = decompose(v)
    R, S = (m << e, 1) if e >= 0 else (m, 1 << -e)
    E = est_k(v)
    while True:
        q = 16 - E
        Rq, Sq = (R * 10 ** q, S) if q >= 0 else (R, S * 10 ** -q)
        D, rem = quot(Rq, Sq)
        if D < 10 ** 16:
            E -= 1
            continue
        if D >= 10 ** 17:
            E += 1
            continue
        break
    c = 2 * rem - Sq
    if c > 0 or (c == 0 and D & 1):
        D += 1
        if D == 10 ** 17:
            D //= 10
            E += 1
    s = str(D).rstrip("0")
    return s, E + 1


def digits_shortest(v):
    """(digits, decpt): dtoa mode 0 (shortest round-trip, closest, ties per
    _Py_dg_dtoa's rules)."""
    m, e, frac0, be = decompose(v)
    even = (m & 1) == 0
    # R / S = v, M- / S = half the gap below, M+ / S = half the gap above (x2 scaled)
    if e >= 0:
        if frac0 and be > 1:
            R, S, Mm, Mp = m << (e + 2), 4, 1 << e, 1 << (e + 1)
        else:
            R, S, Mm, Mp = m << (e + 1), 2, 1 << e, 1 << e
    else:
        if frac0 and be > 1:
            R, S, Mm, Mp = m << 2, 1 << (-e + 2), 1, 2
        else:
            R, S, Mm, Mp = m << 1, 1 << (-e + 1), 1, 1
    k = est_k(v) + 1                      # want 10^(k-1) <= v < 10^k
    if k >= 0:
        S *= 10 ** k
    else:
        f = 10 ** -k
        R, Mm, Mp = R * f, Mm * f, Mp * f
    # fixup: need R < S (i.e. v < 10^k) accounting for the high boundary
    if (R + Mp > S) if not even else (R + Mp >= S):
        k += 1
        S *= 10
    elif (R + Mp) * 10 < S if not even else (R + Mp) * 10 <= S:
        pass
    out = []
    while True:
        R *= 10
        Mm *= 10
        Mp *= 10
        d, R = quot(R, S)
        j = (R > Mm) - (R < Mm)           # cmp(R, M-)
        j1 = 1 if Mp > S else ((R > S - Mp) - (R < S - Mp))  # cmp(R, S - M+)
        if j1 == 0 and even:
            if d == 9:
                return bump(out, 9, k)
            if j > 0:
                d += 1
            out.append(d)
            return fin(out, k)
        if j < 0 or (j == 0 and even):
            if R == 0:
                out.append(d)
                return fin(out, k)
            if j1 > 0:
                c = 2 * R - S
                if c > 0 or (c == 0 and d & 1):
                    if d == 9:
                        return bump(out, 9, k)
                    d += 1
            out.append(d)
            return fin(out, k)
        if j1 > 0:
            if d == 9:
                return bump(out, 9, k)
            out.append(d + 1)
            return fin(out, k)
        out.append(d)


def bump(out, d, k):
    """Append 9 and round the digit string up (carry)."""
    out.append(d)
    i = len(out) - 1
    while i >= 0 and out[i] == 9:
        i -= 1
    if i < 0:
        return "1", k + 1
    out = out[:i] + [out[i] + 1]
    return fin(out, k)


def fin(out, k):
    s = "".join(map(str, out)).rstrip("0") or "0"
    return s, k


def layout(digits, decpt, mode):
    """format_float_short of CPython: mode 'g' (.17g) or 'r' (repr)."""
    nd = len(digits)
    use_exp = (decpt <= -4 or decpt > 17) if mode == "g" else (decpt <= -4 or decpt > 16)
    add_dot0 = mode == "r"
    exp = 0
    if use_exp:
        exp = decpt - 1
        decpt = 1
    vstart = decpt - 1 if decpt <= 0 else 0
    vend = nd
    if not use_exp and add_dot0:
        vend = max(vend, decpt + 1)
    else:
        vend = max(vend, decpt)
    p = []
    if decpt <= 0:
        p.append("0" * (decpt - vstart) + "." + "0" * (-decpt))
    if 0 < decpt <= nd:
        p.append(digits[:decpt] + "." + digits[decpt:])
    else:
        p.append(digits)
    if nd < decpt:
        p.append("0" * (decpt - nd) + "." + "0" * (vend - decpt))
    else:
        p.append("0" * (vend - nd))
    s = "".join(p)
    if s.endswith("."):
        s = s[:-1]
    if use_exp:
        s += "e" + ("-" if exp < 0 else "+") + ("%02d" % abs(exp))
    return s


def fmt(v, mode):
    if v != v:
        return "nan"
    if v in (float("inf"), float("-inf")):
        return "inf" if v > 0 else "-inf"
    neg = math.copysign(1.0, v) < 0
    a = abs(v)
    if a == 0.0:
        s = "0" if mode == "g" else "0.0"
    else:
        d, p = digits_g17(a) if mode == "g" else digits_shortest(a)
        s = layout(d, p, mode)
    return "-" + s if neg else s


def check(vals):
    bad = 0
    for v in vals:
        v = float(v)
        for mode, ref in (("g", format(v, ".17g")), ("r", repr(v))):
            got = fmt(v, mode)
            if got != ref:
                bad += 1
                if bad < 20:
                    print("MISMATCH", mode, repr(v), got, ref)
    return bad


def test_values(n, seed=0):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2 ** 63, n, dtype=np.int64).view(np.float64)
    vals = [x for x in bits if np.isfinite(x)]
    vals += list(rng.random(n // 4) * 10.0 ** rng.integers(-20, 20, n // 4))
    vals += [0.0, -0.0, 1.0, 0.1, 0.5, 1e16, 1e17, 2e16 + 8, 1e-4, 1e-5, 9.999999999999999e22,
             5e-324, 2.2250738585072014e-308, 2.225073858507201e-308, 1.7976931348623157e308,
             2.0 ** 60, 2.0 ** -1074, 123456789012345678.0, 0.3, 2.0 / 3, 1e23, 8.41e21,
             5e-310, 1e22, 1e21, 9007199254740993.0, 4.35e-7, 1234.5, 0.000123456789]
    vals += [2.0 ** e for e in range(-1074, 1024)]
    vals += [np.nextafter(2.0 ** e, 0) for e in range(-1020, 1024, 7)]
    vals += [10.0 ** e for e in range(-323, 309)]
    vals += [-x for x in vals[:2000]]
    return vals


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
    vals = test_values(n)
    print("values", len(vals), "mismatches", check(vals))
