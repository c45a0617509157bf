// trace.cu — batched triangle-descent path tracer (K8).
//
// Reference: pathfield/paths.py:101-307 (triangle_gradient, _Tracer,
// triangle_descent).  One thread advances one (source, field) path through
// the state machine over a device-resident triangle adjacency; thousands of
// paths run per launch.  The kernel reproduces the reference's FP64 rounding
// exactly so that the location sequence (triangle/edge/vertex decisions) is
// bit-identical:
//   * this file is compiled with -fmad=false: no implicit contraction;
//   * the only fused multiply-adds are where numpy's OpenBLAS kernels fuse
//     (re-probed in tests): f @ G and lam @ V as
//     fma(x2,y2, fma(x1,y1, x0*y0)), G @ d as fma(G_i0,d0, G_i1*d1), the 3-dot
//     lam @ f as fma(l2,f2, fma(l1,f1, l0*f0));
//   * np.hypot is glibc 2.39's non-FMA correction kernel, restated below
//     (CUDA's hypot rounds differently);
//   * 3-element sums are ((a+b)+c) (numpy reduce), ties break on the lowest
//     index exactly where the reference's argmax/min/strict-< do.
#include <cmath>

#include <cstdlib>

#include "pf_common.cuh"

namespace pf {

constexpr int kTraceThreads = 128;
constexpr int kTraceSpread = 4;   // lanes per path in trace_kernel (see the launch)

// ---------------------------------------------------------------- hypot --
// glibc sysdeps/ieee754/dbl-64/e_hypot.c (non-FMA kernel); SURVEY A.3.
__device__ __forceinline__ double hypot_kernel(double ax, double ay) {
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    const double delta = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
    t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
  } else {
    const double delta = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

__device__ double np_hypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return INFINITY;
    return x + y;
  }
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  const double kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54, kScale = 0x1p-600;
  if (ax > kLarge) {
    if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
    return __ddiv_rn(hypot_kernel(__dmul_rn(ax, kScale), __dmul_rn(ay, kScale)), kScale);
  }
  if (ay < kTiny) {
    if (ax >= __ddiv_rn(ay, kEps)) return __dadd_rn(ax, ay);
    return __dmul_rn(hypot_kernel(__ddiv_rn(ax, kScale), __ddiv_rn(ay, kScale)), kScale);
  }
  if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
  return hypot_kernel(ax, ay);
}

// ----------------------------------------------------------- geometry --
struct Tri {
  int v[3];
  int nbr[3];       // triangle across the edge opposite each slot (-1: none)
  double G[3][2];   // barycentric gradients (paths.py:105-110)
  double xy[3][2];  // vertex coordinates
  double area;
  double f[3];      // field values at the vertices (set by gradient())
};

__device__ __forceinline__ void tri_G(const pf_mesh_t &m, int64_t ti, const int v[3],
                                      double G[3][2]) {
  const double ax = m.vertices[2 * v[0]], ay = m.vertices[2 * v[0] + 1];
  const double bx = m.vertices[2 * v[1]], by = m.vertices[2 * v[1] + 1];
  const double cx = m.vertices[2 * v[2]], cy = m.vertices[2 * v[2] + 1];
  const double area2 = __dmul_rn(2.0, m.areas[ti]);
  // _perp(v) = [-v[1], v[0]];  rows: perp(pc-pb), perp(pa-pc), perp(pb-pa); / area2
  G[0][0] = __ddiv_rn(-__dsub_rn(cy, by), area2);
  G[0][1] = __ddiv_rn(__dsub_rn(cx, bx), area2);
  G[1][0] = __ddiv_rn(-__dsub_rn(ay, cy), area2);
  G[1][1] = __ddiv_rn(__dsub_rn(ax, cx), area2);
  G[2][0] = __ddiv_rn(-__dsub_rn(by, ay), area2);
  G[2][1] = __ddiv_rn(__dsub_rn(bx, ax), area2);
}

// Triangle record: with the packed per-triangle table (pf_mesh_pack_f64: one
// 128-byte line = vertex coordinates, barycentric gradients, area, vertex ids,
// neighbours) a visit is one round trip; otherwise the separate arrays.  Same
// values either way (the table is built with the same arithmetic).
__device__ __forceinline__ void load_tri(const pf_mesh_t &m, int64_t ti, Tri &t) {
  if (m.pack) {
    const double2 *r = reinterpret_cast<const double2 *>(m.pack + 16 * ti);
    double2 q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) q[u] = __ldg(r + u);
    t.xy[0][0] = q[0].x;
    t.xy[0][1] = q[0].y;
    t.xy[1][0] = q[1].x;
    t.xy[1][1] = q[1].y;
    t.xy[2][0] = q[2].x;
    t.xy[2][1] = q[2].y;
    t.G[0][0] = q[3].x;
    t.G[0][1] = q[3].y;
    t.G[1][0] = q[4].x;
    t.G[1][1] = q[4].y;
    t.G[2][0] = q[5].x;
    t.G[2][1] = q[5].y;
    t.area = q[6].x;
    const long long w0 = __double_as_longlong(q[6].y), w1 = __double_as_longlong(q[7].x),
                    w2 = __double_as_longlong(q[7].y);
    t.v[0] = static_cast<int>(w0 & 0xffffffffLL);
    t.v[1] = static_cast<int>(w0 >> 32);
    t.v[2] = static_cast<int>(w1 & 0xffffffffLL);
    t.nbr[0] = static_cast<int>(w1 >> 32);
    t.nbr[1] = static_cast<int>(w2 & 0xffffffffLL);
    t.nbr[2] = static_cast<int>(w2 >> 32);
    return;
  }
  t.v[0] = m.triangles[3 * ti + 0];
  t.v[1] = m.triangles[3 * ti + 1];
  t.v[2] = m.triangles[3 * ti + 2];
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    t.nbr[s] = m.tri_nbr[3 * ti + s];
    t.xy[s][0] = m.vertices[2 * t.v[s]];
    t.xy[s][1] = m.vertices[2 * t.v[s] + 1];
  }
  t.area = m.areas[ti];
  if (m.G) {
    const double2 *g = reinterpret_cast<const double2 *>(m.G + 6 * ti);
    const double2 g0 = g[0], g1 = g[1], g2 = g[2];
    t.G[0][0] = g0.x;
    t.G[0][1] = g0.y;
    t.G[1][0] = g1.x;
    t.G[1][1] = g1.y;
    t.G[2][0] = g2.x;
    t.G[2][1] = g2.y;
  } else {
    tri_G(m, ti, t.v, t.G);
  }
}

// Speculative prefetch into L1 of the packed records the walk may visit next
// (a triangle's neighbours, a vertex's incident triangles): each visit then
// starts from L1 instead of a DRAM round trip.  Loads only -- the walk's
// arithmetic and order are untouched (bitwise the same paths).
__device__ __forceinline__ void prefetch_rec(const pf_mesh_t &m, int64_t ti) {
  if (m.pack && ti >= 0)
    asm volatile("prefetch.global.L1 [%0];" ::"l"(m.pack + 16 * ti));
}

// a[i] for a 3-element array and a runtime i, as selects: a dynamic index
// would put the array in local memory, an L1 round trip inside the walk's
// serial chain (same values either way)
template <class T>
__device__ __forceinline__ T sel3(int i, const T (&a)[3]) {
  return i == 0 ? a[0] : (i == 1 ? a[1] : a[2]);
}
__device__ __forceinline__ double sel3xy(int i, const double (&xy)[3][2], int c) {
  return i == 0 ? xy[0][c] : (i == 1 ? xy[1][c] : xy[2][c]);
}

// One field's values: vertex v at p[v * s] (s = 1: a field per row of an
// (F, n) block; s = T: a column of the (n, T) output of the batched KL).
struct FieldView {
  const double *p;
  int64_t s;
  __device__ __forceinline__ double operator[](int64_t v) const { return p[v * s]; }
};

// f @ G  (3,)@(3,2): fma(f2,G2j, fma(f1,G1j, f0*G0j))
__device__ __forceinline__ void gradient(Tri &t, const FieldView &vals, double g[2]) {
  const double f0 = vals[t.v[0]], f1 = vals[t.v[1]], f2 = vals[t.v[2]];
  t.f[0] = f0;
  t.f[1] = f1;
  t.f[2] = f2;
#pragma unroll
  for (int j = 0; j < 2; ++j)
    g[j] = __fma_rn(f2, t.G[2][j], __fma_rn(f1, t.G[1][j], __dmul_rn(f0, t.G[0][j])));
}

// G @ d  (3,2)@(2,): fma(G_i0, d0, G_i1*d1); returns scale = max|dl| + 1e-300
__device__ __forceinline__ double dlam_of(const Tri &t, const double d[2], double dl[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) dl[i] = __fma_rn(t.G[i][0], d[0], __dmul_rn(t.G[i][1], d[1]));
  double mx = fabs(dl[0]);
  if (fabs(dl[1]) > mx) mx = fabs(dl[1]);
  if (fabs(dl[2]) > mx) mx = fabs(dl[2]);
  return __dadd_rn(mx, 1e-300);
}

// ------------------------------------------------------------- output --
struct Writer {
  const pf_paths_t *o;
  int64_t path, count;
  double lx, ly;  // pts[-1]
  __device__ void put(int kind, int64_t i, int64_t j, double t, double x, double y) {
    if (count < o->cap) {
      const int64_t at = path * o->cap + count;
      o->kind[at] = static_cast<int8_t>(kind);
      o->i[at] = static_cast<int32_t>(i);
      o->j[at] = static_cast<int32_t>(j);
      o->t[at] = t;
      o->x[at] = x;
      o->y[at] = y;
    }
    ++count;
    lx = x;
    ly = y;
  }
};

enum { ST_REACHED = 0, ST_STUCK = 1, ST_MAX = 2 };
constexpr int64_t kNearestPending = -2;

__global__ void __launch_bounds__(kTraceThreads) trace_kernel(pf_mesh_t m, const double *fields,
                                                              int64_t field_ld, int64_t vertex_ld,
                                                              const int64_t *targets,
                                                              const int64_t *sources,
                                                              const int32_t *field_of,
                                                              int64_t npaths, int64_t cap,
                                                              pf_paths_t out, int spread) {
  // one path per `spread` lanes (fewer paths per warp to diverge)
  const int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gid % spread) return;
  const int64_t p = gid / spread;
  if (p >= npaths) return;
  const int64_t fi = field_of ? field_of[p] : 0;
  const FieldView vals{fields + fi * field_ld, vertex_ld};
  const int64_t target = targets[fi];
  const int64_t source = sources[p];
  const double eps_prog = m.eps_prog;

  Writer w{&out, p, 0, 0.0, 0.0};
  w.put(0, source, -1, 0.0, m.vertices[2 * source], m.vertices[2 * source + 1]);

  bool in_tri = false;
  int64_t v = source, ti = -1;
  double x0 = 0.0, x1 = 0.0, cur = 0.0;
  int status = ST_MAX;
  int64_t stuck = -1;
  double qx = 0.0, qy = 0.0;
  bool carry = false;  // geometry of triangle `ti` already evaluated by _enters
  Tri ct;
  double cnorm = 0.0, cd[2] = {0.0, 0.0}, cdl[3] = {0.0, 0.0, 0.0}, cscale = 0.0;

  for (int64_t it = 0; it < cap; ++it) {
    if (!in_tri) {
      // ---------------- vertex rule (paths.py:162-196)
      if (v == target) {
        status = ST_REACHED;
        break;
      }
      double best_norm = 0.0;
      int64_t best = -1;
      const int64_t e0 = m.vt_ptr[v], e1 = m.vt_ptr[v + 1];
      for (int64_t e = e0; e < e1; ++e) prefetch_rec(m, m.vt_idx[e]);
      for (int64_t e = e0; e < e1; ++e) {
        const int64_t tj = m.vt_idx[e];
        Tri t;
        load_tri(m, tj, t);
        double g[2];
        gradient(t, vals, g);
        const double norm = np_hypot(g[0], g[1]);
        if (norm <= 0.0) continue;
        const double d[2] = {__ddiv_rn(-g[0], norm), __ddiv_rn(-g[1], norm)};
        const int slot = (t.v[0] == v) ? 0 : (t.v[1] == v ? 1 : 2);
        double dl[3];
        const double scale = dlam_of(t, d, dl);
        const int o0 = slot == 0 ? 1 : 0, o1 = slot == 2 ? 1 : 2;
        const double thr = __dmul_rn(1e-12, scale);
        if (sel3(o0, dl) > thr && sel3(o1, dl) > thr) {
          if (best < 0 || norm > best_norm) {
            best_norm = norm;
            best = tj;
          }
        }
      }
      if (best >= 0) {
        in_tri = true;
        ti = best;
        x0 = m.vertices[2 * v];
        x1 = m.vertices[2 * v + 1];
        cur = vals[v];
        continue;
      }
      // steepest incident edge
      const double vx = m.vertices[2 * v], vy = m.vertices[2 * v + 1], fv = vals[v];
      double bs = 0.0;
      int64_t bu = -1;
      for (int64_t e = m.nb_ptr[v]; e < m.nb_ptr[v + 1]; ++e) {
        const int64_t u = m.nb_idx[e];
        const double diff = __dsub_rn(fv, vals[u]);
        const double len =
            np_hypot(__dsub_rn(m.vertices[2 * u], vx), __dsub_rn(m.vertices[2 * u + 1], vy));
        const double slope = __ddiv_rn(diff, len);
        if (bu < 0 || slope > bs) {
          bs = slope;
          bu = u;
        }
      }
      if (bu < 0 || bs <= 0.0) {
        status = ST_STUCK;
        stuck = v;
        break;
      }
      w.put(0, bu, -1, 0.0, m.vertices[2 * bu], m.vertices[2 * bu + 1]);
      v = bu;
      continue;
    }

    // ---------------- triangle rule (paths.py:200-254)
    // The previous step's _enters() already evaluated this triangle's gradient,
    // direction and dlam (the reference recomputes the identical values): reuse.
    Tri t;
    double g[2], norm, d[2], dl[3], scale = 0.0;
    if (carry) {
      t = ct;
      norm = cnorm;
      d[0] = cd[0];
      d[1] = cd[1];
      dl[0] = cdl[0];
      dl[1] = cdl[1];
      dl[2] = cdl[2];
      scale = cscale;
      carry = false;
    } else {
      load_tri(m, ti, t);
      gradient(t, vals, g);
      norm = np_hypot(g[0], g[1]);
      if (norm > 0.0) {
        d[0] = __ddiv_rn(-g[0], norm);
        d[1] = __ddiv_rn(-g[1], norm);
        scale = dlam_of(t, d, dl);
      }
    }
    bool slide_best = norm <= 0.0;
    double lam[3], s_exit = INFINITY;
    int slot_exit = -1;
    if (!slide_best) {
      const double ax = t.xy[0][0], ay = t.xy[0][1];
      const double bx = t.xy[1][0], by = t.xy[1][1];
      const double cx = t.xy[2][0], cy = t.xy[2][1];
      const double area2 = __dmul_rn(2.0, t.area);
      // _cross2(u, w) = u0*w1 - u1*w0 (paths.py:124-134)
      const double la = __ddiv_rn(__dsub_rn(__dmul_rn(__dsub_rn(cx, bx), __dsub_rn(x1, by)),
                                            __dmul_rn(__dsub_rn(cy, by), __dsub_rn(x0, bx))),
                                  area2);
      const double lb = __ddiv_rn(__dsub_rn(__dmul_rn(__dsub_rn(ax, cx), __dsub_rn(x1, cy)),
                                            __dmul_rn(__dsub_rn(ay, cy), __dsub_rn(x0, cx))),
                                  area2);
      lam[0] = la;
      lam[1] = lb;
      lam[2] = __dsub_rn(__dsub_rn(1.0, la), lb);
#pragma unroll
      for (int s = 0; s < 3; ++s) lam[s] = lam[s] < 0.0 ? 0.0 : lam[s];  // np.clip(., 0)
      const double sum = __dadd_rn(__dadd_rn(lam[0], lam[1]), lam[2]);
#pragma unroll
      for (int s = 0; s < 3; ++s) lam[s] = __ddiv_rn(lam[s], sum);
      const double thr = __dmul_rn(-1e-14, scale);
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        if (dl[s] < thr && lam[s] > 0.0) {
          const double cand = __ddiv_rn(lam[s], -dl[s]);
          if (cand < s_exit) {
            s_exit = cand;
            slot_exit = s;
          }
        }
      }
      slide_best = !isfinite(s_exit);
    }
    if (slide_best) {
      // _slide_to_best_vertex (paths.py:276-282): min by (value, index)
      int sb = 0;
#pragma unroll
      for (int s = 1; s < 3; ++s)
        if (t.f[s] < sel3(sb, t.f) || (t.f[s] == sel3(sb, t.f) && t.v[s] < sel3(sb, t.v))) sb = s;
      const int64_t bw = sel3(sb, t.v);
      if (sel3(sb, t.f) >= cur) {
        status = ST_STUCK;
        stuck = bw;
        break;
      }
      w.put(0, bw, -1, 0.0, sel3xy(sb, t.xy, 0), sel3xy(sb, t.xy, 1));
      in_tri = false;
      v = bw;
      continue;
    }
    double le[3];
#pragma unroll
    for (int s = 0; s < 3; ++s) le[s] = __dadd_rn(lam[s], __dmul_rn(s_exit, dl[s]));
#pragma unroll
    for (int s = 0; s < 3; ++s)
      if (s == slot_exit) le[s] = 0.0;
#pragma unroll
    for (int s = 0; s < 3; ++s) le[s] = le[s] < 0.0 ? 0.0 : le[s];
    const double lsum = __dadd_rn(__dadd_rn(le[0], le[1]), le[2]);
#pragma unroll
    for (int s = 0; s < 3; ++s) le[s] = __ddiv_rn(le[s], lsum);
    int hi = 0;
    double lhi = le[0];
    if (le[1] > lhi) {
      hi = 1;
      lhi = le[1];
    }
    if (le[2] > lhi) {
      hi = 2;
      lhi = le[2];
    }
    if (lhi > 1.0 - 1e-12) {
      // exit through a vertex
      const int64_t wv = sel3(hi, t.v);
      const double wx = sel3xy(hi, t.xy, 0), wy = sel3xy(hi, t.xy, 1);
      if (!(np_hypot(__dsub_rn(wx, w.lx), __dsub_rn(wy, w.ly)) >= eps_prog)) {
        status = ST_STUCK;
        stuck = kNearestPending;  // resolved by nearest_resolve_kernel
        qx = x0;
        qy = x1;
        break;
      }
      w.put(0, wv, -1, 0.0, wx, wy);
      in_tri = false;
      v = wv;
      continue;
    }
    int o0 = slot_exit == 0 ? 1 : 0, o1 = slot_exit == 2 ? 1 : 2;
    int64_t ei = sel3(o0, t.v), ej = sel3(o1, t.v);
    if (ei > ej) {
      const int64_t tmp = ei;
      ei = ej;
      ej = tmp;
      const int to = o0;
      o0 = o1;
      o1 = to;
    }
    const double tpar = sel3(o1, le);
    // lam_exit @ V[tri]  (3,)@(3,2)
    const double xe0 = __fma_rn(le[2], t.xy[2][0],
                                __fma_rn(le[1], t.xy[1][0], __dmul_rn(le[0], t.xy[0][0])));
    const double xe1 = __fma_rn(le[2], t.xy[2][1],
                                __fma_rn(le[1], t.xy[1][1], __dmul_rn(le[0], t.xy[0][1])));
    if (!(np_hypot(__dsub_rn(xe0, w.lx), __dsub_rn(xe1, w.ly)) >= eps_prog)) {
      status = ST_STUCK;
      stuck = kNearestPending;
      qx = x0;
      qy = x1;
      break;
    }
    w.put(1, ei, ej, tpar, xe0, xe1);
    // lam_exit @ vals[tri]  (3,)@(3,)
    const double val_exit = __fma_rn(le[2], t.f[2], __fma_rn(le[1], t.f[1], __dmul_rn(le[0], t.f[0])));
    if (target == ei || target == ej) {
      w.put(0, target, -1, 0.0, m.vertices[2 * target], m.vertices[2 * target + 1]);
      status = ST_REACHED;
      break;
    }
    const int64_t nt = sel3(slot_exit, t.nbr);
    bool enters = false;
    if (nt >= 0) {
      // _enters (paths.py:256-266); on success its geometry carries into the
      // next step
      load_tri(m, nt, ct);
      double gu[2];
      gradient(ct, vals, gu);
      cnorm = np_hypot(gu[0], gu[1]);
      if (cnorm > 0.0) {
        cd[0] = __ddiv_rn(-gu[0], cnorm);
        cd[1] = __ddiv_rn(-gu[1], cnorm);
        int so = 0;
        for (int s = 0; s < 3; ++s)
          if (ct.v[s] != ei && ct.v[s] != ej) so = s;
        cscale = dlam_of(ct, cd, cdl);
        enters = sel3(so, cdl) > __dmul_rn(1e-12, cscale);
      }
    }
    if (enters) {
      // the triangle after this one is one of nt's other neighbours
#pragma unroll
      for (int s = 0; s < 3; ++s)
        if (ct.nbr[s] != ti) prefetch_rec(m, ct.nbr[s]);
      carry = true;
      ti = nt;
      x0 = xe0;
      x1 = xe1;
      cur = val_exit;
      continue;
    }
    // _slide_along_edge (paths.py:268-274); stuck-vertex reference point is
    // the entry point for a boundary edge, the exit point otherwise.
    const double rx = nt < 0 ? x0 : xe0, ry = nt < 0 ? x1 : xe1;
    const int ssw = (sel3(o1, t.f) < sel3(o0, t.f)) ? o1 : o0;  // vals[ej] < vals[ei] ? ej : ei
    const int64_t sw = sel3(ssw, t.v);
    if (sel3(ssw, t.f) >= val_exit) {
      status = ST_STUCK;
      stuck = kNearestPending;
      qx = rx;
      qy = ry;
      break;
    }
    w.put(0, sw, -1, 0.0, sel3xy(ssw, t.xy, 0), sel3xy(ssw, t.xy, 1));
    in_tri = false;
    v = sw;
  }
  out.count[p] = w.count;
  out.status[p] = status;
  out.stuck[p] = stuck;
  if (stuck == kNearestPending) {
    out.qx[p] = qx;
    out.qy[p] = qy;
  }
}

// A stuck path's reported vertex is the mesh vertex nearest to a point
// (paths.py:287-289, np.argmin of np.hypot over all n vertices).  That O(n)
// scan would serialise one thread of the tracer for milliseconds, so the
// tracer only records the query point and this kernel resolves it with one
// CTA per pending path: strided per-thread scans, then a (distance, index)
// lexicographic block minimum = numpy's first minimum.
__global__ void __launch_bounds__(256) nearest_resolve_kernel(pf_mesh_t m, int64_t npaths,
                                                              pf_paths_t out) {
  const int64_t p = blockIdx.x;
  if (p >= npaths || out.stuck[p] != kNearestPending) return;
  const double x = out.qx[p], y = out.qy[p];
  double bd = INFINITY;
  int64_t bv = INT64_MAX;
  for (int64_t v = threadIdx.x; v < m.n; v += blockDim.x) {
    const double d = np_hypot(__dsub_rn(m.vertices[2 * v], x), __dsub_rn(m.vertices[2 * v + 1], y));
    if (d < bd) {
      bd = d;
      bv = v;
    }
  }
  __shared__ double sd[256];
  __shared__ int64_t sv[256];
  sd[threadIdx.x] = bd;
  sv[threadIdx.x] = bv;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double d2 = sd[threadIdx.x + o];
      const int64_t v2 = sv[threadIdx.x + o];
      if (d2 < sd[threadIdx.x] || (d2 == sd[threadIdx.x] && v2 < sv[threadIdx.x])) {
        sd[threadIdx.x] = d2;
        sv[threadIdx.x] = v2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out.stuck[p] = sv[0] == INT64_MAX ? 0 : sv[0];
}

// edge_descent (paths.py:71-94): vertex walk to the neighbour with the largest
// value drop (first maximum in ascending neighbour order), one thread per path.
__global__ void __launch_bounds__(kTraceThreads) edge_trace_kernel(
    pf_mesh_t m, const double *fields, int64_t field_ld, int64_t vertex_ld,
    const int64_t *targets, const int64_t *sources, const int32_t *field_of, int64_t npaths,
    int64_t cap, pf_paths_t out) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= npaths) return;
  const int64_t fi = field_of ? field_of[p] : 0;
  const FieldView vals{fields + fi * field_ld, vertex_ld};
  const int64_t target = targets[fi];
  int64_t cur = sources[p];
  Writer w{&out, p, 0, 0.0, 0.0};
  w.put(0, cur, -1, 0.0, m.vertices[2 * cur], m.vertices[2 * cur + 1]);
  int status = ST_MAX;
  int64_t stuck = -1;
  for (int64_t it = 0; it < cap; ++it) {
    if (cur == target) {
      status = ST_REACHED;
      break;
    }
    const double fc = vals[cur];
    int64_t best = -1;
    double bd = 0.0;
    for (int64_t e = m.nb_ptr[cur]; e < m.nb_ptr[cur + 1]; ++e) {
      const int64_t u = m.nb_idx[e];
      const double drop = __dsub_rn(fc, vals[u]);
      if (best < 0 || drop > bd) {
        bd = drop;
        best = u;
      }
    }
    if (best < 0 || bd <= 0.0) {
      status = ST_STUCK;
      stuck = cur;
      break;
    }
    cur = best;
    w.put(0, cur, -1, 0.0, m.vertices[2 * cur], m.vertices[2 * cur + 1]);
  }
  out.count[p] = w.count;
  out.status[p] = status;
  out.stuck[p] = stuck;
}

// find_local_minima (paths.py:314-324): v != target with neighbours, strictly
// below every neighbour.
__global__ void local_minima_kernel(pf_mesh_t m, const double *vals, int64_t target,
                                    uint8_t *out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < m.n;
       v += (int64_t)gridDim.x * blockDim.x) {
    bool mn = v != target && m.nb_ptr[v + 1] > m.nb_ptr[v];
    const double fv = vals[v];
    for (int64_t e = m.nb_ptr[v]; mn && e < m.nb_ptr[v + 1]; ++e) mn = fv < vals[m.nb_idx[e]];
    out[v] = mn ? 1 : 0;
  }
}

__global__ void tri_geometry_kernel(pf_mesh_t m, double *G) {
  for (int64_t ti = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ti < m.nt;
       ti += (int64_t)gridDim.x * blockDim.x) {
    const int v[3] = {m.triangles[3 * ti], m.triangles[3 * ti + 1], m.triangles[3 * ti + 2]};
    double g[3][2];
    tri_G(m, ti, v, g);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      G[6 * ti + 2 * i] = g[i][0];
      G[6 * ti + 2 * i + 1] = g[i][1];
    }
  }
}

// Packed per-triangle records for load_tri (16 doubles = one 128-byte line):
// xy[3][2], G[3][2] (tri_G arithmetic), area, then int32 v0 v1 | v2 nbr0 | nbr1 nbr2.
__global__ void tri_pack_kernel(pf_mesh_t m, double *pack) {
  for (int64_t ti = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; ti < m.nt;
       ti += (int64_t)gridDim.x * blockDim.x) {
    const int v[3] = {m.triangles[3 * ti], m.triangles[3 * ti + 1], m.triangles[3 * ti + 2]};
    double g[3][2];
    tri_G(m, ti, v, g);
    double *r = pack + 16 * ti;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      r[2 * i] = m.vertices[2 * v[i]];
      r[2 * i + 1] = m.vertices[2 * v[i] + 1];
      r[6 + 2 * i] = g[i][0];
      r[7 + 2 * i] = g[i][1];
    }
    r[12] = m.areas[ti];
    auto pair = [](int lo, int hi) {
      return __longlong_as_double(static_cast<long long>(static_cast<uint32_t>(lo)) |
                                  (static_cast<long long>(static_cast<uint32_t>(hi)) << 32));
    };
    r[13] = pair(v[0], v[1]);
    r[14] = pair(v[2], m.tri_nbr[3 * ti]);
    r[15] = pair(m.tri_nbr[3 * ti + 1], m.tri_nbr[3 * ti + 2]);
  }
}

// triangle_gradient for a batch of triangles (paths.py:113-121)
__global__ void tri_gradient_kernel(pf_mesh_t m, const double *vals, const int64_t *tris,
                                    int64_t ntri, double *out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ntri) return;
  Tri t;
  load_tri(m, tris[i], t);
  double g[2];
  gradient(t, FieldView{vals, 1}, g);
  out[2 * i] = g[0];
  out[2 * i + 1] = g[1];
}

__global__ void hypot_kernel_batch(const double *x, const double *y, int64_t n, double *out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = np_hypot(x[i], y[i]);
}


// ---------------------------------------------------------------------------
// Path metric (paths.py:326-368): polyline resampling + Hausdorff distance.
// A "polyline instance" is one side of one compared pair: its points
// (pts[src_off .. src_off + len) as (x, y)), the pair's resampling step, and
// its slice of the resampled output.  Arithmetic follows numpy bit for bit
// (this file is built with -fmad=false): np.hypot segments, a sequential
// cumsum, np.linspace (i * step + 0.0, last = total), np.interp (largest j
// with arc[j] <= s, slope form with its NaN retries), and scipy cKDTree's
// 2-D squared distance (dx*dx) + (dy*dy).

// Thread per instance: arc lengths (arc[src_off + i]) and the shortest
// positive segment (segmin, +inf if none) for the default step.
__global__ void polyline_arc_kernel(const double *__restrict__ pts,
                                    const int64_t *__restrict__ src_off,
                                    const int64_t *__restrict__ len, int64_t ninst,
                                    double *__restrict__ arc, double *__restrict__ segmin) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= ninst) return;
  const int64_t o = src_off[p], L = len[p];
  double a = 0.0, mn = __longlong_as_double(0x7ff0000000000000LL);
  if (L > 0) arc[o] = 0.0;
  for (int64_t i = 1; i < L; ++i) {
    const double dx = __dsub_rn(pts[2 * (o + i)], pts[2 * (o + i - 1)]);
    const double dy = __dsub_rn(pts[2 * (o + i) + 1], pts[2 * (o + i - 1) + 1]);
    const double sg = np_hypot(dx, dy);
    if (sg > 0.0 && sg < mn) mn = sg;
    a = __dadd_rn(a, sg);
    arc[o + i] = a;
  }
  if (segmin) segmin[p] = mn;
}

// One thread per resampled point; instance found by binary search over the
// output offsets.  cnt[p] == 0 marks "copy the input" (fewer than 2 points),
// cnt[p] == -1 "first point only" (zero total length).
__global__ void polyline_resample_kernel(const double *__restrict__ pts,
                                         const int64_t *__restrict__ src_off,
                                         const int64_t *__restrict__ len,
                                         const double *__restrict__ arc,
                                         const int64_t *__restrict__ cnt,
                                         const int64_t *__restrict__ out_off, int64_t ninst,
                                         double *__restrict__ out) {
  const int64_t total_out = out_off[ninst];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total_out;
       g += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = ninst;  // largest p with out_off[p] <= g
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (out_off[mid] <= g) lo = mid; else hi = mid;
    }
    const int64_t p = lo, i = g - out_off[p], o = src_off[p], L = len[p], c = cnt[p];
    if (c <= 0) {  // input copied through (len < 2) or its first point (total <= 0)
      out[2 * g] = pts[2 * (o + i)];
      out[2 * g + 1] = pts[2 * (o + i) + 1];
      continue;
    }
    const double total = arc[o + L - 1];
    const int64_t div = c - 1;
    double s;
    if (i == c - 1) {
      s = total;
    } else {
      const double step = __ddiv_rn(total, static_cast<double>(div));
      s = step == 0.0 ? __dmul_rn(__ddiv_rn(static_cast<double>(i), static_cast<double>(div)), total)
                      : __dmul_rn(static_cast<double>(i), step);
      s = __dadd_rn(s, 0.0);
    }
    // np.interp: j = largest index with arc[j] <= s (s in [arc[0], arc[L-1]])
    int64_t a = 0, b = L;  // arc[a] <= s < arc[b] (arc[L] = +inf)
    while (b - a > 1) {
      const int64_t mid = (a + b) >> 1;
      if (arc[o + mid] <= s) a = mid; else b = mid;
    }
    const int64_t j = a;
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      const double *fp = pts + 2 * o + d;
      double r;
      if (j == L - 1 || arc[o + j] == s) {
        r = fp[2 * j];
      } else {
        const double x0 = arc[o + j], x1 = arc[o + j + 1];
        const double y0 = fp[2 * j], y1 = fp[2 * (j + 1)];
        const double slope = __ddiv_rn(__dsub_rn(y1, y0), __dsub_rn(x1, x0));
        r = __dadd_rn(__dmul_rn(slope, __dsub_rn(s, x0)), y0);
        if (isnan(r)) {
          r = __dadd_rn(__dmul_rn(slope, __dsub_rn(s, x1)), y1);
          if (isnan(r) && y0 == y1) r = y0;
        }
      }
      out[2 * g + d] = r;
    }
  }
}

// Directed squared Hausdorff term for (pair, direction) = blockIdx.y: max over
// the resampled points x of instance X (256 per block) of min over the
// resampled points y of instance Y of (dx*dx) + (dy*dy), folded into best[pair]
// with an atomic max on the bits of a non-negative double (order-preserving).
//
// The resampled points of Y lie on Y's source polyline at uniform arc spacing
// h = total / (cnt - 1), so instead of all |Y| points each x visits Y's source
// segments: the squared distance to segment j is a lower bound for every
// resampled point on it (less a rounding margin), and along the segment the
// nearest resampled point is within two indices of x's projection.  Pass 1
// takes the segment with the smallest bound and evaluates its window; pass 2
// evaluates the window of every segment whose bound does not exceed that
// minimum.  Only window points are measured, with the reference's exact
// arithmetic, so the result is the exhaustive minimum bit for bit.
constexpr int kHdThreads = 256, kHdTile = 512;

struct HdSeg {
  double x0, y0, ex, ey, inv_l2, a0, a1, pad;
};

__device__ __forceinline__ double seg_lower_bound(const HdSeg &g, double px, double py,
                                                  double &tpar) {
  double t = ((px - g.x0) * g.ex + (py - g.y0) * g.ey) * g.inv_l2;
  t = fmin(fmax(t, 0.0), 1.0);
  tpar = t;
  const double qx = px - (g.x0 + t * g.ex), qy = py - (g.y0 + t * g.ey);
  return qx * qx + qy * qy;
}

__device__ __forceinline__ double window_min(const double *__restrict__ ry, int64_t ny, double h,
                                             double s_star, double px, double py, double best) {
  const double fi = rint(s_star / h);
  int64_t i0 = static_cast<int64_t>(fi) - 2, i1 = static_cast<int64_t>(fi) + 2;
  if (i0 < 0) i0 = 0;
  if (i1 > ny - 1) i1 = ny - 1;
  for (int64_t i = i0; i <= i1; ++i) {
    const double dx = __dsub_rn(px, ry[2 * i]), dy = __dsub_rn(py, ry[2 * i + 1]);
    best = fmin(best, __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
  }
  return best;
}

__global__ void __launch_bounds__(kHdThreads) hausdorff_kernel(
    const double *__restrict__ pts, const double *__restrict__ arc,
    const int64_t *__restrict__ src_off, const int64_t *__restrict__ len,
    const int64_t *__restrict__ cnt, const double *__restrict__ rp,
    const int64_t *__restrict__ out_off, const int64_t *__restrict__ inst_a,
    const int64_t *__restrict__ inst_b, unsigned long long *__restrict__ best_bits) {
  __shared__ HdSeg segs[kHdTile];
  const int64_t pair = blockIdx.y >> 1;
  const bool rev = blockIdx.y & 1;
  const int64_t ix = rev ? inst_b[pair] : inst_a[pair];
  const int64_t iy = rev ? inst_a[pair] : inst_b[pair];
  const int64_t xa = out_off[ix], nx = out_off[ix + 1] - xa;
  const int64_t ya = out_off[iy], ny = out_off[iy + 1] - ya;
  const int64_t x0 = static_cast<int64_t>(blockIdx.x) * kHdThreads;
  if (x0 >= nx) return;
  const int64_t xi = x0 + threadIdx.x;
  const bool live = xi < nx;
  const double px = live ? rp[2 * (xa + xi)] : 0.0, py = live ? rp[2 * (xa + xi) + 1] : 0.0;
  const double *ry = rp + 2 * ya;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double best = inf;
  const int64_t c = cnt[iy];
  if (c <= 0) {  // Y is its input copied (< 2 points) or one point: exhaustive
    for (int64_t i = 0; i < ny; ++i) {
      const double dx = __dsub_rn(px, ry[2 * i]), dy = __dsub_rn(py, ry[2 * i + 1]);
      best = fmin(best, __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    }
  } else {
    const int64_t so = src_off[iy], nseg = len[iy] - 1;
    const double total = arc[so + nseg];
    const double h = __ddiv_rn(total, static_cast<double>(c - 1));
    // rounding margin on the bounds: the resampled points sit within a few
    // ulps of their segment, the bound itself is a few ulps off
    const double scale = fabs(px) + fabs(py) + 1.0;
    double lb_min = inf, s_at_min = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
      for (int64_t t0 = 0; t0 < nseg; t0 += kHdTile) {
        const int nt = static_cast<int>(nseg - t0 < kHdTile ? nseg - t0 : kHdTile);
        __syncthreads();
        for (int u = threadIdx.x; u < nt; u += kHdThreads) {
          const int64_t j = so + t0 + u;
          HdSeg g;
          g.x0 = pts[2 * j];
          g.y0 = pts[2 * j + 1];
          g.ex = pts[2 * j + 2] - g.x0;
          g.ey = pts[2 * j + 3] - g.y0;
          const double l2 = g.ex * g.ex + g.ey * g.ey;
          g.inv_l2 = l2 > 0.0 ? 1.0 / l2 : 0.0;
          g.a0 = arc[j];
          g.a1 = arc[j + 1];
          segs[u] = g;
        }
        __syncthreads();
        if (!live) continue;
        for (int u = 0; u < nt; ++u) {
          const HdSeg &g = segs[u];
          double tpar;
          const double lb = seg_lower_bound(g, px, py, tpar);
          const double s_star = g.a0 + tpar * (g.a1 - g.a0);
          if (pass == 0) {
            if (lb < lb_min) {
              lb_min = lb;
              s_at_min = s_star;
            }
          } else {
            const double d = sqrt(lb) - 1e-12 * scale;
            if (d <= 0.0 || d * d <= best) best = window_min(ry, ny, h, s_star, px, py, best);
          }
        }
      }
      if (pass == 0 && live) best = window_min(ry, ny, h, s_at_min, px, py, best);
    }
  }
  double m = live ? best : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0)
    atomicMax(best_bits + pair, static_cast<unsigned long long>(__double_as_longlong(m)));
}

}  // namespace pf

using namespace pf;

extern "C" {

int pf_trace_fields_f64(const pf_mesh_t *mesh, const double *fields, int64_t field_ld,
                        int64_t vertex_ld, const int64_t *targets, const int64_t *sources,
                        const int32_t *field_of, int64_t npaths, int64_t step_cap,
                        const pf_paths_t *out, pf_stream_t stream) {
  if (!mesh || !fields || !targets || !sources || !out) return fail(PF_E_ARG, "trace: null");
  if (npaths <= 0) return 0;
  if (vertex_ld < 1 || field_ld < 0) return fail(PF_E_ARG, "trace: bad field layout");
  if (!out->count || !out->status || !out->stuck) return fail(PF_E_ARG, "trace: null outputs");
  // 8 paths per warp (one per 4 lanes): the walks diverge step by step, and a
  // warp's time is the sum over its steps of every taken branch.  C5 (10,000
  // paths on the C4 mesh): 32 paths per warp 13.4 ms, 16 12.4, ~11 12.1, 8 11.7,
  // ~6 12.1, ~5 17.2, 4 18.2 (tools/probe_trace_layout.py, the spread as a parameter).
  constexpr int spread = kTraceSpread;
  const int64_t blocks = (npaths * spread + kTraceThreads - 1) / kTraceThreads;
  if (!out->qx || !out->qy) return fail(PF_E_ARG, "trace: null qx/qy");
  trace_kernel<<<static_cast<unsigned>(blocks), kTraceThreads, 0, as_stream(stream)>>>(
      *mesh, fields, field_ld, vertex_ld, targets, sources, field_of, npaths, step_cap, *out,
      spread);
  if (int e = check_launch("trace")) return e;
  nearest_resolve_kernel<<<static_cast<unsigned>(npaths), 256, 0, as_stream(stream)>>>(
      *mesh, npaths, *out);
  return check_launch("nearest_resolve");
}

int pf_trace_batch_f64(const pf_mesh_t *mesh, const double *fields, const int64_t *targets,
                       const int64_t *sources, const int32_t *field_of, int64_t npaths,
                       int64_t step_cap, const pf_paths_t *out, pf_stream_t stream) {
  if (!mesh) return fail(PF_E_ARG, "trace: null");
  return pf_trace_fields_f64(mesh, fields, mesh->n, 1, targets, sources, field_of, npaths,
                             step_cap, out, stream);
}

int pf_edge_descent_batch_f64(const pf_mesh_t *mesh, const double *fields,
                              const int64_t *targets, const int64_t *sources,
                              const int32_t *field_of, int64_t npaths, int64_t step_cap,
                              const pf_paths_t *out, pf_stream_t stream) {
  if (!mesh || !fields || !targets || !sources || !out) return fail(PF_E_ARG, "edge: null");
  if (npaths <= 0) return 0;
  const int64_t blocks = (npaths + kTraceThreads - 1) / kTraceThreads;
  edge_trace_kernel<<<static_cast<unsigned>(blocks), kTraceThreads, 0, as_stream(stream)>>>(
      *mesh, fields, mesh->n, 1, targets, sources, field_of, npaths, step_cap, *out);
  return check_launch("edge_descent");
}

int pf_local_minima_f64(const pf_mesh_t *mesh, const double *vals, int64_t target, uint8_t *out,
                        pf_stream_t stream) {
  if (!mesh || !vals || !out) return fail(PF_E_ARG, "local_minima: null");
  if (mesh->n <= 0) return 0;
  local_minima_kernel<<<sm_count() * 4, 256, 0, as_stream(stream)>>>(*mesh, vals, target, out);
  return check_launch("local_minima");
}

int pf_triangle_gradient_f64(const pf_mesh_t *mesh, const double *vals, const int64_t *tris,
                             int64_t ntri, double *out, pf_stream_t stream) {
  if (!mesh || !vals || !tris || !out) return fail(PF_E_ARG, "triangle_gradient: null");
  if (ntri <= 0) return 0;
  tri_gradient_kernel<<<static_cast<unsigned>((ntri + 127) / 128), 128, 0, as_stream(stream)>>>(
      *mesh, vals, tris, ntri, out);
  return check_launch("triangle_gradient");
}

int pf_mesh_geometry_f64(const pf_mesh_t *mesh, double *G, pf_stream_t stream) {
  if (!mesh || !G) return fail(PF_E_ARG, "mesh_geometry: null");
  if (mesh->nt <= 0) return 0;
  pf_mesh_t m = *mesh;
  m.G = nullptr;  // compute, do not read
  tri_geometry_kernel<<<sm_count() * 4, 256, 0, as_stream(stream)>>>(m, G);
  return check_launch("mesh_geometry");
}

int pf_mesh_pack_f64(const pf_mesh_t *mesh, double *pack, pf_stream_t stream) {
  if (!mesh || !pack) return fail(PF_E_ARG, "mesh_pack: null");
  if (mesh->nt <= 0) return 0;
  if (reinterpret_cast<uintptr_t>(pack) & 127) return fail(PF_E_ALIGN, "mesh_pack: 128-byte alignment");
  pf_mesh_t m = *mesh;
  m.G = nullptr;
  m.pack = nullptr;
  tri_pack_kernel<<<sm_count() * 4, 256, 0, as_stream(stream)>>>(m, pack);
  return check_launch("mesh_pack");
}

int pf_np_hypot_f64(const double *x, const double *y, int64_t n, double *out,
                    pf_stream_t stream) {
  if (n <= 0) return 0;
  if (!x || !y || !out) return fail(PF_E_ARG, "np_hypot: null");
  hypot_kernel_batch<<<static_cast<unsigned>((n + 255) / 256), 256, 0, as_stream(stream)>>>(
      x, y, n, out);
  return check_launch("np_hypot");
}

int pf_polyline_arc_f64(const double *pts, const int64_t *src_off, const int64_t *len,
                        int64_t ninst, double *arc, double *segmin, pf_stream_t stream) {
  if (ninst <= 0) return 0;
  if (!pts || !src_off || !len || !arc) return fail(PF_E_ARG, "polyline_arc: null");
  polyline_arc_kernel<<<static_cast<unsigned>((ninst + 127) / 128), 128, 0, as_stream(stream)>>>(
      pts, src_off, len, ninst, arc, segmin);
  return check_launch("polyline_arc");
}

int pf_polyline_resample_f64(const double *pts, const int64_t *src_off, const int64_t *len,
                             const double *arc, const int64_t *cnt, const int64_t *out_off,
                             int64_t ninst, int64_t total_out, double *out, pf_stream_t stream) {
  if (ninst <= 0 || total_out <= 0) return 0;
  if (!pts || !src_off || !len || !arc || !cnt || !out_off || !out)
    return fail(PF_E_ARG, "polyline_resample: null");
  int64_t blocks = (total_out + 255) / 256;
  if (blocks > static_cast<int64_t>(sm_count()) * 32) blocks = static_cast<int64_t>(sm_count()) * 32;
  polyline_resample_kernel<<<static_cast<unsigned>(blocks), 256, 0, as_stream(stream)>>>(
      pts, src_off, len, arc, cnt, out_off, ninst, out);
  return check_launch("polyline_resample");
}

int pf_hausdorff_pairs_f64(const double *pts, const double *arc, const int64_t *src_off,
                           const int64_t *len, const int64_t *cnt, const double *rp,
                           const int64_t *out_off, const int64_t *inst_a, const int64_t *inst_b,
                           int64_t npairs, int64_t max_points, uint64_t *best_bits,
                           pf_stream_t stream) {
  if (npairs <= 0 || max_points <= 0) return 0;
  if (!pts || !arc || !src_off || !len || !cnt || !rp || !out_off || !inst_a || !inst_b ||
      !best_bits)
    return fail(PF_E_ARG, "hausdorff_pairs: null");
  if (2 * npairs > 65535) return fail(PF_E_DOMAIN, "hausdorff_pairs: at most 32767 pairs per call");
  cudaMemsetAsync(best_bits, 0, npairs * sizeof(uint64_t), as_stream(stream));
  dim3 grid(static_cast<unsigned>((max_points + kHdThreads - 1) / kHdThreads),
            static_cast<unsigned>(2 * npairs));
  hausdorff_kernel<<<grid, kHdThreads, 0, as_stream(stream)>>>(
      pts, arc, src_off, len, cnt, rp, out_off, inst_a, inst_b,
      reinterpret_cast<unsigned long long *>(best_bits));
  return check_launch("hausdorff_pairs");
}

}  // extern "C"
