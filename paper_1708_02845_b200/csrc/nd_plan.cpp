// nd_plan.cpp — host-side symbolic phase of the device Poisson-kernel solver.
//
// Replaces the ordering + symbolic factorisation half of SuperLU's
// `splu(-Lc_II)` (laplacian.py:29-45, used by solvers.py:278-303) with a
// plan for a multifrontal Cholesky of the SPD interior block A = -Lc_II:
//
//   * geometric nested dissection of the interior vertices (the mesh is
//     planar with coordinates, so a median split of the wider bounding-box
//     axis plus the smaller one-sided vertex separator gives O(sqrt n)
//     separators without a graph partitioner);
//   * a post-order elimination tree of "fronts": a node owns a contiguous
//     range C of the permuted order (a separator, or a leaf sub-domain) and
//     its front is C plus R, the ancestor vertices coupled to its subtree;
//   * the scatter lists the device kernels consume: where every entry of A
//     lands in its front (`a_dst`), where each child's update matrix lands
//     in its parent (`relmap`), where each entry of the right-hand side
//     B = Lc_IB lands (`b_*`), and which 32-column tiles of B can be non-zero
//     under each node (`act_*`; the forward solve skips the rest).
//
// Nothing here is numeric: values stay on the device (poisson.cu) and are
// addressed by their index in the mesh's neighbour CSR.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <future>
#include <memory>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pathfield_b200.h"

namespace pf {
void set_error(const char *fmt, ...);
}

namespace {

struct Plan {
  // inputs
  int64_t n = 0, m = 0, k = 0;
  int leaf = 64, ta = 32;
  // ordering
  std::vector<int32_t> perm_orig;  // perm position -> original vertex id
  std::vector<int32_t> iperm;      // interior-local id -> perm position
  // nodes (post-order: children before parents)
  std::vector<int32_t> c0, cn, rn, fn, parent, height;
  std::vector<int64_t> foff;
  std::vector<int32_t> ch_ptr, ch_idx;
  std::vector<int64_t> r_ptr;
  std::vector<int32_t> r_pos;   // R as perm positions (sorted)
  std::vector<int32_t> r_orig;  // R as original vertex ids
  std::vector<int64_t> relmap_off;  // per node: offset of its map into the parent front
  std::vector<int32_t> relmap;
  std::vector<int64_t> a_ptr, a_dst, a_src;
  std::vector<int64_t> b_ptr;
  std::vector<int32_t> b_row, b_col;
  std::vector<int64_t> b_src;
  std::vector<int64_t> act_ptr;
  std::vector<int32_t> act_tile;
  std::vector<int64_t> act_voff;  // per active (node, tile): offset of its f x ta block
  std::vector<int64_t> tile_item;  // node*ntiles + tile -> active item index or -1
  std::vector<int32_t> level_ptr, level_nodes;
  int64_t ntiles = 0, f_total = 0, v_total = 0, nnz_l = 0;
  double flops_factor = 0, flops_solve = 0;
  int32_t max_f = 0, max_c = 0, max_r = 0;
};

struct Builder {
  const double *xy;
  const int64_t *nb_ptr;
  const int64_t *nb_idx;
  const std::vector<int32_t> &ilocal;  // orig -> interior-local or -1
  const std::vector<int32_t> &interior;  // interior-local -> orig
  Plan &P;
  std::vector<int8_t> side;  // per interior-local: -1 outside, 0 left, 1 right
  std::vector<std::vector<int32_t>> node_children;
  std::vector<std::vector<int32_t>> node_C;  // interior-local ids (leaf / separator)
  int32_t next_pos = 0;

  Builder(const double *xy_, const int64_t *p, const int64_t *i,
          const std::vector<int32_t> &il, const std::vector<int32_t> &in, Plan &pl)
      : xy(xy_), nb_ptr(p), nb_idx(i), ilocal(il), interior(in), P(pl),
        side(in.size(), -1) {}

  double coord(int32_t v, int axis) const { return xy[2 * (int64_t)interior[v] + axis]; }

  int32_t new_node(std::vector<int32_t> &&C, std::vector<int32_t> &&children) {
    const int32_t id = (int32_t)node_C.size();
    // positions: C is numbered after every vertex of the children (post-order)
    P.c0.push_back(next_pos);
    P.cn.push_back((int32_t)C.size());
    for (int32_t v : C) {
      P.perm_orig[next_pos] = interior[v];
      P.iperm[v] = next_pos;
      ++next_pos;
    }
    node_C.push_back(std::move(C));
    node_children.push_back(std::move(children));
    return id;
  }

  // Nested dissection of S (interior-local ids), in two phases.  partition()
  // splits S recursively into a tree of (C, children) and is where the time
  // goes (a median split and a separator scan per level); below the top
  // kParDepth levels' splits the two halves run on separate threads (they touch
  // disjoint vertices; `side` is written per vertex).  number() then walks the
  // tree in post-order and assigns node ids and permutation positions exactly
  // as the sequential recursion did, so the plan is independent of threading.
  struct Part {
    std::vector<int32_t> C;
    std::vector<std::unique_ptr<Part>> ch;
  };
  static constexpr int kParDepth = 4;  // up to 16 concurrent subtrees

  std::unique_ptr<Part> partition(std::vector<int32_t> &S, int depth) {
    auto node = std::make_unique<Part>();
    if ((int64_t)S.size() <= P.leaf) {
      // leaf: order by the wider axis for locality of the dense front
      node->C = S;
      return node;
    }
    double lo[2] = {1e300, 1e300}, hi[2] = {-1e300, -1e300};
    for (int32_t v : S)
      for (int a = 0; a < 2; ++a) {
        const double c = coord(v, a);
        lo[a] = std::min(lo[a], c);
        hi[a] = std::max(hi[a], c);
      }
    const int axis = (hi[0] - lo[0]) >= (hi[1] - lo[1]) ? 0 : 1;
    const size_t half = S.size() / 2;
    auto less = [&](int32_t a, int32_t b) {
      const double ca = coord(a, axis), cb = coord(b, axis);
      return ca < cb || (ca == cb && a < b);
    };
    std::nth_element(S.begin(), S.begin() + half, S.end(), less);
    for (size_t i = 0; i < S.size(); ++i) side[S[i]] = i < half ? 0 : 1;
    // one-sided separators: vertices of one half adjacent to the other half
    std::vector<int32_t> sep[2];
    for (int32_t v : S) {
      const int8_t sv = side[v];
      const int32_t o = interior[v];
      for (int64_t e = nb_ptr[o]; e < nb_ptr[o + 1]; ++e) {
        const int32_t u = ilocal[nb_idx[e]];
        if (u >= 0 && side[u] == 1 - sv) {
          sep[sv].push_back(v);
          break;
        }
      }
    }
    const int pick = sep[1].size() < sep[0].size() ? 1 : 0;
    for (int32_t v : sep[pick]) side[v] = 2;
    std::vector<int32_t> part[2];
    for (int32_t v : S)
      if (side[v] < 2) part[side[v]].push_back(v);
    for (int32_t v : S) side[v] = -1;
    std::vector<int32_t>().swap(S);
    if (depth < kParDepth && !part[0].empty() && !part[1].empty()) {
      auto left = std::async(std::launch::async,
                             [this, &part, depth] { return partition(part[0], depth + 1); });
      auto right = partition(part[1], depth + 1);
      node->ch.push_back(left.get());
      node->ch.push_back(std::move(right));
    } else {
      for (int h = 0; h < 2; ++h)
        if (!part[h].empty()) node->ch.push_back(partition(part[h], depth + 1));
    }
    std::vector<int32_t> &C = node->C;
    C = std::move(sep[pick]);
    std::sort(C.begin(), C.end(), [&](int32_t a, int32_t b) {
      const double ca = coord(a, 1 - axis), cb = coord(b, 1 - axis);
      return ca < cb || (ca == cb && a < b);
    });
    return node;
  }

  int32_t number(Part &t) {
    std::vector<int32_t> children;
    for (auto &c : t.ch) children.push_back(number(*c));
    t.ch.clear();
    return new_node(std::move(t.C), std::move(children));
  }

  int32_t build(std::vector<int32_t> &S) {
    auto root = partition(S, 0);
    return number(*root);
  }
};

int64_t lower_pos(const std::vector<int32_t> &v, int64_t lo, int64_t hi, int32_t x) {
  return std::lower_bound(v.begin() + lo, v.begin() + hi, x) - v.begin();
}

// f(i) for i in [0, n) on up to 16 host threads, dynamically chunked (fronts
// vary in size); sequential for small n.  f must only write what index i owns.
template <class F>
void parallel_for(int64_t n, F &&f) {
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < 2048 || hw == 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  constexpr int64_t kChunk = 64;
  std::atomic<int64_t> next{0};
  auto work = [&] {
    for (;;) {
      const int64_t a = next.fetch_add(kChunk);
      if (a >= n) return;
      const int64_t b = std::min(n, a + kChunk);
      for (int64_t i = a; i < b; ++i) f(i);
    }
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < hw; ++t) pool.emplace_back(work);
  work();
  for (auto &th : pool) th.join();
}

int build_plan(Plan &P, const double *xy, const int64_t *nb_ptr, const int64_t *nb_idx,
               const uint8_t *is_boundary) {
  const int64_t n = P.n;
  std::vector<int32_t> ilocal(n, -1), interior, bcol(n, -1);
  int64_t k = 0;
  for (int64_t v = 0; v < n; ++v) {
    if (is_boundary[v]) {
      bcol[v] = (int32_t)k++;
    } else {
      ilocal[v] = (int32_t)interior.size();
      interior.push_back((int32_t)v);
    }
  }
  P.k = k;
  P.m = (int64_t)interior.size();
  const int64_t m = P.m;
  P.perm_orig.assign(m, -1);
  P.iperm.assign(m, -1);
  Builder B(xy, nb_ptr, nb_idx, ilocal, interior, P);
  if (m > 0) {
    std::vector<int32_t> S(m);
    for (int64_t i = 0; i < m; ++i) S[i] = (int32_t)i;
    B.build(S);
  }
  const int32_t nn = (int32_t)B.node_C.size();
  // children CSR, parents, heights
  P.parent.assign(nn, -1);
  P.height.assign(nn, 0);
  P.ch_ptr.assign(nn + 1, 0);
  for (int32_t s = 0; s < nn; ++s) {
    P.ch_ptr[s + 1] = P.ch_ptr[s] + (int32_t)B.node_children[s].size();
    int32_t h = 0;
    for (int32_t c : B.node_children[s]) {
      P.parent[c] = s;
      P.ch_idx.push_back(c);
      h = std::max(h, P.height[c] + 1);
    }
    P.height[s] = h;
  }
  // R sets (perm positions > c1), bottom-up (post-order ids)
  P.r_ptr.assign(nn + 1, 0);
  P.rn.assign(nn, 0);
  // R[s] = the sorted positions >= c1 coupled to C (mesh neighbours) or to the
  // children's R; fronts of one height are independent, so each height is one
  // parallel pass (children always have a smaller height)
  std::vector<std::vector<int32_t>> R(nn);
  int32_t hmax_r = 0;
  for (int32_t s = 0; s < nn; ++s) hmax_r = std::max(hmax_r, P.height[s]);
  std::vector<std::vector<int32_t>> by_h(hmax_r + 1);
  for (int32_t s = 0; s < nn; ++s) by_h[P.height[s]].push_back(s);
  for (int32_t h = 0; h <= hmax_r; ++h) {
    const std::vector<int32_t> &nodes = by_h[h];
    parallel_for((int64_t)nodes.size(), [&](int64_t i) {
      const int32_t s = nodes[i];
      const int32_t c1 = P.c0[s] + P.cn[s];
      std::vector<int32_t> tmp;
      for (int32_t v : B.node_C[s]) {
        const int32_t o = interior[v];
        for (int64_t e = nb_ptr[o]; e < nb_ptr[o + 1]; ++e) {
          const int32_t u = ilocal[nb_idx[e]];
          if (u < 0) continue;
          const int32_t p = P.iperm[u];
          if (p >= c1) tmp.push_back(p);
        }
      }
      for (int32_t j = P.ch_ptr[s]; j < P.ch_ptr[s + 1]; ++j)
        for (int32_t p : R[P.ch_idx[j]])
          if (p >= c1) tmp.push_back(p);
      std::sort(tmp.begin(), tmp.end());
      tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
      P.rn[s] = (int32_t)tmp.size();
      R[s] = std::move(tmp);
    });
  }
  for (int32_t s = 0; s < nn; ++s) P.r_ptr[s + 1] = P.r_ptr[s] + P.rn[s];
  P.r_pos.resize(P.r_ptr[nn]);
  P.r_orig.resize(P.r_ptr[nn]);
  for (int32_t s = 0; s < nn; ++s)
    for (int32_t i = 0; i < P.rn[s]; ++i) {
      P.r_pos[P.r_ptr[s] + i] = R[s][i];
      P.r_orig[P.r_ptr[s] + i] = P.perm_orig[R[s][i]];
    }
  std::vector<std::vector<int32_t>>().swap(R);
  // fronts
  P.fn.assign(nn, 0);
  P.foff.assign(nn + 1, 0);
  for (int32_t s = 0; s < nn; ++s) {
    const int64_t c = P.cn[s], r = P.rn[s], f = c + r;
    P.fn[s] = (int32_t)f;
    P.foff[s + 1] = P.foff[s] + f * f;
    P.max_f = std::max<int32_t>(P.max_f, (int32_t)f);
    P.max_c = std::max<int32_t>(P.max_c, (int32_t)c);
    P.max_r = std::max<int32_t>(P.max_r, (int32_t)r);
    P.nnz_l += c * (c + 1) / 2 + c * r;
    P.flops_factor += (double)c * c * c / 3.0 + (double)c * c * r + (double)c * r * r;
    P.flops_solve += 2.0 * ((double)c * c + 2.0 * (double)c * r);
  }
  P.f_total = P.foff[nn];
  // local index of perm position p inside node s's front
  auto local = [&](int32_t s, int32_t p) -> int64_t {
    const int32_t c0 = P.c0[s], c1 = c0 + P.cn[s];
    if (p >= c0 && p < c1) return p - c0;
    const int64_t j = lower_pos(P.r_pos, P.r_ptr[s], P.r_ptr[s + 1], p);
    if (j >= P.r_ptr[s + 1] || P.r_pos[j] != p) return -1;
    return P.cn[s] + (j - P.r_ptr[s]);
  };
  // child -> parent front maps
  P.relmap_off.assign(nn + 1, 0);
  for (int32_t s = 0; s < nn; ++s) P.relmap_off[s + 1] = P.relmap_off[s] + P.rn[s];
  P.relmap.resize(P.relmap_off[nn]);
  std::atomic<int32_t> bad_rel{-1};
  parallel_for(nn, [&](int64_t si) {
    const int32_t s = (int32_t)si;
    const int32_t par = P.parent[s];
    for (int32_t i = 0; i < P.rn[s]; ++i) {
      const int64_t l = par >= 0 ? local(par, P.r_pos[P.r_ptr[s] + i]) : -1;
      if (l < 0) {
        bad_rel.store(s);
        return;
      }
      P.relmap[P.relmap_off[s] + i] = (int32_t)l;
    }
  });
  if (bad_rel.load() >= 0) {
    pf::set_error("nd plan: update row of node %d not in its parent front", (int)bad_rel.load());
    return PF_E_DOMAIN;
  }
  // A entries (lower triangle of each front's C columns) and B entries: counted,
  // then filled per front in parallel (each front owns its slice; same order as
  // a sequential pass)
  P.a_ptr.assign(nn + 1, 0);
  P.b_ptr.assign(nn + 1, 0);
  std::atomic<int32_t> bad_vertex{-1};
  auto front_entries = [&](int32_t s, bool fill) {
    const int64_t f = P.fn[s];
    const int32_t c0 = P.c0[s];
    int64_t ia = fill ? P.a_ptr[s] : 0, ib = fill ? P.b_ptr[s] : 0;
    for (int32_t j = 0; j < P.cn[s]; ++j) {
      const int32_t p = c0 + j;
      const int32_t o = P.perm_orig[p];
      if (fill) {
        P.a_dst[ia] = P.foff[s] + (int64_t)j * f + j;
        P.a_src[ia] = -1 - (int64_t)o;  // diagonal of vertex o
      }
      ++ia;
      for (int64_t e = nb_ptr[o]; e < nb_ptr[o + 1]; ++e) {
        const int64_t u = nb_idx[e];
        const int32_t ul = ilocal[u];
        if (ul < 0) {
          if (fill) {
            P.b_row[ib] = j;
            P.b_col[ib] = bcol[u];
            P.b_src[ib] = e;
          }
          ++ib;
          continue;
        }
        const int32_t pu = P.iperm[ul];
        if (pu <= p) continue;  // upper triangle / already eliminated
        if (fill) {
          const int64_t i = local(s, pu);
          if (i < 0) {
            bad_vertex.store(o);
            return;
          }
          P.a_dst[ia] = P.foff[s] + i * f + j;
          P.a_src[ia] = e;
        }
        ++ia;
      }
    }
    if (!fill) {
      P.a_ptr[s + 1] = ia;
      P.b_ptr[s + 1] = ib;
    }
  };
  parallel_for(nn, [&](int64_t s) { front_entries((int32_t)s, false); });
  for (int32_t s = 0; s < nn; ++s) {
    P.a_ptr[s + 1] += P.a_ptr[s];
    P.b_ptr[s + 1] += P.b_ptr[s];
  }
  P.a_dst.resize(P.a_ptr[nn]);
  P.a_src.resize(P.a_ptr[nn]);
  P.b_row.resize(P.b_ptr[nn]);
  P.b_col.resize(P.b_ptr[nn]);
  P.b_src.resize(P.b_ptr[nn]);
  parallel_for(nn, [&](int64_t s) { front_entries((int32_t)s, true); });
  if (bad_vertex.load() >= 0) {
    pf::set_error("nd plan: coupling of vertex %d not in its front", (int)bad_vertex.load());
    return PF_E_DOMAIN;
  }
  // active 32-column tiles of the forward solve (bottom-up union)
  P.ntiles = (k + P.ta - 1) / P.ta;
  std::vector<std::vector<int32_t>> act(nn);
  for (int32_t s = 0; s < nn; ++s) {
    std::vector<int32_t> &A = act[s];
    for (int64_t e = P.b_ptr[s]; e < P.b_ptr[s + 1]; ++e) A.push_back(P.b_col[e] / P.ta);
    for (int32_t i = P.ch_ptr[s]; i < P.ch_ptr[s + 1]; ++i) {
      const auto &Ac = act[P.ch_idx[i]];
      A.insert(A.end(), Ac.begin(), Ac.end());
    }
    std::sort(A.begin(), A.end());
    A.erase(std::unique(A.begin(), A.end()), A.end());
  }
  P.act_ptr.assign(nn + 1, 0);
  for (int32_t s = 0; s < nn; ++s) P.act_ptr[s + 1] = P.act_ptr[s] + (int64_t)act[s].size();
  P.act_tile.resize(P.act_ptr[nn]);
  P.act_voff.resize(P.act_ptr[nn] + 1);
  P.tile_item.assign((size_t)nn * P.ntiles, -1);
  int64_t voff = 0;
  for (int32_t s = 0; s < nn; ++s)
    for (size_t i = 0; i < act[s].size(); ++i) {
      const int64_t it = P.act_ptr[s] + (int64_t)i;
      P.act_tile[it] = act[s][i];
      P.act_voff[it] = voff;
      P.tile_item[(size_t)s * P.ntiles + act[s][i]] = it;
      voff += (int64_t)P.fn[s] * P.ta;  // [Y_C; V] block of the item
    }
  P.act_voff[P.act_ptr[nn]] = voff;
  P.v_total = voff;
  // levels by height
  int32_t hmax = 0;
  for (int32_t s = 0; s < nn; ++s) hmax = std::max(hmax, P.height[s]);
  P.level_ptr.assign(hmax + 2, 0);
  for (int32_t s = 0; s < nn; ++s) P.level_ptr[P.height[s] + 1]++;
  for (int32_t h = 0; h <= hmax; ++h) P.level_ptr[h + 1] += P.level_ptr[h];
  P.level_nodes.resize(nn);
  std::vector<int32_t> fill(P.level_ptr.begin(), P.level_ptr.end() - 1);
  for (int32_t s = 0; s < nn; ++s) P.level_nodes[fill[P.height[s]]++] = s;
  if (nn == 0) P.level_ptr.assign(1, 0);
  return PF_OK;
}

template <class T>
int64_t copy_out(const std::vector<T> &v, void *dst) {
  if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(T));
  return (int64_t)v.size();
}

}  // namespace

extern "C" {

int pf_nd_plan_build(int64_t n, const double *xy_host, const int64_t *nb_ptr_host,
                     const int64_t *nb_idx_host, const uint8_t *is_boundary_host, int leaf,
                     int tile, void **plan_out) {
  if (!plan_out || n < 0 || (n > 0 && (!xy_host || !nb_ptr_host || !nb_idx_host ||
                                       !is_boundary_host)) || leaf < 1 || tile < 1) {
    pf::set_error("pf_nd_plan_build: bad argument");
    return PF_E_ARG;
  }
  if (n >= (int64_t)1 << 31) {
    pf::set_error("pf_nd_plan_build: n >= 2^31 not supported");
    return PF_E_DOMAIN;
  }
  *plan_out = nullptr;
  Plan *P = new (std::nothrow) Plan();
  if (!P) {
    pf::set_error("pf_nd_plan_build: out of host memory");
    return PF_E_CAPACITY;
  }
  P->n = n;
  P->leaf = leaf;
  P->ta = tile;
  int rc;
  try {
    rc = build_plan(*P, xy_host, nb_ptr_host, nb_idx_host, is_boundary_host);
  } catch (const std::bad_alloc &) {
    pf::set_error("pf_nd_plan_build: out of host memory");
    rc = PF_E_CAPACITY;
  }
  if (rc != PF_OK) {
    delete P;
    return rc;
  }
  *plan_out = P;
  return PF_OK;
}

void pf_nd_plan_free(void *plan) { delete static_cast<Plan *>(plan); }

int64_t pf_nd_plan_array(void *plan, const char *name, void *dst_host) {
  if (!plan || !name) return -1;
  Plan &P = *static_cast<Plan *>(plan);
  const std::string s(name);
#define PF_ARR(field) \
  if (s == #field) return copy_out(P.field, dst_host);
  PF_ARR(perm_orig) PF_ARR(iperm) PF_ARR(c0) PF_ARR(cn) PF_ARR(rn) PF_ARR(fn)
  PF_ARR(parent) PF_ARR(height) PF_ARR(foff) PF_ARR(ch_ptr) PF_ARR(ch_idx) PF_ARR(r_ptr)
  PF_ARR(r_pos) PF_ARR(r_orig) PF_ARR(relmap_off) PF_ARR(relmap) PF_ARR(a_ptr) PF_ARR(a_dst)
  PF_ARR(a_src) PF_ARR(b_ptr) PF_ARR(b_row) PF_ARR(b_col) PF_ARR(b_src) PF_ARR(act_ptr)
  PF_ARR(act_tile) PF_ARR(act_voff) PF_ARR(tile_item) PF_ARR(level_ptr) PF_ARR(level_nodes)
#undef PF_ARR
  pf::set_error("pf_nd_plan_array: unknown array '%s'", name);
  return -1;
}

// Sorted vertex-neighbour CSR of a triangle mesh (mesh.py:151 `neighbors`):
// counting sort of the 6 directed edge entries per triangle by source vertex,
// then a per-vertex sort + unique.  nb_idx_host needs capacity 6 * nt; the
// number of entries is returned in *nnz_out.
int pf_vertex_neighbors(int64_t n, int64_t nt, const int64_t *tri_host, int64_t *nb_ptr_host,
                        int64_t *nb_idx_host, int64_t *nnz_out) {
  if (n < 0 || nt < 0 || (nt && !tri_host) || !nb_ptr_host || (nt && !nb_idx_host) ||
      !nnz_out) {
    pf::set_error("pf_vertex_neighbors: bad argument");
    return PF_E_ARG;
  }
  try {
    std::vector<int64_t> cnt(n + 1, 0);
    for (int64_t t = 0; t < 3 * nt; ++t) {
      const int64_t v = tri_host[t];
      if (v < 0 || v >= n) {
        pf::set_error("pf_vertex_neighbors: vertex index out of range");
        return PF_E_DOMAIN;
      }
      cnt[v + 1] += 2;
    }
    for (int64_t v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
    std::vector<int64_t> cand(cnt[n]);
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int64_t t = 0; t < nt; ++t) {
      const int64_t *T = tri_host + 3 * t;
      for (int a = 0; a < 3; ++a) {
        const int64_t v = T[a];
        cand[fill[v]++] = T[(a + 1) % 3];
        cand[fill[v]++] = T[(a + 2) % 3];
      }
    }
    int64_t out = 0;
    nb_ptr_host[0] = 0;
    for (int64_t v = 0; v < n; ++v) {
      auto b = cand.begin() + cnt[v], e = cand.begin() + cnt[v + 1];
      std::sort(b, e);
      e = std::unique(b, e);
      for (auto it = b; it != e; ++it) nb_idx_host[out++] = *it;
      nb_ptr_host[v + 1] = out;
    }
    *nnz_out = out;
  } catch (const std::bad_alloc &) {
    pf::set_error("pf_vertex_neighbors: out of host memory");
    return PF_E_CAPACITY;
  }
  return PF_OK;
}

int pf_nd_plan_stats(void *plan, double *out_host) {
  if (!plan || !out_host) {
    pf::set_error("pf_nd_plan_stats: bad argument");
    return PF_E_ARG;
  }
  const Plan &P = *static_cast<const Plan *>(plan);
  const double v[] = {(double)P.n, (double)P.m, (double)P.k, (double)P.c0.size(),
                      (double)(P.level_ptr.size() - 1), (double)P.f_total, (double)P.v_total,
                      (double)P.nnz_l, P.flops_factor, P.flops_solve, (double)P.max_f,
                      (double)P.max_c, (double)P.max_r, (double)P.ntiles, (double)P.ta,
                      (double)P.leaf};
  std::memcpy(out_host, v, sizeof(v));
  return PF_OK;
}

}  // extern "C"
