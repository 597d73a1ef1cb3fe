// builder.cpp — host instance builder (include/hmxb.h): seeded points -> cluster tree ->
// interactions (HSS / tau / budget) -> neighbour sampling -> nested interpolative
// decomposition -> blocking + coarsening -> computation-ordered CDS.
//
// This is the producer of the evaluator's input, written for this repo (multi-threaded,
// tree-order point storage); it follows the structure of the reference inspector
// (proj/src/{points,tree,interaction,sampling,compress,structure}.cpp) and adds the
// BASELINE features the reference lacks. Results are pinned at the evaluate
// boundary, not here: the oracle evaluates the same CDS this code produces.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hmxb.h"

namespace hmxb {
namespace {

using u32 = std::uint32_t;
using u64 = std::uint64_t;
using u8 = std::uint8_t;
constexpr u32 kNone = HMXG_NO_NODE;

thread_local std::string g_err;

// ---------------------------------------------------------------- randomness
// splitmix64 and xoshiro256** (Vigna), seeded by chaining splitmix64 over the seed.
inline u64 splitmix64(u64 x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

class Xoshiro {
 public:
  explicit Xoshiro(u64 seed) {
    u64 x = seed;
    for (auto& w : s_) w = x = splitmix64(x);
  }
  u64 next() {
    const u64 out = rotl(s_[1] * 5, 7) * 9;
    const u64 t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return out;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  u64 below(u64 bound) { return next() % bound; }
  double normal() {  // Box-Muller
    double u1 = uniform();
    while (u1 == 0.0) u1 = uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586477 * u2);
  }

 private:
  static u64 rotl(u64 x, int k) { return (x << k) | (x >> (64 - k)); }
  u64 s_[4];
};

// ---------------------------------------------------------------- threading
// Dynamic index claiming; every index runs exactly once and the call returns after all
// workers joined (no state survives the call, unlike a persistent pool).
template <class Fn>
void parallel_for(u64 count, unsigned threads, Fn&& fn) {
  if (count == 0) return;
  const unsigned t = static_cast<unsigned>(std::min<u64>(threads, count));
  if (t <= 1) {
    for (u64 i = 0; i < count; ++i) fn(i);
    return;
  }
  std::atomic<u64> next{0};
  auto body = [&] {
    for (u64 i = next.fetch_add(1); i < count; i = next.fetch_add(1)) fn(i);
  };
  std::vector<std::thread> pool;
  pool.reserve(t - 1);
  for (unsigned k = 1; k < t; ++k) pool.emplace_back(body);
  body();
  for (auto& th : pool) th.join();
}

double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---------------------------------------------------------------- kernel
struct KernelFn {
  int kind;
  double h;
  double den2h2, invh;  // 2 h h formed as (2 h) h, kernel.cpp:42
  KernelFn(int k, double hh) : kind(k), h(hh), den2h2(2.0 * hh * hh), invh(1.0 / hh) {}
  double operator()(const double* x, const double* y, u32 d) const {
    double s = 0.0;
    for (u32 k = 0; k < d; ++k) {
      const double t = x[k] - y[k];
      s += t * t;
    }
    switch (kind) {
      case HMXB_K_GAUSSIAN:
        return std::exp(-s / den2h2);
      case HMXB_K_EXPONENTIAL:
        return std::exp(-std::sqrt(s) * invh);
      default:
        return s == 0.0 ? 1.0 : 1.0 / std::sqrt(s);
    }
  }
};

}  // namespace

struct Instance {
  hmxb_spec spec{};
  u32 d = 0;
  u64 n = 0;
  std::vector<double> pts;   // original order, point major
  std::vector<double> tpts;  // tree order (perm applied), point major
  // cluster tree
  u32 num_nodes = 0;
  u32 height = 0;
  std::vector<u32> parent, lchild, rchild, start, end, level, perm;
  // interactions
  std::vector<std::vector<u32>> near, far;
  std::vector<u8> part;
  // compression
  std::vector<u32> srank;
  std::vector<std::vector<u32>> skel;  // tree positions
  std::vector<std::vector<double>> basis;
  // CDS
  std::vector<u32> near_flat, far_flat, v_order;
  std::vector<u64> dptr, bptr, vptr;
  std::vector<double> dgen, bgen, vgen;
  hmxb_build_stats stats{};

  bool leaf(u32 i) const { return lchild[i] == kNone; }
  u32 size(u32 i) const { return end[i] - start[i]; }
  const double* tp(u32 pos) const { return tpts.data() + static_cast<u64>(pos) * d; }
};

namespace {

// ---------------------------------------------------------------- points
void make_points(Instance& in) {
  const hmxb_spec& s = in.spec;
  in.n = s.n;
  in.d = s.points == HMXB_PTS_GRID2D ? 2 : s.d;
  const u32 d = in.d;
  in.pts.assign(in.n * d, 0.0);
  Xoshiro rng(s.seed);
  switch (s.points) {
    case HMXB_PTS_GRID2D: {
      u64 side = 1;
      while (side * side < in.n) ++side;
      for (u64 i = 0; i < in.n; ++i) {
        in.pts[2 * i] = static_cast<double>(i % side);
        in.pts[2 * i + 1] = static_cast<double>(i / side);
      }
      break;
    }
    case HMXB_PTS_MIXTURE: {
      const u32 comps = s.components ? s.components : 8;
      std::vector<double> centre(static_cast<u64>(comps) * d);
      for (auto& c : centre) c = -5.0 + 10.0 * rng.uniform();
      for (u64 i = 0; i < in.n; ++i) {
        const u64 c = rng.below(comps);
        for (u32 k = 0; k < d; ++k) in.pts[i * d + k] = centre[c * d + k] + rng.normal();
      }
      break;
    }
    case HMXB_PTS_NORMAL: {
      for (auto& x : in.pts) x = rng.normal();
      for (u32 k = 0; k < d; ++k) {
        double mean = 0.0, var = 0.0;
        for (u64 i = 0; i < in.n; ++i) mean += in.pts[i * d + k];
        mean /= static_cast<double>(in.n);
        for (u64 i = 0; i < in.n; ++i) {
          const double t = in.pts[i * d + k] - mean;
          var += t * t;
        }
        const double sd = std::sqrt(var / static_cast<double>(in.n));
        for (u64 i = 0; i < in.n; ++i)
          in.pts[i * d + k] = sd > 0.0 ? (in.pts[i * d + k] - mean) / sd : 0.0;
      }
      break;
    }
    case HMXB_PTS_QUANTIZED: {
      const u32 lv = s.levels > 1 ? s.levels : 16;
      for (auto& x : in.pts) {
        const double q = std::floor(rng.uniform() * lv);
        x = std::min(q, static_cast<double>(lv - 1)) / static_cast<double>(lv - 1);
      }
      break;
    }
    default:
      for (auto& x : in.pts) x = rng.uniform();
  }
}

// ---------------------------------------------------------------- cluster tree
u64 kd_split(const Instance& in, u32* idx, u64 len) {
  const u32 d = in.d;
  u32 best = 0;
  double spread = -1.0;
  for (u32 k = 0; k < d; ++k) {
    double lo = in.pts[static_cast<u64>(idx[0]) * d + k], hi = lo;
    for (u64 a = 0; a < len; ++a) {
      const double c = in.pts[static_cast<u64>(idx[a]) * d + k];
      lo = std::min(lo, c);
      hi = std::max(hi, c);
    }
    if (hi - lo > spread) {
      spread = hi - lo;
      best = k;
    }
  }
  const u64 left = (len + 1) / 2;
  std::nth_element(idx, idx + left, idx + len, [&](u32 a, u32 b) {
    const double ka = in.pts[static_cast<u64>(a) * d + best], kb = in.pts[static_cast<u64>(b) * d + best];
    return ka < kb || (ka == kb && a < b);
  });
  return left;
}

u64 two_means_split(const Instance& in, u32* idx, u64 len, u64 seed) {
  const u32 d = in.d;
  auto pt = [&](u32 p) { return in.pts.data() + static_cast<u64>(p) * d; };
  auto dist2 = [&](const double* a, const double* b) {
    double s = 0.0;
    for (u32 k = 0; k < d; ++k) {
      const double t = a[k] - b[k];
      s += t * t;
    }
    return s;
  };
  Xoshiro rng(seed);
  std::vector<double> c0(pt(idx[0]), pt(idx[0]) + d), c1(pt(idx[len - 1]), pt(idx[len - 1]) + d);
  double best = dist2(c0.data(), c1.data());
  for (int t = 0; t < 48; ++t) {
    const u32 a = idx[rng.below(len)], b = idx[rng.below(len)];
    const double dd = dist2(pt(a), pt(b));
    if (dd > best) {
      best = dd;
      c0.assign(pt(a), pt(a) + d);
      c1.assign(pt(b), pt(b) + d);
    }
  }
  std::vector<u8> side(len, 0);
  u64 n0 = 0, n1 = 0;
  for (int iter = 0; iter < 16; ++iter) {
    bool changed = false;
    n0 = n1 = 0;
    for (u64 a = 0; a < len; ++a) {
      const u8 s = dist2(pt(idx[a]), c1.data()) < dist2(pt(idx[a]), c0.data()) ? 1 : 0;
      changed |= s != side[a];
      side[a] = s;
      (s ? n1 : n0)++;
    }
    if (n0 == 0 || n1 == 0) break;
    std::fill(c0.begin(), c0.end(), 0.0);
    std::fill(c1.begin(), c1.end(), 0.0);
    for (u64 a = 0; a < len; ++a) {
      double* c = side[a] ? c1.data() : c0.data();
      const double* p = pt(idx[a]);
      for (u32 k = 0; k < d; ++k) c[k] += p[k];
    }
    for (u32 k = 0; k < d; ++k) {
      c0[k] /= static_cast<double>(n0);
      c1[k] /= static_cast<double>(n1);
    }
    if (!changed && iter > 0) break;
  }
  const u64 small = std::min(n0, n1);
  if (small == 0 || small * 10 < len) {
    // degenerate or > 90/10: median split along the centroid direction
    std::vector<double> dir(d);
    double nrm = 0.0;
    for (u32 k = 0; k < d; ++k) {
      dir[k] = c1[k] - c0[k];
      nrm += dir[k] * dir[k];
    }
    const u64 left = (len + 1) / 2;
    if (nrm == 0.0) {
      std::sort(idx, idx + len);
      return left;
    }
    std::vector<std::pair<double, u32>> key(len);
    for (u64 a = 0; a < len; ++a) {
      double pr = 0.0;
      const double* p = pt(idx[a]);
      for (u32 k = 0; k < d; ++k) pr += p[k] * dir[k];
      key[a] = {pr, idx[a]};
    }
    std::nth_element(key.begin(), key.begin() + left, key.end());
    for (u64 a = 0; a < len; ++a) idx[a] = key[a].second;
    return left;
  }
  std::vector<u32> tmp(idx, idx + len);
  u64 l = 0, r = n0;
  for (u64 a = 0; a < len; ++a) (side[a] ? idx[r++] : idx[l++]) = tmp[a];
  return n0;
}

void build_tree(Instance& in) {
  const hmxb_spec& s = in.spec;
  const u32 m = std::max<u32>(1, s.leaf);
  int split = s.split;
  if (split == HMXB_SPLIT_AUTO) split = in.d <= 3 ? HMXB_SPLIT_KD : HMXB_SPLIT_TWOMEANS;
  in.perm.resize(in.n);
  std::iota(in.perm.begin(), in.perm.end(), 0u);
  auto add = [&](u32 par, u32 b, u32 e, u32 lvl) {
    const u32 id = in.num_nodes++;
    in.parent.push_back(par);
    in.lchild.push_back(kNone);
    in.rchild.push_back(kNone);
    in.start.push_back(b);
    in.end.push_back(e);
    in.level.push_back(lvl);
    in.height = std::max(in.height, lvl);
    return id;
  };
  add(kNone, 0, static_cast<u32>(in.n), 0);
  // BFS ids (children consecutive, larger than the parent). Splits of one BFS level are
  // independent and run in parallel; ids are assigned afterwards in order.
  std::vector<u32> frontier{0};
  const unsigned threads = s.threads;
  while (!frontier.empty()) {
    std::vector<u64> mid(frontier.size(), 0);
    parallel_for(frontier.size(), threads, [&](u64 f) {
      const u32 node = frontier[f];
      const u32 b = in.start[node], e = in.end[node];
      if (e - b <= m) return;
      u32* idx = in.perm.data() + b;
      mid[f] = b + (split == HMXB_SPLIT_KD ? kd_split(in, idx, e - b)
                                           : two_means_split(in, idx, e - b, splitmix64(s.seed ^ splitmix64(node + 1))));
    });
    std::vector<u32> next;
    for (std::size_t f = 0; f < frontier.size(); ++f) {
      const u32 node = frontier[f];
      if (in.end[node] - in.start[node] <= m) continue;
      const u32 md = static_cast<u32>(mid[f]);
      const u32 l = add(node, in.start[node], md, in.level[node] + 1);
      const u32 r = add(node, md, in.end[node], in.level[node] + 1);
      in.lchild[node] = l;
      in.rchild[node] = r;
      next.push_back(l);
      next.push_back(r);
    }
    frontier.swap(next);
  }
  in.tpts.resize(in.n * in.d);
  for (u64 pos = 0; pos < in.n; ++pos)
    std::memcpy(in.tpts.data() + pos * in.d, in.pts.data() + static_cast<u64>(in.perm[pos]) * in.d,
                in.d * sizeof(double));
}

// ---------------------------------------------------------------- geometry helpers
struct Geometry {
  std::vector<double> centroid;  // num_nodes x d
  std::vector<double> radius;
};

Geometry geometry(const Instance& in) {
  Geometry g;
  const u32 d = in.d;
  g.centroid.assign(static_cast<u64>(in.num_nodes) * d, 0.0);
  g.radius.assign(in.num_nodes, 0.0);
  parallel_for(in.num_nodes, in.spec.threads, [&](u64 i) {
    double* c = g.centroid.data() + i * d;
    for (u32 p = in.start[i]; p < in.end[i]; ++p)
      for (u32 k = 0; k < d; ++k) c[k] += in.tp(p)[k];
    for (u32 k = 0; k < d; ++k) c[k] /= static_cast<double>(in.size(static_cast<u32>(i)));
    double r2 = 0.0;
    for (u32 p = in.start[i]; p < in.end[i]; ++p) {
      double s = 0.0;
      for (u32 k = 0; k < d; ++k) {
        const double t = in.tp(p)[k] - c[k];
        s += t * t;
      }
      r2 = std::max(r2, s);
    }
    g.radius[i] = std::sqrt(r2);
  });
  return g;
}

double centroid_dist2(const Geometry& g, u32 d, u32 a, u32 b) {
  double s = 0.0;
  for (u32 k = 0; k < d; ++k) {
    const double t = g.centroid[static_cast<u64>(a) * d + k] - g.centroid[static_cast<u64>(b) * d + k];
    s += t * t;
  }
  return s;
}

// ---------------------------------------------------------------- k-NN (tree positions)
// Exact k nearest neighbours of every point among the points of the `cand` leaves nearest
// (by centroid) to its own leaf. nbr is n x k in tree positions, self excluded.
std::vector<u32> knn(const Instance& in, const Geometry& g, const std::vector<u32>& leaves, u32 k,
                     u32 cand) {
  const u32 d = in.d;
  const u32 L = static_cast<u32>(leaves.size());
  cand = std::min(cand, L);
  k = static_cast<u32>(std::min<u64>(k, in.n - 1));
  std::vector<u32> nbr(in.n * static_cast<u64>(k), 0);
  if (k == 0) return nbr;
  parallel_for(L, in.spec.threads, [&](u64 li) {
    const u32 leaf = leaves[li];
    std::vector<std::pair<double, u32>> cl(L);
    for (u32 t = 0; t < L; ++t) cl[t] = {centroid_dist2(g, d, leaf, leaves[t]), leaves[t]};
    std::partial_sort(cl.begin(), cl.begin() + cand, cl.end());
    std::vector<u32> pool;
    for (u32 t = 0; t < cand; ++t)
      for (u32 p = in.start[cl[t].second]; p < in.end[cl[t].second]; ++p) pool.push_back(p);
    // top up from other leaves in centroid order until k candidates besides self exist
    for (u32 t = cand; t < L && pool.size() < k + 1; ++t)
      for (u32 p = in.start[cl[t].second]; p < in.end[cl[t].second]; ++p) pool.push_back(p);
    std::vector<std::pair<double, u32>> sc;
    sc.reserve(pool.size());
    for (u32 p = in.start[leaf]; p < in.end[leaf]; ++p) {
      sc.clear();
      const double* x = in.tp(p);
      for (u32 q : pool) {
        if (q == p) continue;
        const double* y = in.tp(q);
        double s = 0.0;
        for (u32 kk = 0; kk < d; ++kk) {
          const double t = x[kk] - y[kk];
          s += t * t;
        }
        sc.emplace_back(s, q);
      }
      const u64 take = std::min<u64>(k, sc.size());
      std::partial_sort(sc.begin(), sc.begin() + take, sc.end());
      for (u64 t = 0; t < take; ++t) nbr[static_cast<u64>(p) * k + t] = sc[t].second;
      for (u64 t = take; t < k; ++t) nbr[static_cast<u64>(p) * k + t] = sc.empty() ? p : sc[0].second;
    }
  });
  return nbr;
}

// ---------------------------------------------------------------- interactions
void interactions_hss(Instance& in) {
  for (u32 i = 0; i < in.num_nodes; ++i) {
    if (in.leaf(i)) {
      in.near[i].push_back(i);
    } else {
      in.far[in.lchild[i]].push_back(in.rchild[i]);
      in.far[in.rchild[i]].push_back(in.lchild[i]);
    }
  }
}

// Geometric admissibility tau*dist(ci,cj) > 2(ri+rj), dual traversal from (root, root)
// splitting the larger-radius node (proj/src/interaction.cpp:49-111).
void interactions_tau(Instance& in, const Geometry& g) {
  const double tau = in.spec.tau;
  std::vector<std::pair<u32, u32>> stack{{0, 0}};
  while (!stack.empty()) {
    auto [i, j] = stack.back();
    stack.pop_back();
    if (i == j) {
      if (in.leaf(i)) {
        in.near[i].push_back(i);
      } else {
        const u32 l = in.lchild[i], r = in.rchild[i];
        stack.push_back({r, r});
        stack.push_back({r, l});
        stack.push_back({l, r});
        stack.push_back({l, l});
      }
      continue;
    }
    if (tau * std::sqrt(centroid_dist2(g, in.d, i, j)) > 2.0 * (g.radius[i] + g.radius[j])) {
      in.far[i].push_back(j);
      continue;
    }
    const bool li = in.leaf(i), lj = in.leaf(j);
    if (li && lj) {
      in.near[i].push_back(j);
      continue;
    }
    bool split_i;
    if (li) split_i = false;
    else if (lj) split_i = true;
    else if (g.radius[i] != g.radius[j]) split_i = g.radius[i] > g.radius[j];
    else if (in.size(i) != in.size(j)) split_i = in.size(i) > in.size(j);
    else split_i = i < j;
    if (split_i) {
      stack.push_back({in.rchild[i], j});
      stack.push_back({in.lchild[i], j});
    } else {
      stack.push_back({i, in.rchild[j]});
      stack.push_back({i, in.lchild[j]});
    }
  }
}

// Budget ("H2-b", GOFMM-style) admissibility: each leaf keeps itself plus its top
// ceil(budget * L) - 1 leaves by k-NN neighbour votes (ties: nearer centroid, lower id) as
// near blocks; the relation is symmetrized. Far pairs come from a dual traversal from
// (root, root): (a, b) is admissible iff no near leaf pair lies under a x b.
void interactions_budget(Instance& in, const Geometry& g, const std::vector<u32>& leaves,
                         const std::vector<u32>& nbr, u32 k) {
  const u32 L = static_cast<u32>(leaves.size());
  std::vector<u32> leaf_of_pos(in.n);
  std::vector<u32> leaf_index(in.num_nodes, kNone);
  for (u32 t = 0; t < L; ++t) {
    leaf_index[leaves[t]] = t;
    for (u32 p = in.start[leaves[t]]; p < in.end[leaves[t]]; ++p) leaf_of_pos[p] = t;
  }
  const u32 per_leaf = std::max<u32>(1, static_cast<u32>(std::ceil(in.spec.budget * L)));
  std::vector<std::vector<u32>> nl(L);
  parallel_for(L, in.spec.threads, [&](u64 t) {
    const u32 leaf = leaves[t];
    std::vector<u32> votes(L, 0);
    for (u32 p = in.start[leaf]; p < in.end[leaf]; ++p)
      for (u32 a = 0; a < k; ++a) ++votes[leaf_of_pos[nbr[static_cast<u64>(p) * k + a]]];
    std::vector<std::tuple<long long, double, u32>> rank;
    rank.reserve(L);
    for (u32 o = 0; o < L; ++o)
      if (o != t) rank.emplace_back(-static_cast<long long>(votes[o]), centroid_dist2(g, in.d, leaf, leaves[o]), o);
    const u32 take = std::min<u32>(per_leaf - 1, static_cast<u32>(rank.size()));
    std::partial_sort(rank.begin(), rank.begin() + take, rank.end());
    nl[t].push_back(static_cast<u32>(t));
    for (u32 a = 0; a < take; ++a) nl[t].push_back(std::get<2>(rank[a]));
  });
  std::vector<std::vector<u32>> sym(L);
  for (u32 t = 0; t < L; ++t)
    for (u32 o : nl[t]) {
      sym[t].push_back(o);
      sym[o].push_back(t);
    }
  // DFS leaf order so that every subtree owns a contiguous leaf range
  std::vector<u32> dfs_rank(L), lo(in.num_nodes), hi(in.num_nodes);
  {
    u32 counter = 0;
    std::vector<std::pair<u32, bool>> st{{0, false}};
    while (!st.empty()) {
      auto [i, done] = st.back();
      st.pop_back();
      if (in.leaf(i)) {
        lo[i] = counter;
        dfs_rank[leaf_index[i]] = counter++;
        hi[i] = counter;
        continue;
      }
      if (done) {
        lo[i] = lo[in.lchild[i]];
        hi[i] = hi[in.rchild[i]];
        continue;
      }
      st.push_back({i, true});
      st.push_back({in.rchild[i], false});
      st.push_back({in.lchild[i], false});
    }
  }
  for (u32 t = 0; t < L; ++t) {
    auto& v = sym[t];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  // near_under[a] = sorted DFS ranks of leaves near to some leaf under a
  std::vector<std::vector<u32>> under(in.num_nodes);
  for (u32 i = in.num_nodes; i-- > 0;) {
    auto& u = under[i];
    if (in.leaf(i)) {
      for (u32 o : sym[leaf_index[i]]) u.push_back(dfs_rank[o]);
      std::sort(u.begin(), u.end());
    } else {
      const auto& a = under[in.lchild[i]];
      const auto& b = under[in.rchild[i]];
      std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(u));
    }
  }
  auto admissible = [&](u32 a, u32 b) {
    const auto& u = under[a];
    const auto it = std::lower_bound(u.begin(), u.end(), lo[b]);
    return it == u.end() || *it >= hi[b];
  };
  std::vector<std::pair<u32, u32>> stack{{0, 0}};
  while (!stack.empty()) {
    auto [i, j] = stack.back();
    stack.pop_back();
    if (i == j) {
      if (in.leaf(i)) {
        in.near[i].push_back(i);
      } else {
        const u32 l = in.lchild[i], r = in.rchild[i];
        stack.push_back({r, r});
        stack.push_back({r, l});
        stack.push_back({l, r});
        stack.push_back({l, l});
      }
      continue;
    }
    if (admissible(i, j)) {
      in.far[i].push_back(j);
      continue;
    }
    const bool li = in.leaf(i), lj = in.leaf(j);
    if (li && lj) {
      in.near[i].push_back(j);
      continue;
    }
    bool split_i;
    if (li) split_i = false;
    else if (lj) split_i = true;
    else if (in.size(i) != in.size(j)) split_i = in.size(i) > in.size(j);
    else split_i = i < j;
    if (split_i) {
      stack.push_back({in.rchild[i], j});
      stack.push_back({in.lchild[i], j});
    } else {
      stack.push_back({i, in.rchild[j]});
      stack.push_back({i, in.lchild[j]});
    }
  }
}

// ---------------------------------------------------------------- sampling
// Sample rows of node i (tree positions, outside node i): its members' k-NN hits outside
// the node by descending multiplicity (ties: lower position), topped up uniformly.
std::vector<u32> sample_rows(const Instance& in, u32 i, const std::vector<u32>& nbr, u32 k,
                             u32 budget) {
  const u32 b = in.start[i], e = in.end[i];
  const u64 outside = in.n - (e - b);
  if (budget == std::numeric_limits<u32>::max()) {  // exact: every non-member row
    std::vector<u32> rows;
    rows.reserve(outside);
    for (u32 p = 0; p < in.n; ++p)
      if (p < b || p >= e) rows.push_back(p);
    return rows;
  }
  const u64 target = std::min<u64>(budget, outside);
  std::vector<u32> hits;
  hits.reserve(static_cast<u64>(e - b) * k);
  for (u32 p = b; p < e; ++p)
    for (u32 a = 0; a < k; ++a) {
      const u32 q = nbr[static_cast<u64>(p) * k + a];
      if (q < b || q >= e) hits.push_back(q);
    }
  std::sort(hits.begin(), hits.end());
  std::vector<std::pair<u32, u32>> w;  // (-count, pos) encoded
  for (std::size_t a = 0; a < hits.size();) {
    std::size_t c = a;
    while (c < hits.size() && hits[c] == hits[a]) ++c;
    w.emplace_back(static_cast<u32>(c - a), hits[a]);
    a = c;
  }
  std::sort(w.begin(), w.end(), [](auto x, auto y) { return x.first > y.first || (x.first == y.first && x.second < y.second); });
  std::vector<u32> rows;
  rows.reserve(target);
  for (std::size_t a = 0; a < w.size() && rows.size() < target; ++a) rows.push_back(w[a].second);
  if (rows.size() < target) {
    std::vector<u8> taken(in.n, 0);
    for (u32 r : rows) taken[r] = 1;
    Xoshiro rng(splitmix64(in.spec.seed ^ splitmix64(0xba5eULL + i)));
    u64 attempts = 16 * target + 64;
    while (rows.size() < target && attempts-- > 0) {
      const u32 p = static_cast<u32>(rng.below(in.n));
      if ((p >= b && p < e) || taken[p]) continue;
      taken[p] = 1;
      rows.push_back(p);
    }
    for (u32 p = 0; rows.size() < target && p < in.n; ++p)
      if ((p < b || p >= e) && !taken[p]) {
        taken[p] = 1;
        rows.push_back(p);
      }
  }
  return rows;
}

// ---------------------------------------------------------------- interpolative decomposition
// Column-pivoted Householder QR of M (r x c, column major, destroyed) with exact trailing
// column norms; stops once the trailing residual's Frobenius norm is <= tol * |M|_F or at
// `cap` columns. Returns the rank k, the pivot order and V (c x k, column major) with
// M ~ M[:, piv[0:k]] V^T (identity rows at the skeleton columns).
u32 interpolative(std::vector<double>& a, u64 r, u64 c, double tol, u64 cap,
                  std::vector<u32>& piv, std::vector<double>& v) {
  cap = std::min({cap, r, c});
  piv.resize(c);
  std::iota(piv.begin(), piv.end(), 0u);
  double total = 0.0;
  for (double x : a) total += x * x;
  const double tl = std::max(tol, 1e-14);
  const double stop = tl * tl * total;
  std::vector<double> nrm(c), hv(r);
  u64 k = 0;
  for (; k < cap; ++k) {
    double rest = 0.0, best = -1.0;
    u64 pv = k;
    for (u64 j = k; j < c; ++j) {
      const double* col = a.data() + j * r;
      double s = 0.0;
      for (u64 i = k; i < r; ++i) s += col[i] * col[i];
      nrm[j] = s;
      rest += s;
      if (s > best) {
        best = s;
        pv = j;
      }
    }
    if (rest <= stop || best <= 0.0) break;
    if (pv != k) {
      std::swap_ranges(a.data() + k * r, a.data() + (k + 1) * r, a.data() + pv * r);
      std::swap(piv[k], piv[pv]);
    }
    double* ck = a.data() + k * r;
    double alpha = std::sqrt(nrm[pv]);
    if (ck[k] > 0) alpha = -alpha;
    const u64 len = r - k;
    hv[0] = ck[k] - alpha;
    for (u64 i = 1; i < len; ++i) hv[i] = ck[k + i];
    double h2 = 0.0;
    for (u64 i = 0; i < len; ++i) h2 += hv[i] * hv[i];
    ck[k] = alpha;
    for (u64 i = k + 1; i < r; ++i) ck[i] = 0.0;
    if (h2 > 0.0) {
      for (u64 j = k + 1; j < c; ++j) {
        double* cj = a.data() + j * r + k;
        double dot = 0.0;
        for (u64 i = 0; i < len; ++i) dot += hv[i] * cj[i];
        // 2 dot / h2 as the reference forms it (compress.cpp:71): with a subnormal h2 (a block
        // of underflowing kernel values) a precomputed 2 / h2 is inf, and 0 * inf a NaN in V
        const double f = 2.0 * dot / h2;
        for (u64 i = 0; i < len; ++i) cj[i] -= f * hv[i];
      }
    }
  }
  v.assign(c * k, 0.0);
  for (u64 j = 0; j < k; ++j) v[piv[j] + j * c] = 1.0;
  std::vector<double> x(k);
  for (u64 t = k; t < c; ++t) {  // R11 x = R12(:, t)
    for (u64 i = k; i-- > 0;) {
      double s = a[t * r + i];
      for (u64 j = i + 1; j < k; ++j) s -= a[j * r + i] * x[j];
      x[i] = s / a[i * r + i];
    }
    for (u64 j = 0; j < k; ++j) v[piv[t] + j * c] = x[j];
  }
  return static_cast<u32>(k);
}

void compress(Instance& in, const std::vector<u32>& nbr, u32 k) {
  const hmxb_spec& s = in.spec;
  const KernelFn K(s.kernel, s.h);
  const u32 sample = s.sample_rows == 0 ? 2 * s.max_rank : s.sample_rows;
  in.srank.assign(in.num_nodes, 0);
  in.skel.assign(in.num_nodes, {});
  in.basis.assign(in.num_nodes, {});
  std::vector<std::vector<u32>> by_level(in.height + 1);
  for (u32 i = 0; i < in.num_nodes; ++i)
    if (in.part[i]) by_level[in.level[i]].push_back(i);
  for (u32 lv = in.height + 1; lv-- > 0;) {
    const auto& nodes = by_level[lv];
    parallel_for(nodes.size(), s.threads, [&](u64 t) {
      const u32 i = nodes[t];
      std::vector<u32> cols;
      if (in.leaf(i)) {
        for (u32 p = in.start[i]; p < in.end[i]; ++p) cols.push_back(p);
      } else {
        const auto& l = in.skel[in.lchild[i]];
        const auto& r = in.skel[in.rchild[i]];
        cols.insert(cols.end(), l.begin(), l.end());
        cols.insert(cols.end(), r.begin(), r.end());
      }
      if (cols.empty()) return;
      const std::vector<u32> rows = sample_rows(in, i, nbr, k, sample);
      if (rows.empty()) throw std::runtime_error("builder: participating node without sample rows");
      std::vector<double> m(rows.size() * cols.size());
      for (u64 c = 0; c < cols.size(); ++c)
        for (u64 r = 0; r < rows.size(); ++r) m[c * rows.size() + r] = K(in.tp(rows[r]), in.tp(cols[c]), in.d);
      std::vector<u32> piv;
      const u32 sr = interpolative(m, rows.size(), cols.size(), s.tol, s.max_rank, piv, in.basis[i]);
      in.srank[i] = sr;
      for (u32 j = 0; j < sr; ++j) in.skel[i].push_back(cols[piv[j]]);
    });
  }
}

// ---------------------------------------------------------------- blocking / coarsening
// Storage order of a pair relation: row groups (i-1)/bs ascending, then column cells
// (j-1)/bs ascending, then i, then j (MatRox Alg. 1; proj/src/structure.cpp:29-61).
std::vector<u32> blocked_order(const Instance& in, const std::vector<std::vector<u32>>& lists, u32 bs) {
  bs = std::max<u32>(1, bs);
  struct P {
    u32 ig, jg, i, j;
  };
  std::vector<P> ps;
  for (u32 i = 0; i < in.num_nodes; ++i)
    for (u32 j : lists[i]) {
      if (i == 0 || j == 0) throw std::runtime_error("builder: root node appears in an interaction");
      ps.push_back({(i - 1) / bs, (j - 1) / bs, i, j});
    }
  std::sort(ps.begin(), ps.end(), [](const P& a, const P& b) {
    return std::tie(a.ig, a.jg, a.i, a.j) < std::tie(b.ig, b.jg, b.i, b.j);
  });
  std::vector<u32> flat;
  flat.reserve(2 * ps.size());
  for (const P& p : ps) {
    flat.push_back(p.i);
    flat.push_back(p.j);
  }
  return flat;
}

// V storage order (MatRox Alg. 2; proj/src/structure.cpp:63-186): height bands of `agg`
// levels from the leaves, disjoint participating sub-trees per band in post-order, packed
// first-fit-decreasing by upward cost into at most p bins; bins laid out in order.
std::vector<u32> coarsened_order(const Instance& in, u32 p, u32 agg) {
  p = std::max<u32>(1, p);
  agg = std::max<u32>(1, agg);
  std::vector<u32> h(in.num_nodes, 0);
  for (u32 i = in.num_nodes; i-- > 0;)
    if (!in.leaf(i)) h[i] = 1 + std::max(h[in.lchild[i]], h[in.rchild[i]]);
  const u32 H = h[0];
  std::vector<u32> order;
  if (H == 0) return order;
  const u32 levels = (H + agg - 1) / agg;
  auto cost = [&](u32 i) {
    const double own = in.srank[i];
    return in.leaf(i) ? in.size(i) * own : (double(in.srank[in.lchild[i]]) + in.srank[in.rchild[i]]) * own;
  };
  for (u32 lvl = 0; lvl < levels; ++lvl) {
    const u32 lo = lvl * agg, hi = lvl + 1 == levels ? H + 1 : (lvl + 1) * agg;
    std::vector<std::vector<u32>> subs;
    std::vector<double> costs;
    for (u32 i = 0; i < in.num_nodes; ++i) {
      if (h[i] < lo || h[i] >= hi) continue;
      const u32 par = in.parent[i];
      if (par != kNone && h[par] < hi) continue;  // not a band root
      std::vector<u32> nodes;
      std::vector<std::pair<u32, bool>> st{{i, false}};
      while (!st.empty()) {
        auto [x, done] = st.back();
        st.pop_back();
        if (h[x] < lo || h[x] >= hi) continue;
        if (done || in.leaf(x)) {
          if (in.part[x]) nodes.push_back(x);
          continue;
        }
        st.push_back({x, true});
        st.push_back({in.rchild[x], false});
        st.push_back({in.lchild[x], false});
      }
      if (nodes.empty()) continue;
      double c = 0.0;
      for (u32 x : nodes) c += cost(x);
      subs.push_back(std::move(nodes));
      costs.push_back(c);
    }
    if (subs.empty()) continue;
    const u32 cnt = static_cast<u32>(subs.size());
    const u32 bins = cnt > p ? p : std::max<u32>(1, cnt / 2);
    std::vector<u32> ord(cnt);
    std::iota(ord.begin(), ord.end(), 0u);
    std::stable_sort(ord.begin(), ord.end(), [&](u32 a, u32 b) { return costs[a] > costs[b]; });
    double total = 0.0, largest = 0.0;
    for (double c : costs) {
      total += c;
      largest = std::max(largest, c);
    }
    const double capy = std::max(largest, std::ceil(total / bins));
    std::vector<double> load(bins, 0.0);
    std::vector<std::vector<u32>> bin_nodes(bins);
    for (u32 r = 0; r < cnt; ++r) {
      const u32 sidx = ord[r];
      u32 chosen = kNone;
      if (total == 0.0) {
        chosen = r % bins;
      } else {
        for (u32 b = 0; b < bins && chosen == kNone; ++b)
          if (load[b] + costs[sidx] <= capy) chosen = b;
        if (chosen == kNone) chosen = static_cast<u32>(std::min_element(load.begin(), load.end()) - load.begin());
      }
      load[chosen] += costs[sidx];
      bin_nodes[chosen].insert(bin_nodes[chosen].end(), subs[sidx].begin(), subs[sidx].end());
    }
    for (auto& b : bin_nodes) order.insert(order.end(), b.begin(), b.end());
  }
  return order;
}

void pack(Instance& in) {
  const KernelFn K(in.spec.kernel, in.spec.h);
  const unsigned th = in.spec.threads;
  in.near_flat = blocked_order(in, in.near, in.spec.near_blocksize);
  in.far_flat = blocked_order(in, in.far, in.spec.far_blocksize);
  in.v_order = coarsened_order(in, in.spec.coarsen_p, in.spec.coarsen_agg);
  const u64 nn = in.near_flat.size() / 2, nf = in.far_flat.size() / 2, nv = in.v_order.size();
  in.dptr.assign(nn + 1, 0);
  in.bptr.assign(nf + 1, 0);
  in.vptr.assign(nv + 1, 0);
  for (u64 s = 0; s < nn; ++s)
    in.dptr[s + 1] = in.dptr[s] + u64(in.size(in.near_flat[2 * s])) * in.size(in.near_flat[2 * s + 1]);
  for (u64 s = 0; s < nf; ++s)
    in.bptr[s + 1] = in.bptr[s] + u64(in.srank[in.far_flat[2 * s]]) * in.srank[in.far_flat[2 * s + 1]];
  for (u64 s = 0; s < nv; ++s) in.vptr[s + 1] = in.vptr[s] + in.basis[in.v_order[s]].size();
  in.dgen.resize(in.spec.skip_near ? 0 : in.dptr[nn]);
  in.bgen.resize(in.bptr[nf]);
  in.vgen.resize(in.vptr[nv]);
  if (!in.spec.skip_near) parallel_for(nn, th, [&](u64 s) {
    const u32 i = in.near_flat[2 * s], j = in.near_flat[2 * s + 1];
    double* out = in.dgen.data() + in.dptr[s];
    const u32 mi = in.size(i);
    for (u32 c = 0; c < in.size(j); ++c)
      for (u32 r = 0; r < mi; ++r) out[c * mi + r] = K(in.tp(in.start[i] + r), in.tp(in.start[j] + c), in.d);
  });
  parallel_for(nf, th, [&](u64 s) {
    const u32 i = in.far_flat[2 * s], j = in.far_flat[2 * s + 1];
    double* out = in.bgen.data() + in.bptr[s];
    const u32 si = in.srank[i];
    for (u32 c = 0; c < in.srank[j]; ++c)
      for (u32 r = 0; r < si; ++r) out[c * si + r] = K(in.tp(in.skel[i][r]), in.tp(in.skel[j][c]), in.d);
  });
  parallel_for(nv, th, [&](u64 s) {
    const auto& b = in.basis[in.v_order[s]];
    std::copy(b.begin(), b.end(), in.vgen.begin() + in.vptr[s]);
  });
}

void build(Instance& in) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  auto& s = in.spec;
  if (s.threads == 0) s.threads = std::max(1u, std::thread::hardware_concurrency());
  if (s.n < 2) throw std::invalid_argument("builder: need n >= 2");
  if (s.points != HMXB_PTS_GRID2D && s.d < 1) throw std::invalid_argument("builder: need d >= 1");
  if (!(s.h > 0.0) && s.kernel != HMXB_K_INVDIST) throw std::invalid_argument("builder: bandwidth must be > 0");
  if (s.leaf < 1 || s.leaf >= s.n) throw std::invalid_argument("builder: need 1 <= leaf < n (one-node trees are rejected, structure.cpp:35-36)");
  if (s.tol < 0.0) throw std::invalid_argument("builder: tol must be >= 0");
  auto t = clk::now();
  make_points(in);
  in.stats.seconds_points = since(t);
  t = clk::now();
  build_tree(in);
  in.stats.seconds_tree = since(t);

  t = clk::now();
  const Geometry g = geometry(in);
  std::vector<u32> leaves;
  for (u32 i = 0; i < in.num_nodes; ++i)
    if (in.leaf(i)) leaves.push_back(i);
  const u32 k = static_cast<u32>(std::min<u64>(s.knn_k ? s.knn_k : 32, in.n - 1));
  const bool exact = s.sample_rows == std::numeric_limits<u32>::max();
  std::vector<u32> nbr;
  if (!exact || s.mode == HMXB_BUDGET) nbr = knn(in, g, leaves, k, 8);
  in.stats.seconds_sampling = since(t);
  t = clk::now();
  in.near.assign(in.num_nodes, {});
  in.far.assign(in.num_nodes, {});
  if (s.mode == HMXB_HSS) interactions_hss(in);
  else if (s.mode == HMXB_TAU) interactions_tau(in, g);
  else interactions_budget(in, g, leaves, nbr, k);
  for (auto& l : in.near) std::sort(l.begin(), l.end());
  for (auto& l : in.far) std::sort(l.begin(), l.end());
  in.part.assign(in.num_nodes, 0);
  for (u32 i = 0; i < in.num_nodes; ++i)
    if (!in.far[i].empty()) in.part[i] = 1;
  for (u32 i = 0; i < in.num_nodes; ++i)  // closed downward; parents precede children
    if (in.part[i] && !in.leaf(i)) in.part[in.lchild[i]] = in.part[in.rchild[i]] = 1;
  in.stats.seconds_interactions = since(t);

  t = clk::now();
  compress(in, nbr, k);
  in.stats.seconds_compress = since(t);
  t = clk::now();
  pack(in);
  in.stats.seconds_blocks = since(t);
  in.stats.seconds_total = since(t0);
  in.stats.leaves = leaves.size();
  in.stats.near_pairs = in.near_flat.size() / 2;
  in.stats.far_pairs = in.far_flat.size() / 2;
  in.stats.height = in.height;
  for (u32 sr : in.srank) in.stats.max_srank = std::max(in.stats.max_srank, sr);
}

}  // namespace
}  // namespace hmxb

struct hmxb_instance {
  hmxb::Instance in;
};

extern "C" {

const char* hmxb_last_error(void) { return hmxb::g_err.c_str(); }

void hmxb_spec_default(hmxb_spec* s) {
  std::memset(s, 0, sizeof *s);
  s->n = 4096;
  s->d = 3;
  s->points = HMXB_PTS_UNIFORM;
  s->components = 8;
  s->levels = 16;
  s->seed = 42;
  s->kernel = HMXB_K_GAUSSIAN;
  s->h = 0.5;
  s->leaf = 128;
  s->split = HMXB_SPLIT_AUTO;
  s->mode = HMXB_HSS;
  s->tau = 0.65;
  s->budget = 0.03;
  s->max_rank = 64;
  s->tol = 1e-5;
  s->sample_rows = 0;
  s->knn_k = 32;
  s->near_blocksize = 2;
  s->far_blocksize = 4;
  s->coarsen_p = 8;
  s->coarsen_agg = 2;
  s->threads = 0;
}

int hmxb_build(const hmxb_spec* spec, hmxb_instance** out) {
  if (!spec || !out) {
    hmxb::g_err = "hmxb_build: null argument";
    return HMXG_EINVAL;
  }
  *out = nullptr;
  try {
    auto inst = std::make_unique<hmxb_instance>();
    inst->in.spec = *spec;
    hmxb::build(inst->in);
    *out = inst.release();
    return HMXG_OK;
  } catch (const std::invalid_argument& e) {
    hmxb::g_err = e.what();
    return HMXG_EINVAL;
  } catch (const std::bad_alloc&) {
    hmxb::g_err = "hmxb_build: out of host memory";
    return HMXG_ENOMEM;
  } catch (const std::exception& e) {
    hmxb::g_err = e.what();
    return HMXG_EINVAL;
  }
}

int hmxb_view(const hmxb_instance* inst, hmxg_cds_view* v) {
  if (!inst || !v) return HMXG_EINVAL;
  const auto& in = inst->in;
  std::memset(v, 0, sizeof *v);
  v->n = in.n;
  v->num_nodes = in.num_nodes;
  v->height = in.height;
  v->parent = in.parent.data();
  v->lchild = in.lchild.data();
  v->rchild = in.rchild.data();
  v->start = in.start.data();
  v->end = in.end.data();
  v->level = in.level.data();
  v->perm = in.perm.data();
  v->sranks = in.srank.data();
  v->participating = in.part.data();
  v->num_near = in.near_flat.size() / 2;
  v->near_pairs = in.near_flat.data();
  v->num_far = in.far_flat.size() / 2;
  v->far_pairs = in.far_flat.data();
  v->num_v = in.v_order.size();
  v->v_order = in.v_order.data();
  v->dptr = in.dptr.data();
  v->bptr = in.bptr.data();
  v->vptr = in.vptr.data();
  v->dgen = in.dgen.data();
  v->bgen = in.bgen.data();
  v->vgen = in.vgen.data();
  return HMXG_OK;
}

int hmxb_points(const hmxb_instance* inst, const double** coords, uint64_t* n, uint32_t* d) {
  if (!inst) return HMXG_EINVAL;
  *coords = inst->in.pts.data();
  *n = inst->in.n;
  *d = inst->in.d;
  return HMXG_OK;
}

int hmxb_stats(const hmxb_instance* inst, hmxb_build_stats* st) {
  if (!inst || !st) return HMXG_EINVAL;
  *st = inst->in.stats;
  return HMXG_OK;
}

int hmxb_dense_rows(const hmxb_instance* inst, const uint32_t* rows, uint64_t nrows, const double* W,
                    uint64_t q, uint64_t ldw, double* out, uint64_t ldo) {
  if (!inst || (nrows && (!rows || !out)) || (q && !W) || ldw < inst->in.n) return HMXG_EINVAL;
  const auto& in = inst->in;
  const hmxb::KernelFn K(in.spec.kernel, in.spec.h);
  for (uint64_t r = 0; r < nrows; ++r)
    if (rows[r] >= in.n) return HMXG_EINVAL;
  hmxb::parallel_for(nrows, in.spec.threads, [&](uint64_t r) {
    const double* x = in.pts.data() + static_cast<uint64_t>(rows[r]) * in.d;
    std::vector<double> kv(in.n);
    for (uint64_t j = 0; j < in.n; ++j) kv[j] = K(x, in.pts.data() + j * in.d, in.d);
    for (uint64_t c = 0; c < q; ++c) {
      double s = 0.0;
      const double* w = W + c * ldw;
      for (uint64_t j = 0; j < in.n; ++j) s += kv[j] * w[j];
      out[r + c * ldo] = s;
    }
  });
  return HMXG_OK;
}

void hmxb_free(hmxb_instance* inst) { delete inst; }

void hmxb_random_w(uint64_t seed, uint64_t n, uint64_t q, double* out) {
  hmxb::Xoshiro rng(hmxb::splitmix64(seed ^ hmxb::splitmix64(0x77a7ULL)));
  for (uint64_t i = 0; i < n * q; ++i) out[i] = rng.uniform() * 2.0 - 1.0;
}

}  // extern "C"
