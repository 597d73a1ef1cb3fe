// plan.cpp — CDS validation and lowering to level-batched task tables (see plan.hpp).
#include "plan.hpp"

#include <algorithm>
#include <cstdlib>
#include <limits>
#include <sstream>

namespace hmxg {

namespace {

constexpr std::uint64_t kNoSlot = std::numeric_limits<std::uint64_t>::max();

template <class... A>
bool fail(std::string& err, A&&... parts) {
  std::ostringstream os;
  (os << ... << parts);
  err = os.str();
  return false;
}

}  // namespace

bool build_plan(const hmxg_cds_view& v, std::uint32_t tile_m, Plan& plan, std::string& err, const SplitSpec& split) {
  plan = Plan{};
  const std::uint32_t nn = v.num_nodes;
  if (nn == 0) return fail(err, "cds: empty tree");
  if (!v.parent || !v.lchild || !v.rchild || !v.start || !v.end || !v.level || !v.perm ||
      !v.sranks || !v.participating || !v.dptr || !v.bptr || !v.vptr)
    return fail(err, "cds: null array in view");
  if ((v.num_near && !v.near_pairs) || (v.num_far && !v.far_pairs) || (v.num_v && !v.v_order))
    return fail(err, "cds: null pair list in view");
  if ((v.dptr[v.num_near] && !v.dgen && !split.generated_near) || (v.bptr[v.num_far] && !v.bgen && !split.generated_far) || (v.vptr[v.num_v] && !v.vgen))
    return fail(err, "cds: null generator array in view");
  if (v.n == 0 || v.n > std::numeric_limits<std::uint32_t>::max())
    return fail(err, "cds: point count out of range");
  if (v.parent[0] != HMXG_NO_NODE || v.start[0] != 0 || v.end[0] != v.n)
    return fail(err, "cds: node 0 must be the root covering [0, n)");
  plan.n = v.n;
  plan.num_nodes = nn;

  // --- tree structure (ClusterTree invariants, proj/src/tree.cpp:27-47)
  std::vector<std::uint8_t> seen(v.n, 0);
  for (std::uint64_t p = 0; p < v.n; ++p) {
    if (v.perm[p] >= v.n || seen[v.perm[p]]) return fail(err, "cds: perm is not a bijection");
    seen[v.perm[p]] = 1;
  }
  auto is_leaf = [&](std::uint32_t i) { return v.lchild[i] == HMXG_NO_NODE; };
  std::vector<std::uint32_t> order;  // BFS from the root
  order.reserve(nn);
  order.push_back(0);
  for (std::size_t qi = 0; qi < order.size(); ++qi) {
    const std::uint32_t i = order[qi];
    if (v.start[i] > v.end[i] || v.end[i] > v.n) return fail(err, "cds: bad range of node ", i);
    if (is_leaf(i)) {
      if (v.rchild[i] != HMXG_NO_NODE) return fail(err, "cds: half-leaf node ", i);
      continue;
    }
    const std::uint32_t l = v.lchild[i], r = v.rchild[i];
    if (l >= nn || r >= nn || l == r) return fail(err, "cds: bad children of node ", i);
    if (v.parent[l] != i || v.parent[r] != i) return fail(err, "cds: bad parent link under ", i);
    if (v.start[l] != v.start[i] || v.end[l] != v.start[r] || v.end[r] != v.end[i])
      return fail(err, "cds: children do not partition node ", i);
    if (v.level[l] != v.level[i] + 1 || v.level[r] != v.level[i] + 1)
      return fail(err, "cds: level of children of node ", i);
    order.push_back(l);
    order.push_back(r);
    if (order.size() > nn) return fail(err, "cds: tree has a cycle");
  }
  if (order.size() != nn) return fail(err, "cds: nodes unreachable from the root");
  std::uint32_t height = 0;
  for (std::uint32_t i = 0; i < nn; ++i) height = std::max(height, v.level[i]);
  std::vector<std::uint32_t> sub_h(nn, 0);  // longest downward path (tree.cpp:19-25)
  for (std::size_t qi = order.size(); qi-- > 0;) {
    const std::uint32_t i = order[qi];
    if (!is_leaf(i)) sub_h[i] = 1 + std::max(sub_h[v.lchild[i]], sub_h[v.rchild[i]]);
  }

  auto active = [&](std::uint32_t i) { return v.participating[i] && v.sranks[i] > 0; };
  auto size_of = [&](std::uint32_t i) { return v.end[i] - v.start[i]; };
  auto v_width = [&](std::uint32_t i) -> std::uint64_t {
    return is_leaf(i) ? size_of(i) : std::uint64_t(v.sranks[v.lchild[i]]) + v.sranks[v.rchild[i]];
  };
  for (std::uint32_t i = 0; i < nn; ++i) {
    if (!active(i) || is_leaf(i)) continue;
    // participation is closed downward (proj/src/interaction.cpp:145-157)
    if (!v.participating[v.lchild[i]] || !v.participating[v.rchild[i]])
      return fail(err, "cds: active node ", i, " has a non-participating child");
  }

  // --- generator slots and sizes (structure.hpp:88-130)
  std::vector<std::uint64_t> vslot(nn, kNoSlot);
  for (std::uint64_t s = 0; s < v.num_v; ++s) {
    const std::uint32_t i = v.v_order[s];
    if (i >= nn || vslot[i] != kNoSlot) return fail(err, "cds: bad v_order entry ", s);
    vslot[i] = s;
    if (v.vptr[s + 1] < v.vptr[s] || v.vptr[s + 1] - v.vptr[s] != v_width(i) * v.sranks[i])
      return fail(err, "cds: V generator of node ", i, " has the wrong size");
  }
  for (std::uint32_t i = 0; i < nn; ++i)
    if (active(i) && vslot[i] == kNoSlot) return fail(err, "cds: node ", i, " has no basis generator");
  std::vector<std::vector<std::uint64_t>> far_of(nn), near_of(nn);
  for (std::uint64_t s = 0; s < v.num_far; ++s) {
    const std::uint32_t i = v.far_pairs[2 * s], j = v.far_pairs[2 * s + 1];
    if (i >= nn || j >= nn) return fail(err, "cds: far pair ", s, " out of range");
    if (v.bptr[s + 1] < v.bptr[s] ||
        v.bptr[s + 1] - v.bptr[s] != std::uint64_t(v.sranks[i]) * v.sranks[j])
      return fail(err, "cds: far generator ", s, " has the wrong size");
    if (v.sranks[i] == 0 || v.sranks[j] == 0) continue;  // no-op pair, executor.cpp:107
    if (!active(i) || !active(j)) return fail(err, "cds: far pair ", s, " touches a non-participating node");
    far_of[i].push_back(s);
  }
  for (std::uint64_t s = 0; s < v.num_near; ++s) {
    const std::uint32_t i = v.near_pairs[2 * s], j = v.near_pairs[2 * s + 1];
    if (i >= nn || j >= nn || !is_leaf(i) || !is_leaf(j)) return fail(err, "cds: near pair ", s, " is not a leaf pair");
    if (v.dptr[s + 1] < v.dptr[s] ||
        v.dptr[s + 1] - v.dptr[s] != std::uint64_t(size_of(i)) * size_of(j))
      return fail(err, "cds: near generator ", s, " has the wrong size");
    near_of[i].push_back(s);
  }
  plan.d_elems = v.dptr[v.num_near];
  plan.b_elems = v.bptr[v.num_far];
  plan.v_elems = v.vptr[v.num_v];
  if (std::max({plan.d_elems, plan.b_elems, plan.v_elems}) >= (std::uint64_t(1) << 62))
    return fail(err, "cds: generator arrays too large");

  // --- padded row layouts: leaves in Wp/Yp, active nodes in T/S, 16-row aligned blocks
  auto pad16 = [](std::uint64_t r) { return (r + kRowAlign - 1) / kRowAlign * kRowAlign; };
  plan.leaf_row.assign(nn, 0);
  std::vector<std::uint32_t> leaves_by_start;
  for (std::uint32_t i = 0; i < nn; ++i)
    if (is_leaf(i)) leaves_by_start.push_back(i);
  std::sort(leaves_by_start.begin(), leaves_by_start.end(),
            [&](std::uint32_t a, std::uint32_t b) { return v.start[a] < v.start[b]; });
  std::uint64_t prow = 0;
  for (std::uint32_t i : leaves_by_start) {
    plan.leaf_row[i] = prow;
    prow += pad16(size_of(i));
  }
  if (prow > std::numeric_limits<std::uint32_t>::max() - kRowAlign) return fail(err, "cds: too many points");
  plan.rows_pad = prow;
  // Leaf point orders (identity rows, below): a leaf basis V_i has a unit row for every
  // skeleton point, so its points are ordered [points dense in V_i, skeleton points]. The
  // upward K range is then a prefix of the leaf's Wp rows and the downward V_i product a
  // prefix of its Y' rows; the skeleton points become row copies.
  std::vector<std::vector<std::uint32_t>> lpt(nn), lpt_pos(nn);  // new row -> old position; inverse
  std::vector<std::vector<std::uint32_t>> leaf_unit_col(nn);     // old position -> V column (kNoMap)
  std::vector<std::vector<std::uint32_t>> leaf_col_src(nn);      // V column -> old position (kNoMap)
  std::vector<std::uint32_t> dense_pts(nn, 0), pt_map_off(nn, kNoMap);
  for (std::uint32_t i = 0; i < nn; ++i) dense_pts[i] = size_of(i);
  if (split.identity_rows && v.num_v) {
    for (std::uint32_t i : leaves_by_start) {
      if (!(v.participating[i] && v.sranks[i] > 0)) continue;
      const std::uint64_t W = size_of(i), K = v.sranks[i];
      const double* V = v.vgen + v.vptr[vslot[i]];
      leaf_unit_col[i].assign(W, kNoMap);
      leaf_col_src[i].assign(K, kNoMap);
      for (std::uint64_t r = 0; r < W; ++r) {
        std::uint64_t nz = 0, col = 0;
        for (std::uint64_t j = 0; j < K && nz < 2; ++j)
          if (V[r + j * W] != 0.0) {
            ++nz;
            col = j;
          }
        if (nz != 1 || V[r + col * W] != 1.0 || leaf_col_src[i][col] != kNoMap) continue;
        leaf_unit_col[i][r] = static_cast<std::uint32_t>(col);
        leaf_col_src[i][col] = static_cast<std::uint32_t>(r);
      }
      for (std::uint32_t r = 0; r < W; ++r)
        if (leaf_unit_col[i][r] == kNoMap) lpt[i].push_back(r);
      dense_pts[i] = static_cast<std::uint32_t>(lpt[i].size());
      if (dense_pts[i] == W) {
        lpt[i].clear();
        continue;
      }
      for (std::uint32_t r = 0; r < W; ++r)
        if (leaf_unit_col[i][r] != kNoMap) lpt[i].push_back(r);
      lpt_pos[i].assign(W, 0);
      for (std::uint32_t q = 0; q < W; ++q) lpt_pos[i][lpt[i][q]] = q;
      pt_map_off[i] = static_cast<std::uint32_t>(plan.maps.size());
      plan.maps.insert(plan.maps.end(), lpt[i].begin(), lpt[i].end());
    }
  }
  plan.pmap.assign(prow, 0xffffffffu);
  plan.ipmap.assign(v.n, 0);
  for (std::uint32_t i : leaves_by_start)
    for (std::uint32_t r = 0; r < size_of(i); ++r) {
      const std::uint32_t orig = v.perm[v.start[i] + (lpt[i].empty() ? r : lpt[i][r])];
      plan.pmap[plan.leaf_row[i] + r] = orig;
      plan.ipmap[orig] = static_cast<std::uint32_t>(plan.leaf_row[i] + r);
    }
  // --- subtree split: owner part of every node (-1: replicated top level)
  if (split.nparts == 0 || split.part >= split.nparts) return fail(err, "split: bad part / nparts");
  plan.nparts = split.nparts;
  plan.part = split.part;
  const bool splitting = split.nparts > 1;
  std::vector<int> owner(nn, 0);
  if (splitting) {
    std::uint32_t top_depth = 0;
    while ((1u << top_depth) < split.nparts) ++top_depth;
    std::vector<std::uint32_t> roots;  // subtree roots in tree-position order
    for (std::uint32_t i : order)
      if (v.level[i] == top_depth || (v.level[i] < top_depth && is_leaf(i))) roots.push_back(i);
    std::sort(roots.begin(), roots.end(), [&](std::uint32_t a, std::uint32_t b) { return v.start[a] < v.start[b]; });
    for (std::uint32_t i = 0; i < nn; ++i) owner[i] = -1;
    for (std::size_t k = 0; k < roots.size(); ++k)
      owner[roots[k]] = static_cast<int>(k * split.nparts / roots.size());
    for (std::uint32_t i : order)  // BFS: parents before children
      if (!is_leaf(i) && owner[i] >= 0) owner[v.lchild[i]] = owner[v.rchild[i]] = owner[i];
    for (std::uint32_t i = 0; i < nn; ++i)
      if (owner[i] >= 0 && owner[i] != static_cast<int>(split.part) && active(i)) plan.remote_t_nodes.push_back(i);
  }
  // Split mode: the T rows a part publishes (the nodes another part's stage 1 reads: children
  // of the replicated top nodes, and far partners of top nodes or of another part's nodes)
  // come first in T, grouped by part, so the exchange is one in-place all-gather of
  // contiguous row ranges (pub_row[p], pub_row[p + 1]) instead of a sum over the whole T.
  // Each part's leaves are contiguous in Wp / Yp: the result rows of part p are
  // [yp_row[p], yp_row[p + 1]).
  std::vector<std::uint8_t> published(nn, 0);
  if (splitting) {
    for (std::uint32_t i = 0; i < nn; ++i) {
      if (owner[i] < 0 || !active(i)) continue;
      const std::uint32_t par = v.parent[i];
      if (par != HMXG_NO_NODE && owner[par] < 0) published[i] = 1;
    }
    for (std::uint32_t c = 0; c < nn; ++c)
      for (std::uint64_t s : far_of[c]) {
        const std::uint32_t j = v.far_pairs[2 * s + 1];
        if (owner[j] >= 0 && (owner[c] < 0 || owner[c] != owner[j])) published[j] = 1;
      }
  }
  plan.node_off.assign(nn, 0);
  std::uint64_t rows = 0;
  plan.pub_row.assign(split.nparts + 1, 0);
  if (splitting) {
    for (std::uint32_t p = 0; p < split.nparts; ++p) {
      plan.pub_row[p] = rows;
      for (std::uint32_t i : order)
        if (published[i] && owner[i] == static_cast<int>(p)) {
          plan.node_off[i] = rows;
          rows += pad16(v.sranks[i]);
        }
    }
    plan.pub_row[split.nparts] = rows;
  }
  for (std::uint32_t i : order)
    if (active(i) && !published[i]) {
      plan.node_off[i] = rows;
      rows += pad16(v.sranks[i]);
    }
  plan.yp_row.assign(split.nparts + 1, 0);
  if (splitting) {
    std::vector<std::uint64_t> lo(split.nparts, ~std::uint64_t(0)), hi(split.nparts, 0), cnt(split.nparts, 0);
    for (std::uint32_t i : leaves_by_start) {
      const int o = owner[i];
      if (o < 0) return fail(err, "split: leaf without an owner part");
      lo[o] = std::min(lo[o], plan.leaf_row[i]);
      hi[o] = std::max(hi[o], plan.leaf_row[i] + pad16(size_of(i)));
      cnt[o] += pad16(size_of(i));
    }
    for (std::uint32_t p = 0; p < split.nparts; ++p) {
      if (cnt[p] == 0) lo[p] = hi[p] = p ? plan.yp_row[p] : 0;
      if (hi[p] - lo[p] != cnt[p] || lo[p] != (p ? plan.yp_row[p] : 0))
        return fail(err, "split: the leaves of part ", p, " are not contiguous");
      plan.yp_row[p + 1] = hi[p];
    }
  }
  if (rows > std::numeric_limits<std::uint32_t>::max() - kRowAlign) return fail(err, "cds: too many skeleton rows");
  plan.skel_rows = std::max<std::uint64_t>(rows, kRowAlign);

  const std::uint32_t bm = tile_m;
  plan.node_tiles.assign(nn, 0);
  for (std::uint32_t i = 0; i < nn; ++i)
    if (active(i)) plan.node_tiles[i] = (v.sranks[i] + bm - 1) / bm;
  std::uint32_t cur_node = 0;
  // identity sources of the current node's output rows (row -> absolute row of id_buf, or
  // kNoMap), set by the pass before add_tiles; empty: none
  std::vector<std::uint32_t> cur_id;
  std::uint16_t cur_id_buf = 0;
  std::uint32_t cur_id_node0 = kNoMap, cur_id_node1 = kNoMap;
  auto add_tiles = [&](std::uint32_t m, Buf cbuf, std::uint64_t c_row, auto&& emit_segs, Phase& ph) {
    const std::uint32_t tiles = m == 0 ? 0 : (m + bm - 1) / bm;
    if (cbuf == kBufYp) plan.leaf_tasks += tiles;
    for (std::uint32_t t = 0; t < tiles; ++t) {
      const std::uint32_t r0 = t * bm;
      Task task{};
      task.c_row = static_cast<std::uint32_t>(c_row + r0);
      task.cbuf = cbuf;
      task.m = static_cast<std::uint16_t>(std::min(bm, m - r0));
      task.node = cur_node;
      task.id_off = kNoMap;
      task.id_node0 = task.id_node1 = kNoMap;
      task.seg_begin = static_cast<std::uint32_t>(plan.segs.size());
      emit_segs(r0, task.m);
      task.seg_end = static_cast<std::uint32_t>(plan.segs.size());
      if (!cur_id.empty()) {
        bool any = false;
        for (std::uint32_t r = r0; r < r0 + task.m; ++r) any = any || cur_id[r] != kNoMap;
        if (any) {
          task.id_off = static_cast<std::uint32_t>(plan.idmap.size());
          plan.idmap.insert(plan.idmap.end(), cur_id.begin() + r0, cur_id.begin() + r0 + task.m);
          task.id_buf = cur_id_buf;
          task.id_node0 = cur_id_node0;
          task.id_node1 = cur_id_node1;
        }
      }
      for (std::uint32_t s = task.seg_begin; s < task.seg_end; ++s) {
        const double k = plan.tile_src[s].k, rows = plan.tile_src[s].m;
        ph.flops_per_col += 2.0 * rows * k;  // executed: identity rows are row copies
        ph.gen_bytes += 8.0 * rows * k;
        if (t == 0) ph.io_bytes_per_col += 8.0 * k;  // B rows, read once per node
      }
      plan.tasks.push_back(task);
    }
    ph.io_bytes_per_col += 8.0 * m;  // C rows, written once
    plan.max_m = std::max(plan.max_m, m);
  };
  // A operand of one segment: tile rows r < m read generator row rmap[r0 + r] (or r0 + r),
  // K index k < kcount reads generator column kmap[k] (or k), of the block at a_off with
  // leading dimension lda; B rows [b_row, b_row + kcount). Only the first `rows` tile rows
  // carry data (the rest are identity rows handled as row copies, zero in A).
  bool seg_overflow = false;
  auto push_seg = [&](Gen gen, bool trans, std::uint64_t a_off, std::uint64_t lda, std::uint64_t k,
                      std::uint32_t m, Buf bbuf, std::uint64_t b_row, std::uint32_t src, std::uint32_t r0,
                      std::uint32_t rmap, std::uint32_t kmap, std::uint32_t rows) {
    rows = std::min(rows, m);
    if (k == 0 || rows == 0) return;
    const std::uint64_t chunks = (k + kRowAlign - 1) / kRowAlign;
    if (chunks > 0xffffu) seg_overflow = true;  // SegDev::nchunks is 16 bits (a K range of 2^20 rows)
    TileSrc ts{};
    ts.a_off = a_off;
    ts.tile_off = plan.tile_elems;
    ts.lda = static_cast<std::uint32_t>(lda);
    ts.k = static_cast<std::uint32_t>(k);
    ts.m = static_cast<std::uint16_t>(rows);
    ts.gen = gen;
    ts.trans = trans ? 1 : 0;
    ts.r0 = r0;
    ts.rmap = rmap;
    ts.kmap = kmap;
    for (std::uint64_t c = 0; c < chunks; ++c) plan.chunk_seg.push_back(static_cast<std::uint32_t>(plan.segs.size()));
    const std::uint64_t k_last = k - (chunks - 1) * kRowAlign;  // 1 .. 16
    plan.segs.push_back(SegDev{plan.tile_elems, static_cast<std::uint32_t>(b_row), static_cast<std::uint16_t>(chunks),
                               static_cast<std::uint8_t>(bbuf), static_cast<std::uint8_t>(k_last == kRowAlign ? 0 : (k_last + 3) / 4),
                               src, rows < m ? rows : 0});
    plan.tile_src.push_back(ts);
    plan.tile_elems += chunks * kRowAlign * bm;
  };
  const int me = static_cast<int>(split.part);
  auto mine = [&](std::uint32_t i) { return !splitting || owner[i] == me; };
  auto top = [&](std::uint32_t i) { return splitting && owner[i] < 0; };

  // --- identity rows of the bases. An interpolative basis V_p has a unit row for every
  // skeleton column (compress.cpp:79-81: V(piv[j], j) = 1, the rest of the row 0), so the
  // rows of a child c that the parent keeps contribute exact row copies: T_p(j) += T_c(row)
  // upward and S_c(row) += S_p(j) downward. Each active child's rows (its T and S order,
  // the columns of its V, the rows / columns of its far blocks) are reordered as
  // [rows dense in V_p, rows copied by V_p]: the upward K range of the child is then a
  // prefix and the downward V_p product covers a prefix of the child's rows. The copies
  // move to the tile epilogue; only multiply-adds by exact zeros and ones are dropped.
  std::vector<std::vector<std::uint32_t>> rperm(nn);  // node row order: new -> old (empty: identity)
  std::vector<std::vector<std::uint32_t>> rpos(nn);   // old -> new
  std::vector<std::vector<std::uint32_t>> idcol(nn);  // old row -> parent column it copies (kNoMap)
  std::vector<std::vector<std::uint64_t>> colsrc(nn); // parent: column -> (child << 32 | old row), or ~0
  std::vector<std::uint32_t> dense(nn, 0);            // rows [0, dense) of a node are dense in V_parent
  std::vector<std::uint32_t> map_off(nn, kNoMap);
  for (std::uint32_t i = 0; i < nn; ++i) dense[i] = v.sranks[i];
  if (split.identity_rows && v.num_v) {
    for (std::uint32_t p = 0; p < nn; ++p) {
      if (!active(p) || is_leaf(p)) continue;
      const std::uint32_t lc = v.lchild[p], rc = v.rchild[p];
      const std::uint64_t W = v_width(p), K = v.sranks[p], klc = v.sranks[lc];
      const double* V = v.vgen + v.vptr[vslot[p]];
      colsrc[p].assign(K, ~std::uint64_t(0));
      for (std::uint32_t c : {lc, rc}) idcol[c].assign(v.sranks[c], kNoMap);
      for (std::uint64_t r = 0; r < W; ++r) {
        std::uint64_t nz = 0, col = 0;
        for (std::uint64_t j = 0; j < K && nz < 2; ++j)
          if (V[r + j * W] != 0.0) {
            ++nz;
            col = j;
          }
        if (nz != 1 || V[r + col * W] != 1.0 || colsrc[p][col] != ~std::uint64_t(0)) continue;
        const std::uint32_t c = r < klc ? lc : rc;
        const std::uint32_t old = static_cast<std::uint32_t>(r < klc ? r : r - klc);
        idcol[c][old] = static_cast<std::uint32_t>(col);
        colsrc[p][col] = (std::uint64_t(c) << 32) | old;
      }
      for (std::uint32_t c : {lc, rc}) {
        if (!active(c)) continue;
        std::vector<std::uint32_t>& order_c = rperm[c];
        for (std::uint32_t r = 0; r < v.sranks[c]; ++r)
          if (idcol[c][r] == kNoMap) order_c.push_back(r);
        dense[c] = static_cast<std::uint32_t>(order_c.size());
        for (std::uint32_t r = 0; r < v.sranks[c]; ++r)
          if (idcol[c][r] != kNoMap) order_c.push_back(r);
        if (dense[c] == v.sranks[c]) {  // nothing copied: keep the natural order
          order_c.clear();
          continue;
        }
        rpos[c].assign(v.sranks[c], 0);
        for (std::uint32_t q = 0; q < v.sranks[c]; ++q) rpos[c][order_c[q]] = q;
        map_off[c] = static_cast<std::uint32_t>(plan.maps.size());
        plan.maps.insert(plan.maps.end(), order_c.begin(), order_c.end());
      }
    }
  }
  auto oldrow = [&](std::uint32_t i, std::uint32_t r) { return rperm[i].empty() ? r : rperm[i][r]; };
  auto newrow = [&](std::uint32_t i, std::uint32_t r) { return rpos[i].empty() ? r : rpos[i][r]; };

  std::uint32_t cur_stage = 0;
  auto open_phase = [&](PhaseKind kind, std::uint32_t level) {
    plan.phases.push_back(
        Phase{kind, cur_stage, static_cast<std::uint32_t>(plan.tasks.size()), 0, level, 0.0, 0.0, 0.0});
  };
  auto close_phase = [&]() {
    Phase& ph = plan.phases.back();
    ph.task_end = static_cast<std::uint32_t>(plan.tasks.size());
    if (ph.task_end == ph.task_begin) plan.phases.pop_back();
  };

  // --- upward, by subtree height: T_i = V_i^T * (leaf ? Wp_i : [T_lc; T_rc])
  std::uint32_t max_h = 0;
  for (std::uint32_t i = 0; i < nn; ++i) max_h = std::max(max_h, sub_h[i]);
  auto upward_pass = [&](auto&& take) {
    for (std::uint32_t h = 0; h <= max_h; ++h) {
      open_phase(kPhaseUp, h);
      for (std::uint32_t i : order) {
        if (sub_h[i] != h || !active(i) || !take(i)) continue;
        const std::uint64_t lda = v_width(i);
        const std::uint64_t vo = v.vptr[vslot[i]];
        cur_node = i;
        cur_id.clear();
        cur_id_node0 = cur_id_node1 = kNoMap;
        if (is_leaf(i) && !lpt[i].empty()) {  // T_i(j) += Wp(skeleton point of column j)
          cur_id.assign(v.sranks[i], kNoMap);
          for (std::uint32_t r = 0; r < v.sranks[i]; ++r) {
            const std::uint32_t pos = leaf_col_src[i][oldrow(i, r)];
            if (pos != kNoMap) cur_id[r] = static_cast<std::uint32_t>(plan.leaf_row[i] + lpt_pos[i][pos]);
          }
          cur_id_buf = kBufWp;  // complete before the launch, or (fused permutes) the leaf's own rows
          cur_id_node0 = i;
        }
        if (!is_leaf(i) && !colsrc[i].empty()) {  // T_i(j) += T_child(copied row)
          cur_id.assign(v.sranks[i], kNoMap);
          for (std::uint32_t r = 0; r < v.sranks[i]; ++r) {
            const std::uint64_t src = colsrc[i][oldrow(i, r)];
            if (src == ~std::uint64_t(0)) continue;
            const std::uint32_t c = static_cast<std::uint32_t>(src >> 32), old = static_cast<std::uint32_t>(src);
            cur_id[r] = static_cast<std::uint32_t>(plan.node_off[c] + newrow(c, old));
          }
          cur_id_buf = kBufT;
          cur_id_node0 = active(v.lchild[i]) ? v.lchild[i] : kNoMap;
          cur_id_node1 = active(v.rchild[i]) ? v.rchild[i] : kNoMap;
        }
        add_tiles(v.sranks[i], kBufT, plan.node_off[i], [&](std::uint32_t r0, std::uint32_t m) {
          // A = V_i^T: tile row r is column oldrow(i, r) of V_i
          if (is_leaf(i)) {  // K: the leaf's dense points (a prefix of its rows)
            push_seg(kGenV, true, vo, lda, dense_pts[i], m, kBufWp, plan.leaf_row[i], i, r0, map_off[i], pt_map_off[i],
                     m);
          } else {
            const std::uint32_t lc = v.lchild[i], rc = v.rchild[i];
            const std::uint64_t srl = v.sranks[lc];
            // K: the child's dense rows (a prefix of its order); copied rows are epilogue adds
            if (active(lc))
              push_seg(kGenV, true, vo, lda, dense[lc], m, kBufT, plan.node_off[lc], lc, r0, map_off[i], map_off[lc], m);
            if (active(rc))
              push_seg(kGenV, true, vo + srl, lda, dense[rc], m, kBufT, plan.node_off[rc], rc, r0, map_off[i],
                       map_off[rc], m);
          }
        }, plan.phases.back());
      }
      close_phase();
    }
  };
  upward_pass(mine);  // stage 0 (everything, without a split)
  cur_stage = splitting ? 1 : 0;
  if (splitting) upward_pass(top);  // stage 1: replicated top levels from the exchanged T

  // --- downward with the far pass folded in, by depth:
  //     S_c = sum_{far (c,j)} B_cj T_j + V_p[rows of c] S_p
  for (std::uint32_t d = 0; d <= height; ++d) {
    open_phase(kPhaseDown, d);
    for (std::uint32_t c : order) {
      if (v.level[c] != d || !active(c) || !(mine(c) || top(c))) continue;
      const std::uint32_t p = v.parent[c];
      cur_node = c;
      cur_id.clear();
      cur_id_node0 = cur_id_node1 = kNoMap;
      if (p != HMXG_NO_NODE && active(p) && !rperm[c].empty()) {  // S_c(row) += S_p(copied column)
        cur_id.assign(v.sranks[c], kNoMap);
        for (std::uint32_t r = dense[c]; r < v.sranks[c]; ++r)
          cur_id[r] = static_cast<std::uint32_t>(plan.node_off[p] + newrow(p, idcol[c][oldrow(c, r)]));
        cur_id_buf = kBufS;
        cur_id_node0 = p;
      }
      add_tiles(v.sranks[c], kBufS, plan.node_off[c], [&](std::uint32_t r0, std::uint32_t m) {
        for (std::uint64_t s : far_of[c]) {
          const std::uint32_t j = v.far_pairs[2 * s + 1];
          push_seg(kGenB, false, v.bptr[s], v.sranks[c], v.sranks[j], m, kBufT, plan.node_off[j], j, r0, map_off[c],
                   map_off[j], m);
        }
        if (p != HMXG_NO_NODE && active(p)) {
          const std::uint64_t row_in_parent = (c == v.lchild[p]) ? 0 : v.sranks[v.lchild[p]];
          const std::uint32_t rows = dense[c] > r0 ? dense[c] - r0 : 0;  // the copied rows sit below
          push_seg(kGenV, false, v.vptr[vslot[p]] + row_in_parent, v_width(p), v.sranks[p], m, kBufS,
                   plan.node_off[p], p, r0, map_off[c], map_off[p], rows);
        }
      }, plan.phases.back());
    }
    close_phase();
  }

  // --- leaves: Y'_i = sum_{near (i,j)} D_ij Wp_j + V_i S_i, one task per leaf row tile
  //     (kPhaseLeaf, every leaf row written once; the D segments first, then the V one,
  //     then the skeleton points' copied S_i rows, kTaskIdLast).
  //     The split variant (Plan::split_phases) runs the same D segments as a near task that
  //     needs only Wp, and the V segment as a leaf task that accumulates onto the near rows:
  //     the DAG can then fill the tree passes' idle slots with near-field tiles. Both
  //     variants share the segments and pre-tiled operands and sum in the same order, so
  //     they give the same bits (every column of Y is independent of how Q is split).
  plan.yp_tiles.assign(nn, 0);
  struct LeafTasks {
    std::uint32_t node, t0, t1;  // combined tasks [t0, t1) in plan.tasks
  };
  std::vector<LeafTasks> leaf_tasks_of;
  const std::uint32_t lt0_all = static_cast<std::uint32_t>(plan.tasks.size());
  open_phase(kPhaseLeaf, 0);
  for (std::uint32_t i : order) {
    if (!is_leaf(i) || !mine(i)) continue;
    const std::uint32_t m = size_of(i);
    cur_node = i;
    cur_id.clear();
    cur_id_node0 = cur_id_node1 = kNoMap;
    if (!lpt[i].empty()) {  // Y'_i(skeleton point) += S_i(its column)
      cur_id.assign(m, kNoMap);
      for (std::uint32_t r = dense_pts[i]; r < m; ++r)
        cur_id[r] = static_cast<std::uint32_t>(plan.node_off[i] + newrow(i, leaf_unit_col[i][lpt[i][r]]));
      cur_id_buf = kBufS;
      cur_id_node0 = i;
    }
    const std::uint32_t t0 = static_cast<std::uint32_t>(plan.tasks.size());
    add_tiles(m, kBufYp, plan.leaf_row[i], [&](std::uint32_t r0, std::uint32_t mt) {
      for (std::uint64_t s : near_of[i]) {
        const std::uint32_t j = v.near_pairs[2 * s + 1];
        push_seg(kGenD, false, v.dptr[s], m, size_of(j), mt, kBufWp, plan.leaf_row[j], j, r0, pt_map_off[i],
                 pt_map_off[j], mt);
      }
      if (active(i))  // the V_i product covers the dense points (a prefix of the rows)
        push_seg(kGenV, false, v.vptr[vslot[i]], m, v.sranks[i], mt, kBufS, plan.node_off[i], i, r0, pt_map_off[i],
                 map_off[i], dense_pts[i] > r0 ? dense_pts[i] - r0 : 0);
    }, plan.phases.back());
    for (std::uint32_t t = t0; t < plan.tasks.size(); ++t) plan.tasks[t].flags |= kTaskIdLast | kTaskFinal;
    leaf_tasks_of.push_back({i, t0, static_cast<std::uint32_t>(plan.tasks.size())});
  }
  close_phase();
  // split variant: near tasks, then leaf tasks accumulating onto them
  auto has_v_seg = [&](const Task& t) { return t.seg_end > t.seg_begin && plan.segs[t.seg_end - 1].bbuf == kBufS; };
  const std::uint32_t near_begin = static_cast<std::uint32_t>(plan.tasks.size());
  std::vector<std::uint8_t> split_leaf(nn, 0);
  for (const LeafTasks& lt : leaf_tasks_of) {
    const std::uint32_t i = lt.node;
    if (active(i) && near_of[i].empty()) continue;  // V only: its leaf task below writes the rows
    const bool with_v = active(i);
    if (with_v) split_leaf[i] = 1;
    plan.yp_tiles[i] = lt.t1 - lt.t0;
    for (std::uint32_t t = lt.t0; t < lt.t1; ++t) {
      Task nt = plan.tasks[t];
      // drop the V segment (the last of the task, when the tile has dense points) and the
      // skeleton-row copies: both belong to the leaf task below
      if (has_v_seg(nt)) nt.seg_end -= 1;
      nt.id_off = nt.id_node0 = nt.id_node1 = kNoMap;
      nt.flags = with_v ? 0 : kTaskFinal;  // an inactive leaf's near rows are its final rows
      plan.tasks.push_back(nt);
    }
  }
  const std::uint32_t near_end = static_cast<std::uint32_t>(plan.tasks.size());
  for (const LeafTasks& lt : leaf_tasks_of) {
    const std::uint32_t i = lt.node;
    if (!active(i)) continue;
    for (std::uint32_t t = lt.t0; t < lt.t1; ++t) {
      Task vt = plan.tasks[t];
      if (split_leaf[i]) {  // V segment (and skeleton copies) accumulated onto the near rows
        vt.seg_begin = has_v_seg(vt) ? vt.seg_end - 1 : vt.seg_end;
        vt.flags |= kTaskAccumulate;
      }
      plan.tasks.push_back(vt);
    }
  }
  const std::uint32_t acc_end = static_cast<std::uint32_t>(plan.tasks.size());
  for (std::uint32_t t = lt0_all; t < acc_end; ++t) {
    Task& tk = plan.tasks[t];
    if ((tk.flags & kTaskIdLast) && tk.id_off != kNoMap && tk.id_node1 == kNoMap && has_v_seg(tk) &&
        plan.segs[tk.seg_end - 1].src == tk.id_node0)
      tk.flags |= kTaskIdSynced;
  }
  auto split_phase = [&](PhaseKind kind, std::uint32_t t0, std::uint32_t t1) {
    Phase ph{kind, cur_stage, t0, t1, 0, 0.0, 0.0, 0.0};
    for (std::uint32_t t = t0; t < t1; ++t) {
      const Task& tk = plan.tasks[t];
      for (std::uint32_t sg = tk.seg_begin; sg < tk.seg_end; ++sg) {
        const double k = plan.tile_src[sg].k, rows = plan.tile_src[sg].m;
        ph.flops_per_col += 2.0 * rows * k;
        ph.gen_bytes += 8.0 * rows * k;
        ph.io_bytes_per_col += 8.0 * k / std::max<std::uint32_t>(1, plan.yp_tiles[tk.node]);
      }
      ph.io_bytes_per_col += 8.0 * tk.m * (tk.flags & kTaskAccumulate ? 2 : 1);
    }
    plan.split_phases.push_back(ph);
  };
  if (near_end > near_begin) split_phase(kPhaseNear, near_begin, near_end);
  if (acc_end > near_end) split_phase(kPhaseLeaf, near_end, acc_end);

  // --- flat tree for small trees (Plan::flat_phases). A chain of dependent GEMM levels costs
  //     ~4 us each through the DAG's gpu-scope counters (cfg1: 11 levels, the whole step),
  //     while a small tree's transfer products are cheap to form once. So every active
  //     internal node's T is taken straight from its leaves' T, T_p = sum_l C_pl T_l with
  //     C_pl = M_p,c C_cl (M_p = V_p^T, its column block of the child c on the path; C_ll = I),
  //     and every leaf's S straight from the T's it depends on,
  //     S_l = sum_{a on the path} sum_{j far from a} (G_la B_aj) T_j with G_ll = I and
  //     G_l,parent(a) = G_la V_parent(a)[rows of a] (executor.cpp:51-110 unrolled). Two
  //     dependent levels replace the internal upward and far+downward ones. The composites
  //     are formed once on the host in FP64, in the nodes' T/S row orders, as generator kGenC.
  //     Used when the tree is small and the extra multiply-adds stay below a quarter of the
  //     evaluation's (plan-wide, so every column count gives the same bits).
  // (the composites read B and V on the host: hmxg_upload_generated_ex brings the far blocks of
  // small trees back from the device first, so generated_far is only set for large trees)
  if (!splitting && split.flat_tree && !split.generated_far && (v.bgen || !v.num_far) && v.vgen) {
    double flat = 0.0, replaced = 0.0, total = 0.0;
    for (const Phase& ph : plan.phases) {
      if (ph.kind == kPhaseLeaf) {
        total += ph.flops_per_col;
        continue;
      }
      total += ph.flops_per_col;
      if (!(ph.kind == kPhaseUp && ph.level == 0)) replaced += ph.flops_per_col;
    }
    // Frontier of an upward composite: the nodes whose T it multiplies. Single stage: the
    // leaves. With a middle height h_mid, the nodes above it start from the nodes at h_mid
    // (one more dependent level, but the top nodes' K -- a segment per leaf under them -- is
    // cut: cfg1's root children stream 32 chunks from 16 leaves, 12 from 4 mid nodes).
    auto frontier_of = [&](std::uint32_t p, std::uint32_t h_mid, auto&& self) -> std::vector<std::uint32_t> {
      std::vector<std::uint32_t> f;
      for (std::uint32_t c : {v.lchild[p], v.rchild[p]}) {
        if (!active(c)) continue;
        if (is_leaf(c) || (h_mid && sub_h[c] == h_mid)) {
          f.push_back(c);
        } else {
          const std::vector<std::uint32_t> g = self(c, h_mid, self);
          f.insert(f.end(), g.begin(), g.end());
        }
      }
      return f;
    };
    auto kchunks = [&](std::uint32_t p, std::uint32_t h_mid) {
      std::uint64_t k = 0;
      for (std::uint32_t f : frontier_of(p, (h_mid && sub_h[p] > h_mid) ? h_mid : 0, frontier_of))
        k += (v.sranks[f] + kRowAlign - 1) / kRowAlign;
      return k;
    };
    std::uint32_t h_mid = 0;
    {
      std::uint64_t best = 0;
      for (std::uint32_t i = 0; i < nn; ++i)
        if (active(i) && !is_leaf(i)) best = std::max(best, kchunks(i, 0));
      if (best > 16)
        for (std::uint32_t h = 1; h + 1 <= max_h; ++h) {
          std::uint64_t worst = 0;
          for (std::uint32_t i = 0; i < nn; ++i)
            if (active(i) && !is_leaf(i)) worst = std::max(worst, kchunks(i, h));
          if (worst < best) {
            best = worst;
            h_mid = h;
          }
        }
    }
    auto stage_mid = [&](std::uint32_t p) { return (h_mid && sub_h[p] > h_mid) ? h_mid : 0u; };
    for (std::uint32_t i = 0; i < nn; ++i)
      if (active(i) && !is_leaf(i))
        for (std::uint32_t f : frontier_of(i, stage_mid(i), frontier_of)) flat += 2.0 * v.sranks[i] * v.sranks[f];
    for (std::uint32_t l = 0; l < nn; ++l) {
      if (!active(l) || !is_leaf(l)) continue;
      for (std::uint32_t a = l;;) {
        for (std::uint64_t s : far_of[a]) flat += 2.0 * v.sranks[l] * v.sranks[v.far_pairs[2 * s + 1]];
        const std::uint32_t par = v.parent[a];
        if (par == HMXG_NO_NODE || !active(par)) break;
        a = par;
      }
    }
    const bool small = v.n <= 65536 && nn <= 1024;
    if (small && flat - replaced <= 0.25 * total && replaced > 0.0) {
      // dense r_a x r_b blocks in the nodes' T/S row orders (column major), appended to cgen
      auto vget = [&](std::uint32_t p, std::uint64_t row, std::uint64_t col) {
        return v.vgen[v.vptr[vslot[p]] + row + col * v_width(p)];
      };
      // C_pf over each node's frontier, old orders: comp[0] = from the leaves, comp[1] = from
      // the leaves and the nodes at h_mid (used above h_mid)
      std::vector<std::vector<std::pair<std::uint32_t, std::vector<double>>>> comps[2] = {
          std::vector<std::vector<std::pair<std::uint32_t, std::vector<double>>>>(nn),
          std::vector<std::vector<std::pair<std::uint32_t, std::vector<double>>>>(h_mid ? nn : 0)};
      for (int st = 0; st < (h_mid ? 2 : 1); ++st)
      for (std::size_t qi = order.size(); qi-- > 0;) {
        auto& comp = comps[st];
        const std::uint32_t p = order[qi];
        if (!active(p) || is_leaf(p)) continue;
        const std::uint32_t rp = v.sranks[p];
        for (std::uint32_t c : {v.lchild[p], v.rchild[p]}) {
          if (!active(c)) continue;
          const std::uint64_t off = c == v.lchild[p] ? 0 : v.sranks[v.lchild[p]];
          const std::uint32_t rc = v.sranks[c];
          auto mpc = [&](std::uint32_t i, std::uint32_t k) { return vget(p, off + k, i); };  // M_p,c(i, k)
          if (is_leaf(c) || (st == 1 && sub_h[c] == h_mid)) {
            std::vector<double> m(std::size_t(rp) * rc);
            for (std::uint32_t k = 0; k < rc; ++k)
              for (std::uint32_t i = 0; i < rp; ++i) m[i + std::size_t(k) * rp] = mpc(i, k);
            comp[p].push_back({c, std::move(m)});
          } else {
            for (const auto& [l, ccl] : comp[c]) {
              const std::uint32_t rl = v.sranks[l];
              std::vector<double> m(std::size_t(rp) * rl, 0.0);
              for (std::uint32_t b = 0; b < rl; ++b)
                for (std::uint32_t k = 0; k < rc; ++k) {
                  const double x = ccl[k + std::size_t(b) * rc];
                  if (x == 0.0) continue;
                  for (std::uint32_t i = 0; i < rp; ++i) m[i + std::size_t(b) * rp] += mpc(i, k) * x;
                }
              comp[p].push_back({l, std::move(m)});
            }
          }
        }
      }
      // a block in new row / column orders into cgen: A(r', c') = M(oldrow(ra, r'), oldrow(cb, c'))
      auto put = [&](std::uint32_t ra, std::uint32_t cb, const std::vector<double>& m) {
        const std::uint32_t R = v.sranks[ra], K = v.sranks[cb];
        const std::uint64_t off = plan.cgen.size();
        plan.cgen.resize(off + std::uint64_t(R) * K);
        for (std::uint32_t c2 = 0; c2 < K; ++c2)
          for (std::uint32_t r2 = 0; r2 < R; ++r2)
            plan.cgen[off + r2 + std::uint64_t(c2) * R] = m[oldrow(ra, r2) + std::size_t(oldrow(cb, c2)) * R];
        return off;
      };
      cur_id.clear();
      cur_id_node0 = cur_id_node1 = kNoMap;
      // flat upward: the active internal nodes up to h_mid (all of them without one) from their
      // leaves, then those above it from the nodes at h_mid
      Phase ups[2];
      for (int st = 0; st < (h_mid ? 2 : 1); ++st) {
        Phase& up = ups[st];
        up = Phase{kPhaseUp, 0, static_cast<std::uint32_t>(plan.tasks.size()), 0, static_cast<std::uint32_t>(1 + st),
                   0.0, 0.0, 0.0};
        for (std::uint32_t p : order) {
          if (!active(p) || is_leaf(p) || (stage_mid(p) != 0) != (st == 1)) continue;
          std::vector<std::pair<std::uint32_t, std::uint64_t>> blocks;  // (frontier node, cgen offset)
          for (const auto& [f, m] : comps[st][p]) blocks.push_back({f, put(p, f, m)});
          cur_node = p;
          add_tiles(v.sranks[p], kBufT, plan.node_off[p], [&](std::uint32_t r0, std::uint32_t m) {
            for (const auto& [f, co] : blocks)
              push_seg(kGenC, false, co, v.sranks[p], v.sranks[f], m, kBufT, plan.node_off[f], f, r0, kNoMap, kNoMap, m);
          }, up);
        }
        up.task_end = static_cast<std::uint32_t>(plan.tasks.size());
      }
      // flat far+downward: every active leaf's S from the T's of the far partners on its path
      Phase down{kPhaseDown, 0, static_cast<std::uint32_t>(plan.tasks.size()), 0, 1, 0.0, 0.0, 0.0};
      for (std::uint32_t l : order) {
        if (!active(l) || !is_leaf(l)) continue;
        const std::uint32_t rl = v.sranks[l];
        std::vector<double> g(std::size_t(rl) * rl, 0.0);  // G_la, r_l x r_a, old orders
        for (std::uint32_t r = 0; r < rl; ++r) g[r + std::size_t(r) * rl] = 1.0;
        std::vector<std::pair<std::uint32_t, std::uint64_t>> blocks;  // (partner j, cgen offset)
        for (std::uint32_t a = l;;) {
          const std::uint32_t ra = v.sranks[a];
          for (std::uint64_t s : far_of[a]) {
            const std::uint32_t j = v.far_pairs[2 * s + 1], rj = v.sranks[j];
            const double* B = v.bgen + v.bptr[s];  // r_a x r_j, column major
            std::vector<double> m(std::size_t(rl) * rj, 0.0);
            for (std::uint32_t b = 0; b < rj; ++b)
              for (std::uint32_t k = 0; k < ra; ++k) {
                const double x = B[k + std::size_t(b) * ra];
                if (x == 0.0) continue;
                for (std::uint32_t i = 0; i < rl; ++i) m[i + std::size_t(b) * rl] += g[i + std::size_t(k) * rl] * x;
              }
            blocks.push_back({j, put(l, j, m)});
          }
          const std::uint32_t par = v.parent[a];
          if (par == HMXG_NO_NODE || !active(par)) break;
          const std::uint64_t off = a == v.lchild[par] ? 0 : v.sranks[v.lchild[par]];
          const std::uint32_t rp = v.sranks[par];
          std::vector<double> g2(std::size_t(rl) * rp, 0.0);  // G_l,par = G_la V_par[rows of a]
          for (std::uint32_t b = 0; b < rp; ++b)
            for (std::uint32_t k = 0; k < ra; ++k) {
              const double x = vget(par, off + k, b);
              if (x == 0.0) continue;
              for (std::uint32_t i = 0; i < rl; ++i) g2[i + std::size_t(b) * rl] += g[i + std::size_t(k) * rl] * x;
            }
          g.swap(g2);
          a = par;
        }
        cur_node = l;
        add_tiles(rl, kBufS, plan.node_off[l], [&](std::uint32_t r0, std::uint32_t m) {
          for (const auto& [j, co] : blocks)
            push_seg(kGenC, false, co, rl, v.sranks[j], m, kBufT, plan.node_off[j], j, r0, kNoMap, kNoMap, m);
        }, down);
      }
      down.task_end = static_cast<std::uint32_t>(plan.tasks.size());
      for (int st = 0; st < (h_mid ? 2 : 1); ++st)
        if (ups[st].task_end > ups[st].task_begin) plan.flat_phases.push_back(ups[st]);
      if (down.task_end > down.task_begin) plan.flat_phases.push_back(down);
      plan.flat_mid_height = h_mid;
      plan.flat = !plan.flat_phases.empty();
      plan.flat_extra_flops_per_col = flat - replaced;
    }
  }
  if (plan.segs.size() > std::numeric_limits<std::uint32_t>::max())
    return fail(err, "cds: too many GEMM segments");
  if (seg_overflow) return fail(err, "cds: a block has more than 1048560 rows in its K range");
  plan.parent.assign(nn, kNoMap);
  plan.depth.assign(nn, 0);
  for (std::uint32_t i = 0; i < nn; ++i) {
    plan.parent[i] = v.parent[i] == HMXG_NO_NODE ? kNoMap : v.parent[i];
    plan.depth[i] = v.level[i];
  }
  return true;
}

}  // namespace hmxg
