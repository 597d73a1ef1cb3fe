// ref_capi.cpp — C entry points over the UNMODIFIED reference library (hmx), compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/libhmx_ref.so.
//
// TEST INFRASTRUCTURE ONLY: the reference is the oracle the B200 evaluator is checked
// against and the CPU baseline it is timed beside. Nothing in paper_1812_07152_b200/
// links or loads this library. No reference source is copied: this file only calls the
// reference's public API (headers under /root/reference/proj/include/hmx).
//
// Entry points mirror the reference test harness:
//   hmxr_instance_new   tst::make_instance      (proj/tests/helpers.hpp:101-118)
//   hmxr_random_matrix  tst::random_matrix      (proj/tests/helpers.hpp:53-58)
//   hmxr_evaluate       hmx::evaluate           (proj/src/executor.cpp:274-302)
//   hmxr_evaluate_ref   hmx::evaluate_reference (proj/src/executor.cpp:304-403)
//   hmxr_dense_apply    hmx::dense_apply        (proj/src/executor.cpp:405-429)
//   hmxr_cds_from_view  an hmx::CDS rebuilt from a hmxg_cds_view (for CDSs produced by
//                       this repo's instance builder) so the reference can evaluate it.
//   hmxr_save_cds       hmx::save_cds    (proj/src/serial.cpp:271-277) -> `hmat.cds`
//   hmxr_load_cds       hmx::load_cds    (proj/src/serial.cpp:299-308)
//   hmxr_save_matrix    hmx::save_matrix (proj/src/serial.cpp:279-285)
//   hmxr_load_matrix    hmx::load_matrix (proj/src/serial.cpp:287-297)
#include <algorithm>
#include <chrono>
#include <vector>
#include <cstring>
#include <exception>
#include <memory>
#include <stdexcept>
#include <string>

#include "hmx/compress.hpp"
#include "hmx/executor.hpp"
#include "hmx/interaction.hpp"
#include "hmx/kernel.hpp"
#include "hmx/parallel.hpp"
#include "hmx/points.hpp"
#include "hmx/rng.hpp"
#include "hmx/sampling.hpp"
#include "hmx/serial.hpp"
#include "hmx/structure.hpp"
#include "hmx/tree.hpp"

#include "../include/hmxg.h"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::bad_alloc& e) {
    return fail(e, 3);
  } catch (const std::exception& e) {
    return fail(e, 5);
  }
}

struct RefInstance {
  hmx::PointSet pts;
  hmx::Kernel kernel;
  hmx::HTree ht;
  hmx::SampleInfo si;
  hmx::CompressedMatrix cm;
  hmx::BlockSet nbs, fbs;
  hmx::CoarsenSet cs;
  hmx::CDS cds;
  // flattened pair lists for the view
  std::vector<std::uint32_t> near_flat, far_flat;
  std::vector<std::uint8_t> part;
  double compress_seconds = 0.0;
};

void flatten(const hmx::CDS& cds, std::vector<std::uint32_t>& nf, std::vector<std::uint32_t>& ff) {
  nf.clear();
  ff.clear();
  for (const auto& [i, j] : cds.near_order) {
    nf.push_back(i);
    nf.push_back(j);
  }
  for (const auto& [i, j] : cds.far_order) {
    ff.push_back(i);
    ff.push_back(j);
  }
}

void fill_view(const hmx::CDS& cds, const std::vector<std::uint32_t>& nf,
               const std::vector<std::uint32_t>& ff, hmxg_cds_view* v) {
  std::memset(v, 0, sizeof *v);
  const auto& t = cds.tree;
  v->n = t.num_points();
  v->num_nodes = t.num_nodes;
  v->height = t.height;
  v->parent = t.parent.data();
  v->lchild = t.lchild.data();
  v->rchild = t.rchild.data();
  v->start = t.start.data();
  v->end = t.end.data();
  v->level = t.level.data();
  v->perm = t.perm.data();
  v->sranks = cds.sranks.data();
  v->participating = cds.participating.data();
  v->num_near = cds.near_order.size();
  v->near_pairs = nf.data();
  v->num_far = cds.far_order.size();
  v->far_pairs = ff.data();
  v->num_v = cds.v_order.size();
  v->v_order = cds.v_order.data();
  v->dptr = cds.dptr.data();
  v->bptr = cds.bptr.data();
  v->vptr = cds.vptr.data();
  v->dgen = cds.dgen.data();
  v->bgen = cds.bgen.data();
  v->vgen = cds.vgen.data();
}

hmx::DenseMatrix to_dense(const double* w, std::size_t n, std::size_t q) {
  hmx::DenseMatrix m(n, q);
  if (n * q) std::memcpy(m.data.data(), w, n * q * sizeof(double));
  return m;
}

hmx::EvalPlan make_plan(std::uint32_t bits, std::uint32_t p) {
  hmx::EvalPlan plan;
  plan.block_lowering_near = bits & 1u;
  plan.block_lowering_far = bits & 2u;
  plan.coarsen_lowering = bits & 4u;
  plan.peel_top = bits & 8u;
  plan.p = p == 0 ? 1 : p;
  return plan;
}

struct ViewCds {
  hmx::CDS cds;
  std::vector<std::uint32_t> near_flat, far_flat;
};

}  // namespace

extern "C" {

typedef struct hmxr_spec {
  std::uint64_t n, d;
  std::int32_t shape;   // 0 grid2d, 1 uniform_random, 2 sphere3d
  std::int32_t mode;    // 0 tau, 1 hss
  double tau;
  std::uint32_t leaf;
  std::int32_t kernel;  // 0 gaussian, 1 inverse distance
  double h;
  double bacc;
  std::uint32_t max_rank;
  std::int32_t sample_exact;
  std::uint32_t budget, knn_k, p, agg, near_bs, far_bs;
  std::uint64_t seed;
} hmxr_spec;

const char* hmxr_last_error(void) { return g_err.c_str(); }

void hmxr_spec_default(hmxr_spec* s) {
  // InstanceSpec defaults, proj/tests/helpers.hpp:81-99
  std::memset(s, 0, sizeof *s);
  s->n = 512;
  s->d = 2;
  s->shape = 1;
  s->mode = 1;
  s->tau = 0.0;
  s->leaf = 64;
  s->kernel = 0;
  s->h = 1.0;
  s->bacc = 1e-5;
  s->max_rank = 64;
  s->sample_exact = 0;
  s->budget = 128;
  s->knn_k = 16;
  s->p = 4;
  s->agg = 2;
  s->near_bs = 2;
  s->far_bs = 4;
  s->seed = 1;
}

int hmxr_instance_new(const hmxr_spec* s, void** out) {
  return guarded([&] {
    auto in = std::make_unique<RefInstance>();
    const auto shape = s->shape == 0 ? hmx::SynthShape::Grid2d
                       : s->shape == 2 ? hmx::SynthShape::Sphere3d
                                       : hmx::SynthShape::UniformRandom;
    in->pts = hmx::synth_points(shape, s->n, s->d, s->seed);
    in->kernel = s->kernel == 1 ? hmx::Kernel::inverse_distance() : hmx::Kernel::gaussian(s->h);
    hmx::ClusterTree tree = hmx::build_cluster_tree(in->pts, s->leaf, hmx::SplitMethod::Auto, s->seed);
    in->ht = hmx::compute_interactions(in->pts, tree,
                                       s->mode == 1 ? hmx::InteractionMode::Hss : hmx::InteractionMode::Tau,
                                       s->tau);
    hmx::KnnParams knn;
    knn.k = s->knn_k;
    knn.seed = s->seed;
    in->si = hmx::build_samples(in->pts, in->ht.tree, knn, s->budget,
                                s->sample_exact ? hmx::SampleMode::Exact : hmx::SampleMode::Neighbor,
                                s->seed);
    const auto tc = std::chrono::steady_clock::now();
    in->cm = hmx::compress(in->ht, in->kernel, in->pts, in->si, s->bacc, s->max_rank);
    in->compress_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - tc).count();
    in->nbs = hmx::blocking(in->ht, s->near_bs, hmx::BlockKind::Near);
    in->fbs = hmx::blocking(in->ht, s->far_bs, hmx::BlockKind::Far);
    in->cs = hmx::coarsening(in->ht.tree, hmx::srank_vector(in->cm), in->cm.participating, s->p, s->agg);
    in->cds = hmx::build_cds(in->cm, in->nbs, in->fbs, in->cs);
    in->cds.dim = static_cast<hmx::index_t>(s->d);
    flatten(in->cds, in->near_flat, in->far_flat);
    *out = in.release();
  });
}

void hmxr_instance_free(void* inst) { delete static_cast<RefInstance*>(inst); }

int hmxr_instance_view(void* inst, hmxg_cds_view* v) {
  auto* in = static_cast<RefInstance*>(inst);
  fill_view(in->cds, in->near_flat, in->far_flat, v);
  return 0;
}

int hmxr_points(void* inst, const double** coords, std::uint64_t* n, std::uint64_t* d) {
  auto* in = static_cast<RefInstance*>(inst);
  *coords = in->pts.coords.data();
  *n = in->pts.n;
  *d = in->pts.d;
  return 0;
}

int hmxr_random_matrix(std::uint64_t rows, std::uint64_t cols, std::uint64_t seed, double* out) {
  // tst::random_matrix, proj/tests/helpers.hpp:53-58
  hmx::Rng rng(hmx::mix64(seed ^ 0x9e3779b97f4a7c15ULL));
  for (std::uint64_t i = 0; i < rows * cols; ++i) out[i] = rng.uniform() * 2.0 - 1.0;
  return 0;
}

int hmxr_evaluate(void* inst, const double* w, std::uint64_t n, std::uint64_t q, double* y,
                  std::uint32_t plan_bits, std::uint32_t p, double* seconds) {
  auto* in = static_cast<RefInstance*>(inst);
  return guarded([&] {
    hmx::EvalStats st;
    const auto out = hmx::evaluate(in->cds, make_plan(plan_bits, p), to_dense(w, n, q), &st);
    if (out.data.size()) std::memcpy(y, out.data.data(), out.data.size() * sizeof(double));
    if (seconds) *seconds = st.seconds;
  });
}

int hmxr_evaluate_ref(void* inst, const double* w, std::uint64_t n, std::uint64_t q, double* y) {
  auto* in = static_cast<RefInstance*>(inst);
  return guarded([&] {
    const auto out = hmx::evaluate_reference(in->cm, to_dense(w, n, q));
    if (out.data.size()) std::memcpy(y, out.data.data(), out.data.size() * sizeof(double));
  });
}

int hmxr_dense_apply(void* inst, const double* w, std::uint64_t n, std::uint64_t q, double* y) {
  auto* in = static_cast<RefInstance*>(inst);
  return guarded([&] {
    const auto out = hmx::dense_apply(in->kernel, in->pts, to_dense(w, n, q));
    if (out.data.size()) std::memcpy(y, out.data.data(), out.data.size() * sizeof(double));
  });
}

int hmxr_relative_error_dense(void* inst, const double* w, std::uint64_t n, std::uint64_t q,
                              double* eps) {
  // acceptance criterion 1 path: relative_error(cds, kernel, points, w, Dense)
  auto* in = static_cast<RefInstance*>(inst);
  return guarded([&] {
    *eps = hmx::relative_error(in->cds, in->kernel, in->pts, to_dense(w, n, q), hmx::ErrorMode::Dense);
  });
}

int hmxr_cds_from_view(const hmxg_cds_view* v, void** out) {
  return guarded([&] {
    auto vc = std::make_unique<ViewCds>();
    hmx::CDS& c = vc->cds;
    auto& t = c.tree;
    t.num_nodes = v->num_nodes;
    t.parent.assign(v->parent, v->parent + v->num_nodes);
    t.lchild.assign(v->lchild, v->lchild + v->num_nodes);
    t.rchild.assign(v->rchild, v->rchild + v->num_nodes);
    t.start.assign(v->start, v->start + v->num_nodes);
    t.end.assign(v->end, v->end + v->num_nodes);
    t.level.assign(v->level, v->level + v->num_nodes);
    t.perm.assign(v->perm, v->perm + v->n);
    t.height = v->height;
    c.sranks.assign(v->sranks, v->sranks + v->num_nodes);
    c.participating.assign(v->participating, v->participating + v->num_nodes);
    // one row group holding one block with every pair keeps the storage order
    // (BlockSet::flat_pairs, structure.cpp:21-27)
    auto one_block = [](const std::uint32_t* pairs, std::uint64_t cnt, hmx::BlockKind kind) {
      hmx::BlockSet bs;
      bs.kind = kind;
      bs.blocksize = 1;
      if (cnt) {
        hmx::BlockRowGroup g;
        hmx::InteractionBlock b;
        for (std::uint64_t s = 0; s < cnt; ++s) b.pairs.emplace_back(pairs[2 * s], pairs[2 * s + 1]);
        g.blocks.push_back(std::move(b));
        bs.groups.push_back(std::move(g));
      }
      return bs;
    };
    c.near_bs = one_block(v->near_pairs, v->num_near, hmx::BlockKind::Near);
    c.far_bs = one_block(v->far_pairs, v->num_far, hmx::BlockKind::Far);
    hmx::CoarsenLevel lvl;
    hmx::SubTree st;
    st.nodes.assign(v->v_order, v->v_order + v->num_v);
    lvl.subtrees.push_back(std::move(st));
    c.coarsenset.levels.push_back(std::move(lvl));
    c.rebuild_order();
    c.dptr.assign(v->dptr, v->dptr + v->num_near + 1);
    c.bptr.assign(v->bptr, v->bptr + v->num_far + 1);
    c.vptr.assign(v->vptr, v->vptr + v->num_v + 1);
    c.dgen.assign(v->dgen, v->dgen + v->dptr[v->num_near]);
    c.bgen.assign(v->bgen, v->bgen + v->bptr[v->num_far]);
    c.vgen.assign(v->vgen, v->vgen + v->vptr[v->num_v]);
    flatten(c, vc->near_flat, vc->far_flat);
    *out = vc.release();
  });
}

void hmxr_cds_free(void* cds) { delete static_cast<ViewCds*>(cds); }

int hmxr_cds_evaluate(void* cds, const double* w, std::uint64_t n, std::uint64_t q, double* y,
                      std::uint32_t plan_bits, std::uint32_t p, double* seconds) {
  auto* vc = static_cast<ViewCds*>(cds);
  return guarded([&] {
    // the rebuilt CDS carries a single coarsen level in post-order; the depth schedule
    // (coarsen lowering off) is used unless the caller asks otherwise
    hmx::EvalStats st;
    const auto out = hmx::evaluate(vc->cds, make_plan(plan_bits, p), to_dense(w, n, q), &st);
    if (out.data.size()) std::memcpy(y, out.data.data(), out.data.size() * sizeof(double));
    if (seconds) *seconds = st.seconds;
  });
}

int hmxr_save_cds(void* inst, const char* path) {
  auto* in = static_cast<RefInstance*>(inst);
  return guarded([&] { hmx::save_cds(path, in->cds); });
}

int hmxr_cds_save(void* cds, const char* path) {
  return guarded([&] { hmx::save_cds(path, static_cast<ViewCds*>(cds)->cds); });
}

int hmxr_load_cds(const char* path, void** out) {
  return guarded([&] {
    auto vc = std::make_unique<ViewCds>();
    vc->cds = hmx::load_cds(path);
    flatten(vc->cds, vc->near_flat, vc->far_flat);
    *out = vc.release();
  });
}

int hmxr_cds_view(void* cds, hmxg_cds_view* v) {
  auto* vc = static_cast<ViewCds*>(cds);
  fill_view(vc->cds, vc->near_flat, vc->far_flat, v);
  return 0;
}

int hmxr_save_matrix(const char* path, const double* data, std::uint64_t rows, std::uint64_t cols) {
  return guarded([&] { hmx::save_matrix(path, to_dense(data, rows, cols)); });
}

// rows/cols of the file in *rows/*cols; data copied to out when out != nullptr
int hmxr_load_matrix(const char* path, double* out, std::uint64_t* rows, std::uint64_t* cols) {
  return guarded([&] {
    const auto m = hmx::load_matrix(path);
    *rows = m.rows;
    *cols = m.cols;
    if (out && m.data.size()) std::memcpy(out, m.data.data(), m.data.size() * sizeof(double));
  });
}

// hmx::relative_error_vs (executor.cpp:431-476) of a given approximation, mode 0 dense /
// 1 sampled; status 6 = numeric_guard_error.
int hmxr_relative_error_vs(void* inst, const double* ya, const double* w, std::uint64_t n, std::uint64_t q,
                           std::int32_t mode, std::uint64_t seed, double* eps) {
  auto* in = static_cast<RefInstance*>(inst);
  try {
    *eps = hmx::relative_error_vs(to_dense(ya, n, q), in->kernel, in->pts, to_dense(w, n, q),
                                  mode == 0 ? hmx::ErrorMode::Dense : hmx::ErrorMode::Sampled, seed);
    return 0;
  } catch (const hmx::numeric_guard_error& e) {
    return fail(e, 6);
  } catch (const std::exception& e) {
    return fail(e, 5);
  }
}

// hmx::dense_apply over any point set (kernel 0 gaussian(h), 1 inverse distance).
int hmxr_dense_apply_points(const double* coords, std::uint64_t n, std::uint64_t d, std::int32_t kernel, double h,
                            const double* w, std::uint64_t q, double* y) {
  return guarded([&] {
    hmx::PointSet pts;
    pts.n = n;
    pts.d = d;
    pts.coords.assign(coords, coords + n * d);
    const hmx::Kernel k = kernel == 1 ? hmx::Kernel::inverse_distance() : hmx::Kernel::gaussian(h);
    const auto out = hmx::dense_apply(k, pts, to_dense(w, n, q));
    if (out.data.size()) std::memcpy(y, out.data.data(), out.data.size() * sizeof(double));
  });
}

// The sampled rows of relative_error_vs (executor.cpp:446-451) drawn with the reference Rng.
std::uint64_t hmxr_sample_rows(std::uint64_t n, std::uint64_t seed, std::uint32_t* rows) {
  const std::uint64_t nr = std::min<std::uint64_t>(n, 256);
  std::vector<std::uint32_t> all(n);
  for (std::uint64_t i = 0; i < n; ++i) all[i] = static_cast<std::uint32_t>(i);
  hmx::Rng rng(hmx::mix64(seed ^ hmx::mix64(0xe44a11ULL)));
  for (std::uint64_t i = 0; i < nr; ++i) std::swap(all[i], all[i + rng.below(n - i)]);
  std::copy(all.begin(), all.begin() + nr, rows);
  return nr;
}

// The compression inputs and outputs of a reference instance (compress.cpp:102-148):
// sample rows per node as CSR, and each node's basis (srank, skeleton, V rows x srank).
int hmxr_samples(void* inst, std::uint64_t* ptr, std::uint32_t* idx) {
  auto* in = static_cast<RefInstance*>(inst);
  std::uint64_t off = 0;
  for (std::size_t node = 0; node < in->si.rows.size(); ++node) {
    if (ptr) ptr[node] = off;
    if (idx) std::copy(in->si.rows[node].begin(), in->si.rows[node].end(), idx + off);
    off += in->si.rows[node].size();
  }
  if (ptr) ptr[in->si.rows.size()] = off;
  return 0;
}

int hmxr_basis(void* inst, std::uint32_t node, std::uint32_t* srank, std::uint64_t* rows, std::uint32_t* skel,
               double* v) {
  auto* in = static_cast<RefInstance*>(inst);
  if (node >= in->cm.bases.size()) return 1;
  const auto& b = in->cm.bases[node];
  *srank = b.srank;
  *rows = b.v.rows;
  if (skel) std::copy(b.skeleton.begin(), b.skeleton.end(), skel);
  if (v && b.v.data.size()) std::memcpy(v, b.v.data.data(), b.v.data.size() * sizeof(double));
  return 0;
}

double hmxr_compress_seconds(void* inst) { return static_cast<RefInstance*>(inst)->compress_seconds; }

// The bases part of hmx::compress alone (compress.cpp:113-146: per participating node,
// deepest level first, the sampled block through hmx::dense_block and the reference's
// interpolative_decomposition), timed on one host thread: the like-for-like CPU figure for
// the GPU's hmxg_compress, which computes the bases only. Returns seconds (< 0: failure);
// *rank_sum gets the sum of the sranks (the same as the instance's bases).
double hmxr_bases_seconds(void* inst, std::uint64_t* rank_sum) {
  auto* in = static_cast<RefInstance*>(inst);
  double secs = -1.0;
  guarded([&] {
    const auto& tree = in->ht.tree;
    std::vector<std::vector<hmx::index_t>> by_level(tree.height + 1);
    for (hmx::index_t i = 0; i < tree.num_nodes; ++i)
      if (in->cm.participating[i]) by_level[tree.level[i]].push_back(i);
    std::vector<std::vector<hmx::index_t>> skel(tree.num_nodes);
    std::uint64_t rs = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (auto lvl = by_level.size(); lvl-- > 0;)
      for (hmx::index_t node : by_level[lvl]) {
        std::vector<hmx::index_t> cols;
        if (tree.is_leaf(node)) {
          const auto members = tree.node_points(node);
          cols.assign(members.begin(), members.end());
        } else {
          cols = skel[tree.lchild[node]];
          cols.insert(cols.end(), skel[tree.rchild[node]].begin(), skel[tree.rchild[node]].end());
        }
        if (cols.empty()) continue;
        const hmx::DenseMatrix block = hmx::dense_block(in->kernel, in->pts, in->si.rows[node], cols);
        const hmx::IdResult id = hmx::interpolative_decomposition(block, in->cm.bacc, in->cm.max_rank);
        for (hmx::index_t local : id.skeleton) skel[node].push_back(cols[local]);
        rs += id.srank;
      }
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (rank_sum) *rank_sum = rs;
  });
  return secs;
}

// hmx::generate_plan (executor.cpp:259-272) over the instance's own tree, blocks and
// coarsening with p workers: the stock plan, as lowering bits for hmxr_evaluate.
int hmxr_generate_plan(void* inst, std::uint32_t p, std::uint32_t* bits) {
  auto* in = static_cast<RefInstance*>(inst);
  return guarded([&] {
    hmx::PlanDefaults d;
    d.p = p;
    const hmx::EvalPlan plan = hmx::generate_plan(in->ht.tree, in->nbs, in->fbs, in->cs, d);
    *bits = (plan.block_lowering_near ? 1u : 0u) | (plan.block_lowering_far ? 2u : 0u) |
            (plan.coarsen_lowering ? 4u : 0u) | (plan.peel_top ? 8u : 0u);
  });
}

// The reference RNG primitives, so the CLI's random W (hmx.cpp:117-122) can be pinned.
std::uint64_t hmxr_mix64(std::uint64_t x) { return hmx::mix64(x); }

void hmxr_rng_fill_pm1(std::uint64_t state_seed, std::uint64_t count, double* out) {
  hmx::Rng rng(state_seed);
  for (std::uint64_t i = 0; i < count; ++i) out[i] = rng.uniform() * 2.0 - 1.0;
}

unsigned hmxr_hardware_workers(void) { return hmx::default_worker_count(); }

}  // extern "C"
