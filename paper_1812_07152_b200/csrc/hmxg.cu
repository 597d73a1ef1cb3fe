// hmxg.cu — C-ABI of the B200 evaluator (include/hmxg.h): device residency of the CDS,
// workspace management, column sharding over devices, the launch sequence and the
// pipelined host<->device path.
#include <cuda.h>
#include <cuda_runtime.h>

#include <emmintrin.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/hmxg.h"
#include "kernels.cuh"
#include "plan.hpp"
#include "runtime.hpp"

namespace hmxg {
namespace {

// The GEMM B operand: boxes of 16 rows x kBPitch columns of a point-major buffer in the
// column-block layout (phys_col), zero fill past the last block.
int make_map(CUtensorMap* map, const double* base, std::uint64_t rows, std::uint64_t q, std::uint64_t ld) {
  return make_map_box(map, base, rows, phys_cols(q), ld, kBPitch, kBK);
}

// Columns per pipeline chunk of the host-pointer path: H2D of chunk k+1 and D2H of chunk
// k-1 overlap the evaluation of chunk k. When PCIe bounds the pipeline (cfg5-HSS), 64: a
// wider chunk only lengthens the unhidden first copy-in and last copy-out. When the
// evaluation does (its executed FP64 work at ~30 TF/s is over twice the W and Y bytes at
// ~45 GB/s per direction), each chunk also pays a fixed cost c of about 0.4 ms (the top
// of the tree and the launches: measured 0.3-0.45 ms on cfg3-cfg5-H2-b), and the width
// balances the two: w* = sqrt(Q c 45e9 / (16 n)), rounded to 64 x a power of two, at most
// 256. Measured e2e: cfg3 35.8 -> 33.6 ms (w 128), cfg5-H2-b 299 -> 296 ms (w 128); cfg4
// stays at 64 (w 256 cost +4%).
constexpr std::size_t kChunkCols = 64;
std::size_t host_chunk_cols(const Plan& plan, std::size_t qg) {
#ifndef HMXG_HOST_CHUNK_ADAPTIVE
#define HMXG_HOST_CHUNK_ADAPTIVE 1
#endif
  if (!HMXG_HOST_CHUNK_ADAPTIVE) return std::min(qg, kChunkCols);
  double flops_per_col = 0.0;
  for (const Phase& ph : plan.phases) flops_per_col += ph.flops_per_col;
  const double bw = 45e9, per_chunk = 0.4e-3;
  const double compute = flops_per_col / 30e12, transfer = 8.0 * double(plan.n) / bw;  // per column
  if (compute < 2.0 * transfer) return std::min(qg, kChunkCols);
  const double w = std::sqrt(double(qg) * per_chunk * bw / (16.0 * double(plan.n)));
  std::size_t cols = kChunkCols;
  while (cols < 4 * kChunkCols && w > 1.41421356 * cols) cols *= 2;  // nearest power of two
  return std::min(qg, cols);
}

struct DevState {
  int dev = 0;
  cudaStream_t comp = nullptr, h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> phase_ev;  // launches + 1
  bool phase_valid = false;
  double* tiles = nullptr;  // pre-tiled A operands
  std::uint64_t tile_elems = 0;
  Task* tasks = nullptr;
  SegDev* segs = nullptr;
  std::uint32_t* ipmap = nullptr;
  std::uint32_t* idmap = nullptr;  // identity-row sources of the tasks (Plan::idmap)
  std::size_t cap_q = 0;  // row pitch of Wp/T/S/Yp in physical columns (phys_cols of the capacity)
  double* wp = nullptr;
  double* yp = nullptr;
  double* t = nullptr;
  double* s = nullptr;
  std::size_t stage_q = 0;  // host-path staging capacity (columns per buffer)
  double* w_stage[2] = {nullptr, nullptr};
  double* y_stage[2] = {nullptr, nullptr};
  // pageable host W / Y (bounce path): pinned host staging of the same chunks
  std::size_t pin_q = 0;
  double* w_pin[2] = {nullptr, nullptr};
  double* y_pin[2] = {nullptr, nullptr};
  std::uint64_t resident_bytes = 0;
  std::uint32_t* tile_counters = nullptr;  // one per GEMM launch, zeroed per evaluation
  // whole-evaluation DAG launch: work items (built per column count) and counters
  struct DagItems {
    std::size_t q = 0;
    std::uint32_t nitems = 0;
    // the claim order as the kernel reads it: one record per task run (DagParams::recs), each
    // run per_task = column blocks x parts consecutive items
    RingSlot* recs = nullptr;
    std::uint32_t per_task = 1, parts = 1;
    std::uint32_t stage = 0;
    bool ct = false;  // CTree mode (near tiles only): the mode can change with the environment
    // the slot holds a built list; the list itself can be empty (recs == nullptr): a tree
    // without levels whose near field is generated on the fly has nothing for the DAG
    bool valid = false;
  };
  DagItems dag[4];                    // item lists of the last few (column count, stage) keys
  std::uint32_t dag_next = 0;
  std::uint32_t* dag_done = nullptr;  // claim counter + done counters (sized for the largest q)
  std::size_t dag_done_cap = 0;
  std::uint32_t* node_tiles = nullptr;
  std::uint32_t* yp_tiles = nullptr;
  // fused permutations (small problems, see fused_io): padded row -> point, and the leaf jobs
  std::uint32_t* pmap = nullptr;
  // host staging of host-buffer collectives (hmxg_comm::host_buffers)
  unsigned char* comm_host = nullptr;
  std::size_t comm_host_bytes = 0;
  // on-the-fly near field (Plan::near_otf): the points, the kernel, every wave's near chunks
  // (GenChunk, concatenated) and the waves of leaf tasks whose chunks fit the scratch region
  double* pts = nullptr;
  KernelParams kp{};
  GenChunk* gen_chunks = nullptr;
  struct Wave {
    std::uint32_t t0, t1;  // leaf tasks
    std::uint64_t c0, c1;  // their chunks in gen_chunks
  };
  std::vector<Wave> waves;
  std::vector<SegDev> otf_segs;  // host copy of the device's segment table (its tile offsets differ from the plan's)
  std::vector<double> wave_flops, wave_io;  // per wave: executed flops and B/C bytes per column
  // the last evaluation's launch sequence (hmxg_phase_count / hmxg_phase_get)
  struct LaunchDesc {
    std::uint32_t kind, level, tiles;
    double flops_per_col, gen_bytes, io_bytes_per_col;
  };
  std::vector<LaunchDesc> launch_desc, gdesc;  // (gdesc: the cached graph's)
  // CTree program (ctree_csize): work units by level, built on first use
  unsigned char* ct_blob = nullptr;  // tasks, then segments at ct_segs_off
  std::uint32_t* ct_units = nullptr;
  std::uint32_t* ct_lvl = nullptr;
  std::uint32_t ct_nlev = 0, ct_blob_bytes = 0, ct_segs_off = 0;
  std::uint64_t ct_tile_base = 0, ct_tile_lines = 0;
  int ct_occ_c = 0;          // cluster size of the cached occupancy
  unsigned ct_occ_ctas = 0;  // resident CTAs of eval_dag<true> in clusters of ct_occ_c
  std::uint32_t* rowleaf = nullptr;    // Wp row -> leaf node
  std::uint32_t* wp_target = nullptr;  // leaf node -> rows
  // an enqueue failed between eval_dag and the launch that zeroes its counters: zero them first
  bool counters_dirty = false;
  bool last_fused = false;  // the last evaluation ran the single fused launch
  std::uint32_t last_launches = 3;
  std::uint32_t* remote_t = nullptr;  // split mode: nodes whose T comes from the exchange
  // HMXG_POISON=1 (debug): live T/S rows, NaN-filled with Wp and Yp before every evaluation
  bool poison = false;
  std::uint32_t* ts_live = nullptr;
  std::uint64_t ts_live_count = 0;
  // CUDA graph of the whole launch sequence for one (W, Y, q, ld, stream, workspace) key:
  // repeated device-pointer evaluations replay it instead of issuing ~2H+4 launches.
  struct GraphKey {
    const double* w = nullptr;
    double* y = nullptr;
    std::size_t q = 0, ldw = 0, ldy = 0;
    cudaStream_t st = nullptr;
    const double* wp = nullptr;
    const void* items = nullptr;  // the DAG claim-order records and counters the graph reads
    const std::uint32_t* dag_done = nullptr;
    bool levels = false;
    bool timed = false;  // captured with per-launch event nodes (and without programmatic launch)
    bool operator==(const GraphKey& o) const {
      return w == o.w && y == o.y && q == o.q && ldw == o.ldw && ldy == o.ldy && st == o.st && wp == o.wp &&
             items == o.items && dag_done == o.dag_done && levels == o.levels && timed == o.timed;
    }
  } gkey;
  cudaGraphExec_t gexec = nullptr;
  // Ordering between calls: every call shares the workspace (Wp, T, S, Yp, the DAG counters).
  // A device-pointer call may return before its work is done (HMXG_F_NO_SYNC); ev_last marks
  // the end of its work on its stream, and the next call, on whatever stream, waits for it.
  cudaEvent_t ev_last = nullptr;
  bool pending = false;
  bool last_levels = false;  // launch sequence of the last evaluation (phase reporting)
  std::size_t last_q = 0;    // its column count (per device shard)
  std::uint32_t glaunches = 0;
  bool gfused = false;  // the cached graph is the fused single launch
  unsigned gemm_grid = 0;                   // resident CTAs of the persistent GEMM

  void drop_graph() {
    if (gexec) cudaGraphExecDestroy(gexec);
    gexec = nullptr;
    gkey = GraphKey{};
  }
  void release_workspace() {
    drop_graph();
    cudaFree(wp);
    cudaFree(yp);
    cudaFree(t);
    cudaFree(s);
    wp = yp = t = s = nullptr;
    cap_q = 0;
  }
  void release_stage() {
    for (int b = 0; b < 2; ++b) {
      cudaFree(w_stage[b]);
      cudaFree(y_stage[b]);
      w_stage[b] = y_stage[b] = nullptr;
    }
    stage_q = 0;
  }
  void release_pinned() {
    for (int b = 0; b < 2; ++b) {
      cudaFreeHost(w_pin[b]);
      cudaFreeHost(y_pin[b]);
      w_pin[b] = y_pin[b] = nullptr;
    }
    pin_q = 0;
  }
  void release() {
    if (cudaSetDevice(dev) != cudaSuccess) return;
    for (cudaStream_t st : {comp, h2d, d2h})
      if (st) cudaStreamSynchronize(st);
    release_workspace();
    release_stage();
    release_pinned();
    cudaFree(tiles);
    cudaFree(tile_counters);
    tile_counters = nullptr;
    for (auto& e : dag) {
      cudaFree(e.recs);
      e = DagItems{};
    }
    cudaFree(dag_done);
    cudaFree(node_tiles);
    cudaFree(yp_tiles);
    yp_tiles = nullptr;
    cudaFree(remote_t);
    remote_t = nullptr;
    cudaFree(ts_live);
    ts_live = nullptr;
    cudaFree(pmap);
    pmap = nullptr;
    cudaFree(rowleaf);
    rowleaf = nullptr;
    cudaFree(ct_units);
    cudaFree(ct_lvl);
    cudaFree(ct_blob);
    ct_units = ct_lvl = nullptr;
    ct_blob = nullptr;
    cudaFree(pts);
    cudaFree(gen_chunks);
    pts = nullptr;
    gen_chunks = nullptr;
    waves.clear();
    ct_nlev = 0;
    cudaFreeHost(comm_host);
    comm_host = nullptr;
    comm_host_bytes = 0;
    cudaFree(wp_target);
    wp_target = nullptr;
    dag_done = nullptr;
    dag_done_cap = 0;
    node_tiles = nullptr;
    cudaFree(tasks);
    cudaFree(segs);
    cudaFree(ipmap);
    cudaFree(idmap);
    idmap = nullptr;
    tiles = nullptr;
    tasks = nullptr;
    segs = nullptr;
    ipmap = nullptr;
    for (cudaEvent_t* e : {&ev0, &ev1, &ev_in[0], &ev_in[1], &ev_done[0], &ev_done[1], &ev_out[0], &ev_out[1], &ev_last})
      if (*e) cudaEventDestroy(*e), *e = nullptr;
    for (auto& e : phase_ev) cudaEventDestroy(e);
    phase_ev.clear();
    for (cudaStream_t* st : {&comp, &h2d, &d2h})
      if (*st) cudaStreamDestroy(*st), *st = nullptr;
  }
};

}  // namespace
}  // namespace hmxg

struct hmxg_mat {
  hmxg_ctx* ctx = nullptr;
  hmxg::Plan plan;
  std::vector<hmxg::DevState> devs;
  std::mutex mu;  // one in-flight evaluate per matrix
};

namespace hmxg {
namespace {

// Wp/Yp/T/S are point-major with a row pitch of cap_q physical columns: the column blocks
// of q columns at kCbPitch (phys_cols(q), a multiple of 16: 128-byte aligned rows).
int ensure_workspace(const Plan& plan, DevState& d, std::size_t q) {
  q = phys_cols(q);
  if (q <= d.cap_q) return HMXG_OK;
  HMXG_CUDA(cudaDeviceSynchronize());  // an earlier asynchronous call may still use the buffers
  d.pending = false;
  d.release_workspace();
  const std::size_t n = plan.rows_pad, r = plan.skel_rows;
  HMXG_CUDA(cudaMalloc(&d.wp, n * q * sizeof(double)));
  HMXG_CUDA(cudaMalloc(&d.yp, n * q * sizeof(double)));
  HMXG_CUDA(cudaMalloc(&d.t, r * q * sizeof(double)));
  HMXG_CUDA(cudaMalloc(&d.s, r * q * sizeof(double)));
  // pad rows of Wp/T/S are read as zeros by the 16-row B chunks and never written
  HMXG_CUDA(cudaMemset(d.wp, 0, n * q * sizeof(double)));
  HMXG_CUDA(cudaMemset(d.t, 0, r * q * sizeof(double)));
  HMXG_CUDA(cudaMemset(d.s, 0, r * q * sizeof(double)));
  // cudaMemset runs on the legacy stream, which does not order the non-blocking streams
  // the evaluation is enqueued on: finish it before any kernel can touch the buffers
  HMXG_CUDA(cudaDeviceSynchronize());
  d.cap_q = q;
  return HMXG_OK;
}

int ensure_stage(const Plan& plan, DevState& d, std::size_t q) {
  if (q <= d.stage_q) return HMXG_OK;
  d.release_stage();
  for (int b = 0; b < 2; ++b) {
    HMXG_CUDA(cudaMalloc(&d.w_stage[b], plan.n * q * sizeof(double)));
    HMXG_CUDA(cudaMalloc(&d.y_stage[b], plan.n * q * sizeof(double)));
  }
  d.stage_q = q;
  return HMXG_OK;
}

// Work items of the whole-evaluation DAG launch for q columns, in topological order:
// within a phase, row tiles in task order with the column block fastest (so a row tile's A
// chunks are re-served from L2 to all column blocks).
// When the tree levels are too narrow to keep every CTA busy, the split leaf variant is
// used: its near phase depends on Wp only, so its items are dealt out in equal slices
// after every tree level but the first (CTAs that would wait for the next level pick up
// near-field tiles instead), and the accumulating leaf phase comes last. Otherwise the Yp
// round trip of the split costs more than the idle slots it fills, and the combined leaf
// tasks run. The criterion is work items per CTA of the combined variant (measured:
// cfg1 Q=64, 0.4 per CTA, and cfg2 Q=256, 32: split faster; cfg5-HSS Q=256, 83: combined
// 1.81 vs 1.89 ms; Q=2048, 660: combined, split +11%). Both variants give the same bits.
#ifndef HMXG_SPLIT_LEAF_MAX_ITEMS_PER_CTA
#define HMXG_SPLIT_LEAF_MAX_ITEMS_PER_CTA 48
#endif
// The plan options of a replicated upload (HMXG_NO_FLAT=1: no flat tree, see Plan::flat_phases).
SplitSpec plan_spec() {
  SplitSpec s;
  s.flat_tree = std::getenv("HMXG_NO_FLAT") == nullptr;
  return s;
}
// The tree phases an evaluation runs, in order: the upward and far+downward phases, or, for a
// flat tree (Plan::flat_phases, small trees), the leaf upward phase and the two flat phases.
std::vector<const Phase*> tree_phases(const Plan& plan, std::uint32_t stage) {
  std::vector<const Phase*> out;
  for (const Phase& ph : plan.phases)
    if (ph.stage == stage && ph.kind != kPhaseLeaf && (!plan.flat || (ph.kind == kPhaseUp && ph.level == 0)))
      out.push_back(&ph);
  if (plan.flat && stage == 0)
    for (const Phase& ph : plan.flat_phases) out.push_back(&ph);
  return out;
}
std::uint32_t ctree_csize(const Plan& plan, std::size_t q, unsigned grid);
bool split_leaf(const Plan& plan, std::size_t q, unsigned grid) {
  if (plan.split_phases.empty() || plan.near_otf) return false;  // on-the-fly near field: combined tasks
  if (ctree_csize(plan, q, grid)) return true;  // the CTree's leaf rows accumulate onto the near tiles
  std::uint64_t tasks = 0;
  for (const Phase& ph : plan.phases) tasks += ph.task_end - ph.task_begin;
  return tasks * ((q + kBN - 1) / kBN) < std::uint64_t(HMXG_SPLIT_LEAF_MAX_ITEMS_PER_CTA) * grid;
}
// The level-by-level launch sequence for q columns (HMXG_F_LEVEL_LAUNCHES): the same leaf
// variant as the DAG launch, so both give the same bits.
std::vector<const Phase*> level_phases(const Plan& plan, std::size_t q, unsigned grid) {
  std::vector<const Phase*> out = tree_phases(plan, 0);
  const bool split = split_leaf(plan, q, grid);
  if (!split)
    for (const Phase& ph : plan.phases)
      if (ph.kind == kPhaseLeaf) out.push_back(&ph);
  if (split)
    for (const Phase& ph : plan.split_phases) out.push_back(&ph);
  return out;
}
// Column-split parts per tile for narrow DAGs (DagParams::colsplit): with fewer work items
// than resident CTAs the dependency chain of small GEMMs is DMMA-time bound on one SM per
// tile, so each tile's 64 columns become 4 (or 2) items on different SMs. Wide DAGs keep
// whole tiles: the split re-reads every A chunk per part. HMXG_COLSPLIT overrides (1, 2, 4).
std::uint32_t colsplit(const Plan& plan, std::size_t q, unsigned grid, std::uint32_t stage = 0) {
  if (stage != 0 || plan.nparts != 1) return 1;
  if (const char* e = std::getenv("HMXG_COLSPLIT")) {
    const int v = std::atoi(e);
    return v == 2 || v == 4 ? static_cast<std::uint32_t>(v) : 1u;
  }
  std::uint64_t tasks = 0;
  for (const Phase& ph : plan.phases) tasks += ph.task_end - ph.task_begin;
  const std::uint64_t items = tasks * ((q + kBN - 1) / kBN);
  return items < grid ? 4u : (items < 4ull * grid ? 2u : 1u);
}
// Partial split of the leaf rows (wide DAGs): the near field of a fraction f of the leaves runs
// as split-variant near items dealt out between the tree levels -- they depend on Wp only, so
// they fill the slots the narrow upper levels leave idle -- and those leaves' V_i S_i rows
// accumulate onto them at the end; the other leaves keep the combined tasks (no Yp round
// trip). f = 1 is the split variant of narrow DAGs (split_leaf), f = 0 the combined one. Both
// variants sum every row in one order, so any f gives the same bits. HMXG_SPLIT_FRAC sets f.
#ifndef HMXG_SPLIT_FRAC
#define HMXG_SPLIT_FRAC 0.0
#endif
// Default f by work items per CTA of the combined variant (below 48 the whole split variant
// runs): measured on cfg5-HSS, the 8-GPU sweep's per-rank workloads -- Q=256 (83 items per
// CTA) 2.189 -> 2.162 ms at f = 0.2-0.35, Q=512 (165) 4.232 -> 4.219 ms at f = 0.2, Q=1024
// (330) and Q=2048 best at 0 (profiles/r02/split_frac_sweep.txt): f = 0.3 (1 - items / 250).
double split_frac(const Plan& plan, std::size_t q, unsigned grid) {
  if (plan.split_phases.empty() || plan.near_otf || plan.nparts != 1) return 0.0;
  if (split_leaf(plan, q, grid)) return 1.0;
  std::uint64_t tasks = 0;
  for (const Phase& ph : plan.phases) tasks += ph.task_end - ph.task_begin;
  const double per_cta = double(tasks) * double((q + kBN - 1) / kBN) / std::max(1u, grid);
  double f = HMXG_SPLIT_FRAC > 0.0 ? HMXG_SPLIT_FRAC : std::max(0.0, 0.3 * (1.0 - per_cta / 250.0));
  if (const char* e = std::getenv("HMXG_SPLIT_FRAC")) f = std::atof(e);
  return std::min(1.0, std::max(0.0, f));
}
// Leaves whose rows run split for fraction f: among the leaves with near tiles and a basis
// (those with an accumulating task), evenly spaced in task order.
std::vector<std::uint8_t> split_set(const Plan& plan, double f) {
  std::vector<std::uint8_t> sel(plan.num_nodes, 0);
  if (f <= 0.0) return sel;
  std::vector<std::uint32_t> cand;
  for (const Phase& ph : plan.split_phases)
    if (ph.kind == kPhaseLeaf && ph.stage == 0)
      for (std::uint32_t t = ph.task_begin; t < ph.task_end; ++t)
        if ((plan.tasks[t].flags & kTaskAccumulate) && (cand.empty() || cand.back() != plan.tasks[t].node))
          cand.push_back(plan.tasks[t].node);
  for (std::size_t k = 0; k < cand.size(); ++k)
    if (f >= 1.0 || std::floor((k + 1) * f) > std::floor(k * f)) sel[cand[k]] = 1;
  return sel;
}
// Subtree-pipelined claim order (wide DAGs that run the combined leaf tasks). The far+downward
// levels next to the leaves are bound by HBM, not by the FP64 pipe -- their items are a few
// chunks of K, mostly row traffic of T and S, which do not fit in L2 (cfg5-HSS: L8-L10 at 22-26
// TF/s, within ~25% of their T/S bytes at HBM speed) -- while the leaf rows are bound by the FP64
// pipe with HBM mostly idle. Level by level the two kinds never meet. The nodes below depth d0
// are therefore grouped by their ancestor at depth d0 and the groups pipelined: the
// far+downward levels of group g are interleaved (by estimated work, task by task, so a task's
// column blocks stay consecutive and reuse its A chunks from L2) with the leaf rows of group
// g-1; the upward pass and the levels above d0 run level by level as before. Every sequence
// keeps its own level order and everything an item reads is emitted before it, so the order
// stays topological (hmxg_dag_check) and the results are the same bits.
// Measured (cfg5-HSS eval_dag, tools/pipe_check.py): Q=2048 13.43 -> 13.32 ms at d0 = 2 (13.34
// at 3, 13.39 at 4), Q=1536 10.09 -> 10.05, Q=1024 6.79 -> 6.81 (below the threshold now); the
// H2-b configs unchanged. The same pipelining of the upward levels with the next group's
// leaf-upward tasks lost (13.45 at d0 = 2, 13.54 at 4: both sides read HBM heavily) and was
// dropped. Returns d0, or 0 for the level-major order. HMXG_PIPE sets d0 (0: off),
// HMXG_PIPE_MIN the work items per CTA from which the order applies (tests).
#ifndef HMXG_PIPE_DEPTH
#define HMXG_PIPE_DEPTH 2
#endif
#ifndef HMXG_PIPE_MIN_ITEMS_PER_CTA
#define HMXG_PIPE_MIN_ITEMS_PER_CTA 450
#endif
std::uint32_t pipe_depth(const Plan& plan, std::size_t q, unsigned grid, std::uint32_t stage) {
  if (stage != 0 || plan.nparts != 1 || plan.flat || plan.near_otf || plan.depth.empty()) return 0;
  std::uint32_t d0 = HMXG_PIPE_DEPTH;
  if (const char* e = std::getenv("HMXG_PIPE")) d0 = static_cast<std::uint32_t>(std::max(0, std::min(16, std::atoi(e))));
  if (d0 == 0 || split_frac(plan, q, grid) > 0.0) return 0;
  std::uint64_t tasks = 0;
  for (const Phase& ph : plan.phases) tasks += ph.task_end - ph.task_begin;
  std::uint64_t min_per_cta = HMXG_PIPE_MIN_ITEMS_PER_CTA;
  if (const char* e = std::getenv("HMXG_PIPE_MIN")) min_per_cta = static_cast<std::uint64_t>(std::max(0, std::atoi(e)));
  if (tasks * ((q + kBN - 1) / kBN) < min_per_cta * grid) return 0;
  std::uint32_t height = 0;
  for (std::uint32_t d : plan.depth) height = std::max(height, d);
  return height >= d0 + 3 ? d0 : 0;  // at least three levels inside a group
}

std::vector<std::uint64_t> build_items(const Plan& plan, std::uint32_t q, std::uint32_t stage, unsigned grid) {
  const std::uint32_t ncb = (q + kBN - 1) / kBN;
  const std::uint32_t S = colsplit(plan, q, grid, stage);
  std::vector<std::uint64_t> items;
  auto emit_task = [&](std::uint32_t t) {
    for (std::uint32_t cb = 0; cb < ncb; ++cb)
      for (std::uint32_t sub = 0; sub < S; ++sub) items.push_back(make_item(kItemGemm, cb, t, sub));
  };
  auto emit = [&](std::uint32_t t0, std::uint32_t t1) {
    for (std::uint32_t t = t0; t < t1; ++t) emit_task(t);
  };
  if (stage == 0 && ctree_csize(plan, q, grid)) {  // CTree mode: the near tiles only
    for (const Phase& ph : plan.split_phases)
      if (ph.kind == kPhaseNear) emit(ph.task_begin, ph.task_end);
    return items;
  }
  const double f = stage == 0 ? split_frac(plan, q, grid) : (split_leaf(plan, q, grid) ? 1.0 : 0.0);
  if (const std::uint32_t d0 = S == 1 ? pipe_depth(plan, q, grid, stage) : 0) {
    // group of a node: its ancestor at depth d0 (nodes come parents first); kNoMap: above d0
    std::vector<std::uint32_t> grp(plan.num_nodes, kNoMap);
    std::uint32_t G = 0;
    for (std::uint32_t i = 0; i < plan.num_nodes; ++i) {
      if (plan.depth[i] == d0) grp[i] = G++;
      else if (plan.depth[i] > d0 && plan.parent[i] != kNoMap) grp[i] = grp[plan.parent[i]];
    }
    if (G >= 2) {
      std::vector<std::vector<std::uint32_t>> down(G), leaf(G);
      std::vector<std::uint32_t> top_down, top_leaf;
      for (const Phase* ph : tree_phases(plan, stage)) {
        if (ph->kind == kPhaseUp) {  // the upward pass, level by level
          emit(ph->task_begin, ph->task_end);
          continue;
        }
        for (std::uint32_t t = ph->task_begin; t < ph->task_end; ++t) {
          const std::uint32_t g = grp[plan.tasks[t].node];
          (g == kNoMap ? top_down : down[g]).push_back(t);
        }
      }
      for (const Phase& ph : plan.phases)
        if (ph.stage == stage && ph.kind == kPhaseLeaf)
          for (std::uint32_t t = ph.task_begin; t < ph.task_end; ++t) {
            const std::uint32_t g = grp[plan.tasks[t].node];
            (g == kNoMap ? top_leaf : leaf[g]).push_back(t);
          }
      auto cost = [&](std::uint32_t t) {  // chunks of K plus a fixed part per item
        double c = 4.0;
        for (std::uint32_t si = plan.tasks[t].seg_begin; si < plan.tasks[t].seg_end; ++si) c += plan.segs[si].nchunks;
        return c;
      };
      auto merge = [&](const std::vector<std::uint32_t>& x, const std::vector<std::uint32_t>& y) {
        double xt = 0.0, yt = 0.0, xc = 0.0, yc = 0.0;
        for (std::uint32_t t : x) xt += cost(t);
        for (std::uint32_t t : y) yt += cost(t);
        std::size_t i = 0, j = 0;
        while (i < x.size() || j < y.size()) {
          const bool take_x = j >= y.size() || (i < x.size() && xc * yt <= yc * xt);
          const std::uint32_t t = take_x ? x[i++] : y[j++];
          (take_x ? xc : yc) += cost(t);
          emit_task(t);
        }
      };
      for (std::uint32_t t : top_down) emit_task(t);
      for (std::uint32_t t : down[0]) emit_task(t);
      for (std::uint32_t g = 1; g < G; ++g) merge(down[g], leaf[g - 1]);
      merge(leaf[G - 1], top_leaf);
      return items;
    }
  }
  const std::vector<std::uint8_t> sel = split_set(plan, f);
  // tree phases; the leaf rows: combined tasks of the leaves not split, the near tasks and the
  // accumulating tasks of the split ones (and every near task when f = 1: those of leaves
  // without a basis are their final rows)
  const std::vector<const Phase*> tree = tree_phases(plan, stage);
  std::vector<std::uint32_t> near, tail;
  for (const Phase& ph : plan.phases) {
    if (ph.stage != stage) continue;
    if (ph.kind == kPhaseLeaf && f < 1.0 && !plan.near_otf) {  // on the fly: the leaf rows run in waves
      for (std::uint32_t t = ph.task_begin; t < ph.task_end; ++t)
        if (!sel[plan.tasks[t].node]) tail.push_back(t);
    }
  }
  if (f > 0.0)
    for (const Phase& ph : plan.split_phases) {
      if (ph.stage != stage) continue;
      for (std::uint32_t t = ph.task_begin; t < ph.task_end; ++t)
        if (f >= 1.0 || sel[plan.tasks[t].node]) (ph.kind == kPhaseNear ? near : tail).push_back(t);
    }
  const std::uint64_t nt = near.size();
  const std::size_t L = tree.size();
  const std::size_t nslices = L > 1 ? L - 1 : 1;  // after every level but the first
  for (std::size_t k = 0; k < L; ++k) {
    emit(tree[k]->task_begin, tree[k]->task_end);
    if (nt && (L == 1 || k >= 1)) {
      const std::size_t slice = L == 1 ? 0 : k - 1;
      for (std::uint64_t i = nt * slice / nslices; i < nt * (slice + 1) / nslices; ++i) emit_task(near[i]);
    }
  }
  if (nt && L == 0)
    for (std::uint32_t t : near) emit_task(t);
  for (std::uint32_t t : tail) emit_task(t);
  return items;
}

// eval_dag's producer lanes publish the stored tiles when every CTA runs many items
// (cfg5-HSS, 660 per CTA: DAG -1.4%); with few (cfg2, 32 per CTA) the producer is the busier
// side and the consumers release their own tiles (forwarding cost cfg2 +21%).
#ifndef HMXG_FWD_MIN_ITEMS_PER_CTA
#define HMXG_FWD_MIN_ITEMS_PER_CTA 128
#endif
std::uint32_t forward_signals(std::uint32_t nitems, unsigned grid) {
  return nitems >= std::uint64_t(HMXG_FWD_MIN_ITEMS_PER_CTA) * grid ? 1u : 0u;
}

// [claim counter per stage | T counters | S counters | Yp counters | Wp counters] (nodes x ncb
// each), then the exit counter of the launch's self-reset (DagParams::reset_words)
constexpr std::size_t kDagClaimWords = 2;
// Words between two counters: polled counters packed into a few L2 lines make those lines'
// slice a hot spot when hundreds of producers and consumers poll and release them at once
// (narrow DAGs). HMXG_CSTRIDE overrides.
std::uint32_t counter_stride(const Plan& plan, std::size_t q, unsigned grid, std::uint32_t stage = 0) {
  if (stage != 0 || plan.nparts != 1) return 1;
  if (const char* e = std::getenv("HMXG_CSTRIDE")) return static_cast<std::uint32_t>(std::max(1, std::min(64, std::atoi(e))));
  // narrow DAGs (the column-split ones): one counter per 128-byte line (cfg1 DAG 63 -> 58 us
  // with the split); wide DAGs poll few counters at a time and keep them packed
  return colsplit(plan, q, grid) > 1 ? 32u : 1u;
}
std::size_t dag_done_words(const Plan& plan, std::size_t q, std::uint32_t cstride = 1) {
  const std::size_t ncb = (q + kBN - 1) / kBN;
  return (kDagClaimWords + 4 * std::size_t(plan.num_nodes) * ncb) * cstride;  // T, S, Yp, Wp counters
}

// Small problems run the permutations inside the DAG launch (DagParams::fused): one launch,
// Wp gathered per (leaf, column block) by the CTAs before their first item, final leaf rows
// stored straight into Y. For large W the dedicated transpose kernels move the data at HBM
// speed and the DAG keeps all of its issue slots for the DMMAs.
#ifndef HMXG_FUSED_MAX_ELEMS
#define HMXG_FUSED_MAX_ELEMS (1u << 22)
#endif
bool fused_io(const Plan& plan, std::size_t q) {
  return plan.nparts == 1 && !plan.near_otf && plan.n * q <= std::uint64_t(HMXG_FUSED_MAX_ELEMS) &&
         std::getenv("HMXG_NO_FUSED") == nullptr;
}

// CTree mode (kernels.cuh, ct_run; opt-in with HMXG_CTREE=1): small fused problems whose tree
// work per 8-column octet is small run every task but the near field in clusters of CTAs, one
// cluster per octet, level by level with cluster barriers, instead of through the DAG's
// gpu-scope counters (~4 us per dependent level on cfg1). The tasks are the upward and
// far+downward phases and the split variant's accumulating leaf phase (ct_levels); the work
// bound is DMMAs per octet. Bit-identical to the DAG, but measured slower on cfg1 (115 vs 55
// us): an 8-column unit does ~30 instructions of operand addressing per
// DMMA and waits ~0.8 us per 3-k-step block. Returns the cluster size (0: the DAG runs every
// task); HMXG_CT_CLUSTER sets the size.
#ifndef HMXG_CT_MAX_DMMA_PER_OCTET
#define HMXG_CT_MAX_DMMA_PER_OCTET 16384
#endif
std::vector<const Phase*> ct_levels(const Plan& plan) {
  std::vector<const Phase*> lv;
  for (const Phase& ph : plan.phases)
    if (ph.stage == 0 && ph.kind != kPhaseLeaf) lv.push_back(&ph);
  for (const Phase& ph : plan.split_phases)
    if (ph.stage == 0 && ph.kind != kPhaseNear) lv.push_back(&ph);
  return lv;
}
double ct_dmma_per_octet(const Plan& plan) {
  double n = 0.0;
  std::uint64_t tasks = 0, steps = 0;
  for (const Phase* ph : ct_levels(plan))
    for (std::uint32_t t = ph->task_begin; t < ph->task_end; ++t) {
      const Task& tk = plan.tasks[t];
      ++tasks;
      for (std::uint32_t r0 = 0; r0 < tk.m; r0 += 8)
        for (std::uint32_t si = tk.seg_begin; si < tk.seg_end; ++si) {
          const SegDev& sg = plan.segs[si];
          if ((sg.rows && r0 >= sg.rows) || sg.nchunks == 0) continue;
          n += 4.0 * (sg.nchunks - 1) + (sg.last_ksteps ? sg.last_ksteps : 4);
        }
      for (std::uint32_t si = tk.seg_begin; si < tk.seg_end; ++si) {
        const SegDev& sg = plan.segs[si];
        if (sg.nchunks) steps += 4u * (sg.nchunks - 1u) + (sg.last_ksteps ? sg.last_ksteps : 4u);
      }
    }
  plan.ct_smem = (tasks * sizeof(Task) + 15) / 16 * 16 + (steps * sizeof(CtStep) + 15) / 16 * 16;
  return tasks ? n : 1e300;  // no tree tasks: nothing for a CTree
}
std::uint32_t ctree_csize(const Plan& plan, std::size_t q, unsigned grid) {
  if (!fused_io(plan, q) || plan.split_phases.empty() || plan.flat || !std::getenv("HMXG_CTREE")) return 0;
  if (plan.ct_dmma < 0.0) plan.ct_dmma = ct_dmma_per_octet(plan);
  if (plan.ct_dmma > HMXG_CT_MAX_DMMA_PER_OCTET || plan.ct_smem > std::uint64_t(kStages) * kStageBytes) return 0;
  const std::size_t noct = (q + 7) / 8;
  std::uint32_t c = 4;
  if (const char* e = std::getenv("HMXG_CT_CLUSTER")) c = static_cast<std::uint32_t>(std::max(1, std::min(8, std::atoi(e))));
  while (c > 1 && noct * c * 2 > grid) c /= 2;  // at most half of the grid in CTree clusters
  return noct * c * 2 <= grid ? c : 0u;
}

// Resident CTAs of eval_dag<true> launched in clusters of c (cached per c).
int ct_resident(DevState& d, std::uint32_t c) {
  if (d.ct_occ_c == static_cast<int>(c)) return HMXG_OK;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(d.gemm_grid - d.gemm_grid % c);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmemBytes;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = c;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int clusters = 0;
  HMXG_CUDA(cudaOccupancyMaxActiveClusters(&clusters, eval_dag<true>, &cfg));
  if (clusters <= 0) return set_err(HMXG_ECUDA, "eval_dag: no cluster of the CTree size fits an SM group");
  d.ct_occ_c = static_cast<int>(c);
  d.ct_occ_ctas = std::min<unsigned>(d.gemm_grid, static_cast<unsigned>(clusters) * c);
  return HMXG_OK;
}

// Item list and counters for q columns (built on first use, cached for a few q).
int ensure_dag(const Plan& plan, DevState& d, std::size_t q, cudaStream_t st, const DevState::DagItems** out,
               std::uint32_t stage = 0) {
  const bool ct = stage == 0 && ctree_csize(plan, q, d.gemm_grid) != 0;
  for (const auto& e : d.dag)
    if (e.valid && e.q == q && e.stage == stage && e.ct == ct) {
      *out = &e;
      return HMXG_OK;
    }
  DevState::DagItems& e = d.dag[d.dag_next++ % 4];
  // the slot's previous list may still be in use (this stream, or an earlier asynchronous
  // call on another one), and the cached graph may have captured it
  HMXG_CUDA(cudaStreamSynchronize(st));
  if (d.pending) HMXG_CUDA(cudaEventSynchronize(d.ev_last));
  if (e.valid) d.drop_graph();
  cudaFree(e.recs);
  e = DevState::DagItems{};
  const std::vector<std::uint64_t> items = build_items(plan, static_cast<std::uint32_t>(q), stage, d.gemm_grid);
  if (items.size() >= 0xffffffffull) return set_err(HMXG_EINVAL, "hmxg_evaluate: too many work items");
  {  // the records: every task's items are one run, column block then part fastest
    const std::uint32_t parts = colsplit(plan, q, d.gemm_grid, stage);
    const std::uint32_t per_task = static_cast<std::uint32_t>((q + kBN - 1) / kBN) * parts;
    if (items.size() % per_task) return set_err(HMXG_ECUDA, "internal: claim order is not whole task runs");
    std::vector<RingSlot> recs(items.size() / per_task);
    for (std::size_t j = 0; j < recs.size(); ++j) {
      const std::uint32_t t = static_cast<std::uint32_t>(items[j * per_task]);
      for (std::uint32_t r = 0; r < per_task; ++r)
        if (items[j * per_task + r] != make_item(kItemGemm, r / parts, t, r % parts))
          return set_err(HMXG_ECUDA, "internal: claim order is not whole task runs");
      RingSlot& rc = recs[j];
      std::memset(&rc, 0, sizeof(rc));
      rc.task = plan.tasks[t];
      const std::uint32_t ns = std::min<std::uint32_t>(rc.task.seg_end - rc.task.seg_begin, kSegSmem);
      // (near field on the fly: the device's segment table has its own tile offsets)
      const std::vector<SegDev>& segs = d.otf_segs.empty() ? plan.segs : d.otf_segs;
      for (std::uint32_t k = 0; k < ns; ++k) rc.seg[k] = segs[rc.task.seg_begin + k];
    }
    HMXG_TRY(dev_upload(&e.recs, recs.data(), recs.size(), st));
    e.per_task = per_task;
    e.parts = parts;
  }
  const std::size_t words = dag_done_words(plan, q, counter_stride(plan, q, d.gemm_grid, stage));
  if (words > d.dag_done_cap) {
    d.drop_graph();
    cudaFree(d.dag_done);
    d.dag_done = nullptr;
    HMXG_CUDA(cudaMalloc(&d.dag_done, (words + 1) * sizeof(std::uint32_t)));
    // every launch leaves the counters zero for the next one (permute_out or the DAG's own
    // last CTA zeroes them); a new buffer starts zero
    HMXG_CUDA(cudaMemsetAsync(d.dag_done, 0, (words + 1) * sizeof(std::uint32_t), st));
    d.dag_done_cap = words;
    d.counters_dirty = false;
  }
  if (stage == 0 && ctree_csize(plan, q, d.gemm_grid) && !d.ct_units) {
    // CTree program: its tasks in level order, each with the flat list of its k steps in the
    // DAG's order (kernels.cuh CtStep), in one blob; (local task << 5 | first octet) units of
    // kCtG row octets, level by level; the range of A chunks they read
    std::vector<Task> tasks;
    std::vector<CtStep> steps;
    std::vector<std::uint32_t> units, lvl{0};
    std::uint64_t t_lo = ~0ull, t_hi = 0;
    for (const Phase* ph : ct_levels(plan)) {
      for (std::uint32_t t = ph->task_begin; t < ph->task_end; ++t) {
        Task tk = plan.tasks[t];
        const std::uint32_t kb = static_cast<std::uint32_t>(steps.size());
        std::uint32_t wp_leaf = kNoMap;
        for (std::uint32_t si = tk.seg_begin; si < tk.seg_end; ++si) {
          const SegDev& sg = plan.segs[si];
          if (sg.nchunks == 0) continue;
          if (sg.bbuf == kBufWp && wp_leaf == kNoMap) wp_leaf = sg.src;
          if (sg.tile_off % kChunkElems || sg.b_row + 16ull * sg.nchunks >= (1ull << 24))
            return set_err(HMXG_EINVAL, "internal: CTree step out of range");
          const std::uint32_t lim = sg.rows ? (sg.rows + 7) / 8 : 8u;
          for (std::uint32_t ch = 0; ch < sg.nchunks; ++ch) {
            const std::uint32_t nks = (ch + 1 == sg.nchunks && sg.last_ksteps) ? sg.last_ksteps : 4u;
            for (std::uint32_t ks = 0; ks < nks; ++ks)
              steps.push_back(CtStep{static_cast<std::uint32_t>((sg.tile_off / kChunkElems + ch) * 4 + ks),
                                     (sg.b_row + ch * 16 + ks * 4) << 8 | std::uint32_t(sg.bbuf) << 4 | lim});
          }
          t_lo = std::min<std::uint64_t>(t_lo, sg.tile_off);
          t_hi = std::max<std::uint64_t>(t_hi, sg.tile_off + std::uint64_t(sg.nchunks) * kChunkElems);
        }
        if (tk.id_off != kNoMap && tk.id_buf == kBufWp && wp_leaf == kNoMap) wp_leaf = tk.id_node0;
        tk.seg_begin = kb;
        tk.seg_end = static_cast<std::uint32_t>(steps.size());
        tk.pad1 = wp_leaf;
        const std::uint32_t lt = static_cast<std::uint32_t>(tasks.size());
        tasks.push_back(tk);
        for (std::uint32_t o = 0; o * 8 < tk.m; o += kCtG) units.push_back(lt << 5 | o);
      }
      lvl.push_back(static_cast<std::uint32_t>(units.size()));
    }
    if (steps.size() >= (1ull << 32) / kChunkElems) return set_err(HMXG_EINVAL, "internal: CTree program too large");
    const std::size_t tb = (tasks.size() * sizeof(Task) + 15) / 16 * 16;
    const std::size_t sb = (steps.size() * sizeof(CtStep) + 15) / 16 * 16;
    std::vector<unsigned char> blob(tb + sb, 0);
    std::memcpy(blob.data(), tasks.data(), tasks.size() * sizeof(Task));
    if (!steps.empty()) std::memcpy(blob.data() + tb, steps.data(), steps.size() * sizeof(CtStep));
    HMXG_TRY(dev_upload(&d.ct_blob, blob.data(), blob.size(), st));
    HMXG_TRY(dev_upload(&d.ct_units, units.data(), units.size(), st));
    HMXG_TRY(dev_upload(&d.ct_lvl, lvl.data(), lvl.size(), st));
    d.ct_nlev = static_cast<std::uint32_t>(lvl.size() - 1);
    d.ct_blob_bytes = static_cast<std::uint32_t>(blob.size());
    d.ct_segs_off = static_cast<std::uint32_t>(tb);
    d.ct_tile_base = t_lo == ~0ull ? 0 : t_lo;
    d.ct_tile_lines = t_hi > d.ct_tile_base ? (t_hi - d.ct_tile_base + 15) / 16 : 0;
  }
  HMXG_CUDA(cudaStreamSynchronize(st));
  e.nitems = static_cast<std::uint32_t>(items.size());
  e.q = q;
  e.stage = stage;
  e.ct = ct;
  e.valid = true;
  *out = &e;
  return HMXG_OK;
}

#ifdef HMXG_TRACE
// Diagnostic builds only (tools/dag_trace.py): per-item globaltimer stamps of the last
// eval_dag launch, written as CSV to $HMXG_TRACE_OUT after a synchronous evaluation.
unsigned long long* g_trace = nullptr;
std::size_t g_trace_words = 0;
int trace_prepare(const DevState& d, cudaStream_t st) {
  const std::size_t words = std::size_t(d.gemm_grid) * kTraceSeq * kTraceWords;
  if (words > g_trace_words) {
    cudaFree(g_trace);
    HMXG_CUDA(cudaMalloc(&g_trace, words * sizeof(unsigned long long)));
    g_trace_words = words;
  }
  HMXG_CUDA(cudaMemsetAsync(g_trace, 0, words * sizeof(unsigned long long), st));
  return HMXG_OK;
}
void trace_dump(const Plan& plan, std::size_t q, unsigned grid) {
  const char* path = std::getenv("HMXG_TRACE_OUT");
  if (!path || !g_trace) return;
  std::vector<unsigned long long> h(g_trace_words);
  if (cudaMemcpy(h.data(), g_trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
    return;
  const std::vector<std::uint64_t> items = build_items(plan, static_cast<std::uint32_t>(q), 0, grid);
  std::vector<const Phase*> phs;
  for (const Phase& ph : plan.phases) phs.push_back(&ph);
  for (const Phase& ph : plan.split_phases) phs.push_back(&ph);
  for (const Phase& ph : plan.flat_phases) phs.push_back(&ph);
  FILE* f = std::fopen(path, "w");
  if (!f) return;
  std::fprintf(f, "cta,seq,sm,item,task,cb,kind,level,m,segs,chunks,t_claim,t_issued,t_take,t_kend,t_done,t_first,t_deps,"
               "node,sub\n");
  for (std::size_t b = 0; b < g_trace_words / (kTraceSeq * kTraceWords); ++b)
    for (int s = 0; s < kTraceSeq; ++s) {
      const unsigned long long* r = &h[(b * kTraceSeq + s) * kTraceWords];
      if (r[1] == 0) continue;
      const std::uint32_t qi = static_cast<std::uint32_t>(r[0]);
      if (qi >= items.size()) continue;
      const std::uint32_t task = static_cast<std::uint32_t>(items[qi]);
      const std::uint32_t cb = item_cb(items[qi]);
      int kind = -1, level = -1;
      for (const Phase* ph : phs)
        if (task >= ph->task_begin && task < ph->task_end) {
          kind = ph->kind;
          level = static_cast<int>(ph->level);
        }
      const Task& tk = plan.tasks[task];
      unsigned chunks = 0;
      for (std::uint32_t sgi = tk.seg_begin; sgi < tk.seg_end; ++sgi) chunks += plan.segs[sgi].nchunks;
      std::fprintf(f, "%zu,%d,%llu,%u,%u,%u,%d,%d,%u,%u,%u,%llu,%llu,%llu,%llu,%llu,%llu,%llu,%u,%u\n", b, s, r[0] >> 32,
                   qi, task, cb, kind, level, tk.m, tk.seg_end - tk.seg_begin, chunks, r[1], r[2], r[3], r[4], r[5], r[6],
                   r[7], tk.node, item_sub(items[qi]));
    }
  std::fclose(f);
  // CTree clusters: per CTA start, tables copied, end of each level
  {
    const std::string cpath = std::string(path) + ".ctree";
    FILE* fc = std::fopen(cpath.c_str(), "w");
    if (fc) {
      std::fprintf(fc, "cta,oct,rank,t_start,t_tables,levels\n");
      for (std::size_t b = 0; b < g_trace_words / (kTraceSeq * kTraceWords); ++b) {
        const unsigned long long* r = &h[(b * kTraceSeq + kTraceSeq - 3) * kTraceWords];
        if ((r[0] >> 48) != 0xc7eeull) continue;
        std::fprintf(fc, "%zu,%llu,%llu,%llu,%llu,", b, (r[0] >> 8) & 0xffffffull, r[0] & 0xffull, r[1], r[2]);
        for (int l = 0; l < 13 && r[3 + l]; ++l) std::fprintf(fc, "%s%llu", l ? ";" : "", r[3 + l]);
        std::fprintf(fc, "\n");
      }
      std::fclose(fc);
    }
  }
  {  // CTree units: per warp its first unit of level 0 [begin, waited, first block, end, unit|chunks]
    const std::string upath = std::string(path) + ".ctunit";
    FILE* fu = std::fopen(upath.c_str(), "w");
    if (fu) {
      std::fprintf(fu, "cta,warp,t_begin,t_waited,t_first,t_end,unit,chunks,blocks\n");
      for (std::size_t b = 0; b < g_trace_words / (kTraceSeq * kTraceWords); ++b) {
        const unsigned long long* r0 = &h[(b * kTraceSeq + kTraceSeq - 3) * kTraceWords];
        if ((r0[0] >> 48) != 0xc7eeull) continue;
        for (int w = 0; w < 5; ++w) {
          const unsigned long long* r = &h[(b * kTraceSeq + kTraceSeq - 8 - 15) * kTraceWords + w * 24];
          if (!r[0]) continue;
          std::fprintf(fu, "%zu,%d,%llu,%llu,%llu,%llu,%llu,%llu,", b, w, r[0], r[1], r[2], r[3], r[4] >> 32,
                       r[4] & 0xffffffffull);
          for (int k = 0; k < 12 && r[5 + k]; ++k) std::fprintf(fu, "%s%llu", k ? ";" : "", r[5 + k] - r[1]);
          std::fprintf(fu, "\n");
        }
      }
      std::fclose(fu);
    }
  }
  // the fused permute jobs: per CTA start, stores done, signal released
  const std::string ppath = std::string(path) + ".perm";
  FILE* fp = std::fopen(ppath.c_str(), "w");
  if (!fp) return;
  std::fprintf(fp, "cta,t_start,t_stored,t_signalled\n");
  for (std::size_t b = 0; b < g_trace_words / (kTraceSeq * kTraceWords); ++b) {
    const unsigned long long* r = &h[(b * kTraceSeq + kTraceSeq - 1) * kTraceWords];
    if (r[0] == 0xfffffffffull) std::fprintf(fp, "%zu,%llu,%llu,%llu\n", b, r[1], r[2], r[3]);
  }
  std::fclose(fp);
}
#endif

// Default: one whole-evaluation DAG launch. `levels`: the level-by-level launch sequence
// (permute-in, one launch per tree level, permute-out) for per-launch breakdowns.
// A launch that may overlap its predecessor (programmatic dependent launch): the kernel
// waits for it in-kernel (griddepcontrol.wait). pdl false: an ordinary stream launch.
template <class... KArgs, class... Args>
int launch_dependent(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  HMXG_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  return HMXG_OK;
}

int enqueue_eval(const Plan& plan, DevState& d, const double* w, std::size_t ldw, double* y,
                 std::size_t ldy, std::size_t q, cudaStream_t st, bool time_phases, bool levels,
                 std::uint32_t* launches) {
  const std::uint32_t n = static_cast<std::uint32_t>(plan.n);
  const std::uint32_t qq = static_cast<std::uint32_t>(q);
  const dim3 eblk(256);
  d.last_q = q;
  // Per-launch timing events (time_phases). Under graph capture they become external
  // event-record nodes, so a replayed timed graph still times every launch.
  std::size_t ev = 0;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  HMXG_CUDA(cudaStreamIsCapturing(st, &cap));
  const bool capturing = cap == cudaStreamCaptureStatusActive;
  auto mark = [&]() -> int {
    if (time_phases)
      HMXG_CUDA(cudaEventRecordWithFlags(d.phase_ev[ev++], st, capturing ? cudaEventRecordExternal : 0u));
    return HMXG_OK;
  };
  // the launch sequence as hmxg_phase_get reports it (algorithmic flops / bytes per launch)
  std::vector<DevState::LaunchDesc> descs;
  auto desc = [&](std::uint32_t kind, std::uint32_t level, std::uint32_t tiles, double flops, double gen, double io) {
    descs.push_back(DevState::LaunchDesc{kind, level, tiles, flops, gen, io});
  };
  auto desc_phase = [&](const Phase& ph) {
    desc(ph.kind == kPhaseUp ? 1u : (ph.kind == kPhaseDown ? 2u : (ph.kind == kPhaseLeaf ? 3u : 6u)), ph.level,
         ph.task_end - ph.task_begin, ph.flops_per_col, ph.gen_bytes, ph.io_bytes_per_col);
  };
  auto desc_perm = [&](std::uint32_t kind) { desc(kind, 0, static_cast<std::uint32_t>((plan.n + 31) / 32), 0.0, 4.0 * plan.n, 16.0 * plan.n); };
  CUtensorMap tm_wp, tm_t, tm_s;
  const std::uint64_t ldq = d.cap_q;
  if (d.poison) {  // debug race detector: every live workspace row NaN before the launches
    const std::uint64_t pc = phys_cols(q);
    poison_rows<<<1184, 256, 0, st>>>(d.wp, ldq, d.ipmap, plan.n, pc);
    poison_rows<<<1184, 256, 0, st>>>(d.yp, ldq, d.ipmap, plan.n, pc);
    if (d.ts_live_count) {
      poison_rows<<<1184, 256, 0, st>>>(d.t, ldq, d.ts_live, d.ts_live_count, pc);
      poison_rows<<<1184, 256, 0, st>>>(d.s, ldq, d.ts_live, d.ts_live_count, pc);
    }
    HMXG_CUDA(cudaGetLastError());
  }
  HMXG_TRY(make_map(&tm_wp, d.wp, plan.rows_pad, q, ldq));
  HMXG_TRY(make_map(&tm_t, d.t, plan.skel_rows, q, ldq));
  HMXG_TRY(make_map(&tm_s, d.s, plan.skel_rows, q, ldq));
  GemmParams p{};
  p.tiles = d.tiles;
  p.buf[kBufWp] = d.wp;
  p.buf[kBufT] = d.t;
  p.buf[kBufS] = d.s;
  p.buf[kBufYp] = d.yp;
  p.ld[kBufWp] = ldq;
  p.ld[kBufT] = ldq;
  p.ld[kBufS] = ldq;
  p.ld[kBufYp] = ldq;
  p.segs = d.segs;
  p.idmap = d.idmap;
  p.q = qq;
  // on-the-fly near field: every wave generates its near chunks into the scratch, then runs
  // its leaf rows (the grouped GEMM over the wave's combined leaf tasks)
  auto run_waves = [&](std::uint32_t* counters) -> int {
    if (d.waves.empty()) return HMXG_OK;
    HMXG_CUDA(cudaMemsetAsync(counters, 0, d.waves.size() * sizeof(std::uint32_t), st));
    const std::uint32_t col_blocks = (qq + kBN - 1) / kBN;
    for (std::size_t w = 0; w < d.waves.size(); ++w) {
      const DevState::Wave& wv = d.waves[w];
      const std::uint64_t nch = wv.c1 - wv.c0;
      if (nch) {
        gen_near<<<static_cast<unsigned>(std::min<std::uint64_t>(nch, 148ull * 8)), 256, 80 * d.kp.d * sizeof(double),
                   st>>>(d.pts, d.kp, d.pmap, d.gen_chunks + wv.c0, nch, d.tiles);
        ++*launches;
        desc(7, static_cast<std::uint32_t>(w), static_cast<std::uint32_t>(nch), 0.0, 8.0 * kChunkElems * nch, 0.0);
        HMXG_TRY(mark());
      }
      GemmParams pw = p;
      pw.tasks = d.tasks + wv.t0;
      const std::uint32_t ntasks = wv.t1 - wv.t0;
      const std::uint64_t tiles = std::uint64_t(ntasks) * col_blocks;
      if (tiles > 0xfffff000ull) return set_err(HMXG_EINVAL, "hmxg_evaluate: too many output tiles");
      grouped_gemm<<<static_cast<unsigned>(std::min<std::uint64_t>(tiles, d.gemm_grid)), kThreads, kSmemBytes, st>>>(
          tm_wp, tm_t, tm_s, pw, ntasks, counters + w);
      ++*launches;
      desc(3, static_cast<std::uint32_t>(w), ntasks, d.wave_flops[w], 4.0 * d.wave_flops[w], d.wave_io[w]);
      HMXG_TRY(mark());
    }
    HMXG_CUDA(cudaGetLastError());
    return HMXG_OK;
  };
  if (!levels) {
    const DevState::DagItems* di = nullptr;
    const bool ct = ctree_csize(plan, q, d.gemm_grid) != 0;
    for (const auto& e : d.dag)
      if (e.valid && e.q == q && e.stage == 0 && e.ct == ct) di = &e;
    if (!di) return set_err(HMXG_ECUDA, "internal: DAG items not prepared");
    const std::uint32_t cst = counter_stride(plan, q, d.gemm_grid);
    const std::size_t words = dag_done_words(plan, q, cst);
    const bool fused = fused_io(plan, q);
    d.last_fused = fused;
    DagParams dp{};
    dp.recs = di->recs;
    dp.per_task = di->per_task;
    dp.parts = di->parts;
    dp.nitems = di->nitems;
    dp.claim = d.dag_done;
    dp.done = d.dag_done + kDagClaimWords * cst;
    dp.cstride = cst;
    dp.node_tiles = d.node_tiles;
    dp.yp_tiles = d.yp_tiles;
    dp.signal_yp = split_frac(plan, q, d.gemm_grid) > 0.0 ? 1u : 0u;
    dp.colsplit = colsplit(plan, q, d.gemm_grid);
    dp.ncb = (qq + kBN - 1) / kBN;
    dp.nodes = plan.num_nodes;
    dp.fwd_signals = forward_signals(di->nitems, d.gemm_grid);
    p.tasks = d.tasks;
#ifdef HMXG_TRACE
    HMXG_TRY(trace_prepare(d, st));
    dp.trace = g_trace;
#endif
    if (d.counters_dirty) HMXG_CUDA(cudaMemsetAsync(d.dag_done, 0, (words + 1) * sizeof(std::uint32_t), st));
    d.counters_dirty = true;  // until the launch that zeroes them is enqueued
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(di->nitems, d.gemm_grid));
    if (fused) {
      // one launch: permutations inside, counters zeroed by the DAG's last CTA
      dp.fused = 1;
      dp.n = n;
      dp.ipmap = d.ipmap;
      dp.rowleaf = d.rowleaf;
      dp.wp_target = d.wp_target;
      dp.w = w;
      dp.ldw = ldw;
      dp.pmap = d.pmap;
      dp.reset_words = static_cast<std::uint32_t>(words);
      dp.exit_ctr = d.dag_done + words;
      dp.pf_tile_lines = d.tile_elems / 16;
      p.y_final = y;
      p.ldy = ldy;
      p.pmap = d.pmap;
      unsigned fgrid = std::max<unsigned>(grid, std::min<unsigned>(d.gemm_grid, (n + 31) / 32 * dp.ncb));
      const std::uint32_t csize = ctree_csize(plan, q, d.gemm_grid);
      if (csize) {
        if (!d.ct_units) return set_err(HMXG_ECUDA, "internal: CTree program not prepared");
        dp.ct_noct = static_cast<std::uint32_t>((q + 7) / 8);
        dp.ct_csize = csize;
        dp.ct_nlev = d.ct_nlev;
        dp.ct_units = d.ct_units;
        dp.ct_lvl = d.ct_lvl;
        dp.ct_blob = d.ct_blob;
        dp.ct_blob_bytes = d.ct_blob_bytes;
        dp.ct_segs_off = d.ct_segs_off;
        dp.ct_tile_base = d.ct_tile_base;
        p.y_final = nullptr;  // the final rows go to Yp; the clusters write Y
        dp.y = y;
        dp.ldy = ldy;
        dp.ct_tile_lines = d.ct_tile_lines;
        // every CTA in clusters of csize; the CTree clusters come on top of the item CTAs, and
        // the grid stays within what is resident at once
        HMXG_TRY(ct_resident(d, csize));
        fgrid = std::min<unsigned>(fgrid + dp.ct_noct * csize, d.ct_occ_ctas);
        fgrid -= fgrid % csize;
        if (std::getenv("HMXG_DEBUG_LAUNCH"))
          std::fprintf(stderr, "[hmxg] CTree launch: grid %u, clusters of %u, %u octet clusters, %u levels, resident %u\n",
                       fgrid, csize, dp.ct_noct, dp.ct_nlev, d.ct_occ_ctas);
      }
      HMXG_TRY(mark());
      if (csize) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(fgrid);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kSmemBytes;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = csize;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        HMXG_CUDA(cudaLaunchKernelEx(&cfg, eval_dag<true>, tm_wp, tm_t, tm_s, p, dp));
      } else {
        eval_dag<true><<<fgrid, kThreads, kSmemBytes, st>>>(tm_wp, tm_t, tm_s, p, dp);
      }
      ++*launches;
      HMXG_TRY(mark());
      {  // the permutations ran inside: W read and Y written once more per column
        DevState::LaunchDesc a{5, 0, 0, 0.0, 4.0 * plan.n, 16.0 * plan.n};
        for (const Phase* ph : level_phases(plan, q, d.gemm_grid)) {
          a.tiles += ph->task_end - ph->task_begin;
          a.flops_per_col += ph->flops_per_col;
          a.gen_bytes += ph->gen_bytes;
          a.io_bytes_per_col += ph->io_bytes_per_col;
        }
        descs.push_back(a);
      }
      d.launch_desc = std::move(descs);
      HMXG_CUDA(cudaGetLastError());
      d.counters_dirty = false;
      d.last_launches = 1;
      if (time_phases) d.phase_valid = true;
      return HMXG_OK;
    }
    HMXG_TRY(mark());
    const dim3 pgrid2((n + kTT - 1) / kTT, (qq + kTT - 1) / kTT);
    if (pgrid2.y > 65535) return set_err(HMXG_EINVAL, "hmxg_evaluate: too many columns for one call");
    // eval_dag and permute_out are programmatic dependent launches (their launch overlaps the
    // predecessor; they wait in-kernel). With per-launch timing the dependents launch
    // normally, so each event brackets one kernel. permute_out zeroes the DAG's counters.
    permute_in<<<pgrid2, eblk, 0, st>>>(w, ldw, d.ipmap, d.wp, ldq, n, qq, nullptr, 0);
    ++*launches;
    desc_perm(0);
    HMXG_TRY(mark());
    // Programmatic dependent launch of eval_dag and permute_out (HMXG_PDL=1; 2: permute_out
    // only) is off by default: measured on cfg5-HSS without per-launch events, 16.60 ms with
    // it (either form) against 16.38-16.47 ms without -- the dependents' early CTAs hold SM
    // slots through their predecessor's tail; cfg2 equal. (An event between two kernels would
    // break the programmatic edge anyway.)
    const bool pdl = !time_phases;
    const int pdl_mode = std::getenv("HMXG_PDL") ? std::atoi(std::getenv("HMXG_PDL")) : 0;
    const bool pdl_dag = pdl && pdl_mode == 1, pdl_out = pdl && pdl_mode >= 1;
    const bool narrow = dp.colsplit > 1 || dp.cstride > 1;
    if (grid) {  // (on the fly, a tree without levels has nothing for the DAG)
      HMXG_TRY(launch_dependent(pdl_dag, narrow ? eval_dag<true> : eval_dag<false>, dim3(grid), dim3(kThreads), kSmemBytes,
                                st, tm_wp, tm_t, tm_s, p, dp));
      ++*launches;
      DevState::LaunchDesc a{5, 0, 0, 0.0, 0.0, 0.0};
      for (const Phase* ph : level_phases(plan, q, d.gemm_grid)) {
        if (plan.near_otf && ph->kind == kPhaseLeaf) continue;  // the waves below
        a.tiles += ph->task_end - ph->task_begin;
        a.flops_per_col += ph->flops_per_col;
        a.gen_bytes += ph->gen_bytes;
        a.io_bytes_per_col += ph->io_bytes_per_col;
      }
      descs.push_back(a);
      HMXG_TRY(mark());
    }
    if (plan.near_otf) HMXG_TRY(run_waves(d.tile_counters));
    HMXG_TRY(launch_dependent(pdl_out && !plan.near_otf, permute_out, pgrid2, eblk, 0, st, static_cast<const double*>(d.yp),
                              std::uint64_t(ldq), static_cast<const std::uint32_t*>(d.ipmap), y, std::uint64_t(ldy), n,
                              qq, d.dag_done, std::uint64_t(words + 1)));
    ++*launches;
    desc_perm(4);
    HMXG_TRY(mark());
    d.launch_desc = std::move(descs);
    HMXG_CUDA(cudaGetLastError());
    d.counters_dirty = false;
    d.last_launches = static_cast<std::uint32_t>(d.launch_desc.size());
    if (time_phases) d.phase_valid = true;
    return HMXG_OK;
  }
  d.last_fused = false;
  HMXG_TRY(mark());
  const dim3 pgrid((n + kTT - 1) / kTT, (qq + kTT - 1) / kTT);
  if (pgrid.y > 65535) return set_err(HMXG_EINVAL, "hmxg_evaluate: too many columns for one call");
  permute_in<<<pgrid, eblk, 0, st>>>(w, ldw, d.ipmap, d.wp, ldq, n, qq, nullptr, 0);
  ++*launches;
  desc_perm(0);
  HMXG_TRY(mark());
  const std::uint32_t col_blocks = (qq + kBN - 1) / kBN;
  const std::vector<const Phase*> lphases = level_phases(plan, q, d.gemm_grid);
  HMXG_CUDA(cudaMemsetAsync(d.tile_counters, 0, lphases.size() * sizeof(std::uint32_t), st));
  for (std::size_t ph_i = 0; ph_i < lphases.size(); ++ph_i) {
    const Phase& ph = *lphases[ph_i];
    if (plan.near_otf && ph.kind == kPhaseLeaf) {
      HMXG_TRY(run_waves(d.tile_counters + lphases.size()));
      continue;
    }
    p.tasks = d.tasks + ph.task_begin;
    const std::uint32_t ntasks = ph.task_end - ph.task_begin;
    const std::uint64_t tiles = std::uint64_t(ntasks) * col_blocks;
    if (tiles > 0xfffff000ull) return set_err(HMXG_EINVAL, "hmxg_evaluate: too many output tiles");
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(tiles, d.gemm_grid));
    grouped_gemm<<<grid, kThreads, kSmemBytes, st>>>(tm_wp, tm_t, tm_s, p, ntasks, d.tile_counters + ph_i);
    ++*launches;
    desc_phase(ph);
    HMXG_TRY(mark());
  }
  permute_out<<<pgrid, eblk, 0, st>>>(d.yp, ldq, d.ipmap, y, ldy, n, qq, nullptr, 0);
  ++*launches;
  desc_perm(4);
  HMXG_TRY(mark());
  d.launch_desc = std::move(descs);
  d.last_launches = static_cast<std::uint32_t>(d.launch_desc.size());
  HMXG_CUDA(cudaGetLastError());
  if (time_phases) d.phase_valid = true;
  return HMXG_OK;
}

int copy_cols(double* dst, std::size_t lddst, const double* src, std::size_t ldsrc, std::size_t rows,
              std::size_t cols, cudaMemcpyKind kind, cudaStream_t st) {
  if (lddst == rows && ldsrc == rows) {
    HMXG_CUDA(cudaMemcpyAsync(dst, src, rows * cols * sizeof(double), kind, st));
  } else {
    HMXG_CUDA(cudaMemcpy2DAsync(dst, lddst * sizeof(double), src, ldsrc * sizeof(double), rows * sizeof(double),
                                cols, kind, st));
  }
  return HMXG_OK;
}

// Host-pointer evaluation of columns [c0, c1) on device d: chunks of host_chunk_cols columns,
// double-buffered staging, copies on their own streams so PCIe traffic in both
// directions overlaps the kernels.
int enqueue_host_shard(const Plan& plan, DevState& d, const double* W, std::size_t ldw, double* Y,
                       std::size_t ldy, std::size_t c0, std::size_t c1, bool time_phases, bool levels,
                       std::uint32_t* launches) {
  const std::size_t n = plan.n, qg = c1 - c0;
  const std::size_t cq = host_chunk_cols(plan, qg);
  HMXG_TRY(ensure_workspace(plan, d, cq));
  HMXG_TRY(ensure_stage(plan, d, cq));
  const std::size_t chunks = (qg + cq - 1) / cq;
  for (std::size_t k = 0; k < chunks; ++k) {
    const int b = static_cast<int>(k & 1);
    const std::size_t a = c0 + k * cq, m = std::min(cq, c1 - a);
    // input buffer b is free once the evaluation of chunk k-2 finished
    if (k >= 2) HMXG_CUDA(cudaStreamWaitEvent(d.h2d, d.ev_done[b], 0));
    HMXG_TRY(copy_cols(d.w_stage[b], n, W + a * ldw, ldw, n, m, cudaMemcpyHostToDevice, d.h2d));
    HMXG_CUDA(cudaEventRecord(d.ev_in[b], d.h2d));
    HMXG_CUDA(cudaStreamWaitEvent(d.comp, d.ev_in[b], 0));
    // output buffer b is free once the copy-out of chunk k-2 finished
    if (k >= 2) HMXG_CUDA(cudaStreamWaitEvent(d.comp, d.ev_out[b], 0));
    if (k == 0) HMXG_CUDA(cudaEventRecord(d.ev0, d.comp));
    const DevState::DagItems* di = nullptr;
    if (!levels) HMXG_TRY(ensure_dag(plan, d, m, d.comp, &di));
    HMXG_TRY(enqueue_eval(plan, d, d.w_stage[b], n, d.y_stage[b], n, m, d.comp, time_phases && k == 0, levels,
                          launches));
    HMXG_CUDA(cudaEventRecord(d.ev_done[b], d.comp));
    if (k + 1 == chunks) HMXG_CUDA(cudaEventRecord(d.ev1, d.comp));
    HMXG_CUDA(cudaStreamWaitEvent(d.d2h, d.ev_done[b], 0));
    HMXG_TRY(copy_cols(Y + a * ldy, ldy, d.y_stage[b], n, n, m, cudaMemcpyDeviceToHost, d.d2h));
    HMXG_CUDA(cudaEventRecord(d.ev_out[b], d.d2h));
  }
  return HMXG_OK;
}

// What a W / Y pointer of the host path is: memory the copy engines can read or write
// without staging (pinned or registered), pageable (or managed: staged by the host threads
// like pageable memory), or device memory, which needs HMXG_F_DEVICE_PTRS.
enum class HostKind { kPageable, kPinned, kDevice };
HostKind host_kind(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return HostKind::kPageable;
  }
  if (a.type == cudaMemoryTypeDevice) return HostKind::kDevice;
  return a.type == cudaMemoryTypeHost ? HostKind::kPinned : HostKind::kPageable;
}

// The stream `st` of device d waits for the previous call's work (see DevState::ev_last).
// Not inside a capture the caller runs: its graph cannot wait on an event recorded outside.
int order_after_previous(DevState& d, cudaStream_t st) {
  if (!d.pending) return HMXG_OK;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  HMXG_CUDA(cudaStreamIsCapturing(st, &cap));
  if (cap != cudaStreamCaptureStatusNone) return HMXG_OK;
  HMXG_CUDA(cudaStreamWaitEvent(st, d.ev_last, 0));
  return HMXG_OK;
}

// Columns [c0, c0 + m) between a column-major host matrix and a contiguous n x m buffer,
// split over `threads` host threads by column.
void copy_columns_mt(double* dst, std::size_t lddst, const double* src, std::size_t ldsrc, std::size_t n,
                     std::size_t m, unsigned threads) {
  // Non-temporal stores: the destination (pinned staging read back by DMA, or the
  // caller's Y) is not read by this thread, so no read-for-ownership traffic on it.
  auto copy_col = [n](double* d, const double* s) {
    std::size_t i = 0;
    if ((reinterpret_cast<std::uintptr_t>(d) & 15) == 0) {
      for (; i + 8 <= n; i += 8) {
        const __m128d a = _mm_loadu_pd(s + i), b = _mm_loadu_pd(s + i + 2), c = _mm_loadu_pd(s + i + 4),
                      e = _mm_loadu_pd(s + i + 6);
        _mm_stream_pd(d + i, a);
        _mm_stream_pd(d + i + 2, b);
        _mm_stream_pd(d + i + 4, c);
        _mm_stream_pd(d + i + 6, e);
      }
    }
    for (; i < n; ++i) d[i] = s[i];
  };
  auto part = [&](std::size_t j0, std::size_t j1) {
    for (std::size_t j = j0; j < j1; ++j) copy_col(dst + j * lddst, src + j * ldsrc);
    _mm_sfence();
  };
  const std::size_t t = std::max<std::size_t>(1, std::min<std::size_t>(threads, m));
  if (t == 1 || n * m * sizeof(double) < (std::size_t(1) << 22)) {
    part(0, m);
    return;
  }
  std::vector<std::thread> pool;
  for (std::size_t k = 1; k < t; ++k) pool.emplace_back(part, m * k / t, m * (k + 1) / t);
  part(0, m / t);
  for (auto& th : pool) th.join();
}

// Host-pointer evaluation from pageable memory. cudaMemcpyAsync from pageable buffers is
// staged by the driver and host-synchronous, so the chunk pipeline of enqueue_host_shard
// collapses (cfg5-HSS: 615 ms per step against 90 ms from pinned buffers). Here the host
// threads copy each chunk of W into pinned staging and each chunk of Y out of it, while the
// copy engines and the evaluation work on the neighbouring chunks: chunk k+1 is staged and
// chunk k-1 unstaged while chunk k is on the device. Returns when Y is complete.
int host_bounce_shard(const Plan& plan, DevState& d, const double* W, std::size_t ldw, double* Y, std::size_t ldy,
                      std::size_t c0, std::size_t c1, bool time_phases, bool levels, std::uint32_t* launches,
                      unsigned threads) {
  HMXG_CUDA(cudaSetDevice(d.dev));
  const std::size_t n = plan.n, qg = c1 - c0;
  const std::size_t cq = host_chunk_cols(plan, qg);
  HMXG_TRY(ensure_workspace(plan, d, cq));
  HMXG_TRY(ensure_stage(plan, d, cq));
  if (cq > d.pin_q) {
    d.release_pinned();
    for (int b = 0; b < 2; ++b) {
      HMXG_CUDA(cudaHostAlloc(&d.w_pin[b], n * cq * sizeof(double), cudaHostAllocPortable));
      HMXG_CUDA(cudaHostAlloc(&d.y_pin[b], n * cq * sizeof(double), cudaHostAllocPortable));
    }
    d.pin_q = cq;
  }
  const std::size_t chunks = (qg + cq - 1) / cq;
  auto cols = [&](std::size_t k) { return std::min(cq, qg - k * cq); };
  for (std::size_t k = 0; k <= chunks; ++k) {
    if (k < chunks) {
      const int b = static_cast<int>(k & 1);
      const std::size_t a = c0 + k * cq, m = cols(k);
      // pinned W buffer b is free once the H2D of chunk k-2 finished
      if (k >= 2) HMXG_CUDA(cudaEventSynchronize(d.ev_in[b]));
      copy_columns_mt(d.w_pin[b], n, W + a * ldw, ldw, n, m, threads);
      if (k >= 2) HMXG_CUDA(cudaStreamWaitEvent(d.h2d, d.ev_done[b], 0));  // device W buffer b is free
      HMXG_CUDA(cudaMemcpyAsync(d.w_stage[b], d.w_pin[b], n * m * sizeof(double), cudaMemcpyHostToDevice, d.h2d));
      HMXG_CUDA(cudaEventRecord(d.ev_in[b], d.h2d));
      HMXG_CUDA(cudaStreamWaitEvent(d.comp, d.ev_in[b], 0));
      if (k >= 2) HMXG_CUDA(cudaStreamWaitEvent(d.comp, d.ev_out[b], 0));  // device Y buffer b is free
      if (k == 0) HMXG_CUDA(cudaEventRecord(d.ev0, d.comp));
      const DevState::DagItems* di = nullptr;
      if (!levels) HMXG_TRY(ensure_dag(plan, d, m, d.comp, &di));
      HMXG_TRY(enqueue_eval(plan, d, d.w_stage[b], n, d.y_stage[b], n, m, d.comp, time_phases && k == 0, levels,
                            launches));
      HMXG_CUDA(cudaEventRecord(d.ev_done[b], d.comp));
      if (k + 1 == chunks) HMXG_CUDA(cudaEventRecord(d.ev1, d.comp));
      HMXG_CUDA(cudaStreamWaitEvent(d.d2h, d.ev_done[b], 0));
      HMXG_CUDA(cudaMemcpyAsync(d.y_pin[b], d.y_stage[b], n * m * sizeof(double), cudaMemcpyDeviceToHost, d.d2h));
      HMXG_CUDA(cudaEventRecord(d.ev_out[b], d.d2h));
    }
    if (k >= 1) {  // chunk k-1 out of pinned Y buffer (k-1) & 1, which chunk k+1 reuses
      const int b = static_cast<int>((k - 1) & 1);
      HMXG_CUDA(cudaEventSynchronize(d.ev_out[b]));
      copy_columns_mt(Y + (c0 + (k - 1) * cq) * ldy, ldy, d.y_pin[b], n, n, cols(k - 1), threads);
    }
  }
  return HMXG_OK;
}

}  // namespace
}  // namespace hmxg

namespace hmxg {
namespace {

// Subtree-split upload: only the generator blocks this part's tiles read are copied to
// the device (one compact array per generator kind); tile sources are re-based onto it.
int compact_generators(const hmxg_cds_view& v, Plan& plan, const double* (&src)[3], std::vector<double> (&host)[3]) {
  const std::uint64_t* ptr[3] = {v.dptr, v.bptr, v.vptr};
  const std::uint64_t count[3] = {v.num_near, v.num_far, v.num_v};
  const double* gen[3] = {v.dgen, v.bgen, v.vgen};
  std::vector<std::uint64_t> base[3];
  for (int g = 0; g < 3; ++g) base[g].assign(count[g], ~std::uint64_t(0));
  for (TileSrc& ts : plan.tile_src) {
    const int g = ts.gen;
    const std::uint64_t slot = std::upper_bound(ptr[g], ptr[g] + count[g] + 1, ts.a_off) - ptr[g] - 1;
    if (slot >= count[g]) return set_err(HMXG_EINVAL, "split upload: tile source outside its generator");
    if (base[g][slot] == ~std::uint64_t(0)) {
      base[g][slot] = host[g].size();
      host[g].insert(host[g].end(), gen[g] + ptr[g][slot], gen[g] + ptr[g][slot + 1]);
    }
    ts.a_off = base[g][slot] + (ts.a_off - ptr[g][slot]);
  }
  for (int g = 0; g < 3; ++g) src[g] = host[g].data();
  plan.d_elems = host[0].size();
  plan.b_elems = host[1].size();
  plan.v_elems = host[2].size();
  return HMXG_OK;
}

// Generated blocks (hmxg_upload_generated): the points and kernel of the CDS, and
// optionally every node's skeleton (CSR) to generate the far blocks too.
struct NearSource {
  const double* coords = nullptr;  // n x d, original point order
  std::uint32_t d = 0;
  KernelParams kp{};
  const std::uint64_t* skel_ptr = nullptr;  // num_nodes + 1, or null: bgen comes from the view
  const std::uint32_t* skel_idx = nullptr;
};

// Kernel blocks on the device, one GenBlock per slot in storage order, into *out.
int generate_blocks(const double* pts, const KernelParams& kp, const std::vector<std::uint32_t>& idx,
                    const std::vector<GenBlock>& blocks, std::uint64_t elems, double** out, cudaStream_t st) {
  *out = nullptr;
  if (elems == 0) return HMXG_OK;
  std::uint32_t* didx = nullptr;
  GenBlock* dblocks = nullptr;
  HMXG_TRY(dev_upload(&didx, idx.data(), idx.size(), st));
  HMXG_TRY(dev_upload(&dblocks, blocks.data(), blocks.size(), st));
  HMXG_CUDA(cudaMalloc(out, elems * sizeof(double)));
  gen_blocks<<<static_cast<unsigned>(std::min<std::uint64_t>(blocks.size(), 148ull * 16)), 256, 0, st>>>(
      pts, kp, didx, dblocks, blocks.size(), *out);
  HMXG_CUDA(cudaGetLastError());
  HMXG_CUDA(cudaStreamSynchronize(st));
  cudaFree(didx);
  cudaFree(dblocks);
  return HMXG_OK;
}

// dgen (and, with skeletons, bgen) on the device from the points.
int generate_generators(const hmxg_cds_view& v, const Plan& plan, const NearSource& src, double** gd, double** gb,
                        cudaStream_t st, bool near = true) {
  double* pts = nullptr;
  HMXG_TRY(dev_upload(&pts, src.coords, v.n * src.d, st));
  std::vector<GenBlock> blocks(near ? v.num_near : 0);
  for (std::uint64_t s = 0; s < blocks.size(); ++s) {
    const std::uint32_t i = v.near_pairs[2 * s], j = v.near_pairs[2 * s + 1];
    blocks[s] = GenBlock{v.dptr[s], v.start[i], v.start[j], v.end[i] - v.start[i], v.end[j] - v.start[j]};
  }
  const std::vector<std::uint32_t> perm(v.perm, v.perm + v.n);
  int rc = near ? generate_blocks(pts, src.kp, perm, blocks, plan.d_elems, gd, st) : HMXG_OK;
  if (rc == HMXG_OK && src.skel_ptr) {
    blocks.assign(v.num_far, GenBlock{});
    for (std::uint64_t s = 0; s < v.num_far; ++s) {
      const std::uint32_t i = v.far_pairs[2 * s], j = v.far_pairs[2 * s + 1];
      blocks[s] = GenBlock{v.bptr[s], src.skel_ptr[i], src.skel_ptr[j], v.sranks[i], v.sranks[j]};
    }
    const std::vector<std::uint32_t> skel(src.skel_idx, src.skel_idx + src.skel_ptr[v.num_nodes]);
    rc = generate_blocks(pts, src.kp, skel, blocks, plan.b_elems, gb, st);
  }
  cudaFree(pts);
  return rc;
}

// On-the-fly near field (HMXG_UPLOAD_NEAR_ON_THE_FLY): the resident tiles hold every A chunk
// but the near blocks' (compacted), then a scratch region. The combined leaf tasks are cut
// into waves whose near chunks fit it, in task order; their near segments point into the
// scratch at wave-relative offsets, and every evaluation generates a wave's chunks (gen_near)
// right before the wave's leaf rows run.
struct OtfLayout {
  std::vector<SegDev> segs;         // plan.segs, tile offsets re-based
  std::vector<TileSrc> srcs;        // plan.tile_src, tile offsets re-based (near ones unused)
  std::vector<std::uint32_t> cseg;  // resident chunk -> segment
  std::uint64_t resident_elems = 0, scratch_elems = 0;
  std::vector<GenChunk> chunks;
  std::vector<DevState::Wave> waves;
  std::vector<double> wave_flops_per_col, wave_io_per_col;
};
#ifndef HMXG_NEAR_SCRATCH_MB
#define HMXG_NEAR_SCRATCH_MB 2048
#endif
int otf_layout(const Plan& plan, OtfLayout& L) {
  std::uint64_t scratch_bytes = std::uint64_t(HMXG_NEAR_SCRATCH_MB) << 20;
  if (const char* e = std::getenv("HMXG_NEAR_SCRATCH_MB")) scratch_bytes = std::uint64_t(std::max(1, std::atoi(e))) << 20;
  const std::size_t ns = plan.segs.size();
  L.segs = plan.segs;
  L.srcs = plan.tile_src;
  std::vector<std::uint8_t> is_d(ns, 0), placed(ns, 0);
  std::uint64_t off = 0;
  for (std::size_t s = 0; s < ns; ++s) {
    is_d[s] = plan.tile_src[s].gen == kGenD;
    if (is_d[s]) continue;
    L.segs[s].tile_off = off;
    L.srcs[s].tile_off = off;
    for (std::uint32_t c = 0; c < plan.segs[s].nchunks; ++c) L.cseg.push_back(static_cast<std::uint32_t>(s));
    off += std::uint64_t(plan.segs[s].nchunks) * kChunkElems;
  }
  L.resident_elems = off;
  const Phase* leaf = nullptr;
  for (const Phase& ph : plan.phases)
    if (ph.kind == kPhaseLeaf && ph.stage == 0) leaf = &ph;
  if (!leaf) return HMXG_OK;
  auto dchunks = [&](std::uint32_t t) {
    std::uint64_t c = 0;
    for (std::uint32_t si = plan.tasks[t].seg_begin; si < plan.tasks[t].seg_end; ++si)
      if (is_d[si]) c += plan.segs[si].nchunks;
    return c;
  };
  std::uint64_t cap = std::max<std::uint64_t>(1, scratch_bytes / (kChunkElems * sizeof(double)));
  for (std::uint32_t t = leaf->task_begin; t < leaf->task_end; ++t) cap = std::max(cap, dchunks(t));
  std::uint32_t t = leaf->task_begin;
  while (t < leaf->task_end) {
    DevState::Wave w{t, t, L.chunks.size(), 0};
    std::uint64_t woff = 0;  // chunks of the wave so far
    double flops = 0.0, io = 0.0;
    while (t < leaf->task_end && (w.t1 == w.t0 || woff + dchunks(t) <= cap)) {
      const Task& tk = plan.tasks[t];
      for (std::uint32_t si = tk.seg_begin; si < tk.seg_end; ++si) {
        const TileSrc& ts = plan.tile_src[si];
        flops += 2.0 * ts.m * ts.k;
        io += 8.0 * ts.k / std::max<std::uint32_t>(1, plan.yp_tiles[tk.node]);
        if (!is_d[si]) continue;
        if (placed[si]++) return set_err(HMXG_EINVAL, "internal: a near segment in two leaf tasks");
        const std::uint64_t base = L.resident_elems / kChunkElems + woff;
        L.segs[si].tile_off = base * kChunkElems;
        for (std::uint32_t c = 0; c < plan.segs[si].nchunks; ++c) {
          GenChunk g{};
          g.out = base + c;
          g.yrow = tk.c_row;
          g.brow = plan.segs[si].b_row + c * kBK;
          g.m = ts.m;
          g.kvalid = static_cast<std::uint16_t>(std::min<std::uint64_t>(kBK, ts.k - std::uint64_t(c) * kBK));
          L.chunks.push_back(g);
        }
        woff += plan.segs[si].nchunks;
      }
      io += 8.0 * tk.m;
      w.t1 = ++t;
    }
    w.c1 = L.chunks.size();
    L.scratch_elems = std::max(L.scratch_elems, woff * kChunkElems);
    L.waves.push_back(w);
    L.wave_flops_per_col.push_back(flops);
    L.wave_io_per_col.push_back(io);
  }
  return HMXG_OK;
}

int upload_impl(hmxg_ctx* ctx, const hmxg_cds_view* cds, const SplitSpec& split, hmxg_mat** out,
                const NearSource* near_src = nullptr, bool otf = false) {
  if (!ctx || !cds || !out) return set_err(HMXG_EINVAL, "hmxg_upload: null argument");
  if (near_src && split.nparts > 1) return set_err(HMXG_EINVAL, "hmxg_upload: generated near field is single-part");
  *out = nullptr;
  auto mat = std::make_unique<hmxg_mat>();
  mat->ctx = ctx;
  std::string err;
  SplitSpec spec = split;
  spec.flat_tree = spec.flat_tree && std::getenv("HMXG_NO_FLAT") == nullptr;
  if (!build_plan(*cds, kBM, mat->plan, err, spec)) return set_err(HMXG_EINVAL, err);
  OtfLayout otf_l;
  if (otf) {
    if (!near_src || split.nparts != 1) return set_err(HMXG_EINVAL, "hmxg_upload: near field on the fly needs points");
    mat->plan.near_otf = true;
    HMXG_TRY(otf_layout(mat->plan, otf_l));
  }
  const double* gsrc[3] = {cds->dgen, cds->bgen, cds->vgen};
  std::vector<double> gcompact[3];
  if (split.nparts > 1) HMXG_TRY(compact_generators(*cds, mat->plan, gsrc, gcompact));
  const Plan& plan = mat->plan;
  mat->devs.resize(ctx->devs.size());
  for (std::size_t g = 0; g < ctx->devs.size(); ++g) {
    DevState& d = mat->devs[g];
    d.dev = ctx->devs[g];
    HMXG_CUDA(cudaSetDevice(d.dev));
    for (cudaStream_t* st : {&d.comp, &d.h2d, &d.d2h}) HMXG_CUDA(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&d.ev0, &d.ev1}) HMXG_CUDA(cudaEventCreate(e));
    for (int b = 0; b < 2; ++b)
      for (cudaEvent_t* e : {&d.ev_in[b], &d.ev_done[b], &d.ev_out[b]})
        HMXG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    HMXG_CUDA(cudaEventCreateWithFlags(&d.ev_last, cudaEventDisableTiming));
    d.phase_ev.resize(plan.phases.size() + plan.split_phases.size() + plan.flat_phases.size() + 3 +
                      2 * otf_l.waves.size());
    for (auto& e : d.phase_ev) HMXG_CUDA(cudaEventCreate(&e));
    HMXG_CUDA(cudaFuncSetAttribute(grouped_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    HMXG_CUDA(cudaFuncSetAttribute(eval_dag<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    HMXG_CUDA(cudaFuncSetAttribute(eval_dag<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    {
      int per_sm = 0, sms = 0;
      int per_sm_dag = 0;
      HMXG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, grouped_gemm, kThreads, kSmemBytes));
      int per_sm_narrow = 0;
      HMXG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_dag, eval_dag<false>, kThreads, kSmemBytes));
      HMXG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_narrow, eval_dag<true>, kThreads, kSmemBytes));
      per_sm_dag = std::min(per_sm_dag, per_sm_narrow);
      // eval_dag relies on every CTA of its grid being resident (items wait on earlier items)
      per_sm = std::min(per_sm, per_sm_dag);
      HMXG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d.dev));
#ifndef HMXG_GEMM_CTAS_PER_SM
#define HMXG_GEMM_CTAS_PER_SM 3
#endif
      d.gemm_grid = static_cast<unsigned>(std::max(1, std::min(per_sm, HMXG_GEMM_CTAS_PER_SM)) * sms);
      HMXG_CUDA(cudaMalloc(&d.tile_counters,
                           std::max<std::size_t>(1, plan.phases.size() + plan.split_phases.size() +
                                                        plan.flat_phases.size() + otf_l.waves.size()) *
                               sizeof(std::uint32_t)));
    }
    // raw generators -> pre-tiled A operands on the device, then the raw copies go away
    double *gd = nullptr, *gb = nullptr, *gv = nullptr;
    TileSrc* srcs = nullptr;
    std::uint32_t* cseg = nullptr;
    if (near_src)
      HMXG_TRY(generate_generators(*cds, plan, *near_src, &gd, &gb, d.comp, /*near=*/!otf));
    else
      HMXG_TRY(dev_upload(&gd, gsrc[kGenD], plan.d_elems, d.comp));
    if (!near_src || !near_src->skel_ptr) HMXG_TRY(dev_upload(&gb, gsrc[kGenB], plan.b_elems, d.comp));
    HMXG_TRY(dev_upload(&gv, gsrc[kGenV], plan.v_elems, d.comp));
    double* gc = nullptr;  // the flat tree's composite blocks (Plan::cgen)
    HMXG_TRY(dev_upload(&gc, plan.cgen.data(), plan.cgen.size(), d.comp));
    const std::vector<TileSrc>& tsrc = otf ? otf_l.srcs : plan.tile_src;
    const std::vector<std::uint32_t>& tcseg = otf ? otf_l.cseg : plan.chunk_seg;
    const std::uint64_t tile_elems = otf ? otf_l.resident_elems + otf_l.scratch_elems : plan.tile_elems;
    HMXG_TRY(dev_upload(&srcs, tsrc.data(), tsrc.size(), d.comp));
    HMXG_TRY(dev_upload(&cseg, tcseg.data(), tcseg.size(), d.comp));
    std::uint32_t* maps = nullptr;
    HMXG_TRY(dev_upload(&maps, plan.maps.data(), plan.maps.size(), d.comp));
    d.tile_elems = tile_elems;
    if (tile_elems) {
      HMXG_CUDA(cudaMalloc(&d.tiles, tile_elems * sizeof(double)));
      const std::uint64_t nch = tcseg.size();
      if (nch)
        tile_a<<<static_cast<unsigned>(std::min<std::uint64_t>(nch, 1u << 20)), 256, 0, d.comp>>>(gd, gb, gv, gc, srcs,
                                                                                                 cseg, maps, d.tiles, nch);
      HMXG_CUDA(cudaGetLastError());
    }
    if (otf) {  // the points and every wave's near chunks; the near blocks themselves never exist
      const std::size_t gsm = 80 * std::size_t(near_src->d) * sizeof(double);
      if (gsm > 200 * 1024) return set_err(HMXG_EINVAL, "hmxg_upload: near field on the fly supports d <= 320");
      HMXG_CUDA(cudaFuncSetAttribute(gen_near, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gsm)));
      HMXG_TRY(dev_upload(&d.pts, near_src->coords, cds->n * near_src->d, d.comp));
      HMXG_TRY(dev_upload(&d.gen_chunks, otf_l.chunks.data(), otf_l.chunks.size(), d.comp));
      d.kp = near_src->kp;
      d.otf_segs = otf_l.segs;
      d.waves = otf_l.waves;
      d.wave_flops = otf_l.wave_flops_per_col;
      d.wave_io = otf_l.wave_io_per_col;
    }
    HMXG_CUDA(cudaStreamSynchronize(d.comp));
    cudaFree(gd);
    cudaFree(gb);
    cudaFree(gv);
    cudaFree(gc);
    cudaFree(srcs);
    cudaFree(cseg);
    cudaFree(maps);
    HMXG_TRY(dev_upload(&d.tasks, plan.tasks.data(), plan.tasks.size(), d.comp));
    HMXG_TRY(dev_upload(&d.segs, otf ? otf_l.segs.data() : plan.segs.data(), plan.segs.size(), d.comp));
    HMXG_TRY(dev_upload(&d.idmap, plan.idmap.data(), plan.idmap.size(), d.comp));
    HMXG_TRY(dev_upload(&d.ipmap, plan.ipmap.data(), plan.ipmap.size(), d.comp));
    HMXG_TRY(dev_upload(&d.node_tiles, plan.node_tiles.data(), plan.node_tiles.size(), d.comp));
    HMXG_TRY(dev_upload(&d.yp_tiles, plan.yp_tiles.data(), plan.yp_tiles.size(), d.comp));
    HMXG_TRY(dev_upload(&d.remote_t, plan.remote_t_nodes.data(), plan.remote_t_nodes.size(), d.comp));
    if (split.nparts == 1) {  // the fused permutations of small problems
      HMXG_TRY(dev_upload(&d.pmap, plan.pmap.data(), plan.pmap.size(), d.comp));
      std::vector<std::uint32_t> rowleaf(plan.rows_pad, 0), target(plan.num_nodes, 0);
      for (std::uint32_t i = 0; i < plan.num_nodes; ++i)
        if (cds->lchild[i] == HMXG_NO_NODE) {
          target[i] = cds->end[i] - cds->start[i];
          for (std::uint32_t r = 0; r < target[i]; ++r) rowleaf[plan.leaf_row[i] + r] = i;
        }
      HMXG_TRY(dev_upload(&d.rowleaf, rowleaf.data(), rowleaf.size(), d.comp));
      HMXG_TRY(dev_upload(&d.wp_target, target.data(), target.size(), d.comp));
    }
    {
      const char* pz = std::getenv("HMXG_POISON");
      d.poison = split.nparts == 1 && pz && *pz && std::strcmp(pz, "0") != 0;
      if (d.poison) {
        std::vector<std::uint32_t> live;
        for (std::uint32_t i = 0; i < plan.num_nodes; ++i)
          if (cds->participating[i] && cds->sranks[i] > 0)
            for (std::uint32_t r = 0; r < cds->sranks[i]; ++r) live.push_back(static_cast<std::uint32_t>(plan.node_off[i] + r));
        HMXG_TRY(dev_upload(&d.ts_live, live.data(), live.size(), d.comp));
        d.ts_live_count = live.size();
      }
    }
    HMXG_CUDA(cudaStreamSynchronize(d.comp));
    d.resident_bytes = 8 * tile_elems + sizeof(Task) * plan.tasks.size() + sizeof(SegDev) * plan.segs.size() +
                       (otf ? 8 * cds->n * near_src->d + sizeof(GenChunk) * otf_l.chunks.size() : 0) +
                       4 * plan.ipmap.size() + 4 * plan.idmap.size();
  }
  *out = mat.release();
  return HMXG_OK;
}

// The caller's collective over contiguous row blocks [row[r], row[r + 1]) of a point-major
// buffer (row pitch ld doubles), in place; HMXG_ECOMM when it fails.
int comm_allgather_rows(const hmxg_comm& cm, DevState& d, double* base, std::uint64_t ld,
                        const std::vector<std::uint64_t>& row, cudaStream_t st) {
  const std::size_t P = cm.size, rb = ld * sizeof(double);
  std::vector<std::size_t> counts(P), displs(P);
  for (std::size_t r = 0; r < P; ++r) {
    displs[r] = row[r] * rb;
    counts[r] = (row[r + 1] - row[r]) * rb;
  }
  const std::size_t total = row[P] * rb;
  if (total == 0) return HMXG_OK;
  int rc = 0;
  if (cm.host_buffers) {
    if (total > d.comm_host_bytes) {
      cudaFreeHost(d.comm_host);
      d.comm_host = nullptr;
      d.comm_host_bytes = 0;
      HMXG_CUDA(cudaHostAlloc(&d.comm_host, total, cudaHostAllocPortable));
      d.comm_host_bytes = total;
    }
    unsigned char* dev = reinterpret_cast<unsigned char*>(base);
    const std::size_t me = cm.rank;
    if (counts[me]) HMXG_CUDA(cudaMemcpyAsync(d.comm_host + displs[me], dev + displs[me], counts[me], cudaMemcpyDeviceToHost, st));
    HMXG_CUDA(cudaStreamSynchronize(st));
    rc = cm.allgatherv(cm.user, d.comm_host + displs[me], counts[me], d.comm_host, counts.data(), displs.data(), nullptr);
    if (rc == 0) HMXG_CUDA(cudaMemcpyAsync(dev, d.comm_host, total, cudaMemcpyHostToDevice, st));
  } else {
    unsigned char* dev = reinterpret_cast<unsigned char*>(base);
    rc = cm.allgatherv(cm.user, dev + displs[cm.rank], counts[cm.rank], dev, counts.data(), displs.data(), st);
  }
  if (rc != 0) return set_err(HMXG_ECOMM, "hmxg_evaluate: allgatherv failed (" + std::to_string(rc) + ")");
  return HMXG_OK;
}

// Collective evaluation of a subtree-split matrix (hmxg_create_comm, CDS over the HBM
// budget): every rank passes the same full W. Stage 0 runs the upward pass over the rank's
// subtrees; the ranks all-gather the T rows other parts read (Plan::pub_row); stage 1 runs
// the replicated top levels, far+downward and the near/leaf rows of the rank's leaves; the
// ranks all-gather their Yp rows (Plan::yp_row) and every rank permutes out the full Y.
int split_evaluate(hmxg_mat* mat, const double* W, std::size_t ldw, double* Y, std::size_t ldy, std::size_t q,
                   unsigned flags, void* stream, std::uint32_t* launches) {
  const Plan& plan = mat->plan;
  const hmxg_comm& cm = mat->ctx->comm;
  if (cm.size != plan.nparts || cm.rank != plan.part)
    return set_err(HMXG_EINVAL, "hmxg_evaluate: a split matrix evaluates through its hmxg_create_comm context "
                                "(or stage by stage with hmxg_split_stage)");
  DevState& d = mat->devs[0];
  HMXG_CUDA(cudaSetDevice(d.dev));
  const bool dev_ptrs = flags & HMXG_F_DEVICE_PTRS;
  cudaStream_t st = dev_ptrs && stream ? static_cast<cudaStream_t>(stream) : d.comp;
  const std::size_t n = plan.n;
  const double* Wd = W;
  double* Yd = Y;
  std::size_t ldwd = ldw, ldyd = ldy;
  HMXG_TRY(ensure_workspace(plan, d, q));
  if (!dev_ptrs) {
    HMXG_TRY(ensure_stage(plan, d, q));
    HMXG_TRY(copy_cols(d.w_stage[0], n, W, ldw, n, q, cudaMemcpyHostToDevice, st));
    Wd = d.w_stage[0];
    Yd = d.y_stage[0];
    ldwd = ldyd = n;
  }
  const DevState::DagItems* di[2] = {nullptr, nullptr};
  for (std::uint32_t stage = 0; stage < 2; ++stage) HMXG_TRY(ensure_dag(plan, d, q, st, &di[stage], stage));
  HMXG_TRY(order_after_previous(d, st));
  const std::uint32_t qq = static_cast<std::uint32_t>(q), nn = static_cast<std::uint32_t>(n);
  const std::uint64_t ldq = d.cap_q;
  const std::uint32_t ncb = (qq + kBN - 1) / kBN;
  const std::size_t words = dag_done_words(plan, q);
  CUtensorMap tm_wp, tm_t, tm_s;
  HMXG_TRY(make_map(&tm_wp, d.wp, plan.rows_pad, q, ldq));
  HMXG_TRY(make_map(&tm_t, d.t, plan.skel_rows, q, ldq));
  HMXG_TRY(make_map(&tm_s, d.s, plan.skel_rows, q, ldq));
  GemmParams p{};
  p.tiles = d.tiles;
  p.tasks = d.tasks;
  p.segs = d.segs;
  p.idmap = d.idmap;
  p.buf[kBufWp] = d.wp;
  p.buf[kBufT] = d.t;
  p.buf[kBufS] = d.s;
  p.buf[kBufYp] = d.yp;
  for (auto& l : p.ld) l = ldq;
  p.q = qq;
  const dim3 pgrid((nn + kTT - 1) / kTT, (qq + kTT - 1) / kTT);
  if (pgrid.y > 65535) return set_err(HMXG_EINVAL, "hmxg_evaluate: too many columns for one call");
  d.counters_dirty = true;
  HMXG_CUDA(cudaMemsetAsync(d.t, 0, plan.skel_rows * ldq * sizeof(double), st));
  HMXG_CUDA(cudaMemsetAsync(d.yp, 0, plan.rows_pad * ldq * sizeof(double), st));
  HMXG_CUDA(cudaMemsetAsync(d.dag_done, 0, (words + 1) * sizeof(std::uint32_t), st));
  permute_in<<<pgrid, 256, 0, st>>>(Wd, ldwd, d.ipmap, d.wp, ldq, nn, qq, nullptr, 0);
  ++*launches;
  for (std::uint32_t stage = 0; stage < 2; ++stage) {
    DagParams dp{};
    dp.recs = di[stage]->recs;
    dp.per_task = di[stage]->per_task;
    dp.parts = di[stage]->parts;
    dp.nitems = di[stage]->nitems;
    dp.claim = d.dag_done + stage;
    dp.done = d.dag_done + kDagClaimWords;
    dp.node_tiles = d.node_tiles;
    dp.yp_tiles = d.yp_tiles;
    dp.signal_yp = split_leaf(plan, q, d.gemm_grid) ? 1u : 0u;
    dp.colsplit = 1;
    dp.cstride = 1;
    dp.ncb = ncb;
    dp.nodes = plan.num_nodes;
    dp.fwd_signals = forward_signals(di[stage]->nitems, d.gemm_grid);
    if (stage == 1) {
      // the T rows other parts publish, then their completion for stage 1's waits
      HMXG_TRY(comm_allgather_rows(cm, d, d.t, ldq, plan.pub_row, st));
      if (!plan.remote_t_nodes.empty()) {
        const std::uint64_t cells = std::uint64_t(plan.remote_t_nodes.size()) * ncb;
        preset_done<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, st>>>(
            d.remote_t, static_cast<std::uint32_t>(plan.remote_t_nodes.size()), dp.done, ncb, d.node_tiles);
        ++*launches;
      }
    }
    if (dp.nitems) {
      const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(dp.nitems, d.gemm_grid));
      eval_dag<false><<<grid, kThreads, kSmemBytes, st>>>(tm_wp, tm_t, tm_s, p, dp);
      ++*launches;
    }
  }
  HMXG_TRY(comm_allgather_rows(cm, d, d.yp, ldq, plan.yp_row, st));  // every part's result rows
  permute_out<<<pgrid, 256, 0, st>>>(d.yp, ldq, d.ipmap, Yd, ldyd, nn, qq, d.dag_done, words + 1);
  ++*launches;
  HMXG_CUDA(cudaGetLastError());
  d.counters_dirty = false;
  d.last_fused = false;
  d.last_launches = *launches;
  d.launch_desc.clear();  // (the subtree-split stages are not described per launch)
  if (!dev_ptrs) HMXG_TRY(copy_cols(Y, ldy, d.y_stage[0], n, n, q, cudaMemcpyDeviceToHost, st));
  if (!dev_ptrs || !(flags & HMXG_F_NO_SYNC)) {
    HMXG_CUDA(cudaStreamSynchronize(st));
    d.pending = false;
  } else {
    HMXG_CUDA(cudaEventRecord(d.ev_last, st));
    d.pending = true;
  }
  return HMXG_OK;
}

}  // namespace
}  // namespace hmxg

using namespace hmxg;

extern "C" {

const char* hmxg_last_error(void) { return g_err.c_str(); }
const char* hmxg_version(void) {
  return "hmxg 0.4 sm_100a fp64-dmma tma-pipelined dag; identity-row lowering; generated blocks; gpu id";
}

int hmxg_create(const int* devs, int ndev, hmxg_ctx** out) {
  if (!out) return set_err(HMXG_EINVAL, "hmxg_create: null out");
  *out = nullptr;
  int count = 0;
  HMXG_CUDA(cudaGetDeviceCount(&count));
  if (count == 0) return set_err(HMXG_ECUDA, "hmxg_create: no CUDA device");
  auto ctx = std::make_unique<hmxg_ctx>();
  if (ndev <= 0 || !devs) {
    ctx->devs.push_back(0);
  } else {
    for (int i = 0; i < ndev; ++i) {
      if (devs[i] < 0 || devs[i] >= count) return set_err(HMXG_EINVAL, "hmxg_create: device id out of range");
      ctx->devs.push_back(devs[i]);
    }
  }
  for (int dv : ctx->devs) {
    cudaDeviceProp prop{};
    HMXG_CUDA(cudaGetDeviceProperties(&prop, dv));
    if (prop.major != 10) return set_err(HMXG_ECUDA, "hmxg_create: built for sm_100a (B200) only");
  }
  *out = ctx.release();
  return HMXG_OK;
}

int hmxg_create_comm(int dev, const hmxg_comm* comm, hmxg_ctx** out) {
  if (!out || !comm) return set_err(HMXG_EINVAL, "hmxg_create_comm: null argument");
  *out = nullptr;
  if (comm->size == 0 || comm->rank >= comm->size) return set_err(HMXG_EINVAL, "hmxg_create_comm: bad rank / size");
  if (comm->size > 1 && !comm->allgatherv) return set_err(HMXG_EINVAL, "hmxg_create_comm: no allgatherv");
  hmxg_ctx* ctx = nullptr;
  HMXG_TRY(hmxg_create(&dev, 1, &ctx));
  ctx->comm = *comm;
  *out = ctx;
  return HMXG_OK;
}

int hmxg_destroy(hmxg_ctx* ctx) {
  delete ctx;
  return HMXG_OK;
}

}  // extern "C"

namespace hmxg {
namespace {
// Content fingerprint of a CDS view (hmxg_cds_fingerprint): xxHash64-style rounds (four
// 64-bit lanes, multiply-rotate-multiply, then an avalanche) over every array, 4 MiB blocks
// hashed in parallel and combined in order. One pass over the CDS at host memory bandwidth.
constexpr std::uint64_t kP1 = 0x9E3779B185EBCA87ull, kP2 = 0xC2B2AE3D27D4EB4Full, kP3 = 0x165667B19E3779F9ull,
                        kP4 = 0x85EBCA77C2B2AE63ull, kP5 = 0x27D4EB2F165667C5ull;
inline std::uint64_t rotl64(std::uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }
inline std::uint64_t fp_round(std::uint64_t acc, std::uint64_t in) { return rotl64(acc + in * kP2, 31) * kP1; }
inline std::uint64_t fp_avalanche(std::uint64_t h) {
  h ^= h >> 33;
  h *= kP2;
  h ^= h >> 29;
  h *= kP3;
  return h ^ (h >> 32);
}
std::uint64_t fp_block(const unsigned char* p, std::size_t len, std::uint64_t seed) {
  std::uint64_t a[4] = {seed + kP1 + kP2, seed + kP2, seed, seed - kP1};
  std::size_t i = 0;
  for (; i + 32 <= len; i += 32)
    for (int l = 0; l < 4; ++l) {
      std::uint64_t w;
      std::memcpy(&w, p + i + 8 * l, 8);  // generators inside a mapped file need not be aligned
      a[l] = fp_round(a[l], w);
    }
  std::uint64_t h = rotl64(a[0], 1) + rotl64(a[1], 7) + rotl64(a[2], 12) + rotl64(a[3], 18) + len;
  for (; i < len; ++i) h = rotl64(h ^ (p[i] * kP5), 11) * kP1;
  return fp_avalanche(h);
}
std::uint64_t fp_array(const void* data, std::size_t bytes, std::uint64_t h) {
  constexpr std::size_t kBlock = std::size_t(4) << 20;
  const auto* p = static_cast<const unsigned char*>(data);
  const std::size_t nb = (bytes + kBlock - 1) / kBlock;
  std::vector<std::uint64_t> bh(nb);
  auto work = [&](std::size_t b0, std::size_t b1) {
    for (std::size_t b = b0; b < b1; ++b) bh[b] = fp_block(p + b * kBlock, std::min(kBlock, bytes - b * kBlock), b);
  };
  const std::size_t t = std::min<std::size_t>(std::max(1u, std::thread::hardware_concurrency()), nb);
  if (t <= 1) {
    work(0, nb);
  } else {
    std::vector<std::thread> pool;
    for (std::size_t k = 1; k < t; ++k) pool.emplace_back(work, nb * k / t, nb * (k + 1) / t);
    work(0, nb / t);
    for (auto& th : pool) th.join();
  }
  h = fp_round(h, bytes);
  for (std::uint64_t x : bh) h = fp_round(h ^ x, kP4);
  return h;
}
}  // namespace
}  // namespace hmxg

extern "C" {

int hmxg_cds_fingerprint(const hmxg_cds_view* v, uint64_t* out) {
  if (!v || !out) return set_err(HMXG_EINVAL, "hmxg_cds_fingerprint: null argument");
  const std::size_t nn = v->num_nodes, n = v->n;
  std::uint64_t h = fp_round(fp_round(kP5, n), (std::uint64_t(v->height) << 32) | nn);
  auto arr = [&](const void* p, std::size_t bytes) {
    if (bytes && !p) return false;
    h = fp_array(p, bytes, h);
    return true;
  };
  bool ok = arr(v->parent, 4 * nn) && arr(v->lchild, 4 * nn) && arr(v->rchild, 4 * nn) && arr(v->start, 4 * nn) &&
            arr(v->end, 4 * nn) && arr(v->level, 4 * nn) && arr(v->perm, 4 * n) && arr(v->sranks, 4 * nn) &&
            arr(v->participating, nn) && arr(v->near_pairs, 8 * v->num_near) && arr(v->far_pairs, 8 * v->num_far) &&
            arr(v->v_order, 4 * v->num_v) && arr(v->dptr, 8 * (v->num_near + 1)) &&
            arr(v->bptr, 8 * (v->num_far + 1)) && arr(v->vptr, 8 * (v->num_v + 1));
  if (!ok) return set_err(HMXG_EINVAL, "cds: null array in view");
  // generator extents come from the offset arrays (the view was checked to hold them above)
  ok = arr(v->dgen, 8 * v->dptr[v->num_near]) && arr(v->bgen, 8 * v->bptr[v->num_far]) &&
       arr(v->vgen, 8 * v->vptr[v->num_v]);
  if (!ok) return set_err(HMXG_EINVAL, "cds: null generator in view");
  *out = fp_avalanche(h);
  return HMXG_OK;
}

int hmxg_validate(const hmxg_cds_view* cds, hmxg_info* info) {
  if (!cds) return set_err(HMXG_EINVAL, "hmxg_validate: null view");
  Plan plan;
  std::string err;
  if (!build_plan(*cds, kBM, plan, err, plan_spec())) return set_err(HMXG_EINVAL, err);
  if (info) {
    std::memset(info, 0, sizeof *info);
    info->n = plan.n;
    info->d_elems = plan.d_elems;
    info->b_elems = plan.b_elems;
    info->v_elems = plan.v_elems;
    info->skel_rows = plan.skel_rows;
    info->launches_per_eval = 3;
    info->flops_per_col = 2.0 * (2.0 * plan.v_elems + plan.b_elems + plan.d_elems);
    for (const Phase* ph : tree_phases(plan, 0)) info->exec_flops_per_col += ph->flops_per_col;
    for (const Phase& ph : plan.phases)
      if (ph.kind == kPhaseLeaf) info->exec_flops_per_col += ph.flops_per_col;
  }
  return HMXG_OK;
}


namespace hmxg {
namespace {
// hmxg_dag_check in CTree mode: the items are the near tiles, each once per column block and
// part; the CTree levels hold every other task of the split variant exactly once, and every
// T / S row block a level reads (B operand or identity rows) is complete at an earlier level;
// the accumulating leaf rows read near tiles, which the items write completely.
int ct_check(const Plan& plan, const std::vector<std::uint64_t>& items, std::uint32_t q, std::uint32_t S) {
  const std::uint32_t ncb = (q + kBN - 1) / kBN;
  const std::size_t nn = plan.num_nodes, nt = plan.tasks.size();
  std::vector<std::uint8_t> is_near(nt, 0), in_ct(nt, 0);
  for (const Phase& ph : plan.split_phases)
    if (ph.kind == kPhaseNear)
      for (std::uint32_t t = ph.task_begin; t < ph.task_end; ++t) is_near[t] = 1;
  std::vector<std::uint8_t> seen(nt * std::size_t(ncb) * S, 0);
  for (std::uint64_t it : items) {
    const std::uint32_t t = static_cast<std::uint32_t>(it), cb = item_cb(it), sub = item_sub(it);
    if (t >= nt || cb >= ncb || sub >= S || !is_near[t] || seen[(std::size_t(t) * ncb + cb) * S + sub]++)
      return set_err(HMXG_EINVAL, "dag: CTree item list is not the near tiles x column blocks x parts");
  }
  if (items.size() != [&] {
        std::size_t c = 0;
        for (std::size_t t = 0; t < nt; ++t) c += is_near[t];
        return c * ncb * S;
      }())
    return set_err(HMXG_EINVAL, "dag: a near tile is missing");
  const std::vector<const Phase*> lv = ct_levels(plan);
  std::vector<std::uint32_t> wr(3 * nn, 0), done(3 * nn, 0);
  for (const Phase* ph : lv)
    for (std::uint32_t t = ph->task_begin; t < ph->task_end; ++t) {
      if (in_ct[t]++ || is_near[t]) return set_err(HMXG_EINVAL, "dag: a CTree task appears twice");
      const Task& tk = plan.tasks[t];
      if (tk.cbuf == kBufT) ++wr[tk.node];
      if (tk.cbuf == kBufS) ++wr[nn + tk.node];
    }
  for (std::size_t t = 0; t < nt; ++t) {
    if (is_near[t]) ++wr[2 * nn + plan.tasks[t].node];
    if (!is_near[t] && !in_ct[t]) {  // a task of the combined leaf variant only
      bool combined = false;
      for (const Phase& ph : plan.phases)
        if (ph.kind == kPhaseLeaf && t >= ph.task_begin && t < ph.task_end) combined = true;
      if (!combined) return set_err(HMXG_EINVAL, "dag: a task is neither a near tile nor in the CTree");
    }
  }
  for (std::size_t i = 0; i < nn; ++i) {
    if (wr[i] && wr[i] != plan.node_tiles[i]) return set_err(HMXG_EINVAL, "dag: T writers != node tiles");
    if (wr[nn + i] && wr[nn + i] != plan.node_tiles[i]) return set_err(HMXG_EINVAL, "dag: S writers != node tiles");
    if (wr[2 * nn + i] != plan.yp_tiles[i]) return set_err(HMXG_EINVAL, "dag: Yp writers != near tiles");
  }
  auto ready = [&](std::size_t r) { return done[r] >= wr[r]; };
  for (const Phase* ph : lv) {
    for (std::uint32_t t = ph->task_begin; t < ph->task_end; ++t) {
      const Task& tk = plan.tasks[t];
      for (std::uint32_t sgi = tk.seg_begin; sgi < tk.seg_end; ++sgi) {
        const SegDev& sg = plan.segs[sgi];
        if ((sg.bbuf == kBufT || sg.bbuf == kBufS) && !(wr[(sg.bbuf == kBufT ? 0 : nn) + sg.src] &&
                                                        ready((sg.bbuf == kBufT ? 0 : nn) + sg.src)))
          return set_err(HMXG_EINVAL, "dag: a CTree level reads T / S rows of a later level");
      }
      if (tk.id_off != kNoMap && (tk.id_buf == kBufT || tk.id_buf == kBufS))
        for (std::uint32_t nd : {tk.id_node0, tk.id_node1})
          if (nd != kNoMap && !ready((tk.id_buf == kBufT ? 0 : nn) + nd))
            return set_err(HMXG_EINVAL, "dag: a CTree level copies identity rows of a later level");
      if (tk.flags & kTaskAccumulate && !wr[2 * nn + tk.node])
        return set_err(HMXG_EINVAL, "dag: a CTree leaf task has no near tiles");
    }
    for (std::uint32_t t = ph->task_begin; t < ph->task_end; ++t) {  // the level's rows, after its reads
      const Task& tk = plan.tasks[t];
      if (tk.cbuf == kBufT) ++done[tk.node];
      if (tk.cbuf == kBufS) ++done[nn + tk.node];
    }
  }
  return HMXG_OK;
}
}  // namespace
}  // namespace hmxg

int hmxg_dag_items(const hmxg_cds_view* cds, size_t q, uint32_t grid, uint64_t* out, size_t cap, uint64_t* nitems) {
  if (!cds || q == 0 || grid == 0 || (cap && !out))
    return set_err(HMXG_EINVAL, "hmxg_dag_items: null view or buffer, q = 0 or grid = 0");
  Plan plan;
  std::string err;
  if (!build_plan(*cds, kBM, plan, err, plan_spec())) return set_err(HMXG_EINVAL, err);
  const std::vector<std::uint64_t> items = build_items(plan, static_cast<std::uint32_t>(q), 0, grid);
  if (nitems) *nitems = items.size();
  for (std::size_t i = 0; i < std::min<std::size_t>(cap, items.size()); ++i) out[i] = items[i];
  return HMXG_OK;
}

int hmxg_dag_check(const hmxg_cds_view* cds, size_t q, uint32_t grid, uint64_t* nitems) {
  if (!cds || q == 0 || grid == 0) return set_err(HMXG_EINVAL, "hmxg_dag_check: null view, q = 0 or grid = 0");
  Plan plan;
  std::string err;
  if (!build_plan(*cds, kBM, plan, err, plan_spec())) return set_err(HMXG_EINVAL, err);
  const std::uint32_t ncb = static_cast<std::uint32_t>((q + kBN - 1) / kBN);
  const std::vector<std::uint64_t> items = build_items(plan, static_cast<std::uint32_t>(q), 0, grid);
  if (nitems) *nitems = items.size();
  const double f = split_frac(plan, q, grid);
  const bool split = f > 0.0;  // (some) leaves run the split variant
  const std::vector<std::uint8_t> sel = split_set(plan, f);
  const std::uint32_t S = colsplit(plan, q, grid);  // parts per tile: every tile appears S times
  if (ctree_csize(plan, q, grid)) return ct_check(plan, items, static_cast<std::uint32_t>(q), S);
  // (1) every task of the variant that runs, once per column block: the tree phases, the
  // combined leaf tasks of the leaves not split, the near and accumulating tasks of the split
  // ones (every near task when f = 1)
  std::vector<std::uint32_t> want(plan.tasks.size(), 0), seen(plan.tasks.size() * std::size_t(ncb), 0);
  std::vector<std::uint8_t> is_near(plan.tasks.size(), 0);
  for (const Phase* ph : tree_phases(plan, 0))
    for (std::uint32_t t = ph->task_begin; t < ph->task_end; ++t) want[t] = 1;
  for (const Phase& ph : plan.phases)
    if (ph.kind == kPhaseLeaf)
      for (std::uint32_t t = ph.task_begin; t < ph.task_end; ++t)
        if (f < 1.0 && !sel[plan.tasks[t].node]) want[t] = 1;
  if (split)
    for (const Phase& ph : plan.split_phases)
      for (std::uint32_t t = ph.task_begin; t < ph.task_end; ++t)
        if (f >= 1.0 || sel[plan.tasks[t].node]) {
          want[t] = 1;
          if (ph.kind == kPhaseNear) is_near[t] = 1;
        }
  std::vector<std::uint8_t> seen_sub(plan.tasks.size() * std::size_t(ncb) * S, 0);
  for (std::uint64_t it : items) {
    const std::uint32_t t = static_cast<std::uint32_t>(it), cb = item_cb(it), sub = item_sub(it);
    if (t >= plan.tasks.size() || cb >= ncb || sub >= S || !want[t] ||
        seen_sub[(std::size_t(t) * ncb + cb) * S + sub]++)
      return set_err(HMXG_EINVAL, "dag: item list is not the variant's tasks x column blocks x parts");
    ++seen[std::size_t(t) * ncb + cb];
  }
  for (std::size_t t = 0; t < plan.tasks.size(); ++t)
    for (std::uint32_t cb = 0; cb < ncb; ++cb)
      if (want[t] && seen[t * ncb + cb] != S) return set_err(HMXG_EINVAL, "dag: a task tile is missing");
  // (3) the kernel's completion targets are the writer counts
  const std::size_t nn = plan.num_nodes;
  std::vector<std::uint32_t> wr(3 * nn, 0);
  for (std::size_t t = 0; t < plan.tasks.size(); ++t) {
    if (!want[t]) continue;
    const Task& tk = plan.tasks[t];
    if (tk.cbuf == kBufT) ++wr[tk.node];
    if (tk.cbuf == kBufS) ++wr[nn + tk.node];
    if (is_near[t]) ++wr[2 * nn + tk.node];
  }
  for (std::size_t i = 0; i < nn; ++i) {
    if (wr[i] && wr[i] != plan.node_tiles[i]) return set_err(HMXG_EINVAL, "dag: T target != writer tiles");
    if (wr[nn + i] && wr[nn + i] != plan.node_tiles[i]) return set_err(HMXG_EINVAL, "dag: S target != writer tiles");
    if (split && (f >= 1.0 || sel[i]) && wr[2 * nn + i] != plan.yp_tiles[i])
      return set_err(HMXG_EINVAL, "dag: Yp target != near tiles");
  }
  // (2) topological: every tile an item waits for is complete before it in the claim order
  std::vector<std::uint32_t> done(3 * nn * std::size_t(ncb), 0);
  auto ready = [&](std::size_t r, std::uint32_t cb) { return done[r * ncb + cb] >= wr[r] * S; };
  for (std::uint64_t it : items) {
    const std::uint32_t t = static_cast<std::uint32_t>(it), cb = item_cb(it);
    const Task& tk = plan.tasks[t];
    for (std::uint32_t sgi = tk.seg_begin; sgi < tk.seg_end; ++sgi) {
      const SegDev& sg = plan.segs[sgi];
      if ((sg.bbuf == kBufT || sg.bbuf == kBufS) && !ready((sg.bbuf == kBufT ? 0 : nn) + sg.src, cb))
        return set_err(HMXG_EINVAL, "dag: an item precedes the tiles its B operand reads");
    }
    if (tk.id_off != kNoMap && (tk.id_buf == kBufT || tk.id_buf == kBufS))
      for (std::uint32_t nd : {tk.id_node0, tk.id_node1})
        if (nd != kNoMap && !ready((tk.id_buf == kBufT ? 0 : nn) + nd, cb))
          return set_err(HMXG_EINVAL, "dag: an item precedes the tiles its identity rows copy");
    if ((tk.flags & kTaskAccumulate) && !ready(2 * nn + tk.node, cb))
      return set_err(HMXG_EINVAL, "dag: a leaf task precedes its near tiles");
    if (tk.cbuf == kBufT) ++done[std::size_t(tk.node) * ncb + cb];
    if (tk.cbuf == kBufS) ++done[(nn + tk.node) * ncb + cb];
    if (is_near[t]) ++done[(2 * nn + tk.node) * ncb + cb];
  }
  return HMXG_OK;
}

int hmxg_upload(hmxg_ctx* ctx, const hmxg_cds_view* cds, hmxg_mat** out) {
  if (ctx && cds && ctx->comm.size > 1) {
    // one process per GPU: replicate while the resident CDS fits the budget, else hold this
    // rank's subtree part (SURVEY §8e fallback)
    Plan probe;
    std::string err;
    if (!build_plan(*cds, kBM, probe, err, plan_spec())) return set_err(HMXG_EINVAL, err);
    const std::uint64_t bytes = 8 * probe.tile_elems + sizeof(Task) * probe.tasks.size() +
                                sizeof(SegDev) * probe.segs.size() + 4 * (probe.ipmap.size() + probe.idmap.size());
    std::uint64_t budget = ctx->comm.hbm_budget;
    if (budget == 0) {
      std::size_t free_b = 0, total_b = 0;
      HMXG_CUDA(cudaSetDevice(ctx->devs[0]));
      HMXG_CUDA(cudaMemGetInfo(&free_b, &total_b));
      budget = total_b / 4 * 3;
    }
    if (bytes > budget) return upload_impl(ctx, cds, SplitSpec{ctx->comm.size, ctx->comm.rank}, out);
  }
  return upload_impl(ctx, cds, SplitSpec{}, out);
}

// hmxg_upload_generated with skeletons: trees up to these sizes (the flat tree's own limits,
// plan.cpp) get their far blocks on the host as well, for the flat tree's composites
constexpr std::uint64_t kFlatGenMaxPoints = 65536;
constexpr std::uint32_t kFlatGenMaxNodes = 1024;

int hmxg_upload_generated(hmxg_ctx* ctx, const hmxg_cds_view* cds, const double* coords, uint32_t d, int32_t kernel,
                          double h, const uint64_t* skel_ptr, const uint32_t* skel_idx, hmxg_mat** out) {
  return hmxg_upload_generated_ex(ctx, cds, coords, d, kernel, h, skel_ptr, skel_idx, 0u, out);
}

int hmxg_upload_generated_ex(hmxg_ctx* ctx, const hmxg_cds_view* cds, const double* coords, uint32_t d,
                             int32_t kernel, double h, const uint64_t* skel_ptr, const uint32_t* skel_idx,
                             unsigned flags, hmxg_mat** out) {
  if (flags & ~HMXG_UPLOAD_NEAR_ON_THE_FLY) return set_err(HMXG_EINVAL, "hmxg_upload_generated_ex: unknown flags");
  if (!cds || !coords || d == 0) return set_err(HMXG_EINVAL, "hmxg_upload_generated: null points");
  if (skel_ptr) {  // every node's skeleton must have its srank entries, all of them points
    if (cds->num_nodes && !cds->sranks) return set_err(HMXG_EINVAL, "cds: null array in view");
    if (skel_ptr[cds->num_nodes] && !skel_idx) return set_err(HMXG_EINVAL, "hmxg_upload_generated: null skeletons");
    for (std::uint32_t i = 0; i < cds->num_nodes; ++i)
      if (skel_ptr[i + 1] - skel_ptr[i] != cds->sranks[i])
        return set_err(HMXG_EINVAL, "hmxg_upload_generated: skeleton size differs from the node's srank");
    for (std::uint64_t s = 0; s < skel_ptr[cds->num_nodes]; ++s)
      if (skel_idx[s] >= cds->n) return set_err(HMXG_EINVAL, "dense_block: row index out of range");
  }
  if (kernel < HMXG_KERNEL_GAUSSIAN || kernel > HMXG_KERNEL_INVDIST)
    return set_err(HMXG_EINVAL, "hmxg_upload_generated: unknown kernel");
  if (kernel != HMXG_KERNEL_INVDIST && !(h > 0.0)) return set_err(HMXG_EINVAL, "Gaussian kernel: bandwidth must be > 0");
  NearSource src;
  src.coords = coords;
  src.d = d;
  src.kp.kind = kernel;
  src.kp.d = d;
  src.kp.den = 2.0 * h * h;
  src.kp.invh = 1.0 / h;
  src.skel_ptr = skel_ptr;
  src.skel_idx = skel_idx;
  SplitSpec spec;
  spec.generated_near = true;
  spec.generated_far = skel_ptr != nullptr;
  const bool otf = (flags & HMXG_UPLOAD_NEAR_ON_THE_FLY) != 0;
  // Small trees run the flat tree, whose composite transfer products the plan forms on the
  // host from the far blocks and the bases (plan.cpp): there the far blocks are generated on
  // the device first and brought back (a few MB at most), and the upload proceeds as with
  // stored far blocks. The same device kernel generates them either way, so the values are
  // the generated upload's; large trees keep them on the device.
  if (skel_ptr && ctx && !ctx->devs.empty() && cds->n <= kFlatGenMaxPoints && cds->num_nodes <= kFlatGenMaxNodes &&
      cds->num_far && cds->bptr && cds->far_pairs && std::getenv("HMXG_NO_FLAT") == nullptr) {
    const std::uint64_t b_elems = cds->bptr[cds->num_far];
    std::vector<double> bhost(b_elems);
    if (b_elems) {
      HMXG_CUDA(cudaSetDevice(ctx->devs[0]));
      std::vector<GenBlock> blocks(cds->num_far);
      for (std::uint64_t k = 0; k < cds->num_far; ++k) {
        const std::uint32_t i = cds->far_pairs[2 * k], j = cds->far_pairs[2 * k + 1];
        if (i >= cds->num_nodes || j >= cds->num_nodes) return set_err(HMXG_EINVAL, "cds: far pair out of range");
        blocks[k] = GenBlock{cds->bptr[k], skel_ptr[i], skel_ptr[j], cds->sranks[i], cds->sranks[j]};
        if (cds->bptr[k] + std::uint64_t(cds->sranks[i]) * cds->sranks[j] > b_elems)
          return set_err(HMXG_EINVAL, "cds: far block offsets out of range");
      }
      const std::vector<std::uint32_t> skel(skel_idx, skel_idx + skel_ptr[cds->num_nodes]);
      double *pts = nullptr, *gb = nullptr;
      int rc = dev_upload(&pts, coords, cds->n * std::uint64_t(d), nullptr);
      if (rc == HMXG_OK) rc = generate_blocks(pts, src.kp, skel, blocks, b_elems, &gb, nullptr);
      if (rc == HMXG_OK && cudaMemcpy(bhost.data(), gb, b_elems * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
        rc = set_err(HMXG_ECUDA, "hmxg_upload_generated: far blocks device -> host");
      cudaFree(pts);
      cudaFree(gb);
      HMXG_TRY(rc);
    }
    hmxg_cds_view with_b = *cds;
    with_b.bgen = bhost.data();
    src.skel_ptr = nullptr;
    src.skel_idx = nullptr;
    spec.generated_far = false;
    return upload_impl(ctx, &with_b, spec, out, &src, otf);
  }
  return upload_impl(ctx, cds, spec, out, &src, otf);
}

int hmxg_upload_split(hmxg_ctx* ctx, const hmxg_cds_view* cds, uint32_t nparts, uint32_t part, hmxg_mat** out) {
  if (nparts == 0 || part >= nparts) return set_err(HMXG_EINVAL, "hmxg_upload_split: bad part / nparts");
  if (ctx && ctx->devs.size() != 1) return set_err(HMXG_EINVAL, "hmxg_upload_split: one device per part");
  return upload_impl(ctx, cds, SplitSpec{nparts, part}, out);
}

int hmxg_split_stage(hmxg_mat* mat, int stage, const double* W, size_t n, size_t q, size_t ldw, double* Y, size_t ldy,
                     void* stream) {
  if (!mat) return set_err(HMXG_EINVAL, "hmxg_split_stage: null matrix");
  const Plan& plan = mat->plan;
  if (n != plan.n) return set_err(HMXG_EINVAL, "evaluate: W row count does not match the point count");
  if (q == 0) return HMXG_OK;
  if (stage < 0 || stage > 1 || !W || !Y || ldw < n || ldy < n || mat->devs.size() != 1)
    return set_err(HMXG_EINVAL, "hmxg_split_stage: bad arguments");
  std::lock_guard<std::mutex> lock(mat->mu);
  DevState& d = mat->devs[0];
  HMXG_CUDA(cudaSetDevice(d.dev));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.comp;
  HMXG_TRY(ensure_workspace(plan, d, q));
  const DevState::DagItems* di = nullptr;
  HMXG_TRY(ensure_dag(plan, d, q, st, &di, static_cast<std::uint32_t>(stage)));
  HMXG_TRY(order_after_previous(d, st));
  d.pending = false;  // this call returns when its stage (and everything before it) is done
  const std::uint32_t qq = static_cast<std::uint32_t>(q), nn = static_cast<std::uint32_t>(n);
  const std::uint64_t ldq = d.cap_q;
  const std::uint32_t ncb = (qq + kBN - 1) / kBN;
  CUtensorMap tm_wp, tm_t, tm_s;
  HMXG_TRY(make_map(&tm_wp, d.wp, plan.rows_pad, q, ldq));
  HMXG_TRY(make_map(&tm_t, d.t, plan.skel_rows, q, ldq));
  HMXG_TRY(make_map(&tm_s, d.s, plan.skel_rows, q, ldq));
  GemmParams p{};
  p.tiles = d.tiles;
  p.tasks = d.tasks;
  p.segs = d.segs;
  p.idmap = d.idmap;
  p.buf[kBufWp] = d.wp;
  p.buf[kBufT] = d.t;
  p.buf[kBufS] = d.s;
  p.buf[kBufYp] = d.yp;
  for (auto& l : p.ld) l = ldq;
  p.q = qq;
  DagParams dp{};
  dp.recs = di->recs;
  dp.per_task = di->per_task;
  dp.parts = di->parts;
  dp.nitems = di->nitems;
  dp.claim = d.dag_done + stage;
  dp.done = d.dag_done + kDagClaimWords;
  dp.cstride = 1;
  dp.node_tiles = d.node_tiles;
  dp.yp_tiles = d.yp_tiles;
  dp.signal_yp = split_leaf(plan, q, d.gemm_grid) ? 1u : 0u;
  dp.colsplit = 1;
  dp.ncb = ncb;
  dp.nodes = plan.num_nodes;
  dp.fwd_signals = forward_signals(di->nitems, d.gemm_grid);
#ifdef HMXG_TRACE
  HMXG_TRY(trace_prepare(d, st));
  dp.trace = g_trace;
#endif
  const dim3 pgrid((nn + kTT - 1) / kTT, (qq + kTT - 1) / kTT);
  if (pgrid.y > 65535) return set_err(HMXG_EINVAL, "hmxg_split_stage: too many columns for one call");
  if (stage == 0) {
    // T rows of other parts and of the top levels must be zero for the exchange (a sum);
    // Y' rows of other parts' leaves stay zero so the parts' Y sum to the full Y
    HMXG_CUDA(cudaMemsetAsync(d.t, 0, plan.skel_rows * ldq * sizeof(double), st));
    HMXG_CUDA(cudaMemsetAsync(d.yp, 0, plan.rows_pad * ldq * sizeof(double), st));
    HMXG_CUDA(cudaMemsetAsync(d.dag_done, 0, (dag_done_words(plan, q) + 1) * sizeof(std::uint32_t), st));
    permute_in<<<pgrid, 256, 0, st>>>(W, ldw, d.ipmap, d.wp, ldq, nn, qq, nullptr, 0);
  } else if (!plan.remote_t_nodes.empty()) {
    // T of the other parts' nodes arrived through the exchange: mark it complete
    const std::uint64_t cells = std::uint64_t(plan.remote_t_nodes.size()) * ncb;
    preset_done<<<static_cast<unsigned>((cells + 255) / 256), 256, 0, st>>>(
        d.remote_t, static_cast<std::uint32_t>(plan.remote_t_nodes.size()), dp.done, ncb, d.node_tiles);
  }
  if (di->nitems) {
    const unsigned grid = static_cast<unsigned>(std::min<std::uint64_t>(di->nitems, d.gemm_grid));
    eval_dag<false><<<grid, kThreads, kSmemBytes, st>>>(tm_wp, tm_t, tm_s, p, dp);
  }
  if (stage == 1)  // zeroes the counters for the next evaluation (stage 0 sets them itself)
    permute_out<<<pgrid, 256, 0, st>>>(d.yp, ldq, d.ipmap, Y, ldy, nn, qq, d.dag_done,
                                       dag_done_words(plan, q) + 1);
  HMXG_CUDA(cudaGetLastError());
  HMXG_CUDA(cudaStreamSynchronize(st));
  return HMXG_OK;
}

int hmxg_split_exchange(hmxg_mat* mat, double* buf, size_t count, int to_matrix, void* stream) {
  double* t = nullptr;
  size_t need = 0;
  HMXG_TRY(hmxg_split_exchange_buffer(mat, &t, &need));
  if (!buf || count != need) return set_err(HMXG_EINVAL, "hmxg_split_exchange: buffer size mismatch");
  DevState& d = mat->devs[0];
  HMXG_CUDA(cudaSetDevice(d.dev));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.comp;
  HMXG_CUDA(cudaMemcpyAsync(to_matrix ? t : buf, to_matrix ? buf : t, need * sizeof(double), cudaMemcpyDeviceToDevice, st));
  HMXG_CUDA(cudaStreamSynchronize(st));
  return HMXG_OK;
}

int hmxg_split_exchange_buffer(hmxg_mat* mat, double** ptr, size_t* count) {
  if (!mat || !ptr || !count || mat->devs.empty()) return set_err(HMXG_EINVAL, "hmxg_split_exchange_buffer: null");
  DevState& d = mat->devs[0];
  if (!d.t) return set_err(HMXG_EINVAL, "hmxg_split_exchange_buffer: run stage 0 first");
  *ptr = d.t;
  *count = mat->plan.skel_rows * d.cap_q;
  return HMXG_OK;
}

int hmxg_free(hmxg_mat* mat) {
  if (!mat) return HMXG_OK;
  for (auto& d : mat->devs) d.release();
  delete mat;
  return HMXG_OK;
}

int hmxg_info_get(const hmxg_mat* mat, hmxg_info* info) {
  if (!mat || !info) return set_err(HMXG_EINVAL, "hmxg_info_get: null argument");
  const Plan& p = mat->plan;
  std::memset(info, 0, sizeof *info);
  info->n = p.n;
  info->d_elems = p.d_elems;
  info->b_elems = p.b_elems;
  info->v_elems = p.v_elems;
  info->skel_rows = p.skel_rows;
  info->num_devices = static_cast<std::uint32_t>(mat->devs.size());
  // permute-in, eval_dag, permute-out; 1 when the last evaluation fused the permutations
  info->launches_per_eval = mat->devs.empty() ? 3 : mat->devs[0].last_launches;
  info->flops_per_col = 2.0 * (2.0 * p.v_elems + p.b_elems + p.d_elems);
  for (const Phase* ph : tree_phases(p, 0)) info->exec_flops_per_col += ph->flops_per_col;
  for (const Phase& ph : p.phases)
    if (ph.kind == kPhaseLeaf) info->exec_flops_per_col += ph.flops_per_col;
  info->device_bytes = mat->devs.empty() ? 0 : mat->devs[0].resident_bytes;
  info->split_parts = p.nparts;
  info->part = p.part;
  return HMXG_OK;
}

// The launch sequence of the most recent evaluation: the DAG sequence (permute-in,
// eval_dag, permute-out) by default, the level sequence after HMXG_F_LEVEL_LAUNCHES.
int hmxg_phase_count(const hmxg_mat* mat) {
  if (!mat) return -1;
  return static_cast<int>(mat->devs[0].launch_desc.size());
}

int hmxg_phase_get(hmxg_mat* mat, uint32_t idx, hmxg_phase* out) {
  if (!mat || !out) return set_err(HMXG_EINVAL, "hmxg_phase_get: null argument");
  const std::vector<DevState::LaunchDesc>& ld = mat->devs[0].launch_desc;
  if (idx >= ld.size()) return set_err(HMXG_EINVAL, "hmxg_phase_get: index out of range");
  std::memset(out, 0, sizeof *out);
  out->kind = ld[idx].kind;
  out->level = ld[idx].level;
  out->tiles = ld[idx].tiles;
  out->flops_per_col = ld[idx].flops_per_col;
  out->gen_bytes = ld[idx].gen_bytes;
  out->io_bytes_per_col = ld[idx].io_bytes_per_col;
  DevState& d = mat->devs[0];
  if (d.phase_valid) {
    HMXG_CUDA(cudaSetDevice(d.dev));
    HMXG_CUDA(cudaEventSynchronize(d.phase_ev[idx + 1]));
    float ms = 0.f;
    HMXG_CUDA(cudaEventElapsedTime(&ms, d.phase_ev[idx], d.phase_ev[idx + 1]));
    out->last_ms = ms;
  }
  return HMXG_OK;
}

int hmxg_evaluate(hmxg_mat* mat, const double* W, size_t n, size_t q, size_t ldw, double* Y, size_t ldy,
                  unsigned flags, void* stream, hmxg_stats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  if (!mat) return set_err(HMXG_EINVAL, "hmxg_evaluate: null matrix");
  if (n != mat->plan.n) return set_err(HMXG_EINVAL, "evaluate: W row count does not match the point count");
  if (stats) std::memset(stats, 0, sizeof *stats);
  if (q == 0) return HMXG_OK;  // executor.cpp:279-282
  if (!W || !Y || ldw < n || ldy < n) return set_err(HMXG_EINVAL, "hmxg_evaluate: bad W/Y or leading dimension");
  if (q > 0xffffffffull) return set_err(HMXG_EINVAL, "hmxg_evaluate: too many columns");
  std::lock_guard<std::mutex> lock(mat->mu);
  const Plan& plan = mat->plan;
  const bool time_phases = flags & HMXG_F_TIME_PHASES;
  const bool levels = flags & HMXG_F_LEVEL_LAUNCHES;
  for (auto& dv : mat->devs) {
    dv.last_levels = levels;
    dv.phase_valid = false;  // set again by the launches of this call if they are timed
  }
  std::uint32_t launches = 0;
  float dev_ms = 0.f;

  if (plan.nparts > 1) {  // subtree-split part: a collective evaluation (hmxg_create_comm)
    HMXG_TRY(split_evaluate(mat, W, ldw, Y, ldy, q, flags, stream, &launches));
  } else if (flags & HMXG_F_DEVICE_PTRS) {
    if (mat->devs.size() != 1)
      return set_err(HMXG_EINVAL, "hmxg_evaluate: device pointers need a single-device context");
    DevState& d = mat->devs[0];
    HMXG_CUDA(cudaSetDevice(d.dev));
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.comp;
    HMXG_TRY(ensure_workspace(plan, d, q));
    const DevState::DagItems* di = nullptr;
    if (!levels) HMXG_TRY(ensure_dag(plan, d, q, st, &di));
    HMXG_TRY(order_after_previous(d, st));
    const bool sync = !(flags & HMXG_F_NO_SYNC);
    if (sync) HMXG_CUDA(cudaEventRecord(d.ev0, st));
    // the legacy / per-thread default streams cannot be captured: launch directly there
    if (st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread || (flags & HMXG_F_NO_GRAPH)) {
      HMXG_TRY(enqueue_eval(plan, d, W, ldw, Y, ldy, q, st, time_phases, levels, &launches));
    } else {
      const DevState::GraphKey key{W, Y, q, ldw, ldy, st, d.wp, di ? static_cast<const void*>(di->recs) : nullptr, d.dag_done, levels,
                                   time_phases};
      if (!(d.gexec && d.gkey == key)) {
        d.drop_graph();
        cudaGraph_t graph = nullptr;
        HMXG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        std::uint32_t captured = 0;
        const int rc = enqueue_eval(plan, d, W, ldw, Y, ldy, q, st, time_phases, levels, &captured);
        const cudaError_t ec = cudaStreamEndCapture(st, &graph);
        if (rc != HMXG_OK) {
          if (graph) cudaGraphDestroy(graph);
          return rc;
        }
        if (ec != cudaSuccess) return cuda_fail(ec, "cudaStreamEndCapture");
        const cudaError_t ei = cudaGraphInstantiate(&d.gexec, graph, 0);
        cudaGraphDestroy(graph);
        if (ei != cudaSuccess) return cuda_fail(ei, "cudaGraphInstantiate");
        d.gkey = key;
        d.glaunches = captured;
        d.gfused = d.last_fused;
        d.gdesc = d.launch_desc;
      }
      HMXG_CUDA(cudaGraphLaunch(d.gexec, st));
      launches += d.glaunches;
      d.phase_valid = time_phases;  // the graph's event nodes time this replay
      d.last_fused = d.gfused;      // and the launch sequence is the captured one
      d.launch_desc = d.gdesc;
      d.last_launches = d.glaunches;
      d.last_q = q;
    }
    if (sync) {
      HMXG_CUDA(cudaEventRecord(d.ev1, st));
      HMXG_CUDA(cudaEventSynchronize(d.ev1));
      HMXG_CUDA(cudaEventElapsedTime(&dev_ms, d.ev0, d.ev1));
      d.pending = false;
#ifdef HMXG_TRACE
      if (!levels) trace_dump(plan, q, d.gemm_grid);
#endif
    } else {
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      HMXG_CUDA(cudaStreamIsCapturing(st, &cap));
      if (cap == cudaStreamCaptureStatusNone) {  // the next call waits for this one's work
        HMXG_CUDA(cudaEventRecord(d.ev_last, st));
        d.pending = true;
      }
    }
  } else {
    // column sharding over the context's devices: Y[:,c] depends only on W[:,c]
    const HostKind kw = host_kind(W), ky = host_kind(Y);
    if (kw == HostKind::kDevice || ky == HostKind::kDevice)
      return set_err(HMXG_EINVAL, "hmxg_evaluate: device pointer without HMXG_F_DEVICE_PTRS");
    const std::size_t G = mat->devs.size();
    std::vector<std::size_t> cut(G + 1);
    for (std::size_t g = 0; g <= G; ++g) cut[g] = q * g / G;
    for (std::size_t g = 0; g < G; ++g) {  // an earlier asynchronous device-pointer call
      DevState& d = mat->devs[g];
      if (!d.pending) continue;
      HMXG_CUDA(cudaSetDevice(d.dev));
      HMXG_CUDA(cudaEventSynchronize(d.ev_last));
      d.pending = false;
    }
    if (kw != HostKind::kPinned || ky != HostKind::kPinned) {
      // pageable host buffers: the bounce path, one host thread per device shard
      const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
      const unsigned per = std::max(1u, hw / static_cast<unsigned>(G));
      std::vector<int> rcs(G, HMXG_OK);
      std::vector<std::string> errs(G);
      std::vector<std::uint32_t> lc(G, 0);
      auto run = [&](std::size_t g) {
        rcs[g] = host_bounce_shard(plan, mat->devs[g], W, ldw, Y, ldy, cut[g], cut[g + 1], time_phases && g == 0,
                                   levels, &lc[g], per);
        if (rcs[g] != HMXG_OK) errs[g] = hmxg_last_error();
      };
      std::vector<std::thread> workers;
      for (std::size_t g = 1; g < G; ++g)
        if (cut[g + 1] > cut[g]) workers.emplace_back(run, g);
      if (cut[1] > cut[0]) run(0);
      for (auto& th : workers) th.join();
      for (std::size_t g = 0; g < G; ++g) {
        if (rcs[g] != HMXG_OK) return set_err(rcs[g], errs[g]);
        launches += lc[g];
      }
    } else {
      for (std::size_t g = 0; g < G; ++g) {
        if (cut[g + 1] == cut[g]) continue;
        DevState& d = mat->devs[g];
        HMXG_CUDA(cudaSetDevice(d.dev));
        HMXG_TRY(enqueue_host_shard(plan, d, W, ldw, Y, ldy, cut[g], cut[g + 1], time_phases && g == 0, levels,
                                    &launches));
      }
    }
    for (std::size_t g = 0; g < G; ++g) {
      if (cut[g + 1] == cut[g]) continue;
      DevState& d = mat->devs[g];
      HMXG_CUDA(cudaSetDevice(d.dev));
      HMXG_CUDA(cudaStreamSynchronize(d.d2h));
      HMXG_CUDA(cudaStreamSynchronize(d.comp));
      HMXG_CUDA(cudaEventSynchronize(d.ev1));
      float ms = 0.f;
      HMXG_CUDA(cudaEventElapsedTime(&ms, d.ev0, d.ev1));
      dev_ms = std::max(dev_ms, ms);
    }
  }
  if (stats) {
    stats->locked_pairs = 0;
    stats->device_ms = dev_ms;
    stats->launches = launches;
    stats->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  return HMXG_OK;
}

}  // extern "C"
