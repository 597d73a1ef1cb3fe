// plan.hpp — host-side lowering of a CDS into level-batched GEMM task tables.
//
// The reference runs the evaluation as four barrier-separated passes over the CDS with a
// fork-join pool (proj/src/executor.cpp:139-243). On the B200 each pass becomes a short
// sequence of batched launches, one per tree level, of a single grouped FP64 GEMM kernel
// whose tasks are output row tiles with a list of K segments:
//
//   gather    Wp = W[perm, :]                                   (executor.cpp:35-39)
//   up-leaf   T_i = V_i^T Wp_i                  one launch       (executor.cpp:56-61)
//   up-h      T_i = V_i^T [T_lc; T_rc]          one per height   (executor.cpp:62-71)
//   down-d    S_c = sum_j B_cj T_j + V_p[c] S_p one per depth    (executor.cpp:105-110, 85-102)
//   leaf      Y'_i = V_i S_i + sum_j D_ij Wp_j  one launch       (executor.cpp:79-84, 112-117)
//   scatter   Y[perm, :] = Y'                                    (executor.cpp:245-254)
//
// The far pass is folded into the downward pass (far terms only need T, which is complete
// after the upward pass), and the leaf downward term is folded into the near pass, so every
// output tile is written exactly once by one CTA: no atomics, no memset, no read-modify-
// write of S (the reference's single-writer invariant, executor.hpp:48-50).
//
// Device layout: every node's row block in Wp / Yp (leaves) and T / S (active nodes) starts
// on a 16-row boundary and is zero-padded to a multiple of 16 rows, so each 16-row B chunk
// the TMA engine fetches lies inside one node block (no foreign rows enter a sum).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hmxg.h"

namespace hmxg {

constexpr std::uint32_t kRowAlign = 16;  // = the kernel's K chunk

// Operand buffers a task can read (B side) or write (C side).
enum Buf : std::uint16_t { kBufWp = 0, kBufT = 1, kBufS = 2, kBufYp = 3, kNumBufs = 4 };
// Generator arrays an A operand is tiled from.
enum Gen : std::uint8_t { kGenD = 0, kGenB = 1, kGenV = 2, kGenC = 3 /* Plan::cgen composites */ };

// Source of one pre-tiled A operand: rows [0, m) of the tile, K columns, from generator
// `gen` at element offset a_off, column major with leading dimension lda; with `trans`
// the stored matrix is A^T (A(r,k) = a[k + r*lda]). Tile row r reads generator row
// rmap[r0 + r] and K index k reads generator column kmap[k] (the node row orders of the
// identity-row lowering, Plan::maps), or r0 + r and k without a map (kNoMap). Tiled to
// tile_off (in doubles).
constexpr std::uint32_t kNoMap = 0xffffffffu;
struct TileSrc {
  std::uint64_t a_off;
  std::uint64_t tile_off;
  std::uint32_t lda;
  std::uint32_t k;
  std::uint16_t m;
  std::uint8_t gen;
  std::uint8_t trans;
  std::uint32_t r0;
  std::uint32_t rmap;
  std::uint32_t kmap;
  std::uint32_t pad;
};
static_assert(sizeof(TileSrc) == 48, "TileSrc layout");

// One K segment of a task as the GEMM kernel sees it: nchunks pre-tiled A chunks at
// tile_off, and B rows [b_row, b_row + 16*nchunks) of buffer bbuf. `last_ksteps`: the
// last chunk's K rows that carry data, in 4-row DMMA k-steps (0: all four); the rest of
// it is zero padding the consumers do not multiply.
// `src` is the node whose T or S rows the segment reads (the DAG kernel waits for that
// node's tiles of the same column block); unused for Wp. `rows`: the segment only
// contributes to the tile's first `rows` output rows (its A operand is zero below), so
// fragments below are not multiplied.
struct SegDev {
  std::uint64_t tile_off;
  std::uint32_t b_row;
  std::uint16_t nchunks;
  std::uint8_t bbuf;
  std::uint8_t last_ksteps;
  std::uint32_t src;
  std::uint32_t rows;
};
static_assert(sizeof(SegDev) == 24, "SegDev layout");

// One output row tile: rows [c_row, c_row + m) of buffer cbuf, all columns (grid.y).
// `node` owns the output rows (T or S of that node; Yp for a leaf).
// Identity rows (the interpolative bases' unit rows): when id_off != kNoMap, output row r
// also adds row idmap[id_off + r] of buffer id_buf (kNoMap: nothing), whose producers are
// the nodes id_node0 / id_node1 (kNoMap: none) the DAG consumer waits for first.
struct Task {
  std::uint32_t c_row;
  std::uint16_t cbuf;
  std::uint16_t m;
  std::uint32_t seg_begin;
  std::uint32_t seg_end;
  std::uint32_t node;
  std::uint32_t id_off;
  std::uint32_t id_node0;
  std::uint32_t id_node1;
  std::uint16_t id_buf;
  std::uint16_t flags;  // kTaskAccumulate, kTaskIdLast
  std::uint32_t pad1;
};
static_assert(sizeof(Task) == 40, "Task layout");
// The accumulator starts from the task's own C rows (the split leaf variant's leaf task).
constexpr std::uint16_t kTaskAccumulate = 1;
// The identity rows are added after the K loop instead of starting the accumulator. Leaf
// (Yp) tasks use it so that both leaf variants sum every row in one order,
// ((sum_j D_ij Wp_j) + V_i S_i) + copied S_i rows, and give the same bits.
constexpr std::uint16_t kTaskIdLast = 2;
// The task's last segment reads the rows of the identity source node (S_i of a leaf): the
// producer acquired that node's completion before streaming it, and the stage barriers
// (arrive: release, wait: acquire) carry it to the consumers, which skip their own poll.
constexpr std::uint16_t kTaskIdSynced = 4;
// The task writes the final value of its Yp rows (the combined leaf tasks, the split
// variant's accumulating leaf tasks, and the near tasks of leaves without a basis): with the
// fused permutations (eval_dag's small-problem mode) they are stored straight into Y.
constexpr std::uint16_t kTaskFinal = 8;

// kPhaseNear: Y'_i = sum_j D_ij Wp_j (depends on Wp only); kPhaseLeaf: Y'_i += V_i S_i
// (accumulates onto the near rows of the same leaf through the task's identity rows).
enum PhaseKind : int { kPhaseUp = 0, kPhaseDown = 1, kPhaseLeaf = 2, kPhaseNear = 3 };

struct Phase {
  PhaseKind kind;
  std::uint32_t stage;      // 0, or 1 = after the skeleton exchange (subtree-split mode)
  std::uint32_t task_begin, task_end;
  std::uint32_t level;      // height (up) or depth (down)
  double flops_per_col;     // 2*sum(m*k) over the phase's tiles, algorithmic
  double gen_bytes;         // generator (A operand) bytes the phase reads once per evaluation
  double io_bytes_per_col;  // B operand rows read + C rows written, once per node, per column
};

struct Plan {
  std::uint64_t n = 0;
  std::uint32_t num_nodes = 0;
  std::uint64_t rows_pad = 0;           // rows of Wp / Yp (padded tree order)
  std::uint64_t skel_rows = 0;          // rows of T and S (padded)
  std::vector<std::uint32_t> pmap;      // padded row -> original point, 0xffffffff for pad
  std::vector<std::uint32_t> ipmap;     // original point -> padded row
  std::vector<std::uint32_t> parent;    // tree parent of each node (kNoMap for the root)
  std::vector<std::uint32_t> depth;     // tree depth of each node
  std::vector<std::uint64_t> leaf_row;  // padded Wp/Yp row of each leaf
  std::vector<std::uint64_t> node_off;  // T/S row of each active node
  std::vector<Task> tasks;
  std::vector<SegDev> segs;
  std::vector<TileSrc> tile_src;        // one per segment (same order as segs)
  std::vector<std::uint32_t> chunk_seg; // pre-tiled chunk -> segment
  std::uint64_t tile_elems = 0;
  std::vector<Phase> phases;
  // the leaf phase as a near phase + an accumulating leaf phase over the same segments
  // (tasks after the phases' ones); the DAG uses it for narrow column counts
  std::vector<Phase> split_phases;
  std::vector<std::uint32_t> node_tiles;  // row tiles of each active node's T (= of its S)
  std::vector<std::uint32_t> yp_tiles;    // near-phase row tiles of each leaf (its Yp rows)
  // subtree-split mode (SURVEY §8e fallback): nodes whose T arrives through the exchange
  std::uint32_t nparts = 1, part = 0;
  std::vector<std::uint32_t> remote_t_nodes;
  std::vector<std::uint64_t> pub_row;     // nparts + 1: T rows each part publishes (in place)
  std::vector<std::uint64_t> yp_row;      // nparts + 1: Wp / Yp rows of each part's leaves
  std::uint32_t leaf_tasks = 0;           // row tiles of the leaf (Yp) phase
  std::uint64_t d_elems = 0, b_elems = 0, v_elems = 0;
  std::uint32_t max_m = 0;
  // identity-row lowering (plan.cpp): node row orders (TileSrc rmap/kmap index them) and
  // the per-row identity sources of tasks (Task::id_off indexes them)
  std::vector<std::uint32_t> maps;
  std::vector<std::uint32_t> idmap;
  double identity_flops_per_col = 0.0;  // multiply-adds by exact 0/1 rows the kernel skips
  bool near_otf = false;                 // near blocks generated per evaluation (hmxg_upload_generated_ex)
  // flat tree (small trees, plan.cpp): the internal upward and far+downward levels replaced by
  // two phases of composite transfer products (kGenC blocks in cgen)
  bool flat = false;
  std::vector<Phase> flat_phases;
  std::vector<double> cgen;
  double flat_extra_flops_per_col = 0.0;
  std::uint32_t flat_mid_height = 0;  // 0: one flat upward phase from the leaves
  mutable double ct_dmma = -1.0;         // CTree work per 8-column octet in DMMAs (hmxg.cu, cached)
  mutable std::uint64_t ct_smem = 0;     // its tables' shared-memory bytes
};

// Validates the view (structure.hpp invariants the evaluator relies on) and lowers it.
// Returns false with `err` set on a malformed view. `tile_m` is the kernel's row tile.
// Subtree split: the nodes below the top ceil(log2 nparts) levels are divided
// by subtree into nparts contiguous parts. Part `part` gets stage 0 = the upward pass over
// its own subtrees; stage 1 = the replicated top levels (upward), far+downward for its own
// and the top nodes, and the leaf/near rows of its own leaves. Between the stages the
// parts exchange T (each holds only its own rows; the sum of the parts' T is the full T).
struct SplitSpec {
  std::uint32_t nparts = 1;
  std::uint32_t part = 0;
  bool identity_rows = true;    // lower the bases' unit rows to row copies (plan.cpp)
  bool generated_near = false;  // dgen may be null: the near blocks are generated on the device
  bool generated_far = false;   // bgen may be null: the far blocks are generated on the device
  bool flat_tree = true;        // small trees: composite (flat) tree phases, see Plan::flat_phases
};
bool build_plan(const hmxg_cds_view& v, std::uint32_t tile_m, Plan& plan, std::string& err,
                const SplitSpec& split = {});

}  // namespace hmxg
