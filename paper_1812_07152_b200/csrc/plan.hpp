// plan.hpp — host-side lowering of a CDS into level-batched GEMM task tables.
//
// The reference runs the evaluation as four barrier-separated passes over the CDS with a
// fork-join pool (proj/src/executor.cpp:139-243). On the B200 each pass becomes a short
// sequence of batched launches, one per tree level, of a single grouped FP64 GEMM kernel
// whose tasks are output row tiles with a list of K segments:
//
//   gather    Wp = W[perm, :]                                   (executor.cpp:35-39)
//   up-leaf   T_i = V_i^T Wp_i                 one launch        (executor.cpp:56-61)
//   up-h      T_i = V_i^T [T_lc; T_rc]         one per height    (executor.cpp:62-71)
//   down-d    S_c = sum_j B_cj T_j + V_p[c] S_p one per depth    (executor.cpp:105-110, 85-102)
//   leaf      Y'_i = V_i S_i + sum_j D_ij Wp_j one launch        (executor.cpp:79-84, 112-117)
//   scatter   Y[perm, :] = Y'                                    (executor.cpp:245-254)
//
// The far pass is folded into the downward pass (far terms only need T, which is complete
// after the upward pass), and the leaf downward term is folded into the near pass, so every
// output tile is written exactly once by one CTA: no atomics, no memset, no read-modify-
// write of S (the reference's single-writer invariant, executor.hpp:48-50).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/hmxg.h"

namespace hmxg {

// Operand buffers a task can read (B side) or write (C side).
enum Buf : std::uint16_t { kBufWp = 0, kBufT = 1, kBufS = 2, kBufYp = 3, kNumBufs = 4 };
// Generator arrays a segment's A operand lives in.
enum Gen : std::uint16_t { kGenD = 0, kGenB = 1, kGenV = 2 };

// One K segment of a task: C_tile += A_seg(tile rows, 0:k) * B_seg(0:k, cols).
// A is column major with leading dimension lda; with `trans` the stored matrix is A^T
// (A(r,k) = a[k + r*lda]). a_off is the element offset (tile row already applied) into
// generator array `gen`; b_row is the first row of the B operand inside buffer `bbuf`.
struct Seg {
  std::uint64_t a_off;
  std::uint32_t lda;
  std::uint32_t k;
  std::uint32_t b_row;
  std::uint16_t gen;
  std::uint16_t bbuf;
};
static_assert(sizeof(Seg) == 24, "Seg layout");

// One output row tile: rows [c_row, c_row + m) of buffer cbuf, all columns (grid.y).
struct Task {
  std::uint32_t c_row;
  std::uint16_t cbuf;
  std::uint16_t m;
  std::uint32_t seg_begin;
  std::uint32_t seg_end;
};
static_assert(sizeof(Task) == 16, "Task layout");

enum PhaseKind : int { kPhaseUp = 0, kPhaseDown = 1, kPhaseLeaf = 2 };

struct Phase {
  PhaseKind kind;
  bool trans_a;          // upward phases read V^T
  std::uint32_t task_begin, task_end;
  std::uint32_t level;   // height (up) or depth (down)
  double flops_per_col;  // 2*sum(m*k) over the phase's tiles, algorithmic
  double gen_bytes;      // generator (A operand) bytes the phase reads once per evaluation
  double io_bytes_per_col;  // B operand rows read + C rows written, once per node, per column
};

struct Plan {
  std::uint64_t n = 0;
  std::uint32_t num_nodes = 0;
  std::uint64_t skel_rows = 0;  // rows of T and S
  std::vector<std::uint64_t> node_off;  // T/S row of each active node
  std::vector<Task> tasks;
  std::vector<Seg> segs;
  std::vector<Phase> phases;
  std::uint64_t d_elems = 0, b_elems = 0, v_elems = 0;
  std::uint32_t max_m = 0;
};

// Validates the view (structure.hpp invariants the evaluator relies on) and lowers it.
// Returns false with `err` set on a malformed view. `tile_m` is the kernel's row tile.
bool build_plan(const hmxg_cds_view& v, std::uint32_t tile_m, Plan& plan, std::string& err);

}  // namespace hmxg
