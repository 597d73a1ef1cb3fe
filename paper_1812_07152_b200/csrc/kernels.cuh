// kernels.cuh — sm_100a kernels of the evaluator.
//
//  * tile_a: one-time (upload) re-layout of every GEMM A operand (V^T, V, B_ij, D_ij
//    row tiles) into zero-padded, XOR-swizzled 64 x 16 FP64 chunks, so the main kernel
//    streams A with one 8 KB bulk copy per chunk and reads it without bank conflicts.
//  * eval_dag: the whole-evaluation persistent launch. One CTA owns one (output row tile,
//    64-column block) work item at a time, claimed in topological order; its K loop walks
//    the tile's segment list, so a whole far+downward sum or a whole leaf row
//    (V_i S_i + sum_j D_ij Wp_j) is accumulated in registers and stored once (single
//    writer, no atomics). A producer lane streams A chunks with cp.async.bulk and B tiles
//    (rows of Wp/T/S, 16 x 68, unswizzled: the 68-double pitch is conflict-free) with TMA
//    (cp.async.bulk.tensor.2d) into a kStages-deep mbarrier ring; four consumer warps run
//    mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4 — tcgen05 has no f64 kind).
//    grouped_gemm is the same tile machinery, one launch per tree level (diagnostics, and
//    the GEMM of the error oracle in krows.cu).
//  * permute_in / permute_out: the permutation into and out of the padded tree order
//    (executor.cpp:35-39, :245-254), fused with the transpose between the user's column-
//    major W/Y and the point-major internal buffers Wp/T/S/Yp (column blocks kCbPitch apart).
//  * gen_blocks: kernel blocks K(x_rows, x_cols) generated on the device (near field and
//    far blocks of hmxg_upload_generated).
#pragma once

#include <cuda.h>

#include <cstdint>

#include "kfun.cuh"
#include "plan.hpp"

namespace hmxg {
// Internal linkage: every translation unit of libhmxg.so that launches these kernels
// gets its own instantiation (no duplicate host stubs at link time).
namespace {

constexpr int kBM = 64;        // output rows per CTA tile
constexpr int kBN = 64;        // output columns per CTA tile
constexpr int kBK = 16;        // K rows per pipeline chunk
#ifndef HMXG_STAGES
#define HMXG_STAGES 4
#endif
#ifndef HMXG_MIN_CTAS  // resident CTAs per SM the GEMM kernels are compiled for (register cap)
#define HMXG_MIN_CTAS (HMXG_STAGES <= 4 ? 3 : 2)
#endif
constexpr int kStages = HMXG_STAGES;
constexpr int kConsumerWarps = 4;  // 2 x 2 warps, each 4 x 4 interleaved 8 x 8 fragments
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kChunkElems = kBM * kBK;               // A chunk: 64 x 16 doubles
constexpr int kChunkBytes = kChunkElems * 8;         // 8 KB
// B tile: 16 rows (k) x kBPitch columns, row major as TMA writes it. The pitch of 68
// doubles (544 B) shifts consecutive k rows by 8 banks, so each half-warp of a fragment
// load (4 k rows x 4 columns) covers all 32 banks once: conflict-free without a swizzle
// pattern. The 4 extra columns are the next column block's (or TMA zero fill past Q).
constexpr int kBPitch = kBN + 4;
constexpr int kBTileBytes = kBPitch * kBK * 8;       // 8704 B
// Column blocks of the point-major buffers Wp/T/S/Yp are kCbPitch = 80 columns apart: 64
// columns of data and a 128-byte gap. A B tile (kBPitch = 68 columns) then reads 4 gap
// columns instead of the first line of the next column block, whose item may be storing
// to it at that moment: no TMA box shares a cache line with another item's stores.
constexpr int kCbPitch = kBN + 16;
__host__ __device__ __forceinline__ std::uint64_t phys_col(std::uint64_t c) {
  return (c / kBN) * kCbPitch + (c % kBN);
}
__host__ __device__ __forceinline__ std::uint64_t phys_cols(std::uint64_t q) {
  return (q + kBN - 1) / kBN * kCbPitch;
}
constexpr int kStageBytes = kChunkBytes + kBTileBytes;

struct GemmParams {
  const double* tiles;          // pre-tiled A chunks
  const Task* tasks;            // first task of the phase
  const SegDev* segs;
  double* buf[kNumBufs];        // Wp, T, S, Yp
  std::uint64_t ld[kNumBufs];
  std::uint32_t q;
  const std::uint32_t* idmap;   // identity-row sources of the tasks (Task::id_off)
  // fused permutations (eval_dag's small-problem mode): final leaf rows go to Y[pmap[row], :]
  double* y_final;              // null: every task stores into its C buffer
  std::uint64_t ldy;
  const std::uint32_t* pmap;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
  return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// Waits trap after ~2^26 suspended polls (seconds): a dependency or transaction-count bug
// then surfaces as a CUDA error instead of a hung GPU.
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
  std::uint32_t done = 0, polls = 0;
  for (;;) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (++polls > (1u << 26)) __trap();
  }
}
// Non-blocking phase test (acquire at CTA scope when it succeeds).
__device__ __forceinline__ bool mbar_test(std::uint64_t* bar, unsigned parity) {
  std::uint32_t done;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
// The producer lane's waits: a short suspended try, then `svc()` (it forwards the
// consumers' tile signals, eval_dag), so that a producer blocked on its own CTA's
// consumers still publishes what they finished.
template <class Svc>
__device__ __forceinline__ void mbar_wait_svc(std::uint64_t* bar, unsigned parity, Svc&& svc) {
  std::uint32_t done = 0, polls = 0;
  for (;;) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(200u)
        : "memory");
    if (done) return;
    svc();
    if (++polls > (1u << 26)) __trap();
  }
}
struct NoSvc {
  __device__ void operator()() const {}
};
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_2d_g2s(void* dst, const CUtensorMap* map, int x, int y, std::uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<std::uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ double lds64(std::uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Programmatic dependent launch (the DAG path launches eval_dag and permute_out with
// cudaLaunchAttributeProgrammaticStreamSerialization): a dependent grid may start while
// its predecessor runs and waits here before reading the predecessor's output; the
// predecessor lets it launch once all of its own CTAs are running. Both are no-ops for
// grids launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" :::); }

// Uniform selects instead of dynamic indexing into parameter arrays (no local copies).
__device__ __forceinline__ double* pick_buf(const GemmParams& p, unsigned b) {
  return b == kBufWp ? p.buf[kBufWp] : (b == kBufT ? p.buf[kBufT] : (b == kBufS ? p.buf[kBufS] : p.buf[kBufYp]));
}
__device__ __forceinline__ std::uint64_t pick_ld(const GemmParams& p, unsigned b) {
  return b == kBufWp ? p.ld[kBufWp] : (b == kBufT ? p.ld[kBufT] : (b == kBufS ? p.ld[kBufS] : p.ld[kBufYp]));
}

// A chunk layout: element (k, r) of a 64 x 16 chunk lives at k*64 + (r ^ ((k & 3) << 2)).
// A 64-bit fragment load is served per half-warp (lanes r = R..R+3, k = kk..kk+3); the
// XOR on bits 2-3 of r moves the four k rows to four disjoint 8-bank groups, so each
// half-warp is one wavefront (rows are 512 B apart and would otherwise collide).
__host__ __device__ __forceinline__ int a_swz(int k, int r) { return k * kBM + (r ^ ((k & 3) << 2)); }

// One generated kernel block: G(a, b) = K(x_{idx[rows + a]}, x_{idx[cols + b]}), m x ncols
// column major at element offset off. Near blocks index the tree permutation
// (idx = perm, rows = start_i: the node's points, compress.cpp:143-147); far blocks index
// the concatenated skeletons (compress.cpp:139-142). dense_block, kernel.cpp:52-65.
struct GenBlock {
  std::uint64_t off;
  std::uint64_t rows, cols;  // offsets into idx
  std::uint32_t m, ncols;
};

__global__ void __launch_bounds__(256) gen_blocks(const double* __restrict__ pts, const KernelParams kp,
                                                  const std::uint32_t* __restrict__ idx,
                                                  const GenBlock* __restrict__ blocks, std::uint64_t nblocks,
                                                  double* __restrict__ out) {
  for (std::uint64_t s = blockIdx.x; s < nblocks; s += gridDim.x) {
    const GenBlock b = blocks[s];
    const std::uint32_t count = b.m * b.ncols;
    for (std::uint32_t e = threadIdx.x; e < count; e += blockDim.x) {
      const std::uint32_t a = e % b.m, c = e / b.m;  // consecutive threads: consecutive rows
      const std::uint64_t pi = idx[b.rows + a], pj = idx[b.cols + c];
      out[b.off + e] = kernel_value(kp, pts + pi * kp.d, pts + pj * kp.d);
    }
  }
}

// ---------------------------------------------------------------- near field on the fly
// One pre-tiled A chunk of a near block (hmxg_upload_generated_ex, HMXG_UPLOAD_NEAR_ON_THE_FLY):
// element (r, k) = K(x_{pmap[yrow + r]}, x_{pmap[brow + k]}) for r < m, k < kvalid, else 0 --
// the tile's Yp row r and the B chunk's Wp row k name the two points (the leaf row orders of
// the identity-row lowering included), so it equals tile_a's chunk of the block that
// gen_blocks generates at upload, bit for bit (same kernel_value, same argument order).
struct GenChunk {
  std::uint64_t out;   // chunk index in the tiles array (the scratch region)
  std::uint32_t yrow;  // Yp row of tile row 0
  std::uint32_t brow;  // Wp row of k = 0
  std::uint16_t m, kvalid;
  std::uint32_t pad;
};
static_assert(sizeof(GenChunk) == 24, "GenChunk layout");

// A wave's near-field chunks into the scratch region of the tiles (one launch per wave, before
// the wave's leaf rows). Per chunk the CTA stages its 64 row points' and 16 column points'
// coordinates in shared memory (dim-major, so consecutive threads read consecutive rows),
// then every thread forms 4 entries with kernel_value's exact operation sequence and writes
// them swizzled. Dynamic shared memory: 80 * d doubles.
__global__ void __launch_bounds__(256) gen_near(const double* __restrict__ pts, const KernelParams kp,
                                                const std::uint32_t* __restrict__ pmap,
                                                const GenChunk* __restrict__ chunks, std::uint64_t nchunks,
                                                double* __restrict__ tiles) {
  extern __shared__ double xs[];  // [d][80]: rows 0..63 then columns 64..79
  const std::uint32_t d = kp.d;
  for (std::uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const GenChunk g = chunks[c];
    for (std::uint32_t e = threadIdx.x; e < 80u * d; e += blockDim.x) {
      const std::uint32_t p = e / d, i = e % d;  // point slot, dimension
      double v = 0.0;
      if (p < 64 ? p < g.m : p - 64 < g.kvalid) {
        const std::uint64_t pt = __ldg(pmap + (p < 64 ? g.yrow + p : g.brow + (p - 64)));
        v = __ldg(pts + pt * d + i);
      }
      xs[i * 80 + p] = v;
    }
    __syncthreads();
    double* out = tiles + g.out * 1024u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + u * 256, r = e & 63, k = e >> 6;
      double v = 0.0;
      if (r < g.m && k < g.kvalid) {
        double s = 0.0;
        for (std::uint32_t i = 0; i < d; ++i) {
          const double t = __dsub_rn(xs[i * 80 + r], xs[i * 80 + 64 + k]);
          s = __dadd_rn(s, __dmul_rn(t, t));
        }
        v = kernel_of_sqdist(kp, s);
      }
      out[k * 64 + (r ^ ((k & 3) << 2))] = v;  // a_swz(k, r)
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- A pre-tiling
__global__ void tile_a(const double* __restrict__ gd, const double* __restrict__ gb, const double* __restrict__ gv,
                       const double* __restrict__ gc, const TileSrc* __restrict__ srcs, const std::uint32_t* __restrict__ chunk_seg,
                       const std::uint32_t* __restrict__ maps, double* __restrict__ tiles, std::uint64_t nchunks) {
  for (std::uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const TileSrc s = srcs[chunk_seg[c]];
    const std::uint64_t chunk_in_seg = (c * kChunkElems - s.tile_off) / kChunkElems;
    const double* a = (s.gen == kGenD ? gd : (s.gen == kGenB ? gb : (s.gen == kGenV ? gv : gc))) + s.a_off;
    double* out = tiles + c * kChunkElems;
    for (int e = threadIdx.x; e < kChunkElems; e += blockDim.x) {
      int k, r;
      if (s.trans) {  // A(r,k) = a[k + r*lda]: let consecutive threads walk k
        k = e % kBK;
        r = e / kBK;
      } else {        // A(r,k) = a[r + k*lda]: consecutive threads walk r
        r = e % kBM;
        k = e / kBM;
      }
      const std::uint64_t kk = chunk_in_seg * kBK + k;
      double v = 0.0;
      if (r < s.m && kk < s.k) {
        const std::uint64_t rs = s.rmap == kNoMap ? s.r0 + r : maps[s.rmap + s.r0 + r];
        const std::uint64_t ks = s.kmap == kNoMap ? kk : maps[s.kmap + kk];
        v = s.trans ? a[ks + rs * s.lda] : a[rs + ks * s.lda];
      }
      out[a_swz(k, r)] = v;
    }
  }
}

// A consumer thread hands a stage (or a work-item slot) back to the producer. The mbarrier
// arrive does not wait for the thread's outstanding ld.shared to return their data, so
// without the fence the producer could refill the stage under an in-flight fragment load
// (measured on B200: with heavy concurrent LSU traffic on the SM, fragment loads returned
// the next chunk's data). fence.acq_rel.cta retires them first.
__device__ __forceinline__ void release_stage(std::uint64_t* empty) {
  asm volatile("fence.acq_rel.cta;\n" ::: "memory");
  mbar_arrive(empty);
}

// Fragment addresses of a consumer warp (shared window, bytes, relative to a stage): A
// fragment i of k step ks sits at a_base + ks*kAStepBytes + i*kFragStride, B fragment j at
// b_base + ks*kBStepBytes + j*kFragStride, so two base registers and compile-time
// immediates replace a 32-entry address table (see frag_addresses).
constexpr std::uint32_t kAStepBytes = 4 * kBM * 8;       // 4 k rows of the A chunk
constexpr std::uint32_t kBStepBytes = 4 * kBPitch * 8;   // 4 k rows of the B tile
constexpr std::uint32_t kFragStride = 16 * 8;            // fragments 2i+wm are 16 rows / columns apart

// One segment's K loop for a consumer warp: LI x LJ live 8 x 8 fragments (compile time).
// Fragments of k step ks+1 are loaded while step ks multiplies (register double buffer).
// `last_ks`: live k steps of the last chunk (SegDev::last_ksteps, 0 = all four). The
// zero-padded tail of a segment's last chunk is not multiplied: that chunk runs a rolled
// loop over its live k steps (a branch; predicated-off DMMAs would still occupy the pipe).
template <int LI, int LJ>
__device__ __forceinline__ void consume_chunks(double (&acc)[4][4][2], std::uint64_t* full, std::uint64_t* empty,
                                               std::uint32_t smem_base, std::uint32_t a_base, std::uint32_t b_base,
                                               std::uint32_t nchunks, int last_ks, std::uint32_t& it) {
  for (std::uint32_t c = 0; c < nchunks; ++c, ++it) {
    const int stage = it % kStages;
    mbar_wait(&full[stage], (it / kStages) & 1);
    const std::uint32_t sa = smem_base + stage * kStageBytes + a_base;
    const std::uint32_t sb = smem_base + stage * kStageBytes + b_base;
    if (LI > 0 && LJ > 0) {
      if (last_ks == 0 || c + 1 < nchunks) {
        double af[2][4], bf[2][4];
#pragma unroll
        for (int i = 0; i < LI; ++i) af[0][i] = lds64(sa + i * kFragStride);
#pragma unroll
        for (int j = 0; j < LJ; ++j) bf[0][j] = lds64(sb + j * kFragStride);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const int cur = ks & 1;
          if (ks + 1 < 4) {
#pragma unroll
            for (int i = 0; i < LI; ++i) af[cur ^ 1][i] = lds64(sa + (ks + 1) * kAStepBytes + i * kFragStride);
#pragma unroll
            for (int j = 0; j < LJ; ++j) bf[cur ^ 1][j] = lds64(sb + (ks + 1) * kBStepBytes + j * kFragStride);
          }
#pragma unroll
          for (int i = 0; i < LI; ++i)
#pragma unroll
            for (int j = 0; j < LJ; ++j) dmma884(acc[i][j], af[cur][i], bf[cur][j]);
        }
      } else {
#pragma unroll 1
        for (int ks = 0; ks < last_ks; ++ks) {
          double af[4], bf[4];
#pragma unroll
          for (int i = 0; i < LI; ++i) af[i] = lds64(sa + ks * kAStepBytes + i * kFragStride);
#pragma unroll
          for (int j = 0; j < LJ; ++j) bf[j] = lds64(sb + ks * kBStepBytes + j * kFragStride);
#pragma unroll
          for (int i = 0; i < LI; ++i)
#pragma unroll
            for (int j = 0; j < LJ; ++j) dmma884(acc[i][j], af[i], bf[j]);
        }
      }
    }
    release_stage(&empty[stage]);  // every consumer thread releases the stage after its last read
  }
}

// Partial column block (Q not a multiple of 64): runtime-predicated fragments.
__device__ __forceinline__ void consume_chunks_pred(double (&acc)[4][4][2], std::uint64_t* full, std::uint64_t* empty,
                                                    std::uint32_t smem_base, std::uint32_t a_base,
                                                    std::uint32_t b_base, std::uint32_t nchunks, int last_ks,
                                                    std::uint32_t& it, int live_i, int live_j) {
  for (std::uint32_t c = 0; c < nchunks; ++c, ++it) {
    const int stage = it % kStages;
    mbar_wait(&full[stage], (it / kStages) & 1);
    const std::uint32_t sa = smem_base + stage * kStageBytes + a_base;
    const std::uint32_t sb = smem_base + stage * kStageBytes + b_base;
    const int nks = (last_ks == 0 || c + 1 < nchunks) ? 4 : last_ks;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      if (ks >= nks) break;
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = i < live_i ? lds64(sa + ks * kAStepBytes + i * kFragStride) : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = j < live_j ? lds64(sb + ks * kBStepBytes + j * kFragStride) : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (i < live_i && j < live_j) dmma884(acc[i][j], af[i], bf[j]);
    }
    release_stage(&empty[stage]);
  }
}

// ---------------------------------------------------------------- tile bodies
// Shared-memory carve-up of one CTA (both GEMM kernels): kStages x {A chunk, B tile}, the
// stage barriers, a kTileRing-deep ring of claimed work items and their barriers.
#ifndef HMXG_TILE_RING
#define HMXG_TILE_RING 4
#endif
constexpr int kTileRing = HMXG_TILE_RING;
// eval_dag: stored tiles travel from the consumer warps to the producer lane, which
// publishes them at gpu scope (kSigRing-deep ring: counter address, 0 = nothing, kSigEnd)
constexpr int kSigRing = 8;
constexpr std::uint64_t kSigEnd = ~std::uint64_t(0);
// A claimed work item as the producer hands it to the consumers: the item word, its task
// and the task's first kSegSmem segment descriptors (the rest are read from global), so the
// consumers start an item without global round trips for its tables.
constexpr int kSegSmem = 6;
struct RingSlot {
  std::uint64_t item;
  Task task;
  SegDev seg[kSegSmem];
};
static_assert(sizeof(RingSlot) == 192, "RingSlot layout");
static_assert((kStages + kTileRing) % 2 == 0, "the ring slots must start on a 16-byte boundary");
constexpr int kSmemBytes = kStages * kStageBytes + (2 * kStages + 2 * kTileRing) * 8 + kTileRing * sizeof(RingSlot) +
                           3 * kSigRing * 8 + 16 + 1024;

struct CtaSmem {
  unsigned char* stage;    // kStages * kStageBytes, 1024-byte aligned
  std::uint64_t* full;     // [kStages]
  std::uint64_t* empty;    // [kStages]
  std::uint64_t* tfull;    // [kTileRing]
  std::uint64_t* tempty;   // [kTileRing]
  RingSlot* ring;          // [kTileRing] claimed work items
  std::uint64_t* sfull;    // [kSigRing] one arrive per consumer warp
  std::uint64_t* sempty;   // [kSigRing] the producer took the record
  std::uint64_t* saddr;    // [kSigRing]
  std::uint64_t* pbar;     // eval_dag fused mode: the CTA's permute jobs are done (stages free)
  std::uint64_t* ctbar;    // eval_dag CTree mode: the program tables have landed
};

__device__ __forceinline__ CtaSmem carve_smem(unsigned char* smem_raw) {
  CtaSmem c;
  c.stage = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                             ~std::uintptr_t(1023));
  c.full = reinterpret_cast<std::uint64_t*>(c.stage + kStages * kStageBytes);
  c.empty = c.full + kStages;
  c.tfull = c.empty + kStages;
  c.tempty = c.tfull + kTileRing;
  c.ring = reinterpret_cast<RingSlot*>(c.tempty + kTileRing);
  c.sfull = reinterpret_cast<std::uint64_t*>(c.ring + kTileRing);
  c.sempty = c.sfull + kSigRing;
  c.saddr = c.sempty + kSigRing;
  c.pbar = c.saddr + kSigRing;
  c.ctbar = c.pbar + 1;
  return c;
}

__device__ __forceinline__ void init_barriers(const CtaSmem& c) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&c.full[s], 1);
      mbar_init(&c.empty[s], kConsumerWarps * 32);
    }
    for (int s = 0; s < kTileRing; ++s) {
      mbar_init(&c.tfull[s], 1);
      mbar_init(&c.tempty[s], kConsumerWarps * 32);
    }
    for (int s = 0; s < kSigRing; ++s) {
      mbar_init(&c.sfull[s], kConsumerWarps);
      mbar_init(&c.sempty[s], 1);
    }
    mbar_init(c.pbar, 1);
    mbar_init(c.ctbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
}

// Producer lane: post a claimed work item to the ring (waits for the slot to be free) with
// its task (`task_idx`, unless the item is the end) and first segment descriptors.
template <class Svc = NoSvc>
__device__ __forceinline__ RingSlot* post_item(const GemmParams& p, const CtaSmem& c, std::uint32_t seq,
                                               std::uint64_t item, bool end, std::uint32_t task_idx,
                                               Svc&& svc = Svc{}) {
  const int slot = seq % kTileRing;
  RingSlot* rs = &c.ring[slot];
  Task task{};
  SegDev seg[kSegSmem];
  if (!end) {  // loads first, so they overlap the wait for the slot
    task = p.tasks[task_idx];
    const std::uint32_t ns = min(task.seg_end - task.seg_begin, static_cast<std::uint32_t>(kSegSmem));
#pragma unroll
    for (int k = 0; k < kSegSmem; ++k)
      if (k < static_cast<int>(ns)) seg[k] = p.segs[task.seg_begin + k];
  }
  if (seq >= kTileRing) mbar_wait_svc(&c.tempty[slot], ((seq / kTileRing) - 1) & 1, svc);
  rs->item = item;
  if (!end) {
    rs->task = task;
    const std::uint32_t ns = min(task.seg_end - task.seg_begin, static_cast<std::uint32_t>(kSegSmem));
#pragma unroll
    for (int k = 0; k < kSegSmem; ++k)
      if (k < static_cast<int>(ns)) rs->seg[k] = seg[k];
  }
  mbar_arrive(&c.tfull[slot]);  // release: consumers read the slot after their wait
  return rs;
}

// eval_dag's form: the whole slot comes from the claim-order record `rec` (null: the end
// item) as twelve independent 16-byte loads, issued before the wait for the slot.
template <class Svc = NoSvc>
__device__ __forceinline__ RingSlot* post_record(const CtaSmem& c, std::uint32_t seq, std::uint64_t item,
                                                 const RingSlot* rec, Svc&& svc = Svc{}) {
  static_assert(sizeof(RingSlot) % 16 == 0, "RingSlot is copied in 16-byte words");
  constexpr int kWords = sizeof(RingSlot) / 16;
  const int slot = seq % kTileRing;
  RingSlot* rs = &c.ring[slot];
  uint4 v[kWords];
  if (rec) {
#pragma unroll
    for (int k = 0; k < kWords; ++k) v[k] = __ldg(reinterpret_cast<const uint4*>(rec) + k);
  }
  if (seq >= kTileRing) mbar_wait_svc(&c.tempty[slot], ((seq / kTileRing) - 1) & 1, svc);
  if (rec) {
#pragma unroll
    for (int k = 0; k < kWords; ++k) reinterpret_cast<uint4*>(rs)[k] = v[k];
  }
  rs->item = item;
  mbar_arrive(&c.tfull[slot]);  // release: consumers read the slot after their wait
  return rs;
}

// Consumers: the next work item's ring slot. It stays theirs until release_item (the
// segment descriptors are read during the item).
__device__ __forceinline__ const RingSlot* take_item(const CtaSmem& c, std::uint32_t seq) {
  const int slot = seq % kTileRing;
  mbar_wait(&c.tfull[slot], (seq / kTileRing) & 1);
  return &c.ring[slot];
}
__device__ __forceinline__ void release_item(const CtaSmem& c, std::uint32_t seq) {
  release_stage(&c.tempty[seq % kTileRing]);  // the slot's ld.shared must retire first
}
// Segment si of a task: from the ring slot for the first kSegSmem, else from global.
__device__ __forceinline__ SegDev seg_at(const GemmParams& p, const RingSlot* rs, const Task& task, std::uint32_t si) {
  const std::uint32_t k = si - task.seg_begin;
  return k < static_cast<std::uint32_t>(kSegSmem) ? rs->seg[k] : p.segs[si];
}

// Producer lane: stream the A chunks and B tiles of one GEMM tile (column block cb).
// `wait_dep(seg)` runs before a segment's first load (the DAG kernel's dependency wait; a
// no-op per level).
template <class WaitDep, class Svc = NoSvc>
__device__ __forceinline__ void produce_gemm_tile(const GemmParams& p, const CtaSmem& c, const RingSlot* rs,
                                                  std::uint32_t cb, const CUtensorMap* tm_wp, const CUtensorMap* tm_t,
                                                  const CUtensorMap* tm_s, std::uint32_t& it, WaitDep&& wait_dep,
                                                  Svc&& svc = Svc{}) {
  const int x = static_cast<int>(cb * kCbPitch);
  const Task& task = rs->task;
  for (std::uint32_t si = task.seg_begin; si < task.seg_end; ++si) {
    const SegDev sg = seg_at(p, rs, task, si);
    wait_dep(sg);
    const CUtensorMap* map = sg.bbuf == kBufWp ? tm_wp : (sg.bbuf == kBufT ? tm_t : tm_s);
    for (std::uint32_t ch = 0; ch < sg.nchunks; ++ch, ++it) {
      const int stage = it % kStages;
      if (it >= kStages) mbar_wait_svc(&c.empty[stage], ((it / kStages) - 1) & 1, svc);
      unsigned char* st = c.stage + stage * kStageBytes;
      mbar_expect_tx(&c.full[stage], kChunkBytes + kBTileBytes);
      bulk_g2s(st, p.tiles + sg.tile_off + static_cast<std::uint64_t>(ch) * kChunkElems, kChunkBytes,
               &c.full[stage]);
      // coordinates: {column (inner, Q-contiguous), row}
      tma_2d_g2s(st + kChunkBytes, map, x, static_cast<int>(sg.b_row + ch * kBK), &c.full[stage]);
    }
  }
}

// Fragment base addresses of a consumer warp. Fragment i of warp (wm, wn) covers rows
// 8*(2i+wm) .. +7 and fragment j columns 8*(2j+wn) .. +7: interleaving spreads a ragged
// tile's live fragments evenly over the four warps. For lane (fr = lane/4, fk = lane%4)
// at k step ks (k = 4 ks + fk):
//   A: 8 a_swz(k, 8(2i+wm) + fr) = ks*kAStepBytes + i*kFragStride + 8 (64 fk + ((8 wm + fr) ^ 4 fk))
//      (the XOR touches bits 2-3 only, which 16 i leaves alone)
//   B: kChunkBytes + 8 (k kBPitch + 8(2j+wn) + fr) = ks*kBStepBytes + j*kFragStride + b_base
struct FragAddr {
  std::uint32_t a, b;
};

__device__ __forceinline__ FragAddr frag_addresses(int wm, int wn, int fr, int fk) {
  FragAddr f;
  f.a = 8u * (fk * kBM + ((wm * 8 + fr) ^ (fk << 2)));
  f.b = kChunkBytes + 8u * (fk * kBPitch + wn * 8 + fr);
  return f;
}

// Consumers: the K loop and epilogue of one GEMM tile (each element stored exactly once).
// `wait_id(task)` runs before the identity rows are read (the DAG kernel's wait for the
// nodes that produce them; a no-op per level, where they ran in an earlier launch).
struct NoHook {
  template <class... A>
  __device__ void operator()(A...) const {}
};
// Column-split items (narrow DAGs, DagParams::colsplit = S): the 64 columns of a tile are S
// items of 64/S columns on different CTAs, so a short dependency chain of small GEMMs runs
// on S times as many SMs (the K loop of one tile is the DMMA time of one SM). Item `sub`
// covers columns [sub 64/S, (sub+1) 64/S) of the block: its warps' fragments shift by that
// many columns, and only 64/(16 S) fragment columns per warp are live.
// kNarrow (eval_dag's narrow instantiation): column-split items and the fused permutations'
// final stores into Y. The wide instantiation keeps the tile loop of the round-1 kernel.
template <bool kNarrow, class WaitId, class KEnd = NoHook, class KStart = NoHook>
__device__ __forceinline__ void consume_gemm_tile(const GemmParams& p, const CtaSmem& c, const RingSlot* rs,
                                                  const Task& task, std::uint32_t cb, const FragAddr& fa0,
                                                  std::uint32_t& it, WaitId&& wait_id, KEnd&& k_end = KEnd{},
                                                  KStart&& k_start = KStart{}, std::uint32_t sub = 0,
                                                  std::uint32_t split = 1) {
  if (!kNarrow) sub = 0, split = 1;
  const std::uint32_t width = kBN / split, cs = sub * width;  // this item's columns in the block
  const std::uint32_t c0 = cb * kBN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp & 1, wn = warp >> 1, fr = lane >> 2, fk = lane & 3;
  FragAddr fa = fa0;
  fa.b += cs * 8u;
  // Warp-uniform trim of fragments outside the valid rows / the last column block.
  const std::uint32_t ncols = c0 + cs < p.q ? min(width, p.q - c0 - cs) : 0u;
  const int frag_cols = (static_cast<int>(ncols) + 7) / 8;
  const int live_j = min(4, max(0, (frag_cols - wn + 1) / 2));

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // The accumulator starts from rows that are already complete: the task's own C rows
  // (kTaskAccumulate: the leaf phase onto the near phase's rows), plus the identity rows
  // of the bases, exact row copies from Wp or T (upward) or S (downward). The loads are
  // issued before the K loop, so they are in flight while the first chunks arrive.
  // `add` false: the rows are the accumulator's first value (assigned, so no instruction
  // waits for the loads before the first DMMA needs the accumulator); true: added to it
  auto add_rows = [&](const double* B, std::uint64_t ldb, const std::uint32_t (&src)[4], bool add) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (src[i] == kNoMap) continue;
      const double* srow = B + static_cast<std::uint64_t>(src[i]) * ldb + cb * kCbPitch + cs;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = (2 * j + wn) * 8 + 2 * fk;
        if (col + 1 < static_cast<int>(ncols)) {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(srow + col));
          acc[i][j][0] = add ? acc[i][j][0] + v.x : v.x;
          acc[i][j][1] = add ? acc[i][j][1] + v.y : v.y;
        } else if (col < static_cast<int>(ncols)) {
          const double v = __ldcg(srow + col);
          acc[i][j][0] = add ? acc[i][j][0] + v : v;
        }
      }
    }
  };
  if (task.flags & kTaskAccumulate) {
    std::uint32_t own[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = (2 * i + wm) * 8 + fr;
      own[i] = row < task.m ? task.c_row + row : kNoMap;
    }
    wait_id(task, true);
    add_rows(pick_buf(p, task.cbuf), pick_ld(p, task.cbuf), own, false);
  }
  // Identity sources are static: fetched while the producing nodes may still run. Leaf
  // tasks (kTaskIdLast) add the copied rows after the K loop, so that the combined and the
  // split leaf variants sum in one order; the other tasks start the accumulator with them.
  const bool has_id = task.id_off != kNoMap;
  const bool id_last = (task.flags & kTaskIdLast) != 0;
  std::uint32_t srcs[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = (2 * i + wm) * 8 + fr;
    srcs[i] = has_id && row < task.m ? __ldg(p.idmap + task.id_off + row) : kNoMap;
  }
  if (has_id && !id_last) {
    wait_id(task, false);
    // `add` must stay a compile-time constant: a runtime select would wait for the loads
    // here, before the K loop, instead of at the first DMMA
    if (task.flags & kTaskAccumulate)
      add_rows(pick_buf(p, task.id_buf), pick_ld(p, task.id_buf), srcs, true);
    else
      add_rows(pick_buf(p, task.id_buf), pick_ld(p, task.id_buf), srcs, false);
  }

  // Predicated-off DMMAs still occupy the tensor pipe, so ragged tiles branch (warp-
  // uniformly, once per segment) to a K loop instantiated for their live fragment count.
  // A segment may cover only the tile's first rows (SegDev::rows).
  const std::uint32_t base = smem_u32(c.stage);
  k_start(it);
  for (std::uint32_t si = task.seg_begin; si < task.seg_end; ++si) {
    const SegDev sg = seg_at(p, rs, task, si);
    const int rows = sg.rows ? static_cast<int>(sg.rows) : static_cast<int>(task.m);
    const int live_i = min(4, max(0, ((rows + 7) / 8 - wm + 1) / 2));
    const std::uint32_t nch = sg.nchunks;
    const int lks = sg.last_ksteps;
    if (live_i <= 0 || live_j <= 0) {
      consume_chunks<0, 0>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it);
    } else if (live_j == 4) {
      switch (live_i) {
        case 4: consume_chunks<4, 4>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
        case 3: consume_chunks<3, 4>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
        case 2: consume_chunks<2, 4>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
        default: consume_chunks<1, 4>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
      }
    } else if (kNarrow && live_j == 1 && split == 4) {  // column-split items: one live fragment column
      switch (live_i) {
        case 4: consume_chunks<4, 1>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
        case 3: consume_chunks<3, 1>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
        case 2: consume_chunks<2, 1>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
        default: consume_chunks<1, 1>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
      }
    } else if (kNarrow && live_j == 2 && split == 2) {
      switch (live_i) {
        case 4: consume_chunks<4, 2>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
        case 3: consume_chunks<3, 2>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
        case 2: consume_chunks<2, 2>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
        default: consume_chunks<1, 2>(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it); break;
      }
    } else {
      consume_chunks_pred(acc, c.full, c.empty, base, fa.a, fa.b, nch, lks, it, live_i, live_j);
    }
  }
  k_end();
  if (has_id && id_last) {
    if (!(task.flags & kTaskIdSynced)) wait_id(task, false);
    add_rows(pick_buf(p, task.id_buf), pick_ld(p, task.id_buf), srcs, true);
  }

  if (kNarrow && p.y_final && (task.flags & kTaskFinal)) {  // scattered into the caller's column-major Y
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = (2 * i + wm) * 8 + fr;
      if (row >= task.m) continue;
      double* ycol = p.y_final + __ldg(p.pmap + task.c_row + row) + static_cast<std::uint64_t>(c0 + cs) * p.ldy;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int col = (2 * j + wn) * 8 + 2 * fk;
        if (col < static_cast<int>(ncols)) ycol[static_cast<std::uint64_t>(col) * p.ldy] = acc[i][j][0];
        if (col + 1 < static_cast<int>(ncols)) ycol[static_cast<std::uint64_t>(col + 1) * p.ldy] = acc[i][j][1];
      }
    }
    return;
  }
  double* C = pick_buf(p, task.cbuf);
  const std::uint64_t ldc = pick_ld(p, task.cbuf);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = (2 * i + wm) * 8 + fr;
    if (row >= task.m) continue;
    double* crow = C + static_cast<std::uint64_t>(task.c_row + row) * ldc + cb * kCbPitch + cs;  // point major
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = (2 * j + wn) * 8 + 2 * fk;
      if (col + 1 < static_cast<int>(ncols))
        *reinterpret_cast<double2*>(crow + col) = make_double2(acc[i][j][0], acc[i][j][1]);
      else if (col < static_cast<int>(ncols))
        crow[col] = acc[i][j][0];
    }
  }
}

// ---------------------------------------------------------------- level-launch GEMM
// Persistent: gridDim.x = resident CTAs (SMs x occupancy). The producer lane claims output
// tiles of one level from a per-launch atomic counter in raster order (column block
// fastest, so a row tile's A chunks are fetched from HBM once and re-served from L2 to
// every column block) and keeps streaming chunks across tile boundaries: the next tile's
// first chunks land while the consumers run the current tile's epilogue. Used for the
// per-launch breakdown (HMXG_F_LEVEL_LAUNCHES); evaluations run eval_dag.
__global__ void __launch_bounds__(kThreads, HMXG_MIN_CTAS)
grouped_gemm(const __grid_constant__ CUtensorMap tm_wp, const __grid_constant__ CUtensorMap tm_t,
             const __grid_constant__ CUtensorMap tm_s, const GemmParams p, std::uint32_t ntasks,
             std::uint32_t* __restrict__ tile_counter) {
  extern __shared__ unsigned char smem_raw[];
  const CtaSmem c = carve_smem(smem_raw);
  const std::uint32_t col_blocks = (p.q + kBN - 1) / kBN;
  const std::uint32_t ntiles = ntasks * col_blocks;
  init_barriers(c);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == kConsumerWarps) {
    if (lane == 0) {
      std::uint32_t it = 0;
      for (std::uint32_t seq = 0;; ++seq) {
        const std::uint32_t t = atomicAdd(tile_counter, 1u);
        const RingSlot* rs = post_item(p, c, seq, t, t >= ntiles, t / col_blocks);
        if (t >= ntiles) break;
        produce_gemm_tile(p, c, rs, t % col_blocks, &tm_wp, &tm_t, &tm_s, it, [](const SegDev&) {});
      }
    }
    return;
  }
  const FragAddr fa = frag_addresses(warp & 1, warp >> 1, lane >> 2, lane & 3);
  std::uint32_t it = 0;
  for (std::uint32_t seq = 0;; ++seq) {
    const RingSlot* rs = take_item(c, seq);
    const std::uint64_t t = rs->item;
    if (t >= ntiles) {
      release_item(c, seq);
      break;
    }
    const Task task = rs->task;
    consume_gemm_tile<false>(p, c, rs, task, static_cast<std::uint32_t>(t % col_blocks), fa, it,
                      [](const Task&, bool) {});  // the copied rows' level ran in an earlier launch
    release_item(c, seq);
  }
}

// ---------------------------------------------------------------- whole-evaluation DAG
// One persistent launch runs every GEMM tile of every tree level (between the permute-in
// and permute-out kernels). Work items are claimed in a host-built topological order
// (every dependency of an item precedes it), so the lowest unfinished item can always run
// and, with all CTAs of the grid resident, the kernel cannot deadlock. Dependencies are
// per (node, column block): before streaming a segment, a GEMM tile's producer waits until
// every row tile of the segment's source node has been stored for the same column block
// (T or S). There are no level boundaries: a level's first tiles start while the
// previous level's last tiles finish, and there is one launch instead of ~2H.
enum ItemKind : std::uint32_t { kItemGemm = 0, kItemEnd = 3 };
// item word: kind (bits 56-63), column-split part (48-55), column block (32-47), task (0-31)
__host__ __device__ __forceinline__ std::uint64_t make_item(std::uint32_t kind, std::uint32_t cb, std::uint32_t idx,
                                                            std::uint32_t sub = 0) {
  return (static_cast<std::uint64_t>(kind) << 56) | (static_cast<std::uint64_t>(sub) << 48) |
         (static_cast<std::uint64_t>(cb) << 32) | idx;
}
__host__ __device__ __forceinline__ std::uint32_t item_cb(std::uint64_t item) {
  return static_cast<std::uint32_t>(item >> 32) & 0xffffu;
}
__host__ __device__ __forceinline__ std::uint32_t item_sub(std::uint64_t item) {
  return static_cast<std::uint32_t>(item >> 48) & 0xffu;
}

struct DagParams {
  // The claim order as one record per task run: a task's items (column blocks x column-split
  // parts) are consecutive in the order, so item q is column block (q % per_task) / parts,
  // part q % parts of record q / per_task. A record is the ring slot the consumers get: the
  // task and its first kSegSmem segment descriptors, 192 contiguous bytes, so the producer
  // fetches everything about a claimed item in one round trip (the item word, then the task,
  // then its segments were three dependent ones, on the critical path of the short tree-level
  // items).
  const RingSlot* recs;
  std::uint32_t per_task, parts;
  std::uint32_t nitems;
  std::uint32_t* claim;        // work-item counter (zeroed per evaluation)
  std::uint32_t* done;         // [T: nodes*ncb | S: nodes*ncb | Yp: nodes*ncb] warp signals (zeroed)
  const std::uint32_t* node_tiles;
  const std::uint32_t* yp_tiles;  // near-phase row tiles per leaf
  std::uint32_t ncb, nodes;
  std::uint32_t signal_yp;        // the split leaf variant runs: Yp tiles are waited on
  std::uint32_t colsplit;         // column-split parts per tile (1, 2 or 4): targets x colsplit
  std::uint32_t cstride;          // words between counters (narrow DAGs: one per 128-byte line)
  std::uint32_t fwd_signals;      // the producer lane publishes the stored tiles (wide DAGs)
  // Small problems (fused): the permutations run inside this launch. The consumer warps
  // first gather W into Wp for (leaf, column block) jobs, each published on its own counter
  // (done_w), and the tasks that write final leaf rows (kTaskFinal) store them straight into
  // Y through pmap. One launch instead of three: the two kernel boundaries and the
  // permute kernels' fixed latency were a quarter of cfg1's step.
  std::uint32_t fused;
  std::uint32_t n;                // points (rows of W)
  const std::uint32_t* ipmap;     // point -> Wp row
  const std::uint32_t* rowleaf;   // Wp row -> leaf node
  const std::uint32_t* wp_target; // per leaf: its rows (the done_w count of a complete block)
  const double* w;
  std::uint64_t ldw;
  double* y;
  std::uint64_t ldy;
  const std::uint32_t* pmap;      // Wp / Yp row -> original point
  // The last CTA to finish zeroes the claim and completion counters for the next launch
  // (reset_words of them from `claim`, then the exit counter itself); 0: counters are left
  // as they are (the split fallback's stage 0, whose T counters stage 1 reads).
  std::uint32_t reset_words;
  std::uint32_t* exit_ctr;
  std::uint64_t pf_tile_lines;  // fused mode: 128-byte lines of the A chunks prefetched into L2 first
  // CTree mode (small problems, fused): every task but the near field runs inside clusters of
  // ct_csize CTAs, one cluster per 8-column octet of W (the first ct_noct * ct_csize CTAs),
  // level by level with cluster barriers in between; the item list holds the near tiles only.
  // ct_blob: the CTree's tasks (k-step ranges) then, at byte ct_segs_off, their k steps
  // (CtStep); copied to shared memory. ct_units: (local task << 5 | log2 G << 3 | first row octet) work
  // units of G octets, level l = [ct_lvl[l], ct_lvl[l + 1]); ct_tile_base / ct_tile_lines: the
  // A chunks they read (128-byte lines from the tiles' element offset ct_tile_base), prefetched
  // into L2. The final rows go to Yp; each cluster then writes its octet of Y through ipmap.
  std::uint32_t ct_noct, ct_csize, ct_nlev, ct_blob_bytes, ct_segs_off;
  const void* ct_blob;
  const std::uint32_t* ct_units;
  const std::uint32_t* ct_lvl;
  std::uint64_t ct_tile_base, ct_tile_lines;
#ifdef HMXG_TRACE
  // diagnostic builds (tools/dag_trace.py): per claimed item, kTraceWords globaltimer stamps
  unsigned long long* trace;
#endif
};
#ifdef HMXG_TRACE
// per (CTA, claim sequence): smid << 32 | item index, claim, producer issued the item's last
// chunk, consumer warp 0 took the item, its K loop ended, its tile was stored and signalled
constexpr int kTraceWords = 8;  // + [6] first chunk ready (consumer), [7] deps met (producer)
constexpr int kTraceSeq = 4096;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
template <class D>
__device__ __forceinline__ unsigned long long* trace_slot(const D& d, std::uint32_t seq) {
  return seq < kTraceSeq ? d.trace + (static_cast<std::uint64_t>(blockIdx.x) * kTraceSeq + seq) * kTraceWords
                         : nullptr;
}
#define HMXG_STAMP(seq, k) \
  do {                                                                    \
    unsigned long long* tr_ = trace_slot(d, seq);                         \
    if (tr_) tr_[k] = gtimer();                                           \
  } while (0)
#else
#define HMXG_STAMP(seq, k) \
  do {                     \
  } while (0)
#endif

#ifndef HMXG_SPIN_MAX_NS
#define HMXG_SPIN_MAX_NS 256
#endif
#ifndef HMXG_SPIN_SVC_MAX_NS
#define HMXG_SPIN_SVC_MAX_NS 128
#endif
__device__ __forceinline__ std::uint32_t ld_acquire(const std::uint32_t* p) {
  std::uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void spin_until(const std::uint32_t* p, std::uint32_t target) {
  if (ld_acquire(p) >= target) return;
  unsigned ns = 32;
  std::uint32_t polls = 0;
  while (ld_acquire(p) < target) {
    __nanosleep(ns);
    ns = min(ns * 2, static_cast<unsigned>(HMXG_SPIN_MAX_NS));
    if (++polls > (1u << 24)) __trap();  // ~4 s: a missing dependency signal, not a slow tile
  }
}
// The producer lane's dependency wait: polls with a short backoff and forwards its own
// CTA's finished tiles in between (`svc`), since the awaited tile may be one of them.
template <class Svc>
__device__ __forceinline__ void spin_until_svc(const std::uint32_t* p, std::uint32_t target, Svc&& svc) {
  if (ld_acquire(p) >= target) return;
  unsigned ns = 32;
  std::uint32_t polls = 0;
  while (ld_acquire(p) < target) {
    svc();
    __nanosleep(ns);
    ns = min(ns * 2, static_cast<unsigned>(HMXG_SPIN_SVC_MAX_NS));
    if (++polls > (1u << 25)) __trap();
  }
}
__device__ __forceinline__ void red_release_gpu(std::uint32_t* counter, std::uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(counter), "r"(v) : "memory");
}
// A consumer warp has stored its part of an item: publish it. __syncwarp orders the
// lanes' stores before lane 0's release-reduction at gpu scope (no CTA barrier, no L1
// invalidating fence). Counters therefore count warps: targets are kConsumerWarps x items.
__device__ __forceinline__ void warp_signal(std::uint32_t* counter) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(counter) : "memory");
}
// Lane 0 waits (acquire), then the warp proceeds.
__device__ __forceinline__ void warp_wait(const std::uint32_t* counter, std::uint32_t target) {
  if ((threadIdx.x & 31) == 0) spin_until(counter, target);
  __syncwarp();
}

// End of an eval_dag CTA: the CTA's warps meet; the last CTA of the grid to get here (every
// other CTA has stopped reading the counters) zeroes them for the next launch.
__device__ __forceinline__ void dag_exit(const DagParams& d) {
  __shared__ std::uint32_t last;
  __syncthreads();
  if (d.reset_words == 0) return;
  if (threadIdx.x == 0) {
    std::uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;\n" : "=r"(old) : "l"(d.exit_ctr) : "memory");
    last = old + 1 == gridDim.x;
  }
  __syncthreads();
  if (!last) return;
  for (std::uint32_t i = threadIdx.x; i < d.reset_words; i += blockDim.x) d.claim[i] = 0u;
  if (threadIdx.x == 0) *d.exit_ctr = 0u;
}

// ---------------------------------------------------------------- CTree (small problems)
// MatRox's coarsened sub-tree execution (executor.cpp:139-190, structure.cpp:147-186: one
// worker runs a whole disjoint sub-tree with no barrier between its internal levels) on the
// B200: the columns of W are independent, so the whole tree of one 8-column octet is the
// disjoint unit. A cluster of CTAs runs its levels -- upward, far+downward and the leaf rows
// -- separated by cluster barriers (shared-memory-speed) instead of the DAG's gpu-scope
// release / poll / L2 reload per level (~4 us each, the whole of cfg1's step). Only the
// near field (the bulk of the flops, no tree dependency) stays in the DAG's item list, and
// the leaf rows wait for its tiles. Operands are read straight from global memory (A from
// the pre-tiled chunks, B rows of T / S from L2, Wp rows as W[pmap[row], col]) and the
// final rows are stored into Y through pmap. Every 8 x 8 output fragment runs the DAG's
// exact DMMA sequence (accumulator start, segments, chunks, k steps, identity rows last for
// leaf rows), so the results are bit-identical to the DAG and the level launches.
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// The CTree program in shared memory (one bulk copy at the start): its tasks and, per task,
// the flat list of its k steps in the DAG's order (segment, chunk, k step), so that no operand
// address waits on a global load and the loop body stays a few dozen instructions (the
// instruction cache, not the math, bounded the first version).
// CtTask: Task with seg_begin / seg_end = the task's k-step range, pad1 = the leaf whose Wp
// rows it reads (kNoMap: none). CtStep: A = chunk * 4 + k step (the lanes add their k and
// row), B = row << 8 | buffer << 4 | live octet limit (ceil(SegDev::rows / 8), 8 = all).
struct CtStep {
  std::uint32_t a, b;
};
struct CtSmem {
  const Task* tasks;
  const CtStep* steps;
};
// An element of a B operand or identity row: buffer b (Wp, T, S, Yp), padded row, logical
// column. Written during this launch by other CTAs: read at L2 (after the acquire).
__device__ __forceinline__ double ct_load(const GemmParams& p, unsigned b, std::uint32_t row, std::uint32_t col) {
  return __ldcg(pick_buf(p, b) + static_cast<std::uint64_t>(row) * pick_ld(p, b) + phys_col(col));
}
// Counter of (node, column block) in a completion region of stride cst.
template <class D>
__device__ __forceinline__ std::uint64_t at_node(const D& d, std::uint32_t node, std::uint32_t cb, std::uint64_t cst) {
  return (static_cast<std::uint64_t>(node) * d.ncb + cb) * cst;
}
// Lane 0 waits for a counter, then every lane acquires it.
__device__ __noinline__ void ct_wait(const std::uint32_t* ctr, std::uint32_t target) {
  if ((threadIdx.x & 31) == 0) spin_until(ctr, target);
  __syncwarp();
  (void)ld_acquire(ctr);
}

#ifndef HMXG_CT_G
#define HMXG_CT_G 2
#endif
constexpr int kCtG = HMXG_CT_G;  // row octets per CTree unit
#ifndef HMXG_CT_ALD
#define HMXG_CT_ALD __ldg
#endif
// One work unit -- G consecutive 8-row octets of a task x the column octet's 8 columns -- on
// one warp: G independent DMMA chains; two register blocks of KB k steps, the next block's
// loads in flight while the current one multiplies.
template <int G>
__device__ __forceinline__ void ct_unit(const GemmParams& p, const DagParams& d, const CtSmem& cs,
                                       std::uint32_t unit, std::uint32_t cb, std::uint32_t col0,
                                       std::uint32_t ncols, std::uint32_t* done_y, std::uint32_t* done_w,
                                       std::uint64_t cst, std::uint32_t wmul, unsigned long long* ust = nullptr) {
  constexpr int KB = G == 1 ? 6 : (G == 2 ? 3 : 2);  // k steps per register block
  const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
  const Task task = cs.tasks[unit >> 5];
  const std::uint32_t oct0 = unit & 7u;
  const int noct = min(G, static_cast<int>((task.m + 7) / 8) - static_cast<int>(oct0));
  const bool bcol_ok = static_cast<std::uint32_t>(fr) < ncols;  // the lane's B column
  const std::uint32_t bcol = col0 + fr;
  const std::uint32_t cc = 2 * fk;  // the lane's C columns cc, cc + 1 within the octet
#ifdef HMXG_TRACE
  if (ust && lane == 0) ust[0] = gtimer();
#endif
  if (task.pad1 != kNoMap) ct_wait(done_w + at_node(d, task.pad1, cb, cst), d.wp_target[task.pad1]);
#ifdef HMXG_TRACE
  if (ust && lane == 0) ust[1] = gtimer();
#endif
  double acc[G][2];
#pragma unroll
  for (int o = 0; o < G; ++o) acc[o][0] = acc[o][1] = 0.0;
  const bool has_id = task.id_off != kNoMap;
  const bool id_last = (task.flags & kTaskIdLast) != 0;
  std::uint32_t src[G];
#pragma unroll
  for (int o = 0; o < G; ++o) {
    const std::uint32_t row = (oct0 + o) * 8 + fr;
    src[o] = has_id && o < noct && row < task.m ? __ldg(p.idmap + task.id_off + row) : kNoMap;
  }
  // rows (own rows, identity rows) into the accumulators: acc[o] = (add ? acc[o] : 0) + row
#define HMXG_CT_ROWS_IN(B, SRC_OF, ADD)                                                 \
  _Pragma("unroll") for (int o = 0; o < G; ++o) {                                        \
    if (o < noct) {                                                                      \
      const std::uint32_t s_ = (SRC_OF);                                                 \
      double v0 = 0.0, v1 = 0.0;                                                         \
      if (s_ != kNoMap) {                                                                \
        if (cc < ncols) v0 = ct_load(p, (B), s_, col0 + cc);                             \
        if (cc + 1 < ncols) v1 = ct_load(p, (B), s_, col0 + cc + 1);                     \
      }                                                                                  \
      acc[o][0] = (ADD) ? acc[o][0] + v0 : v0;                                           \
      acc[o][1] = (ADD) ? acc[o][1] + v1 : v1;                                           \
    }                                                                                    \
  }
  // the k steps of the task, in the DAG's order, skipping those with no live octet here
  const std::uint32_t k0 = task.seg_begin, k1 = task.seg_end;
  const int lane_a = fk * kBM;  // + (row ^ (fk << 2)) per octet
  double a0[KB][G], b0[KB], a1[KB][G], b1[KB];
  std::uint32_t n0 = 0, n1 = 0;  // live octets of k step j at bits 3j
  std::uint32_t kn = k0;
  auto load_blk = [&](double (&a)[KB][G], double (&b)[KB], std::uint32_t& nl) {
    int c = 0;
    nl = 0;
#pragma unroll
    for (int j = 0; j < KB; ++j) {
      int live = 0;
      CtStep st{};
      while (kn < k1) {  // (dead steps: rows-limited segments below this unit's octets)
        st = cs.steps[kn++];
        live = min(noct, static_cast<int>(st.b & 15u) - static_cast<int>(oct0));
        if (live > 0) break;
      }
      if (live > 0) {
        const double* ach = p.tiles + static_cast<std::uint64_t>(st.a >> 2) * kChunkElems + (st.a & 3u) * 4 * kBM + lane_a;
#pragma unroll
        for (int o = 0; o < G; ++o)
          if (o < live) a[j][o] = HMXG_CT_ALD(ach + ((((oct0 + o) * 8 + fr)) ^ (fk << 2)));
        b[j] = bcol_ok ? ct_load(p, (st.b >> 4) & 15u, (st.b >> 8) + fk, bcol) : 0.0;
        nl |= static_cast<std::uint32_t>(live) << (3 * j);
        c = j + 1;
      }
    }
    return c;
  };
  auto mul_blk = [&](const double (&a)[KB][G], const double (&b)[KB], std::uint32_t nl, int c) {
#pragma unroll
    for (int j = 0; j < KB; ++j)
      if (j < c)
#pragma unroll
        for (int o = 0; o < G; ++o)
          if (o < static_cast<int>((nl >> (3 * j)) & 7u)) dmma884(acc[o], a[j][o], b[j]);
  };
  // the first two blocks' operands go out before the accumulator's start rows are waited
  // for (a leaf task's near tiles may still be in flight)
  int c0 = load_blk(a0, b0, n0);
  int c1 = c0 ? load_blk(a1, b1, n1) : 0;
  if (task.flags & kTaskAccumulate) {  // the near tiles of this leaf (DAG items) are stored
    ct_wait(done_y + at_node(d, task.node, cb, cst), d.yp_tiles[task.node] * wmul);
    HMXG_CT_ROWS_IN(task.cbuf, (oct0 + o) * 8 + fr < task.m ? task.c_row + (oct0 + o) * 8 + fr : kNoMap, false)
  }
  if (has_id && !id_last) {
    if (task.flags & kTaskAccumulate) {
      HMXG_CT_ROWS_IN(task.id_buf, src[o], true)
    } else {
      HMXG_CT_ROWS_IN(task.id_buf, src[o], false)
    }
  }
#ifdef HMXG_TRACE
  int blk_ = 0;
  // per block: DMMAs done (the accumulator read forces completion), up to 12 blocks
#define HMXG_CT_BSTAMP()                                                                          \
  if (ust && lane == 0 && blk_ < 12) {                                                           \
    double z_ = acc[0][0];                                                                       \
    asm volatile("" : "+d"(z_));                                                                 \
    ust[5 + blk_] = gtimer() + (z_ == 12345.678 ? 1ull : 0ull);                                  \
  }                                                                                              \
  ++blk_;
#else
#define HMXG_CT_BSTAMP()
#endif
  while (c0) {
    mul_blk(a0, b0, n0, c0);
    HMXG_CT_BSTAMP()
    if (!c1) break;
    c0 = load_blk(a0, b0, n0);
    mul_blk(a1, b1, n1, c1);
    HMXG_CT_BSTAMP()
    if (!c0) break;
    c1 = load_blk(a1, b1, n1);
  }
#undef HMXG_CT_BSTAMP
  if (has_id && id_last) {
    HMXG_CT_ROWS_IN(task.id_buf, src[o], true)
  }
#undef HMXG_CT_ROWS_IN
  double* const cbase = pick_buf(p, task.cbuf);
  const std::uint64_t ldc = pick_ld(p, task.cbuf);
#pragma unroll
  for (int o = 0; o < G; ++o) {
    const std::uint32_t row = (oct0 + o) * 8 + fr;
    if (o >= noct || row >= task.m) continue;
    double* crow = cbase + static_cast<std::uint64_t>(task.c_row + row) * ldc + phys_col(col0 + cc);
    if (cc + 1 < ncols)
      __stcg(reinterpret_cast<double2*>(crow), make_double2(acc[o][0], acc[o][1]));
    else if (cc < ncols)
      __stcg(crow, acc[o][0]);
  }
#ifdef HMXG_TRACE
  if (ust && lane == 0) {
    ust[3] = gtimer();
    ust[4] = (static_cast<unsigned long long>(unit) << 32) | (k1 - k0);
  }
  if (ust && lane == 0) ust[2] = ust[5];
#endif
}

// A CTree cluster: octet `oct` of the columns, this CTA's rank in the cluster. Every thread of
// every CTA of the cluster runs the same number of cluster barriers. `c.stage` holds the
// program tables (the CTA joins the item loop afterwards, when the stages are free again).
__device__ __forceinline__ void ct_run(const GemmParams& p, const DagParams& d, const CtaSmem& c,
                                      std::uint32_t oct, std::uint32_t rank, std::uint32_t* done_y,
                                      std::uint32_t* done_w, std::uint64_t cst, std::uint32_t wmul) {
  const std::uint32_t cb = oct / (kBN / 8), col0 = oct * 8;
  const std::uint32_t ncols = min(8u, p.q - col0);
#ifdef HMXG_TRACE
  const unsigned long long t_start = gtimer();
#endif
  if (threadIdx.x == 0) {  // the tables: bulk copies of <= 32 KB (sizes are multiples of 16)
    mbar_expect_tx(c.ctbar, d.ct_blob_bytes);
    for (std::uint32_t off = 0; off < d.ct_blob_bytes; off += 32768u)
      bulk_g2s(c.stage + off, reinterpret_cast<const unsigned char*>(d.ct_blob) + off,
               min(32768u, d.ct_blob_bytes - off), c.ctbar);
  }
  {  // the A chunks into L2 meanwhile (after an L2 flush they would come from DRAM at the level
     // that first reads them): this cluster's share of the program's range
    const std::uint32_t tid = rank * kThreads + threadIdx.x, nt = d.ct_csize * kThreads;
    for (std::uint64_t l = tid + static_cast<std::uint64_t>(oct) * nt; l < d.ct_tile_lines; l += nt * d.ct_noct)
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p.tiles + d.ct_tile_base + l * 16));
  }
  mbar_wait(c.ctbar, 0);
  const CtSmem cs{reinterpret_cast<const Task*>(c.stage), reinterpret_cast<const CtStep*>(c.stage + d.ct_segs_off)};
#ifdef HMXG_TRACE
  // trace builds: [marker | oct << 8 | rank, start, tables copied, level 0 end, ...] in the
  // CTA's last-but-one two trace slots (16 words)
  unsigned long long* ctr_ = d.trace + (static_cast<std::uint64_t>(blockIdx.x) * kTraceSeq + kTraceSeq - 3) * kTraceWords;
  if (threadIdx.x == 0) {
    ctr_[0] = 0xc7ee000000000000ull | (static_cast<unsigned long long>(oct) << 8) | rank;
    ctr_[1] = t_start;
    ctr_[2] = gtimer();
  }
#endif
  const std::uint32_t warps = kThreads / 32;
  const std::uint32_t gw = rank * warps + (threadIdx.x >> 5), nw = d.ct_csize * warps;
  for (std::uint32_t l = 0; l < d.ct_nlev; ++l) {
    const std::uint32_t u0 = __ldg(d.ct_lvl + l), u1 = __ldg(d.ct_lvl + l + 1);
    for (std::uint32_t u = u0 + gw; u < u1; u += nw) {
      const std::uint32_t unit = __ldg(d.ct_units + u);
      // one instantiation (kCtG octets per unit): two or more inlined bodies make ptxas spill
      // the whole kernel at its 128-register bound
#ifdef HMXG_TRACE
      // per warp, its first unit of level 0 (5 words) in the trace slots below the CTree record
      unsigned long long* ust = nullptr;
      if (u < u0 + nw && l == 0)
        ust = d.trace + (static_cast<std::uint64_t>(blockIdx.x) * kTraceSeq + kTraceSeq - 8 - 3 * 5) * kTraceWords +
              (threadIdx.x >> 5) * 24;
      ct_unit<kCtG>(p, d, cs, unit, cb, col0, ncols, done_y, done_w, cst, wmul, ust);
#else
      ct_unit<kCtG>(p, d, cs, unit, cb, col0, ncols, done_y, done_w, cst, wmul);
#endif
    }
#ifdef HMXG_TRACE
    if (l < 12) {
      __syncthreads();
      if (threadIdx.x == 0) ctr_[3 + l] = gtimer();
    }
#endif
    cluster_sync_all();  // this level's rows before the next level (or the scatter) reads them
  }
  // Y[:, octet] = Yp rows through ipmap, this CTA's share of the points: every near tile is
  // stored (the leaves without a basis have no CTree task that waited for theirs)
  for (std::uint32_t i = threadIdx.x; i < d.nodes; i += kThreads)
    if (d.yp_tiles[i]) {
      const std::uint32_t* ctr = done_y + at_node(d, i, cb, cst);
      spin_until(ctr, d.yp_tiles[i] * wmul);
    }
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  __syncthreads();
  const double* yp = p.buf[kBufYp] + phys_col(col0);
  const std::uint64_t ldyp = p.ld[kBufYp];
  const std::uint32_t per = (d.n + d.ct_csize - 1) / d.ct_csize;
  const std::uint32_t r1 = min(d.n, (rank + 1) * per);
  for (std::uint32_t r = rank * per + threadIdx.x; r < r1; r += kThreads) {
    const double* src = yp + static_cast<std::uint64_t>(__ldg(d.ipmap + r)) * ldyp;
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      const double2 x = __ldcg(reinterpret_cast<const double2*>(src + u));
      v[u] = x.x;
      v[u + 1] = x.y;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (static_cast<std::uint32_t>(u) < ncols) d.y[r + static_cast<std::uint64_t>(col0 + u) * d.ldy] = v[u];
  }
#ifdef HMXG_TRACE
  __syncthreads();
  if (threadIdx.x == 0) ctr_[15] = gtimer();
#endif
  __syncthreads();  // the stage area is the producer's again
}

// kNarrow: the instantiation for narrow DAGs (column-split items, padded counters, fused
// permutations, self-reset); the wide one compiles those paths out (they cost the cfg5 DAG
// 3.8% as runtime branches).
template <bool kNarrow>
__global__ void __launch_bounds__(kThreads, HMXG_MIN_CTAS)
eval_dag(const __grid_constant__ CUtensorMap tm_wp, const __grid_constant__ CUtensorMap tm_t,
         const __grid_constant__ CUtensorMap tm_s, const GemmParams p, const DagParams d) {
  extern __shared__ unsigned char smem_raw[];
  const CtaSmem c = carve_smem(smem_raw);
  init_barriers(c);
  pdl_trigger();  // permute_out may launch; it waits for this grid before reading Yp
  pdl_wait();     // Wp and the zeroed counters of permute_in
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const std::uint64_t cst = kNarrow ? d.cstride : 1, region = static_cast<std::uint64_t>(d.nodes) * d.ncb * cst;
  std::uint32_t* const done_t = d.done;
  std::uint32_t* const done_s = done_t + region;
  std::uint32_t* const done_y = done_s + region;
  std::uint32_t* const done_w = done_y + region;
  auto at = [&](std::uint32_t node, std::uint32_t cb) { return (static_cast<std::uint64_t>(node) * d.ncb + cb) * cst; };
  const std::uint32_t wmul = kConsumerWarps * (kNarrow ? d.colsplit : 1);  // signals per complete row tile
  // CTree mode: the first ct_ctas CTAs are the octet clusters; they run their trees first and
  // then join the item loop (which by then only has the end item for them)
  const std::uint32_t ct_ctas = kNarrow ? d.ct_noct * d.ct_csize : 0u;
  const bool ct_cta = kNarrow && blockIdx.x < ct_ctas;
  if (kNarrow && ct_cta) ct_run(p, d, c, blockIdx.x / d.ct_csize, blockIdx.x % d.ct_csize, done_y, done_w, cst, wmul);

  if (kNarrow && d.fused && d.pf_tile_lines) {
    // Small problems start cold (an L2 flush, or just the previous evaluation's traffic):
    // every CTA sends a share of the A chunks and of W to L2 first, so each level's first
    // loads hit L2 instead of paying a DRAM round trip on the critical chain.
    const std::uint64_t tid = static_cast<std::uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const std::uint64_t nt = static_cast<std::uint64_t>(gridDim.x) * kThreads;
    for (std::uint64_t l = tid; l < d.pf_tile_lines; l += nt)
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p.tiles + l * 16));
    const std::uint64_t wl = (static_cast<std::uint64_t>(d.n) + 15) / 16;  // lines per column of W
    for (std::uint64_t l = tid; l < wl * p.q; l += nt)
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(d.w + (l % wl) * 16 + (l / wl) * d.ldw));
  }
  if (kNarrow && d.fused && warp < kConsumerWarps) {
    // Wp[ipmap[r]][phys(c)] = W[r + c ldw] in source order: a job is 32 consecutive points x
    // one column block, read as whole 256-byte column segments, transposed through shared
    // memory (the stage buffers: this CTA's producer issues no chunk before pbar) and written
    // as whole point rows; each of the job's points then counts toward its leaf's done_w.
    // One HBM round trip per job instead of the dependent pmap -> W gathers.
    const int tid = threadIdx.x;  // 0 .. 127
    double* tile = reinterpret_cast<double*>(c.stage);  // 32 x 65
    std::uint32_t* rows = reinterpret_cast<std::uint32_t*>(tile + 32 * 65);  // Wp rows of the job
#ifdef HMXG_TRACE
    unsigned long long* ptr_ = d.trace + (static_cast<std::uint64_t>(blockIdx.x) * kTraceSeq + kTraceSeq - 1) * kTraceWords;
    if (tid == 0) ptr_[1] = gtimer();
#endif
    const std::uint32_t nblk = (d.n + 31) / 32;
    // the CTree clusters read W directly: the other CTAs gather Wp for the near tiles
    for (std::uint32_t job = ct_cta ? nblk * d.ncb : blockIdx.x - ct_ctas; job < nblk * d.ncb;
         job += gridDim.x - ct_ctas) {
      const std::uint32_t r0 = (job / d.ncb) * 32, cb = job % d.ncb;
      const std::uint32_t ncols = min(static_cast<std::uint32_t>(kBN), p.q - cb * kBN);
      const std::uint32_t nr = min(32u, d.n - r0);
      double v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const std::uint32_t e = u * 128 + tid, r = e & 31, cc = e >> 5;
        v[u] = (r < nr && cc < ncols) ? __ldg(d.w + r0 + r + static_cast<std::uint64_t>(cb * kBN + cc) * d.ldw) : 0.0;
      }
      if (tid < 32) rows[tid] = tid < static_cast<int>(nr) ? __ldg(d.ipmap + r0 + tid) : 0u;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const std::uint32_t e = u * 128 + tid;
        tile[(e & 31) * 65 + (e >> 5)] = v[u];
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumerWarps * 32) : "memory");
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const std::uint32_t e = u * 128 + tid, cc = e & 63, r = e >> 6;
        if (r < nr && cc < ncols)
          p.buf[kBufWp][static_cast<std::uint64_t>(rows[r]) * p.ld[kBufWp] + cb * kCbPitch + cc] = tile[r * 65 + cc];
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumerWarps * 32) : "memory");
#ifdef HMXG_TRACE
      if (tid == 0) ptr_[2] = gtimer();
#endif
      if (tid < static_cast<int>(nr)) {  // the CTA's stores (bar.sync above) before this point's release
        asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
        red_release_gpu(done_w + at(__ldg(d.rowleaf + rows[tid]), cb), 1u);
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumerWarps * 32) : "memory");  // tile / rows reuse
    }
#ifdef HMXG_TRACE
    if (tid == 0) {
      ptr_[3] = gtimer();
      ptr_[0] = 0xfffffffffull;  // marks the permute record (not an item)
    }
#endif
    if (tid == 0) mbar_arrive(c.pbar);  // the stage buffers are the producer's again
  }

  if (warp == kConsumerWarps) {
    if (lane == 0) {
      // Forward the consumers' stored tiles (sig ring, in item order) to the done counters
      // with a gpu-scope release: the consumer warps only arrive on a CTA-scope barrier
      // after their stores, and go on to the next item instead of waiting for their stores
      // to become visible to the whole GPU. Release is cumulative: the stores the
      // consumers made before their arrive (acquired by the test below) are published.
      // Narrow DAGs (few items per CTA) keep the consumers' own release: there the
      // producer lane is the busier side, and its fences would delay its chunk issue.
      std::uint32_t sig_seq = 0;
      bool consumers_done = d.fwd_signals == 0;
      auto service = [&]() {
        while (!consumers_done) {
          const int slot = sig_seq % kSigRing;
          if (!mbar_test(&c.sfull[slot], (sig_seq / kSigRing) & 1)) return;
          const std::uint64_t a = c.saddr[slot];
          if (a == kSigEnd) {
            consumers_done = true;
            return;
          }
          if (a) red_release_gpu(reinterpret_cast<std::uint32_t*>(a), kConsumerWarps);
          mbar_arrive(&c.sempty[slot]);
          ++sig_seq;
        }
      };
      std::uint32_t it = 0;
      bool stages_free = !kNarrow || !d.fused;
      for (std::uint32_t seq = 0;; ++seq) {
        const std::uint32_t q = atomicAdd(d.claim, 1u);
        const std::uint32_t run = q / d.per_task, rem = q - run * d.per_task;
        const std::uint64_t item = q < d.nitems ? make_item(kItemGemm, rem / d.parts, run, rem % d.parts)
                                                : make_item(kItemEnd, 0, 0);
#ifdef HMXG_TRACE
        unsigned long long* tr = trace_slot(d, seq);
        if (tr && q < d.nitems) {
          tr[0] = (static_cast<unsigned long long>(smid()) << 32) | q;
          tr[1] = gtimer();
        }
#endif
        const bool end = static_cast<std::uint32_t>(item >> 56) == kItemEnd;
        const RingSlot* rs = post_record(c, seq, item, end ? nullptr : d.recs + run, service);
        if (end) break;
        const std::uint32_t cb = item_cb(item);
        if (!stages_free) {  // fused mode: the consumers' permute jobs use the stage buffers
          mbar_wait_svc(c.pbar, 0, service);
          stages_free = true;
        }
        produce_gemm_tile(p, c, rs, cb, &tm_wp, &tm_t, &tm_s, it, [&](const SegDev& sg) {
          if (sg.bbuf == kBufWp) {
            if (!kNarrow || !d.fused) return;  // Wp is complete: permute_in ran before this launch
            spin_until_svc(done_w + at(sg.src, cb), d.wp_target[sg.src], service);
          } else {
            spin_until_svc((sg.bbuf == kBufT ? done_t : done_s) + at(sg.src, cb),
                           d.node_tiles[sg.src] * wmul, service);
          }
          // generic-proxy stores of other CTAs, acquired above, before our async-proxy reads
          asm volatile("fence.proxy.async.global;\n" ::: "memory");
          HMXG_STAMP(seq, 7);
        }, service);
        service();
        HMXG_STAMP(seq, 2);
      }
      std::uint32_t polls = 0;
      while (!consumers_done) {  // the last tiles, up to the consumers' end record
        service();
        __nanosleep(64);
        if (++polls > (1u << 26)) __trap();
      }
    }
    if (kNarrow) dag_exit(d);
    return;
  }
  // consumer warps: hand an item's stored tile (or, with kSigEnd, the end) to the producer
  auto post_signal = [&](std::uint32_t seq, std::uint64_t addr) {
    __syncwarp();  // the warp's stores before lane 0's release arrive
    if (lane == 0) {
      const int slot = seq % kSigRing;
      if (seq >= kSigRing) mbar_wait(&c.sempty[slot], ((seq / kSigRing) - 1) & 1);
      if (warp == 0) c.saddr[slot] = addr;
      mbar_arrive(&c.sfull[slot]);
    }
  };

  const FragAddr fa = frag_addresses(warp & 1, warp >> 1, lane >> 2, lane & 3);
  std::uint32_t it = 0;
  for (std::uint32_t seq = 0;; ++seq) {
    const RingSlot* rs = take_item(c, seq);
    const std::uint64_t item = rs->item;
    if (static_cast<std::uint32_t>(item >> 56) == kItemEnd) {
      release_item(c, seq);
      if (d.fwd_signals) post_signal(seq, kSigEnd);
      break;
    }
    const bool stamp = threadIdx.x == 0;
    if (stamp) HMXG_STAMP(seq, 3);
    const std::uint32_t cb = item_cb(item), sub = item_sub(item);
    const Task task = rs->task;
    consume_gemm_tile<kNarrow>(p, c, rs, task, cb, fa, it, [&](const Task& t, bool own_rows) {
      // the rows about to be read are complete for this column block (every lane acquires;
      // the reads are plain L2 loads): the near phase's rows of this leaf, or the nodes
      // whose rows are copied (Wp is complete before the launch)
      // Fast path: every lane acquires the counter(s) in one L2 round trip, both nodes' loads
      // in flight together; the rows are nearly always complete by the time an item is taken
      // (the producer claimed it microseconds earlier). Otherwise lane 0 polls with a backoff
      // and the lanes acquire afterwards. (One poll + one acquire per node in sequence was four
      // dependent round trips, ~2 us, at the start of every upward item of a few chunks.)
      auto wait_for2 = [&](const std::uint32_t* c0, std::uint32_t t0, const std::uint32_t* c1, std::uint32_t t1) {
        const std::uint32_t v0 = ld_acquire(c0);
        const std::uint32_t v1 = c1 ? ld_acquire(c1) : t1;
        if (__all_sync(0xffffffffu, v0 >= t0 && v1 >= t1)) return;
        if (lane == 0) {
          spin_until(c0, t0);
          if (c1) spin_until(c1, t1);
        }
        __syncwarp();
        (void)ld_acquire(c0);
        if (c1) (void)ld_acquire(c1);
      };
      if (own_rows) {
        wait_for2(done_y + at(t.node, cb), d.yp_tiles[t.node] * wmul, nullptr, 0);
        return;
      }
      if (t.id_buf == kBufWp) {
        if (kNarrow && d.fused && t.id_node0 != kNoMap)
          wait_for2(done_w + at(t.id_node0, cb), d.wp_target[t.id_node0], nullptr, 0);
        return;
      }
      std::uint32_t* const reg = t.id_buf == kBufT ? done_t : done_s;
      const std::uint32_t n0 = t.id_node0 != kNoMap ? t.id_node0 : t.id_node1;
      const std::uint32_t n1 = t.id_node0 != kNoMap ? t.id_node1 : kNoMap;
      if (n0 == kNoMap) return;
      wait_for2(reg + at(n0, cb), d.node_tiles[n0] * wmul, n1 != kNoMap ? reg + at(n1, cb) : nullptr,
                n1 != kNoMap ? d.node_tiles[n1] * wmul : 0u);
    }, [&]() {
      if (stamp) HMXG_STAMP(seq, 4);
    }, [&](std::uint32_t it0) {
#ifdef HMXG_TRACE
      if (task.seg_end > task.seg_begin) {  // trace builds: when the first chunk is ready
        mbar_wait(&c.full[it0 % kStages], (it0 / kStages) & 1);
        if (stamp) HMXG_STAMP(seq, 6);
      }
#else
      (void)it0;
#endif
    }, kNarrow ? sub : 0u, kNarrow ? d.colsplit : 1u);
    // Yp rows have a reader inside the launch only in the split leaf variant (the leaf
    // phase accumulates onto the near phase's rows of the same leaf)
    release_item(c, seq);
    // final leaf rows have no reader inside the launch (the split variant's near rows do)
    // (CTree mode: every near tile, the clusters read them all)
    const bool publish = task.cbuf != kBufYp || (d.signal_yp && !(task.flags & kTaskFinal)) || (kNarrow && d.ct_noct);
    std::uint32_t* const ctr = (task.cbuf == kBufT ? done_t : (task.cbuf == kBufS ? done_s : done_y)) + at(task.node, cb);
    if (d.fwd_signals)
      post_signal(seq, publish ? reinterpret_cast<std::uint64_t>(ctr) : 0);
    else if (publish)
      warp_signal(ctr);
    if (stamp) HMXG_STAMP(seq, 5);
  }
  if (kNarrow) dag_exit(d);
}

// Race detector of debug runs (HMXG_POISON=1): every live row of a workspace buffer (the
// rows of `rows`, all physical columns of the call) is set to NaN before the evaluation, so a
// tile read before its producer stored it (or a row nobody writes) surfaces as NaN in Y
// instead of as the previous evaluation's data. Pad rows stay zero: the 16-row B chunks read
// them as zeros by design.
__global__ void __launch_bounds__(256) poison_rows(double* __restrict__ buf, std::uint64_t ld,
                                                   const std::uint32_t* __restrict__ rows, std::uint64_t nrows,
                                                   std::uint64_t ncols) {
  const double nan = __longlong_as_double(0x7ff8dead00000000ll);
  const std::uint64_t total = nrows * ncols;
  for (std::uint64_t e = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<std::uint64_t>(gridDim.x) * blockDim.x)
    buf[static_cast<std::uint64_t>(rows[e / ncols]) * ld + e % ncols] = nan;
}

// Subtree-split stage 1: the T tiles of the other parts' nodes were filled by the
// exchange; mark them complete for every column block.
__global__ void preset_done(const std::uint32_t* __restrict__ nodes, std::uint32_t count, std::uint32_t* done_t,
                            std::uint32_t ncb, const std::uint32_t* __restrict__ node_tiles) {
  const std::uint64_t i = blockIdx.x * static_cast<std::uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= static_cast<std::uint64_t>(count) * ncb) return;
  const std::uint32_t node = nodes[i / ncb], cb = static_cast<std::uint32_t>(i % ncb);
  done_t[static_cast<std::uint64_t>(node) * ncb + cb] = node_tiles[node] * kConsumerWarps;
}


// Transpose-permute into the point-major internal layout: Wp[ipmap[r], c] = W[r, c]
// (column c at physical column phys_col(c)).
// A 32 x 32 tile is read column by column (256 B contiguous per column of W), turned
// around in shared memory and written row by row (256 B contiguous per point row of Wp),
// so both sides move whole cache lines although the rows land in permuted order.
constexpr int kTT = 32;
// `zero` (optional): words the next launch needs zeroed (eval_dag's claim and completion
// counters), cleared here instead of by a separate memset node; the blocks split them.
__global__ void __launch_bounds__(256) permute_in(const double* __restrict__ w, std::uint64_t ldw,
                                                  const std::uint32_t* __restrict__ ipmap, double* __restrict__ wp,
                                                  std::uint64_t ldwp, std::uint32_t n, std::uint32_t q,
                                                  std::uint32_t* __restrict__ zero, std::uint64_t nzero) {
  __shared__ double tile[kTT][kTT + 1];
  pdl_trigger();
  if (zero) {
    const std::uint64_t nb = static_cast<std::uint64_t>(gridDim.x) * gridDim.y;
    const std::uint64_t b = blockIdx.y * static_cast<std::uint64_t>(gridDim.x) + blockIdx.x;
    for (std::uint64_t i = b * blockDim.x + threadIdx.x; i < nzero; i += nb * blockDim.x) zero[i] = 0u;
  }
  const std::uint32_t r0 = blockIdx.x * kTT, c0 = blockIdx.y * kTT;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 warps
#pragma unroll
  for (int k = 0; k < kTT; k += 8) {
    const std::uint32_t r = r0 + tx, c = c0 + ty + k;
    tile[ty + k][tx] = (r < n && c < q) ? __ldg(w + r + static_cast<std::uint64_t>(c) * ldw) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kTT; k += 8) {
    const std::uint32_t r = r0 + ty + k, c = c0 + tx;
    if (r < n && c < q) wp[static_cast<std::uint64_t>(ipmap[r]) * ldwp + phys_col(c)] = tile[tx][ty + k];
  }
}

// Inverse: Y[r, c] = Yp[ipmap[r], c] (point rows read whole, columns of Y written whole).
// `zero` (optional): eval_dag's counters, zeroed for the next launch once the DAG finished.
__global__ void __launch_bounds__(256) permute_out(const double* __restrict__ yp, std::uint64_t ldyp,
                                                   const std::uint32_t* __restrict__ ipmap, double* __restrict__ y,
                                                   std::uint64_t ldy, std::uint32_t n, std::uint32_t q,
                                                   std::uint32_t* __restrict__ zero, std::uint64_t nzero) {
  __shared__ double tile[kTT][kTT + 1];
  pdl_wait();  // Yp is complete (a no-op without programmatic launch)
  if (zero) {
    const std::uint64_t nb = static_cast<std::uint64_t>(gridDim.x) * gridDim.y;
    const std::uint64_t b = blockIdx.y * static_cast<std::uint64_t>(gridDim.x) + blockIdx.x;
    for (std::uint64_t i = b * blockDim.x + threadIdx.x; i < nzero; i += nb * blockDim.x) zero[i] = 0u;
  }
  const std::uint32_t r0 = blockIdx.x * kTT, c0 = blockIdx.y * kTT;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kTT; k += 8) {
    const std::uint32_t r = r0 + ty + k, c = c0 + tx;
    tile[ty + k][tx] = (r < n && c < q) ? __ldg(yp + static_cast<std::uint64_t>(ipmap[r]) * ldyp + phys_col(c)) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kTT; k += 8) {
    const std::uint32_t r = r0 + tx, c = c0 + ty + k;
    if (r < n && c < q) y[r + static_cast<std::uint64_t>(c) * ldy] = tile[tx][ty + k];
  }
}

}  // namespace
}  // namespace hmxg
