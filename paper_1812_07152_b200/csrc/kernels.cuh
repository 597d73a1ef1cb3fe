// kernels.cuh — sm_100a kernels of the evaluator.
//
//  * tile_a: one-time (upload) re-layout of every GEMM A operand (V^T, V, B_ij, D_ij
//    row tiles) into zero-padded, XOR-swizzled 64 x 16 FP64 chunks, so the main kernel
//    streams A with one 8 KB bulk copy per chunk and reads it without bank conflicts.
//  * grouped_gemm: warp-specialized, mbarrier-pipelined grouped FP64 GEMM. One CTA owns
//    one (output row tile, 64-column block); its K loop walks the tile's segment list,
//    so a whole far+downward sum or a whole leaf row (V_i S_i + sum_j D_ij Wp_j) is
//    accumulated in registers and stored once (single writer, no atomics). A producer
//    warp streams A chunks with cp.async.bulk and B tiles (rows of Wp/T/S, 16 x 64) with
//    TMA (cp.async.bulk.tensor, SWIZZLE_128B) into a kStages-deep ring; four consumer
//    warps run mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4 — tcgen05 has no f64 kind).
//  * permute_in / permute_out: the permutation into and out of the padded tree order
//    (executor.cpp:35-39, :245-254), fused with the transpose between the user's column-
//    major W/Y and the point-major (Q-contiguous) internal buffers Wp/T/S/Yp.
#pragma once

#include <cuda.h>

#include <cstdint>

#include "plan.hpp"

namespace hmxg {

constexpr int kBM = 64;        // output rows per CTA tile
constexpr int kBN = 64;        // output columns per CTA tile
constexpr int kBK = 16;        // K rows per pipeline chunk
#ifndef HMXG_STAGES
#define HMXG_STAGES 4
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
constexpr int kStageBytes = kChunkBytes + kBTileBytes;
constexpr int kSmemBytes = kStages * kStageBytes + 2 * kStages * 8 + 4 * 8 + 16 + 1024;  // + barriers, tile ring, align slack

struct GemmParams {
  const double* tiles;          // pre-tiled A chunks
  const Task* tasks;            // first task of the phase
  const SegDev* segs;
  double* buf[kNumBufs];        // Wp, T, S, Yp
  std::uint64_t ld[kNumBufs];
  std::uint32_t q;
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
__device__ __forceinline__ void mbar_wait(std::uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n"
      "@!done bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
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

// ---------------------------------------------------------------- A pre-tiling
__global__ void tile_a(const double* __restrict__ gd, const double* __restrict__ gb, const double* __restrict__ gv,
                       const TileSrc* __restrict__ srcs, const std::uint32_t* __restrict__ chunk_seg,
                       double* __restrict__ tiles, std::uint64_t nchunks) {
  for (std::uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const TileSrc s = srcs[chunk_seg[c]];
    const std::uint64_t chunk_in_seg = (c * kChunkElems - s.tile_off) / kChunkElems;
    const double* a = (s.gen == kGenD ? gd : (s.gen == kGenB ? gb : gv)) + s.a_off;
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
      if (r < s.m && kk < s.k)
        v = s.trans ? a[kk + static_cast<std::uint64_t>(r) * s.lda] : a[r + kk * s.lda];
      out[a_swz(k, r)] = v;
    }
  }
}

// One tile's K loop for a consumer warp: LI x LJ live 8 x 8 fragments (compile time).
// Fragments of k step ks+1 are loaded while step ks multiplies (register double buffer).
template <int LI, int LJ>
__device__ __forceinline__ void consume_chunks(double (&acc)[4][4][2], std::uint64_t* full, std::uint64_t* empty,
                                               std::uint32_t smem_base, const std::uint32_t (&a_off)[4][4],
                                               const std::uint32_t (&b_off)[4][4], std::uint32_t nchunks,
                                               std::uint32_t& it) {
  for (std::uint32_t c = 0; c < nchunks; ++c, ++it) {
    const int stage = it % kStages;
    mbar_wait(&full[stage], (it / kStages) & 1);
    const std::uint32_t st = smem_base + stage * kStageBytes;
    if (LI > 0 && LJ > 0) {
      double af[2][4], bf[2][4];
#pragma unroll
      for (int i = 0; i < LI; ++i) af[0][i] = lds64(st + a_off[0][i]);
#pragma unroll
      for (int j = 0; j < LJ; ++j) bf[0][j] = lds64(st + b_off[0][j]);
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int cur = ks & 1;
        if (ks + 1 < 4) {
#pragma unroll
          for (int i = 0; i < LI; ++i) af[cur ^ 1][i] = lds64(st + a_off[ks + 1][i]);
#pragma unroll
          for (int j = 0; j < LJ; ++j) bf[cur ^ 1][j] = lds64(st + b_off[ks + 1][j]);
        }
#pragma unroll
        for (int i = 0; i < LI; ++i)
#pragma unroll
          for (int j = 0; j < LJ; ++j) dmma884(acc[i][j], af[cur][i], bf[cur][j]);
      }
    }
    mbar_arrive(&empty[stage]);  // every consumer thread releases the stage after its last read
  }
}

// Partial column block (Q not a multiple of 64): runtime-predicated fragments.
__device__ __forceinline__ void consume_chunks_pred(double (&acc)[4][4][2], std::uint64_t* full, std::uint64_t* empty,
                                                 std::uint32_t smem_base, const std::uint32_t (&a_off)[4][4],
                                                 const std::uint32_t (&b_off)[4][4], std::uint32_t nchunks,
                                                 std::uint32_t& it, int live_i, int live_j) {
  for (std::uint32_t c = 0; c < nchunks; ++c, ++it) {
    const int stage = it % kStages;
    mbar_wait(&full[stage], (it / kStages) & 1);
    const std::uint32_t st = smem_base + stage * kStageBytes;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = i < live_i ? lds64(st + a_off[ks][i]) : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = j < live_j ? lds64(st + b_off[ks][j]) : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (i < live_i && j < live_j) dmma884(acc[i][j], af[i], bf[j]);
    }
    mbar_arrive(&empty[stage]);
  }
}

// ---------------------------------------------------------------- grouped GEMM
// Persistent: gridDim.x = resident CTAs (SMs x occupancy). The producer lane claims output
// tiles from a per-launch atomic counter in raster order (column block fastest, so a row
// tile's A chunks are fetched from HBM once and re-served from L2 to every column block),
// posts each tile id to a 2-slot ring for the consumers, and keeps streaming chunks across
// tile boundaries: the next tile's first chunks land while the consumers run the
// current tile's epilogue. Barrier setup happens once per CTA, not once per tile.
constexpr int kTileRing = 2;

__global__ void __launch_bounds__(kThreads, (HMXG_STAGES <= 4 ? 3 : 2))
grouped_gemm(const __grid_constant__ CUtensorMap tm_wp, const __grid_constant__ CUtensorMap tm_t,
             const __grid_constant__ CUtensorMap tm_s, const GemmParams p, std::uint32_t ntasks,
             std::uint32_t* __restrict__ tile_counter) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<std::uintptr_t>(smem_raw) + 1023) &
                                                         ~std::uintptr_t(1023));
  std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kStages * kStageBytes);
  std::uint64_t* empty = full + kStages;
  std::uint64_t* tfull = empty + kStages;
  std::uint64_t* tempty = tfull + kTileRing;
  std::uint32_t* tring = reinterpret_cast<std::uint32_t*>(tempty + kTileRing);

  const std::uint32_t col_blocks = (p.q + kBN - 1) / kBN;
  const std::uint32_t ntiles = ntasks * col_blocks;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps * 32);
    }
    for (int s = 0; s < kTileRing; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kConsumerWarps * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    // ---------------- producer: one lane claims tiles and streams their chunk sequences
    if (lane == 0) {
      std::uint32_t it = 0;  // chunk counter across tiles (stage ring position)
      for (std::uint32_t seq = 0;; ++seq) {
        const std::uint32_t t = atomicAdd(tile_counter, 1u);
        const int slot = seq % kTileRing;
        if (seq >= kTileRing) mbar_wait(&tempty[slot], ((seq / kTileRing) - 1) & 1);
        tring[slot] = t;
        mbar_arrive(&tfull[slot]);  // release: the consumers read tring[slot] after the wait
        if (t >= ntiles) break;
        const Task task = p.tasks[t / col_blocks];
        const std::uint32_t c0 = (t % col_blocks) * kBN;
        for (std::uint32_t si = task.seg_begin; si < task.seg_end; ++si) {
          const SegDev sg = p.segs[si];
          const CUtensorMap* map = sg.bbuf == kBufWp ? &tm_wp : (sg.bbuf == kBufT ? &tm_t : &tm_s);
          for (std::uint32_t ch = 0; ch < sg.nchunks; ++ch, ++it) {
            const int stage = it % kStages;
            if (it >= kStages) mbar_wait(&empty[stage], ((it / kStages) - 1) & 1);
            unsigned char* st = smem + stage * kStageBytes;
            mbar_expect_tx(&full[stage], kStageBytes);
            bulk_g2s(st, p.tiles + sg.tile_off + static_cast<std::uint64_t>(ch) * kChunkElems, kChunkBytes,
                     &full[stage]);
            // coordinates: {column (inner, Q-contiguous), row}
            tma_2d_g2s(st + kChunkBytes, map, static_cast<int>(c0), static_cast<int>(sg.b_row + ch * kBK),
                       &full[stage]);
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers: 2 x 2 warps, interleaved 8 x 8 fragments
  const int wm = warp & 1, wn = warp >> 1;
  const int fr = lane >> 2, fk = lane & 3;
  // Fragment addresses (shared window, bytes) relative to the stage base. A: swizzled
  // 64 x 16 chunk; B: the 16 x kBPitch row-major TMA tile. Fragment i of warp (wm, wn)
  // covers rows 8*(2i+wm) .. +7 and fragment j columns 8*(2j+wn) .. +7: interleaving
  // spreads a ragged tile's live fragments evenly over the four warps.
  std::uint32_t a_off[4][4], b_off[4][4];  // [k step][fragment]
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const int k = ks * 4 + fk;
#pragma unroll
    for (int i = 0; i < 4; ++i) a_off[ks][i] = 8u * a_swz(k, (2 * i + wm) * 8 + fr);
#pragma unroll
    for (int j = 0; j < 4; ++j) b_off[ks][j] = kChunkBytes + (k * kBPitch + (2 * j + wn) * 8 + fr) * 8;
  }
  const std::uint32_t smem_base = smem_u32(smem);
  std::uint32_t it = 0;
  for (std::uint32_t seq = 0;; ++seq) {
    const int slot = seq % kTileRing;
    mbar_wait(&tfull[slot], (seq / kTileRing) & 1);
    const std::uint32_t t = tring[slot];
    mbar_arrive(&tempty[slot]);
    if (t >= ntiles) break;
    const Task task = p.tasks[t / col_blocks];
    const std::uint32_t c0 = (t % col_blocks) * kBN;
    std::uint32_t nchunks = 0;
    for (std::uint32_t si = task.seg_begin; si < task.seg_end; ++si) nchunks += p.segs[si].nchunks;
    // Warp-uniform trim of fragments outside the task's valid rows / the last column
    // block: their DMMAs are skipped.
    const std::uint32_t ncols = min(static_cast<std::uint32_t>(kBN), p.q - c0);
    const int frag_rows = (static_cast<int>(task.m) + 7) / 8, frag_cols = (static_cast<int>(ncols) + 7) / 8;
    const int live_i = min(4, max(0, (frag_rows - wm + 1) / 2));
    const int live_j = min(4, max(0, (frag_cols - wn + 1) / 2));

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // Predicated-off DMMAs still occupy the tensor pipe, so ragged tiles branch (warp-
    // uniformly, once per tile) to a K loop instantiated for their live fragment count.
    if (live_j == 4) {
      switch (live_i) {
        case 4: consume_chunks<4, 4>(acc, full, empty, smem_base, a_off, b_off, nchunks, it); break;
        case 3: consume_chunks<3, 4>(acc, full, empty, smem_base, a_off, b_off, nchunks, it); break;
        case 2: consume_chunks<2, 4>(acc, full, empty, smem_base, a_off, b_off, nchunks, it); break;
        case 1: consume_chunks<1, 4>(acc, full, empty, smem_base, a_off, b_off, nchunks, it); break;
        default: consume_chunks<0, 0>(acc, full, empty, smem_base, a_off, b_off, nchunks, it); break;
      }
    } else {
      consume_chunks_pred(acc, full, empty, smem_base, a_off, b_off, nchunks, it, live_i, live_j);
    }

    // epilogue: every valid element of the tile is stored exactly once (zeros for empty tasks)
    double* C = pick_buf(p, task.cbuf);
    const std::uint64_t ldc = pick_ld(p, task.cbuf);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int row = (2 * i + wm) * 8 + fr;
      if (row >= task.m) continue;
      double* crow = C + static_cast<std::uint64_t>(task.c_row + row) * ldc + c0;  // row major, Q contiguous
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
}

// Transpose-permute into the point-major internal layout: Wp[ipmap[r], c] = W[r, c].
// A 32 x 32 tile is read column by column (256 B contiguous per column of W), turned
// around in shared memory and written row by row (256 B contiguous per point row of Wp),
// so both sides move whole cache lines although the rows land in permuted order.
constexpr int kTT = 32;
__global__ void __launch_bounds__(256) permute_in(const double* __restrict__ w, std::uint64_t ldw,
                                                  const std::uint32_t* __restrict__ ipmap, double* __restrict__ wp,
                                                  std::uint64_t ldwp, std::uint32_t n, std::uint32_t q) {
  __shared__ double tile[kTT][kTT + 1];
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
    if (r < n && c < q) wp[static_cast<std::uint64_t>(ipmap[r]) * ldwp + c] = tile[tx][ty + k];
  }
}

// Inverse: Y[r, c] = Yp[ipmap[r], c] (point rows read whole, columns of Y written whole).
__global__ void __launch_bounds__(256) permute_out(const double* __restrict__ yp, std::uint64_t ldyp,
                                                   const std::uint32_t* __restrict__ ipmap, double* __restrict__ y,
                                                   std::uint64_t ldy, std::uint32_t n, std::uint32_t q) {
  __shared__ double tile[kTT][kTT + 1];
  const std::uint32_t r0 = blockIdx.x * kTT, c0 = blockIdx.y * kTT;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kTT; k += 8) {
    const std::uint32_t r = r0 + ty + k, c = c0 + tx;
    tile[ty + k][tx] = (r < n && c < q) ? __ldg(yp + static_cast<std::uint64_t>(ipmap[r]) * ldyp + c) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kTT; k += 8) {
    const std::uint32_t r = r0 + tx, c = c0 + ty + k;
    if (r < n && c < q) y[r + static_cast<std::uint64_t>(c) * ldy] = tile[tx][ty + k];
  }
}

}  // namespace hmxg
