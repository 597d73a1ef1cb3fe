/*
 * hmxb.h — C-ABI of the host instance builder (libhmxb.so).
 *
 * Produces the evaluator's input: a computation-ordered CDS (hmxg_cds_view) from seeded
 * synthetic points. It covers the reference inspector pipeline
 *   synth_points -> build_cluster_tree -> compute_interactions -> build_samples ->
 *   compress -> blocking x2 -> coarsening -> build_cds
 *   (/root/reference/proj/tests/helpers.hpp:101-118, proj/src/pipeline.cpp:115-215)
 * plus what BASELINE.json's configs need and the reference lacks: budget
 * ("H2-b") admissibility, the exponential kernel, and the Gaussian-mixture,
 * standardized-normal and quantized-uniform point generators.
 * It is this repo's own (multi-threaded) host code; the reference stays the oracle.
 */
#ifndef HMXB_H_
#define HMXB_H_

#include <stdint.h>

#include "hmxg.h"

#ifdef __cplusplus
extern "C" {
#endif

enum hmxb_points_kind {
  HMXB_PTS_UNIFORM = 0,   /* U[0,1]^d (reference synth_points UniformRandom) */
  HMXB_PTS_GRID2D = 1,    /* integer grid, d = 2 (reference Grid2d) */
  HMXB_PTS_MIXTURE = 2,   /* isotropic Gaussian mixture, centres U[-5,5]^d, unit variance */
  HMXB_PTS_NORMAL = 3,    /* N(0,1)^d, every coordinate standardized over the set */
  HMXB_PTS_QUANTIZED = 4  /* U[0,1]^d quantized to `levels` values */
};
enum hmxb_kernel_kind {
  HMXB_K_GAUSSIAN = 0,    /* exp(-|x-y|^2 / (2 h h)), the reference's operation order */
  HMXB_K_EXPONENTIAL = 1, /* exp(-|x-y| / h) */
  HMXB_K_INVDIST = 2      /* 1/|x-y|, 1 on coincident points */
};
enum hmxb_mode { HMXB_HSS = 0, HMXB_TAU = 1, HMXB_BUDGET = 2 };
enum hmxb_split { HMXB_SPLIT_AUTO = 0, HMXB_SPLIT_KD = 1, HMXB_SPLIT_TWOMEANS = 2 };

typedef struct hmxb_spec {
  uint64_t n;
  uint32_t d;
  int32_t points;      /* hmxb_points_kind */
  uint32_t components; /* mixture components (default 8) */
  uint32_t levels;     /* quantization levels (default 16) */
  uint64_t seed;
  int32_t kernel;      /* hmxb_kernel_kind */
  double h;
  uint32_t leaf;       /* leaf size m */
  int32_t split;       /* hmxb_split */
  int32_t mode;        /* hmxb_mode */
  double tau;          /* TAU mode admissibility */
  double budget;       /* BUDGET mode: near fraction of leaf pairs per leaf row */
  uint32_t max_rank;   /* s */
  double tol;          /* compression tolerance (relative Frobenius of the ID residual) */
  uint32_t sample_rows;/* ID sample rows per node (0 -> 2 s); UINT32_MAX -> exact (all rows) */
  uint32_t knn_k;      /* neighbours per point for sampling / budget votes */
  uint32_t near_blocksize, far_blocksize, coarsen_p, coarsen_agg;
  uint32_t threads;    /* 0 -> hardware concurrency */
  uint32_t skip_near;  /* 1: leave dgen empty (dptr still sized): the evaluator generates the
                        * near blocks from the points (hmxg_upload_generated) */
} hmxb_spec;

typedef struct hmxb_build_stats {
  double seconds_points, seconds_tree, seconds_interactions, seconds_sampling,
      seconds_compress, seconds_blocks, seconds_total;
  uint64_t leaves, near_pairs, far_pairs;
  uint32_t max_srank, height;
} hmxb_build_stats;

typedef struct hmxb_instance hmxb_instance;

void hmxb_spec_default(hmxb_spec* spec);
int hmxb_build(const hmxb_spec* spec, hmxb_instance** out);
int hmxb_view(const hmxb_instance* inst, hmxg_cds_view* view);
int hmxb_points(const hmxb_instance* inst, const double** coords, uint64_t* n, uint32_t* d);
int hmxb_stats(const hmxb_instance* inst, hmxb_build_stats* stats);
/* Exact kernel rows: out[r + c*ldo] = sum_j K(x_rows[r], x_j) W[j, c] (dense oracle rows,
 * reference dense_apply / relative_error_vs sampled mode, executor.cpp:405-476). */
int hmxb_dense_rows(const hmxb_instance* inst, const uint32_t* rows, uint64_t nrows,
                    const double* W, uint64_t q, uint64_t ldw, double* out, uint64_t ldo);
void hmxb_free(hmxb_instance* inst);
/* The reference CLI's random right-hand side (proj/tools/hmx.cpp:117-122): uniform[-1, 1)
 * from xoshiro256** seeded with splitmix64(seed ^ splitmix64(0x77a7)), column major. */
void hmxb_random_w(uint64_t seed, uint64_t n, uint64_t q, double* out);
const char* hmxb_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* HMXB_H_ */
