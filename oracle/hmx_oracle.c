/*
 * hmx_oracle.c — CPU restatement of the reference evaluation phase.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker for the B200 evaluator;
 * it is never linked into, loaded by, or called from the product path
 * (paper_1812_07152_b200/). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it.
 *
 * Parity pin: built with the reference's Release flags (no FMA contraction, no
 * reassociation) this restatement reproduces hmx::evaluate(cds, plan{p=1}, w) BIT FOR
 * BIT on every instance checked (tests/test_oracle.py, against oracle/_ref built from
 * /root/reference/proj/src and against the committed fixtures in tests/golden/).
 *
 * Semantics follow /root/reference/proj/src/executor.cpp:
 *   EvalRun ctor        :32-47   gather Wp = W[perm], zero T/S for active nodes
 *   upward_node/pass    :51-72, :139-163
 *   far_pair/far_pass   :105-110, :229-235 (flat order == blocked order per target)
 *   downward_node/pass  :74-103, :165-190
 *   near_pair/near_pass :112-117, :237-243
 *   scatter             :245-254
 * and the two dense kernels of /root/reference/proj/src/dense.cpp:13-66, whose exact
 * summation order (Kc=256 K-blocks, 4-way grouped rank-1 updates, 2-accumulator dot
 * products) is restated below so that the rounding matches.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/hmxg.h"

#define ORC_KC 256

/* C(m x n) += A(m x k) B(k x n), column major — dense.cpp:13-43. Within each K block of
 * 256, products are grouped four at a time, the group summed left to right and then
 * added to C; the M blocking of the reference does not change any value. */
static void orc_gemm_acc(size_t m, size_t n, size_t k, const double* a, size_t lda,
                         const double* b, size_t ldb, double* c, size_t ldc) {
  for (size_t k0 = 0; k0 < k; k0 += ORC_KC) {
    const size_t kb = (k - k0 < ORC_KC) ? k - k0 : ORC_KC;
    for (size_t j = 0; j < n; ++j) {
      const double* bcol = b + j * ldb + k0;
      double* ccol = c + j * ldc;
      size_t p = 0;
      for (; p + 4 <= kb; p += 4) {
        const double* x0 = a + (k0 + p) * lda;
        const double* x1 = x0 + lda;
        const double* x2 = x1 + lda;
        const double* x3 = x2 + lda;
        const double w0 = bcol[p], w1 = bcol[p + 1], w2 = bcol[p + 2], w3 = bcol[p + 3];
        for (size_t i = 0; i < m; ++i) {
          const double grp = x0[i] * w0 + x1[i] * w1 + x2[i] * w2 + x3[i] * w3;
          ccol[i] += grp;
        }
      }
      for (; p < kb; ++p) {
        const double* x = a + (k0 + p) * lda;
        const double w = bcol[p];
        for (size_t i = 0; i < m; ++i) ccol[i] += x[i] * w;
      }
    }
  }
}

/* C(m x n) += A^T B with A (k x m) column major — dense.cpp:45-66: even and odd terms
 * of each dot product go to separate accumulators, a tail term to the even one. */
static void orc_gemm_trans_acc(size_t m, size_t n, size_t k, const double* a, size_t lda,
                               const double* b, size_t ldb, double* c, size_t ldc) {
  for (size_t j = 0; j < n; ++j) {
    const double* bcol = b + j * ldb;
    double* ccol = c + j * ldc;
    for (size_t i = 0; i < m; ++i) {
      const double* acol = a + i * lda;
      double even = 0.0, odd = 0.0;
      size_t p = 0;
      for (; p + 2 <= k; p += 2) {
        even += acol[p] * bcol[p];
        odd += acol[p + 1] * bcol[p + 1];
      }
      if (p < k) even += acol[p] * bcol[p];
      ccol[i] += even + odd;
    }
  }
}

typedef struct {
  const hmxg_cds_view* v;
  size_t n, q;
  double* wp;
  double* yp;
  double** t;        /* per node, sr x q or NULL */
  double** s;
  uint64_t* vslot;   /* node -> V slot, UINT64_MAX when absent */
} orc_run;

static int orc_active(const orc_run* r, uint32_t i) {
  return r->v->participating[i] && r->v->sranks[i] > 0;
}

static int orc_is_leaf(const hmxg_cds_view* v, uint32_t i) { return v->lchild[i] == HMXG_NO_NODE; }

static const double* orc_vgen(const orc_run* r, uint32_t node) {
  return r->v->vgen + r->v->vptr[r->vslot[node]];
}

/* executor.cpp:51-72 */
static void orc_upward_node(orc_run* r, uint32_t i) {
  const hmxg_cds_view* v = r->v;
  if (!orc_active(r, i)) return;
  const uint32_t sr = v->sranks[i];
  const double* vb = orc_vgen(r, i);
  if (orc_is_leaf(v, i)) {
    const size_t sz = v->end[i] - v->start[i];
    orc_gemm_trans_acc(sr, r->q, sz, vb, sz, r->wp + v->start[i], r->n, r->t[i], sr);
    return;
  }
  const uint32_t lc = v->lchild[i], rc = v->rchild[i];
  const size_t srl = v->sranks[lc], srr = v->sranks[rc], width = srl + srr;
  double* scratch = (double*)calloc(width * r->q + 1, sizeof(double));
  for (size_t c = 0; c < r->q; ++c) {
    if (srl) memcpy(scratch + c * width, r->t[lc] + c * srl, srl * sizeof(double));
    if (srr) memcpy(scratch + c * width + srl, r->t[rc] + c * srr, srr * sizeof(double));
  }
  orc_gemm_trans_acc(sr, r->q, width, vb, width, scratch, width, r->t[i], sr);
  free(scratch);
}

/* executor.cpp:74-103 */
static void orc_downward_node(orc_run* r, uint32_t i) {
  const hmxg_cds_view* v = r->v;
  if (!orc_active(r, i)) return;
  const uint32_t sr = v->sranks[i];
  const double* vb = orc_vgen(r, i);
  if (orc_is_leaf(v, i)) {
    const size_t sz = v->end[i] - v->start[i];
    orc_gemm_acc(sz, r->q, sr, vb, sz, r->s[i], sr, r->yp + v->start[i], r->n);
    return;
  }
  const uint32_t lc = v->lchild[i], rc = v->rchild[i];
  const size_t srl = v->sranks[lc], srr = v->sranks[rc], width = srl + srr;
  if (width == 0) return;
  double* scratch = (double*)calloc(width * r->q, sizeof(double));
  orc_gemm_acc(width, r->q, sr, vb, width, r->s[i], sr, scratch, width);
  for (size_t c = 0; c < r->q; ++c) {
    const double* src = scratch + c * width;
    if (srl) {
      double* dst = r->s[lc] + c * srl;
      for (size_t k = 0; k < srl; ++k) dst[k] += src[k];
    }
    if (srr) {
      double* dst = r->s[rc] + c * srr;
      for (size_t k = 0; k < srr; ++k) dst[k] += src[srl + k];
    }
  }
  free(scratch);
}

/*
 * Y = K~ W for the CDS in `v`; W (n x q, ldw), Y (n x q, ldy), column major.
 * Returns 0, or 1 on a shape mismatch / malformed view (executor.cpp:277-278),
 * or 3 on allocation failure. q == 0 is a no-op (executor.cpp:279-282).
 */
int hmxo_evaluate(const hmxg_cds_view* v, const double* w, size_t n, size_t q, size_t ldw,
                  double* y, size_t ldy) {
  if (!v || n != v->n || ldw < n || ldy < n) return 1;
  if (q == 0) return 0;
  const uint32_t nn = v->num_nodes;
  orc_run r;
  memset(&r, 0, sizeof r);
  r.v = v;
  r.n = n;
  r.q = q;
  r.wp = (double*)malloc(n * q * sizeof(double));
  r.yp = (double*)calloc(n * q, sizeof(double));
  r.t = (double**)calloc(nn, sizeof(double*));
  r.s = (double**)calloc(nn, sizeof(double*));
  r.vslot = (uint64_t*)malloc(nn * sizeof(uint64_t));
  if (!r.wp || !r.yp || !r.t || !r.s || !r.vslot) return 3;
  for (uint32_t i = 0; i < nn; ++i) r.vslot[i] = UINT64_MAX;
  for (uint64_t s = 0; s < v->num_v; ++s) r.vslot[v->v_order[s]] = s;

  /* EvalRun ctor, executor.cpp:32-47 */
  for (size_t c = 0; c < q; ++c)
    for (size_t pos = 0; pos < n; ++pos) r.wp[c * n + pos] = w[c * ldw + v->perm[pos]];
  for (uint32_t i = 0; i < nn; ++i)
    if (orc_active(&r, i)) {
      if (r.vslot[i] == UINT64_MAX) return 1; /* CDS::v_slot throws, structure.cpp:217-221 */
      r.t[i] = (double*)calloc((size_t)v->sranks[i] * q, sizeof(double));
      r.s[i] = (double*)calloc((size_t)v->sranks[i] * q, sizeof(double));
    }

  /* upward: depth descending (executor.cpp:158-162); any children-first order gives the
   * same bits because each T_i is produced by one GEMM */
  for (uint32_t d = v->height + 1; d-- > 0;)
    for (uint32_t i = 0; i < nn; ++i)
      if (v->level[i] == d) orc_upward_node(&r, i);

  /* far: storage order (executor.cpp:105-110, 209-235) */
  for (uint64_t slot = 0; slot < v->num_far; ++slot) {
    const uint32_t i = v->far_pairs[2 * slot], j = v->far_pairs[2 * slot + 1];
    const size_t sri = v->sranks[i], srj = v->sranks[j];
    if (sri == 0 || srj == 0) continue;
    orc_gemm_acc(sri, q, srj, v->bgen + v->bptr[slot], sri, r.t[j], srj, r.s[i], sri);
  }

  /* downward: depth ascending (executor.cpp:185-189) */
  for (uint32_t d = 0; d <= v->height; ++d)
    for (uint32_t i = 0; i < nn; ++i)
      if (v->level[i] == d) orc_downward_node(&r, i);

  /* near: storage order (executor.cpp:112-117) */
  for (uint64_t slot = 0; slot < v->num_near; ++slot) {
    const uint32_t i = v->near_pairs[2 * slot], j = v->near_pairs[2 * slot + 1];
    const size_t szi = v->end[i] - v->start[i], szj = v->end[j] - v->start[j];
    orc_gemm_acc(szi, q, szj, v->dgen + v->dptr[slot], szi, r.wp + v->start[j], n,
                 r.yp + v->start[i], n);
  }

  /* scatter, executor.cpp:245-254 */
  for (size_t c = 0; c < q; ++c)
    for (size_t pos = 0; pos < n; ++pos) y[c * ldy + v->perm[pos]] = r.yp[c * n + pos];

  for (uint32_t i = 0; i < nn; ++i) {
    free(r.t[i]);
    free(r.s[i]);
  }
  free(r.t);
  free(r.s);
  free(r.vslot);
  free(r.wp);
  free(r.yp);
  return 0;
}

/* Algorithmic work of one evaluation column: 2*(2|V| + |B| + |D|). */
double hmxo_flops_per_col(const hmxg_cds_view* v) {
  const double dv = (double)v->vptr[v->num_v], db = (double)v->bptr[v->num_far],
               dd = (double)v->dptr[v->num_near];
  return 2.0 * (2.0 * dv + db + dd);
}
