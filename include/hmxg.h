/*
 * hmxg.h — C-ABI of the B200 HMatrix x W evaluator (libhmxg.so).
 *
 * Drop-in boundary for the reference's evaluation phase
 *   hmx::evaluate(const CDS&, const EvalPlan&, const DenseMatrix& w, [WorkerPool&,] EvalStats*)
 *   (/root/reference/proj/include/hmx/executor.hpp:51-54,
 *    /root/reference/proj/src/executor.cpp:274-302).
 * The caller keeps building the tree / interactions / compression / CDS on the host
 * (reference inspector, or this repo's instance builder) and hands the CDS over as a
 * POD view of raw arrays; nothing here knows about torch or C++ types.
 *
 * Status codes: 0 ok, 1 invalid argument, 2 CUDA error, 3 out of memory,
 * 4 NCCL/collective error, 5 file I/O or format error (reference exit code 3, io_error). A thread-local message is kept for hmxg_last_error().
 */
#ifndef HMXG_H_
#define HMXG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HMXG_OK 0
#define HMXG_EINVAL 1
#define HMXG_ECUDA 2
#define HMXG_ENOMEM 3
#define HMXG_ECOMM 4
#define HMXG_EIO 5
#define HMXG_EGUARD 6 /* hmx::numeric_guard_error (dense error oracle beyond n = 16384) */

#define HMXG_NO_NODE 0xffffffffu

/* hmxg_evaluate flags */
#define HMXG_F_DEVICE_PTRS 0x1u /* W and Y are device pointers on the matrix's (single) device */
#define HMXG_F_NO_SYNC 0x2u     /* with DEVICE_PTRS: enqueue on `stream` and return */
#define HMXG_F_NO_GRAPH 0x8u    /* with DEVICE_PTRS: issue the launches instead of replaying the
                                   cached CUDA graph of the launch sequence (the graph is keyed
                                   on W, Y, q, leading dimensions, a non-NULL stream and
                                   HMXG_F_TIME_PHASES) */
#define HMXG_F_LEVEL_LAUNCHES 0x10u /* run the level-by-level launch sequence (one launch per
                                       tree level) instead of the single whole-evaluation DAG
                                       launch: same results, per-launch timing breakdown */
#define HMXG_F_TIME_PHASES 0x4u /* record a CUDA event pair around every launch (device 0; a
                                   graph captured with it keeps them as event nodes);
                                   read back with hmxg_phase_get. Without it, eval_dag and
                                   permute-out are programmatic dependent launches (their
                                   launch overlaps the preceding kernel) */

/*
 * View of a computation-ordered CDS (reference struct hmx::CDS,
 * /root/reference/proj/include/hmx/structure.hpp:83-130). All arrays are borrowed for
 * the duration of hmxg_upload only.
 *   tree arrays            : num_nodes entries (ClusterTree, tree.hpp:19-33), kNoNode = HMXG_NO_NODE
 *   perm                   : n entries, node i owns perm[start[i], end[i])
 *   near_pairs / far_pairs : 2*num_near / 2*num_far (i,j) in storage order
 *                            (= BlockSet::flat_pairs(), structure.cpp:21-27)
 *   v_order                : num_v node ids in V storage order (coarsenset traversal,
 *                            structure.cpp:197-202)
 *   dptr / bptr / vptr     : num_near+1 / num_far+1 / num_v+1 element offsets
 *   dgen / bgen / vgen     : FP64 generators, column major: D_ij m_i x m_j, B_ij sr_i x sr_j,
 *                            V_i v_width(i) x sr_i (v_width = leaf size or sr_lc + sr_rc).
 */
typedef struct hmxg_cds_view {
  uint64_t n;
  uint32_t num_nodes;
  uint32_t height;
  const uint32_t* parent;
  const uint32_t* lchild;
  const uint32_t* rchild;
  const uint32_t* start;
  const uint32_t* end;
  const uint32_t* level;
  const uint32_t* perm;
  const uint32_t* sranks;
  const uint8_t* participating;
  uint64_t num_near;
  const uint32_t* near_pairs;
  uint64_t num_far;
  const uint32_t* far_pairs;
  uint64_t num_v;
  const uint32_t* v_order;
  const uint64_t* dptr;
  const uint64_t* bptr;
  const uint64_t* vptr;
  const double* dgen;
  const double* bgen;
  const double* vgen;
} hmxg_cds_view;

/* EvalStats (executor.hpp:43-46) plus device-side accounting. */
typedef struct hmxg_stats {
  uint64_t locked_pairs; /* always 0: every output tile has one writer */
  double seconds;        /* host wall time of the call (reference semantics) */
  double device_ms;      /* device time of the evaluation launches (max over devices) */
  uint32_t launches;     /* kernel launches issued by this call (all devices) */
} hmxg_stats;

/* Static description of an uploaded matrix (roofline accounting). */
typedef struct hmxg_info {
  uint64_t n;
  uint64_t d_elems, b_elems, v_elems; /* |Dgen|, |Bgen|, |Vgen| */
  uint64_t skel_rows;                 /* sum of active sranks (T/S rows) */
  uint32_t num_devices;
  uint32_t launches_per_eval;         /* kernels per evaluate call per device (3: permute-in,
                                         the whole-evaluation DAG launch, permute-out) */
  double flops_per_col;               /* 2*(2|V|+|B|+|D|), the reference's count */
  uint64_t device_bytes;              /* resident generator + table bytes per device */
  double exec_flops_per_col;          /* flops the kernels execute per column (the bases'
                                         identity rows become row copies) */
  uint32_t split_parts;               /* 1: the CDS is replicated on this device; P > 1: this
                                         device holds one of P subtree parts (hmxg_create_comm
                                         contexts whose CDS exceeds the HBM budget, or
                                         hmxg_upload_split), and evaluation is collective */
  uint32_t part;                      /* the part this device holds */
} hmxg_info;

/* One launch of the per-evaluation launch sequence (SURVEY §7.3 / DESIGN.md):
 * kind 0 gather, 1 upward (level = subtree height), 2 far+downward (level = depth),
 * 3 near+leaf-downward (level = wave with HMXG_UPLOAD_NEAR_ON_THE_FLY), 4 scatter, 5 the
 * whole-evaluation DAG launch (every GEMM tile of every level; the default sequence is
 * gather, DAG, scatter), 6 near field alone (the split leaf variant of narrow column counts),
 * 7 near blocks generated into the scratch (on the fly; level = wave). Byte/flop fields are ALGORITHMIC (each operand block
 * counted once): the roofline numerators of bench.py. last_ms is the device time of that
 * launch in the last evaluation run with HMXG_F_TIME_PHASES on device 0. */
typedef struct hmxg_phase {
  uint32_t kind;
  uint32_t level;
  uint32_t tiles;            /* row tiles (grid.x); grid.y = ceil(q / 64) */
  uint32_t reserved;
  double flops_per_col;
  double gen_bytes;          /* generator bytes read once per evaluation */
  double io_bytes_per_col;   /* operand rows read + output rows written, per column */
  double last_ms;
} hmxg_phase;

typedef struct hmxg_ctx hmxg_ctx;
typedef struct hmxg_mat hmxg_mat;

/* Context over `ndev` CUDA devices (devs may repeat a device id: each entry is one
 * column shard). ndev = 0 / devs = NULL means {0}. */
int hmxg_create(const int* devs, int ndev, hmxg_ctx** out);

/* ---- One process per GPU. The caller provides the collective:
 * allgatherv(user, sendbuf, sendbytes, recvbuf, recvbytes[size], displs[size], stream):
 * every rank contributes sendbytes bytes and receives rank r's block at recvbuf + displs[r]
 * (recvbytes[r] bytes). The library always calls it in place (sendbuf == recvbuf +
 * displs[rank]) on contiguous blocks in rank order. Buffers are device pointers ordered on
 * `stream` (a cudaStream_t; e.g. ncclGroupStart + one ncclBroadcast per rank), or host
 * memory with a NULL stream when host_buffers != 0 (the library stages; e.g. MPI, gloo).
 * A non-zero return is reported as HMXG_ECOMM.
 * hbm_budget: device bytes the resident CDS may use (0: 3/4 of the device's memory). While
 * the CDS fits, hmxg_upload replicates it and every rank evaluates its own columns with no
 * communication. When it does not, hmxg_upload holds only the rank's subtree part (the
 * subtree-split fallback, hmxg_info.split_parts = size) and hmxg_evaluate becomes
 * collective: every rank passes the same full W and receives the full Y; inside, the parts
 * all-gather the skeleton weights T other parts read (children of the replicated top levels
 * and far partners) and then their rows of the result. (Replaces the reference's in-process
 * WorkerPool fork-join, /root/reference/proj/include/hmx/parallel.hpp:19-114, at process
 * scale; the reference itself has no multi-process evaluation.) */
typedef int (*hmxg_allgatherv_fn)(void* user, const void* sendbuf, size_t sendbytes, void* recvbuf,
                                  const size_t* recvbytes, const size_t* displs, void* stream);
typedef struct hmxg_comm {
  uint32_t rank;
  uint32_t size;
  hmxg_allgatherv_fn allgatherv;
  void* user;
  int32_t host_buffers;
  uint32_t reserved;
  uint64_t hbm_budget;
} hmxg_comm;
int hmxg_create_comm(int dev, const hmxg_comm* comm, hmxg_ctx** out);
int hmxg_destroy(hmxg_ctx* ctx);

/* Validate the view, derive the level-batched task tables and copy the generators to
 * every device of the context (replicated CDS). */
int hmxg_upload(hmxg_ctx* ctx, const hmxg_cds_view* cds, hmxg_mat** out);
int hmxg_free(hmxg_mat* mat);
/* Host-only check of a view (no device needed): the structural invariants hmxg_upload
 * enforces. Returns HMXG_OK or HMXG_EINVAL with the reason in hmxg_last_error(). On
 * success, if info != NULL, the size fields (n, *_elems, skel_rows, launches_per_eval,
 * flops_per_col) are filled. */
int hmxg_validate(const hmxg_cds_view* cds, hmxg_info* info);
/* Content fingerprint of a view (host only, no device needed): a 64-bit hash of every
 * structure array and every generator element, one multi-threaded pass at host memory
 * bandwidth. The drop-in hmx_gpu::evaluate / Python evaluate() key their resident upload on
 * it, so an edited or reallocated CDS is never evaluated from a stale upload (the reference
 * evaluate, executor.cpp:274-302, reads the CDS on every call). */
int hmxg_cds_fingerprint(const hmxg_cds_view* cds, uint64_t* out);
/* Host-only check of the whole-evaluation DAG launch for q columns and a grid of `grid`
 * resident CTAs (no device needed): the claim order holds every task tile of the leaf
 * variant that runs exactly once, every tile an item waits for (B operand rows, identity
 * rows, the split leaf tasks' near rows) comes before it, and the completion targets equal
 * the writer tile counts. These are what eval_dag's deadlock freedom rests on. */
int hmxg_dag_check(const hmxg_cds_view* cds, size_t q, uint32_t grid, uint64_t* nitems);
/* The claim order itself (host only, diagnostics and tests): up to `cap` work-item words into
 * `items` (task index in bits 0-31, column block in bits 32-47, column-split part in 48-55),
 * the total count into *nitems. */
int hmxg_dag_items(const hmxg_cds_view* cds, size_t q, uint32_t grid, uint64_t* items, size_t cap, uint64_t* nitems);
int hmxg_info_get(const hmxg_mat* mat, hmxg_info* info);

/* Subtree-split fallback for a CDS larger than one GPU's HBM. Part `part` of
 * `nparts` (one single-device context per part, e.g. one rank per GPU) owns the subtrees
 * below the top ceil(log2 nparts) tree levels assigned to it and holds only the
 * generators its tiles read; W and Y are full-size on every part. Evaluation is two
 * stages around an exchange of the skeleton weights T:
 *   hmxg_split_stage(mat, 0, ...)  permute-in + upward pass over the part's subtrees
 *   -- sum the parts' T buffers (hmxg_split_exchange_buffer; e.g. ncclAllReduce, sum) --
 *   hmxg_split_stage(mat, 1, ...)  replicated top levels, far+downward and near/leaf for
 *                                  the part's targets, permute-out
 *   -- sum the parts' Y (rows of other parts are zero) --
 * W / Y are device pointers on the part's device; each call returns when its stage is
 * complete on `stream` (NULL = internal stream). */
int hmxg_upload_split(hmxg_ctx* ctx, const hmxg_cds_view* cds, uint32_t nparts, uint32_t part, hmxg_mat** out);
int hmxg_split_stage(hmxg_mat* mat, int stage, const double* W, size_t n, size_t q, size_t ldw, double* Y,
                     size_t ldy, void* stream);
int hmxg_split_exchange_buffer(hmxg_mat* mat, double** ptr, size_t* count);
/* Copy the T exchange buffer (count = skel rows x row pitch doubles, see _buffer) to a
 * device buffer (to_matrix = 0) or back into the matrix (to_matrix = 1). */
int hmxg_split_exchange(hmxg_mat* mat, double* buf, size_t count, int to_matrix, void* stream);

/* Y = K~ W. W is n x q column major with leading dimension ldw >= n, Y likewise.
 * Host pointers (default): columns are sharded over the context's devices, copied in,
 * evaluated and copied back; returns when Y is complete.
 * HMXG_F_DEVICE_PTRS: W/Y live on the matrix's device (single-device contexts only);
 * `stream` (cudaStream_t, may be NULL = internal stream) orders the work.
 * q == 0 is a no-op (Y is n x 0); a row mismatch (n != cds.n) is HMXG_EINVAL. */
int hmxg_evaluate(hmxg_mat* mat, const double* W, size_t n, size_t q, size_t ldw, double* Y,
                  size_t ldy, unsigned flags, void* stream, hmxg_stats* stats);

/* Upload with the kernel blocks generated on the device: cds.dgen is
 * ignored (it may be NULL; dptr must still size every block) and every near block is
 * evaluated from the points instead, D_ij(a, b) = K(x_{perm[start_i+a]}, x_{perm[start_j+b]})
 * (compress.cpp:143-147), with the kernels of hmxg_points_upload. coords: n x d, point
 * major, original point order (hmx::PointSet::coords). The host never forms or ships D.
 * With skel_ptr (num_nodes + 1 CSR offsets into skel_idx: every node's skeleton point
 * indices, srank of them, e.g. from hmxg_compress) the far blocks are generated as well,
 * B_ij = K(skeleton_i, skeleton_j) (compress.cpp:139-142), and cds.bgen is ignored. */
int hmxg_upload_generated(hmxg_ctx* ctx, const hmxg_cds_view* cds, const double* coords, uint32_t d, int32_t kernel,
                          double h, const uint64_t* skel_ptr, const uint32_t* skel_idx, hmxg_mat** out);

/* hmxg_upload_generated with flags. HMXG_UPLOAD_NEAR_ON_THE_FLY: the near blocks are never
 * resident. Every evaluation generates them from the points into a bounded scratch region of
 * the tiles (HMXG_NEAR_SCRATCH_MB, default 2048), wave by wave: the leaf rows run in waves of
 * leaf tasks whose near blocks fit it, each right after its blocks are generated. The
 * resident CDS drops by |D| (cfg5 H2-b: 18.6 GB) for one generation of every near element
 * per evaluation (its FP64 cost is ~Q/50 of the D products it feeds). Results are
 * bit-identical to hmxg_upload_generated. Single device per context entry; no split. */
#define HMXG_UPLOAD_NEAR_ON_THE_FLY 1u
int hmxg_upload_generated_ex(hmxg_ctx* ctx, const hmxg_cds_view* cds, const double* coords, uint32_t d,
                             int32_t kernel, double h, const uint64_t* skel_ptr, const uint32_t* skel_idx,
                             unsigned flags, hmxg_mat** out);

/* Launch sequence description; phase_get synchronizes the timing events of the last
 * HMXG_F_TIME_PHASES evaluation before filling last_ms. */
int hmxg_phase_count(const hmxg_mat* mat);
int hmxg_phase_get(hmxg_mat* mat, uint32_t idx, hmxg_phase* out);

/* The reference's on-disk CDS (`hmat.cds`, format CDS1 v1, written by `hmx inspect` /
 * hmx::save_cds: /root/reference/proj/src/serial.cpp:160-211, 271-308). The file is
 * memory-mapped; the view's generator pointers point into the mapping (not necessarily
 * 8-byte aligned), valid until hmxg_cds_file_close. Truncated files, a bad tag or version
 * and inconsistent offsets are refused with HMXG_EIO (hmxg_cds_file_error()). */
typedef struct hmxg_cds_file hmxg_cds_file;
int hmxg_cds_file_open(const char* path, hmxg_cds_file** out);
int hmxg_cds_file_view(const hmxg_cds_file* file, hmxg_cds_view* view);
int hmxg_cds_file_header(const hmxg_cds_file* file, uint32_t* dim, double* bacc, uint32_t* max_rank);
void hmxg_cds_file_close(hmxg_cds_file* file);
const char* hmxg_cds_file_error(void);

/* ---- Exact kernel products: the GPU error oracle.
 * dense_apply (/root/reference/proj/src/executor.cpp:405-429) and relative_error_vs
 * (:431-476) on the device. Points are uploaded once (n x d, point major, as
 * hmx::PointSet::coords); every kernel tile is generated on the fly from them:
 *   gaussian     exp(-|x-y|^2 / (2 h h))       (kernel.cpp:35-45)
 *   invdist      |x-y| == 0 ? 1 : 1/|x-y|      (kernel.cpp:46-47)
 *   exponential  exp(-|x-y| * (1/h))           (the builder's kernel, hmxb.h)
 * and multiplied into W by the evaluator's FP64 DMMA GEMM. */
typedef struct hmxg_points hmxg_points;
#define HMXG_KERNEL_GAUSSIAN 0
#define HMXG_KERNEL_EXPONENTIAL 1
#define HMXG_KERNEL_INVDIST 2
#define HMXG_ERR_DENSE 0
#define HMXG_ERR_SAMPLED 1
int hmxg_points_upload(hmxg_ctx* ctx, const double* coords, uint64_t n, uint32_t d, int32_t kernel, double h,
                       hmxg_points** out);
int hmxg_points_free(hmxg_points* pts);
/* Y[i + c*ldy] = sum_j K(x_{rows[i]}, x_j) W[j + c*ldw] for i < nrows, c < q; rows is a
 * host array, or NULL for every point in order (nrows must then be n: dense_apply).
 * HMXG_F_DEVICE_PTRS: W and Y are device pointers (else host). */
int hmxg_kernel_rows(hmxg_points* pts, const uint32_t* rows, uint64_t nrows, const double* W, size_t n, size_t q,
                     size_t ldw, double* Y, size_t ldy, unsigned flags, void* stream, hmxg_stats* stats);
/* The sampled-mode row choice of relative_error_vs (executor.cpp:446-451): min(n, 256)
 * rows by a partial Fisher-Yates shuffle seeded with mix64(seed ^ mix64(0xe44a11)).
 * Host only; returns the row count written to rows[] (capacity >= min(n, 256)). */
uint64_t hmxg_sample_rows(uint64_t n, uint64_t seed, uint32_t* rows);
/* relative_error_vs: ||Y_approx - K W||_F / ||K W||_F over every entry (HMXG_ERR_DENSE,
 * n <= 16384 else HMXG_EGUARD) or over the sampled rows (HMXG_ERR_SAMPLED). q == 0
 * gives 0. HMXG_F_DEVICE_PTRS: Y_approx and W are device pointers. */
int hmxg_relative_error(hmxg_points* pts, const double* Y_approx, size_t ldya, const double* W, size_t n, size_t q,
                        size_t ldw, int mode, uint64_t seed, unsigned flags, double* eps);

/* ---- GPU compression: the interpolative decomposition of every
 * participating node, bottom-up (compress.cpp:17-148). Inputs: the points (n x d, original
 * order) and kernel, the tree (lchild/rchild/start/end/level/perm, num_nodes entries, perm n),
 * participation flags, and the sample rows per node in CSR form (sample_ptr[num_nodes + 1]
 * offsets into sample_idx, point indices; hmx::SampleInfo::rows). Per node the result is
 * its srank, its skeleton (point indices) and V (rows = the node's column count, srank
 * columns, column major), read with hmxg_compressed_get (CSR over nodes). */
typedef struct hmxg_compressed hmxg_compressed;
int hmxg_compress(hmxg_ctx* ctx, const double* coords, uint64_t n, uint32_t d, int32_t kernel, double h,
                  uint32_t num_nodes, const uint32_t* lchild, const uint32_t* rchild, const uint32_t* start,
                  const uint32_t* end, const uint32_t* level, const uint32_t* perm, const uint8_t* participating,
                  const uint64_t* sample_ptr, const uint32_t* sample_idx, double bacc, uint32_t max_rank,
                  hmxg_compressed** out);
int hmxg_compressed_get(const hmxg_compressed* c, const uint32_t** srank, const uint64_t** skel_ptr,
                        const uint32_t** skel, const uint64_t** v_ptr, const uint64_t** v_rows, const double** v);
void hmxg_compressed_free(hmxg_compressed* c);

const char* hmxg_last_error(void);
const char* hmxg_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HMXG_H_ */
