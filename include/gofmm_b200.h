/* gofmm_b200.h — C-ABI of the B200-native GOFMM evaluation phase (u = K~ W).
 *
 * Drop-in boundary for the reference hot path
 *     Potentials gfmm::evaluate(const HMatrix& h, const Matrix& w, const EvalOptions& opts)
 *         /root/reference/proj/include/gfmm/evaluate.hpp:287-317
 * The reference has no C ABI; these entry points are what a C/ctypes/cgo binding
 * of that function would bind. Plain pointers and sizes only; no torch or Eigen types.
 *
 * Semantics that follow the reference exactly:
 *   - w is N x r in ORIGINAL index order (column-major, ldw >= N);      evaluate.hpp:285-295
 *   - u is returned N x r in PERMUTED (tree) order (column-major);       evaluate.hpp:16,312-313
 *   - stats.flops is the reference's own flop counter formula;          evaluate.hpp:154-214
 *   - r < 1 or a wrong row count fails with GOFMM_ERR_INVALID (the reference throws
 *     std::invalid_argument, which its CLI maps to exit code 2);        evaluate.hpp:288-289,
 *                                                                        gfmm_cli.cpp:289-305
 *   - accumulation order per output block follows the reference task bodies: partners in
 *     ascending node id (evaluate.hpp:68-70,165-174), D then near blocks in ascending block index
 *     then proj^T c (evaluate.hpp:196-215), downward = cfar + parent term (evaluate.hpp:178-193).
 *
 * The compressed structure is the reference HMatrix (compress.hpp:65-79) flattened: node table
 * (tree.hpp:13-46), skeletons (compress.hpp:39-47), near/far block lists. Arrays are copied at
 * gofmm_create; the caller keeps ownership of everything it passes in.
 */
#ifndef GOFMM_B200_H
#define GOFMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes: mirror the reference's exception -> CLI exit code map (gfmm_cli.cpp:289-305). */
#define GOFMM_OK 0
#define GOFMM_ERR_INVALID 2 /* std::invalid_argument */
#define GOFMM_ERR_IO 3      /* gfmm::io_error */
#define GOFMM_ERR_NUMERIC 4 /* gfmm::numeric_error */
#define GOFMM_ERR_CUDA 5    /* device failure / no device (no reference counterpart) */

/* Entry sources. Kernel ids match the reference generators (oracle.hpp:141-256) plus the
 * Exponential (Matern-1/2) kernel BASELINE config 4 needs. */
#define GOFMM_SOURCE_STORED 0 /* D / near / far blocks supplied (DenseOracle-backed trees) */
#define GOFMM_SOURCE_KERNEL 1 /* entries generated on device from point coordinates */

#define GOFMM_KERNEL_GAUSSIAN 0    /* exp(-|xi-xj|^2 * (1/(2h^2)))      oracle.hpp:148-159, kparam[0]=h */
#define GOFMM_KERNEL_LAPLACE 1     /* max(|xi-xj|,delta)^-(d-2)         oracle.hpp:178-192, kparam[0]=delta */
#define GOFMM_KERNEL_POLYNOMIAL 2  /* (xi.xj + c)^p                     oracle.hpp:208-218, kparam={c,p} */
#define GOFMM_KERNEL_EXPONENTIAL 4 /* exp(-|xi-xj| * (1/h))             Matern-1/2, kparam[0]=h */

/* Arithmetic precision of a handle (gofmm_options.precision). The reference computes in FP64
 * only (common.hpp:18, Matrix = Eigen::MatrixXd); FP32 is north_star's second tolerance class
 * (relative 2-norm error 1e-5 vs the reference), computed as 3xTF32 on the tcgen05 tensor cores.
 * An FP32 handle is evaluated with the *_f32 entry points, an FP64 handle with the others;
 * mixing them fails with GOFMM_ERR_INVALID. */
#define GOFMM_PRECISION_F64 0
#define GOFMM_PRECISION_F32 1

/* Block materialisation modes (GOFMM_SOURCE_KERNEL only). */
#define GOFMM_BLOCKS_MATRIX_FREE 0 /* regenerate K entries inside the tile GEMM (never stored) */
#define GOFMM_BLOCKS_MATERIALIZE 1 /* generate once on device at create, keep in HBM */

typedef struct gofmm_tree_desc {
  int32_t n;         /* matrix size N (HMatrix::n) */
  int32_t num_nodes; /* nodes in BFS order, id == index, root 0 (tree.hpp:33,213-217) */
  const int32_t* parent; /* [num_nodes] -1 for the root */
  const int32_t* left;   /* [num_nodes] -1 at leaves; right == left + 1 */
  const int32_t* right;  /* [num_nodes] */
  const int32_t* level;  /* [num_nodes] root 0 */
  const int32_t* start;  /* [num_nodes] [start,end) in permuted order */
  const int32_t* end;    /* [num_nodes] */
  const int32_t* iperm;  /* [n] iperm[new] = old (tree.hpp:34) */

  /* skeletons (compress.hpp:39-47) */
  const int32_t* rank;        /* [num_nodes] skeleton rank, -1 = invalid (root) */
  const int64_t* skel_offset; /* [num_nodes+1] into skel_idx */
  const int32_t* skel_idx;    /* original indices in CPQR pivot order (compress.hpp:174-175) */
  const int64_t* proj_offset; /* [num_nodes+1] into proj (doubles) */
  const double* proj;         /* per node rank x ncand, column-major (compress.hpp:177-185);
                                 ncand = leaf size for leaves, rank(left)+rank(right) otherwise */

  /* interaction lists, each pair stored once with a < b, sorted ascending (compress.hpp:261-263) */
  int64_t num_near;
  const int32_t* near_a; /* leaf node ids */
  const int32_t* near_b;
  int64_t num_far;
  const int32_t* far_a; /* node ids, never the root; may sit on different levels */
  const int32_t* far_b;

  /* entry source */
  int32_t source; /* GOFMM_SOURCE_* */
  /* GOFMM_SOURCE_KERNEL */
  int32_t kernel;       /* GOFMM_KERNEL_* */
  int32_t dim;          /* d */
  const double* coords; /* d x n column-major, ORIGINAL order (PointCloud::coords, oracle.hpp:13) */
  double kparam[4];
  /* GOFMM_SOURCE_STORED (column-major blocks exactly as HMatrix stores them) */
  const int64_t* diag_offset; /* [num_nodes+1]; leaf_diag[id] is n_id x n_id (compress.hpp:365-371) */
  const double* diag_blocks;
  const int64_t* near_offset; /* [num_near+1]; K(idx a, idx b), n_a x n_b (compress.hpp:374-380) */
  const double* near_blocks;
  const int64_t* far_offset; /* [num_far+1]; K(skel a, skel b), k_a x k_b (compress.hpp:416-420) */
  const double* far_blocks;
} gofmm_tree_desc;

typedef struct gofmm_options {
  int32_t device;     /* CUDA device ordinal */
  int32_t near_mode;  /* GOFMM_BLOCKS_* for D and near (S) blocks; default matrix-free */
  int32_t far_mode;   /* GOFMM_BLOCKS_* for far (coupling) blocks */
  int32_t max_rhs_chunk; /* columns per internal pass; 0 = as many as fit in free HBM */
  int32_t precision;     /* GOFMM_PRECISION_* (default FP64) */
} gofmm_options;

typedef struct gofmm_eval_stats {
  int64_t flops;      /* reference flop counter (Potentials::flops) */
  double seconds;     /* wall time of the call incl. permutation (Potentials::seconds) */
  double ms_permute;  /* device time per phase (CUDA events) */
  double ms_upward;   /* N2S */
  double ms_downward; /* S2S + S2N */
  double ms_output;   /* L2L + leaf S2N */
  double ms_h2d;      /* gofmm_evaluate only: host->device copy of w */
  double ms_d2h;      /* gofmm_evaluate only: device->host copy of u */
} gofmm_eval_stats;

typedef struct gofmm_handle gofmm_handle;

/* Build the device-resident flattened tree. opts may be NULL (defaults). */
int gofmm_create(const gofmm_tree_desc* desc, const gofmm_options* opts, gofmm_handle** out);

/* Concurrency (concurrent evaluate() calls on one HMatrix with different w are
 * allowed): every call on a handle may come from any thread. Calls are serialised on the handle
 * (host side), and each enqueue waits for the previous one's device work on the handle's
 * workspace, whatever stream either was issued on — so results are bitwise those of the same
 * calls made one after another. Device-buffer calls still return before their work completes;
 * the caller's stream orders its own buffers.
 * Handles created by gofmm_create_dist with nranks > 1 hold one rank's share of the tree: the
 * whole-matrix evaluate entry points reject them (GOFMM_ERR_INVALID). */

/* u_perm = K~ w with HOST buffers (pinned or pageable); the drop-in for gfmm::evaluate. */
int gofmm_evaluate(gofmm_handle* h, const double* w, int64_t ldw, int32_t r, double* u_perm,
                   int64_t ldu, gofmm_eval_stats* stats);

/* Same with DEVICE buffers on `stream` (cudaStream_t, NULL = the handle's stream). Enqueues and
 * returns; stats->flops is filled, the phase times are filled only when stats_sync != 0. */
int gofmm_evaluate_device(gofmm_handle* h, const double* d_w, int64_t ldw, int32_t r, double* d_u_perm,
                          int64_t ldu, void* stream, int32_t stats_sync, gofmm_eval_stats* stats);

/* FP32 variants (handles created with precision GOFMM_PRECISION_F32): same semantics, float
 * buffers. Single-GPU handles only. */
int gofmm_evaluate_f32(gofmm_handle* h, const float* w, int64_t ldw, int32_t r, float* u_perm, int64_t ldu,
                       gofmm_eval_stats* stats);
int gofmm_evaluate_device_f32(gofmm_handle* h, const float* d_w, int64_t ldw, int32_t r, float* d_u_perm,
                              int64_t ldu, void* stream, int32_t stats_sync, gofmm_eval_stats* stats);
int gofmm_unpermute_device_f32(gofmm_handle* h, const float* d_u_perm, int64_t ldp, int32_t r, float* d_u,
                               int64_t ldu, void* stream);

/* Precision the handle was created with (GOFMM_PRECISION_*), -1 for a null handle. */
int32_t gofmm_precision(const gofmm_handle* h);

/* unpermute (evaluate.hpp:21-25) on device: u[iperm[t], :] = u_perm[t, :]. */
int gofmm_unpermute_device(gofmm_handle* h, const double* d_u_perm, int64_t ldp, int32_t r, double* d_u,
                           int64_t ldu, void* stream);

/* Reference flop count (Potentials::flops) for r right-hand sides, without evaluating. */
int64_t gofmm_flops(const gofmm_handle* h, int32_t r);

/* Reference flops split by phase for r right-hand sides: out3 = {upward (N2S),
 * downward (S2S + S2N), output (L2L + leaf S2N)}. */
int gofmm_phase_flops(const gofmm_handle* h, int32_t r, int64_t* out3);

/* Per-launch breakdown of one evaluation (for roofline reporting): the plan's grouped-GEMM
 * launches in issue order; ms is the CUDA-event duration from the last evaluation run with
 * stats (gofmm_evaluate, or gofmm_evaluate_device with stats_sync), -1 if none yet. */
typedef struct gofmm_launch_info {
  int32_t phase;     /* 0 upward (N2S), 1 downward (S2S + S2N), 2 output (L2L + leaf S2N) */
  int32_t level;     /* tree level (-1 for the output launch) */
  int64_t ctas;      /* grid size for this r */
  int64_t flops;     /* reference-counted flops of this launch for r columns */
  double ms;         /* measured duration */
  int32_t generated; /* 1 if the launch generates K entries from coordinates */
  int32_t reserved;
} gofmm_launch_info;

/* Fill up to cap entries of `out`; *count receives the number of launches. */
int gofmm_launch_profile(const gofmm_handle* h, int32_t r, int32_t cap, gofmm_launch_info* out, int32_t* count);

/* ---- multi-GPU: subtree split (north_star (4)) ------------------------------
 * nranks = 2^l GPUs; the tree is split at level s = l + up to 3 (split_level), and rank g owns a
 * contiguous, work-balanced run of the level-s subtrees (permuted rows [own_row_begin,
 * own_row_end)); nodes above level s are evaluated redundantly on every rank.
 * W is replicated: every rank receives the full N x r input and permutes all of it, so the W rows
 * of cross-subtree near-field partners are never exchanged.
 * One all-gather per evaluation: stage1 packs this rank's exports (the skeleton weights `what`
 * other ranks need — all level-s nodes plus cross-subtree far-field partners) into a send buffer
 * of max_send_rows x r doubles; the nranks send buffers are all-gathered into recv
 * (nranks * max_send_rows * r doubles, rank order) — by the library (gofmm_dist_evaluate, below)
 * or by the caller between gofmm_dist_stage1 and gofmm_dist_stage2 — and stage2 consumes it and
 * writes this rank's rows of u_perm. No reduction of outputs is needed. */
typedef struct gofmm_dist_info {
  int32_t rank, nranks, split_level, n_exports;
  int64_t send_rows;          /* rows (multiple of 16) this rank exports */
  int64_t max_send_rows;      /* all-gather slot size in rows (max over ranks) */
  int64_t own_row_begin, own_row_end;  /* this rank's permuted rows of u */
  int64_t flops_per_rhs;      /* this rank's reference-counted flops (incl. redundant top) */
  int64_t full_flops_per_rhs; /* the whole evaluation (reference counter) */
} gofmm_dist_info;

int gofmm_create_dist(const gofmm_tree_desc* desc, const gofmm_options* opts, int32_t rank, int32_t nranks,
                      gofmm_handle** out);
int gofmm_dist_get_info(const gofmm_handle* h, gofmm_dist_info* info);
/* Host-only plan (no device touched): info and up to cap exported ids (what: node id,
 * W rows: -(leaf id + 1)), in send-buffer order. */
int gofmm_dist_plan_host(const gofmm_tree_desc* desc, int32_t rank, int32_t nranks, gofmm_dist_info* info,
                         int32_t cap, int32_t* export_ids);
/* d_w: full N x r W in original order (device); d_send: max_send_rows x r doubles. */
int gofmm_dist_stage1(gofmm_handle* h, const double* d_w, int64_t ldw, int32_t r, double* d_send, void* stream);
/* d_recv: nranks x max_send_rows x r doubles (all-gathered); writes u_perm rows of this rank. */
int gofmm_dist_stage2(gofmm_handle* h, const double* d_recv, int32_t r, double* d_u_perm, int64_t ldu, void* stream);

/* In-library data plane: one call per evaluation on every rank. Stage 1 (permutation of the full
 * replicated W, own-subtree N2S, pack of the exported skeleton weights) -> ncclAllGather on a
 * high-priority stream of the handle -> unpack, top-of-tree N2S, downward pass and the proj^T c
 * output terms; the own leaves' D + near output terms read only W and run on `stream` while the
 * all-gather is in flight. u_perm receives this rank's rows [own_row_begin, own_row_end).
 * The communicator is either created by the library from a unique id that rank 0 obtained with
 * gofmm_nccl_unique_id and the caller broadcast (gofmm_dist_init_comm — collective over all
 * ranks), or borrowed (gofmm_dist_attach_comm: an ncclComm_t of the NCCL instance loaded in the
 * process, e.g. torch's ProcessGroupNCCL._comm_ptr(); its size / rank must match the handle).
 * NCCL is resolved at run time (the already-loaded libnccl.so.2 first); without it these calls
 * fail with GOFMM_ERR_CUDA. A single-rank handle needs no communicator.
 * timed != 0 synchronises and fills ms3 = {stage 1, all-gather, whole evaluation} (ms). */
#define GOFMM_NCCL_UNIQUE_ID_BYTES 128
int gofmm_nccl_unique_id(void* id_out /* GOFMM_NCCL_UNIQUE_ID_BYTES */);
int gofmm_dist_init_comm(gofmm_handle* h, const void* unique_id);
int gofmm_dist_attach_comm(gofmm_handle* h, void* nccl_comm);
int gofmm_dist_evaluate(gofmm_handle* h, const double* d_w, int64_t ldw, int32_t r, double* d_u_perm, int64_t ldu,
                        void* stream, int32_t timed, double* ms3);
int gofmm_dist_evaluate_f32(gofmm_handle* h, const float* d_w, int64_t ldw, int32_t r, float* d_u_perm,
                            int64_t ldu, void* stream, int32_t timed, double* ms3);

/* The same with HOST buffers: W (n x r, original order) is uploaded, the evaluation above runs on
 * the handle's stream, and this rank's rows [own_row_begin, own_row_end) of u_perm are written back
 * (other rows are not touched). Synchronous; ms3 may be NULL (else timed as above). */
int gofmm_dist_evaluate_host(gofmm_handle* h, const double* w, int64_t ldw, int32_t r, double* u_perm, int64_t ldu,
                             double* ms3);

/* FP32 handles: the same two stages; the send buffer is 2 * max_send_rows * r floats (hi then
 * lo halves of the 3xTF32 operands), recv is nranks of those slots in rank order. */
int gofmm_dist_stage1_f32(gofmm_handle* h, const float* d_w, int64_t ldw, int32_t r, float* d_send, void* stream);
int gofmm_dist_stage2_f32(gofmm_handle* h, const float* d_recv, int32_t r, float* d_u_perm, int64_t ldu,
                          void* stream);

/* ---- error_eps2 support (evaluate.hpp:330-373) ---------------------------------------------
 * Exact rows of K W for nrows ORIGINAL indices `rows` (host array), W on the device in original
 * order; out is nrows x r column-major (device). Matrix-free kernel sources only. */
int gofmm_exact_rows(gofmm_handle* h, const int32_t* rows, int32_t nrows, const double* d_w, int64_t ldw, int32_t r,
                     double* d_out, int64_t ldo, void* stream);
/* error_eps2's draws from the reference Rng (common.hpp:40-104): Rng(seed, 0xe952), the sorted
 * row sample (min(sample_rows, n) rows), then W column-major (host). w_out may be NULL. */
int gofmm_rng_eps2_draw(uint64_t seed, int32_t n, int32_t r, int32_t sample_rows, int32_t* rows_out, double* w_out,
                        int64_t ldw);
/* The same draws for resample `attempt` (0, 1, 2): error_eps2 redraws W from the same stream up to
 * three times while the sampled rows of K W vanish (evaluate.hpp:343-372); attempt a's W follows
 * the r * n normals of attempts 0..a-1. rows_out may be NULL. */
int gofmm_rng_eps2_draw_attempt(uint64_t seed, int32_t n, int32_t r, int32_t sample_rows, int32_t attempt,
                                int32_t* rows_out, double* w_out, int64_t ldw);

/* ---- compress-side skeletonisation ------------------------------------
 * Replaces gfmm::skeletonize_node (compress.hpp:149-187) for a batch of nodes: column-pivoted
 * Householder QR of each node's sampled block K(sample_cols, candidates) in the reference's
 * Eigen 3.4 ColPivHouseholderQR operation order, rank = #{l : |R_ll| > tau |R_11|} clamped to
 * [1, min(s, rows, cols)], skeleton = the first rank pivots, proj = [I | R11^-1 R12] in pivot
 * order. Bit-identical to the reference on the same block (tests/test_skel_gpu.py).
 * blocks: node t's block column-major rows[t] x cols[t] at blocks + block_off[t] (host).
 * Outputs (host): rank_out[t]; achieved_out[t] (Skeleton::achieved_tol); perm_out: cols[t]
 * column-pivot indices per node, concatenated (skeleton = candidates[perm[0..rank)]);
 * proj_out: per node a slot of min(s, rows, cols) * cols doubles, concatenated, of which the
 * first rank * cols hold proj column-major (ld = rank). */
typedef struct gofmm_skel_stats {
  double seconds;   /* wall time of the call (uploads, kernel, downloads) */
  double kernel_ms; /* device time of the batched kernel (CUDA events) */
  double bytes;     /* algorithmic bytes streamed by the kernel (3 passes over each trailing block) */
  double flops;     /* Householder application flops (4 per trailing element per step) */
} gofmm_skel_stats;
int gofmm_skeletonize_batch(int32_t nnodes, const int32_t* rows, const int32_t* cols, const int64_t* block_off,
                            const double* blocks, int32_t s, double tau, int32_t device, int32_t* rank_out,
                            double* achieved_out, int32_t* perm_out, double* proj_out, gofmm_skel_stats* stats);
const char* gofmm_skeletonize_last_error(void);

/* ---- ANN leaf pass -----------------------------------------------------
 * The per-leaf body of ann_iteration (neighbors.hpp:88-106) for all leaves of one random tree:
 * pairwise distances inside each leaf (kind 0: GeometricL2, bit-identical to the reference;
 * kind 1: KernelL2 over a Gaussian oracle of bandwidth h) merged into every index's list as the
 * kappa smallest distinct indices under (distance, index) (merge_candidates, :35-63).
 * coords: d x n column-major (host). Leaves: leaf_idx[leaf_off[l] .. leaf_off[l+1]) (host; from
 * the host-built random tree). Table (host, updated in place): table_j / table_d n x kappa
 * row-major, table_len[i] entries valid. kappa = NeighborTable::k (<= 32); leaves <= 1024. */
int gofmm_ann_leaf_merge(int32_t n, int32_t d, const double* coords, int32_t kind, double h, int32_t kappa,
                         int32_t nleaves, const int32_t* leaf_off, const int32_t* leaf_idx, int32_t device,
                         int32_t* table_j, double* table_d, int32_t* table_len, double* kernel_ms);
const char* gofmm_ann_last_error(void);

/* ---- compress: the input of gofmm_create from a point cloud ---------------
 * gfmm::compress (compress.hpp:331-434) with its kernel oracle, metric, ANN search, metric tree,
 * near-field selection, structure walk, column sampling and skeletonisation: host pipeline with
 * the ANN leaf passes, the per-level sampled blocks and the per-level batched CPQR / ID on the
 * GPU. D / near / far blocks are not stored (gofmm_create regenerates them matrix-free); their
 * entries are counted as the reference's CountingOracle counts them.
 * entries = GOFMM_ENTRIES_HOST: every entry that steers a decision is computed on the host with
 * the reference's formulas and reduction order -> tree, neighbour lists, skeletons, proj and all
 * statistics bit-identical to the reference compress. GOFMM_ENTRIES_DEVICE: ANN leaf passes
 * (geometric, or kernel L2 over a Gaussian) and sampled blocks generated on the GPU (libdevice
 * exp/pow: a few ulps from glibc, so exact near-ties may resolve differently). */
#define GOFMM_DIST_GEOMETRIC 0 /* DistanceKind::GeometricL2 (metric.hpp:8) */
#define GOFMM_DIST_KERNEL 1    /* DistanceKind::KernelL2 (the reference default) */
#define GOFMM_DIST_ANGLE 2     /* DistanceKind::Angle */
#define GOFMM_ENTRIES_HOST 0
#define GOFMM_ENTRIES_DEVICE 1

typedef struct gofmm_compress_config { /* RunConfig (compress.hpp:12-34) + device knobs */
  int32_t m, s;
  double tau;
  int32_t kappa;
  double budget;
  int32_t distance; /* GOFMM_DIST_* */
  uint64_t seed;
  int32_t ann_iterations;
  int32_t threads; /* host threads */
  int32_t entries; /* GOFMM_ENTRIES_* */
  int32_t device;
} gofmm_compress_config;

typedef struct gofmm_compress_stats { /* CompressStats (compress.hpp:49-59) + structure sizes */
  int64_t entries_evaluated, compress_flops, near_field_entries;
  int32_t max_skeleton, ann_iterations_done;
  double mean_skeleton, compress_seconds, tree_seconds;
  double ann_recall[64]; /* per ANN iteration (first ann_iterations_done) */
  double ann_seconds, ann_kernel_ms, skeleton_seconds, skel_kernel_ms;
  int32_t depth, num_nodes, num_leaves, reserved;
  int64_t num_near, num_far;
} gofmm_compress_stats;

typedef struct gofmm_compressed gofmm_compressed;

/* RunConfig defaults (m = s = 256, tau 1e-5, kappa 32, budget 0.03, kernel distance, seed 0,
 * 10 ANN iterations), all host threads, device entries, device 0. */
void gofmm_compress_default_config(gofmm_compress_config* cfg);
/* kernel: GOFMM_KERNEL_*; kparam[0..1] as gofmm_tree_desc::kparam (Laplace: the resolved floor);
 * coords d x n column-major, original order (copied). */
int gofmm_compress(int32_t kernel, const double* kparam, int32_t dim, int32_t n, const double* coords,
                   const gofmm_compress_config* cfg, gofmm_compressed** out);
/* The flattened HMatrix as a gofmm_tree_desc (GOFMM_SOURCE_KERNEL); pointers stay valid until
 * gofmm_compressed_free. */
int gofmm_compressed_desc(const gofmm_compressed* c, gofmm_tree_desc* desc);
int gofmm_compressed_stats(const gofmm_compressed* c, gofmm_compress_stats* stats);
int gofmm_compressed_free(gofmm_compressed* c);
const char* gofmm_compress_last_error(void);

/* ---- error_eps2 (evaluate.hpp:330-373) ------------------------------------------------------
 * ErrorReport (evaluate.hpp:319-326) of this handle's evaluation against exact rows of K: the
 * reference's draws (gofmm_rng_eps2_draw_attempt, up to 3 W draws), u = K~ W on the device, the exact
 * rows K(rows, :) W generated matrix-free on the device (kernel sources only). rows_out (optional)
 * receives the min(sample_rows, n) sampled original indices. A degenerate draw three times in a
 * row -> GOFMM_ERR_NUMERIC (the reference's numeric_error). */
typedef struct gofmm_eps2_report {
  double eps2;
  double per_entry[10]; /* relative row errors of the first 10 sampled rows */
  int32_t num_per_entry;
  double mean_sample;   /* average relative row error over the sample */
  int64_t eval_flops;
  double eval_seconds;
} gofmm_eps2_report;
int gofmm_error_eps2(gofmm_handle* h, int32_t r, int32_t sample_rows, uint64_t seed, gofmm_eps2_report* rep,
                     int32_t* rows_out);

/* ---- point sources of the CLI (tools/gfmm_cli.cpp:55-92) ---------------------------------------
 * PointCloud::random_gaussian(n, d, seed) (oracle.hpp:18-25) into out (d x n column-major), and
 * default_laplace_floor(points, seed) (oracle.hpp:274-288). */
int gofmm_points_gaussian(int32_t n, int32_t d, uint64_t seed, double* out);
int gofmm_default_laplace_floor(int32_t d, int32_t n, const double* coords, uint64_t seed, double* out);
/* Rng(seed, stream).gauss() (common.hpp:52-77) column-major into w (n x r, leading dimension ldw). */
int gofmm_rng_gauss_stream(uint64_t seed, uint64_t stream, int32_t n, int32_t r, double* w, int64_t ldw);

/* Bytes of device memory held by the handle (tree + workspace). */
int64_t gofmm_device_bytes(const gofmm_handle* h);

/* Number of kernel launches one evaluation issues (for the bench's gpu_launches). */
int32_t gofmm_launches_per_eval(const gofmm_handle* h);

int gofmm_destroy(gofmm_handle* h);

/* Message of the last failure on the calling thread ("" if none). */
const char* gofmm_last_error(void);

int32_t gofmm_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GOFMM_B200_H */
