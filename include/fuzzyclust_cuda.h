/*
 * fuzzyclust_cuda.h -- C ABI of the B200-native GPA/FISTA solver
 * (libfuzzyclust_cuda.so, built from paper_2506_04045_b200/csrc/).
 *
 * The reference (arXiv 2506.04045, /root/reference/proj) is a header-only C++
 * library with no FFI; its "operator API" is the inline header API that callers
 * #include (fuzzyclust.hpp:1-14).  This ABI is what those header bodies bind to
 * (see the headers under include/fuzzyclust/ and INTEGRATION.md).  Each entry point names the
 * reference interface it replaces.
 *
 * Conventions:
 *  - Plain pointers and sizes; no C++ or torch types.
 *  - Dense matrices are the reference's C x N column-major layout
 *    (dense.hpp:12-27), i.e. U = N x C row-major: node i's C memberships are
 *    contiguous.  Host buffers belong to the caller; the context owns device memory.
 *  - The similarity is the reference's symmetric CSC == CSR (sparse.hpp:18-20):
 *    row_ptr int64[N+1], col_idx uint32[nnz] strictly increasing per row,
 *    values f64[nnz] or NULL meaning "every value is 1.0".
 *  - Return codes: 0 ok, 1 I/O (IoError), 2 invalid input (InvalidInput, incl. the
 *    non-finite projection input of simplex.hpp:21-23), 3 CUDA/NCCL failure.
 *    fc_last_error() returns the message (same text as the reference exception).
 *  - Arithmetic is IEEE FP64 with no FMA contraction in the reference's
 *    summation orders, so results are bitwise identical to the reference CPU
 *    solver for any GPU count.
 *  - One control thread per context; a context is not thread-safe.
 */
#ifndef FUZZYCLUST_CUDA_H
#define FUZZYCLUST_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FC_ABI_VERSION 1

enum { FC_OK = 0, FC_IO = 1, FC_INVALID = 2, FC_DEVICE = 3 };
/* Method (solver.hpp:18) plus the new backtracking FISTA */
enum { FC_GPA = 0, FC_FISTA = 1, FC_FISTA_BT = 2 };
/* TerminationReason (solver.hpp:20) */
enum { FC_TOL_REACHED = 0, FC_MAX_ITER = 1, FC_LOSS_INCREASE_FISTA = 2 };

typedef struct fc_ctx fc_ctx;

/* SolverConfig (solver.hpp:31-48).  `workers` is replaced by the context's
 * device set; bt_* are new (backtracking, no reference). */
typedef struct {
    double step_size;       /* <= 0 (exactly 0) selects default_step_size, solver.hpp:78-85 */
    uint64_t max_iter;
    double tol;
    int32_t method;         /* FC_GPA | FC_FISTA | FC_FISTA_BT */
    int32_t fista_restart;
    uint64_t trace_every;
    double bt_eta;          /* backtracking growth factor for L = 1/step (> 1) */
    uint32_t bt_max;        /* max backtracks per iteration */
    uint32_t flags;         /* reserved, 0 */
} fc_solver_config;

/* TraceRecord (solver.hpp:50-55) plus backtracking fields */
typedef struct {
    uint64_t iteration;
    double loss;
    double elapsed_ms;      /* device %globaltimer since solve start */
    int32_t loss_increased;
    int32_t backtracks;
    double step;            /* step actually used (== step_size unless backtracking) */
} fc_trace_record;

/* SolverTrace scalars (solver.hpp:57-63) */
typedef struct {
    int32_t reason;
    int32_t pad;
    uint64_t iterations;
    double final_loss;
    double step_size;
    uint64_t n_records;     /* records produced (may exceed trace_cap; extra dropped) */
} fc_solve_summary;

/* ---- library / context -------------------------------------------------- */
const char* fc_version(void);
int fc_abi_version(void);
/* Message for the last failing call on `ctx` (or on this thread if ctx == NULL). */
const char* fc_last_error(const fc_ctx* ctx);

/* NCCL unique id (128 bytes) for multi-rank contexts; rank 0 makes it and the
 * launcher broadcasts it (bench.py uses torch.distributed for that plumbing). */
int fc_nccl_unique_id(unsigned char id[128]);

/* One process per GPU.  world == 1: nccl_id may be NULL. */
int fc_create(fc_ctx** out, int device, int rank, int world, const unsigned char* nccl_id);
/* Test topology: `shards` row shards emulated on ONE device (same kernels,
 * same partition and ordered cross-shard chain, no NCCL). */
int fc_create_virtual(fc_ctx** out, int device, int shards);
/* Numerical contract of the solver entry points (fc_solve / fc_solver_*):
 *   0 (default) bitwise: the reference's operation order, no FMA -- results equal the
 *     reference CPU solver bit for bit;
 *   1 tolerance (north star: loss within 1e-9 relative at every record, U within 1e-7,
 *     identical supports): FISTA gathers one operand per sweep (S X_ext^{n+1} formed by
 *     linearity from S bar^n and S bar^{n-1}, solver.hpp:261 applied to S x) and the
 *     Gram / gradient contractions use fused multiply-add.  GPA and FISTA without
 *     backtracking, C <= 128.  Granular operators stay bitwise. */
int fc_set_parity_mode(fc_ctx* ctx, int mode);
int fc_get_parity_mode(const fc_ctx* ctx);

/* Multi-rank exchange plan chosen at fc_upload_csr: 1 = halo exchange (only the rows
 * other shards' columns name move each iteration; locality graphs), 0 = full
 * allgather.  FC_HALO=0/1 forces it; default: halo when every rank then receives less
 * than half of what the allgather would move.  Rows received / sent per exchange. */
int fc_halo_info(const fc_ctx* ctx, uint64_t* recv_rows, uint64_t* send_rows);

/* In-process loopback group (tests / single-GPU validation of the multi-rank path):
 * `world` rank contexts in ONE process on `device`, one host thread per rank, each
 * created with fc_create_loopback.  The collectives are stream-ordered device copies
 * pulled from the peer after a CUDA event (no NCCL); the ranks run exactly the
 * multi-rank code of fc_create(rank, world, nccl_id): shard partition, allgather,
 * ordered recv -> combine -> send chain, broadcast from the last rank. */
typedef struct fc_loopback fc_loopback;
int fc_loopback_create(fc_loopback** out, int device, int world);
void fc_loopback_destroy(fc_loopback* group);
int fc_create_loopback(fc_ctx** out, fc_loopback* group, int rank);
void fc_destroy(fc_ctx* ctx);

/* SparseSimilarity (sparse.hpp:21-146).  Every rank passes the FULL CSR; the
 * context keeps its nnz-balanced, 1024-row-aligned shard on the device.
 * frob_sq is SparseSimilarity::frob_sq() (sum of v*v in stored order). */
int fc_upload_csr(fc_ctx* ctx, uint64_t n, uint64_t nnz, const int64_t* row_ptr,
                  const uint32_t* col_idx, const double* values, double frob_sq);
/* ---- second order (granular, single-rank) --------------- */
/* cross_share(A, B) = A B^T (objective.hpp:61-90): g_out C x C row-major; A, B n x c
 * node-major; c <= 128 (computed as the Gram of the stacked n x 2c matrix). */
int fc_cross_share(fc_ctx* ctx, uint32_t c, const double* a, const double* b, double* g_out);
/* hessian_vector_product(xbar, v, s) (objective.hpp:182-217) against the resident
 * similarity: out_i = -4 (V s_i - A x_i - A^T x_i - B v_i), A = cross_share(V, X),
 * B = share_matrix(X); x, v, out n x c node-major; c <= 128. */
int fc_hessian_vector_product(fc_ctx* ctx, uint32_t c, const double* x, const double* v, double* out);
/* The pairwise part of refine (secondorder.hpp:132-330) for a critical point x with
 * gradient grad (both n x c node-major): the kept pair directions V = e_k - e_l at
 * node i (critical_cone_directions' filter and order) are enumerated and evaluated
 * on the device without materialising them; condition (a) <H V, V> (bit-identical
 * to quadratic_form) and condition (b) <grad, W> over the W each V admits, both over
 * the first `budget` directions, ties to the first in enumeration order.
 * triples_out (optional, 3 * min(pairs, triples_cap)): (node, plus, minus) per pair. */
typedef struct fc_refine_pairs_out {
    uint64_t pairs;                            /* kept pair directions */
    double a_worst;                            /* min(0, min <H V, V>) */
    uint64_t a_index;                          /* its direction index (UINT64_MAX: none < 0) */
    uint32_t a_col, a_plus, a_minus, pad0;     /* that direction: node, +1 row, -1 row */
    double b_worst;                            /* min(0, min <grad, W>) */
    uint64_t b_index;                          /* index of the base direction V (UINT64_MAX: none) */
    uint32_t b_col, b_plus, b_minus;           /* W = e_plus - e_minus at node b_col */
    uint32_t b_base_plus, b_base_minus, pad1;  /* V = e_base_plus - e_base_minus at b_col */
} fc_refine_pairs_out;
int fc_refine_pairs(fc_ctx* ctx, uint32_t c, const double* x, const double* grad, double eps_active,
                    double eps_grad_orth, uint64_t budget, uint32_t* triples_out, uint64_t triples_cap,
                    fc_refine_pairs_out* out);
/* frob_inner (dense.hpp:40-46) on the host: sum_k a[k] * b[k], strictly sequential
 * (quadratic_form = frob_inner(HVP, V)). */
double fc_frob_inner(const double* a, const double* b, uint64_t count);

/* ---- edge-list ingest ----------------------------------- */
typedef struct fc_ingest_result {
    uint64_t parsed_nodes;   /* nodes after parse_edge_list */
    uint64_t lcc_nodes;      /* nodes of the largest connected component (stages >= 1) */
    uint64_t num_nodes;      /* nodes of the returned graph */
    uint64_t num_edges;      /* edges of the returned graph */
    uint32_t* edges;         /* 2 * num_edges ids, (u < v) pairs sorted ascending; fc_free */
    int64_t* original_ids;   /* num_nodes input ids of the returned nodes; fc_free */
} fc_ingest_result;
/* The reference's load_pipeline (tools/fuzzyclust.cpp:62-89) on `len` bytes of
 * "u v" text: stages 0 = parse_edge_list only (graph.hpp:63-103, ids compacted by
 * first appearance, self-loops / duplicates dropped, symmetrised), 1 = + largest
 * connected component (graph.hpp:146-175, ties to the smallest id), 2 = + 2-core
 * (graph.hpp:185-219).  Parse errors: FC_IO with the reference's messages and line
 * numbers ("edge list is empty" when no edge line). */
int fc_ingest_edge_list(fc_ctx* ctx, const char* text, uint64_t len, int stages, fc_ingest_result* out);
/* largest_connected_component_nodes / two_core_nodes (graph.hpp:146-169, :206-213)
 * of a Graph given as its edge list (2 * num_edges ids); *nodes_out (ascending,
 * malloc'ed: fc_free) and *count. */
int fc_graph_lcc_nodes(fc_ctx* ctx, uint64_t num_nodes, uint64_t num_edges, const uint32_t* edges,
                       uint32_t** nodes_out, uint64_t* count);
int fc_graph_two_core_nodes(fc_ctx* ctx, uint64_t num_nodes, uint64_t num_edges, const uint32_t* edges,
                            uint32_t** nodes_out, uint64_t* count);

/* SparseSimilarity::from_triplets (sparse.hpp:28-62) on the device: triplets
 * (row i, column j, value; values NULL = all 1.0) are validated, sorted by
 * (column, row), checked for duplicates and exact symmetry (the reference's
 * messages, first failing entry in its loop order), and the CSR is written to
 * row_ptr_out[n+1] / col_idx_out[nnz] / values_out[nnz] (may be NULL) with
 * frob_sq and whether every value is 1.0.  The result becomes the context's
 * resident similarity (as fc_upload_csr: a multi-rank context keeps its shard). */
int fc_build_from_triplets(fc_ctx* ctx, uint64_t n, uint64_t nnz, const uint32_t* rows, const uint32_t* cols,
                           const double* values, int64_t* row_ptr_out, uint32_t* col_idx_out, double* values_out,
                           double* frob_sq_out, int* pattern_only_out);
/* SparseSimilarity::build_similarity (sparse.hpp:66-75) on the device: A + I
 * from `num_edges` (u, v) pairs (a normalised Graph's edge list); nnz =
 * num_nodes + 2 num_edges, all values 1.0. */
int fc_build_similarity(fc_ctx* ctx, uint64_t num_nodes, uint64_t num_edges, const uint32_t* edges,
                        int64_t* row_ptr_out, uint32_t* col_idx_out, double* frob_sq_out);
/* Row bounds of every shard after fc_upload_csr: bounds[0..world]. */
int fc_partition(const fc_ctx* ctx, uint64_t* bounds, int max_world);

/* ---- granular operators (host buffers in / out) ---------------------------
 * share_matrix, objective.hpp:92-95 -> g_out C x C row-major */
int fc_share_matrix(fc_ctx* ctx, uint32_t c, const double* x, double* g_out);
/* fused_column_pass, objective.hpp:151-173 -> xs_out C x N col-major (may be NULL), merge */
int fc_fused_column_pass(fc_ctx* ctx, uint32_t c, const double* x, double* xs_out, double* merge_out);
/* loss_decomposed, objective.hpp:176-180 (g is the caller's share matrix) */
int fc_loss_decomposed(fc_ctx* ctx, uint32_t c, const double* x, const double* g, double* loss_out);
/* gpa_step_fused, solver.hpp:89-107 */
int fc_gpa_step_fused(fc_ctx* ctx, uint32_t c, const double* x, const double* g, const double* xs,
                      double tau, double* x_out);
/* gpa_step, solver.hpp:110-114 */
int fc_gpa_step(fc_ctx* ctx, uint32_t c, const double* x, const double* g, double tau, double* x_out);
/* project_simplex_inplace (simplex.hpp:18-59) applied to `rows` vectors of
 * length c stored contiguously (init_membership's per-column projection). */
int fc_project_simplex_rows(fc_ctx* ctx, uint32_t c, uint64_t rows, double* x);

/* Per-row pieces used by the reference's single-column API (host buffers):
 *   gradient_column_fused (objective.hpp:113-118): out_i = -4 (xs_i - G x_i)
 *   loss_terms_column     (objective.hpp:131-135): out_i = sum_k xs_i[k] x_i[k]
 * g is C x C row-major; xs, x, out are `rows` vectors of length c. */
int fc_gradient_rows(fc_ctx* ctx, uint32_t c, uint64_t rows, const double* g, const double* xs,
                     const double* x, double* out);
int fc_loss_terms_rows(fc_ctx* ctx, uint32_t c, uint64_t rows, const double* xs, const double* x,
                       double* out);

/* ---- solver ---------------------------------------------------------------
 * solve / run_gpa / run_fista, solver.hpp:137-277: the whole loop on device.
 * x_out receives result.membership (C x N col-major). */
int fc_solve(fc_ctx* ctx, const fc_solver_config* cfg, uint32_t c, const double* x0,
             double* x_out, fc_trace_record* trace, uint64_t trace_cap, fc_solve_summary* out);

/* Stateful form of fc_solve (bench timing, warm restarts):
 *   begin  : validate, upload x0, run the iteration-0 pass (FISTA loss record 0)
 *   run    : enqueue up to `iterations` more iterations (async; finished runs are no-ops)
 *   sync   : wait for the device; *done = 1 once the stop rule fired
 *   end    : download membership + trace.  */
int fc_solver_begin(fc_ctx* ctx, const fc_solver_config* cfg, uint32_t c, const double* x0);
int fc_solver_run(fc_ctx* ctx, uint64_t iterations);
int fc_solver_sync(fc_ctx* ctx, int* done);
int fc_solver_end(fc_ctx* ctx, double* x_out, fc_trace_record* trace, uint64_t trace_cap,
                  fc_solve_summary* out);
/* Run the session's remaining iterations (same stop rule and pass budget as
 * fc_solve), then fc_solver_end. */
int fc_solver_finish(fc_ctx* ctx, double* x_out, fc_trace_record* trace, uint64_t trace_cap,
                     fc_solve_summary* out);

/* ---- checkpoint / resume (new) ---------------------------
 * fc_solver_checkpoint waits for the enqueued iterations, then writes the whole
 * session (device control state, trace so far, every iterate / sweep / Gram
 * buffer the next iteration reads) to `path`.  fc_solver_resume loads it into a
 * context holding the same similarity (n, nnz, frob_sq and shard layout are
 * checked) and reopens the session: continuing with fc_solver_run/finish gives
 * the same trace and membership, bit for bit, as the uninterrupted run.
 * Single-rank contexts (virtual shards allowed). FC_IO on file errors. */
int fc_solver_checkpoint(fc_ctx* ctx, const char* path);
int fc_solver_resume(fc_ctx* ctx, const char* path);

/* ---- instrumentation (bench.py) ------------------------------------------ */
/* The CUDA stream every kernel and collective of ctx is enqueued on. */
void* fc_stream(fc_ctx* ctx);
/* Kernel launches enqueued by this context since creation. */
uint64_t fc_launch_count(const fc_ctx* ctx);
/* Per-kernel-class device time (ms) and launch counts since the last reset,
 * measured with CUDA events on ctx's stream when profiling is enabled.
 * Classes: 0 step, 1 gram, 2 sweep, 3 rowsum, 4 combine, 5 finalize, 6 comm. */
int fc_set_profiling(fc_ctx* ctx, int enabled);
int fc_kernel_times(fc_ctx* ctx, double* ms, uint64_t* launches, int n_classes);

/* ---- host utilities (no GPU needed) -------------------------------------- */
/* nnz-balanced partition of rows into `world` contiguous shards whose
 * boundaries are multiples of 1024 (parallel.hpp:15 kReductionBlock). */
int fc_plan_partition(uint64_t n, const int64_t* row_ptr, int world, uint64_t* bounds);

/* Synthetic graphs (new: the reference generator, generator.hpp:46-97, is the
 * O(n^2) two-cluster ER model).  Output is build_similarity's A+I CSR.
 * kind 0: stochastic block model; kind 1: power-law citation-like. */
typedef struct {
    int32_t kind;
    uint32_t blocks;        /* SBM: number of equal blocks */
    uint64_t n;             /* nodes */
    uint64_t m;             /* undirected edge draws (duplicates merged) */
    uint64_t seed;
    double p_in;            /* SBM: probability an edge stays inside its block */
    double alpha;           /* citation: out-degree power-law exponent */
    double gamma;           /* citation: age-bias exponent of cited node (>= 1) */
    int32_t locality;       /* citation: 1 keeps time order ids, 0 random relabel */
    int32_t threads;        /* 0 = hardware concurrency */
} fc_graph_spec;

int fc_generate_graph(const fc_graph_spec* spec, uint64_t* nnz_out, int64_t** row_ptr_out,
                      uint32_t** col_idx_out);
void fc_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
