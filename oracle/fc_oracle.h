/*
 * fc_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, single-threaded CPU restatement of the reference GPA/FISTA hot path
 * (arXiv 2506.04045 reference, /root/reference/proj/include/fuzzyclust/).  It is
 * the CHECKER for the CUDA path: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.  The product path
 * (paper_2506_04045_b200/ and include/) never links or calls it.
 *
 * Parity of this restatement is PINNED two ways (tests/test_oracle.py):
 *   - against the reference itself, compiled from /root/reference headers into
 *     oracle/_ref/libfcref.so (oracle/ref_driver.cpp), bitwise, on random instances;
 *   - against the reference's own known-answer tests (7-node goldens 12.25 /
 *     11.5 / 6.49 / 8.84, the splitmix64 golden stream, the known projections)
 *     and the committed fixtures under tests/golden/.
 * The backtracking FISTA variant (fco_solve with method FCO_FISTA_BT) has no
 * reference implementation (SPEC.md:354 lists line search as a non-goal):
 * its parity is UNPINNED ("parity by restatement").
 *
 * Arithmetic: IEEE binary64, round-to-nearest, no FMA contraction (build with
 * -ffp-contract=off and no -march, matching the reference Release flags,
 * proj/CMakeLists.txt:7-9).
 */
#ifndef FC_ORACLE_H
#define FC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { FCO_OK = 0, FCO_IO = 1, FCO_INVALID = 2 };
enum { FCO_GPA = 0, FCO_FISTA = 1, FCO_FISTA_BT = 2 };
enum { FCO_TOL_REACHED = 0, FCO_MAX_ITER = 1, FCO_LOSS_INCREASE_FISTA = 2 };

typedef struct {
    uint64_t n;
    uint64_t nnz;
    const int64_t* row_ptr;   /* n+1 */
    const uint32_t* col_idx;  /* nnz, strictly increasing per row */
    const double* values;     /* nnz, or NULL = every value 1.0 */
    double frob_sq;           /* sum of v*v in stored order (sparse.hpp:59-60) */
} fco_csr;

typedef struct {
    double step_size;      /* <= 0 -> default_step_size (solver.hpp:78-85) */
    uint64_t max_iter;
    double tol;
    int method;            /* FCO_GPA | FCO_FISTA | FCO_FISTA_BT */
    uint64_t trace_every;
    int fista_restart;
    /* backtracking only (new functionality, parity unpinned) */
    double bt_eta;         /* L <- eta * L on a failed sufficient-decrease test */
    uint32_t bt_max;       /* max backtracks per iteration */
} fco_config;

typedef struct {
    uint64_t iteration;
    double loss;
    int32_t loss_increased;
    int32_t backtracks;
    double step;           /* step actually used at this iteration */
} fco_record;

typedef struct {
    int32_t reason;
    int32_t pad;
    uint64_t iterations;
    double final_loss;
    double step_size;
    uint64_t n_records;
} fco_summary;

const char* fco_last_error(void);

/* rng.hpp:14-38 */
uint64_t fco_splitmix_next(uint64_t* state);
double fco_splitmix_next_double(uint64_t* state);

/* simplex.hpp:18-59 -- returns FCO_INVALID on empty / non-finite input */
int fco_project_simplex(double* x, size_t c);

/* membership.hpp:86-94 (kRandom); x is C x N column-major */
int fco_init_random(size_t n, size_t c, uint64_t seed, double* x);
/* membership.hpp:49-61 feasibility_error / validate */
double fco_feasibility_error(const double* x, size_t c, size_t n);

/* objective.hpp:61-95 -- G = X X^T, C x C row-major */
void fco_share_matrix(const double* x, size_t c, size_t n, double* g);
/* objective.hpp:25-29 */
double fco_share_frob_sq(const double* g, size_t c);
/* objective.hpp:61-90 cross_share(A, B) = A B^T (C x C, row-major) */
void fco_cross_share(const double* a, const double* b, size_t c, size_t n, double* g);
/* objective.hpp:186-217 hessian_vector_product(xbar, v, s) (N x C, node-major) */
int fco_hessian_vector_product(const double* x, const double* v, size_t c, const fco_csr* s, double* out);
/* dense.hpp:40-46 frob_inner */
double fco_frob_inner(const double* a, const double* b, size_t count);
/* objective.hpp:151-173 -- xs is C x N column-major */
int fco_fused_column_pass(const double* x, size_t c, const fco_csr* s, double* xs, double* merge);
/* objective.hpp:176-180 */
double fco_loss_decomposed(const double* x, size_t c, const fco_csr* s, const double* g);
/* solver.hpp:89-107 */
int fco_gpa_step_fused(const double* x, size_t c, size_t n, const double* g, const double* xs,
                       double tau, double* out);
/* solver.hpp:72, 78-85 */
double fco_fista_t_next(double t);
double fco_default_step_size(const fco_csr* s, size_t n);

/* solver.hpp:137-277 (run_gpa / run_fista / solve), plus the unpinned
 * backtracking FISTA.  x_out (C x N) receives result.membership. */
int fco_solve(const fco_csr* s, const fco_config* cfg, size_t c, const double* x0,
              double* x_out, fco_record* trace, uint64_t trace_cap, fco_summary* out);

#ifdef __cplusplus
}
#endif
#endif
