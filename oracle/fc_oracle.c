/*
 * fc_oracle.c -- TEST INFRASTRUCTURE ONLY (see fc_oracle.h).
 *
 * Single-threaded restatement of the reference hot path.  Each function cites the
 * reference lines it follows (paths relative to /root/reference/proj/include/fuzzyclust).
 * The reference's block-parallel reductions (parallel.hpp:15-68) are restated as
 * their fixed serial order: per-1024-column block partials combined in ascending
 * block order.  That order is what makes the reference bitwise independent of
 * its worker count, so a serial loop reproduces every worker count.
 */
#include "fc_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define FCO_BLOCK 1024u /* parallel.hpp:15 kReductionBlock */

static char g_err[512];

const char* fco_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* ---------------------------------------------------------------- rng.hpp:21-32 */
uint64_t fco_splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double fco_splitmix_next_double(uint64_t* state) {
    return (double)(fco_splitmix_next(state) >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------ simplex.hpp:18-59 */
static int cmp_desc(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) ? -1 : (x < y) ? 1 : 0;
}

/* std::max(a, b) == (a < b) ? b : a  (keeps -0.0 when a == -0.0, b == +0.0) */
static inline double ref_max(double a, double b) { return (a < b) ? b : a; }

int fco_project_simplex(double* x, size_t c) {
    if (c == 0) return fail(FCO_INVALID, "project_simplex: empty vector");
    for (size_t k = 0; k < c; ++k)
        if (!isfinite(x[k])) return fail(FCO_INVALID, "project_simplex: non-finite entry");
    if (c == 1) { x[0] = 1.0; return FCO_OK; }

    double stack_buf[256];
    double* sorted = c <= 256 ? stack_buf : (double*)malloc(c * sizeof(double));
    memcpy(sorted, x, c * sizeof(double));
    qsort(sorted, c, sizeof(double), cmp_desc); /* any correct descending sort: see DESIGN.md */

    double cumsum = 0.0, threshold = 0.0;
    for (size_t k = 0; k < c; ++k) {                       /* simplex.hpp:31-36 */
        cumsum += sorted[k];
        const double t = (cumsum - 1.0) / (double)(k + 1);
        if (sorted[k] - t >= 0.0) threshold = t;
    }
    if (sorted != stack_buf) free(sorted);

    for (size_t k = 0; k < c; ++k) x[k] = ref_max(x[k] - threshold, 0.0);   /* :38 */

    for (int round = 0; round < 4; ++round) {              /* simplex.hpp:43-55 */
        double sum = 0.0;
        for (size_t k = 0; k < c; ++k) sum += x[k];
        const double residual = sum - 1.0;
        if (residual == 0.0) break;
        double top = x[0];                                 /* std::max_element */
        for (size_t k = 1; k < c; ++k) if (top < x[k]) top = x[k];
        size_t ties = 0;
        for (size_t k = 0; k < c; ++k) ties += (x[k] == top);
        const double share = residual / (double)ties;
        for (size_t k = 0; k < c; ++k)
            if (x[k] == top) x[k] = ref_max(x[k] - share, 0.0);
    }
    return FCO_OK;
}

/* -------------------------------------------------------- membership.hpp:79-94 */
int fco_init_random(size_t n, size_t c, uint64_t seed, double* x) {
    if (n == 0 || c == 0) return fail(FCO_INVALID, "init_membership: dimensions must be positive");
    uint64_t st = seed;
    for (size_t i = 0; i < n; ++i) {
        double* col = x + i * c;
        for (size_t k = 0; k < c; ++k) col[k] = fco_splitmix_next_double(&st);
        int rc = fco_project_simplex(col, c);
        if (rc) return rc;
    }
    return FCO_OK;
}

/* -------------------------------------------------------- membership.hpp:49-61 */
double fco_feasibility_error(const double* x, size_t c, size_t n) {
    double worst = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double sum = 0.0;
        for (size_t k = 0; k < c; ++k) {
            const double v = x[i * c + k];
            sum += v;
            if (v < 0.0) worst = worst < -v ? -v : worst;            /* std::max(worst, -v) */
            if (v > 1.0) worst = worst < v - 1.0 ? v - 1.0 : worst;
        }
        const double dev = fabs(sum - 1.0);
        worst = worst < dev ? dev : worst;
    }
    return worst;
}

static int validate_membership(const double* x, size_t c, size_t n, double tol) {
    if (c == 0 || n == 0) return fail(FCO_INVALID, "membership: empty matrix");
    for (size_t k = 0; k < c * n; ++k)
        if (!isfinite(x[k])) return fail(FCO_INVALID, "membership: non-finite entry");
    const double err = fco_feasibility_error(x, c, n);
    if (err > tol)
        return fail(FCO_INVALID,
                    "membership: columns violate the simplex constraint by %g (tolerance %g)", err, tol);
    return FCO_OK;
}

/* ----------------------------------------------------------- objective.hpp:61-95 */
void fco_share_matrix(const double* x, size_t c, size_t n, double* g) {
    double* acc = (double*)malloc(c * c * sizeof(double));
    memset(g, 0, c * c * sizeof(double));
    for (size_t begin = 0; begin < n; begin += FCO_BLOCK) {
        const size_t end = begin + FCO_BLOCK < n ? begin + FCO_BLOCK : n;
        memset(acc, 0, c * c * sizeof(double));
        for (size_t i = begin; i < end; ++i) {            /* :72-79 */
            const double* ci = x + i * c;
            for (size_t r = 0; r < c; ++r)
                for (size_t s = 0; s < c; ++s) acc[r * c + s] += ci[r] * ci[s];
        }
        for (size_t k = 0; k < c * c; ++k) g[k] += acc[k]; /* :83-88, ascending blocks */
    }
    free(acc);
}

/* objective.hpp:61-90: A B^T, per-1024-column-block partials summed in ascending order */
void fco_cross_share(const double* a, const double* b, size_t c, size_t n, double* g) {
    double* acc = (double*)malloc(c * c * sizeof(double));
    memset(g, 0, c * c * sizeof(double));
    for (size_t begin = 0; begin < n; begin += FCO_BLOCK) {
        const size_t end = begin + FCO_BLOCK < n ? begin + FCO_BLOCK : n;
        memset(acc, 0, c * c * sizeof(double));
        for (size_t i = begin; i < end; ++i) {
            const double* ca = a + i * c;
            const double* cb = b + i * c;
            for (size_t r = 0; r < c; ++r)
                for (size_t q = 0; q < c; ++q) acc[r * c + q] += ca[r] * cb[q];
        }
        for (size_t k = 0; k < c * c; ++k) g[k] += acc[k];
    }
    free(acc);
}

/* objective.hpp:186-217: column i of -4 V (S - X^T X) + 4 X (V^T X + X^T V), i.e.
 * -4 (V s_i - A x_i - A^T x_i - B v_i) with A = cross_share(V, X), B = share_matrix(X);
 * ShareMatrix::apply / transpose_apply (objective.hpp:37-51) are sequential in l. */
int fco_hessian_vector_product(const double* x, const double* v, size_t c, const fco_csr* s, double* out) {
    const size_t n = (size_t)s->n;
    double* A = (double*)malloc(c * c * sizeof(double));
    double* B = (double*)malloc(c * c * sizeof(double));
    double* vs = (double*)malloc(c * sizeof(double));
    fco_cross_share(v, x, c, n, A);
    fco_share_matrix(x, c, n, B);
    for (size_t i = 0; i < n; ++i) {
        for (size_t k = 0; k < c; ++k) vs[k] = 0.0;             /* similarity_column_product */
        for (int64_t e = s->row_ptr[i]; e < s->row_ptr[i + 1]; ++e) {
            const double* vj = v + (size_t)s->col_idx[e] * c;
            const double w = s->values ? s->values[e] : 1.0;
            for (size_t r = 0; r < c; ++r) vs[r] += w * vj[r];
        }
        const double* xi = x + i * c;
        const double* vi = v + i * c;
        for (size_t k = 0; k < c; ++k) {
            double ax = 0.0, atx = 0.0, bv = 0.0;
            for (size_t l = 0; l < c; ++l) ax += A[k * c + l] * xi[l];
            for (size_t l = 0; l < c; ++l) atx += A[l * c + k] * xi[l];
            for (size_t l = 0; l < c; ++l) bv += B[k * c + l] * vi[l];
            out[i * c + k] = -4.0 * (vs[k] - ax - atx - bv);
        }
    }
    free(A);
    free(B);
    free(vs);
    return FCO_OK;
}

/* dense.hpp:40-46 frob_inner: one sequential sum over the storage order */
double fco_frob_inner(const double* a, const double* b, size_t count) {
    double acc = 0.0;
    for (size_t k = 0; k < count; ++k) acc += a[k] * b[k];
    return acc;
}

/* objective.hpp:25-29 */
double fco_share_frob_sq(const double* g, size_t c) {
    double s = 0.0;
    for (size_t k = 0; k < c * c; ++k) s += g[k] * g[k];
    return s;
}

/* objective.hpp:98-109 + :131-135 + :151-173 */
int fco_fused_column_pass(const double* x, size_t c, const fco_csr* s, double* xs, double* merge) {
    const size_t n = (size_t)s->n;
    double total = 0.0;
    for (size_t begin = 0; begin < n; begin += FCO_BLOCK) {
        const size_t end = begin + FCO_BLOCK < n ? begin + FCO_BLOCK : n;
        double local = 0.0;
        for (size_t i = begin; i < end; ++i) {
            double* out = xs + i * c;
            for (size_t k = 0; k < c; ++k) out[k] = 0.0;
            for (int64_t e = s->row_ptr[i]; e < s->row_ptr[i + 1]; ++e) {
                const double* xj = x + (size_t)s->col_idx[e] * c;
                const double w = s->values ? s->values[e] : 1.0;
                for (size_t r = 0; r < c; ++r) out[r] += w * xj[r];
            }
            double prod = 0.0;                               /* loss_terms_column */
            for (size_t k = 0; k < c; ++k) prod += out[k] * x[i * c + k];
            local += prod;
        }
        total += local;                                      /* :171 */
    }
    *merge = total;
    return FCO_OK;
}

/* objective.hpp:176-180 */
double fco_loss_decomposed(const double* x, size_t c, const fco_csr* s, const double* g) {
    double* xs = (double*)malloc(c * (size_t)s->n * sizeof(double));
    double merge = 0.0;
    fco_fused_column_pass(x, c, s, xs, &merge);
    free(xs);
    return s->frob_sq + fco_share_frob_sq(g, c) - 2.0 * merge;
}

/* objective.hpp:37-43 (ShareMatrix::apply) + :113-118 (gradient_column_fused) */
static void gradient_column(const double* g, size_t c, const double* xs_i, const double* x_i,
                            double* out) {
    for (size_t k = 0; k < c; ++k) {
        double acc = 0.0;
        for (size_t l = 0; l < c; ++l) acc += g[k * c + l] * x_i[l];
        out[k] = acc;
    }
    for (size_t k = 0; k < c; ++k) out[k] = -4.0 * (xs_i[k] - out[k]);
}

/* solver.hpp:89-107 */
int fco_gpa_step_fused(const double* x, size_t c, size_t n, const double* g, const double* xs,
                       double tau, double* out) {
    double* grad = (double*)malloc(c * sizeof(double));
    for (size_t i = 0; i < n; ++i) {
        const double* x_i = x + i * c;
        double* o = out + i * c;
        gradient_column(g, c, xs + i * c, x_i, grad);
        for (size_t k = 0; k < c; ++k) o[k] = x_i[k] - tau * grad[k];
        int rc = fco_project_simplex(o, c);
        if (rc) { free(grad); return rc; }
    }
    free(grad);
    return FCO_OK;
}

/* Backtracking helpers (no reference: parity unpinned).  Same step as
 * gpa_step_fused, plus the sufficient-decrease terms
 *   lin = <grad f(y), p - y>,  sq = ||p - y||^2
 * reduced in the library's fixed order: sequential over k within a column,
 * sequential over columns within a 1024-column block, blocks ascending. */
static int step_with_terms(const double* y, size_t c, size_t n, const double* g, const double* xs,
                           double tau, double* out, double* lin_out, double* sq_out) {
    double* grad = (double*)malloc(c * sizeof(double));
    double lin = 0.0, sq = 0.0;
    for (size_t begin = 0; begin < n; begin += FCO_BLOCK) {
        const size_t end = begin + FCO_BLOCK < n ? begin + FCO_BLOCK : n;
        double lb = 0.0, sb = 0.0;
        for (size_t i = begin; i < end; ++i) {
            const double* y_i = y + i * c;
            double* o = out + i * c;
            gradient_column(g, c, xs + i * c, y_i, grad);
            for (size_t k = 0; k < c; ++k) o[k] = y_i[k] - tau * grad[k];
            int rc = fco_project_simplex(o, c);
            if (rc) { free(grad); return rc; }
            double li = 0.0, si = 0.0;
            for (size_t k = 0; k < c; ++k) {
                const double d = o[k] - y_i[k];
                li += grad[k] * d;
                si += d * d;
            }
            lb += li;
            sb += si;
        }
        lin += lb;
        sq += sb;
    }
    free(grad);
    *lin_out = lin;
    *sq_out = sq;
    return FCO_OK;
}

/* solver.hpp:72 */
double fco_fista_t_next(double t) { return (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0; }

/* solver.hpp:78-81 (frob_norm = sqrt(frob_sq), sparse.hpp:105) */
double fco_default_step_size(const fco_csr* s, size_t n) {
    return 1.0 / (4.0 * sqrt(s->frob_sq) + 12.0 * (double)n);
}

static void push_record(fco_record* trace, uint64_t cap, uint64_t* count, uint64_t it, double loss,
                        int increased, int backtracks, double step) {
    if (*count < cap) {
        trace[*count].iteration = it;
        trace[*count].loss = loss;
        trace[*count].loss_increased = increased;
        trace[*count].backtracks = backtracks;
        trace[*count].step = step;
    }
    ++*count;
}

/* SolverConfig::validate, solver.hpp:40-47 */
static int validate_config(const fco_config* cfg) {
    if (cfg->max_iter < 1) return fail(FCO_INVALID, "solver: max_iter must be >= 1");
    if (cfg->tol < 0.0) return fail(FCO_INVALID, "solver: tol must be >= 0");
    if (cfg->trace_every < 1) return fail(FCO_INVALID, "solver: trace_every must be >= 1");
    if (!(cfg->step_size > 0.0) && cfg->step_size != 0.0)
        return fail(FCO_INVALID, "solver: step_size must be positive (or 0 for auto)");
    if (cfg->method == FCO_FISTA_BT && !(cfg->bt_eta > 1.0))
        return fail(FCO_INVALID, "solver: backtracking eta must be > 1");
    return FCO_OK;
}

/* run_gpa, solver.hpp:137-180 */
static int run_gpa(const fco_csr* s, const fco_config* cfg, size_t c, const double* x0,
                   double* x_out, fco_record* trace, uint64_t cap, fco_summary* out) {
    const size_t n = (size_t)s->n;
    const double tau = cfg->step_size > 0.0 ? cfg->step_size : fco_default_step_size(s, n);
    double* x = x_out;
    double* next = (double*)malloc(c * n * sizeof(double));
    double* xs = (double*)malloc(c * n * sizeof(double));
    double* g = (double*)malloc(c * c * sizeof(double));
    memcpy(x, x0, c * n * sizeof(double));
    uint64_t count = 0;
    out->step_size = tau;
    double loss_prev = (double)n * (double)n;
    int rc = FCO_OK;
    for (uint64_t it = 0;; ++it) {
        double merge;
        fco_share_matrix(x, c, n, g);
        fco_fused_column_pass(x, c, s, xs, &merge);
        const double loss = s->frob_sq + fco_share_frob_sq(g, c) - 2.0 * merge;
        const int increased = it > 0 && loss > loss_prev;
        const int stop_tol = loss_prev - loss <= cfg->tol;
        const int stop_iter = it >= cfg->max_iter;
        if (stop_tol || stop_iter || it % cfg->trace_every == 0)
            push_record(trace, cap, &count, it, loss, increased, 0, tau);
        out->iterations = it;
        out->final_loss = loss;
        if (stop_tol) { out->reason = FCO_TOL_REACHED; break; }
        if (stop_iter) { out->reason = FCO_MAX_ITER; break; }
        rc = fco_gpa_step_fused(x, c, n, g, xs, tau, next);
        if (rc) break;
        memcpy(x, next, c * n * sizeof(double));
        loss_prev = loss;
    }
    out->n_records = count;
    free(next); free(xs); free(g);
    return rc;
}

/* run_fista, solver.hpp:188-272; with cfg->method == FCO_FISTA_BT the fixed
 * step is replaced by Beck-Teboulle backtracking (new; parity unpinned):
 *   L starts at 1/tau_0 and never decreases; at each iteration, while
 *   f(p) > f(y) + <grad f(y), p - y> + (L/2)||p - y||^2 and fewer than bt_max
 *   backtracks were taken, L <- eta*L and p is recomputed. */
static int run_fista(const fco_csr* s, const fco_config* cfg, size_t c, const double* x0,
                     double* x_out, fco_record* trace, uint64_t cap, fco_summary* out) {
    const size_t n = (size_t)s->n;
    const size_t bytes = c * n * sizeof(double);
    const int bt = cfg->method == FCO_FISTA_BT;
    const double tau0 = cfg->step_size > 0.0 ? cfg->step_size : fco_default_step_size(s, n);
    double L = 1.0 / tau0;
    double* bar_prev = (double*)malloc(bytes);
    double* ext = (double*)malloc(bytes);
    double* bar = (double*)malloc(bytes);
    double* xs = (double*)malloc(bytes);
    double* g = (double*)malloc(c * c * sizeof(double));
    double* gb = (double*)malloc(c * c * sizeof(double));
    memcpy(bar_prev, x0, bytes);
    memcpy(ext, x0, bytes);
    uint64_t count = 0;
    out->step_size = tau0;
    int rc = FCO_OK;
    double loss_prev;
    {
        double merge0;
        fco_share_matrix(x0, c, n, g);
        fco_fused_column_pass(x0, c, s, xs, &merge0);
        loss_prev = s->frob_sq + fco_share_frob_sq(g, c) - 2.0 * merge0;
        push_record(trace, cap, &count, 0, loss_prev, 0, 0, tau0);
    }
    memcpy(x_out, x0, bytes);
    out->final_loss = loss_prev;
    out->iterations = 0;
    out->reason = FCO_MAX_ITER;

    double t = 1.0;
    for (uint64_t it = 1; it <= cfg->max_iter; ++it) {
        double merge_y;
        fco_share_matrix(ext, c, n, g);                       /* :218 */
        fco_fused_column_pass(ext, c, s, xs, &merge_y);        /* :219 */
        double loss = 0.0;
        int backtracks = 0;
        double tau = tau0;
        for (;;) {
            double lin = 0.0, sq = 0.0, merge_b;
            tau = bt ? 1.0 / L : tau0;
            rc = bt ? step_with_terms(ext, c, n, g, xs, tau, bar, &lin, &sq)
                    : fco_gpa_step_fused(ext, c, n, g, xs, tau, bar);   /* :220 */
            if (rc) goto done;
            double* xs_b = (double*)malloc(bytes);
            fco_share_matrix(bar, c, n, gb);                   /* :222 */
            fco_fused_column_pass(bar, c, s, xs_b, &merge_b);  /* :223 */
            free(xs_b);
            loss = s->frob_sq + fco_share_frob_sq(gb, c) - 2.0 * merge_b;   /* :224 */
            if (!bt) break;
            const double f_y = s->frob_sq + fco_share_frob_sq(g, c) - 2.0 * merge_y;
            const double q = (f_y + lin) + (0.5 * L) * sq;
            if (loss <= q || (uint32_t)backtracks >= cfg->bt_max) break;
            L = cfg->bt_eta * L;
            ++backtracks;
        }
        const int increased = loss > loss_prev;                 /* :225 */
        const double decrease = loss_prev - loss;
        const int stop_tol = decrease <= cfg->tol && !(increased && cfg->fista_restart);
        const int stop_iter = it >= cfg->max_iter;
        if (stop_tol || stop_iter || it % cfg->trace_every == 0)
            push_record(trace, cap, &count, it, loss, increased, backtracks, tau);
        memcpy(x_out, bar, bytes);                              /* :233 */
        out->iterations = it;
        out->final_loss = loss;
        if (stop_tol) {
            out->reason = increased ? FCO_LOSS_INCREASE_FISTA : FCO_TOL_REACHED;
            goto done;
        }
        if (stop_iter) { out->reason = FCO_MAX_ITER; goto done; }
        if (increased && cfg->fista_restart) {                  /* :247-249 */
            t = 1.0;
            memcpy(ext, bar, bytes);
        } else {                                                /* :251-266 */
            const double t_next = fco_fista_t_next(t);
            const double beta = (t - 1.0) / t_next;
            for (size_t k = 0; k < c * n; ++k) ext[k] = bar[k] + beta * (bar[k] - bar_prev[k]);
            t = t_next;
        }
        { double* tmp = bar_prev; bar_prev = bar; bar = tmp; }  /* :268 */
        loss_prev = loss;
    }
done:
    out->n_records = count;
    free(bar_prev); free(ext); free(bar); free(xs); free(g); free(gb);
    return rc;
}

/* solve, solver.hpp:274-277 (plus validation at :139-143 / :190-195) */
int fco_solve(const fco_csr* s, const fco_config* cfg, size_t c, const double* x0,
              double* x_out, fco_record* trace, uint64_t trace_cap, fco_summary* out) {
    memset(out, 0, sizeof *out);
    int rc = validate_config(cfg);
    if (rc) return rc;
    rc = validate_membership(x0, c, (size_t)s->n, 1e-9);
    if (rc) return rc;
    if (cfg->method == FCO_GPA) return run_gpa(s, cfg, c, x0, x_out, trace, trace_cap, out);
    return run_fista(s, cfg, c, x0, x_out, trace, trace_cap, out);
}
