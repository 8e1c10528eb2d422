// fc_kernels.cuh -- sm_100a kernels of the GPA/FISTA hot path.
//
// Arithmetic contract: IEEE FP64, round-to-nearest, no FMA
// contraction (the whole library is compiled with --fmad=false and the critical
// expressions below use explicit __dmul_rn/__dadd_rn/__dsub_rn), every reduction
// in the reference's fixed order.  The results are therefore bitwise identical to
// the reference CPU solver (/root/reference/proj/include/fuzzyclust).
//
// Layout in HBM:
//   U  : N x C f64 row-major (== the reference's C x N column-major X), node i's
//        C memberships contiguous.  Three full replicas rotate (bar^n, bar^{n-1},
//        bar^{n-2}) for FISTA, two for GPA.
//   S  : CSR (== the reference's CSC, S symmetric) row_ptr i64, col u32, val f64
//        (val absent when every value is 1.0: 1.0*x == x exactly).
//   xs : shard rows x C f64 (S U products), two slots (0 = extrapolated point, 1 = bar).
//   per-1024-row-block partials: Gram (packed upper triangle) and scalar terms.
#pragma once
#include <type_traits>

#include <cstdint>
#include <cuda.h>
#include <climits>
#include <cuda_runtime.h>

namespace fc {

constexpr uint32_t kBlock = 1024;   // parallel.hpp:15 kReductionBlock
constexpr unsigned kFull = 0xffffffffu;

enum : int { kLiteral = 0, kExtrap = 1 };
enum : int { kMatExt = 0, kMatBar = 1 };
// scalar partial / total slots
enum : int { kScalMerge = 0, kScalLin = 1, kScalSq = 2, kScalMergeY = 3, kNumScal = 4 };
enum : int { kFinPrelude = 0, kFinFista = 1, kFinGpa = 2, kFinGranular = 3 };

// Solver state in device memory.  Kernels read the "plan" fields; only
// k_finalize (one thread) writes them, so a whole iteration can be enqueued
// (or graph-replayed) without host round trips.
struct DevState {
    unsigned long long iter;        // iteration whose pass is being computed
    unsigned long long n_records;
    unsigned long long iterations;  // SolverTrace::iterations
    unsigned long long max_iter;
    unsigned long long trace_every;
    unsigned long long trace_cap;
    int done;
    int error;                      // 1: non-finite projection input
    int reason;
    int method;
    int restart;                    // fista_restart
    int bt;                         // backtracking enabled
    int bt_max;
    int backtracks;                 // backtracks taken in the current iteration
    double loss_prev;
    double final_loss;
    double t;                       // FISTA t_n
    double tau;                     // step used by the next k_step
    double tau0;
    double L;                       // backtracking: 1/tau
    double bt_eta;
    double frob_s;                  // ||S||_F^2
    double tol;
    double frob_gy;                 // backtracking: ||G(y)||^2 of the current y
    // plan of the next k_step
    int step_mode;                  // kLiteral | kExtrap
    int step_a;                     // U index of bar^{n-1} (or literal source)
    int step_b;                     // U index of bar^{n-2}
    int step_dst;                   // U index receiving bar^n
    int step_sel;                   // 0: use (G, xs) of the extrapolated point, 1: of bar
    int sw_b;                       // U index of the point swept / Gram'd (bar^n)
    int sw_p;                       // U index of bar^{n-1} (dual pass)
    int result_buf;                 // U index holding result.membership
    double beta_step;               // beta used to rebuild X_ext^n in k_step
    double beta_next;               // beta_n: X_ext^{n+1} = bar^n + beta_n (bar^n - bar^{n-1})
    long long t0_ns;
    int xs_r;                       // xs set read by k_step (S y of the current y)
    int xs_w;                       // xs set written by k_sweep (differs only with backtracking)
    unsigned long long err_bits;    // validation: max feasibility error (as bits)
    unsigned int nonfinite;
    unsigned int pad;
    // tolerance mode (fc_set_parity_mode 1): FISTA's S X_ext by linearity from two S bar sweeps
    int tolmode;
    int xs_a;                       // xs set holding S bar^{n-1} (read by the step of iteration n)
    int xs_b;                       // xs set holding S bar^{n-2}
    int pad_tol;
};

struct TraceRec {                   // == fc_trace_record
    unsigned long long iteration;
    double loss;
    double elapsed_ms;
    int loss_increased;
    int backtracks;
    double step;
};

// Everything a kernel needs, passed by value.  Row-indexed shard arrays (xs,
// prod, rowterm) and block-indexed partials are pre-offset to the shard.
struct Bufs {
    const long long* row_ptr;       // shard-local, rebased (row_ptr[0] == 0)
    const unsigned* col;
    const double* val;              // nullptr => pattern only
    double* U[3];
    double* xs[4];                  // [set*2 + slot]; set = DevState::xs_r / xs_w
    double* prod;                   // per row: <xs_bar_i, bar_i> (or <xs_i, x_i>)
    double* rowterm[3];             // backtracking: lin_i, sq_i, <xs_y_i, y_i>
    double* gpart[2];               // [blk][npairs]
    double* spart;                  // [scal][spart_stride]
    double* totals;                 // [2*npairs + kNumScal]
    double* gfull[2];               // C x C, read as Gt[l*C + r] == G[r][l]
    TraceRec* trace;
    DevState* st;
    unsigned* counter;              // dynamic row scheduler of k_sweep
    const unsigned* heavy;          // shard-local rows of degree >= heavy_deg, by degree descending
    unsigned nheavy;
    unsigned heavy_deg;
    unsigned* hcounter;             // scheduler of the heavy rows
    double* pair;                   // C <= 8 dual sweep: rows [bar^n | bar^{n-1}] interleaved (2C doubles)
};

struct Geo {
    unsigned C;
    unsigned npairs;
    unsigned long long N;
    unsigned long long row0;        // first global row of the shard (multiple of 1024)
    unsigned long long nrows;
    unsigned long long nblk;        // blocks of the shard
    unsigned long long spart_stride;
    unsigned chunk;                 // k_sweep rows per scheduler grab: 32, fewer when N is small
};

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
// acc + a*b: the reference's two roundings (bitwise mode), or one fused rounding (TOL)
template <bool TOL>
__device__ __forceinline__ double madd(double acc, double a, double b) {
    if constexpr (TOL) return __fma_rn(a, b, acc);
    else return __dadd_rn(acc, __dmul_rn(a, b));
}
// std::max(a, b) as the reference uses it: (a < b) ? b : a
__device__ __forceinline__ double ref_max(double a, double b) { return (a < b) ? b : a; }
// FISTA extrapolation, solver.hpp:261: b + beta * (b - p)
__device__ __forceinline__ double extrap(double b, double p, double beta) {
    return dadd(b, dmul(beta, dsub(b, p)));
}
__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// Ampere-style async global->shared copies (no register staging).
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ unsigned long long l2_policy_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_policy_evict_normal() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ldg_hint(const double* p, unsigned long long pol) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
// Column indices carry a "hot row" flag in bit 31 (set by k_flag_hot).
constexpr unsigned kHotBit = 0x80000000u;
constexpr unsigned kIdxMask = 0x7fffffffu;

// Device-side bounds checks of the debug build (-DFC_DEBUG_CHECKS,
// lib/libfuzzyclust_cuda_debug.so; compute-sanitizer is not available on the GPU pool):
// every gathered / scattered row index is checked against its array before use; a failed
// check prints the location and traps (the context reports a device error).
#ifdef FC_DEBUG_CHECKS
#define FC_DCHECK(cond)                                                                    \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("FC_DCHECK failed: %s at %s:%d\n", #cond, __FILE__, __LINE__);          \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define FC_DCHECK(cond) \
    do {                \
    } while (0)
#endif

__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_n() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__host__ __device__ __forceinline__ unsigned pair_index(unsigned r, unsigned s, unsigned C) {
    // packed upper triangle, r <= s, row-major
    return r * C - (r * (r - 1u)) / 2u + (s - r);
}

// =============================================================================
// Per-row simplex projection, lane-parallel within a group of G lanes
// (component r lives in lane r % G, slot r / G).  Follows simplex.hpp:18-59
// operation for operation:
//   sort descending; cumsum; t_k = (cs_k - 1)/(k+1); last k with s_k - t_k >= 0;
//   y = max(y - thr, 0); up to 4 residual folds onto the (tied) maxima.
// sm: G*S doubles of group-private shared scratch.
// Returns false if any entry was non-finite (the reference throws InvalidInput).
// =============================================================================
template <int G, int S>
__device__ __forceinline__ bool project_group(double (&y)[S], int C, int lg, double* sm) {
    const unsigned lane = threadIdx.x & 31u;
    const unsigned gbase = lane & ~(unsigned)(G - 1);
    const unsigned gbits = (G == 32) ? kFull : (((1u << G) - 1u) << gbase);

    __syncwarp();   // sm is reused row after row: finish the previous row's reads
    bool fin = true;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int r = lg + s * G;
        if (r < C && !isfinite(y[s])) fin = false;
    }
    const bool all_fin = (__ballot_sync(kFull, !fin) & gbits) == 0u;
    if (C == 1) {   // uniform across the warp
        if (lg == 0) y[0] = 1.0;
        return all_fin;
    }
    if (!all_fin) {
        // the reference throws; keep this group's lanes convergent with the rest
        // of the warp on harmless values (the caller raises the error flag)
#pragma unroll
        for (int s = 0; s < S; ++s) y[s] = 0.0;
    }

    // rank of each of my components in the descending order (ties by index)
    int rank[S];
#pragma unroll
    for (int s = 0; s < S; ++s) rank[s] = 0;
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) {
#pragma unroll
        for (int l2 = 0; l2 < G; ++l2) {
            const int l = s2 * G + l2;
            const double v = __shfl_sync(kFull, y[s2], l2, G);
            if (l < C) {
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int r = lg + s * G;
                    rank[s] += (v > y[s]) || (v == y[s] && l < r);
                }
            }
        }
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int r = lg + s * G;
        if (r < C) sm[rank[s]] = y[s];
    }
    __syncwarp();

    // cumsum in sorted order (sequential, as the reference) -- each lane-slot
    // keeps the partial sum at the sorted position it owns (k = lg + s*G)
    double mycs[S];
    double cs = 0.0;
    for (int k = 0; k < C; ++k) {
        cs = dadd(cs, sm[k]);
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (k == lg + s * G) mycs[s] = cs;
    }
    double tk[S];
    int best = -1;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int k = lg + s * G;
        bool cond = false;
        tk[s] = 0.0;
        if (k < C) {
            tk[s] = dsub(mycs[s], 1.0) / (double)(k + 1);
            cond = dsub(sm[k], tk[s]) >= 0.0;
        }
        const unsigned bal = (__ballot_sync(kFull, cond) & gbits) >> gbase;
        if (bal) best = max(best, s * G + (31 - __clz(bal)));
    }
    double thr = 0.0;
    if (best >= 0) {
        const int bl = best % G, bs = best / G;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const double v = __shfl_sync(kFull, tk[s], bl, G);
            if (s == bs) thr = v;
        }
    } else {
        // keep the shuffles warp-convergent for other groups of the warp
#pragma unroll
        for (int s = 0; s < S; ++s) (void)__shfl_sync(kFull, tk[s], 0, G);
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int r = lg + s * G;
        if (r < C) y[s] = ref_max(dsub(y[s], thr), 0.0);
    }

    // residual folds (simplex.hpp:43-55)
    bool live = true;
    for (int round = 0; round < 4; ++round) {
        double sum = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2) {
#pragma unroll
            for (int l2 = 0; l2 < G; ++l2) {
                const double v = __shfl_sync(kFull, y[s2], l2, G);
                if (s2 * G + l2 < C) sum = dadd(sum, v);
            }
        }
        const double residual = dsub(sum, 1.0);
        if (residual == 0.0) live = false;
        double top = -INFINITY;
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (lg + s * G < C) top = (top < y[s]) ? y[s] : top;
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            const double v = __shfl_xor_sync(kFull, top, o, G);
            top = (top < v) ? v : top;
        }
        int ties = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const bool eq = (lg + s * G < C) && (y[s] == top);
            ties += __popc(__ballot_sync(kFull, eq) & gbits);
        }
        if (!__any_sync(kFull, live)) break;
        if (live) {
            const double share = residual / (double)ties;
#pragma unroll
            for (int s = 0; s < S; ++s)
                if (lg + s * G < C && y[s] == top) y[s] = ref_max(dsub(y[s], share), 0.0);
        }
    }
    return all_fin;
}

// Sequential (index-order) sum over a group's components of a[]:
//   p = 0; p += a_0; p += a_1; ...  (loss_terms_column, objective.hpp:131-135)
template <int G, int S>
__device__ __forceinline__ double group_seq_sum(const double (&a)[S], int C) {
    double p = 0.0;
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) {
#pragma unroll
        for (int l2 = 0; l2 < G; ++l2) {
            const double v = __shfl_sync(kFull, a[s2], l2, G);
            if (s2 * G + l2 < C) p = dadd(p, v);
        }
    }
    return p;
}

// Same, restricted to one group's lanes (group-divergent code paths).
template <int G, int S>
__device__ __forceinline__ double group_seq_sum_m(const double (&a)[S], int C, unsigned gmask) {
    double p = 0.0;
#pragma unroll
    for (int s2 = 0; s2 < S; ++s2) {
#pragma unroll
        for (int l2 = 0; l2 < G; ++l2) {
            const double v = __shfl_sync(gmask, a[s2], l2, G);
            if (s2 * G + l2 < C) p = dadd(p, v);
        }
    }
    return p;
}

// =============================================================================
// K1: CSR SpMM sweep with the loss-term epilogue.
//   xs_i[r] = sum_{k in row i, ascending} w_k * X[j_k][r]      (objective.hpp:98-109)
//   prod_i  = sum_r xs_i[r] * x_i[r]                            (objective.hpp:131-135)
// DUAL (the FISTA single-sweep schedule): one pass over
// the CSR gathers bar^n_j and bar^{n-1}_j and accumulates both
//   S bar^n                and   S X_ext^{n+1},  X_ext^{n+1}_j = bar_j + beta (bar_j - prev_j)
// where each X_ext entry is formed exactly as solver.hpp:261 forms it, so both
// sums are bit-identical to the reference's two separate sweeps.
// Work: groups of G lanes own a row (lane = component); warps pull 32-row
// chunks from a counter (power-law rows balance dynamically).  The lane that
// loads a column index pre-multiplies it by C (32-bit element offset, host
// guarantees N*C < 2^32) and shuffles the offset; full G-wide index chunks
// take a predicate-free path with U gathers (x2 when DUAL) in flight per lane.
// EXACT: C == G*S (no idle lanes).
// =============================================================================
// Gathers in flight per lane per batch (x2 when DUAL): measured at config C
// (C=32) 16 -> 36.7 ms vs 8 -> 38.8 ms per sweep; C=16 (config B) prefers 8.
#ifndef FC_SWEEP16_MINB
#define FC_SWEEP16_MINB 4
#endif
template <int G, int S = 1>
struct SweepTune {
    static constexpr int U = G == 32 ? (16 / S > 2 ? 16 / S : 2) : (G < 8 ? G : 8);
    static constexpr int MINB = G == 32 ? (S == 1 ? 3 : 2) : (G == 16 ? FC_SWEEP16_MINB : 4);   // CTAs per SM
};

// Single-gather sweeps (GPA, prelude, tolerance-mode FISTA) gather one operand and keep
// half the dual sweep's loads in flight.  -DFC_SWEEP1_WIDE=1 gives them 2U at 2 CTAs per
// SM: measured slower (tolerance-mode C sweep 19.7 vs 16.7-17.5 ms), so off.
#ifndef FC_SWEEP1_WIDE
#define FC_SWEEP1_WIDE 0
#endif
template <int G, int S, bool DUAL>
struct SweepTuneD {
    static constexpr bool WIDE = !DUAL && G == 32 && FC_SWEEP1_WIDE;
    static constexpr int U = WIDE ? 2 * SweepTune<G, S>::U : SweepTune<G, S>::U;
    static constexpr int MINB = WIDE ? 2 : SweepTune<G, S>::MINB;
};

template <int G, int S, bool DUAL, bool W, bool EXACT>
__device__ __forceinline__ void sweep_chunk(const double* __restrict__ B, const double* __restrict__ P, double beta,
                                            unsigned myidx, double myw, int cnt, unsigned gmask, unsigned lg,
                                            unsigned C, double (&ab)[S], double (&ae)[S], unsigned long long pol_hot,
                                            unsigned long long pol_cold, unsigned long long N) {
    constexpr int U = SweepTuneD<G, S, DUAL>::U;
    if (cnt == G) {
#pragma unroll
        for (int k0 = 0; k0 < G; k0 += U) {
            double vb[U][S];
            double vp[DUAL ? U : 1][S];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned raw = __shfl_sync(gmask, myidx, k0 + u, G);
                const unsigned o = (raw & kIdxMask) * C;
                const unsigned long long pol = (raw & kHotBit) ? pol_hot : pol_cold;
                FC_DCHECK((raw & kIdxMask) < N);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const bool okc = EXACT || lg + s * G < C;
                    vb[u][s] = okc ? ldg_hint(B + o + s * G, pol) : 0.0;
                    if (DUAL) vp[u][s] = okc ? ldg_hint(P + o + s * G, pol) : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double w = W ? __shfl_sync(gmask, myw, k0 + u, G) : 1.0;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    ab[s] = W ? dadd(ab[s], dmul(w, vb[u][s])) : dadd(ab[s], vb[u][s]);
                    if (DUAL) {
                        const double e = extrap(vb[u][s], vp[u][s], beta);
                        ae[s] = W ? dadd(ae[s], dmul(w, e)) : dadd(ae[s], e);
                    }
                }
            }
        }
    } else {
        for (int k0 = 0; k0 < cnt; k0 += U) {
            double vb[U][S];
            double vp[DUAL ? U : 1][S];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const unsigned raw = __shfl_sync(gmask, myidx, k0 + u, G);
                const unsigned o = (raw & kIdxMask) * C;
                const unsigned long long pol = (raw & kHotBit) ? pol_hot : pol_cold;
                const bool ok = k0 + u < cnt;
                FC_DCHECK(!ok || (raw & kIdxMask) < N);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const bool okc = ok && (EXACT || lg + s * G < C);
                    vb[u][s] = okc ? ldg_hint(B + o + s * G, pol) : 0.0;
                    if (DUAL) vp[u][s] = okc ? ldg_hint(P + o + s * G, pol) : 0.0;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double w = W ? __shfl_sync(gmask, myw, k0 + u, G) : 1.0;
                if (k0 + u < cnt) {
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        ab[s] = W ? dadd(ab[s], dmul(w, vb[u][s])) : dadd(ab[s], vb[u][s]);
                        if (DUAL) {
                            const double e = extrap(vb[u][s], vp[u][s], beta);
                            ae[s] = W ? dadd(ae[s], dmul(w, e)) : dadd(ae[s], e);
                        }
                    }
                }
            }
        }
    }
}

// Work decomposition: warps pull 32-row chunks from a counter; inside a chunk
// each G-lane group owns a strip of G consecutive rows, i.e. one contiguous
// stretch of the CSR.  The group walks that stretch in G-wide index chunks and
// prefetches the NEXT chunk's column offsets (same row or the next row) before
// gathering the current one, so no row waits on its index load.
// Heavy rows (G == 32, degree >= b.heavy_deg; b.heavy lists them by degree,
// descending) are handed out FIRST, one per warp, and skipped by the strips:
// a power-law hub (114k entries at config C) is one sequential chain per
// component, and started late it would set the kernel's tail.
template <int G, int S, bool DUAL, bool W, bool EXACT>
__global__ void __launch_bounds__(256, SweepTuneD<G, S, DUAL>::MINB) k_sweep(Bufs b, Geo g) {
    const DevState* st = b.st;
    if (st->done) return;
    const unsigned kChunk = g.chunk;                        // rows per counter grab (<= 32)
    const unsigned C = g.C;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned lg = lane % G;
    const unsigned sub = lane / G;
    const unsigned gmask = (G == 32) ? kFull : (((1u << G) - 1u) << (sub * G));
    const double* __restrict__ B = b.U[st->sw_b] + lg;
    const double* __restrict__ P = DUAL ? b.U[st->sw_p] + lg : nullptr;
    const double beta = st->beta_next;
    double* xs_main = (DUAL ? b.xs[st->xs_w * 2 + kMatBar] : b.xs[st->xs_w * 2 + kMatExt]) + lg;
    double* xs_ext = b.xs[st->xs_w * 2 + kMatExt] + lg;
    const unsigned long long pol_hot = l2_policy_evict_last();
    const unsigned long long pol_cold = l2_policy_evict_normal();
    constexpr bool kHeavy = G == 32;                         // heavy-row phase: full-warp groups only
    const long long heavy_deg = (kHeavy && b.nheavy) ? (long long)b.heavy_deg : LLONG_MAX;

    // rows [rb, rb + nrow) of the shard; rows of degree >= tdeg are skipped
    auto strip = [&](unsigned long long rb, unsigned nrow, long long tdeg) {
        const long long myrp = __ldg(b.row_ptr + rb + min(lg, nrow));
        const long long e_hi = __ldg(b.row_ptr + rb + nrow);
        unsigned skip = 0;
        if (kHeavy && tdeg != LLONG_MAX) {
            const long long nb = __shfl_down_sync(gmask, myrp, 1, G);
            const long long d = ((lg + 1 < (unsigned)G) ? nb : e_hi) - myrp;
            skip = (__ballot_sync(gmask, lg < nrow && d >= tdeg) >> (sub * G)) & (G == 32 ? kFull : ((1u << G) - 1u));
        }
        long long e = __shfl_sync(gmask, myrp, 0, G);
        unsigned nxt_idx = 0;                                // raw index: multiplied at use, so the
        double nxt_w = 1.0;                                  // prefetch never waits on its load
        bool stale = true;
        for (unsigned j = 0; j < nrow; ++j) {
            const long long e0 = e;
            const long long e1 = (j + 1 < (unsigned)G) ? __shfl_sync(gmask, myrp, j + 1, G) : e_hi;
            if (kHeavy && ((skip >> j) & 1u)) {              // heavy row: done in the first phase
                e = e1;
                stale = true;
                continue;
            }
            if (stale) {
                nxt_idx = 0;
                if (e0 + lg < e_hi) {
                    nxt_idx = __ldg(b.col + e0 + lg);
                    if (W) nxt_w = ldg(b.val + e0 + lg);
                }
                stale = false;
            }
            const unsigned long long row = rb + j;
            const size_t own = (size_t)(g.row0 + row) * C;
            double xi[S];
#pragma unroll
            for (int s = 0; s < S; ++s) xi[s] = (EXACT || lg + s * G < C) ? ldg(B + own + s * G) : 0.0;
            double ab[S], ae[S];
#pragma unroll
            for (int s = 0; s < S; ++s) { ab[s] = 0.0; ae[s] = 0.0; }
            for (long long eb = e0; eb < e1; eb += G) {
                const unsigned myidx = nxt_idx;
                const double myw = nxt_w;
                const int cnt = (int)min((long long)G, e1 - eb);
                const long long pn = eb + cnt;               // next chunk: this row or the next one
                if (pn + lg < e_hi) {
                    nxt_idx = __ldg(b.col + pn + lg);
                    if (W) nxt_w = ldg(b.val + pn + lg);
                }
                sweep_chunk<G, S, DUAL, W, EXACT>(B, P, beta, myidx, myw, cnt, gmask, lg, C, ab, ae, pol_hot, pol_cold, g.N);
            }
            e = e1;
            double a[S];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                a[s] = dmul(ab[s], xi[s]);
                if (EXACT || lg + s * G < C) {
                    xs_main[(size_t)row * C + s * G] = ab[s];
                    if (DUAL) xs_ext[(size_t)row * C + s * G] = ae[s];
                }
            }
            const double pr = group_seq_sum_m<G, S>(a, (int)C, gmask);
            if (lg == 0) b.prod[row] = pr;
        }
    };

    // one call site (a second inlined copy of strip() costs registers): heavy rows
    // first, longest first, then the 32-row chunks
    bool heavy_phase = kHeavy && heavy_deg != LLONG_MAX;
    for (;;) {
        unsigned long long rb;
        unsigned nrow;
        long long tdeg;
        if (heavy_phase) {
            unsigned h = 0;
            if (lane == 0) h = atomicAdd(b.hcounter, 1u);
            h = __shfl_sync(kFull, h, 0);
            if (h >= b.nheavy) {
                heavy_phase = false;
                continue;
            }
            rb = b.heavy[h];
            nrow = 1;
            tdeg = LLONG_MAX;
        } else {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(b.counter, kChunk);
            base = __shfl_sync(kFull, base, 0);
            if (base >= g.nrows) break;
            const unsigned nr = (unsigned)min((unsigned long long)kChunk, g.nrows - base);
            const unsigned r_lo = sub * G;                   // this group's strip [r_lo, r_hi)
            if (r_lo >= nr) continue;                        // group-divergent from here on
            rb = base + r_lo;
            nrow = min((unsigned)G, nr - r_lo);
            tdeg = heavy_deg;
        }
        strip(rb, nrow, tdeg);
    }
}

// ---- TMA bulk-copy helpers (sm_90+/sm_100a) ------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int r0, int r1, int r2, int r3,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"(smem_u32(bar))
        : "memory");
}

// Tensor maps of the three U replicas (2-D [N][C] f64, box {C, 1}: one
// tile::gather4 lands 4 whole rows).
struct UMaps {
    CUtensorMap m[3];
};

// =============================================================================
// K1 (TMA gather4 variant) for C in (16, 256], C % 4 == 0, pattern-only S: the same
// sums in the same order as k_sweep, with the gathered rows brought in by the
// Blackwell TMA row gather (cp.async.bulk.tensor...tile::gather4).  A warp owns
// a 32-row chunk (one contiguous stretch of the CSR) and walks its nonzeros in
// chunks of Q (multiple of 4); for each chunk lane 0 issues Q/4 gather4s per
// operand (bar^n, bar^{n-1}) into a kSwStages-deep shared-memory ring completed
// on per-stage mbarriers.  The next kSwStages-1 chunks stay in flight while the
// current one is accumulated (lane = component; conflict-free reads),
// independent of row boundaries; rows are flushed (xs stores, prod_i) as the
// stream crosses them.  Selected with FC_SWEEP=tma.  Measured on B200 at config C
// (n=1e7, k=32): 80 ms per sweep vs 38 ms for the LDG-gather k_sweep -- TMA row
// gathers of 256-B rows sustain only ~2.5 TB/s here -- so LDG stays the default.
// =============================================================================
constexpr int kSwTmaThreads = 128;
constexpr int kSwStages = 3;

__host__ __device__ inline int sweep_tma_q(int C) {
    int q = 8192 / (16 * C);                // ~8 KB of (bar, prev) rows per stage
    q = q < 4 ? 4 : (q > 16 ? 16 : q);
    return q & ~3;
}
__host__ __device__ inline size_t sweep_tma_stage_bytes(int C, int dual) {
    return (size_t)sweep_tma_q(C) * 8 * C * (dual ? 2 : 1);
}
__host__ __device__ inline size_t sweep_tma_smem(int C, int dual) {
    return (kSwTmaThreads / 32) * (kSwStages * sweep_tma_stage_bytes(C, dual) + kSwStages * 8) + 128;
}

template <int S, bool DUAL>
__global__ void __launch_bounds__(kSwTmaThreads) k_sweep_tma(Bufs b, Geo g, const __grid_constant__ UMaps maps) {
    const DevState* st = b.st;
    if (st->done) return;
    extern __shared__ __align__(1024) unsigned char sw_raw[];
    constexpr unsigned kChunk = 32;
    const int C = (int)g.C;
    const int Q = sweep_tma_q(C);
    const unsigned rowbytes = 8u * (unsigned)C;
    const size_t stage_bytes = sweep_tma_stage_bytes(C, DUAL);
    const unsigned lane = threadIdx.x & 31u;
    const int warp = threadIdx.x >> 5;
    unsigned char* wbuf = sw_raw + (size_t)warp * kSwStages * stage_bytes;
    unsigned long long* bars =
        reinterpret_cast<unsigned long long*>(sw_raw + (size_t)(kSwTmaThreads / 32) * kSwStages * stage_bytes) +
        warp * kSwStages;
    if (lane == 0)
        for (int k = 0; k < kSwStages; ++k) mbar_init(bars + k, 1);
    mbar_fence_init();
    __syncwarp();
    unsigned phases = 0;                                   // bit k: parity of stage k's next completion
    const CUtensorMap* mapB = &maps.m[st->sw_b];
    const CUtensorMap* mapP = &maps.m[st->sw_p];

    const double* __restrict__ Bg = b.U[st->sw_b];
    const double beta = st->beta_next;
    double* xs_main = DUAL ? b.xs[st->xs_w * 2 + kMatBar] : b.xs[st->xs_w * 2 + kMatExt];
    double* xs_ext = b.xs[st->xs_w * 2 + kMatExt];

    for (;;) {
        unsigned base = 0;
        if (lane == 0) base = atomicAdd(b.counter, kChunk);
        base = __shfl_sync(kFull, base, 0);
        if (base >= g.nrows) break;
        const unsigned nr = (unsigned)min((unsigned long long)kChunk, g.nrows - base);
        const long long myrp = __ldg(b.row_ptr + base + min(lane, nr));
        const long long e_hi = __ldg(b.row_ptr + base + nr);
        const long long e_lo = __shfl_sync(kFull, myrp, 0);
        const long long nchunks = (e_hi - e_lo + Q - 1) / Q;

        long long next_issue = 0;
        int idx_pf = 0;                                    // prefetched column index (lane k < Q)
        if ((long long)lane < (long long)Q && e_lo + lane < e_hi) idx_pf = (int)(__ldg(b.col + e_lo + lane) & kIdxMask);
        auto issue = [&](long long c) {
            const int sidx = (int)(c % kSwStages);
            const long long p0 = e_lo + c * Q;
            const int cnt = (int)min((long long)Q, e_hi - p0);
            int idx = idx_pf;
            const long long pn = p0 + Q;
            if ((long long)lane < (long long)Q && pn + lane < e_hi) idx_pf = (int)(__ldg(b.col + pn + lane) & kIdxMask);
            const int last = __shfl_sync(kFull, idx, cnt - 1);
            if ((int)lane >= cnt) idx = last;              // pad a partial gather4 with a valid row
            const int ng = (cnt + 3) >> 2;
            unsigned char* sb = wbuf + (size_t)sidx * stage_bytes;
            if (lane == 0) mbar_expect_tx(bars + sidx, (unsigned)ng * 4u * rowbytes * (DUAL ? 2u : 1u));
            for (int q = 0; q < ng; ++q) {
                const int r0 = __shfl_sync(kFull, idx, 4 * q), r1 = __shfl_sync(kFull, idx, 4 * q + 1);
                const int r2 = __shfl_sync(kFull, idx, 4 * q + 2), r3 = __shfl_sync(kFull, idx, 4 * q + 3);
                if (lane == 0) {
                    tma_gather4(sb + (size_t)4 * q * rowbytes, mapB, r0, r1, r2, r3, bars + sidx);
                    if (DUAL) tma_gather4(sb + (size_t)(Q + 4 * q) * rowbytes, mapP, r0, r1, r2, r3, bars + sidx);
                }
            }
        };
        for (; next_issue < nchunks && next_issue < kSwStages; ++next_issue) issue(next_issue);

        unsigned j = 0;                                    // current row of the chunk
        long long row_end = (nr > 1) ? __shfl_sync(kFull, myrp, 1) : e_hi;
        double xi[S], ab[S], ae[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int r = (int)lane + 32 * s;
            xi[s] = (r < C) ? ldg(Bg + (size_t)(g.row0 + base) * C + r) : 0.0;
            ab[s] = 0.0;
            ae[s] = 0.0;
        }
        for (long long c = 0;; ++c) {
            const bool have = c < nchunks;
            const int sidx = (int)(c % kSwStages);
            long long p0 = e_hi;
            int cnt = 0;
            if (have) {
                mbar_wait(bars + sidx, (phases >> sidx) & 1u);
                phases ^= 1u << sidx;
                p0 = e_lo + c * Q;
                cnt = (int)min((long long)Q, e_hi - p0);
            }
            const double* sbar = reinterpret_cast<const double*>(wbuf + (size_t)sidx * stage_bytes);
            const double* sprev = sbar + (size_t)Q * C;
            for (int k = 0; k <= cnt; ++k) {
                // flush every row that ends at stream position p0 + k (incl. empty rows)
                while (j < nr && p0 + k == row_end && (k < cnt || !have)) {
                    const unsigned long long row = base + j;
                    double a[S];
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const int r = (int)lane + 32 * s;
                        a[s] = dmul(ab[s], xi[s]);
                        if (r < C) {
                            xs_main[(size_t)row * C + r] = ab[s];
                            if (DUAL) xs_ext[(size_t)row * C + r] = ae[s];
                        }
                    }
                    const double pr = group_seq_sum<32, S>(a, C);
                    if (lane == 0) b.prod[row] = pr;
                    ++j;
                    const long long nxt = __shfl_sync(kFull, myrp, (j + 1) & 31u);
                    row_end = (j + 1 < nr) ? nxt : e_hi;
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const int r = (int)lane + 32 * s;
                        xi[s] = (r < C && j < nr) ? ldg(Bg + (size_t)(g.row0 + base + j) * C + r) : 0.0;
                        ab[s] = 0.0;
                        ae[s] = 0.0;
                    }
                }
                if (k == cnt) break;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int r = (int)lane + 32 * s;
                    if (r < C) {
                        const double vb = sbar[k * C + r];
                        ab[s] = dadd(ab[s], vb);
                        if (DUAL) ae[s] = dadd(ae[s], extrap(vb, sprev[k * C + r], beta));
                    }
                }
            }
            if (!have) break;
            __syncwarp();
            if (next_issue < nchunks) {
                fence_proxy_async();                       // generic reads of this stage precede the refill
                issue(next_issue);
                ++next_issue;
            }
        }
    }
}

// =============================================================================
// K1 for C <= G <= 16: one row per warp at a time; lane = (nonzero slot q,
// component c) with Q = 32/G slots, so one load instruction gathers Q
// neighbour rows of the same row i.  The values are then shuffled to the
// q = 0 lanes in ascending nonzero order and accumulated sequentially there
// (the reference's order), keeping the warp converged (no per-group row loops).
// A warp owns a 32-row chunk and walks its rows in order; column indices of the
// next 32 nonzeros are prefetched.
// =============================================================================
struct NoLightChunk {
    __device__ void operator()(unsigned long long, unsigned) const {}
};

// MODE 0: heavy rows, then every chunk through strip(); MODE 2: chunks without a heavy
// row go to light(base, nr) instead (k_sweep_async)
template <int G, bool DUAL, bool W, bool PAIR, int MODE = 0, class Light = NoLightChunk>
__device__ __forceinline__ void k_sweep_small_body(Bufs& b, Geo& g, Light light = Light()) {
    const DevState* st = b.st;
    if (st->done) return;

    const unsigned kChunk = g.chunk;                        // rows per counter grab (<= 32)
    constexpr int Q = 32 / G;                 // nonzeros per load instruction
    constexpr int U = (32 / Q) < 8 ? (32 / Q) : 8;  // loads per lane in flight per batch (x2 DUAL)
    const unsigned C = g.C;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned c = lane % G, q = lane / G;
    const bool okc = c < C;
    const double* __restrict__ B = b.U[st->sw_b] + c;
    const double* __restrict__ P = DUAL ? b.U[st->sw_p] + c : nullptr;
    const double beta = st->beta_next;
    double* xs_main = (DUAL ? b.xs[st->xs_w * 2 + kMatBar] : b.xs[st->xs_w * 2 + kMatExt]) + c;
    double* xs_ext = b.xs[st->xs_w * 2 + kMatExt] + c;

    const long long heavy_deg = b.nheavy ? (long long)b.heavy_deg : LLONG_MAX;
    // rows [base, base + nr); rows of degree >= tdeg were done in the heavy phase
    auto strip = [&](unsigned long long base, unsigned nr, long long tdeg) {
        const long long myrp = __ldg(b.row_ptr + base + min(lane, nr));
        const long long e_hi = __ldg(b.row_ptr + base + nr);
        unsigned skip = 0;
        if (tdeg != LLONG_MAX) {
            const long long nb = __shfl_down_sync(kFull, myrp, 1);
            const long long d = ((lane + 1 < 32u) ? nb : e_hi) - myrp;
            skip = __ballot_sync(kFull, lane < nr && d >= tdeg);
        }
        long long e = __shfl_sync(kFull, myrp, 0);
        unsigned nxt = 0;
        double nxtw = 1.0;
        bool stale = true;
        for (unsigned j = 0; j < nr; ++j) {
            const long long e0 = e;
            const long long e1 = (j + 1 < 32u) ? __shfl_sync(kFull, myrp, (j + 1) & 31u) : e_hi;
            if ((skip >> j) & 1u) {
                e = e1;
                stale = true;
                continue;
            }
            if (stale) {
                nxt = 0;
                if (e0 + lane < e_hi) {
                    nxt = __ldg(b.col + e0 + lane);
                    if (W) nxtw = ldg(b.val + e0 + lane);
                }
                stale = false;
            }
            const unsigned long long row = base + j;
            const double xi = okc ? ldg(B + (size_t)(g.row0 + row) * C) : 0.0;
            double ab = 0.0, ae = 0.0;
            for (long long eb = e0; eb < e1; eb += 32) {
                const unsigned myidx = nxt;
                const double myw = nxtw;
                const int cnt = (int)min(32LL, e1 - eb);
                const long long pn = eb + cnt;
                if (pn + lane < e_hi) {
                    nxt = __ldg(b.col + pn + lane);
                    if (W) nxtw = ldg(b.val + pn + lane);
                }
                if constexpr (PAIR) {
                    // 2G lanes per neighbour: lane cp < G reads bar component cp, lane G + cp the
                    // prev component cp of the same interleaved row; bar lanes pull prev by shuffle
                    constexpr int GP = 2 * G, QP = 32 / GP, UP = U;
                    const unsigned qp = lane / GP, cp = lane % GP;
                    const bool okp = (cp % G) < C;
                    const unsigned poff = cp < (unsigned)G ? cp : C + (cp - G);
                    for (int t0 = 0; t0 < cnt; t0 += QP * UP) {
                        double vb[UP], ve[UP];
#pragma unroll
                        for (int u = 0; u < UP; ++u) {
                            const int k = t0 + u * QP + (int)qp;
                            const unsigned raw = __shfl_sync(kFull, myidx, k & 31);
                            const double w = W ? __shfl_sync(kFull, myw, k & 31) : 1.0;
                            const bool ok = k < cnt && okp;
                            FC_DCHECK(!ok || (raw & kIdxMask) < g.N);
                            const double v = ok ? ldg(b.pair + (size_t)(raw & kIdxMask) * (2 * C) + poff) : 0.0;
                            const double pv = __shfl_down_sync(kFull, v, G);
                            const double ev = extrap(v, pv, beta);
                            ve[u] = ok ? (W ? dmul(w, ev) : ev) : -0.0;     // -0.0: exact no-op addend
                            vb[u] = ok ? (W ? dmul(w, v) : v) : -0.0;
                        }
#pragma unroll
                        for (int u = 0; u < UP; ++u) {
#pragma unroll
                            for (int qq = 0; qq < QP; ++qq) {
                                ab = dadd(ab, __shfl_sync(kFull, vb[u], qq * GP + c));
                                ae = dadd(ae, __shfl_sync(kFull, ve[u], qq * GP + c));
                            }
                        }
                    }
                } else {
                // one batch = UU load slots per lane = Q * UU nonzeros; a row's last batch
                // shrinks to the half / quarter batch that covers its remainder (fewer
                // padded slots: shuffles and adds are per slot, not per nonzero)
                auto batch = [&](auto uc, const int t0) {
                    constexpr int UU = decltype(uc)::value;
                    double vb[UU], ve[DUAL ? UU : 1];
#pragma unroll
                    for (int u = 0; u < UU; ++u) {
                        const int k = t0 + u * Q + (int)q;           // this lane's nonzero slot
                        const unsigned raw = __shfl_sync(kFull, myidx, k & 31);
                        const double w = W ? __shfl_sync(kFull, myw, k & 31) : 1.0;
                        const bool ok = k < cnt && okc;
                        const unsigned o = (raw & kIdxMask) * C;
                        FC_DCHECK(!ok || (raw & kIdxMask) < g.N);
                        const double bv = ok ? ldg(B + o) : 0.0;
                        if (DUAL) {
                            const double pv = ok ? ldg(P + o) : 0.0;
                            const double ev = extrap(bv, pv, beta);
                            ve[u] = ok ? (W ? dmul(w, ev) : ev) : -0.0;
                        }
                        vb[u] = ok ? (W ? dmul(w, bv) : bv) : -0.0;
                    }
                    // slots past the row's end hold -0.0, and x + (-0.0) == x for every x in
                    // round-to-nearest (+0 + -0 = +0, -0 + -0 = -0): the additions are
                    // unconditional (no per-slot select) and the chains stay bitwise
#pragma unroll
                    for (int u = 0; u < UU; ++u) {
#pragma unroll
                        for (int qq = 0; qq < Q; ++qq) {
                            const double bb = __shfl_sync(kFull, vb[u], qq * G + c);
                            ab = dadd(ab, bb);
                            if (DUAL) {
                                const double ee = __shfl_sync(kFull, ve[u], qq * G + c);
                                ae = dadd(ae, ee);
                            }
                        }
                    }
                };
                int t0 = 0;
                for (; cnt - t0 > Q * U / 2; t0 += Q * U) batch(std::integral_constant<int, U>{}, t0);
                if (t0 < cnt) {
                    if constexpr (U >= 4) {
                        if (cnt - t0 > Q * U / 4) batch(std::integral_constant<int, U / 2>{}, t0);
                        else batch(std::integral_constant<int, U / 4>{}, t0);
                    } else if constexpr (U == 2) {
                        batch(std::integral_constant<int, 1>{}, t0);
                    } else {
                        batch(std::integral_constant<int, U>{}, t0);
                    }
                }
                }
            }
            e = e1;
            // flush row (q = 0 lanes hold the sums; every lane computed the same chain)
            if (q == 0 && okc) {
                xs_main[(size_t)row * C] = ab;
                if (DUAL) xs_ext[(size_t)row * C] = ae;
            }
            const double a1[1] = {dmul(ab, xi)};
            const double pr = group_seq_sum<G, 1>(a1, (int)C);
            if (lane == 0) b.prod[row] = pr;
        }
    };
    bool heavy_phase = heavy_deg != LLONG_MAX;              // heavy rows first, longest first
    for (;;) {
        unsigned long long rb;
        unsigned nrow;
        long long tdeg;
        if (heavy_phase) {
            unsigned h = 0;
            if (lane == 0) h = atomicAdd(b.hcounter, 1u);
            h = __shfl_sync(kFull, h, 0);
            if (h >= b.nheavy) {
                heavy_phase = false;
                continue;
            }
            rb = b.heavy[h];
            nrow = 1;
            tdeg = LLONG_MAX;
        } else {
            unsigned base = 0;
            if (lane == 0) base = atomicAdd(b.counter, kChunk);
            base = __shfl_sync(kFull, base, 0);
            if (base >= g.nrows) break;
            rb = base;
            nrow = (unsigned)min((unsigned long long)kChunk, g.nrows - base);
            tdeg = heavy_deg;
            if (MODE == 2) {
                bool hv = false;
                if (tdeg != LLONG_MAX) {
                    const long long a0 = __ldg(b.row_ptr + rb + min(lane, nrow));
                    const long long a1 = __ldg(b.row_ptr + rb + min(lane + 1, nrow));
                    hv = __any_sync(kFull, a1 - a0 >= tdeg);
                }
                if (!hv) {
                    light(rb, nrow);
                    continue;
                }
            }
        }
        strip(rb, nrow, tdeg);
    }
}

template <int G, bool DUAL, bool W>
__global__ void __launch_bounds__(256, 4) k_sweep_small(Bufs b, Geo g) {
    k_sweep_small_body<G, DUAL, W, false>(b, g);
}

// PAIR (dual, C <= 8): the neighbours' bar and prev rows are read as ONE interleaved row
// [bar | prev] of 2C doubles from b.pair (k_pair_pack): 2G lanes per neighbour, one
// 8C..16C-byte contiguous segment per neighbour instead of two half-size ones -- a
// random-gather microbenchmark at E8 size measured 3.15 vs 5.76 ms
// (scripts/gather_ceiling_c8_pair.cu).  Same values, same summation order.
template <int G, bool W>
__global__ void __launch_bounds__(256, 4) k_sweep_small_pair(Bufs b, Geo g) {
    k_sweep_small_body<G, true, W, true>(b, g);
}

// =============================================================================
// K1 async-copy variant (dual, C <= G <= 8, PAIR layout).  k_sweep_small's
// gathers are register-staged (every nonzero in flight holds registers in 8-16
// lanes) and its per-slot value shuffles + padded row tails cost ~32 warp
// instructions per nonzero (ncu, E8).  Here G lanes form a group (lane =
// component), each group owns G consecutive rows of the warp's 32-row chunk
// and walks their nonzeros as ONE flat stream, staged through a shared-memory
// ring with cp.async: S stages of U interleaved [bar | prev] rows (lane c
// copies bytes [16c, 16c+16) of each 16C-byte row), the column indices copied
// S stages ahead of the values, so S-1 stages are in flight per group without
// holding registers and without an index load on the issue path.  The groups
// of a warp advance in lockstep (warp-uniform stage loop; a group past its
// stream is predicated off; row flushes under __any_sync), so the warp never
// serialises divergent groups.  Per row: the same chains ab = sum w*bar,
// ae = sum w*extrap(bar, prev) from 0.0 in CSR order as k_sweep_small (bitwise
// identical).  Chunks holding a heavy row go through k_sweep_small's strip,
// after the heavy phase.
// =============================================================================
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int G, bool W, int S, int U>
struct SweepRing {                                 // one per lane group
    double val[S][U][2 * G];                       // stage slot: U rows [bar | prev] (2C of 2G used)
    double w[W ? 2 * S : 1][U];                    // weights, with the indices
    unsigned idx[2 * S][U];                        // column indices, S stages ahead of the values
};

// rows [base, base + nr) of the shard (nr <= 32, no heavy row among them).  Positions are
// 32-bit offsets into the group's stream; a slot past the stream is zero-filled in shared
// memory (weight 0): its addends are +0.0, and x + (+0.0) == x for every x != -0.0 -- the
// chains start at +0.0 and a round-to-nearest sum is -0.0 only when both operands are, so
// they never hold -0.0 and the padding is exact without per-slot selects.
template <int G, bool W, int S, int U>
__device__ __forceinline__ void sweep_async_chunk(Bufs& b, Geo& g, unsigned long long base, unsigned nr,
                                                  SweepRing<G, W, S, U>& ring) {
    static_assert(U <= G, "one index per lane per stage");
    const DevState* st = b.st;
    const unsigned C = g.C;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned gi = lane / G, c = lane % G;
    const unsigned r_lo = min(nr, gi * G), r_hi = min(nr, (gi + 1) * G);
    const unsigned nrg = r_hi - r_lo;             // this group's rows (0 for idle groups)
    const unsigned long long gbase = base + r_lo;
    const bool okc = c < C;
    const double beta = st->beta_next;
    const double* __restrict__ Xown = b.U[st->sw_b] + c;
    double* xs_main = b.xs[st->xs_w * 2 + kMatBar] + c;
    double* xs_ext = b.xs[st->xs_w * 2 + kMatExt] + c;
    const char* pairb = reinterpret_cast<const char*>(b.pair) + 16 * c;
    const unsigned rowbytes = 16 * C;

    const long long e0 = __ldg(b.row_ptr + gbase);
    const unsigned my_end = c < nrg ? (unsigned)(__ldg(b.row_ptr + gbase + c + 1) - e0) : 0xffffffffu;
    const unsigned last = __shfl_sync(kFull, my_end, nrg ? nrg - 1 : 0, G);
    const unsigned len = nrg ? last : 0;          // stream length
    const unsigned nst = (len + U - 1) / U;
    unsigned nst_max = nst;
#pragma unroll
    for (int o = G; o < 32; o <<= 1) nst_max = max(nst_max, __shfl_xor_sync(kFull, nst_max, o));
    const unsigned* __restrict__ colp = b.col + e0;
    const double* __restrict__ valp = W ? b.val + e0 : nullptr;

    auto issue_idx = [&](unsigned t) {             // column indices (and weights) of stage t
        const unsigned k = t * U + c;
        if (c < (unsigned)U) {
            if (k < len) {
                cp_async4(&ring.idx[t % (2 * S)][c], colp + k);
                if (W) cp_async8(&ring.w[t % (2 * S)][c], valp + k);
            } else if (W) {
                ring.w[t % (2 * S)][c] = 0.0;
            }
        }
    };
    auto issue_val = [&](unsigned t) {             // the stage's rows; its indices have landed
        const unsigned* ix = ring.idx[t % (2 * S)];
        double* dst = &ring.val[t % S][0][2 * c];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!okc) continue;
            if (t * U + u < len)
                cp_async16(dst + u * 2 * G, pairb + (size_t)(ix[u] & kIdxMask) * rowbytes);
            else                                   // past the stream: +0.0 addends
                *reinterpret_cast<double2*>(dst + u * 2 * G) = make_double2(0.0, 0.0);
        }
    };
    auto load_xi = [&](unsigned r) -> double {
        return (okc && r < nrg) ? ldg(Xown + (size_t)(g.row0 + gbase + r) * C) : 0.0;
    };
    // flush row r of the groups with `need` (the shuffles run on every lane)
    auto flush = [&](bool need, unsigned r, double ab, double ae, double xi) {
        const unsigned long long row = gbase + r;
        if (need && okc) {
            xs_main[(size_t)row * C] = ab;
            xs_ext[(size_t)row * C] = ae;
        }
        const double a = dmul(ab, xi);
        double p = 0.0;
#pragma unroll
        for (int l2 = 0; l2 < G; ++l2) {
            const double v = __shfl_sync(kFull, a, l2, G);
            if ((unsigned)l2 < C) p = dadd(p, v);
        }
        if (need && c == 0) b.prod[row] = p;
    };

#pragma unroll
    for (int t = 0; t < S; ++t) issue_idx(t);
    cp_async_commit();
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll
    for (int t = 0; t < S; ++t) {
        if ((unsigned)t < nst_max) issue_val(t);
        issue_idx(t + S);
        cp_async_commit();
    }
    unsigned cur = 0;
    unsigned cur_end = __shfl_sync(kFull, my_end, 0, G);
    double xi = load_xi(0);
    double ab = 0.0, ae = 0.0;
    for (unsigned s = 0; s < nst_max; ++s) {
        cp_async_wait<S - 1>();                    // stage s (and the indices of stage s + S) landed
        __syncwarp();
        const double* sv = &ring.val[s % S][0][c];
        const double* sw = W ? ring.w[s % (2 * S)] : nullptr;
        const unsigned k0 = s * U;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const unsigned k = k0 + u;
            const double bv = sv[u * 2 * G];
            const double pv = sv[u * 2 * G + C];
            double xb = bv, xe = extrap(bv, pv, beta);
            if (W) {
                const double w = sw[u];
                xb = dmul(w, xb);
                xe = dmul(w, xe);
            }
            bool need = k == cur_end && cur < nrg;  // row `cur` ends before nonzero k (empty rows too)
            while (__any_sync(kFull, need)) {
                flush(need, cur, ab, ae, xi);
                if (need) {
                    ab = 0.0;
                    ae = 0.0;
                    ++cur;
                }
                cur_end = __shfl_sync(kFull, my_end, min(cur, (unsigned)G - 1u), G);
                if (need) xi = load_xi(cur);
                need = k == cur_end && cur < nrg;
            }
            ab = dadd(ab, xb);
            ae = dadd(ae, xe);
        }
        __syncwarp();                              // slot s % S is free
        if (s + S < nst_max) issue_val(s + S);
        issue_idx(s + 2 * S);
        cp_async_commit();
    }
    bool need = cur < nrg;                         // each group's last row, then trailing empty rows
    while (__any_sync(kFull, need)) {
        flush(need, cur, ab, ae, xi);
        if (need) {
            ab = 0.0;
            ae = 0.0;
            ++cur;
            xi = load_xi(cur);
        }
        need = cur < nrg;
    }
    cp_async_wait<0>();                            // no copy may land in a ring the next chunk reuses
    __syncwarp();
}

template <int G, bool W, int S, int U>
__global__ void __launch_bounds__(128) k_sweep_async(Bufs b, Geo g) {
    extern __shared__ __align__(16) unsigned char sweep_ring_smem[];
    using Ring = SweepRing<G, W, S, U>;
    Ring* ring = reinterpret_cast<Ring*>(sweep_ring_smem) + (threadIdx.x / G);
    k_sweep_small_body<G, true, W, true, 2>(b, g, [&](unsigned long long base, unsigned nr) {
        sweep_async_chunk<G, W, S, U>(b, g, base, nr, *ring);
    });
}

// Interleave [bar^n | bar^{n-1}] rows for the PAIR sweep (after the row exchange).
__global__ void k_pair_pack(Bufs b, Geo g) {
    const DevState* st = b.st;
    if (st->done) return;
    const unsigned C = g.C;
    const double* __restrict__ B = b.U[st->sw_b];
    const double* __restrict__ P = b.U[st->sw_p];
    const unsigned long long total = g.N * 2ull * C;
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < total;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long i = e / (2 * C), k = e % (2 * C);
        b.pair[e] = k < C ? B[i * C + k] : P[i * C + k - C];
    }
}

// =============================================================================
// Per-block sequential sums of per-row scalars (objective.hpp:160-170 order):
//   part[s][blk] = ((0 + v_{1024 blk}) + v_{1024 blk + 1}) + ...
// One CTA per (scalar, block): the block's values are staged into shared
// memory by all threads (coalesced), then one thread adds them in order.
// =============================================================================
constexpr int kRowsumThreads = 128;

__global__ void __launch_bounds__(kRowsumThreads) k_rowsum(Bufs b, Geo g, int nscal, const double* a0,
                                                           const double* a1, const double* a2, const double* a3,
                                                           int slot0) {
    if (b.st->done) return;
    __shared__ double v[kBlock];
    const int which = (int)(blockIdx.x / g.nblk);
    const unsigned long long blk = blockIdx.x % g.nblk;
    const double* a = which == 0 ? a0 : which == 1 ? a1 : which == 2 ? a2 : a3;
    const unsigned long long r0 = blk * kBlock;
    const int n = (int)(min(r0 + kBlock, g.nrows) - r0);
    for (int k = threadIdx.x; k < n; k += kRowsumThreads) v[k] = a[r0 + k];
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        int k = 0;
        for (; k + 8 <= n; k += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) m = dadd(m, v[k + u]);
        }
        for (; k < n; ++k) m = dadd(m, v[k]);
        b.spart[(size_t)(slot0 + which) * g.spart_stride + blk] = m;
    }
}

// =============================================================================
// K2: Gram partials per 1024-row block, objective.hpp:69-80:
//   P_b[r][s] = sum_{i in block b, ascending} x_i[r] * x_i[s]
// x_i[r]*x_i[s] == x_i[s]*x_i[r] in IEEE, so only r <= s is accumulated (the
// reference's matrix is exactly symmetric).  Each thread owns a 4x4 register
// tile of (r, s) of one matrix and walks the block's rows in order from
// shared-memory chunks.  dual: matrix 1 = bar^n, matrix 0 = X_ext^{n+1}
// (formed as in solver.hpp:261); single: matrix 0 = the swept point.
// grid = (blocks, tile groups); blockDim = 128.
// =============================================================================
constexpr int kGramMaxThreads = 320;   // blockDim = min(320, tiles rounded up to a warp)

// Number of TR x TC tiles of one C x C Gram that hold at least one pair r <= s.
__host__ __device__ inline int gram_tiles(int C, int TR, int TC) {
    const int nR = (C + TR - 1) / TR, nC = (C + TC - 1) / TC;
    int t = 0;
    for (int J = 0; J < nC; ++J) t += min(nR - 1, (TC * J + TC - 1) / TR) + 1;
    return t;
}

// Shared memory of k_gram: 2 stages x (bar [+ prev]) x R x C4, + the ext tile (dual).
__host__ __device__ inline size_t gram_smem(int C, int dual, int R, int TS = 4) {
    const int PADW = TS > 4 ? TS : 4;
    const int C4 = (C + PADW - 1) / PADW * PADW;
    return sizeof(double) * (size_t)R * C4 * (dual ? 5 : 2);
}

// TS x TS register tiles: TS = 4 in general; TS = 1 when there are few 1024-row
// blocks (small N): every (r, s) pair gets its own thread, so the 1024-long
// sequential chains of all pairs run in parallel instead of 16 per thread.
template <int TR, int TC = TR, bool TOL = false>
__global__ void __launch_bounds__(kGramMaxThreads) k_gram(Bufs b, Geo g, int dual, int rows_per_chunk) {
    const DevState* st = b.st;
    if (st->done) return;
    extern __shared__ double smg[];
    const int C = (int)g.C;
    constexpr int PADW = (TR > TC ? TR : TC) > 4 ? (TR > TC ? TR : TC) : 4;
    const int C4 = (C + PADW - 1) / PADW * PADW;         // row stride in shared memory
    const int nR = (C + TR - 1) / TR, nC = (C + TC - 1) / TC;
    // tiles (I, J) of TR x TC that hold at least one pair r <= s: I <= (TC J + TC - 1) / TR
    const int tiles_per_mat = gram_tiles(C, TR, TC);
    const int nmat = dual ? 2 : 1;
    const int tile = blockIdx.y * blockDim.x + threadIdx.x;
    const bool has = tile < tiles_per_mat * nmat;
    const int mat_local = has ? tile / tiles_per_mat : 0;
    int tt = has ? tile % tiles_per_mat : 0;
    int I = 0, J = 0;
    for (; J < nC; ++J) {
        const int cnt = min(nR - 1, (TC * J + TC - 1) / TR) + 1;
        if (tt < cnt) {
            I = tt;
            break;
        }
        tt -= cnt;
    }
    // dual: local matrix 0 -> bar (slot kMatBar), 1 -> ext (slot kMatExt)
    const int out_mat = dual ? (mat_local == 0 ? kMatBar : kMatExt) : kMatExt;

    const double* __restrict__ Bm = b.U[st->sw_b];
    const double* __restrict__ Pm = dual ? b.U[st->sw_p] : nullptr;
    const double beta = st->beta_next;
    // grid-stride over blocks (a persistent grid can run next to the sweep, FC_OVERLAP=2)
    for (unsigned long long blk = blockIdx.x; blk < g.nblk; blk += gridDim.x) {
    const unsigned long long r0 = blk * kBlock;
    const unsigned long long r1 = min(r0 + kBlock, g.nrows);
    const int R = rows_per_chunk;
    const size_t tsz = (size_t)R * C4;
    // stage k: bar at smg + k*tsz, prev at smg + (2+k)*tsz; ext tile after them (dual)
    double* te = smg + (dual ? 4 : 2) * tsz;

    auto issue = [&](int sidx, unsigned long long cr) {
        const int rows = (int)min((unsigned long long)R, r1 - cr);
        if (C == C4) {
            // unpadded rows: the chunk is one contiguous run of rows * C doubles in U and
            // in the tile -- 16-byte copies, no per-element row / column split
            const size_t a0 = (size_t)(g.row0 + cr) * C;
            for (int e = 2 * threadIdx.x; e < rows * C; e += 2 * blockDim.x) {
                cp_async16(smg + sidx * tsz + e, Bm + a0 + e);
                if (dual) cp_async16(smg + (2 + sidx) * tsz + e, Pm + a0 + e);
            }
            cp_async_commit();
            return;
        }
        for (int e = threadIdx.x; e < rows * C4; e += blockDim.x) {
            const int rr = e / C4, cc = e % C4;
            if (cc < C) {
                const size_t a = (size_t)(g.row0 + cr + rr) * C + cc;
                cp_async8(smg + sidx * tsz + e, Bm + a);
                if (dual) cp_async8(smg + (2 + sidx) * tsz + e, Pm + a);
            } else {
                smg[sidx * tsz + e] = 0.0;
                if (dual) smg[(2 + sidx) * tsz + e] = 0.0;
            }
        }
        cp_async_commit();
    };

    double acc[TR][TC];
#pragma unroll
    for (int a = 0; a < TR; ++a)
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[a][c] = 0.0;

    issue(0, r0);
    int sidx = 0;
    for (unsigned long long cr = r0; cr < r1; cr += R, sidx ^= 1) {
        const int rows = (int)min((unsigned long long)R, r1 - cr);
        if (cr + R < r1) {
            issue(sidx ^ 1, cr + R);
            cp_async_wait_1();
        } else {
            cp_async_wait_all();
        }
        __syncthreads();
        const double* tb = smg + sidx * tsz;
        if (dual) {
            const double* tp = smg + (2 + sidx) * tsz;
            for (int e = threadIdx.x; e < rows * C4; e += blockDim.x) te[e] = extrap(tb[e], tp[e], beta);
            __syncthreads();
        }
        if (has) {
            const double* t = mat_local == 0 ? tb : te;
            for (int rr = 0; rr < rows; ++rr) {
                double xr[TR], xq[TC];
                if constexpr (TR % 2 == 0 && TC % 2 == 0) {   // 16-byte aligned (C4 % 4 == 0)
                    const double2* rowp = reinterpret_cast<const double2*>(t + rr * C4);
#pragma unroll
                    for (int a = 0; a < TR / 2; ++a) {
                        const double2 rv = rowp[(TR / 2) * I + a];
                        xr[2 * a] = rv.x;
                        xr[2 * a + 1] = rv.y;
                    }
#pragma unroll
                    for (int a = 0; a < TC / 2; ++a) {
                        const double2 qv = rowp[(TC / 2) * J + a];
                        xq[2 * a] = qv.x;
                        xq[2 * a + 1] = qv.y;
                    }
                } else {
#pragma unroll
                    for (int a = 0; a < TR; ++a) xr[a] = t[rr * C4 + TR * I + a];
#pragma unroll
                    for (int a = 0; a < TC; ++a) xq[a] = t[rr * C4 + TC * J + a];
                }
#pragma unroll
                for (int a = 0; a < TR; ++a)
#pragma unroll
                    for (int c = 0; c < TC; ++c) acc[a][c] = madd<TOL>(acc[a][c], xr[a], xq[c]);
            }
        }
        __syncthreads();                                     // stage sidx is re-filled next round
    }
    if (has) {
        double* out = b.gpart[out_mat] + (size_t)blk * g.npairs;
#pragma unroll
        for (int a = 0; a < TR; ++a)
#pragma unroll
            for (int c = 0; c < TC; ++c) {
                const int r = TR * I + a, s = TC * J + c;
                if (r <= s && s < C) out[pair_index(r, s, C)] = acc[a][c];
            }
    }
    __syncthreads();                                         // stages are re-filled by the next block
    }
}

// =============================================================================
// K4a: ordered combine of block partials (objective.hpp:82-88, :171):
//   total = ((init + part_0) + part_1) + ...
// Chains: [mat 0 pairs][mat 1 pairs][scalars]; chain c's block-b partial is at
// base_c + b * stride_c.  A CTA owns up to 32 chains: all its warps stage
// [kCombTile blocks][32 chains] tiles into shared memory (coalesced: 32
// consecutive pairs of one block are contiguous), and warp 0 (lane = chain)
// adds them in ascending block order.  `init` carries the previous shard's
// running totals (ordered multi-GPU chain) or is null (0.0).
// grid.x = matrix-chain groups of 32, + one CTA per scalar chain.
// =============================================================================
constexpr int kCombTile = 128;
constexpr int kCombThreads = 256;
constexpr int kCombStages = 4;                                // tiles in flight per CTA
constexpr size_t kCombSmem = (size_t)kCombStages * kCombTile * 32 * sizeof(double);

// Every thread loads one chain column (lane) of 16 block rows per tile through a
// kCombStages-deep cp.async ring (source pointers hoisted: one add per element);
// warp 0 (lane = chain) adds the landed tiles in ascending block order.
__global__ void __launch_bounds__(kCombThreads) k_combine(Bufs b, Geo g, int mat_mask, int scal_mask,
                                                          const double* init) {
    if (b.st->done) return;
    extern __shared__ double ctile[];                       // [kCombStages][kCombTile][32]
    const int np = (int)g.npairs;
    const int mat_groups = (2 * np + 31) / 32;
    const double* sbase = nullptr;
    int c0, nch;
    if ((int)blockIdx.x < mat_groups) {
        c0 = blockIdx.x * 32;
        nch = min(32, 2 * np - c0);
    } else {
        const int s = blockIdx.x - mat_groups;
        if (s >= kNumScal || !((scal_mask >> s) & 1)) return;
        c0 = 2 * np + s;
        nch = 1;
        sbase = b.spart + (size_t)s * g.spart_stride;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int my_c = c0 + lane;
    bool live = lane < nch;
    if (!sbase && live) live = (mat_mask >> (my_c / np)) & 1;
    const unsigned long long nb = g.nblk;
    const unsigned long long ntiles = (nb + kCombTile - 1) / kCombTile;
    // this thread's column source: block partial blk of chain my_c at col + blk * step
    const double* col = nullptr;
    size_t step = 0;
    if (live) {
        if (sbase) {
            col = sbase;
            step = 1;
        } else {
            col = b.gpart[my_c / np] + (my_c % np);
            step = (size_t)np;
        }
    }
    constexpr int kRowsPerThread = kCombTile / (kCombThreads / 32);
    auto stage = [&](unsigned long long t) {
        double* dst = ctile + (size_t)(t % kCombStages) * kCombTile * 32 + lane;
        const unsigned long long b0 = t * kCombTile;
#pragma unroll 4
        for (int i = 0; i < kRowsPerThread; ++i) {
            const int r = warp + (kCombThreads / 32) * i;
            const unsigned long long blk = b0 + r;
            if (col && blk < nb) cp_async8(dst + r * 32, col + blk * step);
            else dst[r * 32] = 0.0;
        }
    };
    double acc = (live && init) ? init[my_c] : 0.0;
#pragma unroll
    for (int k = 0; k < kCombStages - 1; ++k) {
        if ((unsigned long long)k < ntiles) stage(k);
        cp_async_commit();
    }
    for (unsigned long long t = 0; t < ntiles; ++t) {
        cp_async_wait_n<kCombStages - 2>();                  // tile t landed (own copies)
        __syncthreads();                                     // ... everyone's; tile t-1 fully summed
        if (t + kCombStages - 1 < ntiles) stage(t + kCombStages - 1);
        cp_async_commit();
        if (warp == 0) {
            const double* tl = ctile + (size_t)(t % kCombStages) * kCombTile * 32 + lane;
            const int rows = (int)min((unsigned long long)kCombTile, nb - t * kCombTile);
            if (rows == kCombTile) {
#pragma unroll 16
                for (int r = 0; r < kCombTile; ++r) acc = dadd(acc, tl[r * 32]);
            } else {
                for (int r = 0; r < rows; ++r) acc = dadd(acc, tl[r * 32]);
            }
        }
    }
    cp_async_wait_all();
    if (warp == 0 && live) b.totals[my_c] = acc;
}

__device__ __forceinline__ double packed_at(const double* tot, int r, int s, int C) {
    return r <= s ? tot[pair_index(r, s, C)] : tot[pair_index(s, r, C)];
}

// ||G||_F^2, sequential over the row-major entries (objective.hpp:25-29)
__device__ double frob_packed(const double* tot, int C) {
    double f = 0.0;
    for (int r = 0; r < C; ++r)
        for (int s = 0; s < C; ++s) {
            const double v = packed_at(tot, r, s, C);
            f = dadd(f, dmul(v, v));
        }
    return f;
}

__device__ double fista_t_next(double t) {     // solver.hpp:72
    return (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
}

// The last trace slot is reserved for the terminating record (the reference always
// appends it, solver.hpp:157-173, :225-241): past the capacity, intermediate records are
// dropped (n_records keeps counting them, so n_records > trace_cap flags the loss) and
// the terminating one lands in slot trace_cap - 1.
__device__ __forceinline__ void push_record(Bufs& b, DevState* st, unsigned long long it, double loss,
                                            int increased, int backtracks, double step, bool terminal = false) {
    unsigned long long k = st->n_records++;
    if (st->trace_cap == 0) return;
    if (k >= st->trace_cap - 1) {
        if (!terminal) return;
        k = st->trace_cap - 1;
    }
    {
        long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        TraceRec& r = b.trace[k];
        r.iteration = it;
        r.loss = loss;
        r.elapsed_ms = (double)(now - st->t0_ns) * 1e-6;
        r.loss_increased = increased;
        r.backtracks = backtracks;
        r.step = step;
    }
}

// =============================================================================
// K4b: loss, stop rule, trace record and next-iteration plan (one CTA).
//   loss = (||S||^2 + ||G||^2) - 2 merge          solver.hpp:156 / :224
//   GPA stop:   loss_prev - loss <= tol           solver.hpp:157-173
//   FISTA stop: (loss_prev - loss <= tol) && !(increased && restart), restart
//               and momentum update               solver.hpp:224-269
// Expands the combined Gram(s) to full C x C (gfull) for the next k_step.
// =============================================================================
// Decision part of k_finalize (thread 0).  Returns whether the combined Gram
// matrices become the next step's (false only on a rejected backtracking trial,
// which must keep G(y) and S y of the current extrapolated point).
__device__ bool finalize_decide(Bufs& b, Geo& g, int kind) {
    DevState* st = b.st;
    const int C = (int)g.C;
    const int np = (int)g.npairs;
    const double* scal = b.totals + 2 * (size_t)np;
    if (kind == kFinGranular) return true;

    const int gm = (kind == kFinFista) ? kMatBar : kMatExt;
    const double frob_g = frob_packed(b.totals + (size_t)gm * np, C);
    const double loss = dsub(dadd(st->frob_s, frob_g), dmul(2.0, scal[kScalMerge]));
    const unsigned long long n = st->iter;

    if (kind == kFinPrelude) {                    // solver.hpp:206-215
        st->loss_prev = loss;
        st->final_loss = loss;
        st->iterations = 0;
        st->reason = 1;                           // kMaxIter unless a stop rule fires
        push_record(b, st, 0, loss, 0, 0, st->tau);
        st->t = 1.0;
        st->step_mode = kLiteral;
        st->step_a = st->sw_b;
        st->step_sel = kMatExt;
        st->step_dst = (st->sw_b + 1) % 3;
        st->beta_step = 0.0;
        st->beta_next = (st->t - 1.0) / fista_t_next(st->t);
        st->sw_p = st->sw_b;
        st->sw_b = st->step_dst;
        st->result_buf = st->sw_p;
        if (st->bt) st->frob_gy = frob_g;
        st->xs_r = st->xs_w;                      // S x0 is the first step's S y
        if (st->bt) st->xs_w = 1 - st->xs_w;
        if (st->tolmode) {                        // single-gather sweeps alternate between two sets
            st->xs_a = st->xs_w;
            st->xs_b = st->xs_w;
            st->xs_w = 1 - st->xs_w;
        }
        st->iter = 1;
        return true;
    }

    if (kind == kFinGpa) {                        // solver.hpp:153-178
        const int increased = n > 0 && loss > st->loss_prev;
        const bool stop_tol = dsub(st->loss_prev, loss) <= st->tol;
        const bool stop_iter = n >= st->max_iter;
        if (stop_tol || stop_iter || n % st->trace_every == 0)
            push_record(b, st, n, loss, increased, 0, st->tau, stop_tol || stop_iter);
        st->iterations = n;
        st->final_loss = loss;
        st->result_buf = st->sw_b;
        if (stop_tol || stop_iter) {
            st->reason = stop_tol ? 0 : 1;
            st->done = 1;
            return true;
        }
        st->step_mode = kLiteral;
        st->step_a = st->sw_b;
        st->step_sel = kMatExt;
        st->step_dst = 1 - st->sw_b;
        st->sw_b = st->step_dst;
        st->loss_prev = loss;
        st->iter = n + 1;
        if (st->tolmode) st->xs_a = st->xs_w;     // literal step: S bar of this sweep
        return true;
    }

    // kFinFista
    if (st->bt) {                                 // Beck-Teboulle sufficient decrease
        const double f_y = dsub(dadd(st->frob_s, st->frob_gy), dmul(2.0, scal[kScalMergeY]));
        const double q = dadd(dadd(f_y, scal[kScalLin]), dmul(dmul(0.5, st->L), scal[kScalSq]));
        if (loss > q && st->backtracks < st->bt_max) {
            st->L = dmul(st->bt_eta, st->L);
            st->tau = 1.0 / st->L;
            st->backtracks += 1;
            return false;                         // same iteration, same y, new step: keep G(y)
        }
    }
    const int increased = loss > st->loss_prev;
    const double decrease = dsub(st->loss_prev, loss);
    const bool stop_tol = decrease <= st->tol && !(increased && st->restart);
    const bool stop_iter = n >= st->max_iter;
    if (stop_tol || stop_iter || n % st->trace_every == 0)
        push_record(b, st, n, loss, increased, st->backtracks, st->tau, stop_tol || stop_iter);
    st->result_buf = st->sw_b;
    st->iterations = n;
    st->final_loss = loss;
    st->backtracks = 0;
    if (stop_tol) {
        st->reason = increased ? 2 : 0;
        st->done = 1;
        return true;
    }
    if (stop_iter) {
        st->reason = 1;
        st->done = 1;
        return true;
    }
    const int bar_idx = st->sw_b, prev_idx = st->sw_p;
    st->xs_r = st->xs_w;                          // this pass's S bar / S X_ext feed the next step
    if (st->bt) st->xs_w = 1 - st->xs_w;
    if (st->tolmode) {                            // S bar^n (this sweep) and S bar^{n-1} (the previous)
        st->xs_a = st->xs_w;
        st->xs_b = 1 - st->xs_w;
        st->xs_w = 1 - st->xs_w;                  // the next sweep overwrites S bar^{n-1} after the step read it
    }
    if (increased && st->restart) {               // solver.hpp:247-249
        st->t = 1.0;
        st->step_mode = kLiteral;
        st->step_a = bar_idx;
        st->step_sel = kMatBar;
        if (st->bt) st->frob_gy = frob_g;
    } else {                                      // solver.hpp:251-266
        const double t_next = fista_t_next(st->t);
        st->step_mode = kExtrap;
        st->step_a = bar_idx;
        st->step_b = prev_idx;
        st->beta_step = st->beta_next;            // == (t - 1) / t_next
        st->step_sel = kMatExt;
        st->t = t_next;
        if (st->bt) st->frob_gy = frob_packed(b.totals + (size_t)kMatExt * np, C);
    }
    st->beta_next = (st->t - 1.0) / fista_t_next(st->t);
    st->step_dst = 3 - bar_idx - prev_idx;
    st->sw_p = bar_idx;
    st->sw_b = st->step_dst;
    st->loss_prev = loss;
    st->iter = n + 1;
    return true;
}

__global__ void __launch_bounds__(256) k_finalize(Bufs b, Geo g, int kind, int mat_mask) {
    DevState* st = b.st;
    if (st->done) return;
    __shared__ int expand;
    const int C = (int)g.C;
    const int np = (int)g.npairs;
    if (threadIdx.x == 0) expand = finalize_decide(b, g, kind) ? 1 : 0;
    __syncthreads();
    if (!expand) return;
    for (int m = 0; m < 2; ++m) {
        if (!((mat_mask >> m) & 1)) continue;
        const double* tot = b.totals + (size_t)m * np;
        for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
            const int r = e / C, s = e % C;
            b.gfull[m][e] = packed_at(tot, r, s, C);
        }
    }
}

// =============================================================================
// K3: gradient step + simplex projection (solver.hpp:89-107), with the FISTA
// extrapolated point rebuilt on the fly (solver.hpp:261) instead of stored:
//   x   = literal ? A_i : A_i + beta (A_i - B_i)
//   o_r = sum_l G[r][l] x_l                    (ShareMatrix::apply, objective.hpp:37-43)
//   g_r = -4 (xs_r - o_r)                      (objective.hpp:116-117)
//   y_r = x_r - tau g_r ; bar = P_simplex(y)
// bt: also lin_i = sum_r g_r (bar_r - x_r), sq_i = sum_r (bar_r - x_r)^2,
//     <xs_i, x_i> (merge term of f at the extrapolated point).
// =============================================================================
template <int G, int S>
__global__ void __launch_bounds__(256) k_step(Bufs b, Geo g, int bt) {
    DevState* st = b.st;
    if (st->done) return;
    __shared__ double smp[256 / 32][32 / G][G * S];
    const int C = (int)g.C;
    const unsigned lane = threadIdx.x & 31u;
    const int lg = (int)(lane % G);
    const int sub = (int)(lane / G);
    double* sm = &smp[threadIdx.x >> 5][sub][0];
    const int mode = st->step_mode;
    const double* __restrict__ A = b.U[st->step_a];
    const double* __restrict__ Bp = b.U[st->step_b];
    double* __restrict__ D = b.U[st->step_dst];
    const double beta = st->beta_step;
    const double tau = st->tau;
    const int sel = st->step_sel;
    const double* __restrict__ Gt = b.gfull[sel];
    const double* __restrict__ XS = b.xs[st->xs_r * 2 + sel];

    const unsigned long long warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    constexpr int RPW = 32 / G;
    bool bad = false;
    for (unsigned long long rb = w0 * RPW; rb < g.nrows; rb += warps * RPW) {
        const unsigned long long row = rb + sub;
        const bool active = row < g.nrows;
        const unsigned long long grow = g.row0 + row;
        double x[S], xs[S], y[S], gr[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int r = lg + s * G;
            x[s] = 0.0;
            xs[s] = 0.0;
            if (active && r < C) {
                const size_t a = (size_t)grow * C + r;
                const double av = A[a];
                x[s] = (mode == kLiteral) ? av : extrap(av, Bp[a], beta);
                xs[s] = XS[(size_t)row * C + r];
            }
        }
        double o[S];
#pragma unroll
        for (int s = 0; s < S; ++s) o[s] = 0.0;
#pragma unroll
        for (int s2 = 0; s2 < S; ++s2) {
#pragma unroll
            for (int l2 = 0; l2 < G; ++l2) {
                const int l = s2 * G + l2;
                const double xl = __shfl_sync(kFull, x[s2], l2, G);
                if (l < C) {
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        const int r = lg + s * G;
                        if (r < C) o[s] = dadd(o[s], dmul(ldg(Gt + (size_t)l * C + r), xl));
                    }
                }
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            gr[s] = dmul(-4.0, dsub(xs[s], o[s]));
            y[s] = dsub(x[s], dmul(tau, gr[s]));
        }
        const bool ok = project_group<G, S>(y, C, lg, sm);
        if (!ok && active) bad = true;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int r = lg + s * G;
            if (active && r < C) D[(size_t)grow * C + r] = y[s];
        }
        if (bt) {
            double al[S], aq[S], am[S];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const double d = dsub(y[s], x[s]);
                al[s] = dmul(gr[s], d);
                aq[s] = dmul(d, d);
                am[s] = dmul(xs[s], x[s]);
            }
            const double li = group_seq_sum<G, S>(al, C);
            const double qi = group_seq_sum<G, S>(aq, C);
            const double mi = group_seq_sum<G, S>(am, C);
            if (active && lg == 0) {
                b.rowterm[0][row] = li;
                b.rowterm[1][row] = qi;
                b.rowterm[2][row] = mi;
            }
        }
    }
    if (bad) {
        st->error = 1;
        st->done = 1;
    }
}

// Row-wise gradient / loss term for the single-column API (not on the
// iteration path): one thread per row, the reference's loops verbatim.
__global__ void k_gradient_rows(const double* g, const double* xs, const double* x, double* out,
                                unsigned long long rows, int C) {
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (i >= rows) return;
    const double* xi = x + i * C;
    const double* xsi = xs + i * C;
    double* o = out + i * C;
    for (int k = 0; k < C; ++k) {
        double acc = 0.0;
        for (int l = 0; l < C; ++l) acc = dadd(acc, dmul(g[k * C + l], xi[l]));
        o[k] = dmul(-4.0, dsub(xsi[k], acc));
    }
}

__global__ void k_loss_terms_rows(const double* xs, const double* x, double* out, unsigned long long rows, int C) {
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double acc = 0.0;
    for (int k = 0; k < C; ++k) acc = dadd(acc, dmul(xs[i * C + k], x[i * C + k]));
    out[i] = acc;
}

// Set / clear the hot-row flag (bit 31) of every stored column index:
// hot iff deg[j] >= threshold (threshold 0xFFFFFFFF clears all flags).
__global__ void k_flag_hot(unsigned* col, unsigned long long nnz, const unsigned* deg, unsigned threshold) {
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < nnz;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned j = col[e] & kIdxMask;
        col[e] = j | (deg[j] >= threshold ? kHotBit : 0u);
    }
}

// Device clock origin of TraceRecord::elapsed_ms.
// ---- second order (objective.hpp:61-90, :186-217) ------------------------------------
// Z = [A | B] row by row (N x 2C): the Gram of Z holds cross_share(A, B) = A B^T in its
// upper-right C x C block with exactly the reference's per-block products and order.
__global__ void k_stack2(const double* a, const double* b, double* z, unsigned long long n, int C) {
    const unsigned long long total = n * (unsigned long long)(2 * C);
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < total;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long i = e / (2 * C);
        const int k = (int)(e - i * 2 * C);
        z[e] = k < C ? a[i * C + k] : b[i * C + (k - C)];
    }
}

// out_i[k] = -4 (vs[k] - ax[k] - atx[k] - bv[k]); g2 = the 2C x 2C Gram of [V | X]:
// A[k][l] = g2[k][C+l], B[k][l] = g2[C+k][C+l]; each sum sequential in l from 0.0.
__global__ void k_hvp_rows(const double* g2, const double* vs, const double* x, const double* v, double* out,
                           unsigned long long n, int C) {
    const unsigned long long total = n * (unsigned long long)C;
    const int W = 2 * C;
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < total;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long i = e / C;
        const int k = (int)(e - i * C);
        const double* xi = x + i * C;
        const double* vi = v + i * C;
        double ax = 0.0, atx = 0.0, bv = 0.0;
        for (int l = 0; l < C; ++l) ax = dadd(ax, dmul(g2[k * W + C + l], xi[l]));
        for (int l = 0; l < C; ++l) atx = dadd(atx, dmul(g2[l * W + C + k], xi[l]));
        for (int l = 0; l < C; ++l) bv = dadd(bv, dmul(g2[(C + k) * W + C + l], vi[l]));
        out[e] = dmul(-4.0, dsub(dsub(dsub(vs[e], ax), atx), bv));
    }
}

// Halo exchange (locality graphs, multi-rank): rows of U listed in `rows` <-> a packed
// buffer [i][C].  Lanes run over components, so each row moves as one coalesced segment.
__global__ void k_halo_pack(const double* __restrict__ U, const unsigned* __restrict__ rows, unsigned long long n,
                            unsigned C, double* __restrict__ out) {
    const unsigned long long total = n * C;
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < total;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long i = e / C, k = e % C;
        FC_DCHECK(rows[i] < 0x80000000u);
        out[e] = U[(size_t)rows[i] * C + k];
    }
}

__global__ void k_halo_unpack(const double* __restrict__ in, const unsigned* __restrict__ rows, unsigned long long n,
                              unsigned C, double* __restrict__ U) {
    const unsigned long long total = n * C;
    for (unsigned long long e = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; e < total;
         e += (unsigned long long)gridDim.x * blockDim.x) {
        const unsigned long long i = e / C, k = e % C;
        U[(size_t)rows[i] * C + k] = in[e];
    }
}

// Structural check of an uploaded CSR (fc_upload_csr accepts caller arrays): row_ptr
// monotone, column indices < n and strictly ascending within a row -- the invariants
// from_triplets establishes (sparse.hpp:43-58) and every gathering kernel relies on.
// Warp per row; the first failing row wins: out = min over failures of (row << 2 | code),
// code 1 = row_ptr decreases, 2 = column out of range, 3 = columns not strictly ascending.
__global__ void k_check_csr(const long long* row_ptr, unsigned long long rows, const unsigned* col,
                            unsigned long long n, unsigned long long* out) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned long long warps = (unsigned long long)gridDim.x * (blockDim.x >> 5);
    for (unsigned long long i = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5; i < rows;
         i += warps) {
        const long long a = row_ptr[i], b = row_ptr[i + 1];
        unsigned code = 0;
        if (b < a) {
            code = 1;
        } else {
            for (long long k = a + lane; k < b; k += 32) {
                const unsigned c0 = col[k];
                if (c0 >= n) { code = 2; break; }
                if (k + 1 < b && col[k + 1] <= c0) { code = code ? code : 3u; }
            }
        }
        // lowest code of the row's failing lanes (2 before 3 at equal rows is fine: either reports the row)
        const unsigned any = __ballot_sync(0xffffffffu, code != 0);
        if (any && lane == (unsigned)(__ffs(any) - 1)) atomicMin(out, (i << 2) | code);
    }
}

__global__ void k_degrees(const long long* row_ptr, unsigned long long n, unsigned* deg) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const long long d = row_ptr[i + 1] - row_ptr[i];
        deg[i] = (unsigned)(d < 0xFFFFFFFELL ? d : 0xFFFFFFFELL);
    }
}

// Fingerprint of the resident CSR (checkpoint compatibility, not cryptographic):
// sum over entries of (column + 1) * (2 * position + 1) (+ the value bits when
// weighted) and of row_ptr[r] * (2r + 1) -- order-sensitive, one 64-bit multiply each.
__global__ void k_fingerprint(const long long* row_ptr, unsigned long long rows, const unsigned* col,
                              const double* val, unsigned long long nnz, unsigned long long* out) {
    unsigned long long acc = 0;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; k < nnz; k += stride) {
        unsigned long long h = (unsigned long long)((col[k] & kIdxMask) + 1u);
        if (val) h ^= (unsigned long long)__double_as_longlong(val[k]);
        acc += h * (2ULL * k + 1ULL);
    }
    for (unsigned long long r = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; r <= rows; r += stride)
        acc += (unsigned long long)row_ptr[r] * (0x9E3779B97F4A7C15ULL ^ (2ULL * r + 1ULL));
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

__global__ void k_stamp(DevState* st) {
    long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    st->t0_ns = now;
}

// =============================================================================
// Thread-per-row projection (simplex.hpp:18-59) for C <= CP <= 32: the row's
// C values live in registers, so the reference's sequential loops (cumsum,
// residual sums, max, ties) cost C instructions per THREAD instead of C per
// warp and row.  Same operations in the same order as the reference.
// =============================================================================
template <int CP>
__device__ __forceinline__ void bitonic_desc(double (&v)[CP]) {
#pragma unroll
    for (int k = 2; k <= CP; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int i = 0; i < CP; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const double a = v[i], b = v[l];
                    const bool sw = ((i & k) == 0) ? (a < b) : (b < a);
                    v[i] = sw ? b : a;
                    v[l] = sw ? a : b;
                }
            }
        }
    }
}

// cond_k of simplex.hpp:36: sorted_k - RN(a / d) >= 0, with a = RN(cs_k - 1),
// d = k + 1.  Decided from RN(s*d) when it is clear of the rounding band
// (|RN(s d) - s d| <= eps |s d|, d ulp(s)/2 <= eps |s d|: an 8 eps margin is
// conservative), otherwise by the exact IEEE division the reference performs.
__device__ __forceinline__ bool threshold_cond(double s, double a, double d) {
    const double p = dmul(s, d);
    const double mag = fmax(fabs(a), fabs(p));
    if (mag >= 0x1p-900 && mag <= 0x1p+1000) {
        const double margin = dmul(mag, 0x1p-50);
        if (p >= dadd(a, margin)) return true;
        if (p <= dsub(a, margin)) return false;
    }
    return dsub(s, a / d) >= 0.0;
}

// Threshold of simplex.hpp:29-36 for the row stored at r[0..C) (shared
// memory, index order); only the sorted copy is held in registers.
template <int CP>
__device__ __forceinline__ double row_threshold(const double* r, int C) {
    double v[CP];
#pragma unroll
    for (int k = 0; k < CP; ++k) v[k] = (k < C) ? r[k] : -INFINITY;
    bitonic_desc<CP>(v);
    double cs = 0.0, a_star = 0.0;
    int k_star = -1;
#pragma unroll
    for (int k = 0; k < CP; ++k) {
        if (k < C) {
            cs = dadd(cs, v[k]);
            const double a = dsub(cs, 1.0);
            if (threshold_cond(v[k], a, (double)(k + 1))) {
                k_star = k;
                a_star = a;
            }
        }
    }
    return k_star >= 0 ? a_star / (double)(k_star + 1) : 0.0;
}

// Residual folds of simplex.hpp:43-55 (up to 4 rounds: sequential sum, max,
// ties, subtract residual/ties from the maxima).  Same values as the
// reference's loops, cheaper bookkeeping: the maxima are tracked as a bit mask
// together with the second-largest value.  All maxima hold the same value
// (equal doubles; if the maximum is 0 every entry is +-0 and the fold adds the
// same 1/ties to each), so after a fold they all become v = max(top - share, 0);
// if v still exceeds the runner-up the mask is unchanged, otherwise everything
// is recomputed from scratch.
template <int CP>
__device__ __forceinline__ void top_two(const double (&w)[CP], int C, double& top, unsigned& tmask) {
    top = w[0];
#pragma unroll
    for (int k = 1; k < CP; ++k)
        if (k < C) top = (top < w[k]) ? w[k] : top;
    tmask = 0u;
#pragma unroll
    for (int k = 0; k < CP; ++k)
        if (k < C && w[k] == top) tmask |= 1u << k;
}

template <int CP>
__device__ __forceinline__ void fold_residual(double (&w)[CP], int C) {
    double top;
    unsigned tmask;
    top_two<CP>(w, C, top, tmask);
    double second = -INFINITY;
#pragma unroll
    for (int k = 0; k < CP; ++k)
        if (k < C && !((tmask >> k) & 1u)) second = (second < w[k]) ? w[k] : second;
#pragma unroll 1
    for (int round = 0; round < 4; ++round) {
        double sum = 0.0;
#pragma unroll
        for (int k = 0; k < CP; ++k)
            if (k < C) sum = dadd(sum, w[k]);
        const double residual = dsub(sum, 1.0);
        if (residual == 0.0) break;
        const double share = residual / (double)__popc(tmask);
        const double v = ref_max(dsub(top, share), 0.0);
#pragma unroll
        for (int k = 0; k < CP; ++k)
            if ((tmask >> k) & 1u) w[k] = v;
        if (v > second) {
            top = v;
        } else {
            top_two<CP>(w, C, top, tmask);
            second = -INFINITY;
#pragma unroll
            for (int k = 0; k < CP; ++k)
                if (k < C && !((tmask >> k) & 1u)) second = (second < w[k]) ? w[k] : second;
        }
    }
}

// K3 (C <= 32, no backtracking terms).  Each warp handles batches of 32 rows
// through three per-warp shared tiles [32][G+1] (stride G+1: conflict-free
// row-per-thread access):
//   1 lane = component: cp.async of bar^{n-1} rows (A), bar^{n-2} rows (B, when
//     extrapolating) and S X_ext rows into the tiles -- the whole batch's loads
//     in flight at once, one round trip per batch
//   2 thread = row: x = A + beta (A - B) (solver.hpp:261), g_k = -4 (xs_k -
//     sum_l G[k][l] x_l) (4 independent k chains, G broadcast from shared memory
//     as double2), y_k = x_k - tau g_k, projection -- the reference's order
//   3 lane = component: coalesced store of bar^n.
// G (power of two, 2..32) is the padded row width, C <= G; EXACT: C == G.
constexpr int kStepThreads = 128;

#ifndef FC_STEP_KU
#define FC_STEP_KU 4
#endif

// Tolerance mode's projection threshold (Michelot 1986): theta = (sum_S y - 1) / |S| with
// S = {y > theta}, starting from S = all entries; theta only grows and S only shrinks, so
// the loop stops when a pass drops nothing (typically 2-4 passes over the row).  Equals the
// sorted-prefix threshold of simplex.hpp:29-36 in exact arithmetic.
__device__ __forceinline__ double michelot_threshold(const double* y, int C) {
    double sum = 0.0;
    for (int k = 0; k < C; ++k) sum += y[k];
    int cnt = C;
    double thr = (sum - 1.0) / (double)cnt;
    for (int it = 0; it < C; ++it) {
        double s2 = 0.0;
        int c2 = 0;
        for (int k = 0; k < C; ++k)
            if (y[k] > thr) {
                s2 += y[k];
                ++c2;
            }
        if (c2 == cnt || c2 == 0) break;
        cnt = c2;
        thr = (s2 - 1.0) / (double)cnt;
    }
    return thr;
}

// Per-kernel invariants of a k_step_t / k_step_gram batch (read from the plan once).
struct StepPlan {
    const double* A;                                         // bar^{n-1} (or the literal point)
    const double* Bp;                                        // bar^{n-2}
    double* D;                                               // receives bar^n
    const double* XS;                                        // S X_ext^n (or S bar); TOL: S bar^{n-1}
    const double* XSB;                                       // TOL: S bar^{n-2} (S X_ext^n by linearity)
    double beta, tau;
    int mode;
};

__device__ __forceinline__ StepPlan step_plan(const Bufs& b) {
    const DevState* st = b.st;
    StepPlan p;
    p.mode = st->step_mode;
    p.A = b.U[st->step_a];
    p.Bp = b.U[st->step_b];
    p.D = b.U[st->step_dst];
    p.beta = st->beta_step;
    p.tau = st->tau;
    if (st->tolmode) {
        p.XS = b.xs[st->xs_a * 2];
        p.XSB = b.xs[st->xs_b * 2];
    } else {
        p.XS = b.xs[st->xs_r * 2 + st->step_sel];
        p.XSB = nullptr;
    }
    return p;
}

// Gr[k*G + l] = G[k][l] (zero padded to G x G) from the expanded C x C matrix of the plan.
template <int G>
__device__ __forceinline__ void stage_gram_matrix(const Bufs& b, double* Gr, int C) {
    const double* __restrict__ Gt = b.gfull[b.st->step_sel];   // Gt[l*C + k] == G[k][l]
    for (int e = threadIdx.x; e < G * G; e += blockDim.x) {
        const int k = e / G, l = e % G;
        Gr[e] = (k < C && l < C) ? Gt[l * C + k] : 0.0;
    }
}

// One warp, rows [rb, min(rb + 32, rend)) of the shard: the K3 batch described above.
// Tiles TA/TB/TX are the warp's [32][G+1]; on return TA holds the A rows (bar^{n-1})
// and TX the new rows bar^n (already stored to D).  Returns false on a non-finite y.
// BT: also the backtracking row terms (as k_step): lin_i = sum_r g_r (bar_r - x_r),
// sq_i = sum_r (bar_r - x_r)^2, <xs_i, x_i>; g is parked in the thread's A-tile row.
template <int G, bool EXACT, bool BT, bool TOL = false, bool NO_TB = false>
__device__ __forceinline__ bool step_t_batch(const StepPlan& sp, const Bufs& b, const Geo& g, const double* Gr,
                                             int C, double* TA, double* TB, double* TX, unsigned long long rb,
                                             unsigned long long rend) {
    constexpr int LD = G + 1;
    constexpr int RPW = 32 / G;
    constexpr int KU = G < FC_STEP_KU ? G : FC_STEP_KU;   // independent gradient chains per thread
    const unsigned lane = threadIdx.x & 31u;
    const int lg = (int)(lane % G);
    const int sub = (int)(lane / G);
    const bool lane_ok = EXACT || lg < C;
    const int mode = sp.mode;
    const double* __restrict__ A = sp.A;
    const double* __restrict__ Bp = sp.Bp;
    const double* __restrict__ XS = sp.XS;
    double* ra = TA + lane * LD;                             // this thread's row in phase 2
    const double* rb_ = TB + lane * LD;
    double* tr = TX + lane * LD;
    bool bad = false;
    const bool row_ok = rb + lane < rend;
    // 1: async loads of the batch
    for (int p = 0; p < 32; p += RPW) {
        const unsigned long long row = rb + p + sub;
        if (row < rend && lane_ok) {
            const size_t a = (size_t)(g.row0 + row) * C + lg;
            const int t = (p + sub) * LD + lg;
            cp_async8(TA + t, A + a);
            if (!NO_TB && mode != kLiteral) cp_async8(TB + t, Bp + a);
            cp_async8(TX + t, XS + (size_t)row * C + lg);
        }
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    double xr[G];
    if (row_ok) {
        if constexpr (NO_TB) {
            // bar^{n-2} straight from global into registers, thread per row (no B tile:
            // a third less shared memory per warp, one more CTA per SM)
            const double* brow = Bp + (size_t)(g.row0 + rb + lane) * C;
#pragma unroll
            for (int l = 0; l < G; ++l) xr[l] = (EXACT || l < C) ? ra[l] : 0.0;
            if (mode != kLiteral) {
                double bv[G];
#pragma unroll
                for (int l = 0; l < G; ++l) bv[l] = (EXACT || l < C) ? ldg(brow + l) : 0.0;
#pragma unroll
                for (int l = 0; l < G; ++l)
                    if (EXACT || l < C) xr[l] = extrap(xr[l], bv[l], sp.beta);
            }
        } else {
#pragma unroll
            for (int l = 0; l < G; ++l)
                xr[l] = (EXACT || l < C) ? ((mode == kLiteral) ? ra[l] : extrap(ra[l], rb_[l], sp.beta)) : 0.0;
        }
    }
    if constexpr (TOL) {
        // S X_ext = S bar + beta (S bar - S bar_prev): S bar_prev rows into the B tile,
        // which is dead once x is in registers (a second round trip, coalesced)
        if (mode != kLiteral) {
            __syncwarp();
            for (int p = 0; p < 32; p += RPW) {
                const unsigned long long row = rb + p + sub;
                if (row < rend && lane_ok) cp_async8(TB + (p + sub) * LD + lg, sp.XSB + (size_t)row * C + lg);
            }
            cp_async_commit();
            cp_async_wait_all();
            __syncwarp();
            for (int p = 0; p < 32; p += RPW) {
                const int t = (p + sub) * LD + lg;
                if (rb + p + sub < rend && lane_ok) TX[t] = extrap(TX[t], TB[t], sp.beta);
            }
            __syncwarp();
        }
    }
    if (row_ok) {
        double mi = 0.0;                                     // BT: <xs_i, x_i>, component order
        if constexpr (BT) {
#pragma unroll
            for (int k = 0; k < G; ++k)
                if (EXACT || k < C) mi = dadd(mi, dmul(tr[k], xr[k]));
        }
        // gradient (objective.hpp:37-43, :116-117), KU independent chains
#pragma unroll 1
        for (int k0 = 0; k0 < C; k0 += KU) {
            double o[KU];
#pragma unroll
            for (int u = 0; u < KU; ++u) o[u] = 0.0;
#pragma unroll
            for (int l2 = 0; l2 < G / 2; ++l2) {
#pragma unroll
                for (int u = 0; u < KU; ++u) {
                    const double2 gg = reinterpret_cast<const double2*>(Gr + (k0 + u) * G)[l2];
                    if (EXACT || 2 * l2 < C) o[u] = madd<TOL>(o[u], gg.x, xr[2 * l2]);
                    if (EXACT || 2 * l2 + 1 < C) o[u] = madd<TOL>(o[u], gg.y, xr[2 * l2 + 1]);
                }
            }
#pragma unroll
            for (int u = 0; u < KU; ++u) {
                if (EXACT || k0 + u < C) tr[k0 + u] = dmul(-4.0, dsub(tr[k0 + u], o[u]));
            }
        }
        // y = x - tau * grad (solver.hpp:102)
        bool fin = true;
#pragma unroll
        for (int k = 0; k < G; ++k) {
            if (EXACT || k < C) {
                if constexpr (BT) ra[k] = tr[k];            // keep g_k for lin_i
                const double y = dsub(xr[k], dmul(sp.tau, tr[k]));
                fin = fin && isfinite(y);
                tr[k] = y;
            }
        }
        if (!fin) {
            bad = true;
        } else if (C == 1) {
            tr[0] = 1.0;
        } else if constexpr (TOL) {
            // tolerance mode: sort-free Michelot projection (same threshold in exact
            // arithmetic, any summation order; no residual folds -- they move the top
            // entries by rounding-size amounts only)
            const double thr = michelot_threshold(tr, C);
#pragma unroll
            for (int k = 0; k < G; ++k)
                if (EXACT || k < C) tr[k] = ref_max(tr[k] - thr, 0.0);
        } else {
            const double thr = row_threshold<G>(tr, C);
            double w[G];
#pragma unroll
            for (int k = 0; k < G; ++k) w[k] = (EXACT || k < C) ? ref_max(dsub(tr[k], thr), 0.0) : 0.0;
            fold_residual<G>(w, C);
#pragma unroll
            for (int k = 0; k < G; ++k)
                if (EXACT || k < C) tr[k] = w[k];
        }
        if constexpr (BT) {
            double li = 0.0, qi = 0.0;
#pragma unroll
            for (int k = 0; k < G; ++k) {
                if (EXACT || k < C) {
                    const double d = dsub(tr[k], xr[k]);
                    li = dadd(li, dmul(ra[k], d));
                    qi = dadd(qi, dmul(d, d));
                }
            }
            b.rowterm[0][rb + lane] = li;
            b.rowterm[1][rb + lane] = qi;
            b.rowterm[2][rb + lane] = mi;
        }
    }
    __syncwarp();
    // 3: store bar^n
#pragma unroll 4
    for (int p = 0; p < 32; p += RPW) {
        const unsigned long long r2 = rb + p + sub;
        FC_DCHECK(r2 >= rend || g.row0 + r2 < g.N);
        if (r2 < rend && lane_ok) sp.D[(size_t)(g.row0 + r2) * C + lg] = TX[(p + sub) * LD + lg];
    }
    __syncwarp();
    return !bad;
}

template <int G, bool EXACT, bool BT = false, bool TOL = false>
__global__ void __launch_bounds__(kStepThreads, 2) k_step_t(Bufs b, Geo g) {
    DevState* st = b.st;
    if (st->done) return;
    extern __shared__ double smt[];
    constexpr int LD = G + 1;
    const int C = EXACT ? G : (int)g.C;
    const int warp = threadIdx.x >> 5;
    double* Gr = smt;                                        // Gr[k*G + l] = G[k][l]
    double* TA = smt + G * G + warp * 3 * 32 * LD;
    double* TB = TA + 32 * LD;
    double* TX = TB + 32 * LD;
    const StepPlan sp = step_plan(b);
    stage_gram_matrix<G>(b, Gr, C);
    __syncthreads();
    const unsigned long long warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    bool ok = true;
    for (unsigned long long rb = w0 * 32; rb < g.nrows; rb += warps * 32)
        ok = step_t_batch<G, EXACT, BT, TOL>(sp, b, g, Gr, C, TA, TB, TX, rb, g.nrows) && ok;
    if (!ok) {
        st->error = 1;
        st->done = 1;
    }
}

// K3 variant with two tiles per warp (A and S X_ext; bar^{n-2} read per thread): 75 KB of
// shared memory per 4-warp CTA, so three CTAs (12 warps) fit an SM when the registers
// allow (launch bound 128 x 3).  FC_STEP=t2 (C <= 32, no backtracking, bitwise).
inline size_t step_t2_smem(int G) { return sizeof(double) * ((size_t)G * G + (kStepThreads / 32) * 2 * 32 * (G + 1)); }

template <int G, bool EXACT>
__global__ void __launch_bounds__(kStepThreads, 3) k_step_t2(Bufs b, Geo g) {
    DevState* st = b.st;
    if (st->done) return;
    extern __shared__ double smt[];
    constexpr int LD = G + 1;
    const int C = EXACT ? G : (int)g.C;
    const int warp = threadIdx.x >> 5;
    double* Gr = smt;
    double* TA = smt + G * G + warp * 2 * 32 * LD;
    double* TX = TA + 32 * LD;
    const StepPlan sp = step_plan(b);
    stage_gram_matrix<G>(b, Gr, C);
    __syncthreads();
    const unsigned long long warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    bool ok = true;
    for (unsigned long long rb = w0 * 32; rb < g.nrows; rb += warps * 32)
        ok = step_t_batch<G, EXACT, false, false, true>(sp, b, g, Gr, C, TA, TA, TX, rb, g.nrows) && ok;
    if (!ok) {
        st->error = 1;
        st->done = 1;
    }
}

// =============================================================================
// K3 + K2 fused (C <= 32, FISTA without backtracking): the step kernel of
// iteration n also accumulates the Gram partials of bar^n and of the next
// extrapolated point X_ext^{n+1} = bar^n + beta_n (bar^n - bar^{n-1})
// (solver.hpp:261), which it holds on chip anyway -- k_gram's separate pass
// re-read both from HBM.  A CTA owns whole 1024-row blocks (grid-stride) and
// walks each in 128-row chunks: every warp steps 32 rows (step_t_batch), the
// extrapolated rows replace bar^{n-1} in the A tile, then the CTA's Gram
// threads (one 4x4 tile of (r, s), r <= s, of one matrix each) add the chunk's
// rows in ascending order -- the per-block sequential order of objective.hpp:71-80
// is kept exactly, so the partials equal k_gram's bit for bit.
// =============================================================================
template <int G, bool EXACT>
__global__ void __launch_bounds__(kStepThreads, 2) k_step_gram(Bufs b, Geo g) {
    DevState* st = b.st;
    if (st->done) return;
    extern __shared__ double smt[];
    constexpr int LD = G + 1;
    constexpr int TS = G < 4 ? G : 4;
    constexpr int NW = kStepThreads / 32;
    const int C = EXACT ? G : (int)g.C;
    const int warp = threadIdx.x >> 5;
    double* Gr = smt;
    double* TA0 = smt + G * G;                               // warp w: TA0 + w * 3 * 32 * LD
    double* TA = TA0 + warp * 3 * 32 * LD;
    double* TB = TA + 32 * LD;
    double* TX = TB + 32 * LD;
    const StepPlan sp = step_plan(b);
    const double beta_n = st->beta_next;
    // Gram tile of this thread: matrix 0 = bar^n (slot kMatBar), 1 = X_ext^{n+1} (kMatExt)
    const int nT = (C + TS - 1) / TS;
    const int tiles_per_mat = nT * (nT + 1) / 2;
    const int tile = threadIdx.x;
    const bool has = tile < 2 * tiles_per_mat;
    const int mat = has ? tile / tiles_per_mat : 0;
    int tt = has ? tile % tiles_per_mat : 0;
    int I = 0;
    while (tt >= nT - I) { tt -= nT - I; ++I; }
    const int J = I + tt;
    const int toff = mat == 0 ? 2 * 32 * LD : 0;             // bar^n in TX, ext in TA
    // zero the padding columns once (never written; read by the Gram tiles)
    if (!EXACT)
        for (int e = threadIdx.x; e < NW * 3 * 32 * LD; e += blockDim.x)
            if (e % LD >= C) TA0[e] = 0.0;
    stage_gram_matrix<G>(b, Gr, C);
    __syncthreads();
    const unsigned lane = threadIdx.x & 31u;
    bool ok = true;
    for (unsigned long long blk = blockIdx.x; blk < g.nblk; blk += gridDim.x) {
        const unsigned long long r0 = blk * kBlock;
        const unsigned long long r1 = min(r0 + kBlock, g.nrows);
        double acc[TS][TS];
#pragma unroll
        for (int a = 0; a < TS; ++a)
#pragma unroll
            for (int c = 0; c < TS; ++c) acc[a][c] = 0.0;
        for (unsigned long long c0 = r0; c0 < r1; c0 += 32 * NW) {
            const unsigned long long rb = c0 + 32 * warp;
            if (rb < r1) {
                ok = step_t_batch<G, EXACT, false>(sp, b, g, Gr, C, TA, TB, TX, rb, r1) && ok;
                // X_ext^{n+1} rows in place of bar^{n-1} (lane = component)
                constexpr int RPW = 32 / G;
                const int lg = (int)(lane % G), sub = (int)(lane / G);
                if (EXACT || lg < C)
                    for (int p = 0; p < 32; p += RPW) {
                        const int t = (p + sub) * LD + lg;
                        TA[t] = extrap(TX[t], TA[t], beta_n);
                    }
            }
            __syncthreads();
            if (has) {
                const int rows = (int)min((unsigned long long)(32 * NW), r1 - c0);
                for (int q = 0; q < rows; ++q) {
                    const double* row = TA0 + (q >> 5) * 3 * 32 * LD + toff + (q & 31) * LD;
                    double xr[TS], xq[TS];
#pragma unroll
                    for (int a = 0; a < TS; ++a) {
                        xr[a] = row[TS * I + a];
                        xq[a] = row[TS * J + a];
                    }
#pragma unroll
                    for (int a = 0; a < TS; ++a)
#pragma unroll
                        for (int c = 0; c < TS; ++c) acc[a][c] = dadd(acc[a][c], dmul(xr[a], xq[c]));
                }
            }
            __syncthreads();
        }
        if (has) {
            double* out = b.gpart[mat == 0 ? kMatBar : kMatExt] + blk * g.npairs;
#pragma unroll
            for (int a = 0; a < TS; ++a)
#pragma unroll
                for (int c = 0; c < TS; ++c) {
                    const int r = TS * I + a, s = TS * J + c;
                    if (r <= s && s < C) out[pair_index(r, s, C)] = acc[a][c];
                }
        }
    }
    if (!ok) {
        st->error = 1;
        st->done = 1;
    }
}

// =============================================================================
// K3 for C in (32, 256] (no backtracking terms): thread-per-row like k_step_t
// but with the row data in shared memory (CP doubles do not fit registers).
// Per warp, batches of RB rows:
//   1 lane-parallel: X_ext rows -> TX (computed in registers), S X_ext rows -> TY (cp.async)
//   2 thread = row: gradient (4 independent k chains over l ascending; G read
//     as warp-broadcast double2 from global/L1), y -> TY; projection with a
//     loop-form bitonic sort of a copy (in TX), the exact threshold test, folds
//   3 lane-parallel store.
// CP (64, 128, 256) is the padded width; rows have stride CP+1 (conflict-free).
// =============================================================================
template <int CP>
__device__ void bitonic_desc_smem(double* v) {
    for (int k = 2; k <= CP; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll 4
            for (int i = 0; i < CP; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const double a = v[i], b = v[l];
                    const bool sw = ((i & k) == 0) ? (a < b) : (b < a);
                    if (sw) {
                        v[i] = b;
                        v[l] = a;
                    }
                }
            }
        }
    }
}

constexpr int kStepBigThreads = 64;

template <int CP>
struct StepBigCfg {
    static constexpr int RB = CP <= 64 ? 32 : 16;       // rows per warp batch
    static constexpr int LDB = CP + 1;
    static size_t smem() { return sizeof(double) * (size_t)(kStepBigThreads / 32) * 2 * RB * LDB; }
};

template <int CP>
__global__ void __launch_bounds__(kStepBigThreads) k_step_big(Bufs b, Geo g) {
    DevState* st = b.st;
    if (st->done) return;
    constexpr int RB = StepBigCfg<CP>::RB;
    constexpr int LDB = StepBigCfg<CP>::LDB;
    constexpr int S = CP / 32;
    extern __shared__ double smb[];
    const int C = (int)g.C;
    const unsigned lane = threadIdx.x & 31u;
    const int warp = threadIdx.x >> 5;
    double* TX = smb + (size_t)warp * 2 * RB * LDB;
    double* TY = TX + RB * LDB;
    const int mode = st->step_mode;
    const double* __restrict__ A = b.U[st->step_a];
    const double* __restrict__ Bp = b.U[st->step_b];
    double* __restrict__ D = b.U[st->step_dst];
    const double beta = st->beta_step;
    const double tau = st->tau;
    const int sel = st->step_sel;
    const double* __restrict__ XS = b.xs[st->xs_r * 2 + sel];
    const double* __restrict__ Gt = b.gfull[sel];            // Gt[l*C + k] == G[k][l]
    const bool gvec = (C & 1) == 0;                           // double2 loads of (k, k+1)

    const unsigned long long warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    bool bad = false;
    for (unsigned long long rb = w0 * RB; rb < g.nrows; rb += warps * RB) {
        // 1: x rows (registers -> TX), xs rows (cp.async -> TY)
        for (int p = 0; p < RB; ++p) {
            const unsigned long long row = rb + p;
            if (row >= g.nrows) break;
#pragma unroll
            for (int s2 = 0; s2 < S; ++s2) {
                const int r = (int)lane + 32 * s2;
                if (r < C) {
                    const size_t a = (size_t)(g.row0 + row) * C + r;
                    const double av = A[a];
                    TX[p * LDB + r] = (mode == kLiteral) ? av : extrap(av, Bp[a], beta);
                    cp_async8(TY + p * LDB + r, XS + (size_t)row * C + r);
                }
            }
        }
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();
        const unsigned long long row = rb + lane;
        if ((int)lane < RB && row < g.nrows) {
            double* tx = TX + lane * LDB;
            double* ty = TY + lane * LDB;
            // gradient: o_k = sum_l G[k][l] x_l, g_k = -4 (xs_k - o_k) -> ty
            for (int k0 = 0; k0 < C; k0 += 4) {
                double o[4] = {0.0, 0.0, 0.0, 0.0};
                for (int l = 0; l < C; ++l) {
                    const double xl = tx[l];
                    const double* gl = Gt + (size_t)l * C + k0;
                    double gk[4];
                    if (gvec && k0 + 3 < C) {
                        const double2 g01 = __ldg(reinterpret_cast<const double2*>(gl));
                        const double2 g23 = __ldg(reinterpret_cast<const double2*>(gl + 2));
                        gk[0] = g01.x; gk[1] = g01.y; gk[2] = g23.x; gk[3] = g23.y;
                    } else {
#pragma unroll
                        for (int u = 0; u < 4; ++u) gk[u] = (k0 + u < C) ? __ldg(gl + u) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) o[u] = dadd(o[u], dmul(gk[u], xl));
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (k0 + u < C) ty[k0 + u] = dmul(-4.0, dsub(ty[k0 + u], o[u]));
            }
            bool fin = true;
            for (int k = 0; k < C; ++k) {
                const double y = dsub(tx[k], dmul(tau, ty[k]));   // solver.hpp:102
                fin = fin && isfinite(y);
                ty[k] = y;
            }
            if (!fin) {
                bad = true;
            } else if (C == 1) {
                ty[0] = 1.0;
            } else {
                // sorted copy in tx (x is dead), -inf padding
                for (int k = 0; k < CP; ++k) tx[k] = (k < C) ? ty[k] : -INFINITY;
                bitonic_desc_smem<CP>(tx);
                double cs = 0.0, a_star = 0.0;
                int k_star = -1;
                for (int k = 0; k < C; ++k) {
                    cs = dadd(cs, tx[k]);
                    const double a = dsub(cs, 1.0);
                    if (threshold_cond(tx[k], a, (double)(k + 1))) {
                        k_star = k;
                        a_star = a;
                    }
                }
                const double thr = k_star >= 0 ? a_star / (double)(k_star + 1) : 0.0;
                for (int k = 0; k < C; ++k) ty[k] = ref_max(dsub(ty[k], thr), 0.0);
                // residual folds (simplex.hpp:43-55), loop form
                for (int round = 0; round < 4; ++round) {
                    double sum = 0.0;
                    for (int k = 0; k < C; ++k) sum = dadd(sum, ty[k]);
                    const double residual = dsub(sum, 1.0);
                    if (residual == 0.0) break;
                    double top = ty[0];
                    for (int k = 1; k < C; ++k) top = (top < ty[k]) ? ty[k] : top;
                    int ties = 0;
                    for (int k = 0; k < C; ++k) ties += (ty[k] == top);
                    const double share = residual / (double)ties;
                    for (int k = 0; k < C; ++k)
                        if (ty[k] == top) ty[k] = ref_max(dsub(ty[k], share), 0.0);
                }
            }
        }
        __syncwarp();
        // 3: store bar^n
        for (int p = 0; p < RB; ++p) {
            const unsigned long long r2 = rb + p;
            if (r2 >= g.nrows) break;
#pragma unroll
            for (int s2 = 0; s2 < S; ++s2) {
                const int r = (int)lane + 32 * s2;
                if (r < C) D[(size_t)(g.row0 + r2) * C + r] = TY[p * LDB + r];
            }
        }
        __syncwarp();
    }
    if (bad) {
        st->error = 1;
        st->done = 1;
    }
}

// =============================================================================
// K3 for C in (32, 256] (no backtracking terms), CTA-cooperative:
//   batch of 32 rows per CTA (128 threads):
//   1 X_ext rows -> TX, S X_ext rows -> TY (shared, stride CP+1)
//   2 gradient as a register-tiled GEMM: thread (row group of 4, k group of
//     KT = CP/16) accumulates o[r][k] = sum_{l ascending} G[k][l] x_r[l] (each
//     output one sequential DMUL+DADD chain, the reference's order); G streamed
//     through shared memory in l-chunks (cp.async, double-buffered, l-major:
//     Gt[l*C + k] == G[k][l] is already that layout)
//   3 y = x - tau * (-4 (xs - o)) elementwise
//   4 projection, 4 lanes per row: bitonic sort of a copy (in TX), sequential
//     cumsum/threshold by the row's first lane, parallel max / tie counts,
//     sequential residual sums -- values identical to simplex.hpp:18-59
//   5 coalesced store of bar^n.
// =============================================================================
constexpr int kWideThreads = 128;
constexpr int kWideRows = 32;
constexpr int kWideLC = 16;                                  // l-chunk of G per stage

template <int CP>
struct WideCfg {
    static constexpr int LD = CP + 1;
    static constexpr int KT = CP / 16;                       // k per thread
    static size_t smem() {
        return sizeof(double) * ((size_t)2 * kWideRows * LD + (size_t)2 * kWideLC * CP);
    }
};

template <int CP>
__global__ void __launch_bounds__(kWideThreads) k_step_wide(Bufs b, Geo g) {
    DevState* st = b.st;
    if (st->done) return;
    constexpr int LD = WideCfg<CP>::LD;
    constexpr int KT = WideCfg<CP>::KT;
    constexpr int R = kWideRows;
    extern __shared__ double smw[];
    double* TX = smw;
    double* TY = TX + R * LD;
    double* GS = TY + R * LD;                                // [2][kWideLC][CP]
    __shared__ double thr_s[R];
    __shared__ int flag_s[R];
    const int C = (int)g.C;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int mode = st->step_mode;
    const double* __restrict__ A = b.U[st->step_a];
    const double* __restrict__ Bp = b.U[st->step_b];
    double* __restrict__ D = b.U[st->step_dst];
    const double beta = st->beta_step;
    const double tau = st->tau;
    const int sel = st->step_sel;
    const double* __restrict__ XS = b.xs[st->xs_r * 2 + sel];
    const double* __restrict__ Gt = b.gfull[sel];
    const int rg = tid / 16, kg = tid % 16;                  // GEMM: rows 4rg..4rg+3, k = kg + 16 j
    const int pr = tid / 4, pq = tid % 4;                    // projection: row pr, quarter pq
    const unsigned qmask = 0xFu << (lane & ~3);
    bool bad = false;

    for (unsigned long long rb = (unsigned long long)blockIdx.x * R; rb < g.nrows;
         rb += (unsigned long long)gridDim.x * R) {
        const int rows = (int)min((unsigned long long)R, g.nrows - rb);
        // 1: stage rows through cp.async: A -> TX, B -> TY, X_ext formed in place in TX,
        //    then S X_ext -> TY, which lands while the GEMM runs
        for (int e = tid; e < rows * CP; e += kWideThreads) {
            const int r = e / CP, k = e % CP;                // CP constexpr: shifts
            if (k < C) {
                const size_t a = (size_t)(g.row0 + rb + r) * C + k;
                cp_async8(TX + r * LD + k, A + a);
                if (mode != kLiteral) cp_async8(TY + r * LD + k, Bp + a);
            }
        }
        cp_async_commit();
        cp_async_wait_all();
        __syncthreads();
        if (mode != kLiteral) {
            for (int e = tid; e < rows * CP; e += kWideThreads) {
                const int r = e / CP, k = e % CP;
                if (k < C) TX[r * LD + k] = extrap(TX[r * LD + k], TY[r * LD + k], beta);
            }
            __syncthreads();
        }
        for (int e = tid; e < rows * CP; e += kWideThreads) {
            const int r = e / CP, k = e % CP;
            if (k < C) cp_async8(TY + r * LD + k, XS + (size_t)(rb + r) * C + k);
        }
        cp_async_commit();
        // 2: GEMM over l-chunks of G
        auto stage_g = [&](int buf, int l0) {
            const int nl = min(kWideLC, C - l0);
            double* dst = GS + (size_t)buf * kWideLC * CP;
            for (int e = tid; e < nl * C; e += kWideThreads) {
                const int l = e / C, k = e % C;
                cp_async8(dst + l * CP + k, Gt + (size_t)(l0 + l) * C + k);
            }
            cp_async_commit();
        };
        double o[4][KT];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < KT; ++j) o[i][j] = 0.0;
        stage_g(0, 0);
        int buf = 0;
        for (int l0 = 0; l0 < C; l0 += kWideLC, buf ^= 1) {
            // groups in flight: S X_ext rows, G chunk l0 [, G chunk l0 + LC]; the rows'
            // group is the oldest, so waiting for chunk l0 covers it too
            if (l0 + kWideLC < C) {
                stage_g(buf ^ 1, l0 + kWideLC);
                cp_async_wait_1();
            } else {
                cp_async_wait_all();
            }
            __syncthreads();
            const double* gb = GS + (size_t)buf * kWideLC * CP + kg;
            const int nl = min(kWideLC, C - l0);
            for (int l = 0; l < nl; ++l) {
                double xv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) xv[i] = TX[(4 * rg + i) * LD + l0 + l];
                double gv[KT];
#pragma unroll
                for (int j = 0; j < KT; ++j) gv[j] = gb[l * CP + 16 * j];   // k = kg + 16 j
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < KT; ++j) o[i][j] = dadd(o[i][j], dmul(gv[j], xv[i]));
            }
            __syncthreads();
        }
        // 3: grad and step (objective.hpp:116-117, solver.hpp:102)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = 4 * rg + i;
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                const int k = kg + 16 * j;
                if (r < rows && k < C) {
                    const double grad = dmul(-4.0, dsub(TY[r * LD + k], o[i][j]));
                    TY[r * LD + k] = dsub(TX[r * LD + k], dmul(tau, grad));
                }
            }
        }
        __syncthreads();
        // 4: projection, 4 lanes per row
        const bool live = pr < rows;
        double* ty = TY + pr * LD;
        double* tx = TX + pr * LD;
        bool fin = true;
        for (int k = pq; k < C; k += 4)
            if (live && !isfinite(ty[k])) fin = false;
        const bool row_fin = __all_sync(qmask, fin);
        if (live && !row_fin) bad = true;
        const bool work = live && row_fin && C > 1;
        for (int k = pq; k < CP; k += 4) tx[k] = (work && k < C) ? ty[k] : -INFINITY;
        __syncwarp();
        // bitonic network over the row copy: each of the 4 lanes takes every 4th
        // compare-exchange pair of a stage (pair p -> lower index = p with a 0 bit
        // inserted at log2(jj)), a fixed trip count so the loads pipeline
        {
            constexpr int LOGCP = CP == 64 ? 6 : (CP == 128 ? 7 : 8);
            for (int ks = 1; ks <= LOGCP; ++ks) {
                for (int js = ks - 1; js >= 0; --js) {
                    const int jj = 1 << js;
#pragma unroll 8
                    for (int t = 0; t < CP / 8; ++t) {
                        const int pp = pq + 4 * t;
                        const int i = ((pp >> js) << (js + 1)) | (pp & (jj - 1));
                        const int l = i | jj;
                        const double a = tx[i], c2 = tx[l];
                        const bool sw = ((i >> ks) & 1) == 0 ? (a < c2) : (c2 < a);
                        tx[i] = sw ? c2 : a;
                        tx[l] = sw ? a : c2;
                    }
                    __syncwarp();
                }
            }
        }
        if (pq == 0 && work) {
            double cs = 0.0, a_star = 0.0;
            int k_star = -1;
            for (int k = 0; k < C; ++k) {
                cs = dadd(cs, tx[k]);
                const double a = dsub(cs, 1.0);
                if (threshold_cond(tx[k], a, (double)(k + 1))) {
                    k_star = k;
                    a_star = a;
                }
            }
            thr_s[pr] = k_star >= 0 ? a_star / (double)(k_star + 1) : 0.0;
        }
        __syncwarp();
        if (work) {
            const double thr = thr_s[pr];
            for (int k = pq; k < C; k += 4) ty[k] = ref_max(dsub(ty[k], thr), 0.0);
        }
        __syncwarp();
        // residual folds: sequential sum by lane pq == 0, max / ties by the 4 lanes
        for (int round = 0; round < 4; ++round) {
            if (pq == 0) {
                double sum = 0.0;
                if (work)
                    for (int k = 0; k < C; ++k) sum = dadd(sum, ty[k]);
                const double residual = dsub(sum, 1.0);
                thr_s[pr] = residual;
                flag_s[pr] = work && residual != 0.0;
            }
            __syncwarp();
            const bool go = flag_s[pr] != 0;
            double top = -INFINITY;
            if (go)
                for (int k = pq; k < C; k += 4) top = (top < ty[k]) ? ty[k] : top;
#pragma unroll
            for (int o2 = 1; o2 < 4; o2 <<= 1) {
                const double v = __shfl_xor_sync(qmask, top, o2);
                top = (top < v) ? v : top;
            }
            int ties = 0;
            if (go)
                for (int k = pq; k < C; k += 4) ties += (ty[k] == top);
#pragma unroll
            for (int o2 = 1; o2 < 4; o2 <<= 1) ties += __shfl_xor_sync(qmask, ties, o2);
            if (go) {
                const double share = thr_s[pr] / (double)ties;
                for (int k = pq; k < C; k += 4)
                    if (ty[k] == top) ty[k] = ref_max(dsub(ty[k], share), 0.0);
            }
            __syncwarp();
            if (!__any_sync(0xffffffffu, go)) break;
        }
        if (live && row_fin && C == 1 && pq == 0) ty[0] = 1.0;
        __syncthreads();
        // 5: store bar^n
        for (int e = tid; e < rows * CP; e += kWideThreads) {
            const int r = e / CP, k = e % CP;
            if (k < C) D[(size_t)(g.row0 + rb + r) * C + k] = TY[r * LD + k];
        }
        __syncthreads();
    }
    if (bad) {
        st->error = 1;
        st->done = 1;
    }
}

// =============================================================================
// K3 for 32 < C <= 128 (no backtracking terms), v2: G resident in shared memory
// for the whole launch, batches of 32 rows per CTA of 256 threads:
//   1 X_ext rows -> TX (formed in registers, solver.hpp:261), S X_ext -> TY (cp.async)
//   2 gradient as a register-tiled GEMM: thread (row group of 4 = its warp, KT = CP/32
//     components k = 64p + 2kg + {0,1}) accumulates o[r][k] = sum_{l ascending}
//     G[k][l] x_r[l] -- each output one sequential DMUL+DADD chain, the reference's
//     order (objective.hpp:37-43); no barrier inside the l loop
//   3 y = x - tau (-4 (xs - o)) in place of xs (objective.hpp:116-117, solver.hpp:102)
//   4 projection (simplex.hpp:18-59): 8 lanes per row hold VPL = CP/8 values each and
//     run a register bitonic network (in-lane stages, cross-lane stages by shuffle);
//     the sorted row goes to TX, where one thread per row does the sequential cumsum /
//     threshold and the residual folds (sequential sums in index order)
//   5 coalesced store of bar^n.
// Padding: G is zero outside C x C and x is zero beyond C, so the padded GEMM terms
// add +0 to chains that start at +0 and can never be -0: exact.
// =============================================================================
constexpr int kW2Threads = 256;                             // NG = 256 / GT independent groups

template <int CP>
struct Wide2Cfg {
    static constexpr int LD = CP + 1;
    static constexpr int KT = CP / 32;                      // k per thread in the GEMM
    static constexpr int VPL = CP / 8;                      // values per lane in the projection
    // threads per group (measured: CP = 128 -> 128 threads: E128 step 26.2 vs 30.2 ms with 64;
    // CP = 64 -> 64 threads: E64 step 11.2 vs 11.9 ms with 128)
    static constexpr int GT = CP == 64 ? 64 : 128;
    static constexpr int NG = kW2Threads / GT;
    static constexpr int R = GT / 8;                        // rows per group batch (8 lanes per row)
    static size_t smem() { return sizeof(double) * ((size_t)CP * CP + (size_t)NG * 3 * R * LD); }
};

// barrier of one group (ids 1..NG; 0 is __syncthreads)
template <int GT>
__device__ __forceinline__ void group_sync(int grp) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(GT) : "memory");
}

template <int CP, bool TOL = false>
__global__ void __launch_bounds__(kW2Threads, 1) k_step_wide2(Bufs b, Geo g) {
    DevState* st = b.st;
    if (st->done) return;
    constexpr int LD = Wide2Cfg<CP>::LD;
    constexpr int KT = Wide2Cfg<CP>::KT;
    constexpr int VPL = Wide2Cfg<CP>::VPL;
    constexpr int R = Wide2Cfg<CP>::R;
    constexpr int kW2Group = Wide2Cfg<CP>::GT;
    extern __shared__ double smw2[];
    // two groups of 128 threads share G and work on separate 16-row batches with their own
    // tiles and barriers, so one group's FP64 GEMM overlaps the other's projection
    const int grp = threadIdx.x / kW2Group;
    const int tid = threadIdx.x % kW2Group;
    double* GS = smw2;                                       // GS[l*CP + k] = G[k][l]
    double* TX = GS + CP * CP + (size_t)grp * 3 * R * LD;
    constexpr int NG = Wide2Cfg<CP>::NG;
    double* TY = TX + R * LD;
    double* CS = TY + R * LD;                                // running sums of the sorted rows
    const int C = (int)g.C;
    const StepPlan sp = step_plan(b);
    {
        const double* __restrict__ Gt = b.gfull[st->step_sel];   // Gt[l*C + k] == G[k][l]
        for (int e = threadIdx.x; e < CP * CP; e += kW2Threads) {
            const int l = e / CP, k = e % CP;
            GS[e] = (l < C && k < C) ? Gt[l * C + k] : 0.0;
        }
    }
    __syncthreads();
    const int rg = tid >> 5, kg = tid & 31;                  // GEMM: rows 4rg..4rg+3 (rg < 4), k map below
    const int pr = tid >> 3, pq = tid & 7;                   // projection: row pr, lane pq of 8
    const unsigned gmask = 0xFFu << ((tid & 31) & ~7);
    bool bad = false;
    for (unsigned long long rb = ((unsigned long long)blockIdx.x * NG + grp) * R; rb < g.nrows;
         rb += (unsigned long long)gridDim.x * NG * R) {
        const int rows = (int)min((unsigned long long)R, g.nrows - rb);
        group_sync<kW2Group>(grp);                                     // previous batch's tiles consumed
        // 1: A -> TX, B -> TY (cp.async), X_ext formed in place in TX (solver.hpp:261), then
        //    S X_ext -> TY, which lands while the GEMM runs (it is read only after it)
#pragma unroll 4
        for (int e = tid; e < R * CP; e += kW2Group) {
            const int r = e / CP, k = e % CP;
            if (r < rows && k < C) {
                const size_t a = (size_t)(g.row0 + rb + r) * C + k;
                cp_async8(TX + r * LD + k, sp.A + a);
                if (sp.mode != kLiteral) cp_async8(TY + r * LD + k, sp.Bp + a);
            } else {
                TX[r * LD + k] = 0.0;                        // padding: x_l = 0 beyond C
            }
        }
        cp_async_commit();
        cp_async_wait_all();
        group_sync<kW2Group>(grp);
        if (sp.mode != kLiteral) {
#pragma unroll 4
            for (int e = tid; e < rows * CP; e += kW2Group) {
                const int r = e / CP, k = e % CP;
                if (k < C) TX[r * LD + k] = extrap(TX[r * LD + k], TY[r * LD + k], sp.beta);
            }
            group_sync<kW2Group>(grp);
        }
#pragma unroll 4
        for (int e = tid; e < rows * CP; e += kW2Group) {
            const int r = e / CP, k = e % CP;
            if (k < C) {
                const size_t q = (size_t)(rb + r) * C + k;
                cp_async8(TY + r * LD + k, sp.XS + q);
                if (TOL && sp.mode != kLiteral) cp_async8(CS + r * LD + k, sp.XSB + q);   // S bar_prev
            }
        }
        cp_async_commit();
        // 2: GEMM
        double o[4][KT];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < KT; ++j) o[i][j] = 0.0;
        {
            const double* xrow = TX + (4 * rg) * LD;
            // lane kg owns components k = 64 p + 2 kg + {0, 1} (p < KT/2): each double2 load of
            // a G row is then 16 consecutive bytes per lane, conflict-free across the warp
            const double* gcol = GS + 2 * kg;
            // register double buffer: the operands of l + 1 are loaded while l is multiplied
            double xa[4], ga[KT], xb[4], gb[KT];
            auto load = [&](double (&xv)[4], double (&gv)[KT], int l) {
#pragma unroll
                for (int i = 0; i < 4; ++i) xv[i] = xrow[i * LD + l];
#pragma unroll
                for (int j = 0; j < KT; j += 2) {
                    const double2 t = *reinterpret_cast<const double2*>(gcol + l * CP + 32 * j);
                    gv[j] = t.x;
                    gv[j + 1] = t.y;
                }
            };
            auto fma_step = [&](const double (&xv)[4], const double (&gv)[KT]) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < KT; ++j) o[i][j] = madd<TOL>(o[i][j], gv[j], xv[i]);
            };
            load(xa, ga, 0);
#pragma unroll 2
            for (int l = 0; l < CP; l += 2) {
                load(xb, gb, l + 1);
                fma_step(xa, ga);
                if (l + 2 < CP) load(xa, ga, l + 2);
                fma_step(xb, gb);
            }
        }
        // 3: grad and step, in place of xs
        cp_async_wait_all();
        group_sync<kW2Group>(grp);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = 4 * rg + i;
#pragma unroll
            for (int j = 0; j < KT; ++j) {
                const int k = 32 * (j & ~1) + 2 * kg + (j & 1);   // the GEMM's component map
                if (r < rows && k < C) {
                    double xsv = TY[r * LD + k];
                    if (TOL && sp.mode != kLiteral)          // S X_ext = S bar + beta (S bar - S bar_prev)
                        xsv = extrap(xsv, CS[r * LD + k], sp.beta);
                    const double grad = dmul(-4.0, dsub(xsv, o[i][j]));
                    TY[r * LD + k] = dsub(TX[r * LD + k], dmul(sp.tau, grad));
                }
            }
        }
        group_sync<kW2Group>(grp);
        // 4: projection, warp-local: warp w owns rows 4w..4w+3, 8 lanes per row
        // 4a: finiteness, register bitonic sort (descending) -> TX (x is dead)
        const bool live = pr < rows;
        double v[VPL];
        bool fin = true;
#pragma unroll
        for (int m = 0; m < VPL; ++m) {
            const int k = VPL * pq + m;
            const double y = (live && k < C) ? TY[pr * LD + k] : -INFINITY;
            if (live && k < C && !isfinite(y)) fin = false;
            v[m] = y;
        }
        const bool row_fin = __all_sync(gmask, fin);
        if (live && !row_fin) bad = true;
        const bool work = live && row_fin && C > 1;
        double* yrow = TY + pr * LD;
        if constexpr (TOL) {
            // tolerance mode: sort-free Michelot threshold over the 8 lanes' slots
            // (michelot_threshold's iteration; partial sums reduced across the lanes)
            if (work) {
                double sum = 0.0;
#pragma unroll
                for (int m = 0; m < VPL; ++m)
                    if (VPL * pq + m < C) sum += v[m];
#pragma unroll
                for (int o2 = 1; o2 < 8; o2 <<= 1) sum += __shfl_xor_sync(gmask, sum, o2);
                int cnt = C;
                double thr = (sum - 1.0) / (double)cnt;
                for (int it = 0; it < C; ++it) {
                    double s2 = 0.0;
                    int c2 = 0;
#pragma unroll
                    for (int m = 0; m < VPL; ++m)
                        if (VPL * pq + m < C && v[m] > thr) {
                            s2 += v[m];
                            ++c2;
                        }
#pragma unroll
                    for (int o2 = 1; o2 < 8; o2 <<= 1) {
                        s2 += __shfl_xor_sync(gmask, s2, o2);
                        c2 += __shfl_xor_sync(gmask, c2, o2);
                    }
                    if (c2 == cnt || c2 == 0) break;
                    cnt = c2;
                    thr = (s2 - 1.0) / (double)cnt;
                }
#pragma unroll
                for (int m = 0; m < VPL; ++m) {
                    const int k = VPL * pq + m;
                    if (k < C) yrow[k] = ref_max(v[m] - thr, 0.0);
                }
            } else if (live && row_fin && C == 1 && pq == 0) {
                yrow[0] = 1.0;
            }
        } else {
#pragma unroll
        for (int kk = 2; kk <= CP; kk <<= 1) {
#pragma unroll
            for (int j = kk >> 1; j > 0; j >>= 1) {
                if (j >= VPL) {                              // partner in lane pq ^ (j / VPL), same slot
                    const int i0 = VPL * pq;
                    const bool lower = (i0 & j) == 0;
                    const bool keep_max = lower == ((i0 & kk) == 0);
#pragma unroll
                    for (int m = 0; m < VPL; ++m) {
                        const double p = __shfl_xor_sync(gmask, v[m], j / VPL);
                        const double mx = (v[m] < p) ? p : v[m];
                        const double mn = (v[m] < p) ? v[m] : p;
                        v[m] = keep_max ? mx : mn;
                    }
                } else {
#pragma unroll
                    for (int m = 0; m < VPL; ++m) {
                        const int l = m ^ j;
                        if (l > m) {
                            const int i = VPL * pq + m;
                            const double a = v[m], c2 = v[l];
                            const bool sw = ((i & kk) == 0) ? (a < c2) : (c2 < a);
                            v[m] = sw ? c2 : a;
                            v[l] = sw ? a : c2;
                        }
                    }
                }
            }
        }
        double* srow = TX + pr * LD;                         // sorted values
        double* crow = CS + pr * LD;                         // their running sums
#pragma unroll
        for (int m = 0; m < VPL; ++m) srow[VPL * pq + m] = v[m];
        __syncwarp();
        // 4b: the only sequential part of the threshold (simplex.hpp:29-36): cs_k = cs_{k-1} + s_k,
        //     one lane per row; the tests then run on all 8 lanes of the row
        if (pq == 0 && work) {
            double cs = 0.0;
            for (int k = 0; k < C; ++k) {
                cs = dadd(cs, srow[k]);
                crow[k] = cs;
            }
        }
        __syncwarp();
        int kbest = -1;                                      // last k whose test holds
        if (work) {
#pragma unroll
            for (int m = 0; m < VPL; ++m) {
                const int k = VPL * pq + m;
                if (k < C && threshold_cond(srow[k], dsub(crow[k], 1.0), (double)(k + 1))) kbest = k;
            }
        }
#pragma unroll
        for (int o2 = 1; o2 < 8; o2 <<= 1) kbest = max(kbest, __shfl_xor_sync(gmask, kbest, o2));
        if (work) {
            const double thr = kbest >= 0 ? dsub(crow[kbest], 1.0) / (double)(kbest + 1) : 0.0;
#pragma unroll
            for (int m = 0; m < VPL; ++m) {                  // 4c: clip
                const int k = VPL * pq + m;
                if (k < C) yrow[k] = ref_max(dsub(yrow[k], thr), 0.0);
            }
        } else if (live && row_fin && C == 1 && pq == 0) {
            yrow[0] = 1.0;
        }
        __syncwarp();
        // 4d: residual folds (simplex.hpp:43-55): the sum in index order by one lane, max /
        //     ties / update on the 8 lanes
        for (int round = 0; round < 4; ++round) {
            double residual = 0.0;
            if (pq == 0 && work) {
                double sum = 0.0;
                for (int k = 0; k < C; ++k) sum = dadd(sum, yrow[k]);
                residual = dsub(sum, 1.0);
            }
            residual = __shfl_sync(gmask, residual, (tid & 31) & ~7);
            const bool go = work && residual != 0.0;
            if (!__any_sync(0xffffffffu, go)) break;
            double top = -INFINITY;
            if (go)
                for (int k = pq; k < C; k += 8) top = (top < yrow[k]) ? yrow[k] : top;
#pragma unroll
            for (int o2 = 1; o2 < 8; o2 <<= 1) {
                const double t2 = __shfl_xor_sync(gmask, top, o2);
                top = (top < t2) ? t2 : top;
            }
            int ties = 0;
            if (go)
                for (int k = pq; k < C; k += 8) ties += (yrow[k] == top);
#pragma unroll
            for (int o2 = 1; o2 < 8; o2 <<= 1) ties += __shfl_xor_sync(gmask, ties, o2);
            __syncwarp();
            if (go) {
                const double share = residual / (double)ties;
                for (int k = pq; k < C; k += 8)
                    if (yrow[k] == top) yrow[k] = ref_max(dsub(yrow[k], share), 0.0);
            }
            __syncwarp();
        }
        }
        group_sync<kW2Group>(grp);
        // 5: store bar^n
        for (int e = tid; e < rows * CP; e += kW2Group) {
            const int r = e / CP, k = e % CP;
            FC_DCHECK(g.row0 + rb + r < g.N);
            if (k < C) sp.D[(size_t)(g.row0 + rb + r) * C + k] = TY[r * LD + k];
        }
    }
    if (bad) {
        st->error = 1;
        st->done = 1;
    }
}

inline size_t step_t_smem(int G) { return sizeof(double) * ((size_t)G * G + (kStepThreads / 32) * 3 * 32 * (G + 1)); }

// Batched in-place projection, C <= 32, thread per row (init_membership's
// per-column projection and project_simplex): the step kernel's projection
// (register bitonic sort, exact threshold, mask folds) without the gradient.
// A warp stages 32 rows through a [32][G+1] tile (coalesced both ways).
template <int G, bool EXACT>
__global__ void __launch_bounds__(128) k_project_t(double* x, unsigned long long rows, int C, unsigned* bad_flag) {
    constexpr int LD = G + 1;
    constexpr int RPW = 32 / G;
    __shared__ double tiles[4][32 * LD];
    const unsigned lane = threadIdx.x & 31u;
    const int lg = (int)(lane % G);
    const int sub = (int)(lane / G);
    double* T = tiles[threadIdx.x >> 5];
    double* tr = T + lane * LD;
    const bool lane_ok = EXACT || lg < C;
    const unsigned long long warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    bool bad = false;
    for (unsigned long long rb = w0 * 32; rb < rows; rb += warps * 32) {
        for (int p = 0; p < 32; p += RPW) {
            const unsigned long long row = rb + p + sub;
            if (row < rows && lane_ok) T[(p + sub) * LD + lg] = x[row * C + lg];
        }
        __syncwarp();
        if (rb + lane < rows) {
            double w[G];
            bool fin = true;
#pragma unroll
            for (int k = 0; k < G; ++k) {
                w[k] = (EXACT || k < C) ? tr[k] : 0.0;
                if ((EXACT || k < C) && !isfinite(w[k])) fin = false;
            }
            if (!fin) {
                bad = true;
            } else if (C == 1) {
                tr[0] = 1.0;
            } else {
                const double thr = row_threshold<G>(tr, C);
#pragma unroll
                for (int k = 0; k < G; ++k) w[k] = (EXACT || k < C) ? ref_max(dsub(w[k], thr), 0.0) : 0.0;
                fold_residual<G>(w, C);
#pragma unroll
                for (int k = 0; k < G; ++k)
                    if (EXACT || k < C) tr[k] = w[k];
            }
        }
        __syncwarp();
        for (int p = 0; p < 32; p += RPW) {
            const unsigned long long row = rb + p + sub;
            if (row < rows && lane_ok) x[row * C + lg] = T[(p + sub) * LD + lg];
        }
        __syncwarp();
    }
    if (bad) atomicOr(bad_flag, 1u);
}

// Batched in-place projection (init_membership's per-column projection).
template <int G, int S>
__global__ void __launch_bounds__(256) k_project(double* x, unsigned long long rows, int C,
                                                 unsigned* bad_flag) {
    __shared__ double smp[256 / 32][32 / G][G * S];
    const unsigned lane = threadIdx.x & 31u;
    const int lg = (int)(lane % G);
    const int sub = (int)(lane / G);
    double* sm = &smp[threadIdx.x >> 5][sub][0];
    const unsigned long long warps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    constexpr int RPW = 32 / G;
    for (unsigned long long rb = w0 * RPW; rb < rows; rb += warps * RPW) {
        const unsigned long long row = rb + sub;
        const bool active = row < rows;
        double y[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int r = lg + s * G;
            y[s] = (active && r < C) ? x[row * C + r] : 0.0;
        }
        const bool ok = project_group<G, S>(y, C, lg, sm);
        if (!ok && active) atomicOr(bad_flag, 1u);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int r = lg + s * G;
            if (active && r < C) x[row * C + r] = y[s];
        }
    }
}

// x0.validate(1e-9) (membership.hpp:49-61): non-finite flag + max feasibility
// error (max is order independent; the per-column sum is sequential).
__global__ void __launch_bounds__(256) k_validate(const double* x, unsigned long long n, int C, DevState* st) {
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double sum = 0.0, worst = 0.0;
    bool fin = true;
    for (int k = 0; k < C; ++k) {
        const double v = x[i * C + k];
        if (!isfinite(v)) fin = false;
        sum = dadd(sum, v);
        if (v < 0.0) worst = worst < -v ? -v : worst;
        if (v > 1.0) worst = worst < dsub(v, 1.0) ? dsub(v, 1.0) : worst;
    }
    const double dev = fabs(dsub(sum, 1.0));
    worst = worst < dev ? dev : worst;
    if (!fin) atomicOr(&st->nonfinite, 1u);
    else if (worst > 0.0) atomicMax(&st->err_bits, (unsigned long long)__double_as_longlong(worst));
}

}  // namespace fc
