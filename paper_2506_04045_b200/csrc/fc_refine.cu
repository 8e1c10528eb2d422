// fc_refine.cu -- the pairwise part of the second-order refinement (SURVEY.md 8(f)3,
// secondorder.hpp:132-330) without materialising a single direction.
//
// critical_cone_directions' pairs are V = e_k - e_l placed at node i (kept when
// x_il > eps_active and |g_ik - g_il| / sqrt(2) <= eps_grad_orth), enumerated node by
// node, k-major.  For such a V every sum of the reference's HVP path collapses to
// exact closed forms (the other terms are signed zeros, which never change a sum
// that starts at +0.0):
//   A = cross_share(V, X) has rows A_k = x_i, A_l = -x_i (zeros normalised to +0),
//   (V s)_i = s_ii v_i,  out_i[m] = -4 (vs_m - <A_m, x_i> - sum_m' A[m'][m] x_im'
//                                        - (B v_i)_m),  B = share_matrix(X),
//   <H V, V>_F = out_i[k] - out_i[l]   (frob_inner adds +-0 everywhere else),
// each evaluated with the reference's operation order, so q is bit-identical to
// quadratic_form(xbar, V, s) -- at O(C) per direction instead of a CSR sweep and a
// Gram (tests/test_gpu_refine.py checks it against the compiled reference).
// Condition (b) for a pair direction: only l' = k can be an active coordinate that
// V escapes, so the candidates are W = e_k' - e_k at node i with value g_ik' - g_ik.
// Both minima keep the reference's tie rule (first in enumeration order) through a
// two-pass atomicMin: value first, then the smallest (direction, k') key at it.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "fc_internal.h"
#include "fuzzyclust_cuda.h"

namespace {

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// total order of doubles as unsigned keys (for atomicMin)
__device__ __forceinline__ unsigned long long okey(double v) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(v);
    return (u >> 63) ? ~u : (u | 0x8000000000000000ULL);
}
__device__ __forceinline__ double from_okey(unsigned long long k) {
    const unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
    return __longlong_as_double((long long)u);
}

__device__ __forceinline__ bool keep_pair(const double* xi, const double* gi, int k, int l, double eps_active,
                                          double eps_orth, double sqrt2) {
    if (k == l) return false;
    if (xi[l] <= eps_active) return false;                               // -1 entry at an active zero
    if (__ddiv_rn(fabs(dsub(gi[k], gi[l])), sqrt2) > eps_orth) return false;
    return true;
}

__global__ void k_pair_count(const double* x, const double* g, unsigned long long n, int C, double eps_active,
                             double eps_orth, double sqrt2, unsigned long long* count) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const double* xi = x + i * C;
        const double* gi = g + i * C;
        unsigned long long c = 0;
        for (int k = 0; k < C; ++k)
            for (int l = 0; l < C; ++l) c += keep_pair(xi, gi, k, l, eps_active, eps_orth, sqrt2) ? 1 : 0;
        count[i] = c;
    }
}

// <H V, V> for V = e_k - e_l at node i (closed form of the reference's HVP path)
__device__ double pair_q(const double* xi, const double* B, double sii, int C, int k, int l) {
    double out[2];
    for (int t = 0; t < 2; ++t) {
        const int m = t == 0 ? k : l;
        const double vm = t == 0 ? 1.0 : -1.0;
        const double vs = dadd(0.0, dmul(sii, vm));
        double ax = 0.0, atx = 0.0, bv = 0.0;
        for (int mp = 0; mp < C; ++mp) ax = dadd(ax, dmul(dadd(0.0, dmul(vm, xi[mp])), xi[mp]));
        for (int mp = 0; mp < C; ++mp) {
            const double a = mp == k ? dadd(0.0, xi[m]) : (mp == l ? dadd(0.0, dmul(-1.0, xi[m])) : 0.0);
            atx = dadd(atx, dmul(a, xi[mp]));
        }
        for (int mp = 0; mp < C; ++mp) {
            const double v = mp == k ? 1.0 : (mp == l ? -1.0 : 0.0);
            bv = dadd(bv, dmul(B[m * C + mp], v));
        }
        out[t] = dmul(-4.0, dsub(dsub(dsub(vs, ax), atx), bv));
    }
    return dsub(out[0], out[1]);
}

// pass 1 (phase 0): minimum values; pass 2 (phase 1): smallest key attaining them
__global__ void k_pair_eval(const double* x, const double* g, const double* B, const double* diag,
                            const unsigned long long* offset, unsigned long long n, int C, double eps_active,
                            double eps_orth, double sqrt2, unsigned long long budget, int phase,
                            unsigned long long* best, unsigned* triples, unsigned long long triples_cap) {
    const double best_a = phase ? from_okey(best[0]) : 0.0;
    const double best_b = phase ? from_okey(best[2]) : 0.0;
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const double* xi = x + i * C;
        const double* gi = g + i * C;
        unsigned long long d = offset[i];
        if (d >= budget && !triples) continue;
        for (int k = 0; k < C; ++k) {
            for (int l = 0; l < C; ++l) {
                if (!keep_pair(xi, gi, k, l, eps_active, eps_orth, sqrt2)) continue;
                if (phase == 0 && triples && d < triples_cap) {
                    triples[3 * d] = (unsigned)i;
                    triples[3 * d + 1] = (unsigned)k;
                    triples[3 * d + 2] = (unsigned)l;
                }
                if (d < budget) {
                    const double q = pair_q(xi, B, diag[i], C, k, l);
                    if (phase == 0) {
                        if (q < 0.0) atomicMin(best, okey(q));
                    } else if (q == best_a && q < 0.0) {
                        atomicMin(best + 1, d);
                    }
                    if (xi[k] <= eps_active) {                            // condition (b): W = e_k' - e_k
                        for (int kp = 0; kp < C; ++kp) {
                            if (kp == k) continue;
                            const double val = dsub(gi[kp], gi[k]);
                            if (phase == 0) {
                                if (val < 0.0) atomicMin(best + 2, okey(val));
                            } else if (val == best_b && val < 0.0) {
                                atomicMin(best + 3, d * (unsigned long long)C + kp);
                            }
                        }
                    }
                }
                ++d;
            }
        }
    }
}

__global__ void k_diag(const long long* row_ptr, const unsigned* col, const double* val, unsigned long long n,
                       double* diag) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += (unsigned long long)gridDim.x * blockDim.x) {
        long long lo = row_ptr[i], hi = row_ptr[i + 1];
        while (lo < hi) {
            const long long mid = (lo + hi) / 2;
            if ((col[mid] & 0x7fffffffu) < i) lo = mid + 1;
            else hi = mid;
        }
        double d = 0.0;
        if (lo < row_ptr[i + 1] && (col[lo] & 0x7fffffffu) == i) d = val ? val[lo] : 1.0;
        diag[i] = d;
    }
}

struct Dev {
    std::vector<void*> ptrs;
    cudaStream_t s;
    explicit Dev(cudaStream_t st) : s(st) {}
    template <class T>
    cudaError_t alloc(T** p, size_t count) {
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), (count ? count : 1) * sizeof(T), s);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    ~Dev() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
    }
};

#define RT(call)                                                                                       \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess) return fc_internal_fail(ctx, FC_DEVICE, std::string("CUDA error in refine: ") + cudaGetErrorString(e_)); \
    } while (0)

}  // namespace

extern "C" int fc_refine_pairs(fc_ctx* ctx, uint32_t c, const double* x, const double* grad, double eps_active,
                               double eps_grad_orth, uint64_t budget, uint32_t* triples_out, uint64_t triples_cap,
                               fc_refine_pairs_out* out) {
    if (!ctx || !out) return fc_internal_fail(ctx, FC_INVALID, "refine: null argument");
    if (c == 0 || c > 256) return fc_internal_fail(ctx, FC_INVALID, "refine: C outside [1, 256]");
    RT(cudaSetDevice(fc_internal_device(ctx)));
    uint64_t n = 0;
    const long long* d_rp = nullptr;
    const unsigned* d_col = nullptr;
    const double* d_val = nullptr;
    int rc = fc_internal_csr(ctx, &n, &d_rp, &d_col, &d_val);
    if (rc) return rc;
    // B = share_matrix(X) through the library's Gram (same bits as fc_share_matrix)
    std::vector<double> B((size_t)c * c);
    if ((rc = fc_share_matrix(ctx, c, x, B.data()))) return rc;
    Dev dev(fc_internal_stream(ctx));
    double *dx = nullptr, *dg = nullptr, *dB = nullptr, *ddiag = nullptr;
    unsigned long long *dcount = nullptr, *doff = nullptr, *dbest = nullptr;
    unsigned* dtri = nullptr;
    RT(dev.alloc(&dx, n * c));
    RT(dev.alloc(&dg, n * c));
    RT(dev.alloc(&dB, (size_t)c * c));
    RT(dev.alloc(&ddiag, n));
    RT(dev.alloc(&dcount, n));
    RT(dev.alloc(&doff, n));
    RT(dev.alloc(&dbest, 4));
    if ((rc = fc_internal_h2d(ctx, dx, x, n * c * sizeof(double)))) return rc;
    if ((rc = fc_internal_h2d(ctx, dg, grad, n * c * sizeof(double)))) return rc;
    RT(cudaMemcpyAsync(dB, B.data(), B.size() * sizeof(double), cudaMemcpyHostToDevice, dev.s));
    const unsigned grid = (unsigned)std::min<uint64_t>((n + 127) / 128, 148ull * 16);
    const double sqrt2 = std::sqrt(2.0);
    k_diag<<<grid, 128, 0, dev.s>>>(d_rp, d_col, d_val, n, ddiag);
    k_pair_count<<<grid, 128, 0, dev.s>>>(dx, dg, n, (int)c, eps_active, eps_grad_orth, sqrt2, dcount);
    // exclusive scan of the per-node counts (host: n words, once per refine)
    std::vector<unsigned long long> cnt(n);
    RT(cudaMemcpyAsync(cnt.data(), dcount, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost, dev.s));
    RT(cudaStreamSynchronize(dev.s));
    uint64_t total = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t ci = cnt[i];
        cnt[i] = total;
        total += ci;
    }
    RT(cudaMemcpyAsync(doff, cnt.data(), n * sizeof(unsigned long long), cudaMemcpyHostToDevice, dev.s));
    if (triples_out && total) RT(dev.alloc(&dtri, 3 * std::min<uint64_t>(total, triples_cap)));
    const unsigned long long init[4] = {~0ULL, ~0ULL, ~0ULL, ~0ULL};
    RT(cudaMemcpyAsync(dbest, init, sizeof init, cudaMemcpyHostToDevice, dev.s));
    for (int phase = 0; phase < 2; ++phase)
        k_pair_eval<<<grid, 128, 0, dev.s>>>(dx, dg, dB, ddiag, doff, n, (int)c, eps_active, eps_grad_orth, sqrt2,
                                             budget, phase, dbest, phase == 0 ? dtri : nullptr,
                                             std::min<uint64_t>(total, triples_cap));
    unsigned long long best[4];
    RT(cudaMemcpyAsync(best, dbest, sizeof best, cudaMemcpyDeviceToHost, dev.s));
    if (dtri) RT(cudaMemcpyAsync(triples_out, dtri, 3 * std::min<uint64_t>(total, triples_cap) * sizeof(unsigned),
                                 cudaMemcpyDeviceToHost, dev.s));
    RT(cudaStreamSynchronize(dev.s));
    auto val_of = [](unsigned long long k) {
        const unsigned long long u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
        double d;
        std::memcpy(&d, &u, sizeof d);
        return d;
    };
    std::memset(out, 0, sizeof *out);
    out->pairs = total;
    out->a_worst = best[0] == ~0ULL ? 0.0 : val_of(best[0]);
    out->a_index = best[0] == ~0ULL ? UINT64_MAX : best[1];
    out->b_worst = best[2] == ~0ULL ? 0.0 : val_of(best[2]);
    out->b_index = best[2] == ~0ULL ? UINT64_MAX : best[3] / c;
    out->b_plus = best[2] == ~0ULL ? 0u : (uint32_t)(best[3] % c);
    // locate the (node, k, l) of the two winning directions from the offsets
    auto locate = [&](uint64_t d, uint32_t* node, uint32_t* kk, uint32_t* ll) {
        uint64_t lo = 0, hi = n;                                 // last node with offset <= d
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) / 2;
            if (cnt[mid] <= d) lo = mid;
            else hi = mid;
        }
        *node = (uint32_t)lo;
        const double* xi = x + lo * c;
        const double* gi = grad + lo * c;
        uint64_t t = cnt[lo];
        for (uint32_t k = 0; k < c; ++k)
            for (uint32_t l = 0; l < c; ++l) {
                if (k == l || !(xi[l] > eps_active) || std::fabs(gi[k] - gi[l]) / sqrt2 > eps_grad_orth) continue;
                if (t++ == d) {
                    *kk = k;
                    *ll = l;
                    return;
                }
            }
    };
    if (out->a_index != UINT64_MAX) locate(out->a_index, &out->a_col, &out->a_plus, &out->a_minus);
    if (out->b_index != UINT64_MAX) {
        uint32_t node, k, l;
        locate(out->b_index, &node, &k, &l);
        out->b_col = node;
        out->b_minus = k;          // W = e_k' - e_k at the node (k' in b_plus)
        out->b_base_plus = k;
        out->b_base_minus = l;
    }
    return FC_OK;
}
