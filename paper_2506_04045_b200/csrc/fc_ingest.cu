// fc_ingest.cu -- edge-list ingest at scale: the reference's
// load_pipeline (tools/fuzzyclust.cpp:62-89) = parse_edge_list (graph.hpp:63-103)
// -> largest_connected_component_nodes (graph.hpp:146-169) -> induced_subgraph
// (graph.hpp:107-120) -> optional two_core_nodes (graph.hpp:185-213).
//
// Text is parsed on the host by all cores (chunks split at newlines; the first
// error in line order is reported with the reference's message).  Everything
// after the tokens is on the device:
//   * id compaction by FIRST APPEARANCE: tokens (id, position) radix-sorted by id
//     (stable, so each id's run starts at its first position), run heads sorted
//     by position -> rank = compacted id, scattered back to the tokens;
//   * edges: self-loops dropped, (min, max) packed into 64-bit keys, radix sort +
//     unique (normalize_edges);
//   * components: union-find with min-hooking (atomicMin on roots) + pointer
//     jumping until no edge joins two roots; each component's root is its
//     smallest node, so "largest, ties to the smallest id" (the reference's BFS
//     labelling order) is one 64-bit atomicMax over (size, ~root);
//   * 2-core: frontier peeling of degree <= 1 nodes over a CSR of the LCC (the
//     2-core is unique whatever the order);
//   * induced subgraphs: exclusive scan of the keep mask (order-preserving ids),
//     so the filtered edge list stays sorted and unique.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cctype>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "fc_internal.h"
#include "fuzzyclust_cuda.h"

namespace {

// ---- host parser: std::istringstream >> int64 semantics --------------------------
inline bool is_ws(char ch) { return ch == ' ' || ch == '\t' || ch == '\n' || ch == '\v' || ch == '\f' || ch == '\r'; }

// operator>>(long long&): skip whitespace, optional sign, >= 1 digit, stop at the
// first non-digit; overflow fails.
bool read_int64(const char*& p, const char* end, int64_t& out) {
    while (p < end && is_ws(*p)) ++p;
    const char* q = p;
    bool neg = false;
    if (q < end && (*q == '+' || *q == '-')) {
        neg = *q == '-';
        ++q;
    }
    if (q >= end || *q < '0' || *q > '9') return false;
    unsigned long long mag = 0;
    const unsigned long long lim = neg ? (unsigned long long)LLONG_MAX + 1ULL : (unsigned long long)LLONG_MAX;
    bool over = false;
    while (q < end && *q >= '0' && *q <= '9') {
        const unsigned d = (unsigned)(*q - '0');
        if (mag > (lim - d) / 10ULL) over = true;
        else mag = mag * 10ULL + d;
        ++q;
    }
    p = q;
    if (over) return false;
    out = neg ? (int64_t)(0ULL - mag) : (int64_t)mag;
    return true;
}

struct Chunk {
    const char* begin;
    const char* end;
    std::vector<int64_t> tok;   // a0 b0 a1 b1 ...
    uint64_t lines = 0;          // lines in the chunk
    uint64_t err_line = 0;       // 1-based within the chunk, 0 = none
    std::string err;
    bool saw_edge = false;
};

void parse_chunk(Chunk& c) {
    const char* p = c.begin;
    while (p < c.end) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(c.end - p)));
        const char* le = nl ? nl : c.end;
        ++c.lines;
        const char* f = p;
        while (f < le && (*f == ' ' || *f == '\t' || *f == '\r')) ++f;
        if (f < le && *f != '#') {
            const char* q = p;
            int64_t a = 0, b = 0;
            if (!read_int64(q, le, a) || !read_int64(q, le, b)) {
                c.err_line = c.lines;
                c.err = "expected two integer tokens, got \"" + std::string(p, le) + "\"";
                return;
            }
            while (q < le && is_ws(*q)) ++q;
            if (q < le) {
                const char* t = q;
                while (t < le && !is_ws(*t)) ++t;
                c.err_line = c.lines;
                c.err = "trailing token \"" + std::string(q, t) + "\"";
                return;
            }
            c.saw_edge = true;
            c.tok.push_back(a);
            c.tok.push_back(b);
        }
        p = nl ? nl + 1 : c.end;
    }
}

// ---- device kernels ----------------------------------------------------------------
unsigned grid_of(uint64_t items) { return (unsigned)std::min<uint64_t>((items + 255) / 256, 148ull * 32); }
#define GS(i, n) for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (n); i += (uint64_t)gridDim.x * blockDim.x)

__global__ void k_iota(uint64_t* p, uint64_t n) { GS(i, n) p[i] = i; }
__global__ void k_iota32(unsigned* p, uint64_t n) { GS(i, n) p[i] = (unsigned)i; }

// run heads of the id-sorted tokens
__global__ void k_heads(const long long* ids, uint64_t n, unsigned* head) {
    GS(i, n) head[i] = (i == 0 || ids[i] != ids[i - 1]) ? 1u : 0u;
}
// head i (run r = scan[i]) -> first position of run r
__global__ void k_run_first(const unsigned* head, const unsigned* scan, const uint64_t* pos, uint64_t n,
                            uint64_t* first_pos, long long* run_id, const long long* ids) {
    GS(i, n) if (head[i]) {
        first_pos[scan[i]] = pos[i];
        run_id[scan[i]] = ids[i];
    }
}
// ranks: runs sorted by first position -> rank[run] = order
__global__ void k_rank(const unsigned* run_sorted, uint64_t u, unsigned* rank_of_run) { GS(k, u) rank_of_run[run_sorted[k]] = (unsigned)k; }
// token i of the id-sorted order belongs to run (inclusive count of heads) - 1
__global__ void k_token_cid(const unsigned* head, const unsigned* scan, const uint64_t* pos,
                            const unsigned* rank_of_run, uint64_t n, unsigned* cid) {
    GS(i, n) cid[pos[i]] = rank_of_run[scan[i] + head[i] - 1u];
}
__global__ void k_edge_keys(const unsigned* cid, uint64_t m, unsigned long long* key, unsigned* valid) {
    GS(k, m) {
        const unsigned u = cid[2 * k], v = cid[2 * k + 1];
        valid[k] = u != v ? 1u : 0u;
        key[k] = u < v ? ((unsigned long long)u << 32 | v) : ((unsigned long long)v << 32 | u);
    }
}

// union-find: hook the larger root under the smaller one
__device__ __forceinline__ unsigned find_root(unsigned* parent, unsigned v) {
    unsigned p = parent[v];
    while (p != v) {
        const unsigned g = parent[p];
        if (g != p) parent[v] = g;   // path halving (benign race: values only decrease)
        v = p;
        p = g;
    }
    return v;
}
__global__ void k_hook(const unsigned long long* edges, uint64_t m, unsigned* parent, int* changed) {
    GS(k, m) {
        const unsigned u = (unsigned)(edges[k] >> 32), v = (unsigned)edges[k];
        const unsigned ru = find_root(parent, u), rv = find_root(parent, v);
        if (ru != rv) {
            const unsigned hi = ru > rv ? ru : rv, lo = ru > rv ? rv : ru;
            atomicMin(parent + hi, lo);
            *changed = 1;
        }
    }
}
__global__ void k_flatten(unsigned* parent, uint64_t n) { GS(v, n) parent[v] = find_root(parent, (unsigned)v); }
__global__ void k_comp_size(const unsigned* label, uint64_t n, unsigned* size) { GS(v, n) atomicAdd(size + label[v], 1u); }
__global__ void k_best(const unsigned* size, uint64_t n, unsigned long long* best) {
    GS(v, n) if (size[v]) atomicMax(best, ((unsigned long long)size[v] << 32) | (0xFFFFFFFFu - (unsigned)v));
}
__global__ void k_keep_label(const unsigned* label, uint64_t n, const unsigned long long* best, unsigned* keep) {
    const unsigned root = 0xFFFFFFFFu - (unsigned)(*best & 0xFFFFFFFFu);
    GS(v, n) keep[v] = label[v] == root ? 1u : 0u;
}

// induced subgraph: keep both ends, remap through the exclusive scan of keep
__global__ void k_sub_flags(const unsigned long long* e, uint64_t m, const unsigned* keep, unsigned* f) {
    GS(k, m) f[k] = (keep[(unsigned)(e[k] >> 32)] && keep[(unsigned)e[k]]) ? 1u : 0u;
}
__global__ void k_sub_map(unsigned long long* e, uint64_t m, const unsigned* new_id) {
    GS(k, m) {
        const unsigned u = (unsigned)(e[k] >> 32), v = (unsigned)e[k];
        e[k] = ((unsigned long long)new_id[u] << 32) | new_id[v];
    }
}

// 2-core peeling over CSR adjacency
__global__ void k_adj_pairs(const unsigned long long* e, uint64_t m, unsigned long long* both) {
    GS(k, m) {
        const unsigned u = (unsigned)(e[k] >> 32), v = (unsigned)e[k];
        both[2 * k] = e[k];
        both[2 * k + 1] = ((unsigned long long)v << 32) | u;
    }
}
__global__ void k_row_ptr(const unsigned long long* both, uint64_t m2, uint64_t n, unsigned long long* rp) {
    GS(v, n + 1) {
        uint64_t lo = 0, hi = m2;
        const unsigned long long x = (unsigned long long)v << 32;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if (both[mid] < x) lo = mid + 1;
            else hi = mid;
        }
        rp[v] = lo;
    }
}
__global__ void k_deg_init(const unsigned long long* rp, uint64_t n, int* deg, unsigned* removed, unsigned* frontier,
                           unsigned* fcount) {
    GS(v, n) {
        deg[v] = (int)(rp[v + 1] - rp[v]);
        if (deg[v] <= 1) {
            removed[v] = 1;
            frontier[atomicAdd(fcount, 1u)] = (unsigned)v;
        } else {
            removed[v] = 0;
        }
    }
}
// one peel round: neighbours of the frontier lose a degree; those reaching 1 join the next frontier
__global__ void k_peel(const unsigned long long* rp, const unsigned long long* both, const unsigned* frontier,
                       unsigned fsize, int* deg, unsigned* removed, unsigned* next, unsigned* ncount) {
    GS(t, fsize) {
        const unsigned v = frontier[t];
        for (unsigned long long k = rp[v]; k < rp[v + 1]; ++k) {
            const unsigned w = (unsigned)both[k];
            if (removed[w]) continue;
            if (atomicSub(deg + w, 1) == 2 && atomicExch(removed + w, 1u) == 0u) next[atomicAdd(ncount, 1u)] = w;
        }
    }
}
__global__ void k_not(const unsigned* removed, uint64_t n, unsigned* keep) { GS(v, n) keep[v] = removed[v] ? 0u : 1u; }

struct Dev {
    std::vector<void*> ptrs;
    cudaStream_t s;
    explicit Dev(cudaStream_t st) : s(st) {}
    template <class T>
    cudaError_t alloc(T** p, size_t count) {
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T), s);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    ~Dev() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
        cudaStreamSynchronize(s);
    }
};

#define IT(call)                                                                                        \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess) return fc_internal_fail(ctx, FC_DEVICE, std::string("CUDA error in ingest: ") + cudaGetErrorString(e_)); \
    } while (0)

// exclusive scan of flags (unsigned) into out; returns the total
template <class T>
int scan_count(fc_ctx* ctx, Dev& dev, const unsigned* flags, unsigned* out, uint64_t n, uint64_t* total) {
    size_t tb = 0;
    IT(cub::DeviceScan::ExclusiveSum(nullptr, tb, flags, out, (int64_t)n, dev.s));
    void* tmp = nullptr;
    IT(dev.alloc(reinterpret_cast<char**>(&tmp), tb));
    IT(cub::DeviceScan::ExclusiveSum(tmp, tb, flags, out, (int64_t)n, dev.s));
    unsigned last_f = 0, last_s = 0;
    if (n) {
        IT(cudaMemcpyAsync(&last_f, flags + n - 1, 4, cudaMemcpyDeviceToHost, dev.s));
        IT(cudaMemcpyAsync(&last_s, out + n - 1, 4, cudaMemcpyDeviceToHost, dev.s));
    }
    IT(cudaStreamSynchronize(dev.s));
    *total = n ? (uint64_t)last_f + last_s : 0;
    return FC_OK;
}

// compact the 64-bit edge keys where flag == 1 (order kept)
int select_edges(fc_ctx* ctx, Dev& dev, unsigned long long* in, const unsigned* flags, uint64_t m,
                 unsigned long long** out, uint64_t* kept) {
    unsigned long long* o = nullptr;
    uint64_t* d_num = nullptr;
    IT(dev.alloc(&o, m));
    IT(dev.alloc(&d_num, 1));
    size_t tb = 0;
    IT(cub::DeviceSelect::Flagged(nullptr, tb, in, flags, o, d_num, (int64_t)m, dev.s));
    void* tmp = nullptr;
    IT(dev.alloc(reinterpret_cast<char**>(&tmp), tb));
    IT(cub::DeviceSelect::Flagged(tmp, tb, in, flags, o, d_num, (int64_t)m, dev.s));
    IT(cudaMemcpyAsync(kept, d_num, sizeof(uint64_t), cudaMemcpyDeviceToHost, dev.s));
    IT(cudaStreamSynchronize(dev.s));
    *out = o;
    return FC_OK;
}

// node-set step: keep[v] -> new ids, edges filtered + remapped, ids carried along
int induce(fc_ctx* ctx, Dev& dev, unsigned long long*& edges, uint64_t& m, uint64_t& n, const unsigned* keep,
           long long*& ids) {
    unsigned* new_id = nullptr;
    IT(dev.alloc(&new_id, n));
    uint64_t kept_n = 0;
    int rc = scan_count<unsigned>(ctx, dev, keep, new_id, n, &kept_n);
    if (rc) return rc;
    unsigned* f = nullptr;
    IT(dev.alloc(&f, m));
    if (m) k_sub_flags<<<grid_of(m), 256, 0, dev.s>>>(edges, m, keep, f);
    unsigned long long* e2 = nullptr;
    uint64_t m2 = 0;
    if ((rc = select_edges(ctx, dev, edges, f, m, &e2, &m2))) return rc;
    if (m2) k_sub_map<<<grid_of(m2), 256, 0, dev.s>>>(e2, m2, new_id);
    // ids of the kept nodes, in order
    long long* ids2 = nullptr;
    uint64_t* d_num = nullptr;
    IT(dev.alloc(&ids2, kept_n));
    IT(dev.alloc(&d_num, 1));
    size_t tb = 0;
    IT(cub::DeviceSelect::Flagged(nullptr, tb, ids, keep, ids2, d_num, (int64_t)n, dev.s));
    void* tmp = nullptr;
    IT(dev.alloc(reinterpret_cast<char**>(&tmp), tb));
    IT(cub::DeviceSelect::Flagged(tmp, tb, ids, keep, ids2, d_num, (int64_t)n, dev.s));
    IT(cudaStreamSynchronize(dev.s));
    edges = e2;
    m = m2;
    n = kept_n;
    ids = ids2;
    return FC_OK;
}

// LCC keep mask (graph.hpp:146-169 semantics)
int lcc_keep(fc_ctx* ctx, Dev& dev, const unsigned long long* edges, uint64_t m, uint64_t n, unsigned** keep_out) {
    unsigned *parent = nullptr, *size = nullptr, *keep = nullptr;
    int* d_changed = nullptr;
    unsigned long long* d_best = nullptr;
    IT(dev.alloc(&parent, n));
    IT(dev.alloc(&size, n));
    IT(dev.alloc(&keep, n));
    IT(dev.alloc(&d_changed, 1));
    IT(dev.alloc(&d_best, 1));
    IT(cudaMemsetAsync(size, 0, n * sizeof(unsigned), dev.s));
    k_iota32<<<grid_of(n), 256, 0, dev.s>>>(parent, n);                 // every node its own root
    for (int round = 0;; ++round) {
        if (round == 100000) return fc_internal_fail(ctx, FC_DEVICE, "ingest: connected components did not converge");
        IT(cudaMemsetAsync(d_changed, 0, sizeof(int), dev.s));
        if (m) k_hook<<<grid_of(m), 256, 0, dev.s>>>(edges, m, parent, d_changed);
        k_flatten<<<grid_of(n), 256, 0, dev.s>>>(parent, n);
        int changed = 0;
        IT(cudaMemcpyAsync(&changed, d_changed, sizeof(int), cudaMemcpyDeviceToHost, dev.s));
        IT(cudaStreamSynchronize(dev.s));
        if (!changed) break;
    }
    k_comp_size<<<grid_of(n), 256, 0, dev.s>>>(parent, n, size);
    IT(cudaMemsetAsync(d_best, 0, sizeof(unsigned long long), dev.s));
    k_best<<<grid_of(n), 256, 0, dev.s>>>(size, n, d_best);
    k_keep_label<<<grid_of(n), 256, 0, dev.s>>>(parent, n, d_best, keep);
    *keep_out = keep;
    return FC_OK;
}

// 2-core keep mask (graph.hpp:185-213 semantics)
int core_keep(fc_ctx* ctx, Dev& dev, const unsigned long long* edges, uint64_t m, uint64_t n, unsigned** keep_out) {
    unsigned long long *both = nullptr, *both_s = nullptr, *rp = nullptr;
    IT(dev.alloc(&both, 2 * m));
    IT(dev.alloc(&both_s, 2 * m));
    IT(dev.alloc(&rp, n + 1));
    if (m) k_adj_pairs<<<grid_of(m), 256, 0, dev.s>>>(edges, m, both);
    size_t tb = 0;
    IT(cub::DeviceRadixSort::SortKeys(nullptr, tb, both, both_s, (int64_t)(2 * m), 0, 64, dev.s));
    void* tmp = nullptr;
    IT(dev.alloc(reinterpret_cast<char**>(&tmp), tb));
    IT(cub::DeviceRadixSort::SortKeys(tmp, tb, both, both_s, (int64_t)(2 * m), 0, 64, dev.s));
    k_row_ptr<<<grid_of(n + 1), 256, 0, dev.s>>>(both_s, 2 * m, n, rp);
    int* deg = nullptr;
    unsigned *removed = nullptr, *fa = nullptr, *fb = nullptr, *cnt = nullptr, *keep = nullptr;
    IT(dev.alloc(&deg, n));
    IT(dev.alloc(&removed, n));
    IT(dev.alloc(&fa, n));
    IT(dev.alloc(&fb, n));
    IT(dev.alloc(&cnt, 2));
    IT(dev.alloc(&keep, n));
    IT(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned), dev.s));
    k_deg_init<<<grid_of(n), 256, 0, dev.s>>>(rp, n, deg, removed, fa, cnt);
    unsigned fsize = 0;
    IT(cudaMemcpyAsync(&fsize, cnt, 4, cudaMemcpyDeviceToHost, dev.s));
    IT(cudaStreamSynchronize(dev.s));
    while (fsize) {
        IT(cudaMemsetAsync(cnt + 1, 0, sizeof(unsigned), dev.s));
        k_peel<<<grid_of(fsize), 256, 0, dev.s>>>(rp, both_s, fa, fsize, deg, removed, fb, cnt + 1);
        IT(cudaMemcpyAsync(&fsize, cnt + 1, 4, cudaMemcpyDeviceToHost, dev.s));
        IT(cudaStreamSynchronize(dev.s));
        std::swap(fa, fb);
    }
    k_not<<<grid_of(n), 256, 0, dev.s>>>(removed, n, keep);
    *keep_out = keep;
    return FC_OK;
}

// tokens (host) -> compacted edges (device, sorted unique u < v) + original ids
int compact(fc_ctx* ctx, Dev& dev, const std::vector<int64_t>& tok, unsigned long long** edges_out, uint64_t* m_out,
            long long** ids_out, uint64_t* n_out) {
    const uint64_t t = tok.size(), m = t / 2;
    long long *ids = nullptr, *ids_s = nullptr, *run_id = nullptr;
    uint64_t *pos = nullptr, *pos_s = nullptr, *first = nullptr, *first_s = nullptr;
    unsigned *head = nullptr, *scan = nullptr, *runs = nullptr, *runs_s = nullptr, *rank = nullptr, *cid = nullptr;
    IT(dev.alloc(&ids, t));
    IT(dev.alloc(&ids_s, t));
    IT(dev.alloc(&pos, t));
    IT(dev.alloc(&pos_s, t));
    IT(dev.alloc(&head, t));
    IT(dev.alloc(&scan, t));
    IT(cudaMemcpyAsync(ids, tok.data(), t * sizeof(int64_t), cudaMemcpyHostToDevice, dev.s));
    k_iota<<<grid_of(t), 256, 0, dev.s>>>(pos, t);
    size_t tb = 0;
    IT(cub::DeviceRadixSort::SortPairs(nullptr, tb, ids, ids_s, pos, pos_s, (int64_t)t, 0, 64, dev.s));
    void* tmp = nullptr;
    IT(dev.alloc(reinterpret_cast<char**>(&tmp), tb));
    IT(cub::DeviceRadixSort::SortPairs(tmp, tb, ids, ids_s, pos, pos_s, (int64_t)t, 0, 64, dev.s));
    k_heads<<<grid_of(t), 256, 0, dev.s>>>(ids_s, t, head);
    uint64_t u = 0;
    int rc = scan_count<unsigned>(ctx, dev, head, scan, t, &u);
    if (rc) return rc;
    IT(dev.alloc(&first, u));
    IT(dev.alloc(&first_s, u));
    IT(dev.alloc(&run_id, u));
    IT(dev.alloc(&runs, u));
    IT(dev.alloc(&runs_s, u));
    IT(dev.alloc(&rank, u));
    IT(dev.alloc(&cid, t));
    k_run_first<<<grid_of(t), 256, 0, dev.s>>>(head, scan, pos_s, t, first, run_id, ids_s);
    {
        k_iota32<<<grid_of(u), 256, 0, dev.s>>>(runs, u);
        size_t tb2 = 0;
        IT(cub::DeviceRadixSort::SortPairs(nullptr, tb2, first, first_s, runs, runs_s, (int64_t)u, 0, 64, dev.s));
        void* tmp2 = nullptr;
        IT(dev.alloc(reinterpret_cast<char**>(&tmp2), tb2));
        IT(cub::DeviceRadixSort::SortPairs(tmp2, tb2, first, first_s, runs, runs_s, (int64_t)u, 0, 64, dev.s));
        IT(cudaStreamSynchronize(dev.s));
    }
    k_rank<<<grid_of(u), 256, 0, dev.s>>>(runs_s, u, rank);
    k_token_cid<<<grid_of(t), 256, 0, dev.s>>>(head, scan, pos_s, rank, t, cid);
    // original ids in compacted order: ids_by_rank[k] = run_id[runs_s[k]]
    long long* ids_rank = nullptr;
    IT(dev.alloc(&ids_rank, u));
    {
        std::vector<long long> rid(u);
        std::vector<unsigned> rs(u);
        IT(cudaMemcpyAsync(rid.data(), run_id, u * sizeof(long long), cudaMemcpyDeviceToHost, dev.s));
        IT(cudaMemcpyAsync(rs.data(), runs_s, u * sizeof(unsigned), cudaMemcpyDeviceToHost, dev.s));
        IT(cudaStreamSynchronize(dev.s));
        std::vector<long long> out(u);
        for (uint64_t k = 0; k < u; ++k) out[k] = rid[rs[k]];
        IT(cudaMemcpyAsync(ids_rank, out.data(), u * sizeof(long long), cudaMemcpyHostToDevice, dev.s));
        IT(cudaStreamSynchronize(dev.s));
    }
    // edges
    unsigned long long *key = nullptr, *key_s = nullptr;
    unsigned *valid = nullptr, *uniq = nullptr;
    IT(dev.alloc(&key, m));
    IT(dev.alloc(&key_s, m));
    IT(dev.alloc(&valid, m));
    IT(dev.alloc(&uniq, m));
    if (m) k_edge_keys<<<grid_of(m), 256, 0, dev.s>>>(cid, m, key, valid);
    unsigned long long* nz = nullptr;
    uint64_t mz = 0;
    if ((rc = select_edges(ctx, dev, key, valid, m, &nz, &mz))) return rc;
    size_t tb3 = 0;
    IT(cub::DeviceRadixSort::SortKeys(nullptr, tb3, nz, key_s, (int64_t)mz, 0, 64, dev.s));
    void* tmp3 = nullptr;
    IT(dev.alloc(reinterpret_cast<char**>(&tmp3), tb3));
    IT(cub::DeviceRadixSort::SortKeys(tmp3, tb3, nz, key_s, (int64_t)mz, 0, 64, dev.s));
    if (mz) k_heads<<<grid_of(mz), 256, 0, dev.s>>>(reinterpret_cast<const long long*>(key_s), mz, uniq);
    unsigned long long* ue = nullptr;
    uint64_t mu = 0;
    if ((rc = select_edges(ctx, dev, key_s, uniq, mz, &ue, &mu))) return rc;
    *edges_out = ue;
    *m_out = mu;
    *ids_out = ids_rank;
    *n_out = u;
    return FC_OK;
}

int download_result(fc_ctx* ctx, Dev& dev, const unsigned long long* edges, uint64_t m, const long long* ids,
                    uint64_t n, fc_ingest_result* out) {
    std::vector<unsigned long long> e(m);
    if (m) IT(cudaMemcpyAsync(e.data(), edges, m * sizeof(unsigned long long), cudaMemcpyDeviceToHost, dev.s));
    out->original_ids = static_cast<int64_t*>(std::malloc(std::max<uint64_t>(n, 1) * sizeof(int64_t)));
    out->edges = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(2 * m, 1) * sizeof(uint32_t)));
    if (!out->original_ids || !out->edges) return fc_internal_fail(ctx, FC_DEVICE, "ingest: host allocation failed");
    if (n && ids) IT(cudaMemcpyAsync(out->original_ids, ids, n * sizeof(int64_t), cudaMemcpyDeviceToHost, dev.s));
    IT(cudaStreamSynchronize(dev.s));
    for (uint64_t k = 0; k < m; ++k) {
        out->edges[2 * k] = (uint32_t)(e[k] >> 32);
        out->edges[2 * k + 1] = (uint32_t)e[k];
    }
    out->num_nodes = n;
    out->num_edges = m;
    return FC_OK;
}

int upload_edges(fc_ctx* ctx, Dev& dev, uint64_t m, const uint32_t* edges, unsigned long long** out) {
    std::vector<unsigned long long> h(m);
    for (uint64_t k = 0; k < m; ++k) h[k] = ((unsigned long long)edges[2 * k] << 32) | edges[2 * k + 1];
    unsigned long long* d = nullptr;
    IT(dev.alloc(&d, m));
    if (m) IT(cudaMemcpyAsync(d, h.data(), m * sizeof(unsigned long long), cudaMemcpyHostToDevice, dev.s));
    IT(cudaStreamSynchronize(dev.s));
    *out = d;
    return FC_OK;
}

int download_nodes(fc_ctx* ctx, Dev& dev, const unsigned* keep, uint64_t n, uint32_t** nodes_out, uint64_t* count) {
    std::vector<unsigned> k(n);
    if (n) IT(cudaMemcpyAsync(k.data(), keep, n * sizeof(unsigned), cudaMemcpyDeviceToHost, dev.s));
    IT(cudaStreamSynchronize(dev.s));
    uint64_t c = 0;
    for (uint64_t v = 0; v < n; ++v) c += k[v];
    *nodes_out = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(c, 1) * sizeof(uint32_t)));
    if (!*nodes_out) return fc_internal_fail(ctx, FC_DEVICE, "ingest: host allocation failed");
    uint64_t p = 0;
    for (uint64_t v = 0; v < n; ++v)
        if (k[v]) (*nodes_out)[p++] = (uint32_t)v;
    *count = c;
    return FC_OK;
}

}  // namespace

extern "C" int fc_ingest_edge_list(fc_ctx* ctx, const char* text, uint64_t len, int stages, fc_ingest_result* out) {
    if (!ctx) return fc_internal_fail(nullptr, FC_INVALID, "null context");
    if (!out) return fc_internal_fail(ctx, FC_INVALID, "ingest: null result");
    std::memset(out, 0, sizeof *out);
    IT(cudaSetDevice(fc_internal_device(ctx)));
    // ---- parse (host, all cores) ----
    const unsigned hw = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    const uint64_t nthreads = len < (1u << 20) ? 1 : hw;
    std::vector<Chunk> chunks(nthreads);
    {
        uint64_t start = 0;
        for (uint64_t k = 0; k < nthreads; ++k) {
            uint64_t stop = (k + 1 == nthreads) ? len : std::max<uint64_t>(start, (k + 1) * len / nthreads);
            while (stop < len && text[stop - 1] != '\n' && stop > start) ++stop;
            if (stop < start) stop = start;
            chunks[k].begin = text + start;
            chunks[k].end = text + stop;
            start = stop;
        }
        chunks.back().end = text + len;
        std::vector<std::thread> pool;
        for (uint64_t k = 1; k < nthreads; ++k) pool.emplace_back(parse_chunk, std::ref(chunks[k]));
        parse_chunk(chunks[0]);
        for (auto& th : pool) th.join();
    }
    uint64_t line0 = 0;
    bool saw = false;
    size_t ntok = 0;
    for (auto& c : chunks) {
        if (c.err_line) {
            return fc_internal_fail(ctx, FC_IO, "edge list parse error at line " + std::to_string(line0 + c.err_line) +
                                                    ": " + c.err);
        }
        line0 += c.lines;
        saw = saw || c.saw_edge;
        ntok += c.tok.size();
    }
    if (!saw) return fc_internal_fail(ctx, FC_IO, "edge list is empty");
    std::vector<int64_t> tok;
    tok.reserve(ntok);
    for (auto& c : chunks) {
        tok.insert(tok.end(), c.tok.begin(), c.tok.end());
        std::vector<int64_t>().swap(c.tok);
    }
    if (tok.size() / 2 >= 0x80000000ULL) return fc_internal_fail(ctx, FC_INVALID, "ingest: 2^31 or more edge lines");
    // ---- device stages ----
    Dev dev(fc_internal_stream(ctx));
    unsigned long long* edges = nullptr;
    long long* ids = nullptr;
    uint64_t m = 0, n = 0;
    int rc = compact(ctx, dev, tok, &edges, &m, &ids, &n);
    if (rc) return rc;
    out->parsed_nodes = n;
    if (stages >= 1) {
        unsigned* keep = nullptr;
        if ((rc = lcc_keep(ctx, dev, edges, m, n, &keep))) return rc;
        if ((rc = induce(ctx, dev, edges, m, n, keep, ids))) return rc;
        out->lcc_nodes = n;
        if (stages >= 2) {
            if ((rc = core_keep(ctx, dev, edges, m, n, &keep))) return rc;
            if ((rc = induce(ctx, dev, edges, m, n, keep, ids))) return rc;
        }
    }
    return download_result(ctx, dev, edges, m, ids, n, out);
}

extern "C" int fc_graph_lcc_nodes(fc_ctx* ctx, uint64_t num_nodes, uint64_t num_edges, const uint32_t* edges,
                                  uint32_t** nodes_out, uint64_t* count) {
    if (!ctx) return fc_internal_fail(nullptr, FC_INVALID, "null context");
    if (num_nodes == 0) return fc_internal_fail(ctx, FC_INVALID, "largest_connected_component: empty graph");
    IT(cudaSetDevice(fc_internal_device(ctx)));
    Dev dev(fc_internal_stream(ctx));
    unsigned long long* e = nullptr;
    int rc = upload_edges(ctx, dev, num_edges, edges, &e);
    if (rc) return rc;
    unsigned* keep = nullptr;
    if ((rc = lcc_keep(ctx, dev, e, num_edges, num_nodes, &keep))) return rc;
    return download_nodes(ctx, dev, keep, num_nodes, nodes_out, count);
}

extern "C" int fc_graph_two_core_nodes(fc_ctx* ctx, uint64_t num_nodes, uint64_t num_edges, const uint32_t* edges,
                                       uint32_t** nodes_out, uint64_t* count) {
    if (!ctx) return fc_internal_fail(nullptr, FC_INVALID, "null context");
    IT(cudaSetDevice(fc_internal_device(ctx)));
    Dev dev(fc_internal_stream(ctx));
    unsigned long long* e = nullptr;
    int rc = upload_edges(ctx, dev, num_edges, edges, &e);
    if (rc) return rc;
    unsigned* keep = nullptr;
    if (num_nodes == 0) {
        *nodes_out = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t)));
        *count = 0;
        return FC_OK;
    }
    if ((rc = core_keep(ctx, dev, e, num_edges, num_nodes, &keep))) return rc;
    return download_nodes(ctx, dev, keep, num_nodes, nodes_out, count);
}
