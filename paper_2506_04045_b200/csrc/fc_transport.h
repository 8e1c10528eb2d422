// fc_transport.h -- the four collectives of a multi-rank solve behind one interface.
//
// A multi-rank iteration exchanges exactly four things:
//   allgather_rows  every rank's new rows of U into every replica
//   recv_prev       block-partial running totals from rank - 1   (ordered chain,
//   send_next       ... and on to rank + 1                        objective.hpp:82-88)
//   bcast_last      the final totals from rank world - 1 to everyone
// Two implementations:
//   NcclTransport      one process per GPU, NCCL over NVLink / NVSwitch (production)
//   LoopbackTransport  W rank contexts in ONE process on one device (tests): every
//                      collective is a stream-ordered device copy pulled from the
//                      peer's buffer after a CUDA event the peer recorded, with a
//                      host-side rendezvous (publish / consume slots) standing in for
//                      NCCL's matching.  Kernels never wait on each other; only the
//                      copies wait on events, so the GPU cannot deadlock.
// Both run the same rank>0 code in fc_capi.cu (recv, combine with the received
// running total, send, broadcast root, per-rank row offsets).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

namespace fc {

struct Transport {
    virtual ~Transport() = default;
    virtual const char* name() const = 0;
    // rows [bounds[r], bounds[r+1]) x c of `buf` (this rank's replica) from their owner r
    virtual int allgather_rows(double* buf, const uint64_t* bounds, uint32_t c, cudaStream_t s, std::string* err) = 0;
    virtual int recv_prev(double* dst, size_t n, cudaStream_t s, std::string* err) = 0;
    virtual int send_next(const double* src, size_t n, cudaStream_t s, std::string* err) = 0;
    virtual int bcast_last(double* buf, size_t n, cudaStream_t s, std::string* err) = 0;
    // halo exchange (locality graphs): send[send_off[p] .. send_off[p+1]) to every peer p,
    // recv[recv_off[p] .. recv_off[p+1]) from every peer p (offsets in doubles, world + 1
    // entries each).  peer_off[p]: where this rank's segment starts in p's send buffer
    // (used by the loopback, which pulls; NCCL matches send/recv pairs itself).
    virtual int exchange(const double* send, const uint64_t* send_off, double* recv, const uint64_t* recv_off,
                         const uint64_t* peer_off, cudaStream_t s, std::string* err) = 0;
};

inline int transport_fail(std::string* err, const char* what, const char* detail) {
    char b[512];
    std::snprintf(b, sizeof b, "%s: %s", what, detail);
    *err = b;
    return 3;   // FC_DEVICE
}

// ---- NCCL --------------------------------------------------------------------------------
struct NcclTransport final : Transport {
    ncclComm_t comm;
    int rank, world;
    NcclTransport(ncclComm_t c, int r, int w) : comm(c), rank(r), world(w) {
        if (const char* a = std::getenv("FC_ALLGATHER")) padded = std::strcmp(a, "padded") == 0;
    }
    ~NcclTransport() override {
        if (staging) cudaFree(staging);
        ncclCommDestroy(comm);
    }
    const char* name() const override { return "nccl"; }
    static int chk(ncclResult_t r, std::string* err, const char* what) {
        return r == ncclSuccess ? 0 : transport_fail(err, what, ncclGetErrorString(r));
    }
    // FC_ALLGATHER=padded: one ncclAllGather of max-shard-sized slices into a staging
    // buffer, then device copies to each owner's row offset (NCCL's allgather algorithms --
    // ring / NVLS -- for one padded collective, at the price of one extra N x C device copy)
    bool padded = false;
    double* staging = nullptr;
    size_t staging_cap = 0;
    int allgather_padded(double* buf, const uint64_t* bounds, uint32_t c, cudaStream_t s, std::string* err) {
        uint64_t maxrows = 0;
        for (int r = 0; r < world; ++r) maxrows = std::max<uint64_t>(maxrows, bounds[r + 1] - bounds[r]);
        const size_t slice = maxrows * c, need = slice * world;
        if (need > staging_cap) {
            if (staging) cudaFree(staging);
            staging = nullptr;
            staging_cap = 0;
            const cudaError_t e = cudaMalloc(&staging, std::max<size_t>(need, 1) * sizeof(double));
            if (e != cudaSuccess) return transport_fail(err, "padded allgather staging", cudaGetErrorString(e));
            staging_cap = need;
        }
        const size_t own = (bounds[rank + 1] - bounds[rank]) * c;
        cudaError_t e = cudaMemcpyAsync(staging + rank * slice, buf + bounds[rank] * c, own * sizeof(double),
                                        cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return transport_fail(err, "padded allgather copy", cudaGetErrorString(e));
        if (int x = chk(ncclAllGather(staging + rank * slice, staging, slice, ncclDouble, comm, s), err,
                        "ncclAllGather"))
            return x;
        for (int r = 0; r < world; ++r) {
            if (r == rank) continue;
            const size_t cnt = (bounds[r + 1] - bounds[r]) * c;
            if (!cnt) continue;
            e = cudaMemcpyAsync(buf + bounds[r] * c, staging + r * slice, cnt * sizeof(double),
                                cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return transport_fail(err, "padded allgather scatter", cudaGetErrorString(e));
        }
        return 0;
    }
    // unequal shards: one broadcast per owner, grouped (NCCL allgather needs equal counts)
    int allgather_rows(double* buf, const uint64_t* bounds, uint32_t c, cudaStream_t s, std::string* err) override {
        if (padded) return allgather_padded(buf, bounds, c, s, err);
        if (int e = chk(ncclGroupStart(), err, "ncclGroupStart")) return e;
        for (int r = 0; r < world; ++r) {
            const size_t off = bounds[r] * c, cnt = (bounds[r + 1] - bounds[r]) * c;
            if (int e = chk(ncclBroadcast(buf + off, buf + off, cnt, ncclDouble, r, comm, s), err, "ncclBroadcast"))
                return e;
        }
        return chk(ncclGroupEnd(), err, "ncclGroupEnd");
    }
    int recv_prev(double* dst, size_t n, cudaStream_t s, std::string* err) override {
        return chk(ncclRecv(dst, n, ncclDouble, rank - 1, comm, s), err, "ncclRecv");
    }
    int send_next(const double* src, size_t n, cudaStream_t s, std::string* err) override {
        return chk(ncclSend(src, n, ncclDouble, rank + 1, comm, s), err, "ncclSend");
    }
    int bcast_last(double* buf, size_t n, cudaStream_t s, std::string* err) override {
        return chk(ncclBroadcast(buf, buf, n, ncclDouble, world - 1, comm, s), err, "ncclBroadcast");
    }
    int exchange(const double* send, const uint64_t* send_off, double* recv, const uint64_t* recv_off,
                 const uint64_t*, cudaStream_t s, std::string* err) override {
        if (int e = chk(ncclGroupStart(), err, "ncclGroupStart")) return e;
        for (int p = 0; p < world; ++p) {
            if (p == rank) continue;
            const size_t ns = send_off[p + 1] - send_off[p], nr = recv_off[p + 1] - recv_off[p];
            if (ns)
                if (int e = chk(ncclSend(send + send_off[p], ns, ncclDouble, p, comm, s), err, "ncclSend")) return e;
            if (nr)
                if (int e = chk(ncclRecv(recv + recv_off[p], nr, ncclDouble, p, comm, s), err, "ncclRecv")) return e;
        }
        return chk(ncclGroupEnd(), err, "ncclGroupEnd");
    }
};

}  // namespace fc

// ---- in-process loopback group (shared by the W rank contexts) ---------------------------
struct fc_loopback {
    enum Kind { kAllgather = 0, kChain = 1, kBcast = 2, kHalo = 3, kKinds = 4 };
    static constexpr int kRing = 8;
    struct Slot {
        uint64_t seq = ~0ULL;          // publication held in this slot
        const void* ptr = nullptr;     // publisher's device buffer
        cudaEvent_t ev = nullptr;      // recorded on the publisher's stream when the data is ready
        int left = 0;                  // consumers still to issue their wait + copy
    };
    int world = 0;
    int device = 0;
    std::mutex mu;
    std::condition_variable cv;
    std::vector<Slot> slots;           // [kind][rank][seq % kRing]
    bool failed = false;
    double timeout_s = 120.0;

    Slot& slot(int kind, int rank, uint64_t seq) { return slots[((size_t)kind * world + rank) * kRing + seq % kRing]; }

    template <class Pred>
    bool wait(std::unique_lock<std::mutex>& lk, Pred p) {
        const bool ok = cv.wait_for(lk, std::chrono::duration<double>(timeout_s), [&] { return failed || p(); });
        if (!ok) failed = true;
        cv.notify_all();
        return ok && !failed;
    }
    // record `s`'s current tail for (kind, rank, seq); `consumers` peers will pull from `ptr`
    int publish(int kind, int rank, uint64_t seq, const void* ptr, cudaStream_t s, int consumers, std::string* err) {
        std::unique_lock<std::mutex> lk(mu);
        Slot& sl = slot(kind, rank, seq);
        if (!wait(lk, [&] { return sl.left == 0; }))
            return fc::transport_fail(err, "loopback", "timed out waiting for peers to consume a slot");
        const cudaError_t e = cudaEventRecord(sl.ev, s);
        if (e != cudaSuccess) return fc::transport_fail(err, "loopback cudaEventRecord", cudaGetErrorString(e));
        sl.seq = seq;
        sl.ptr = ptr;
        sl.left = consumers;
        cv.notify_all();
        return 0;
    }
    // stream `s` waits for (kind, src, seq); `copy(ptr)` enqueues the pull on `s`
    template <class F>
    int consume(int kind, int src, uint64_t seq, cudaStream_t s, std::string* err, F&& copy) {
        std::unique_lock<std::mutex> lk(mu);
        Slot& sl = slot(kind, src, seq);
        if (!wait(lk, [&] { return sl.seq == seq && sl.left > 0; }))
            return fc::transport_fail(err, "loopback", "timed out waiting for a peer rank's data");
        cudaError_t e = cudaStreamWaitEvent(s, sl.ev, 0);
        if (e == cudaSuccess) e = copy(sl.ptr);
        sl.left -= 1;
        cv.notify_all();
        if (e != cudaSuccess) return fc::transport_fail(err, "loopback copy", cudaGetErrorString(e));
        return 0;
    }
};

namespace fc {

struct LoopbackTransport final : Transport {
    fc_loopback* g;
    int rank, world;
    uint64_t ag_seq = 0, send_seq = 0, recv_seq = 0, bc_seq = 0, halo_seq = 0;
    LoopbackTransport(fc_loopback* grp, int r) : g(grp), rank(r), world(grp->world) {}
    const char* name() const override { return "loopback"; }
    int allgather_rows(double* buf, const uint64_t* bounds, uint32_t c, cudaStream_t s, std::string* err) override {
        const uint64_t seq = ag_seq++;
        if (int e = g->publish(fc_loopback::kAllgather, rank, seq, buf, s, world - 1, err)) return e;
        for (int q = 0; q < world; ++q) {
            if (q == rank) continue;
            const size_t off = bounds[q] * c, bytes = (bounds[q + 1] - bounds[q]) * c * sizeof(double);
            if (int e = g->consume(fc_loopback::kAllgather, q, seq, s, err, [&](const void* p) {
                    return bytes ? cudaMemcpyAsync(buf + off, static_cast<const double*>(p) + off, bytes,
                                                   cudaMemcpyDeviceToDevice, s)
                                 : cudaSuccess;
                }))
                return e;
        }
        return 0;
    }
    int recv_prev(double* dst, size_t n, cudaStream_t s, std::string* err) override {
        return g->consume(fc_loopback::kChain, rank - 1, recv_seq++, s, err, [&](const void* p) {
            return cudaMemcpyAsync(dst, p, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
        });
    }
    int send_next(const double* src, size_t n, cudaStream_t s, std::string* err) override {
        (void)n;
        return g->publish(fc_loopback::kChain, rank, send_seq++, src, s, 1, err);
    }
    int exchange(const double* send, const uint64_t* send_off, double* recv, const uint64_t* recv_off,
                 const uint64_t* peer_off, cudaStream_t s, std::string* err) override {
        const uint64_t seq = halo_seq++;
        int consumers = 0;
        for (int p = 0; p < world; ++p) consumers += (p != rank && send_off[p + 1] > send_off[p]);
        if (consumers)
            if (int e = g->publish(fc_loopback::kHalo, rank, seq, send, s, consumers, err)) return e;
        for (int p = 0; p < world; ++p) {
            const size_t nr = recv_off[p + 1] - recv_off[p];
            if (p == rank || !nr) continue;
            if (int e = g->consume(fc_loopback::kHalo, p, seq, s, err, [&](const void* ptr) {
                    return cudaMemcpyAsync(recv + recv_off[p], static_cast<const double*>(ptr) + peer_off[p],
                                           nr * sizeof(double), cudaMemcpyDeviceToDevice, s);
                }))
                return e;
        }
        return 0;
    }
    int bcast_last(double* buf, size_t n, cudaStream_t s, std::string* err) override {
        const uint64_t seq = bc_seq++;
        if (rank == world - 1) return g->publish(fc_loopback::kBcast, rank, seq, buf, s, world - 1, err);
        return g->consume(fc_loopback::kBcast, world - 1, seq, s, err, [&](const void* p) {
            return cudaMemcpyAsync(buf, p, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
        });
    }
};

}  // namespace fc
