// fuzzyclust/device.hpp -- the process-wide device context the drop-in headers
// bind to (new: the reference runs on std::thread workers, parallel.hpp).
// One context per process on device FUZZYCLUST_DEVICE (default 0); a
// similarity is uploaded once and re-used while it stays the resident one.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <string>

#include "fuzzyclust/common.hpp"
#include "fuzzyclust_cuda.h"

namespace fuzzyclust {
namespace device {

[[noreturn]] inline void raise(int code, fc_ctx* ctx) {
    const std::string msg = fc_last_error(ctx);
    if (code == FC_IO) throw IoError(msg);
    if (code == FC_INVALID) throw InvalidInput(msg);
    throw DeviceError(msg);
}

inline void check(int code, fc_ctx* ctx) {
    if (code != FC_OK) raise(code, ctx);
}

struct Context {
    fc_ctx* ctx = nullptr;
    std::uint64_t resident = 0;   // id of the similarity currently on the device
    std::size_t resident_n = 0;   // its size
    Context() {
        int dev = 0;
        if (const char* e = std::getenv("FUZZYCLUST_DEVICE")) dev = std::atoi(e);
        check(fc_create(&ctx, dev, 0, 1, nullptr), nullptr);
    }
    ~Context() { fc_destroy(ctx); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
};

inline Context& context() {
    static Context c;
    return c;
}

/// Second context for operators that only need N (share_matrix / cross_share of an X
/// whose size differs from the resident similarity): it holds an N-node identity
/// pattern, so the caller's resident similarity on context() is never evicted.
inline Context& aux_context() {
    static Context c;
    return c;
}

inline std::uint64_t next_id() {
    static std::uint64_t id = 0;
    return ++id;
}

}  // namespace device
}  // namespace fuzzyclust
