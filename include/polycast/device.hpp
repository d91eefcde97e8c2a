// polycast-b200: process-wide GPU context used by the drop-in C++ API.
//
// The reference spawns a std::thread pool per classify_batch call
// (proj/include/polycast/batch.hpp:212-229).  Here the data-parallel engine is
// libpolycast_cuda.so; the C++ API talks to it through one lazily created
// context over all visible GPUs (or the set chosen with set_devices()).
// There is no CPU fallback: without a usable GPU every batched call throws
// polycast::DeviceError.
#pragma once

#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../polycast_cuda.h"

namespace polycast {

/// Raised when the GPU engine reports a failure (status != PC_OK).
struct DeviceError : std::runtime_error {
    int status;
    DeviceError(int code, const std::string& what) : std::runtime_error(what), status(code) {}
};

namespace device {

struct Holder {
    std::mutex mu;
    pc_ctx* ctx = nullptr;
    std::vector<int> ids; // empty: all visible GPUs
};

inline Holder& holder() {
    static Holder* h = new Holder(); // intentionally leaked: no teardown after the CUDA runtime
    return *h;
}

/// The shared context, created on first use.
inline pc_ctx* context() {
    Holder& h = holder();
    std::lock_guard<std::mutex> lk(h.mu);
    if (!h.ctx) {
        const int rc = h.ids.empty() ? pc_create(&h.ctx, 0)
                                     : pc_create_devices(&h.ctx, h.ids.data(), static_cast<int>(h.ids.size()));
        if (rc != PC_OK || !h.ctx) {
            h.ctx = nullptr;
            throw DeviceError(rc, "polycast: no usable CUDA device for libpolycast_cuda (status " +
                                      std::to_string(rc) + ")");
        }
    }
    return h.ctx;
}

/// Restricts the shared context to the given GPUs (takes effect immediately).
inline void set_devices(const std::vector<int>& ids) {
    Holder& h = holder();
    std::lock_guard<std::mutex> lk(h.mu);
    if (h.ctx) pc_destroy(h.ctx);
    h.ctx = nullptr;
    h.ids = ids;
}

inline void throw_on(int rc, pc_ctx* ctx, const char* where) {
    if (rc != PC_OK) throw DeviceError(rc, std::string(where) + ": " + pc_last_error(ctx));
}

} // namespace device
} // namespace polycast
