// bsm/detail_cabi.hpp -- glue between the C++ shim and the C ABI: status ->
// exception mapping and the per-thread device context.  The reference's
// functions are pure and thread-safe; the shim keeps that contract with one
// bsm_ctx per calling thread (re-entrant, no shared mutable state).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "../bsm_cuda.h"
#include "bsm/errors.hpp"

namespace bsm::detail {

inline void throw_status(int rc) {
    if (rc == BSM_OK) return;
    const std::string msg = bsm_last_error();
    switch (rc) {
        case BSM_INVALID_ARGUMENT: throw InvalidArgument(msg);
        case BSM_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        default: throw Error(msg);
    }
}

class Context {
public:
    Context() {
        const char* lr = std::getenv("LOCAL_RANK");
        throw_status(bsm_ctx_create(lr ? std::atoi(lr) : 0, &ctx_));
    }
    ~Context() { bsm_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    bsm_ctx* get() const { return ctx_; }

    // Upload the pattern when it differs from the resident one.
    void use_pattern(const std::vector<int16_t>& flat, int n, int window) {
        if (n == n_ && window == window_ && flat == flat_) return;
        n_ = 0;  // a failed upload leaves the context without a pattern
        throw_status(bsm_set_pattern(ctx_, flat.data(), n, window));
        flat_ = flat;
        n_ = n;
        window_ = window;
    }

private:
    bsm_ctx* ctx_ = nullptr;
    std::vector<int16_t> flat_;
    int n_ = 0, window_ = 0;
};

inline Context& context() {
    thread_local Context ctx;
    return ctx;
}

}  // namespace bsm::detail
