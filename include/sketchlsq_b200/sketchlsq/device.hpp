// sketchlsq/device.hpp (B200 drop-in) -- the per-thread device context the
// drop-in functions run on, and the slq_status -> exception mapping.
// Not a reference header: the reference has no device.  One slq_ctx per
// thread on device 0 unless b200::set_device() is called first; multi-GPU
// callers attach a communicator with b200::init_comm() (distsim.hpp).
#pragma once

#include <string>

#include "sketchlsq/errors.hpp"
#include "slq_b200.h"

namespace sketchlsq {
namespace b200 {

inline void check(int st) {
    if (st == SLQ_OK) return;
    const std::string msg = slq_last_error();
    switch (st) {
        case SLQ_INVALID_SPARSITY: throw InvalidSparsity(msg);
        case SLQ_INVALID_DIMS: throw InvalidDims(msg);
        case SLQ_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case SLQ_RANK_DEFICIENT: throw RankDeficient(msg);
        case SLQ_SINGULAR_TRIANGULAR: throw SingularTriangular(msg);
        case SLQ_INVALID_DISTORTION: throw InvalidDistortion(msg);
        case SLQ_DIVERGENCE: throw Divergence(msg);
        default: throw DeviceError(msg);
    }
}

struct Ctx {
    slq_ctx* h = nullptr;
    int device = 0;
    Ctx() = default;
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;
    ~Ctx() {
        if (h) slq_ctx_destroy(h);
    }
};
inline Ctx& tls() {
    thread_local Ctx c;
    return c;
}
inline void set_device(int device) {
    Ctx& c = tls();
    if (c.h && c.device != device) {
        slq_ctx_destroy(c.h);
        c.h = nullptr;
    }
    c.device = device;
}
inline slq_ctx* ctx() {
    Ctx& c = tls();
    if (!c.h) check(slq_ctx_create(c.device, &c.h));
    return c.h;
}

}  // namespace b200
}  // namespace sketchlsq
