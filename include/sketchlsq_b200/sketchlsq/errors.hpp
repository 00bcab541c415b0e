// sketchlsq/errors.hpp (B200 drop-in) -- the reference's exception hierarchy
// (errors.hpp:9-76), so `catch (const sketchlsq::RankDeficient&)` and friends
// work unchanged, plus DeviceError for CUDA / NCCL / allocation failures of
// the device path.  slq_status codes map one-to-one (device.hpp: check()).
#pragma once

#include <stdexcept>
#include <string>

namespace sketchlsq {

struct Error : std::runtime_error {
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

#define SKETCHLSQ_B200_ERROR(Name) \
    struct Name : Error {          \
        using Error::Error;        \
    }
SKETCHLSQ_B200_ERROR(RankDeficient);
SKETCHLSQ_B200_ERROR(SingularTriangular);
SKETCHLSQ_B200_ERROR(DimensionMismatch);
SKETCHLSQ_B200_ERROR(InvalidSparsity);
SKETCHLSQ_B200_ERROR(AllocationTooLarge);
SKETCHLSQ_B200_ERROR(InvalidDistortion);
SKETCHLSQ_B200_ERROR(InvalidDims);
SKETCHLSQ_B200_ERROR(NegativeArgument);
SKETCHLSQ_B200_ERROR(InvalidResidual);
SKETCHLSQ_B200_ERROR(UnsupportedFormat);
SKETCHLSQ_B200_ERROR(Divergence);
SKETCHLSQ_B200_ERROR(BreakdownIfZero);
SKETCHLSQ_B200_ERROR(ConfigError);
// device-path failures (no reference counterpart: the reference has no device)
SKETCHLSQ_B200_ERROR(DeviceError);
#undef SKETCHLSQ_B200_ERROR

}  // namespace sketchlsq
