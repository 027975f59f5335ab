// Error hierarchy of the drop-in library: the same class names and bases as the
// reference (proj/include/spgsim/errors.hpp:9-58) so catch sites port
// unchanged. Each maps one-to-one to an spg_status code of the C ABI.
#pragma once

#include <stdexcept>
#include <string>

namespace spgsim {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DimensionError : Error {
    using Error::Error;
};
struct ParameterError : Error {
    using Error::Error;
};
struct ParseError : Error {
    ParseError(const std::string& what, long ln) : Error(what + " (line " + std::to_string(ln) + ")"), line(ln) {}
    long line;
};
struct UnsupportedFormat : Error {
    using Error::Error;
};
struct GridError : Error {
    using Error::Error;
};
struct IncompleteTileSet : Error {
    using Error::Error;
};
struct RoutingError : Error {
    using Error::Error;
};
struct ScheduleError : Error {
    using Error::Error;
};
struct DeadlockError : Error {
    using Error::Error;
};
// Device-side failure (CUDA error, out of device memory, no sm_100 device).
// Not in the reference: the simulator never touches a device.
struct DeviceError : Error {
    using Error::Error;
};

}  // namespace spgsim
