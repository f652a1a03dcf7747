// csd/error.hpp — exception classes of the csd:: API (mirror of the reference's
// include/csd/error.hpp:8-46).  The GPU library reports csd_status codes through the C ABI;
// the host mirror (libcsd_host.so) rethrows them as these types.
#pragma once

#include <stdexcept>
#include <string>

namespace csd {

struct Error : std::runtime_error {
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};
struct ShapeError : Error { using Error::Error; };    // shape / divisibility mismatch
struct IndexError : Error { using Error::Error; };    // id out of range or duplicated
struct NumericError : Error { using Error::Error; };  // non-finite input
struct StateError : Error { using Error::Error; };    // sparse step before a dense step
struct ValueError : Error { using Error::Error; };    // parameter out of range
struct ConfigError : Error { using Error::Error; };   // invalid model / voxel configuration
struct IoError : Error { using Error::Error; };       // malformed input file / text

}  // namespace csd
