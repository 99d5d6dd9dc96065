// latsum/errors.hpp -- drop-in for the reference's error types
// (/root/reference/proj/include/latsum/errors.hpp:9-20). Same names and
// meaning: validation_error for bad input (CLI exit 2), resource_guard_error
// for a tripped guard (CLI exit 4). Also maps liblatsum_cuda.so status codes
// onto them.
#pragma once

#include <stdexcept>
#include <string>

#include "latsum_cuda.h"

namespace latsum {

class validation_error : public std::runtime_error {
public:
    explicit validation_error(const std::string& what) : std::runtime_error(what) {}
};

class resource_guard_error : public std::runtime_error {
public:
    explicit resource_guard_error(const std::string& what) : std::runtime_error(what) {}
};

// A CUDA failure inside the device engine (no reference counterpart: the
// reference never leaves the host).
class device_error : public std::runtime_error {
public:
    explicit device_error(const std::string& what) : std::runtime_error(what) {}
};

namespace cuda {
// Rethrows a non-zero ls_* status as the mirrored exception type.
inline void check(int status, const char* call) {
    if (status == LS_OK) return;
    const std::string msg = std::string(call) + ": " + ls_last_error();
    if (status == LS_EVALIDATION) throw validation_error(msg);
    if (status == LS_EGUARD) throw resource_guard_error(msg);
    throw device_error(msg);
}
// Same, with the library's message alone: the host validation entry points
// (ls_validate_*) already word it exactly like the reference's exceptions.
inline void check_bare(int status) {
    if (status == LS_OK) return;
    const std::string msg = ls_last_error();
    if (status == LS_EVALIDATION) throw validation_error(msg);
    if (status == LS_EGUARD) throw resource_guard_error(msg);
    throw device_error(msg);
}
}  // namespace cuda

}  // namespace latsum
