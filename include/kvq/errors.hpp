// kvq/errors.hpp — drop-in for the reference's error classes (errors.hpp:11-33) plus the
// status -> exception bridge used by every drop-in header (C-ABI status codes from
// include/kvq_capi.h). Header-only; links against libkvq_b200.so.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "kvq_capi.h"

namespace kvq {

class config_error : public std::runtime_error {  // bad widths / bitwidth / kernel config
public:
    explicit config_error(const std::string& msg) : std::runtime_error(msg) {}
};

class domain_error : public std::runtime_error {  // shape mismatch, empty input, range
public:
    explicit domain_error(const std::string& msg) : std::runtime_error(msg) {}
};

class format_error : public std::runtime_error {  // malformed serialized data
public:
    format_error(const std::string& msg, std::uint64_t at)
        : std::runtime_error(msg + " (byte offset " + std::to_string(at) + ")"), offset_(at) {}
    std::uint64_t offset() const noexcept { return offset_; }

private:
    std::uint64_t offset_;
};

// A CUDA failure or a missing device: the B200 library has no CPU fallback.
class device_error : public std::runtime_error {
public:
    explicit device_error(const std::string& msg) : std::runtime_error(msg) {}
};

namespace capi {

inline std::string last_error() {
    char buf[1024];
    kvq_last_error(buf, sizeof(buf));
    return buf;
}

// Maps a C-ABI status onto the reference's exception classes.
inline void check(int status) {
    switch (status) {
        case KVQ_OK: return;
        case KVQ_ERR_CONFIG: throw config_error(last_error());
        case KVQ_ERR_DOMAIN: throw domain_error(last_error());
        case KVQ_ERR_FORMAT: throw format_error(last_error(), kvq_last_error_offset());
        default: throw device_error(last_error());
    }
}

}  // namespace capi
}  // namespace kvq
