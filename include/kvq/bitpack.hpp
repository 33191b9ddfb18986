// kvq/bitpack.hpp — PackedBuffer / pack / unpack (reference bitpack.hpp:15-106).
// Packing and unpacking run on the GPU through kvq_pack / kvq_unpack.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "kvq/errors.hpp"

namespace kvq {

// N-bit codes, M-bit little-endian words, MSB-first within a word; zero pad codes.
struct PackedBuffer {
    std::vector<std::uint8_t> bytes;
    int code_bits = 0;               // N
    int word_bits = 8;               // M
    std::size_t logical_count = 0;   // codes before padding

    std::size_t codes_per_word() const { return static_cast<std::size_t>(word_bits / code_bits); }
    std::size_t word_count() const { return (logical_count + codes_per_word() - 1) / codes_per_word(); }
    std::size_t byte_size() const { return bytes.size(); }
    std::uint32_t word_at(std::size_t i) const {
        const std::size_t nb = static_cast<std::size_t>(word_bits / 8);
        std::uint32_t w = 0;
        for (std::size_t b = 0; b < nb; ++b) w |= static_cast<std::uint32_t>(bytes[i * nb + b]) << (8 * b);
        return w;
    }
};

inline PackedBuffer pack(std::span<const std::uint32_t> codes, int code_bits, int word_bits = 8) {
    PackedBuffer out;
    out.code_bits = code_bits;
    out.word_bits = word_bits;
    out.logical_count = codes.size();
    out.bytes.resize(kvq_packed_bytes(codes.size(), code_bits, word_bits));
    capi::check(kvq_pack(codes.data(), codes.size(), code_bits, word_bits, out.bytes.data(), out.bytes.size()));
    return out;
}

inline std::vector<std::uint32_t> unpack(const PackedBuffer& buf) {
    std::vector<std::uint32_t> codes(buf.logical_count);
    capi::check(kvq_unpack(buf.bytes.data(), buf.bytes.size(), buf.logical_count, buf.code_bits, buf.word_bits,
                           codes.data()));
    return codes;
}

}  // namespace kvq
