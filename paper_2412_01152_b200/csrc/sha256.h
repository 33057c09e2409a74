// Incremental SHA-256 (host), see sha256.cpp.
#pragma once
#include <cstddef>
#include <cstdint>

namespace emesh_b200 {

struct Sha256 {
    uint32_t h[8];
    uint64_t total;
    uint8_t buf[64];
    size_t fill;
    Sha256() { reset(); }
    void reset();
    void update(const void* data, size_t n);
    void finish(uint8_t out[32]);
};

bool sha256_uses_shani();

}  // namespace emesh_b200
