// SHA-256 (FIPS 180-4) for the checkpoint file/stream integrity digest
// (checkpoint.hpp:68-80,190-224 hash the canonical payload with
// emesh::Sha256, sha256.hpp). Host code: the digest is a strictly sequential
// chain over the payload, so it runs on the CPU next to the device copies;
// the x86 SHA extensions are used when the host has them (cpuid), otherwise a
// portable scalar compression.
#include "sha256.h"

#include <cpuid.h>
#include <immintrin.h>

#include <cstdlib>
#include <cstring>

namespace emesh_b200 {
namespace {

constexpr uint32_t kK[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

inline uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

void blocks_scalar(uint32_t st[8], const uint8_t* p, size_t nblocks) {
    for (; nblocks; --nblocks, p += 64) {
        uint32_t w[64];
        for (int t = 0; t < 16; ++t)
            w[t] = (uint32_t)p[4 * t] << 24 | (uint32_t)p[4 * t + 1] << 16 | (uint32_t)p[4 * t + 2] << 8 | p[4 * t + 3];
        for (int t = 16; t < 64; ++t) {
            const uint32_t s0 = rotr(w[t - 15], 7) ^ rotr(w[t - 15], 18) ^ (w[t - 15] >> 3);
            const uint32_t s1 = rotr(w[t - 2], 17) ^ rotr(w[t - 2], 19) ^ (w[t - 2] >> 10);
            w[t] = w[t - 16] + s0 + w[t - 7] + s1;
        }
        uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
        for (int t = 0; t < 64; ++t) {
            const uint32_t t1 = h + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) + kK[t] + w[t];
            const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
            h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
        st[0] += a; st[1] += b; st[2] += c; st[3] += d; st[4] += e; st[5] += f; st[6] += g; st[7] += h;
    }
}

// SHA-NI: the state lives as {ABEF, CDGH}; each sha256rnds2 does two rounds,
// sha256msg1/msg2 extend the schedule four words at a time.
__attribute__((target("sha,sse4.1,ssse3"))) void blocks_shani(uint32_t st[8], const uint8_t* p, size_t nblocks) {
    const __m128i bswap = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
    __m128i tmp = _mm_loadu_si128(reinterpret_cast<const __m128i*>(st));
    __m128i s1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(st + 4));
    tmp = _mm_shuffle_epi32(tmp, 0xB1);             // CDAB
    s1 = _mm_shuffle_epi32(s1, 0x1B);               // EFGH
    __m128i s0 = _mm_alignr_epi8(tmp, s1, 8);       // ABEF
    s1 = _mm_blend_epi16(s1, tmp, 0xF0);            // CDGH
    for (; nblocks; --nblocks, p += 64) {
        const __m128i abef = s0, cdgh = s1;
        __m128i x[4];
        for (int g = 0; g < 16; ++g) {
            __m128i m;
            if (g < 4) {
                m = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 16 * g)), bswap);
            } else {
                // W[t] = s1(W[t-2]) + W[t-7] + s0(W[t-15]) + W[t-16]
                m = _mm_sha256msg1_epu32(x[g & 3], x[(g + 1) & 3]);
                m = _mm_add_epi32(m, _mm_alignr_epi8(x[(g + 3) & 3], x[(g + 2) & 3], 4));
                m = _mm_sha256msg2_epu32(m, x[(g + 3) & 3]);
            }
            x[g & 3] = m;
            __m128i wk = _mm_add_epi32(m, _mm_loadu_si128(reinterpret_cast<const __m128i*>(kK + 4 * g)));
            s1 = _mm_sha256rnds2_epu32(s1, s0, wk);
            wk = _mm_shuffle_epi32(wk, 0x0E);
            s0 = _mm_sha256rnds2_epu32(s0, s1, wk);
        }
        s0 = _mm_add_epi32(s0, abef);
        s1 = _mm_add_epi32(s1, cdgh);
    }
    tmp = _mm_shuffle_epi32(s0, 0x1B);              // FEBA
    s1 = _mm_shuffle_epi32(s1, 0xB1);               // DCHG
    s0 = _mm_blend_epi16(tmp, s1, 0xF0);            // DCBA
    s1 = _mm_alignr_epi8(s1, tmp, 8);               // HGFE
    _mm_storeu_si128(reinterpret_cast<__m128i*>(st), s0);
    _mm_storeu_si128(reinterpret_cast<__m128i*>(st + 4), s1);
}

bool host_has_shani() {
    unsigned a, b, c, d;
    if (!__get_cpuid(1, &a, &b, &c, &d)) return false;
    const bool sse41 = c & (1u << 19), ssse3 = c & (1u << 9);
    if (!__get_cpuid_count(7, 0, &a, &b, &c, &d)) return false;
    return sse41 && ssse3 && (b & (1u << 29));
}

const bool g_shani = host_has_shani() && !std::getenv("EMESH_SHA_SCALAR");

void blocks(uint32_t st[8], const uint8_t* p, size_t nblocks) {
    if (g_shani) blocks_shani(st, p, nblocks);
    else blocks_scalar(st, p, nblocks);
}

}  // namespace

void Sha256::reset() {
    static constexpr uint32_t kH0[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                        0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    std::memcpy(h, kH0, sizeof h);
    total = 0;
    fill = 0;
}

void Sha256::update(const void* data, size_t n) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    total += n;
    if (fill) {
        const size_t take = n < 64 - fill ? n : 64 - fill;
        std::memcpy(buf + fill, p, take);
        fill += take; p += take; n -= take;
        if (fill < 64) return;
        blocks(h, buf, 1);
        fill = 0;
    }
    if (n >= 64) {
        blocks(h, p, n / 64);
        p += n & ~(size_t)63;
        n &= 63;
    }
    if (n) { std::memcpy(buf, p, n); fill = n; }
}

void Sha256::finish(uint8_t out[32]) {
    const uint64_t bits = total * 8;
    const uint8_t pad = 0x80;
    update(&pad, 1);
    const uint8_t zero[64] = {};
    update(zero, fill <= 56 ? 56 - fill : 120 - fill);
    uint8_t len[8];
    for (int i = 0; i < 8; ++i) len[i] = (uint8_t)(bits >> (56 - 8 * i));
    update(len, 8);
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 4; ++j) out[4 * i + j] = (uint8_t)(h[i] >> (24 - 8 * j));
}

bool sha256_uses_shani() { return g_shani; }

}  // namespace emesh_b200
