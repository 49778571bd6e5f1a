// Device SHA-256 and Keccak-256 for the Merkle commitment (north_star (4)).
//
// Both functions are specialised for the two message shapes the tree needs:
//   leaf     = H(0x00 || chunk)   (commitments.py:137-138)
//   internal = H(0x01 || L || R)  (commitments.py:125)
// i.e. a one-byte domain tag followed by a word-aligned payload.  The payload
// is consumed as little-endian 32-bit words D[m]; the tag shifts every
// message word by one byte, which is one PRMT (SHA-256) or one SHF (Keccak)
// per word instead of a byte-granular copy.  A generic byte-oriented path
// handles odd-length leaves (canon headers, JSON chunks).
#pragma once
#include <stdint.h>

namespace nao {

enum : int { kSHA256 = NAO_HASH_SHA256, kKECCAK256 = NAO_HASH_KECCAK256 };

// ------------------------------------------------------------------ SHA-256

__device__ __forceinline__ uint32_t rotr32(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__constant__ uint32_t c_sha256_k[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u,
    0x923f82a4u, 0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u,
    0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u,
    0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u,
    0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u,
    0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,
    0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au,
    0x5b9cca4fu, 0x682e6ff3u, 0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u,
    0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

__device__ __forceinline__ void sha256_init(uint32_t st[8]) {
    st[0] = 0x6a09e667u; st[1] = 0xbb67ae85u; st[2] = 0x3c6ef372u; st[3] = 0xa54ff53au;
    st[4] = 0x510e527fu; st[5] = 0x9b05688cu; st[6] = 0x1f83d9abu; st[7] = 0x5be0cd19u;
}

// One compression; W holds the 16 big-endian message words (clobbered).
__device__ __forceinline__ void sha256_compress(uint32_t st[8], uint32_t W[16]) {
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3];
    uint32_t e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll
    for (int i = 0; i < 64; i++) {
        uint32_t w;
        if (i < 16) {
            w = W[i];
        } else {
            uint32_t w15 = W[(i + 1) & 15], w2 = W[(i + 14) & 15];
            uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
            uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
            w = W[i & 15] = W[i & 15] + s0 + W[(i + 9) & 15] + s1;
        }
        uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
        uint32_t ch = (e & f) ^ (~e & g);
        uint32_t t1 = h + S1 + ch + c_sha256_k[i] + w;
        uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
        uint32_t mj = (a & b) | (c & (a | b));
        h = g; g = f; f = e; e = d + t1;
        d = c; c = b; b = a; a = t1 + S0 + mj;
    }
    st[0] += a; st[1] += b; st[2] += c; st[3] += d;
    st[4] += e; st[5] += f; st[6] += g; st[7] += h;
}

// Message word j given the previous and current little-endian data words:
// bytes (prev.b3, cur.b0, cur.b1, cur.b2) big-endian.
__device__ __forceinline__ uint32_t sha_shift(uint32_t prev, uint32_t cur) {
    return __byte_perm(prev, cur, 0x3456);
}

// H(tag || D[0..nw)) for a word-aligned payload.  `Load` provides
//   uint4 v4(i)  -> words 4i..4i+3   (only called for i < nw/4 full vectors)
//   uint32_t w(i)-> word i           (i < nw)
template <class Load>
__device__ __forceinline__ void sha256_tagged(const Load& ld, uint32_t nw, uint32_t tag,
                                              uint32_t st[8]) {
    sha256_init(st);
    uint32_t carry = tag << 24;
    const uint32_t nfull = nw >> 4;
#pragma unroll 1
    for (uint32_t b = 0; b < nfull; b++) {
        uint32_t D[16];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint4 v = ld.v4(4 * b + q);
            D[4 * q] = v.x; D[4 * q + 1] = v.y; D[4 * q + 2] = v.z; D[4 * q + 3] = v.w;
        }
        uint32_t W[16];
        W[0] = sha_shift(carry, D[0]);
#pragma unroll
        for (int j = 1; j < 16; j++) W[j] = sha_shift(D[j - 1], D[j]);
        carry = D[15];
        sha256_compress(st, W);
    }
    // tail: rem real words, then the 0x80 pad byte, zeros, 64-bit length
    const uint32_t rem = nw - (nfull << 4);
    const uint32_t base = nfull << 4;
    const uint64_t bits = (1ull + 4ull * nw) * 8ull;
    const int nblk = (rem <= 13) ? 1 : 2;
    uint32_t E[32];
#pragma unroll
    for (int k = 0; k < 32; k++) {
        uint32_t v = 0;
        if ((uint32_t)k < rem) v = ld.w(base + k);
        else if ((uint32_t)k == rem) v = 0x80u;
        E[k] = v;
    }
#pragma unroll
    for (int t = 0; t < 2; t++) {
        if (t < nblk) {
            uint32_t W[16];
#pragma unroll
            for (int j = 0; j < 16; j++) {
                int k = 16 * t + j;
                uint32_t prev = (k == 0) ? carry : E[(k + 31) & 31];
                W[j] = sha_shift(prev, E[k]);
            }
            if (t == nblk - 1) {
                W[14] = (uint32_t)(bits >> 32);
                W[15] = (uint32_t)bits;
            }
            sha256_compress(st, W);
        }
    }
}

// ---------------------------------------------------------------- Keccak-f

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int n) {
    return (x << n) | (x >> (64 - n));
}

__constant__ uint64_t c_keccak_rc[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808aull,
    0x8000000080008000ull, 0x000000000000808bull, 0x0000000080000001ull,
    0x8000000080008081ull, 0x8000000000008009ull, 0x000000000000008aull,
    0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000aull,
    0x000000008000808bull, 0x800000000000008bull, 0x8000000000008089ull,
    0x8000000000008003ull, 0x8000000000008002ull, 0x8000000000000080ull,
    0x000000000000800aull, 0x800000008000000aull, 0x8000000080008081ull,
    0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};

__device__ __forceinline__ uint64_t chi(uint64_t a, uint64_t b, uint64_t c) { return a ^ (~b & c); }

// Keccak-f[1600]; A[x + 5y].
__device__ __forceinline__ void keccak_f1600(uint64_t A[25]) {
#pragma unroll 1
    for (int r = 0; r < 24; r++) {
        uint64_t C0 = A[0] ^ A[5] ^ A[10] ^ A[15] ^ A[20];
        uint64_t C1 = A[1] ^ A[6] ^ A[11] ^ A[16] ^ A[21];
        uint64_t C2 = A[2] ^ A[7] ^ A[12] ^ A[17] ^ A[22];
        uint64_t C3 = A[3] ^ A[8] ^ A[13] ^ A[18] ^ A[23];
        uint64_t C4 = A[4] ^ A[9] ^ A[14] ^ A[19] ^ A[24];
        uint64_t D0 = C4 ^ rotl64(C1, 1), D1 = C0 ^ rotl64(C2, 1), D2 = C1 ^ rotl64(C3, 1);
        uint64_t D3 = C2 ^ rotl64(C4, 1), D4 = C3 ^ rotl64(C0, 1);
        // theta + rho + pi:  B[y + 5*((2x+3y)%5)] = rotl(A[x+5y] ^ D[x], r[x][y])
        uint64_t B00 = A[0] ^ D0;
        uint64_t B10 = rotl64(A[6] ^ D1, 44);
        uint64_t B20 = rotl64(A[12] ^ D2, 43);
        uint64_t B30 = rotl64(A[18] ^ D3, 21);
        uint64_t B40 = rotl64(A[24] ^ D4, 14);
        uint64_t B01 = rotl64(A[3] ^ D3, 28);
        uint64_t B11 = rotl64(A[9] ^ D4, 20);
        uint64_t B21 = rotl64(A[10] ^ D0, 3);
        uint64_t B31 = rotl64(A[16] ^ D1, 45);
        uint64_t B41 = rotl64(A[22] ^ D2, 61);
        uint64_t B02 = rotl64(A[1] ^ D1, 1);
        uint64_t B12 = rotl64(A[7] ^ D2, 6);
        uint64_t B22 = rotl64(A[13] ^ D3, 25);
        uint64_t B32 = rotl64(A[19] ^ D4, 8);
        uint64_t B42 = rotl64(A[20] ^ D0, 18);
        uint64_t B03 = rotl64(A[4] ^ D4, 27);
        uint64_t B13 = rotl64(A[5] ^ D0, 36);
        uint64_t B23 = rotl64(A[11] ^ D1, 10);
        uint64_t B33 = rotl64(A[17] ^ D2, 15);
        uint64_t B43 = rotl64(A[23] ^ D3, 56);
        uint64_t B04 = rotl64(A[2] ^ D2, 62);
        uint64_t B14 = rotl64(A[8] ^ D3, 55);
        uint64_t B24 = rotl64(A[14] ^ D4, 39);
        uint64_t B34 = rotl64(A[15] ^ D0, 41);
        uint64_t B44 = rotl64(A[21] ^ D1, 2);
        // chi (row y: lanes Bxy for x=0..4) + iota
        A[0] = chi(B00, B10, B20) ^ c_keccak_rc[r];
        A[1] = chi(B10, B20, B30); A[2] = chi(B20, B30, B40);
        A[3] = chi(B30, B40, B00); A[4] = chi(B40, B00, B10);
        A[5] = chi(B01, B11, B21); A[6] = chi(B11, B21, B31); A[7] = chi(B21, B31, B41);
        A[8] = chi(B31, B41, B01); A[9] = chi(B41, B01, B11);
        A[10] = chi(B02, B12, B22); A[11] = chi(B12, B22, B32); A[12] = chi(B22, B32, B42);
        A[13] = chi(B32, B42, B02); A[14] = chi(B42, B02, B12);
        A[15] = chi(B03, B13, B23); A[16] = chi(B13, B23, B33); A[17] = chi(B23, B33, B43);
        A[18] = chi(B33, B43, B03); A[19] = chi(B43, B03, B13);
        A[20] = chi(B04, B14, B24); A[21] = chi(B14, B24, B34); A[22] = chi(B24, B34, B44);
        A[23] = chi(B34, B44, B04); A[24] = chi(B44, B04, B14);
    }
}

// lane bytes (prev.b3, cur.b0..b2, nxt.b3?) : lo32 = bytes (p.b3,c.b0,c.b1,c.b2)
__device__ __forceinline__ uint32_t kk_shift(uint32_t prev, uint32_t cur) {
    return __funnelshift_r(prev, cur, 24);
}

// Keccak-256 (pad 0x01) of tag || D[0..nw).  `Load` provides
//   uint2 v2(i) -> words 2i, 2i+1   (i < nw/2)
//   uint32_t w(i)
template <class Load>
__device__ __forceinline__ void keccak256_tagged(const Load& ld, uint32_t nw, uint32_t tag,
                                                 uint64_t out4[4]) {
    uint64_t A[25];
#pragma unroll
    for (int i = 0; i < 25; i++) A[i] = 0;
    uint32_t carry = tag << 24;
    const uint32_t nfull = nw / 34;
#pragma unroll 1
    for (uint32_t b = 0; b < nfull; b++) {
        uint32_t D[34];
#pragma unroll
        for (int q = 0; q < 17; q++) {
            uint2 v = ld.v2(17 * b + q);
            D[2 * q] = v.x; D[2 * q + 1] = v.y;
        }
#pragma unroll
        for (int i = 0; i < 17; i++) {
            uint32_t prev = (i == 0) ? carry : D[2 * i - 1];
            uint32_t lo = kk_shift(prev, D[2 * i]);
            uint32_t hi = kk_shift(D[2 * i], D[2 * i + 1]);
            A[i] ^= ((uint64_t)hi << 32) | lo;
        }
        carry = D[33];
        keccak_f1600(A);
    }
    const uint32_t rem = nw - nfull * 34;
    const uint32_t base = nfull * 34;
    uint32_t E[34];
#pragma unroll
    for (int k = 0; k < 34; k++) {
        uint32_t v = 0;
        if ((uint32_t)k < rem) v = ld.w(base + k);
        else if ((uint32_t)k == rem) v = 0x01u;
        E[k] = v;
    }
#pragma unroll
    for (int i = 0; i < 17; i++) {
        uint32_t prev = (i == 0) ? carry : E[2 * i - 1];
        uint32_t lo = kk_shift(prev, E[2 * i]);
        uint32_t hi = kk_shift(E[2 * i], E[2 * i + 1]);
        if (i == 16) hi ^= 0x80000000u;
        A[i] ^= ((uint64_t)hi << 32) | lo;
    }
    keccak_f1600(A);
#pragma unroll
    for (int i = 0; i < 4; i++) out4[i] = A[i];
}

// ------------------------------------------------------------ loaders

struct GlobalWords {  // 16-byte aligned global payload, read-only path
    const uint32_t* __restrict__ p;
    __device__ __forceinline__ uint4 v4(uint32_t i) const {
        return __ldg(reinterpret_cast<const uint4*>(p) + i);
    }
    __device__ __forceinline__ uint2 v2(uint32_t i) const {
        return __ldg(reinterpret_cast<const uint2*>(p) + i);
    }
    __device__ __forceinline__ uint32_t w(uint32_t i) const { return __ldg(p + i); }
};

struct RegWords16 {  // two 32-byte digests held in registers (internal node)
    uint32_t m[16];
    __device__ __forceinline__ uint4 v4(uint32_t i) const {
        return make_uint4(m[4 * i], m[4 * i + 1], m[4 * i + 2], m[4 * i + 3]);
    }
    __device__ __forceinline__ uint2 v2(uint32_t i) const {
        return make_uint2(m[2 * i], m[2 * i + 1]);
    }
    __device__ __forceinline__ uint32_t w(uint32_t i) const { return m[i]; }
};

// Digest of tag || words, written as 8 little-endian words = the digest bytes.
template <int ALG, class Load>
__device__ __forceinline__ void hash_tagged_words(const Load& ld, uint32_t nw, uint32_t tag,
                                                  uint32_t out[8]) {
    if (ALG == kSHA256) {
        uint32_t st[8];
        sha256_tagged(ld, nw, tag, st);
#pragma unroll
        for (int i = 0; i < 8; i++) out[i] = bswap32(st[i]);
    } else {
        uint64_t o[4];
        keccak256_tagged(ld, nw, tag, o);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            out[2 * i] = (uint32_t)o[i];
            out[2 * i + 1] = (uint32_t)(o[i] >> 32);
        }
    }
}

// Internal node H(0x01 || L || R) of two digests in little-endian words.
template <int ALG>
__device__ __forceinline__ void hash_node(const uint32_t L[8], const uint32_t R[8],
                                          uint32_t out[8]) {
    RegWords16 ld;
#pragma unroll
    for (int i = 0; i < 8; i++) { ld.m[i] = L[i]; ld.m[8 + i] = R[i]; }
    hash_tagged_words<ALG>(ld, 16, 1u, out);
}

// ----------------------------------------------------- generic byte leaves

// Byte k of the padded message for an arbitrary-length leaf tag || p[0..len).
struct ByteMsg {
    const uint8_t* p;
    uint64_t len;
    uint8_t tag;
    __device__ __forceinline__ uint32_t byte_at(uint64_t k, uint8_t pad) const {
        if (k == 0) return tag;
        uint64_t d = k - 1;
        if (d < len) return p[d];
        return d == len ? pad : 0u;
    }
};

template <int ALG>
__device__ void hash_bytes_generic(const ByteMsg& m, uint32_t out[8]) {
    const uint64_t total = m.len + 1;
    if (ALG == kSHA256) {
        uint32_t st[8];
        sha256_init(st);
        const uint64_t nblk = (total + 1 + 8 + 63) / 64;
        const uint64_t bits = total * 8ull;
        for (uint64_t b = 0; b < nblk; b++) {
            uint32_t W[16];
            for (int j = 0; j < 16; j++) {
                uint64_t k = 64 * b + 4 * j;
                W[j] = (m.byte_at(k, 0x80) << 24) | (m.byte_at(k + 1, 0x80) << 16) |
                       (m.byte_at(k + 2, 0x80) << 8) | m.byte_at(k + 3, 0x80);
            }
            if (b == nblk - 1) {
                W[14] = (uint32_t)(bits >> 32);
                W[15] = (uint32_t)bits;
            }
            sha256_compress(st, W);
        }
        for (int i = 0; i < 8; i++) out[i] = bswap32(st[i]);
    } else {
        uint64_t A[25];
        for (int i = 0; i < 25; i++) A[i] = 0;
        const uint64_t nblk = total / 136 + 1;
        for (uint64_t b = 0; b < nblk; b++) {
            for (int i = 0; i < 17; i++) {
                uint64_t lane = 0;
                for (int q = 0; q < 8; q++)
                    lane |= (uint64_t)m.byte_at(136 * b + 8 * i + q, 0x01) << (8 * q);
                if (b == nblk - 1 && i == 16) lane ^= 0x8000000000000000ull;
                A[i] ^= lane;
            }
            keccak_f1600(A);
        }
        for (int i = 0; i < 4; i++) {
            out[2 * i] = (uint32_t)A[i];
            out[2 * i + 1] = (uint32_t)(A[i] >> 32);
        }
    }
}

}  // namespace nao
