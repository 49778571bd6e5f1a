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


__constant__ uint64_t c_keccak_rc[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808aull,
    0x8000000080008000ull, 0x000000000000808bull, 0x0000000080000001ull,
    0x8000000080008081ull, 0x8000000000008009ull, 0x000000000000008aull,
    0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000aull,
    0x000000008000808bull, 0x800000000000008bull, 0x8000000000008089ull,
    0x8000000000008003ull, 0x8000000000008002ull, 0x8000000000000080ull,
    0x000000000000800aull, 0x800000008000000aull, 0x8000000080008081ull,
    0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};


// Keccak-f[1600]; A[x + 5y].  The permutation runs on 32-bit halves: a 64-bit
// rotation is two funnel shifts (SHF.L.W) -- or a free half swap -- and the
// 3-input XOR / chi terms map to one LOP3 per half (~180 ALU ops per round).
struct Lane { uint32_t lo, hi; };
__device__ __forceinline__ Lane lxor(Lane a, Lane b) { return {a.lo ^ b.lo, a.hi ^ b.hi}; }

template <int N>
__device__ __forceinline__ Lane lrot(Lane x) {
    static_assert(N > 0 && N < 64, "rotation");
    if constexpr (N == 32) {
        return {x.hi, x.lo};
    } else if constexpr (N < 32) {
        return {__funnelshift_l(x.hi, x.lo, N), __funnelshift_l(x.lo, x.hi, N)};
    } else {
        return {__funnelshift_l(x.lo, x.hi, N - 32), __funnelshift_l(x.hi, x.lo, N - 32)};
    }
}
// The same rotation on the FMA pipe (the ALU pipe is the Keccak bound):
// IMAD.WIDE by 2^M from constant memory (opaque to ptxas, so it is not
// strength-reduced back to ALU shifts); the two halves never overlap, so the
// ORs are additions and fold into the multiply-adds.
__constant__ uint32_t c_pow2[32] = {
    1u << 0,  1u << 1,  1u << 2,  1u << 3,  1u << 4,  1u << 5,  1u << 6,  1u << 7,
    1u << 8,  1u << 9,  1u << 10, 1u << 11, 1u << 12, 1u << 13, 1u << 14, 1u << 15,
    1u << 16, 1u << 17, 1u << 18, 1u << 19, 1u << 20, 1u << 21, 1u << 22, 1u << 23,
    1u << 24, 1u << 25, 1u << 26, 1u << 27, 1u << 28, 1u << 29, 1u << 30, 1u << 31};
template <int N>
__device__ __forceinline__ Lane lrot_fma(Lane x) {
    static_assert(N > 0 && N < 64 && N != 32, "rotation");
    constexpr int M = N < 32 ? N : N - 32;
    const uint32_t L = N < 32 ? x.lo : x.hi, H = N < 32 ? x.hi : x.lo;
    const uint32_t p = c_pow2[M];
    const uint64_t P = (uint64_t)L * p;                 // {L << M, L >> (32-M)}
    const uint64_t Q = (uint64_t)H * p + (P >> 32);     // {(H << M) | (L >> (32-M)), H >> (32-M)}
    uint32_t lo;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(lo) : "r"((uint32_t)(Q >> 32)), "r"(c_pow2[0]),
        "r"((uint32_t)P));
    return {lo, (uint32_t)Q};
}
// 32-bit form: (H << M) | (L >> (32-M)) = H * 2^M + umulhi(L, 2^M), no register pairs
template <int N>
__device__ __forceinline__ Lane lrot_fma32(Lane x) {
    static_assert(N > 0 && N < 64 && N != 32, "rotation");
    constexpr int M = N < 32 ? N : N - 32;
    const uint32_t L = N < 32 ? x.lo : x.hi, H = N < 32 ? x.hi : x.lo;
    const uint32_t p = c_pow2[M];
    return {L * p + __umulhi(H, p), H * p + __umulhi(L, p)};
}
template <int N, int FMA>  // 0 ALU funnel shifts, 1 IMAD.WIDE form, 2 32-bit IMAD form
__device__ __forceinline__ Lane lrot_sel(Lane x) {
    if constexpr (FMA == 1 && N != 32) return lrot_fma<N>(x);
    else if constexpr (FMA == 2 && N != 32) return lrot_fma32<N>(x);
    else return lrot<N>(x);
}
#ifndef NAO_KECCAK_FMA_MASK
#define NAO_KECCAK_FMA_MASK 0u
#endif

__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
// a ^ c ^ r as one LOP3 per half (theta's D = c ^ r is never materialised)
__device__ __forceinline__ Lane lxor3(Lane a, Lane c, Lane r) {
    return {xor3(a.lo, c.lo, r.lo), xor3(a.hi, c.hi, r.hi)};
}
__device__ __forceinline__ Lane lxor5(Lane a, Lane b, Lane c, Lane d, Lane e) {
    return {xor3(xor3(a.lo, b.lo, c.lo), d.lo, e.lo), xor3(xor3(a.hi, b.hi, c.hi), d.hi, e.hi)};
}
__device__ __forceinline__ Lane lchi(Lane a, Lane b, Lane c) {
    return {a.lo ^ (~b.lo & c.lo), a.hi ^ (~b.hi & c.hi)};
}

#ifndef NAO_KECCAK_UNROLL
#define NAO_KECCAK_UNROLL 1
#endif
constexpr int kKeccakUnroll = NAO_KECCAK_UNROLL;  // rounds per loop iteration
// MASK bit j moves rotation j (0..23: rho in the order below, 24..28: theta)
// to the FMA pipe; bit 31 picks the 32-bit IMAD form over IMAD.WIDE.
template <uint32_t MASK>
__device__ __forceinline__ void keccak_f1600_m(uint64_t Aw[25]) {
    Lane A[25];
#pragma unroll
    for (int i = 0; i < 25; i++) A[i] = {(uint32_t)Aw[i], (uint32_t)(Aw[i] >> 32)};
#pragma unroll kKeccakUnroll
    for (int r = 0; r < 24; r++) {
        const Lane C0 = lxor5(A[0], A[5], A[10], A[15], A[20]);
        const Lane C1 = lxor5(A[1], A[6], A[11], A[16], A[21]);
        const Lane C2 = lxor5(A[2], A[7], A[12], A[17], A[22]);
        const Lane C3 = lxor5(A[3], A[8], A[13], A[18], A[23]);
        const Lane C4 = lxor5(A[4], A[9], A[14], A[19], A[24]);
        // theta + rho + pi:  B[y + 5*((2x+3y)%5)] = rotl(A[x+5y] ^ D[x], r[x][y]),
        // D[x] = C[x-1] ^ rotl(C[x+1], 1)
#define NAO_R(N, j) lrot_sel<N, ((MASK >> (j)) & 1u) ? ((MASK >> 31) ? 2 : 1) : 0>
        const Lane R0 = NAO_R(1, 24)(C1), R1 = NAO_R(1, 25)(C2), R2 = NAO_R(1, 26)(C3),
                   R3 = NAO_R(1, 27)(C4), R4 = NAO_R(1, 28)(C0);
#define NAO_TH(i, x) lxor3(A[i], C##x##m, R##x)
        const Lane C0m = C4, C1m = C0, C2m = C1, C3m = C2, C4m = C3;
        const Lane B00 = NAO_TH(0, 0);
        const Lane B10 = NAO_R(44, 0)(NAO_TH(6, 1));
        const Lane B20 = NAO_R(43, 1)(NAO_TH(12, 2));
        const Lane B30 = NAO_R(21, 2)(NAO_TH(18, 3));
        const Lane B40 = NAO_R(14, 3)(NAO_TH(24, 4));
        const Lane B01 = NAO_R(28, 4)(NAO_TH(3, 3));
        const Lane B11 = NAO_R(20, 5)(NAO_TH(9, 4));
        const Lane B21 = NAO_R(3, 6)(NAO_TH(10, 0));
        const Lane B31 = NAO_R(45, 7)(NAO_TH(16, 1));
        const Lane B41 = NAO_R(61, 8)(NAO_TH(22, 2));
        const Lane B02 = NAO_R(1, 9)(NAO_TH(1, 1));
        const Lane B12 = NAO_R(6, 10)(NAO_TH(7, 2));
        const Lane B22 = NAO_R(25, 11)(NAO_TH(13, 3));
        const Lane B32 = NAO_R(8, 12)(NAO_TH(19, 4));
        const Lane B42 = NAO_R(18, 13)(NAO_TH(20, 0));
        const Lane B03 = NAO_R(27, 14)(NAO_TH(4, 4));
        const Lane B13 = NAO_R(36, 15)(NAO_TH(5, 0));
        const Lane B23 = NAO_R(10, 16)(NAO_TH(11, 1));
        const Lane B33 = NAO_R(15, 17)(NAO_TH(17, 2));
        const Lane B43 = NAO_R(56, 18)(NAO_TH(23, 3));
        const Lane B04 = NAO_R(62, 19)(NAO_TH(2, 2));
        const Lane B14 = NAO_R(55, 20)(NAO_TH(8, 3));
        const Lane B24 = NAO_R(39, 21)(NAO_TH(14, 4));
        const Lane B34 = NAO_R(41, 22)(NAO_TH(15, 0));
        const Lane B44 = NAO_R(2, 23)(NAO_TH(21, 1));
#undef NAO_TH
#undef NAO_R
        // chi (row y: lanes Bxy for x=0..4) + iota
        const uint64_t rc = c_keccak_rc[r];
        A[0] = lchi(B00, B10, B20);
        A[0].lo ^= (uint32_t)rc; A[0].hi ^= (uint32_t)(rc >> 32);
        A[1] = lchi(B10, B20, B30); A[2] = lchi(B20, B30, B40);
        A[3] = lchi(B30, B40, B00); A[4] = lchi(B40, B00, B10);
        A[5] = lchi(B01, B11, B21); A[6] = lchi(B11, B21, B31); A[7] = lchi(B21, B31, B41);
        A[8] = lchi(B31, B41, B01); A[9] = lchi(B41, B01, B11);
        A[10] = lchi(B02, B12, B22); A[11] = lchi(B12, B22, B32); A[12] = lchi(B22, B32, B42);
        A[13] = lchi(B32, B42, B02); A[14] = lchi(B42, B02, B12);
        A[15] = lchi(B03, B13, B23); A[16] = lchi(B13, B23, B33); A[17] = lchi(B23, B33, B43);
        A[18] = lchi(B33, B43, B03); A[19] = lchi(B43, B03, B13);
        A[20] = lchi(B04, B14, B24); A[21] = lchi(B14, B24, B34); A[22] = lchi(B24, B34, B44);
        A[23] = lchi(B34, B44, B04); A[24] = lchi(B44, B04, B14);
    }
#pragma unroll
    for (int i = 0; i < 25; i++) Aw[i] = ((uint64_t)A[i].hi << 32) | A[i].lo;
}
__device__ __forceinline__ void keccak_f1600(uint64_t Aw[25]) {
    keccak_f1600_m<NAO_KECCAK_FMA_MASK>(Aw);
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
            uint2 v = ld.v2c(17 * b + q, q);  // q: compile-time pair index in the block
            D[2 * q] = v.x; D[2 * q + 1] = v.y;
        }
        ld.block_end(b);
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
        if ((uint32_t)k < rem) v = ld.wc(base + k, k);
        else if ((uint32_t)k == rem) v = 0x01u;
        E[k] = v;
    }
    ld.block_end(nfull);
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

// Loaders.  The Keccak sponge reads a 136-byte block as 17 word pairs
// (v2c(i, q), q the compile-time pair index within the block) or, for the
// last block, words (wc(i, k)), then calls block_end(b): hooks for loaders
// that inspect what they load (the fused check's CheckedWords); plain
// loaders forward to v2 / w and ignore block_end.
struct GlobalWords {  // 16-byte aligned global payload, read-only path
    const uint32_t* __restrict__ p;
    __device__ __forceinline__ uint4 v4(uint32_t i) const {
        return __ldg(reinterpret_cast<const uint4*>(p) + i);
    }
    __device__ __forceinline__ uint2 v2(uint32_t i) const {
        return __ldg(reinterpret_cast<const uint2*>(p) + i);
    }
    __device__ __forceinline__ uint32_t w(uint32_t i) const { return __ldg(p + i); }
    __device__ __forceinline__ uint2 v2c(uint32_t i, int) const { return v2(i); }
    __device__ __forceinline__ uint32_t wc(uint32_t i, int) const { return w(i); }
    __device__ __forceinline__ void block_end(uint32_t) const {}
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
    __device__ __forceinline__ uint2 v2c(uint32_t i, int) const { return v2(i); }
    __device__ __forceinline__ uint32_t wc(uint32_t i, int) const { return w(i); }
    __device__ __forceinline__ void block_end(uint32_t) const {}
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
