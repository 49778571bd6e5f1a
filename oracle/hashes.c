/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and only
 * as the checker.  The product (paper_2510_16028_b200) never links it.
 *
 * Plain-C restatement of the two hash functions the commitment layer uses:
 *   - SHA-256 (FIPS 180-4).  The reference hashes with OpenSSL via hashlib
 *     (/root/reference/pkg/src/fpverify/commitments.py:31-32); this C copy is
 *     cross-checked against hashlib in tests/test_oracle.py.
 *   - Keccak-256 (the original Keccak submission padding 0x01, as used by
 *     Ethereum).  The reference has NO Keccak: parity for this
 *     mode is pinned by known-answer tests (keccak256("") / ("abc")) and by
 *     reproducing hashlib.sha3_256 when the pad byte is switched to 0x06.
 *
 * Also exports the chunked Merkle construction used by the oracle's tensor
 * commitment (leaf = H(0x00||x), node = H(0x01||L||R), odd node pairs with
 * itself; commitments.py:112-142), multi-threaded over leaves with OpenMP so it
 * can serve as the CPU baseline.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ SHA-256 */

static const uint32_t K256[64] = {
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

#define ROR32(x, n) (((x) >> (n)) | ((x) << (32 - (n))))

static void sha256_compress(uint32_t st[8], const uint8_t blk[64]) {
    uint32_t w[64];
    for (int i = 0; i < 16; i++)
        w[i] = ((uint32_t)blk[4 * i] << 24) | ((uint32_t)blk[4 * i + 1] << 16) |
               ((uint32_t)blk[4 * i + 2] << 8) | (uint32_t)blk[4 * i + 3];
    for (int i = 16; i < 64; i++) {
        uint32_t s0 = ROR32(w[i - 15], 7) ^ ROR32(w[i - 15], 18) ^ (w[i - 15] >> 3);
        uint32_t s1 = ROR32(w[i - 2], 17) ^ ROR32(w[i - 2], 19) ^ (w[i - 2] >> 10);
        w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3];
    uint32_t e = st[4], f = st[5], g = st[6], h = st[7];
    for (int i = 0; i < 64; i++) {
        uint32_t S1 = ROR32(e, 6) ^ ROR32(e, 11) ^ ROR32(e, 25);
        uint32_t ch = (e & f) ^ (~e & g);
        uint32_t t1 = h + S1 + ch + K256[i] + w[i];
        uint32_t S0 = ROR32(a, 2) ^ ROR32(a, 13) ^ ROR32(a, 22);
        uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        uint32_t t2 = S0 + mj;
        h = g; g = f; f = e; e = d + t1;
        d = c; c = b; b = a; a = t1 + t2;
    }
    st[0] += a; st[1] += b; st[2] += c; st[3] += d;
    st[4] += e; st[5] += f; st[6] += g; st[7] += h;
}

/* SHA-256 over the concatenation prefix(plen) || data(len). */
static void sha256_2(const uint8_t* pre, size_t plen, const uint8_t* data, size_t len,
                     uint8_t out[32]) {
    uint32_t st[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                      0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
    uint8_t blk[64];
    size_t fill = 0;
    uint64_t total = (uint64_t)plen + (uint64_t)len;
    const uint8_t* srcs[2] = {pre, data};
    size_t lens[2] = {plen, len};
    for (int s = 0; s < 2; s++) {
        const uint8_t* p = srcs[s];
        size_t n = lens[s];
        while (n) {
            size_t take = 64 - fill < n ? 64 - fill : n;
            memcpy(blk + fill, p, take);
            fill += take; p += take; n -= take;
            if (fill == 64) { sha256_compress(st, blk); fill = 0; }
        }
    }
    blk[fill++] = 0x80;
    if (fill > 56) {
        memset(blk + fill, 0, 64 - fill);
        sha256_compress(st, blk);
        fill = 0;
    }
    memset(blk + fill, 0, 56 - fill);
    uint64_t bits = total * 8u;
    for (int i = 0; i < 8; i++) blk[56 + i] = (uint8_t)(bits >> (56 - 8 * i));
    sha256_compress(st, blk);
    for (int i = 0; i < 8; i++) {
        out[4 * i] = (uint8_t)(st[i] >> 24); out[4 * i + 1] = (uint8_t)(st[i] >> 16);
        out[4 * i + 2] = (uint8_t)(st[i] >> 8); out[4 * i + 3] = (uint8_t)st[i];
    }
}

/* ---------------------------------------------------------------- Keccak-f */

static const uint64_t KRC[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808aull,
    0x8000000080008000ull, 0x000000000000808bull, 0x0000000080000001ull,
    0x8000000080008081ull, 0x8000000000008009ull, 0x000000000000008aull,
    0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000aull,
    0x000000008000808bull, 0x800000000000008bull, 0x8000000000008089ull,
    0x8000000000008003ull, 0x8000000000008002ull, 0x8000000000000080ull,
    0x000000000000800aull, 0x800000008000000aull, 0x8000000080008081ull,
    0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};

/* rotation offsets r[x][y] from the Keccak reference, lane index x + 5y */
static const int KROT[25] = {0, 1, 62, 28, 27, 36, 44, 6, 55, 20, 3, 10, 43,
                             25, 39, 41, 45, 15, 21, 8, 18, 2, 61, 56, 14};

#define ROL64(x, n) ((n) == 0 ? (x) : (((x) << (n)) | ((x) >> (64 - (n)))))

static void keccak_f1600(uint64_t A[25]) {
    for (int round = 0; round < 24; round++) {
        uint64_t C[5], D[5], B[25];
        for (int x = 0; x < 5; x++)
            C[x] = A[x] ^ A[x + 5] ^ A[x + 10] ^ A[x + 15] ^ A[x + 20];
        for (int x = 0; x < 5; x++) D[x] = C[(x + 4) % 5] ^ ROL64(C[(x + 1) % 5], 1);
        for (int i = 0; i < 25; i++) A[i] ^= D[i % 5];
        /* rho + pi: B[y, 2x+3y] = rot(A[x,y], r[x,y]) */
        for (int x = 0; x < 5; x++)
            for (int y = 0; y < 5; y++) {
                int X = y, Y = (2 * x + 3 * y) % 5;
                B[X + 5 * Y] = ROL64(A[x + 5 * y], KROT[x + 5 * y]);
            }
        for (int y = 0; y < 5; y++)
            for (int x = 0; x < 5; x++)
                A[x + 5 * y] = B[x + 5 * y] ^ (~B[(x + 1) % 5 + 5 * y] & B[(x + 2) % 5 + 5 * y]);
        A[0] ^= KRC[round];
    }
}

/* Keccak sponge, rate 136 B, 32-byte output, domain pad byte `pad`
 * (0x01 = Keccak-256, 0x06 = FIPS-202 SHA3-256), over prefix || data. */
static void keccak256_2(const uint8_t* pre, size_t plen, const uint8_t* data, size_t len,
                        uint8_t pad, uint8_t out[32]) {
    uint64_t A[25];
    memset(A, 0, sizeof A);
    uint8_t blk[136];
    size_t fill = 0;
    const uint8_t* srcs[2] = {pre, data};
    size_t lens[2] = {plen, len};
    for (int s = 0; s < 2; s++) {
        const uint8_t* p = srcs[s];
        size_t n = lens[s];
        while (n) {
            size_t take = 136 - fill < n ? 136 - fill : n;
            memcpy(blk + fill, p, take);
            fill += take; p += take; n -= take;
            if (fill == 136) {
                for (int i = 0; i < 17; i++) {
                    uint64_t v = 0;
                    for (int b = 0; b < 8; b++) v |= (uint64_t)blk[8 * i + b] << (8 * b);
                    A[i] ^= v;
                }
                keccak_f1600(A);
                fill = 0;
            }
        }
    }
    memset(blk + fill, 0, 136 - fill);
    blk[fill] ^= pad;
    blk[135] ^= 0x80;
    for (int i = 0; i < 17; i++) {
        uint64_t v = 0;
        for (int b = 0; b < 8; b++) v |= (uint64_t)blk[8 * i + b] << (8 * b);
        A[i] ^= v;
    }
    keccak_f1600(A);
    for (int i = 0; i < 4; i++)
        for (int b = 0; b < 8; b++) out[8 * i + b] = (uint8_t)(A[i] >> (8 * b));
}

/* ------------------------------------------------------------------ exports */

/* alg: 0 = SHA-256, 1 = Keccak-256 (pad 0x01), 2 = SHA3-256 (pad 0x06, test only) */
void oracle_hash(int alg, const uint8_t* pre, size_t plen, const uint8_t* data, size_t len,
                 uint8_t out[32]) {
    if (alg == 0) sha256_2(pre, plen, data, len, out);
    else keccak256_2(pre, plen, data, len, alg == 2 ? 0x06 : 0x01, out);
}

/* Leaf digests H(0x00 || chunk_i) for payload split into chunk_bytes pieces
 * (the last piece may be short).  n_chunks = ceil(len / chunk_bytes). */
void oracle_chunk_leaves(int alg, const uint8_t* data, uint64_t len, uint64_t chunk_bytes,
                         uint8_t* out, int n_threads) {
    const uint8_t tag = 0x00;
    int64_t n = (int64_t)((len + chunk_bytes - 1) / chunk_bytes);
#pragma omp parallel for schedule(static) num_threads(n_threads) if (n_threads > 1)
    for (int64_t i = 0; i < n; i++) {
        uint64_t off = (uint64_t)i * chunk_bytes;
        uint64_t take = len - off < chunk_bytes ? len - off : chunk_bytes;
        oracle_hash(alg, &tag, 1, data + off, take, out + 32 * i);
    }
}

/* One Merkle level: out[j] = H(0x01 || in[2j] || in[2j+1]) with the odd last
 * node paired with itself (commitments.py:119-126). */
void oracle_tree_level(int alg, const uint8_t* in, int64_t n_in, uint8_t* out, int n_threads) {
    int64_t n_out = (n_in + 1) / 2;
#pragma omp parallel for schedule(static) num_threads(n_threads) if (n_threads > 1)
    for (int64_t j = 0; j < n_out; j++) {
        uint8_t buf[64];
        const uint8_t* l = in + 64 * j;
        const uint8_t* r = (2 * j + 1 < n_in) ? in + 64 * j + 32 : l;
        memcpy(buf, l, 32);
        memcpy(buf + 32, r, 32);
        const uint8_t tag = 0x01;
        oracle_hash(alg, &tag, 1, buf, 64, out + 32 * j);
    }
}
