// Chunked Merkle commitment of traced tensors (north_star (4)).
//
// Per tensor:  leaves = [canon header] + [payload chunk_i]  (chunk = C bytes)
//              root   = MerkleTree(H(0x00||leaf)).root     (commitments.py:112-142)
// Kernels:
//   k_chunk_leaves : one thread per payload chunk, batched over up to kMaxSegs
//                    tensors per launch (a whole layer's node outputs), so the
//                    grid fills 148 SMs even for 33 MB tensors.
//   k_bytes_leaves : generic odd-length leaves (headers, JSON chunks).
//   k_tree_reduce  : each CTA folds an aligned group of 2^lg nodes of one level
//                    through lg levels in shared memory (odd node pairs with
//                    itself; aligned groups reproduce the global tree exactly).
#include <cstdio>
#include <cstdarg>
#include <vector>
#include <algorithm>
#include <cstdlib>

#include <array>
#include <map>
#include <mutex>
#include "common.cuh"
#include "check_common.cuh"
#include "unary.cuh"
#include "hash.cuh"

namespace nao {

constexpr int kMaxSegs = 128;
constexpr int kTreeThreads = 256;  // a CTA folds up to 512 nodes
constexpr uint64_t kFlatLevelMin = 1u << 16;  // live nodes from which levels run flat

struct ChunkTable {
    int n;
    uint32_t chunk_words;
    const uint32_t* payload[kMaxSegs];
    uint64_t nbytes[kMaxSegs];
    uint64_t chunk_prefix[kMaxSegs + 1];  // cumulative chunk counts
    uint64_t out_index[kMaxSegs];         // digest index of chunk 0
};

constexpr int kMaxHeader = 136;  // canon header of rank <= 8: 5 + 16*rank bytes

struct HeaderTable {  // passed by value: no host->device staging, no sync
    int n;
    uint32_t len[kMaxSegs];
    uint64_t out_index[kMaxSegs];
    uint8_t bytes[kMaxSegs][kMaxHeader];
};

struct TreeTable {
    int n;
    int lg;                                // levels folded per CTA
    int full_levels[kMaxSegs];             // 1: fold exactly lg levels (>1 group)
    uint64_t in_index[kMaxSegs];
    uint64_t n_in[kMaxSegs];
    uint64_t out_index[kMaxSegs];
    uint64_t group_prefix[kMaxSegs + 1];
};

__device__ __forceinline__ int find_seg(const uint64_t* prefix, int n, uint64_t t) {
    int lo = 0, hi = n;  // prefix[lo] <= t < prefix[hi]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (prefix[mid] <= t) lo = mid; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ void store_digest(uint32_t* dst, const uint32_t d[8]) {
    uint4* p = reinterpret_cast<uint4*>(dst);
    p[0] = make_uint4(d[0], d[1], d[2], d[3]);
    p[1] = make_uint4(d[4], d[5], d[6], d[7]);
}

template <int ALG>
__global__ void __launch_bounds__(128) k_chunk_leaves(const __grid_constant__ ChunkTable tab,
                                                      uint32_t* __restrict__ digests) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= tab.chunk_prefix[tab.n]) return;
    const int s = find_seg(tab.chunk_prefix, tab.n, t);
    const uint64_t c = t - tab.chunk_prefix[s];
    const uint64_t off_w = c * tab.chunk_words;
    const uint64_t total_w = tab.nbytes[s] >> 2;
    const uint32_t nw = (uint32_t)(total_w - off_w < tab.chunk_words ? total_w - off_w : tab.chunk_words);
    GlobalWords ld{tab.payload[s] + off_w};
    uint32_t d[8];
    hash_tagged_words<ALG>(ld, nw, 0u, d);
    store_digest(digests + 8 * (tab.out_index[s] + c), d);
}

// ------------------------------------------ commit with the check fused in
//
// k_chunk_leaves_check: the same leaf hashing, plus the acceptance check of
// the claimed tensor against the locally recomputed one (nao_check's verdict,
// check.cu) folded into the loads: every claimed word the sponge absorbs is
// compared with the local word at the same offset.  Equal finite words (the
// common case) cost a load + two integer ops; the others take a divergent
// slow path (exact FP64 keys, bound, histogram buckets).  Keccak is
// integer-ALU bound (~33 ops/byte), so the check's extra HBM read rides under
// it instead of costing a separate 8 B/element pass.
// A CTA covers 128 consecutive chunks of ONE tensor; the last CTA of a tensor
// decides its verdict (histogram verdict + rare exact second pass).

#ifndef NAO_CC_PROBE
#define NAO_CC_PROBE 0
#endif
constexpr int kLeafThreads = 128;

struct CheckDesc {  // == nao_check_desc (include/nao_b200.h)
    const float* local;
    const void* eps;
    const VerdictSpec* spec;
    nao_check_result* result;
    double eps_scale;
    double lo_factor;
    int32_t eps_kind;
    int32_t flags;
    unsigned long long* border_list;
    long long border_cap;
};
static_assert(sizeof(CheckDesc) == sizeof(nao_check_desc), "nao_check_desc layout");
static_assert(sizeof(nao_check_partial) == 8 * (5 + 2 * 33 + 4 * 33), "nao_check_partial layout");

struct CCTable {
    int n;
    uint32_t chunk_words;
    const uint32_t* payload[kMaxSegs];
    uint64_t nbytes[kMaxSegs];
    uint64_t out_index[kMaxSegs];
    uint64_t block_prefix[kMaxSegs + 1];
    CheckDesc chk[kMaxSegs];
    uint64_t reuse_out[kMaxSegs];    // digest index of the source's chunk 0, or ~0 (none)
    uint64_t reuse_block[kMaxSegs];  // chunks per source block
    uint64_t reuse_span[kMaxSegs];   // block_chunks * repeats
    const uint32_t* reuse_src[kMaxSegs];  // same-offset mode: the source's claimed payload
    uint32_t row_chunks[kMaxSegs];   // chunk -> CTA mapping (0: identity)
    const uint32_t* ref_payload[kMaxSegs];  // broadcast reference tensor, or null
    const uint32_t* ref_digests[kMaxSegs];  // its chunk digests
    uint64_t ref_chunks[kMaxSegs];
    uint32_t zero_digest[8];         // H(0x00 || zeros(chunk)), valid if zero_ok
    int zero_ok;
};

constexpr int kLeafWarps = kLeafThreads / 32;
__device__ unsigned long long g_reused_chunks = 0;  // nao_commit_stats
#ifndef NAO_SCAN_U
#define NAO_SCAN_U 4  // 16-byte words per lane in flight in the shortcut scan (x3 tensors)
#endif
constexpr int kMaxFusedChunkWords = 4096;  // 16 KiB chunks: 64 mask words per thread
constexpr float kGuard32 = 1.0f / 524288.0f;  // 2^-19 guard of the FP32 relative-key search

struct LeafCheckSmem {
    double t_abs[kMaxGrid], t_rel[kMaxGrid];
    float f_rel[kMaxGrid], f_rel_lo[kMaxGrid], f_rel_hi[kMaxGrid];
    float f_abs[kMaxGrid], f_abs_lo[kMaxGrid], f_abs_hi[kMaxGrid];
    unsigned int wc[kLeafWarps][2][kMaxGrid + 1];  // warp-private interval counters
    unsigned long long q[kLeafWarps][96];           // warp queue of flagged element indices
    unsigned long long bmax[2][kMaxGrid + 1];       // partial mode: per-bucket key range
    unsigned long long bmin_inv[2][kMaxGrid + 1];
    unsigned long long viol, border, nonfin, nslow;
    unsigned long long maxr_bits;
    int is_last;
    VerdictSmem vs;
};

__device__ __forceinline__ bool word_needs_check(uint32_t c, uint32_t y) {
    return (c != y) | ((c & 0x7f800000u) == 0x7f800000u);  // differs, or inf/nan
}
// The check's filter as FP32 compares (FSETP, off the integer-ALU pipe the
// sponge saturates): flags words that differ as floats or are inf / nan.
// +0 / -0 pairs pass unflagged -- their difference is exactly 0, the same
// verdict as equal words (the hash still absorbs the raw claimed bits).
__device__ __forceinline__ bool word_needs_check_f(uint32_t c, uint32_t y) {
    const float fc = __uint_as_float(c), fy = __uint_as_float(y);
    return !((fc == fy) & (fabsf(fc) <= 3.402823466e38f));
}
// warp-aggregated increment of a per-warp shared counter (lanes hitting the
// same bucket -- the common case -- add once instead of serialising)
__device__ __forceinline__ void agg_inc(unsigned int* ctr, unsigned key, unsigned active) {
    const unsigned peers = __match_any_sync(active, key);
    if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(ctr, (unsigned)__popc(peers));
}

// Claimed payload words for the sponge; a word that differs from the local
// word at the same offset (or is inf/nan) sets bit i%64 of this thread's
// mask word i/64 in shared memory -- the check itself runs after the hash.
// Check flags: one 64-bit mask entry per BW-word group of a thread's chunk
// (bit j = word BW*g + j needs the exact check).  Keccak-256: BW = 34, one
// entry per 136-byte sponge block, bit positions known at compile time (the
// block loop is unrolled), so a word costs two FP32 compares and one
// predicated LOP3 with an immediate -- no branch, no shifts.  SHA-256: BW = 64
// groups filled word by word.
template <int ALG> struct MaskGeom { static constexpr uint32_t BW = ALG == kKECCAK256 ? 34u : 64u; };

template <int ALG>
struct CheckedWords {
    const uint32_t* __restrict__ p;  // claimed (hashed)
    const uint32_t* __restrict__ q;  // local
    unsigned long long* mask;        // this thread's mask entries (stride kLeafThreads)
    mutable uint32_t lo = 0, hi = 0, grp = 0;
    __device__ __forceinline__ void put(bool f, int bitpos) const {  // bitpos: compile time
        if (bitpos < 32) lo |= f ? (1u << (bitpos & 31)) : 0u;
        else hi |= f ? (1u << (bitpos & 31)) : 0u;
    }
    __device__ __forceinline__ void store(uint32_t g) const {
        mask[g * kLeafThreads] = ((unsigned long long)hi << 32) | lo;
        lo = hi = 0;
    }
    // Keccak hooks
    __device__ __forceinline__ uint2 v2c(uint32_t i, int qp) const {
        const uint2 c = __ldg(reinterpret_cast<const uint2*>(p) + i);
#if NAO_CC_PROBE != 2
        const uint2 y = __ldg(reinterpret_cast<const uint2*>(q) + i);
        put(word_needs_check_f(c.x, y.x), 2 * qp);
        put(word_needs_check_f(c.y, y.y), 2 * qp + 1);
#endif
        return c;
    }
    __device__ __forceinline__ uint32_t wc(uint32_t i, int k) const {
        const uint32_t c = __ldg(p + i);
#if NAO_CC_PROBE != 2
        put(word_needs_check_f(c, __ldg(q + i)), k);
#endif
        return c;
    }
    __device__ __forceinline__ void block_end(uint32_t b) const { store(b); }
    // SHA-256 path: word by word into 64-word groups
    __device__ __forceinline__ void cmp(uint32_t c, uint32_t y, uint32_t i) const {
#if NAO_CC_PROBE != 2
        const uint32_t g = i >> 6;
        if (g != grp) { store(grp); grp = g; }
        const uint32_t bit = 1u << (i & 31);
        const bool f = word_needs_check_f(c, y);
        if (i & 32) hi |= f ? bit : 0u;
        else lo |= f ? bit : 0u;
#endif
    }
    __device__ __forceinline__ void finish() const { if (ALG != kKECCAK256) store(grp); }
    __device__ __forceinline__ uint4 v4(uint32_t i) const {
        const uint4 c = __ldg(reinterpret_cast<const uint4*>(p) + i);
        const uint4 y = __ldg(reinterpret_cast<const uint4*>(q) + i);
        cmp(c.x, y.x, 4 * i); cmp(c.y, y.y, 4 * i + 1);
        cmp(c.z, y.z, 4 * i + 2); cmp(c.w, y.w, 4 * i + 3);
        return c;
    }
    __device__ __forceinline__ uint2 v2(uint32_t i) const {
        const uint2 c = __ldg(reinterpret_cast<const uint2*>(p) + i);
        const uint2 y = __ldg(reinterpret_cast<const uint2*>(q) + i);
        cmp(c.x, y.x, 2 * i); cmp(c.y, y.y, 2 * i + 1);
        return c;
    }
    __device__ __forceinline__ uint32_t w(uint32_t i) const {
        const uint32_t c = __ldg(p + i), y = __ldg(q + i);
        cmp(c, y, i);
        return c;
    }
};

// Per-lane check state (the standalone k_check's `process`, check.cu).
struct LaneCheck {
    unsigned long long viol = 0, border = 0, nonfin = 0;
    double best_num = 0.0, best_den = 1.0;  // running max of diff/eps as a fraction
    bool best_inf = false;
};

struct Flagged { float y, c; double eps; unsigned long long idx; };

__device__ __forceinline__ Flagged load_flagged(const CheckDesc& d, const float* claimed,
                                                uint64_t idx) {
    Flagged f;
    f.idx = idx;
    f.y = __ldg(d.local + idx);
    f.c = __ldg(claimed + idx);
    f.eps = 0.0;
    if (d.eps_kind == NAO_EPS_TENSOR_F32) f.eps = (double)__ldg(static_cast<const float*>(d.eps) + idx);
    else if (d.eps_kind == NAO_EPS_TENSOR_F64) f.eps = __ldg(static_cast<const double*>(d.eps) + idx);
    return f;
}

__device__ __forceinline__ void process_finite(const CheckDesc& d, const Flagged& f, int G,
                                               double epsilon, LeafCheckSmem& sm, int w,
                                               LaneCheck& lc, unsigned active_all);

// `active`: the lanes calling (all of them in the full-queue path); the
// histogram counters are incremented warp-aggregated over equal buckets
__device__ __forceinline__ void process_flagged(const CheckDesc& d, const Flagged& f, int G,
                                                double epsilon, LeafCheckSmem& sm, int w,
                                                LaneCheck& lc, unsigned active) {
    const bool fin = isfinite(f.y) && isfinite(f.c);
    const unsigned finm = __ballot_sync(active, fin);
    if (!fin) {
        lc.nonfin++; lc.viol++;
        agg_inc(&sm.wc[w][0][G], (unsigned)G, active & ~finm);
        agg_inc(&sm.wc[w][1][G], (unsigned)G, active & ~finm);
        return;
    }
    process_finite(d, f, G, epsilon, sm, w, lc, finm);
}

__device__ __forceinline__ void process_finite(const CheckDesc& d, const Flagged& f, int G,
                                               double epsilon, LeafCheckSmem& sm, int w,
                                               LaneCheck& lc, unsigned active_all) {
    const float y = f.y, c = f.c;
    double eps = f.eps;
    if (d.eps_kind == NAO_EPS_SCALED_LOCAL) eps = __dmul_rn(d.eps_scale, fabs((double)y));
    const double diff = abs_key(y, c);
    if (diff > eps) lc.viol++;
    else if (diff > eps * d.lo_factor) {
        lc.border++;
        if (d.border_list) list_push(d.border_list, d.border_cap, f.idx);
    }
    if (eps > 0.0) {
        if (!lc.best_inf && diff * lc.best_den > lc.best_num * eps) { lc.best_num = diff; lc.best_den = eps; }
    } else if (diff > 0.0) {
        lc.best_inf = true;
    }
    int pa = 0, q = 0;
    if (d.flags & NAO_CHECK_PARTIAL) {  // exact keys + per-bucket key ranges
        const double rel = rel_key(diff, y, epsilon);
        if (diff != 0.0) {
            pa = bsearch_pos(sm.t_abs, G, diff);
            q = bsearch_pos(sm.t_rel, G, rel);
        }
        const unsigned long long ba = (unsigned long long)__double_as_longlong(diff);
        const unsigned long long br = (unsigned long long)__double_as_longlong(rel);
        atomicMax(&sm.bmax[0][pa], ba); atomicMax(&sm.bmin_inv[0][pa], ~ba);
        atomicMax(&sm.bmax[1][q], br); atomicMax(&sm.bmin_inv[1][q], ~br);
    } else if (diff != 0.0) {
        // FP32 bucket searches with a 2^-19 guard band around every threshold;
        // keys inside a band (or tiny) take the exact FP64 search
        const float d32 = (float)diff;
        pa = bsearch_pos32(sm.f_abs, G, d32);
        const bool safe_a = (d32 >= 1e-30f) && isfinite(d32) &&
                            (pa == G || d32 < sm.f_abs_lo[pa]) && (pa == 0 || d32 > sm.f_abs_hi[pa - 1]);
        if (!safe_a) pa = bsearch_pos(sm.t_abs, G, diff);
        const float r32 = __fdividef(d32, __fadd_rn(fabsf(y), (float)epsilon));  // ~2 ulp
        q = bsearch_pos32(sm.f_rel, G, r32);
        const bool safe = (d32 >= 1e-30f) && (r32 >= 1e-30f) && isfinite(r32) &&
                          (q == G || r32 < sm.f_rel_lo[q]) && (q == 0 || r32 > sm.f_rel_hi[q - 1]);
        if (!safe) q = bsearch_pos(sm.t_rel, G, rel_key(diff, y, epsilon));
    }
    agg_inc(&sm.wc[w][0][pa], (unsigned)pa, active_all);
    agg_inc(&sm.wc[w][1][q], (unsigned)q, active_all);
}

template <int ALG>
__device__ __forceinline__ void leaf_check_block(const CCTable& tab, uint32_t* __restrict__ digests,
                                                 CheckAccum* __restrict__ accs, LeafCheckSmem& sm,
                                                 unsigned long long* s_mask, uint64_t vb) {
    const int s = find_seg(tab.block_prefix, tab.n, vb);  // block-uniform
    const CheckDesc& d = tab.chk[s];
    const bool check = d.local != nullptr;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t total_w = tab.nbytes[s] >> 2;
    const uint32_t cw = tab.chunk_words;
    constexpr uint32_t BW = MaskGeom<ALG>::BW;
    // mask entries per thread: Keccak one per sponge block (the tail block's
    // entry always exists), SHA-256 one per 64 words
    const uint32_t groups = ALG == kKECCAK256 ? cw / BW + 1 : (cw + 63) >> 6;
    const uint64_t nchunks = (total_w + cw - 1) / cw;
    // chunk of this thread.  Rows of rc > 1 whole chunks: virtual block vl
    // takes chunk position vl % rc of 128 consecutive rows, so one CTA meets
    // one kind of chunk (e.g. the all-zero right halves of causal softmax
    // rows) and a CTA whose chunks all take a digest shortcut ends early.
    const uint64_t vl = vb - tab.block_prefix[s];
    const uint32_t rc = tab.row_chunks[s];
    uint64_t c, cta_words;
    bool active;
    if (rc > 1) {
        const uint64_t nrows = nchunks / rc, r0 = (vl / rc) * kLeafThreads;
        c = (r0 + threadIdx.x) * rc + vl % rc;
        active = r0 + threadIdx.x < nrows;
        cta_words = (nrows - r0 < (uint64_t)kLeafThreads ? nrows - r0 : (uint64_t)kLeafThreads) * cw;
    } else {
        const uint64_t c0 = vl * kLeafThreads;
        c = c0 + threadIdx.x;
        active = c < nchunks;
        const uint64_t c1 = c0 + kLeafThreads < nchunks ? c0 + kLeafThreads : nchunks;
        cta_words = (c1 * cw < total_w ? c1 * cw : total_w) - c0 * cw;
    }
    int G = 0;
    double epsilon = 0.0;
    if (check) {
        const VerdictSpec* v = d.spec;
        G = v->G;
        epsilon = v->epsilon;
        if (threadIdx.x < kMaxGrid) {
            const int i = threadIdx.x;
            const double ta = i < G ? v->t_abs[i] : INFINITY;
            const float fa = (float)ta;
            sm.f_abs[i] = fa;
            sm.f_abs_lo[i] = fa * (1.0f - kGuard32);
            sm.f_abs_hi[i] = fa * (1.0f + kGuard32);
            const double tr = i < G ? v->t_rel[i] : INFINITY;
            sm.t_abs[i] = ta;
            sm.t_rel[i] = tr;
            const float fr = (float)tr;
            sm.f_rel[i] = fr;
            sm.f_rel_lo[i] = fr * (1.0f - kGuard32);
            sm.f_rel_hi[i] = fr * (1.0f + kGuard32);
        }
        for (int b = lane; b <= kMaxGrid; b += 32) { sm.wc[w][0][b] = 0u; sm.wc[w][1][b] = 0u; }
        if (threadIdx.x < 2 * kMaxGrid) sm.vs.amb[threadIdx.x] = 0;
        for (int b = threadIdx.x; b < 2 * (kMaxGrid + 1); b += blockDim.x) {
            (&sm.bmax[0][0])[b] = 0ull;
            (&sm.bmin_inv[0][0])[b] = 0ull;
        }
        if (threadIdx.x == 0) {
            sm.viol = sm.border = sm.nonfin = sm.nslow = 0ull;
            sm.maxr_bits = 0ull;
            sm.is_last = 0;
        }
        for (uint32_t g = 0; g < groups; g++) s_mask[g * kLeafThreads + threadIdx.x] = 0ull;
        __syncthreads();
    }
    const uint64_t off_w = c * cw;
    const uint32_t nw = active ? (uint32_t)(total_w - off_w < cw ? total_w - off_w : cw) : 0u;
    bool reused = false;
    if (active && check && tab.reuse_out[s] != ~0ull && tab.reuse_src[s] == nullptr) {
        // data-movement node: claimed chunk == local chunk (word for word,
        // finite) means the source's chunk digest is this chunk's digest
        const uint32_t* cp = tab.payload[s] + off_w;
        const uint32_t* lp = reinterpret_cast<const uint32_t*>(d.local) + off_w;
        bool eq = true;
        uint32_t i = 0;
        for (; i + 4 <= nw; i += 4) {
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(cp + i));
            const uint4 b = __ldg(reinterpret_cast<const uint4*>(lp + i));
            eq &= !(word_needs_check(a.x, b.x) | word_needs_check(a.y, b.y) |
                    word_needs_check(a.z, b.z) | word_needs_check(a.w, b.w));
        }
        for (; i < nw; i++) eq &= !word_needs_check(__ldg(cp + i), __ldg(lp + i));
        if (eq) {
            const uint64_t span = tab.reuse_span[s], blk = tab.reuse_block[s];
            const uint64_t sc = (c / span) * blk + c % blk;
            const uint4* src = reinterpret_cast<const uint4*>(digests + 8 * (tab.reuse_out[s] + sc));
            uint4* dst = reinterpret_cast<uint4*>(digests + 8 * (tab.out_index[s] + c));
            dst[0] = src[0];
            dst[1] = src[1];
            reused = true;
        }
    }
    if (ALG == kKECCAK256 && check &&
        (tab.reuse_src[s] != nullptr || tab.ref_payload[s] != nullptr || tab.zero_ok) &&
        (cw & 3u) == 0u) {
        // digest shortcut: a claimed chunk equal to the same-offset chunk of the
        // source (REUSE_SAME_OFFSET), to a chunk of the broadcast reference
        // tensor, or to zeros, takes that chunk's digest.  Each lane probes its
        // chunk's first and last 16 bytes against the candidates; the warp then
        // scans every candidate chunk together (coalesced 16-byte loads of
        // claimed, local and reference), setting the owner's check flags at the
        // sponge-block bit positions the hash pass would use.  Candidates that
        // turn out to differ are hashed.
        const uint32_t* refp = nullptr;  // reference words of this lane's chunk (null: zeros)
        const uint32_t* digp = nullptr;  // its digest
        bool cand = false;
        if (active && !reused && nw == cw) {
            const uint32_t* cp = tab.payload[s] + off_w;
            const uint4 a0 = __ldg(reinterpret_cast<const uint4*>(cp));
            const uint4 a1 = __ldg(reinterpret_cast<const uint4*>(cp + cw - 4));
            auto probe = [&](const uint32_t* r) {
                const uint4 b0 = __ldg(reinterpret_cast<const uint4*>(r));
                const uint4 b1 = __ldg(reinterpret_cast<const uint4*>(r + cw - 4));
                return ((a0.x ^ b0.x) | (a0.y ^ b0.y) | (a0.z ^ b0.z) | (a0.w ^ b0.w) |
                        (a1.x ^ b1.x) | (a1.y ^ b1.y) | (a1.z ^ b1.z) | (a1.w ^ b1.w)) == 0u;
            };
            if (tab.reuse_src[s] != nullptr && probe(tab.reuse_src[s] + off_w)) {
                cand = true;
                refp = tab.reuse_src[s] + off_w;
                digp = digests + 8 * (tab.reuse_out[s] + c);
            }
            if (!cand && tab.ref_payload[s] != nullptr) {
                const uint64_t rcix = c % tab.ref_chunks[s];
                if (probe(tab.ref_payload[s] + rcix * cw)) {
                    cand = true;
                    refp = tab.ref_payload[s] + rcix * cw;
                    digp = tab.ref_digests[s] + 8 * rcix;
                }
            }
            if (!cand && tab.zero_ok &&
                ((a0.x | a0.y | a0.z | a0.w | a1.x | a1.y | a1.z | a1.w) == 0u)) {
                cand = true;
                digp = tab.zero_digest;
            }
        }
        unsigned cm = __ballot_sync(0xffffffffu, cand);
        while (cm) {
            const int j = __ffs(cm) - 1;
            cm &= cm - 1u;
            const uint64_t joff = __shfl_sync(0xffffffffu, off_w, j);
            const uint4* cj = reinterpret_cast<const uint4*>(tab.payload[s] + joff);
            const uint4* lj = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(d.local) + joff);
            const uint4* rj = reinterpret_cast<const uint4*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(refp), j));
            unsigned long long* mj = s_mask + (threadIdx.x & ~31u) + j;
            uint32_t diff = 0u;
            const uint32_t nq = cw / 4;
            for (uint32_t q0 = lane; q0 < nq; q0 += 32 * NAO_SCAN_U) {  // U x 3 loads in flight per lane
                uint4 a[NAO_SCAN_U], y[NAO_SCAN_U], r[NAO_SCAN_U];
#pragma unroll
                for (int u = 0; u < NAO_SCAN_U; u++) {
                    const uint32_t q = q0 + 32 * u;
                    a[u] = y[u] = r[u] = make_uint4(0u, 0u, 0u, 0u);
                    if (q < nq) {
                        a[u] = __ldg(cj + q);
                        y[u] = __ldg(lj + q);
                        if (rj) r[u] = __ldg(rj + q);
                    }
                }
#pragma unroll
                for (int u = 0; u < NAO_SCAN_U; u++) {
                    const uint32_t q = q0 + 32 * u;
                    diff |= (a[u].x ^ r[u].x) | (a[u].y ^ r[u].y) | (a[u].z ^ r[u].z) | (a[u].w ^ r[u].w);
                    const uint32_t av[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
                    const uint32_t yv[4] = {y[u].x, y[u].y, y[u].z, y[u].w};
#pragma unroll
                    for (int e = 0; e < 4; e++)
                        if (q < nq && word_needs_check_f(av[e], yv[e])) {
                            const uint32_t w = 4 * q + e;
                            atomicOr(mj + (w / MaskGeom<ALG>::BW) * kLeafThreads,
                                     1ull << (w % MaskGeom<ALG>::BW));
                        }
                }
            }
            const bool same = __all_sync(0xffffffffu, diff == 0u);
            if (lane == j && same) {
                uint32_t* dst = digests + 8 * (tab.out_index[s] + c);
#pragma unroll
                for (int k = 0; k < 8; k++) dst[k] = digp[k];
                reused = true;
            }
            __syncwarp();
        }
    }
    {  // chunks whose digest was copied (one atomic per warp)
        const unsigned rb = __ballot_sync(0xffffffffu, active && reused);
        if (lane == 0 && rb) atomicAdd(&g_reused_chunks, (unsigned long long)__popc(rb));
    }
    if (active && !reused) {
        uint32_t dg[8];
        if (check) {
            // (re)writes every mask entry of this chunk: stale bits of a failed
            // shortcut scan are overwritten
            CheckedWords<ALG> ld{tab.payload[s] + off_w,
                                 reinterpret_cast<const uint32_t*>(d.local) + off_w,
                                 s_mask + threadIdx.x};
            hash_tagged_words<ALG>(ld, nw, 0u, dg);
            ld.finish();
        } else {
            GlobalWords ld{tab.payload[s] + off_w};
            hash_tagged_words<ALG>(ld, nw, 0u, dg);
        }
        store_digest(digests + 8 * (tab.out_index[s] + c), dg);
    }
    if (!check) return;
    __syncwarp();
    // ---- warp-cooperative check of the flagged words: lanes push their
    // flagged element indices into the warp queue (one per lane per round),
    // 32 queued elements are processed with every lane busy
    LaneCheck lc;
    const float* claimed = reinterpret_cast<const float*>(tab.payload[s]);
    const uint64_t lane_base = c * cw;  // element index of this lane's word 0
    int qn = 0;                         // warp-uniform
    unsigned long long nflag = 0;
    // NAO_CC_PROBE >= 1: timing probe, flagged words are not processed (wrong verdicts)
    const uint32_t groups_proc = NAO_CC_PROBE >= 1 ? 0u : groups;
    for (uint32_t g = 0; g < groups_proc; g++) {
        unsigned long long m = s_mask[g * kLeafThreads + threadIdx.x];
        for (;;) {
            const bool has = m != 0ull;
            const unsigned b = __ballot_sync(0xffffffffu, has);
            if (b == 0u) break;
            if (has) {
                const int bit = __ffsll((long long)m) - 1;
                m &= m - 1ull;
                sm.q[w][qn + __popc(b & ((1u << lane) - 1u))] = lane_base + (uint64_t)BW * g + bit;
            }
            qn += __popc(b);
            nflag += has;
            if (qn >= 64) {  // two entries per lane: four loads in flight before the math
                __syncwarp();
                const Flagged f0 = load_flagged(d, claimed, sm.q[w][lane]);
                const Flagged f1 = load_flagged(d, claimed, sm.q[w][32 + lane]);
                process_flagged(d, f0, G, epsilon, sm, w, lc, 0xffffffffu);
                process_flagged(d, f1, G, epsilon, sm, w, lc, 0xffffffffu);
                __syncwarp();
                if (lane < qn - 64) sm.q[w][lane] = sm.q[w][64 + lane];
                __syncwarp();
                qn -= 64;
            }
        }
    }
    __syncwarp();
    for (int base = 0; base < qn; base += 32) {
        const unsigned act = __ballot_sync(0xffffffffu, base + lane < qn);
        if (base + lane < qn) {
            const Flagged f = load_flagged(d, claimed, sm.q[w][base + lane]);
            process_flagged(d, f, G, epsilon, sm, w, lc, act);
        }
    }
    __syncwarp();
    // ---- block reduction -> the tensor's accumulator
    const unsigned long long viol = warp_sum(lc.viol), border = warp_sum(lc.border),
                             nonfin = warp_sum(lc.nonfin), nf = warp_sum(nflag);
    double r = lc.best_inf ? INFINITY : (lc.best_num > 0.0 ? lc.best_num / lc.best_den : 0.0);
    r = warp_max(r);
    if (lane == 0) {
        atomicAdd(&sm.viol, viol);
        atomicAdd(&sm.border, border);
        atomicAdd(&sm.nonfin, nonfin);
        atomicAdd(&sm.nslow, nf);
        if (r > 0.0) atomicMax(&sm.maxr_bits, (unsigned long long)__double_as_longlong(r));
    }
    __syncthreads();
    CheckAccum* acc = accs + s;
    if (threadIdx.x <= G) {
        unsigned long long ha = 0, hr = 0;
        for (int ww = 0; ww < kLeafWarps; ww++) {
            ha += sm.wc[ww][0][threadIdx.x];
            hr += sm.wc[ww][1][threadIdx.x];
        }
        if (threadIdx.x == 0) {  // equal words: bucket 0 of both arrays
            const unsigned long long eq = cta_words - sm.nslow;
            ha += eq;
            hr += eq;
        }
        if (ha) atomicAdd(&acc->hist_abs[threadIdx.x], ha);
        if (hr) atomicAdd(&acc->hist_rel[threadIdx.x], hr);
        if (d.flags & NAO_CHECK_PARTIAL) {
            const int b = threadIdx.x;
            unsigned long long mx0 = sm.bmax[0][b], mn0 = sm.bmin_inv[0][b];
            unsigned long long mx1 = sm.bmax[1][b], mn1 = sm.bmin_inv[1][b];
            if (b == 0) {  // the equal words: key 0 in bucket 0 of both arrays
                if (cta_words > sm.nslow) { mn0 = ~0ull; mn1 = ~0ull; }
            }
            if (mx0) atomicMax(&acc->bmax[0][b], mx0);
            if (mn0) atomicMax(&acc->bmin_inv[0][b], mn0);
            if (mx1) atomicMax(&acc->bmax[1][b], mx1);
            if (mn1) atomicMax(&acc->bmin_inv[1][b], mn1);
        }
    }
    if (threadIdx.x == 0) {
        if (sm.viol) atomicAdd(&acc->n_viol, sm.viol);
        if (sm.border) atomicAdd(&acc->n_border, sm.border);
        if (sm.nonfin) atomicAdd(&acc->n_nonfinite, sm.nonfin);
        if (sm.maxr_bits) atomicMax(&acc->max_ratio_bits, sm.maxr_bits);
        __threadfence();
        const unsigned int nblk = (unsigned int)(tab.block_prefix[s + 1] - tab.block_prefix[s]);
        sm.is_last = atomicAdd(&acc->blocks_done, 1u) == nblk - 1;
    }
    __syncthreads();
    if (!sm.is_last) return;
    __threadfence();
    const VerdictSpec& v = *d.spec;
    const int64_t n = (int64_t)total_w;
    if (d.flags & NAO_CHECK_PARTIAL) {  // combinable shard record, no verdict here
        nao_check_partial* out = reinterpret_cast<nao_check_partial*>(d.result);
        const volatile CheckAccum* va = acc;
        if (threadIdx.x <= kMaxGrid) {
            const int b = threadIdx.x;
            out->hist_abs[b] = va->hist_abs[b];
            out->hist_rel[b] = va->hist_rel[b];
            out->max_abs[b] = __longlong_as_double((long long)va->bmax[0][b]);
            out->max_rel[b] = __longlong_as_double((long long)va->bmax[1][b]);
            const unsigned long long i0 = va->bmin_inv[0][b], i1 = va->bmin_inv[1][b];
            out->min_abs[b] = i0 ? __longlong_as_double((long long)~i0) : INFINITY;
            out->min_rel[b] = i1 ? __longlong_as_double((long long)~i1) : INFINITY;
        }
        if (threadIdx.x == 0) {
            out->n = (uint64_t)n;
            out->n_violations = va->n_viol;
            out->n_borderline = va->n_border;
            out->n_nonfinite = va->n_nonfinite;
            out->max_ratio = __longlong_as_double((long long)va->max_ratio_bits);
        }
        __syncthreads();
        unsigned long long* zp = reinterpret_cast<unsigned long long*>(acc);
        for (int i = threadIdx.x; i < (int)(sizeof(CheckAccum) / 8); i += blockDim.x) zp[i] = 0ull;
        return;
    }
    decide_targets(v, n, acc->hist_abs, acc->hist_rel, sm.vs, false);
    if (sm.vs.n_amb > 0) {
        settle_ambiguous(v, d.local, claimed, n, sm.vs);
        decide_targets(v, n, acc->hist_abs, acc->hist_rel, sm.vs, true);
    }
    if (threadIdx.x == 0) {
        nao_check_result* out = d.result;
        out->n = (uint64_t)n;
        out->n_violations = acc->n_viol;
        out->n_borderline = acc->n_border;
        out->n_nonfinite = acc->n_nonfinite;
        out->max_ratio = __longlong_as_double((long long)acc->max_ratio_bits);
        out->threshold_exceeded = sm.vs.exceeded;
        out->first_exceeded = sm.vs.exceeded ? sm.vs.first : -1;
        out->n_ambiguous = sm.vs.n_amb;
        out->reserved = 0;
    }
    __syncthreads();
    unsigned long long* z = reinterpret_cast<unsigned long long*>(acc);
    for (int i = threadIdx.x; i < (int)(sizeof(CheckAccum) / 8); i += blockDim.x) z[i] = 0ull;
}

// Persistent over virtual blocks (grid may be smaller than the block count, so
// the commit can share SMs with concurrently running forward kernels).
#ifndef NAO_LEAF_MINB
#define NAO_LEAF_MINB 4  // <= 128 registers: 4 CTAs (16 warps) per SM for the sponge
#endif
template <int ALG>
__global__ void __launch_bounds__(kLeafThreads, NAO_LEAF_MINB) k_chunk_leaves_check(
    const __grid_constant__ CCTable tab, uint32_t* __restrict__ digests,
    CheckAccum* __restrict__ accs) {
    __shared__ LeafCheckSmem sm;
    extern __shared__ unsigned long long s_mask[];  // [groups][kLeafThreads]
    const uint64_t nvb = tab.block_prefix[tab.n];
    for (uint64_t vb = blockIdx.x; vb < nvb; vb += gridDim.x) {
        leaf_check_block<ALG>(tab, digests, accs, sm, s_mask, vb);
        __syncthreads();
    }
}

template <int ALG>
__global__ void __launch_bounds__(64) k_header_leaves(const __grid_constant__ HeaderTable tab,
                                                      uint32_t* __restrict__ digests) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= tab.n) return;
    ByteMsg m{tab.bytes[s], tab.len[s], 0};
    uint32_t d[8];
    hash_bytes_generic<ALG>(m, d);
    store_digest(digests + 8 * tab.out_index[s], d);
}

// Generic leaves laid out contiguously in device memory (offsets in device memory).
template <int ALG>
__global__ void __launch_bounds__(64) k_packed_leaves(const uint8_t* __restrict__ data,
                                                      const int64_t* __restrict__ offsets,
                                                      int64_t n, uint32_t* __restrict__ digests) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    ByteMsg m{data + offsets[s], (uint64_t)(offsets[s + 1] - offsets[s]), 0};
    uint32_t d[8];
    hash_bytes_generic<ALG>(m, d);
    store_digest(digests + 8 * s, d);
}

template <int ALG>
__global__ void __launch_bounds__(kTreeThreads) k_tree_reduce(const __grid_constant__ TreeTable tab,
                                                              const uint32_t* __restrict__ in,
                                                              uint32_t* __restrict__ out) {
    __shared__ uint4 sm[2 * kTreeThreads][2];  // up to 512 digests
    const int s = find_seg(tab.group_prefix, tab.n, blockIdx.x);
    const uint64_t g = blockIdx.x - tab.group_prefix[s];
    const uint64_t group = 1ull << tab.lg;
    const uint64_t first = g * group;
    uint64_t m = (tab.n_in[s] - first < group ? tab.n_in[s] - first : group);  // live nodes in this group
    const uint32_t* src = in + 8 * (tab.in_index[s] + first);
    // level 0 -> smem
    for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint4* p = reinterpret_cast<const uint4*>(src + 8 * i);
        sm[i][0] = p[0];
        sm[i][1] = p[1];
    }
    __syncthreads();
    const int levels = tab.full_levels[s] ? tab.lg : 64;
    for (int l = 0; l < levels; l++) {
        if (!tab.full_levels[s] && m <= 1) break;
        const uint64_t mo = (m + 1) >> 1;
        uint32_t res[8];
        const uint64_t j = threadIdx.x;
        if (j < mo) {
            uint32_t L[8], R[8];
            uint4 a0 = sm[2 * j][0], a1 = sm[2 * j][1];
            uint64_t r = (2 * j + 1 < m) ? 2 * j + 1 : 2 * j;  // odd node pairs with itself
            uint4 b0 = sm[r][0], b1 = sm[r][1];
            L[0] = a0.x; L[1] = a0.y; L[2] = a0.z; L[3] = a0.w;
            L[4] = a1.x; L[5] = a1.y; L[6] = a1.z; L[7] = a1.w;
            R[0] = b0.x; R[1] = b0.y; R[2] = b0.z; R[3] = b0.w;
            R[4] = b1.x; R[5] = b1.y; R[6] = b1.z; R[7] = b1.w;
            hash_node<ALG>(L, R, res);
        }
        __syncthreads();
        if (j < mo) {
            sm[j][0] = make_uint4(res[0], res[1], res[2], res[3]);
            sm[j][1] = make_uint4(res[4], res[5], res[6], res[7]);
        }
        __syncthreads();
        m = mo;
    }
    if (threadIdx.x == 0) {
        uint4* p = reinterpret_cast<uint4*>(out + 8 * (tab.out_index[s] + g));
        p[0] = sm[0][0];
        p[1] = sm[0][1];
    }
}

// One tree level for many segments at once, one parent hash per thread (the
// large lower levels: every lane busy; k_tree_reduce takes over once the
// levels are small).  parent j of a segment = H(0x01 || in[2j] || in[2j+1]),
// an odd last node pairing with itself (commitments.py:119-127).
template <int ALG>
__global__ void __launch_bounds__(128) k_tree_level(const __grid_constant__ TreeTable tab,
                                                   const uint32_t* __restrict__ in,
                                                   uint32_t* __restrict__ out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= tab.group_prefix[tab.n]) return;
    const int s = find_seg(tab.group_prefix, tab.n, t);
    const uint64_t j = t - tab.group_prefix[s];
    const uint64_t a = 2 * j, b = (2 * j + 1 < tab.n_in[s]) ? 2 * j + 1 : 2 * j;
    const uint4* pa = reinterpret_cast<const uint4*>(in + 8 * (tab.in_index[s] + a));
    const uint4* pb = reinterpret_cast<const uint4*>(in + 8 * (tab.in_index[s] + b));
    const uint4 a0 = __ldg(pa), a1 = __ldg(pa + 1), b0 = __ldg(pb), b1 = __ldg(pb + 1);
    const uint32_t L[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const uint32_t R[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    uint32_t res[8];
    hash_node<ALG>(L, R, res);
    store_digest(out + 8 * (tab.out_index[s] + j), res);
}

// ----------------------------------------------------------------- host side

struct ZeroWords {  // an all-zero payload for the sponge
    __device__ __forceinline__ uint2 v2c(uint32_t, int) const { return make_uint2(0u, 0u); }
    __device__ __forceinline__ uint32_t wc(uint32_t, int) const { return 0u; }
    __device__ __forceinline__ void block_end(uint32_t) const {}
    __device__ __forceinline__ uint4 v4(uint32_t) const { return make_uint4(0u, 0u, 0u, 0u); }
    __device__ __forceinline__ uint2 v2(uint32_t) const { return make_uint2(0u, 0u); }
    __device__ __forceinline__ uint32_t w(uint32_t) const { return 0u; }
};

__global__ void k_zero_chunk_digest(uint32_t cw, uint32_t* out) {
    uint32_t d[8];
    hash_tagged_words<kKECCAK256>(ZeroWords{}, cw, 0u, d);
    for (int i = 0; i < 8; i++) out[i] = d[i];
}

// H(0x00 || zeros(4 cw)) with Keccak-256, cached per chunk size.  Computed on
// the device the first time a size is seen on a stream that is not capturing
// (the eager warm-up run); during a capture an uncached size disables the
// shortcut for that call (*ok = 0).
static int zero_chunk_digest(uint32_t cw, uint32_t out[8], int* ok, cudaStream_t st) {
    static std::mutex mu;
    static std::map<uint32_t, std::array<uint32_t, 8>> cache;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(cw);
        if (it != cache.end()) {
            memcpy(out, it->second.data(), 32);
            *ok = 1;
            return NAO_OK;
        }
    }
    *ok = 0;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    NAO_CHECK_CUDA(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone) return NAO_OK;
    uint32_t* dev = nullptr;
    NAO_CHECK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dev), 32, st));
    k_zero_chunk_digest<<<1, 1, 0, st>>>(cw, dev);
    NAO_CHECK_LAUNCH();
    std::array<uint32_t, 8> h{};
    NAO_CHECK_CUDA(cudaMemcpyAsync(h.data(), dev, 32, cudaMemcpyDeviceToHost, st));
    NAO_CHECK_CUDA(cudaFreeAsync(dev, st));
    NAO_CHECK_CUDA(cudaStreamSynchronize(st));
    std::lock_guard<std::mutex> lk(mu);
    cache[cw] = h;
    memcpy(out, h.data(), 32);
    *ok = 1;
    return NAO_OK;
}

static int launch_chunk_leaves(int alg, ChunkTable& tab, uint32_t* digests, cudaStream_t st) {
    uint64_t total = tab.chunk_prefix[tab.n];
    if (total == 0) return NAO_OK;
    const int threads = 128;
    uint64_t blocks = (total + threads - 1) / threads;
    if (alg == kSHA256) k_chunk_leaves<kSHA256><<<(unsigned)blocks, threads, 0, st>>>(tab, digests);
    else k_chunk_leaves<kKECCAK256><<<(unsigned)blocks, threads, 0, st>>>(tab, digests);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

static int launch_header_leaves(int alg, HeaderTable& tab, uint32_t* digests, cudaStream_t st) {
    if (tab.n == 0) return NAO_OK;
    int blocks = (tab.n + 63) / 64;
    if (alg == kSHA256) k_header_leaves<kSHA256><<<blocks, 64, 0, st>>>(tab, digests);
    else k_header_leaves<kKECCAK256><<<blocks, 64, 0, st>>>(tab, digests);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

// Reduce `nseg` level-0 digest ranges to one root each.  Level arrays
// ping-pong between two scratch buffers; roots land in roots_out[k].
// If levels_out != nullptr (single segment only) every level is stored
// consecutively there and lg is forced to 1.
static int reduce_trees(int alg, int nseg, const uint64_t* in_index, const uint64_t* n_leaves,
                        const uint32_t* level0, uint32_t* scratch_a, uint32_t* scratch_b,
                        uint32_t* roots_out, uint32_t* levels_out, cudaStream_t st) {
    std::vector<uint64_t> cur_n(n_leaves, n_leaves + nseg);
    std::vector<uint64_t> cur_idx(in_index, in_index + nseg);
    const uint32_t* cur = level0;
    uint32_t* bufs[2] = {scratch_a, scratch_b};
    int which = 0;
    const int lg = levels_out ? 1 : 9;
    uint64_t level_store_off = 0;
    if (levels_out) {
        NAO_CHECK_CUDA(cudaMemcpyAsync(levels_out, level0 + 8 * in_index[0], 32 * n_leaves[0],
                                       cudaMemcpyDeviceToDevice, st));
        level_store_off = n_leaves[0];
    }
    // segments with a single leaf: root == leaf digest
    for (int k = 0; k < nseg; k++)
        if (cur_n[k] == 1)
            NAO_CHECK_CUDA(cudaMemcpyAsync(roots_out + 8 * k, level0 + 8 * in_index[k], 32,
                                           cudaMemcpyDeviceToDevice, st));
    for (int iter = 0; iter < 64; iter++) {
        std::vector<int> live;
        uint64_t live_nodes = 0;
        for (int k = 0; k < nseg; k++)
            if (cur_n[k] > 1) { live.push_back(k); live_nodes += cur_n[k]; }
        if (live.empty()) break;
        uint32_t* dst = levels_out ? levels_out : bufs[which];
        uint64_t dst_base = levels_out ? level_store_off : 0;
        std::vector<uint64_t> next_n(nseg), next_idx(nseg);
        // big levels: one flat launch per level (all lanes busy)
        const int lg_it = (live_nodes >= kFlatLevelMin || levels_out) ? 1 : lg;
        for (size_t b0 = 0; b0 < live.size(); b0 += kMaxSegs) {
            TreeTable tab;
            memset(&tab, 0, sizeof tab);
            tab.lg = lg;
            int cnt = 0;
            tab.group_prefix[0] = 0;
            tab.lg = lg_it;
            for (size_t q = b0; q < live.size() && cnt < kMaxSegs; q++, cnt++) {
                int k = live[q];
                uint64_t groups = (cur_n[k] + (1ull << lg_it) - 1) >> lg_it;
                tab.full_levels[cnt] = groups > 1 ? 1 : 0;
                tab.in_index[cnt] = cur_idx[k];
                tab.n_in[cnt] = cur_n[k];
                tab.out_index[cnt] = dst_base;
                next_n[k] = groups;
                next_idx[k] = dst_base;
                dst_base += groups;
                tab.group_prefix[cnt + 1] = tab.group_prefix[cnt] + groups;
            }
            tab.n = cnt;
            uint64_t blocks = tab.group_prefix[cnt];
            if (lg_it == 1 && !levels_out) {  // flat level: thread per parent
                const uint64_t fb = (blocks + 127) / 128;
                if (alg == kSHA256)
                    k_tree_level<kSHA256><<<(unsigned)fb, 128, 0, st>>>(tab, cur, dst);
                else
                    k_tree_level<kKECCAK256><<<(unsigned)fb, 128, 0, st>>>(tab, cur, dst);
            } else if (alg == kSHA256)
                k_tree_reduce<kSHA256><<<(unsigned)blocks, kTreeThreads, 0, st>>>(tab, cur, dst);
            else
                k_tree_reduce<kKECCAK256><<<(unsigned)blocks, kTreeThreads, 0, st>>>(tab, cur, dst);
            NAO_CHECK_LAUNCH();
        }
        for (int k : live) {
            cur_n[k] = next_n[k];
            cur_idx[k] = next_idx[k];
            if (cur_n[k] == 1)
                NAO_CHECK_CUDA(cudaMemcpyAsync(roots_out + 8 * k, dst + 8 * cur_idx[k], 32,
                                               cudaMemcpyDeviceToDevice, st));
        }
        if (levels_out) level_store_off = dst_base;
        cur = dst;
        which ^= 1;
    }
    return NAO_OK;
}

static uint64_t seg_chunks(uint64_t nbytes, uint64_t chunk) { return (nbytes + chunk - 1) / chunk; }

}  // namespace nao

using namespace nao;

extern "C" {

size_t nao_merkle_commit_workspace(int64_t n_tensors, const uint64_t* payload_bytes,
                                   uint64_t chunk_bytes) {
    if (n_tensors <= 0 || chunk_bytes == 0) return 0;
    uint64_t leaves = 0;
    for (int64_t i = 0; i < n_tensors; i++) leaves += 1 + seg_chunks(payload_bytes[i], chunk_bytes);
    // level-0 digests + two ping-pong level buffers (each <= leaves/2 + 2n)
    uint64_t lvl = leaves / 2 + 2 * (uint64_t)n_tensors + 16;  // flat first levels: n/2
    return (size_t)(32 * (leaves + 2 * lvl) + 3 * 256);
}

}  // extern "C"

namespace nao {

static int commit_tensors_impl(int64_t n_tensors, const void* const* payloads,
                               const uint64_t* payload_bytes, const uint8_t* const* headers,
                               const uint32_t* header_lens, uint64_t chunk_bytes, int hash_alg,
                               const nao_check_desc* checks, const nao_chunk_reuse* reuse,
                               uint8_t* roots_out, uint8_t* leaf_digests_out, void* accum,
                               void* workspace, size_t workspace_bytes, cudaStream_t st) {
    NAO_REQUIRE(n_tensors > 0, "n_tensors must be positive");
    NAO_REQUIRE(hash_alg == NAO_HASH_SHA256 || hash_alg == NAO_HASH_KECCAK256, "bad hash_alg %d",
                hash_alg);
    NAO_REQUIRE(chunk_bytes >= 64 && chunk_bytes % 64 == 0 && chunk_bytes <= (1ull << 30),
                "chunk_bytes must be a positive multiple of 64 (got %llu)",
                (unsigned long long)chunk_bytes);
    NAO_REQUIRE(roots_out != nullptr, "roots_out is null");
    std::vector<uint64_t> in_index(n_tensors), n_leaves(n_tensors);
    uint64_t leaves = 0;
    for (int64_t i = 0; i < n_tensors; i++) {
        NAO_REQUIRE(payload_bytes[i] % 4 == 0, "payload %lld: byte size not a multiple of 4",
                    (long long)i);
        NAO_REQUIRE(payload_bytes[i] == 0 ||
                        (reinterpret_cast<uintptr_t>(payloads[i]) % 16 == 0),
                    "payload %lld: not 16-byte aligned", (long long)i);
        NAO_REQUIRE(headers[i] != nullptr && header_lens[i] > 0 && header_lens[i] <= kMaxHeader,
                    "header %lld missing or longer than %d bytes", (long long)i, kMaxHeader);
        if (checks && checks[i].local) {
            const nao_check_desc& c = checks[i];
            NAO_REQUIRE(reinterpret_cast<uintptr_t>(c.local) % 16 == 0,
                        "check %lld: local must be 16-byte aligned", (long long)i);
            NAO_REQUIRE(c.eps_kind >= NAO_EPS_TENSOR_F32 && c.eps_kind <= NAO_EPS_ZERO,
                        "check %lld: bad eps_kind %d", (long long)i, c.eps_kind);
            NAO_REQUIRE(c.eps_kind == NAO_EPS_SCALED_LOCAL || c.eps_kind == NAO_EPS_ZERO ||
                            c.eps != nullptr, "check %lld: eps tensor missing", (long long)i);
            NAO_REQUIRE(c.spec != nullptr && c.result != nullptr,
                        "check %lld: spec/result missing", (long long)i);
            NAO_REQUIRE(accum != nullptr, "checks need the accumulator scratch");
        }
        in_index[i] = leaves;
        n_leaves[i] = 1 + seg_chunks(payload_bytes[i], chunk_bytes);
        leaves += n_leaves[i];
    }
    // chunk-digest reuse: phase = 1 + the source's phase (sources hash first)
    std::vector<int> phase(n_tensors, 0);
    int n_phases = 1;
    for (int64_t i = 0; reuse && i < n_tensors; i++) {
        const nao_chunk_reuse& r = reuse[i];
        NAO_REQUIRE(r.row_chunks <= 1 || (r.row_chunks <= (uint32_t)kLeafThreads &&
                                           kLeafThreads % r.row_chunks == 0),
                    "reuse %lld: row_chunks must divide %d", (long long)i, kLeafThreads);
        if (r.ref_payload != nullptr)
            NAO_REQUIRE(r.ref_digests != nullptr && r.ref_bytes > 0 &&
                            r.ref_bytes % chunk_bytes == 0 && payload_bytes[i] % r.ref_bytes == 0 &&
                            reinterpret_cast<uintptr_t>(r.ref_payload) % 16 == 0,
                        "reuse %lld: the reference must be whole chunks dividing the payload",
                        (long long)i);
        if (r.src < 0 || payload_bytes[i] == 0) continue;
        NAO_REQUIRE(r.src < i, "reuse %lld: source %lld must come earlier", (long long)i,
                    (long long)r.src);
        NAO_REQUIRE(checks && checks[i].local, "reuse %lld needs the fused check", (long long)i);
        NAO_REQUIRE(r.mode == NAO_REUSE_LOCAL_COPY || r.mode == NAO_REUSE_SAME_OFFSET,
                    "reuse %lld: bad mode %d", (long long)i, r.mode);
        const uint64_t sb = payload_bytes[r.src];
        if (r.mode == NAO_REUSE_SAME_OFFSET) {
            NAO_REQUIRE(payload_bytes[i] == sb,
                        "reuse %lld: same-offset reuse needs the source's size", (long long)i);
            phase[i] = phase[r.src] + 1;
            n_phases = std::max(n_phases, phase[i] + 1);
            continue;
        }
        NAO_REQUIRE(r.repeats >= 1 && r.block_chunks >= 1, "reuse %lld: bad block", (long long)i);
        if (r.repeats == 1)
            NAO_REQUIRE(payload_bytes[i] == sb && r.block_chunks == seg_chunks(sb, chunk_bytes),
                        "reuse %lld: a reshape must have the source's bytes", (long long)i);
        else
            NAO_REQUIRE(sb % (r.block_chunks * chunk_bytes) == 0 && payload_bytes[i] == sb * r.repeats,
                        "reuse %lld: repeated blocks must be whole chunks", (long long)i);
        phase[i] = phase[r.src] + 1;
        n_phases = std::max(n_phases, phase[i] + 1);
    }
    Workspace ws(workspace, workspace_bytes);
    uint32_t* lvl0 = leaf_digests_out ? reinterpret_cast<uint32_t*>(leaf_digests_out)
                                      : ws.take<uint32_t>(8 * leaves);
    uint64_t lvl = leaves / 2 + 2 * (uint64_t)n_tensors + 16;  // flat first levels: n/2
    uint32_t* sa = ws.take<uint32_t>(8 * lvl);
    uint32_t* sb = ws.take<uint32_t>(8 * lvl);
    NAO_REQUIRE(lvl0 && sa && sb, "workspace too small (%zu bytes)", workspace_bytes);
    // header leaves: host bytes travel as kernel parameters (<= 136 B each)
    for (int64_t b0 = 0; b0 < n_tensors; b0 += kMaxSegs) {
        static thread_local HeaderTable ht;
        ht.n = 0;
        for (int64_t i = b0; i < n_tensors && ht.n < kMaxSegs; i++) {
            memcpy(ht.bytes[ht.n], headers[i], header_lens[i]);
            ht.len[ht.n] = header_lens[i];
            ht.out_index[ht.n] = in_index[i];
            ht.n++;
        }
        int rc = launch_header_leaves(hash_alg, ht, lvl0, st);
        if (rc) return rc;
    }
    bool any_check = false;
    for (int64_t i = 0; checks && i < n_tensors; i++) any_check |= checks[i].local != nullptr;
    NAO_REQUIRE(!any_check || chunk_bytes / 4 <= (uint64_t)kMaxFusedChunkWords,
                "the fused check supports chunk_bytes <= %d", 4 * kMaxFusedChunkWords);
    // digest of the all-zero chunk (Keccak-256 fused check only), computed once
    // per chunk size on the device outside graph capture
    uint32_t zero_digest[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int zero_ok = 0;
    if (any_check && hash_alg == kKECCAK256) {
        int rc = zero_chunk_digest((uint32_t)(chunk_bytes / 4), zero_digest, &zero_ok, st);
        if (rc) return rc;
    }
    std::vector<int64_t> order;  // tensors by phase, canonical order within a phase
    std::vector<int64_t> phase_end;
    for (int ph = 0; ph < n_phases; ph++) {
        for (int64_t i = 0; i < n_tensors; i++)
            if (phase[i] == ph) order.push_back(i);
        phase_end.push_back((int64_t)order.size());
    }
    for (int64_t b0 = 0, ph = 0; b0 < n_tensors;) {
        while (b0 >= phase_end[ph]) ph++;
        const int64_t b1 = std::min<int64_t>(b0 + kMaxSegs, phase_end[ph]);
        if (!any_check) {
            ChunkTable ct;
            memset(&ct, 0, sizeof ct);
            ct.chunk_words = (uint32_t)(chunk_bytes / 4);
            int cnt = 0;
            ct.chunk_prefix[0] = 0;
            for (int64_t k = b0; k < b1; k++, cnt++) {
                const int64_t i = order[k];
                ct.payload[cnt] = static_cast<const uint32_t*>(payloads[i]);
                ct.nbytes[cnt] = payload_bytes[i];
                ct.out_index[cnt] = in_index[i] + 1;
                ct.chunk_prefix[cnt + 1] =
                    ct.chunk_prefix[cnt] + seg_chunks(payload_bytes[i], chunk_bytes);
            }
            ct.n = cnt;
            b0 = b1;
            int rc = launch_chunk_leaves(hash_alg, ct, lvl0, st);
            if (rc) return rc;
            continue;
        }
        static thread_local CCTable ct;
        memset(&ct, 0, sizeof ct);
        ct.chunk_words = (uint32_t)(chunk_bytes / 4);
        int cnt = 0;
        ct.block_prefix[0] = 0;
        for (int64_t k = b0; k < b1; k++, cnt++) {
            const int64_t i = order[k];
            ct.payload[cnt] = static_cast<const uint32_t*>(payloads[i]);
            ct.nbytes[cnt] = payload_bytes[i];
            ct.out_index[cnt] = in_index[i] + 1;
            // row mapping only where rows are whole chunks (else identity)
            uint32_t rcs = reuse && reuse[i].row_chunks > 1 ? reuse[i].row_chunks : 0u;
            if (rcs && payload_bytes[i] % (rcs * chunk_bytes) != 0) rcs = 0u;
            const int64_t nch = (int64_t)seg_chunks(payload_bytes[i], chunk_bytes);
            ct.block_prefix[cnt + 1] = ct.block_prefix[cnt] +
                (rcs ? ceil_div(nch / (int64_t)rcs, kLeafThreads) * rcs : ceil_div(nch, kLeafThreads));
            if (checks && payload_bytes[i] > 0) memcpy(&ct.chk[cnt], &checks[i], sizeof(CheckDesc));
            ct.reuse_out[cnt] = ~0ull;
            ct.reuse_src[cnt] = nullptr;
            ct.row_chunks[cnt] = rcs;
            ct.ref_payload[cnt] = nullptr;
            ct.ref_digests[cnt] = nullptr;
            ct.ref_chunks[cnt] = 1;
            if (reuse && reuse[i].ref_payload != nullptr && payload_bytes[i] > 0) {
                ct.ref_payload[cnt] = static_cast<const uint32_t*>(reuse[i].ref_payload);
                ct.ref_digests[cnt] = static_cast<const uint32_t*>(reuse[i].ref_digests);
                ct.ref_chunks[cnt] = reuse[i].ref_bytes / chunk_bytes;
            }
            if (phase[i] > 0) {
                const nao_chunk_reuse& r = reuse[i];
                ct.reuse_out[cnt] = in_index[r.src] + 1;
                ct.reuse_block[cnt] = r.block_chunks;
                ct.reuse_span[cnt] = r.block_chunks * r.repeats;
                if (r.mode == NAO_REUSE_SAME_OFFSET)
                    ct.reuse_src[cnt] = static_cast<const uint32_t*>(payloads[r.src]);
            }
        }
        ct.n = cnt;
        ct.zero_ok = zero_ok;
        memcpy(ct.zero_digest, zero_digest, sizeof zero_digest);
        b0 = b1;
        uint64_t blocks = ct.block_prefix[cnt];
        if (blocks == 0) continue;
        static const uint64_t max_ctas = [] {
            const char* e = getenv("NAO_COMMIT_CTAS");
            return (uint64_t)(e ? atoll(e) : 0);
        }();
        if (max_ctas && blocks > max_ctas) blocks = max_ctas;
        CheckAccum* accs = static_cast<CheckAccum*>(accum);
        const uint32_t mgroups = hash_alg == kKECCAK256 ? ct.chunk_words / MaskGeom<kKECCAK256>::BW + 1
                                                        : (ct.chunk_words + 63) / 64;
        const size_t dsm = (size_t)mgroups * kLeafThreads * 8;
        static const int carve = [] {  // experiment knob: shared-memory carveout (%)
            const char* e = getenv("NAO_COMMIT_CARVEOUT");
            return e ? atoi(e) : -1;
        }();
        static bool carve_set = false;
        if (carve >= 0 && !carve_set) {
            NAO_CHECK_CUDA(cudaFuncSetAttribute(k_chunk_leaves_check<kSHA256>,
                                                cudaFuncAttributePreferredSharedMemoryCarveout, carve));
            NAO_CHECK_CUDA(cudaFuncSetAttribute(k_chunk_leaves_check<kKECCAK256>,
                                                cudaFuncAttributePreferredSharedMemoryCarveout, carve));
            carve_set = true;
        }
        if (hash_alg == kSHA256) {
            NAO_CHECK_CUDA(cudaFuncSetAttribute(k_chunk_leaves_check<kSHA256>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
            k_chunk_leaves_check<kSHA256><<<(unsigned)blocks, kLeafThreads, dsm, st>>>(ct, lvl0,
                                                                                     accs);
        } else {
            NAO_CHECK_CUDA(cudaFuncSetAttribute(k_chunk_leaves_check<kKECCAK256>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
            k_chunk_leaves_check<kKECCAK256><<<(unsigned)blocks, kLeafThreads, dsm, st>>>(
                ct, lvl0, accs);
        }
        NAO_CHECK_LAUNCH();
    }
    return reduce_trees(hash_alg, (int)n_tensors, in_index.data(), n_leaves.data(), lvl0, sa, sb,
                        reinterpret_cast<uint32_t*>(roots_out), nullptr, st);
}

}  // namespace nao

extern "C" {

int nao_merkle_commit_tensors(int64_t n_tensors, const void* const* payloads,
                              const uint64_t* payload_bytes, const uint8_t* const* headers,
                              const uint32_t* header_lens, uint64_t chunk_bytes, int hash_alg,
                              uint8_t* roots_out, uint8_t* leaf_digests_out, void* workspace,
                              size_t workspace_bytes, void* stream) {
    return commit_tensors_impl(n_tensors, payloads, payload_bytes, headers, header_lens,
                               chunk_bytes, hash_alg, nullptr, nullptr, roots_out, leaf_digests_out,
                               nullptr, workspace, workspace_bytes,
                               static_cast<cudaStream_t>(stream));
}

size_t nao_commit_check_accum_bytes(void) { return sizeof(CheckAccum) * kMaxSegs; }

int nao_commit_stats(uint64_t* reused_chunks, int reset) {
    NAO_REQUIRE(reused_chunks != nullptr, "reused_chunks is null");
    unsigned long long v = 0;
    NAO_CHECK_CUDA(cudaDeviceSynchronize());
    NAO_CHECK_CUDA(cudaMemcpyFromSymbol(&v, nao::g_reused_chunks, sizeof v));
    *reused_chunks = v;
    if (reset) {
        const unsigned long long z = 0;
        NAO_CHECK_CUDA(cudaMemcpyToSymbol(nao::g_reused_chunks, &z, sizeof z));
    }
    return NAO_OK;
}

int nao_commit_check_tensors(int64_t n_tensors, const void* const* payloads,
                             const uint64_t* payload_bytes, const uint8_t* const* headers,
                             const uint32_t* header_lens, uint64_t chunk_bytes, int hash_alg,
                             const nao_check_desc* checks, const nao_chunk_reuse* reuse,
                             uint8_t* roots_out, void* accum, void* workspace,
                             size_t workspace_bytes, void* stream) {
    return commit_tensors_impl(n_tensors, payloads, payload_bytes, headers, header_lens,
                               chunk_bytes, hash_alg, checks, reuse, roots_out, nullptr, accum,
                               workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

int nao_merkle_hash_leaves(const uint8_t* data, const int64_t* offsets, int64_t n_leaves,
                           int hash_alg, uint8_t* digests_out, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    NAO_REQUIRE(n_leaves > 0, "n_leaves must be positive");
    NAO_REQUIRE(hash_alg == NAO_HASH_SHA256 || hash_alg == NAO_HASH_KECCAK256, "bad hash_alg");
    int64_t blocks = (n_leaves + 63) / 64;
    if (hash_alg == kSHA256)
        k_packed_leaves<kSHA256><<<(unsigned)blocks, 64, 0, st>>>(
            data, offsets, n_leaves, reinterpret_cast<uint32_t*>(digests_out));
    else
        k_packed_leaves<kKECCAK256><<<(unsigned)blocks, 64, 0, st>>>(
            data, offsets, n_leaves, reinterpret_cast<uint32_t*>(digests_out));
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

size_t nao_merkle_root_workspace(int64_t n_leaves) {
    if (n_leaves <= 0) return 0;
    return (size_t)(2 * 32 * ((uint64_t)n_leaves / 2 + 16) + 512);
}

int nao_merkle_root_of(const uint8_t* leaf_digests, int64_t n_leaves, int hash_alg,
                       uint8_t* root_out, uint8_t* levels_out, void* workspace,
                       size_t workspace_bytes, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    NAO_REQUIRE(n_leaves > 0, "merkle tree requires at least one leaf");
    NAO_REQUIRE(hash_alg == NAO_HASH_SHA256 || hash_alg == NAO_HASH_KECCAK256, "bad hash_alg");
    Workspace ws(workspace, workspace_bytes);
    uint64_t lvl = (uint64_t)n_leaves / 2 + 16;
    uint32_t* sa = ws.take<uint32_t>(8 * lvl);
    uint32_t* sb = ws.take<uint32_t>(8 * lvl);
    if (levels_out == nullptr) NAO_REQUIRE(sa && sb, "workspace too small");
    uint64_t idx = 0, n = (uint64_t)n_leaves;
    return reduce_trees(hash_alg, 1, &idx, &n, reinterpret_cast<const uint32_t*>(leaf_digests), sa,
                        sb, reinterpret_cast<uint32_t*>(root_out),
                        reinterpret_cast<uint32_t*>(levels_out), st);
}

}  // extern "C"
