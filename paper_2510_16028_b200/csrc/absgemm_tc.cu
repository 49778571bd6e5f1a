// Abs-GEMM bound on the 5th-gen tensor cores (north_star (1), tcgen05 path).
//
//   eps[b,m,n] >= c * sum_k |A[b,m,k]| |B[b,k,n]|    (bounds.py:100-111)
//
// 3xTF32 split with outward rounding.  For a = |x| (x FP32):
//   hi = a truncated to TF32 (<= a),   lo = (a - hi) rounded UP to TF32,
// so a <= hi + lo < a (1 + 2^-20).  Products use hi*hi + hi*lo + lo*hi; the
// dropped lo*lo <= 1.002 * 2^-20 a b is restored by the factor
// 1/(1 - 1.002*2^-20).  Tensor-core accumulation of non-negative terms is
// modelled as losing at most kMmaRel = 3*2^-23 of the running sum per MMA
// instruction (products exact, aligned sum truncated), so:
//   * acc0 (hi*hi) lives in TMEM for only KCHUNK = 128 k (16 MMAs), then the
//     epilogue warps drain it into FP64 registers (double-buffered TMEM, the
//     MMA warp never waits) and the chunk sum is scaled by 1/(1 - 16 kMmaRel);
//   * acc1 (hi*lo + lo*hi, <= 2^-9 of acc0) accumulates over all of K and is
//     scaled by 1/(1 - J1 kMmaRel); its relative weight keeps that inside 2^-9.
// Worst-case over-estimate ~6.7e-6 < rtol 1e-5 (exact data, exact TC sums).
// Subnormal split parts are lifted to FLT_MIN and an absolute floor
// K*2^-120*c covers any flush-to-zero of products, so the result stays >= the
// exact bound.  Chunk length: 64 k made the FP64 drain (F2F + DADD, stall_math)
// pace the kernel (148 TFLOP/s algorithmic at 2048x4096x12288); 128 k -> 172,
// within 3 % of the no-epilogue probe (NAO_TC_EPI=9), which is L2->SM feed bound.
//
// Kernel anatomy (one CTA per 128x128 output tile, 384 threads):
//   warp 0      TMA producer: A_hi, A_lo, B_hi, B_lo tiles (128 x 16 fp32,
//               SWIZZLE_64B) into a 6-stage smem ring (32 KB / stage)
//   warp 1      single-thread tcgen05.mma.kind::tf32 issuer (6 MMAs / stage)
//   warp 2      TMEM allocator (512 columns: acc0 x2, acc1)
//   warps 4-11  epilogue: tcgen05.ld -> FP64 accumulate -> eps store
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace nao {
namespace tc {

#ifndef NAO_TC_BK
#define NAO_TC_BK 16
#endif
// BK = 16: 64 B rows (SWIZZLE_64B), 32 KB stages, 6 in flight;  BK = 32: 128 B
// rows (SWIZZLE_128B), 64 KB stages, 3 in flight.  Same bytes in flight.
constexpr int BM = 128, BN = 128, BK = NAO_TC_BK;
#ifndef NAO_TC_STAGES
#define NAO_TC_STAGES (NAO_TC_BK == 16 ? 6 : 3)
#endif
constexpr int STAGES = NAO_TC_STAGES;
#ifndef NAO_TC_KCHUNK
#define NAO_TC_KCHUNK 128
#endif
constexpr int KCHUNK = NAO_TC_KCHUNK;  // k per TMEM acc0 chunk (drained to the epilogue)
constexpr int KCHUNK_KB = KCHUNK / BK;  // k-blocks per chunk
constexpr int TILE_BYTES = BM * BK * 4;     // 16 KB (BM == BN)
constexpr int STAGE_BYTES = 4 * TILE_BYTES;  // A_hi, A_lo, B_hi, B_lo
constexpr int NUM_THREADS = 384;
constexpr uint32_t TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct TcArgs {
    int64_t M, N, K;
    int nkb;
    int a_batched, b_batched;
    void* C;
    const float* Y;
    int64_t ldc, sC;
    int out_f64;
    double scale0, scale1, abs_floor, u;
    // FP32 images rounded up (short-K epilogue, all-FP32 with round-up arithmetic)
    float scale0f, scale1f, abs_floorf, uf;
    // FP16 format only: power-of-two operand scales, x = 2^e * (hi + 2^-10 lo)
    const int32_t* a_exp;   // [batch_a, M]
    const int32_t* b_exp;   // [batch_b, N]
    const int32_t* a_tiny;  // [batch_a, M] parts below the normal half range
    const int32_t* b_tiny;
    double fix_thr;         // flag when e_scaled <= fix_thr * (tiny_a + tiny_b)
    float fix_thrf;
    unsigned long long* fix_count;  // flagged outputs (exact FP64 recompute)
    unsigned long long* fix_list;
    unsigned long long fix_cap;
};

// Record an output element for the exact FP64 fix-up pass.
__device__ __forceinline__ void flag_fix(const TcArgs& g, int bz, int64_t m, int64_t n) {
    const unsigned long long i = atomicAdd(g.fix_count, 1ull);
    if (i < g.fix_cap)
        g.fix_list[i] = ((unsigned long long)bz * (unsigned long long)g.M + (unsigned long long)m) *
                            (unsigned long long)g.N + (unsigned long long)n;
}

enum : int { kFmtTF32 = 0, kFmtF16 = 1 };

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// One lane of a converged warp (the lowest): the MMA issuer loops run on the
// whole warp so descriptors / TMEM addresses stay in uniform registers, and
// only the tcgen05.mma / commit instructions are issued by the elected lane
// (an `if (lane == 0)` issuer costs ~20 R2UR/ELECT instructions per MMA).
__device__ __forceinline__ bool elect_one() {
    uint32_t p = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                 : "=r"(p));
    return p != 0;
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// K-major swizzled smem operand descriptor: rows of BK*4 bytes, 8-row groups
// 8*BK*4 bytes apart (SWIZZLE_128B for 128 B rows, SWIZZLE_64B for 64 B rows)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;                        // LBO (unused for swizzled K-major)
    d |= (uint64_t)((8u * BK * 4u) >> 4) << 32;     // SBO
    d |= (uint64_t)1u << 46;                        // descriptor version (sm_100)
    d |= (uint64_t)(BK == 32 ? 2u : 4u) << 61;      // SWIZZLE_128B / SWIZZLE_64B
    return d;
}
// kind::tf32, D=F32, A=B=TF32, both K-major, N=BN, M=BM
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

// kind::f16, D=F32, A=B=F16, both K-major, N=BN, M=BM (64-byte rows = 32 halves:
// the same smem tile geometry and 32-byte K-steps as the TF32 tiles)
constexpr uint32_t kIdescF16 = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                               ((uint32_t)(BM >> 4) << 24);

// elements per 64-byte k-block of a format
template <int FMT>
struct FmtK { static constexpr int kb = FMT == 1 ? 32 : BK; };

template <int FMT>
__device__ __forceinline__ void umma_fmt(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
    if constexpr (FMT == kFmtF16) umma_f16(d, a, b, kIdescF16, acc);
    else umma_tf32(d, a, b, kIdesc, acc);
}

// 2^(ea + eb) as an exact FP64 power of two (|ea + eb| < 1000): a b = a_s b_s 2^(ea+eb)
__device__ __forceinline__ double pow2_sum(int ea, int eb) {
    return __hiloint2double((1023 + ea + eb) << 20, 0);
}
__device__ __forceinline__ float pow2f(int t) { return __int_as_float((127 + t) << 23); }  // |t|<=126
// e * 2^-t in FP32, rounded toward +inf (two steps keep 2^-t1 / 2^-t2 normal)
__device__ __forceinline__ float mul_pow2_ru(float e, int t) {
    const int t1 = t > 126 ? 126 : (t < -127 ? -127 : t);
    int t2 = t - t1;
    t2 = t2 > 126 ? 126 : (t2 < -127 ? -127 : t2);
    e = __fmul_ru(e, __int_as_float((127 - t1) << 23));
    return t2 ? __fmul_ru(e, __int_as_float((127 - t2) << 23)) : e;
}

#define TMEM_LD_X32(taddr, v)                                                                     \
    asm volatile(                                                                                 \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"  \
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"        \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),     \
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),              \
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),           \
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),           \
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),           \
          "=r"(v[31])                                                                             \
        : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}


// Per-thread FP64 accumulation of the TMEM chunk sums of acc0 (64 columns).
// NAO_TC_EPI 9 is a timing probe that skips the accumulation (wrong results):
// it measured the epilogue at ~16 % of the kernel with 64-k chunks, ~2 % with
// 128-k chunks.  (An FP32 TwoSum accumulator was measured slower than F2F+DADD.)
#ifndef NAO_TC_EPI
#define NAO_TC_EPI 0
#endif
struct EpiAcc {
    double a[64];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < 64; i++) a[i] = 0.0;
    }
    __device__ __forceinline__ void add(int i, float x) {
#if NAO_TC_EPI == 9
        a[i] = (double)x;
#else
        a[i] = __dadd_rn(a[i], (double)x);
#endif
    }
    __device__ __forceinline__ double get(int i) const { return a[i]; }
};


// Final epilogue of one 128x128 tile, per epilogue warp (32 rows = its TMEM lane
// quarter, 64 columns = its half): e = scale0*acc0sum + scale1*acc1 + floor is
// staged row-per-lane in smem (the drained stage ring; row stride 65 doubles),
// then written back row by row with lanes on consecutive columns, so the eps
// stores and the y reads of the linear u|y| term are coalesced 128 B segments
// (lane = row direct stores were ~8x sector-amplified: 32 rows per instruction).
__device__ __noinline__ void long_flag(const TcArgs& g, double e, int i, int tbh, int ta, int bz,
                                       int64_t mrow, int64_t n) {
    const int nt = ta + __shfl_sync(0xffffffffu, tbh, i);
    if (nt > 0 && n < g.N && mrow < g.M && e <= g.fix_thr * (double)nt) flag_fix(g, bz, mrow, n);
}

template <int FMT>
__device__ __forceinline__ void tile_epilogue(const TcArgs& g, const EpiAcc& acc, uint32_t col1,
                                              double* stg, int lane, int quarter, int half,
                                              int64_t m0, int64_t n0, int bz) {
    const int64_t mrow = m0 + quarter * 32 + lane;
    int ea = 0, ta = 0, eb[2] = {0, 0}, tb[2] = {0, 0};
    bool tiny_tile = false;
    double flag_lim = -1.0;
    if constexpr (FMT == kFmtF16) {
        const int64_t ao = (g.a_batched ? (int64_t)bz * g.M : 0) + mrow;
        if (mrow < g.M) { ea = __ldg(g.a_exp + ao); ta = __ldg(g.a_tiny + ao); }
        const int64_t bo = g.b_batched ? (int64_t)bz * g.N : 0;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int64_t n = n0 + half * 64 + 32 * h + lane;
            if (n < g.N) { eb[h] = __ldg(g.b_exp + bo + n); tb[h] = __ldg(g.b_tiny + bo + n); }
        }
        tiny_tile = __any_sync(0xffffffffu, (ta | tb[0] | tb[1]) != 0);
        int tmax = tb[0] > tb[1] ? tb[0] : tb[1];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        flag_lim = g.fix_thr * (double)(ta + tmax);
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {
        uint32_t v[32];
        TMEM_LD_X32(col1 + 32 * h, v);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; i++) {
            double e = __dadd_rn(__dmul_rn(g.scale0, acc.get(32 * h + i)),
                                 __dmul_rn(g.scale1, (double)__uint_as_float(v[i])));
            if constexpr (FMT == kFmtF16) {
                if (tiny_tile && __any_sync(0xffffffffu, e <= flag_lim))
                    long_flag(g, e, i, tb[h], ta, bz, mrow, n0 + half * 64 + 32 * h + i);
                e = __dmul_rn(e, pow2_sum(ea, __shfl_sync(0xffffffffu, eb[h], i)));
            }
            stg[lane * 65 + 32 * h + i] = __dadd_rn(e, g.abs_floor);
        }
    }
    __syncwarp();
    // rows in groups of 8: the 16 y loads of a group are issued before any eps
    // store (C may alias Y as far as the compiler knows, so a row-by-row loop
    // paid one L2 round trip per row -- ~10 us per tile, the largest part of
    // the per-tile fixed cost)
    const int64_t rows_left = g.M - (m0 + quarter * 32);
    for (int r0 = 0; r0 < 32 && r0 < rows_left; r0 += 8) {
        float yv[8][2];
#pragma unroll
        for (int k = 0; k < 8; k++)
#pragma unroll
            for (int j = 0; j < 2; j++) {
                const int64_t m = m0 + quarter * 32 + r0 + k;
                const int64_t n = n0 + half * 64 + 32 * j + lane;
                yv[k][j] = (g.Y && r0 + k < rows_left && n < g.N)
                               ? __ldg(g.Y + (int64_t)bz * g.sC + m * g.ldc + n) : 0.0f;
            }
#pragma unroll
        for (int k = 0; k < 8; k++)
#pragma unroll
            for (int j = 0; j < 2; j++) {
                const int64_t m = m0 + quarter * 32 + r0 + k;
                const int64_t n = n0 + half * 64 + 32 * j + lane;
                if (r0 + k < rows_left && n < g.N) {
                    double e = stg[(r0 + k) * 65 + 32 * j + lane];
                    const int64_t o = (int64_t)bz * g.sC + m * g.ldc + n;
                    if (g.Y) e = __dadd_rn(e, __dmul_rn(g.u, fabs((double)yv[k][j])));
                    if (g.out_f64) static_cast<double*>(g.C)[o] = e;
                    else static_cast<float*>(g.C)[o] = __double2float_ru(e);
                }
            }
    }
}

// NAO_TC_REGSPLIT: launched with 128 registers per thread (49152 per CTA) so a
// commit CTA (128 threads x 128 registers) fits beside it on the SM; the
// producer / MMA / TMEM-alloc warps give registers back (setmaxnreg.dec 48),
// the 8 epilogue warps take 168 (the FP64 running sums of their 64 columns).
#ifndef NAO_TC_REGSPLIT
#define NAO_TC_REGSPLIT 0
#endif
#if NAO_TC_REGSPLIT
#define NAO_TC_KERNEL_BOUNDS __maxnreg__(128)
#else
#define NAO_TC_KERNEL_BOUNDS __launch_bounds__(NUM_THREADS, 1)
#endif

template <int FMT>
__global__ void NAO_TC_KERNEL_BOUNDS
    k_absgemm_tc(const __grid_constant__ CUtensorMap map_ahi,
                 const __grid_constant__ CUtensorMap map_alo,
                 const __grid_constant__ CUtensorMap map_bhi,
                 const __grid_constant__ CUtensorMap map_blo, const __grid_constant__ TcArgs g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full = bars;                      // [STAGES]
    uint64_t* empty = bars + STAGES;            // [STAGES]
    uint64_t* tfull = bars + 2 * STAGES;        // [2]
    uint64_t* tempty = bars + 2 * STAGES + 2;   // [2]
    uint64_t* acc1_full = bars + 2 * STAGES + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 5);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // grouped rasterization: consecutive CTAs sweep GROUP_M row tiles per column
    // tile, so the B tiles in flight are shared by GROUP_M CTAs through L2
    const int tiles_m = (int)((g.M + BM - 1) / BM), tiles_n = (int)((g.N + BN - 1) / BN);
#ifndef NAO_TC_GROUP_M
#define NAO_TC_GROUP_M 8
#endif
    constexpr int GROUP_M = NAO_TC_GROUP_M;
    const int pid = blockIdx.x;
    const int group = pid / (GROUP_M * tiles_n);
    const int first_m = group * GROUP_M;
    const int gm = (tiles_m - first_m) < GROUP_M ? (tiles_m - first_m) : GROUP_M;
    const int tm = first_m + (pid % (GROUP_M * tiles_n)) % gm;
    const int tn = (pid % (GROUP_M * tiles_n)) / gm;
    const int n0 = tn * BN, m0 = tm * BM, bz = blockIdx.z;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; b++) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 8); }
        mbar_init(acc1_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)));
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nkb = g.nkb;
    constexpr int KBE = FmtK<FMT>::kb;  // k elements per stage
#if NAO_TC_REGSPLIT
#define NAO_REG_DEC() asm volatile("setmaxnreg.dec.sync.aligned.u32 48;")
#define NAO_REG_INC() asm volatile("setmaxnreg.inc.sync.aligned.u32 168;")
#else
#define NAO_REG_DEC()
#define NAO_REG_INC()
#endif

    if (warp == 0) {
        NAO_REG_DEC();
        if (lane == 0) {  // ---------------- TMA producer
            const int za = g.a_batched ? bz : 0, zb = g.b_batched ? bz : 0;
            for (int kb = 0; kb < nkb; kb++) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
#ifdef NAO_TC_NOWAIT
                if (kb >= STAGES) break;
#endif
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* st = smem + s * STAGE_BYTES;
                mbar_expect_tx(&full[s], STAGE_BYTES);
                tma_load_3d(st, &map_ahi, &full[s], kb * KBE, m0, za);
                tma_load_3d(st + TILE_BYTES, &map_alo, &full[s], kb * KBE, m0, za);
                tma_load_3d(st + 2 * TILE_BYTES, &map_bhi, &full[s], kb * KBE, n0, zb);
                tma_load_3d(st + 3 * TILE_BYTES, &map_blo, &full[s], kb * KBE, n0, zb);
            }
        }
    } else if (warp == 1) {  // ---------------- MMA issuer (whole warp, one elected lane issues)
        NAO_REG_DEC();
        const uint64_t desc0 = make_desc(smem_u32(smem));
        const uint32_t acc1 = tmem + 2 * BN;
        for (int kb = 0; kb < nkb; kb++) {
            const int s = kb % STAGES;
            const uint32_t ph = (kb / STAGES) & 1;
            const int chunk = kb / KCHUNK_KB, buf = chunk & 1;
            const bool first = (kb % KCHUNK_KB) == 0;
            if (first) mbar_wait(&tempty[buf], ((chunk >> 1) & 1) ^ 1);
#ifdef NAO_TC_NOWAIT  // timing probe only (wrong results): MMA rate without the TMA feed
            if (kb < STAGES) mbar_wait(&full[s], ph);
#else
            mbar_wait(&full[s], ph);
#endif
            fence_after();
            // descriptor of this stage's first operand tile: the start-address field
            // is (addr >> 4) in the low 14 bits, so offsets within the ring are adds
            const uint64_t dst = desc0 + (uint64_t)((s * STAGE_BYTES) >> 4);
            const uint32_t acc0 = tmem + buf * BN;
            if (elect_one()) {
#pragma unroll
                for (int j = 0; j < BK / 8; j++) {
                    const uint64_t ahi = dst + (uint64_t)((j * 32) >> 4);
                    const uint64_t alo = dst + (uint64_t)((TILE_BYTES + j * 32) >> 4);
                    const uint64_t bhi = dst + (uint64_t)((2 * TILE_BYTES + j * 32) >> 4);
                    const uint64_t blo = dst + (uint64_t)((3 * TILE_BYTES + j * 32) >> 4);
                    umma_fmt<FMT>(acc0, ahi, bhi, (first && j == 0) ? 0u : 1u);
                    umma_fmt<FMT>(acc1, ahi, blo, (kb == 0 && j == 0) ? 0u : 1u);
                    umma_fmt<FMT>(acc1, alo, bhi, 1u);
                }
                umma_commit(&empty[s]);
                if ((kb % KCHUNK_KB) == KCHUNK_KB - 1 || kb == nkb - 1) umma_commit(&tfull[buf]);
            }
            __syncwarp();
        }
        if (elect_one()) umma_commit(acc1_full);
        __syncwarp();
    } else if (warp >= 4) {  // ---------------- epilogue
        NAO_REG_INC();
        const int ew = warp - 4, quarter = warp & 3, half = ew >> 2;
        const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
        EpiAcc acc;
        acc.zero();
        const int nchunks = (nkb + KCHUNK_KB - 1) / KCHUNK_KB;
        for (int c = 0; c < nchunks; c++) {
            const int buf = c & 1;
            mbar_wait(&tfull[buf], (c >> 1) & 1);
            fence_after();
            uint32_t v[32];
            const uint32_t col = tmem + lane_addr + buf * BN + half * 64;
            TMEM_LD_X32(col, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; i++) acc.add(i, __uint_as_float(v[i]));
            TMEM_LD_X32(col + 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; i++)
                acc.add(32 + i, __uint_as_float(v[i]));
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[buf]);
        }
        mbar_wait(acc1_full, 0);
        fence_after();
        const uint32_t col1 = tmem + lane_addr + 2 * BN + half * 64;
        double* stg = reinterpret_cast<double*>(smem) + ew * (32 * 65);
        tile_epilogue<FMT>(g, acc, col1, stg, lane, quarter, half, m0, n0, bz);
    } else {  // warps 2, 3 (TMEM allocator, spare)
        NAO_REG_DEC();
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(TMEM_COLS));
    }
}


// ---------------------------------------------------------------------------
// Persistent variant for short K (K <= KCHUNK: one TMEM chunk per tile), e.g.
// attention scores q k^T with K = head_dim.  There the per-tile fixed costs
// (TMEM alloc, barrier init, pipeline fill, epilogue) of the one-CTA-per-tile
// kernel dominate (8192 tiles of 24 MMAs for Qwen3-8B scores).  One CTA per SM
// walks tiles t = blockIdx.x + i*gridDim.x; TMEM holds two tile slots
// (acc0 | acc1, 256 columns each), so the MMAs of tile i+1 overlap the
// epilogue of tile i; the stage ring streams k-blocks across tile boundaries;
// the epilogue stages FP32 (rounded up) rows in a dedicated smem area and
// stores coalesced.  FP32 eps output only (the streaming verifier's format).
namespace shortk {
constexpr int STAGES = 4;
constexpr int RING_BYTES = STAGES * STAGE_BYTES;
constexpr int STG_BYTES = 8 * 32 * 65 * 4;
constexpr int SMEM_BYTES = RING_BYTES + STG_BYTES + 1024 + 256;
}  // namespace shortk

// FP16 short-K epilogue, rare element path (tiles with tiny parts or extreme
// exponents): tiny-part flag for the exact fix-up, and the two-step scaling.
__device__ __noinline__ float short_rare(const TcArgs& g, float e, int k, int tbh, int ebh, int ta,
                                         int ea, int bz, int64_t mrow, int64_t n, bool tiny) {
    const int nt = ta + __shfl_sync(0xffffffffu, tbh, k);
    const int ebk = __shfl_sync(0xffffffffu, ebh, k);
    if (tiny && nt > 0 && n < g.N && mrow < g.M && e <= g.fix_thrf * (float)nt)
        flag_fix(g, bz, mrow, n);
    return mul_pow2_ru(e, -(ea + ebk));
}

template <int FMT>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_absgemm_tc_short(const __grid_constant__ CUtensorMap map_ahi,
                       const __grid_constant__ CUtensorMap map_alo,
                       const __grid_constant__ CUtensorMap map_bhi,
                       const __grid_constant__ CUtensorMap map_blo, const __grid_constant__ TcArgs g,
                       int batch) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float* stg_all = reinterpret_cast<float*>(smem + shortk::RING_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + shortk::RING_BYTES + shortk::STG_BYTES);
    uint64_t* full = bars;                              // [STAGES]
    uint64_t* empty = bars + shortk::STAGES;            // [STAGES]
    uint64_t* tfull = bars + 2 * shortk::STAGES;        // [2] tile slots
    uint64_t* tempty = bars + 2 * shortk::STAGES + 2;   // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * shortk::STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tiles_m = (int)((g.M + BM - 1) / BM), tiles_n = (int)((g.N + BN - 1) / BN);
    const int64_t tiles_per_b = (int64_t)tiles_m * tiles_n;
    const int64_t n_tiles = tiles_per_b * batch;

    if (threadIdx.x == 0) {
        for (int s = 0; s < shortk::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; b++) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)));
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nkb = g.nkb;
    constexpr int KBE = FmtK<FMT>::kb;  // k elements per stage

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            int kg = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                const int bz = (int)(t / tiles_per_b);
                const int64_t r = t % tiles_per_b;
                const int m0 = (int)(r / tiles_n) * BM, n0 = (int)(r % tiles_n) * BN;
                const int za = g.a_batched ? bz : 0, zb = g.b_batched ? bz : 0;
                for (int kb = 0; kb < nkb; kb++, kg++) {
                    const int s = kg % shortk::STAGES;
                    const uint32_t ph = (kg / shortk::STAGES) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* st = smem + s * STAGE_BYTES;
                    mbar_expect_tx(&full[s], STAGE_BYTES);
                    tma_load_3d(st, &map_ahi, &full[s], kb * KBE, m0, za);
                    tma_load_3d(st + TILE_BYTES, &map_alo, &full[s], kb * KBE, m0, za);
                    tma_load_3d(st + 2 * TILE_BYTES, &map_bhi, &full[s], kb * KBE, n0, zb);
                    tma_load_3d(st + 3 * TILE_BYTES, &map_blo, &full[s], kb * KBE, n0, zb);
                }
            }
        }
    } else if (warp == 1) {  // ---------------- MMA issuer (whole warp, one elected lane issues)
        const uint64_t desc0 = make_desc(smem_u32(smem));
        int kg = 0, i = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, i++) {
            const int slot = i & 1;
            mbar_wait(&tempty[slot], ((i >> 1) & 1) ^ 1);
            fence_after();
            const uint32_t acc0 = tmem + slot * 256, acc1 = acc0 + BN;
            for (int kb = 0; kb < nkb; kb++, kg++) {
                const int s = kg % shortk::STAGES;
                const uint32_t ph = (kg / shortk::STAGES) & 1;
                mbar_wait(&full[s], ph);
                fence_after();
                const uint64_t dst = desc0 + (uint64_t)((s * STAGE_BYTES) >> 4);
                if (elect_one()) {
#pragma unroll
                    for (int j = 0; j < BK / 8; j++) {
                        const uint64_t ahi = dst + (uint64_t)((j * 32) >> 4);
                        const uint64_t alo = dst + (uint64_t)((TILE_BYTES + j * 32) >> 4);
                        const uint64_t bhi = dst + (uint64_t)((2 * TILE_BYTES + j * 32) >> 4);
                        const uint64_t blo = dst + (uint64_t)((3 * TILE_BYTES + j * 32) >> 4);
                        const uint32_t first = (kb == 0 && j == 0) ? 0u : 1u;
                        umma_fmt<FMT>(acc0, ahi, bhi, first);
                        umma_fmt<FMT>(acc1, ahi, blo, first);
                        umma_fmt<FMT>(acc1, alo, bhi, 1u);
                    }
                    umma_commit(&empty[s]);
                }
                __syncwarp();
            }
            if (elect_one()) umma_commit(&tfull[slot]);
            __syncwarp();
        }
    } else if (warp >= 4) {  // ---------------- epilogue
        const int ew = warp - 4, quarter = warp & 3, half = ew >> 2;
        const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
        float* stg = stg_all + ew * (32 * 65);
        int i = 0;
        for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, i++) {
            const int slot = i & 1;
            const int bz = (int)(t / tiles_per_b);
            const int64_t r = t % tiles_per_b;
            const int64_t m0 = (r / tiles_n) * BM, n0 = (r % tiles_n) * BN;
            // FP16: per-thread row scale, per-lane column scales broadcast by shuffles;
            // 2^(ea+eb) = rowf * colf when both exponents are in FP32 range
            const int64_t mrow = m0 + quarter * 32 + lane;
            int ea = 0, ta = 0, eb[2] = {0, 0}, tb[2] = {0, 0};
            bool tiny_tile = false, in_range = true;
            float rowf = 1.f, colf[2] = {1.f, 1.f}, flag_lim = -1.f;
            if constexpr (FMT == kFmtF16) {
                const int64_t ao = (g.a_batched ? (int64_t)bz * g.M : 0) + mrow;
                if (mrow < g.M) { ea = __ldg(g.a_exp + ao); ta = __ldg(g.a_tiny + ao); }
                const int64_t bo = g.b_batched ? (int64_t)bz * g.N : 0;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int64_t n = n0 + half * 64 + 32 * h + lane;
                    if (n < g.N) { eb[h] = __ldg(g.b_exp + bo + n); tb[h] = __ldg(g.b_tiny + bo + n); }
                    colf[h] = pow2f(eb[h] < -126 ? -126 : (eb[h] > 126 ? 126 : eb[h]));
                }
                rowf = pow2f(ea < -126 ? -126 : (ea > 126 ? 126 : ea));
                tiny_tile = __any_sync(0xffffffffu, (ta | tb[0] | tb[1]) != 0);
                // no element of this row can need the exact fix-up unless its value is
                // <= fix_thr * (ta + max tb over the tile's columns)
                int tmax = tb[0] > tb[1] ? tb[0] : tb[1];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
                flag_lim = g.fix_thrf * (float)(ta + tmax);
                in_range = __all_sync(0xffffffffu, ea >= -126 && ea <= 126 && eb[0] >= -126 &&
                                                       eb[0] <= 126 && eb[1] >= -126 && eb[1] <= 126);
            }
            mbar_wait(&tfull[slot], (i >> 1) & 1);
            fence_after();
            const uint32_t c0 = tmem + lane_addr + slot * 256 + half * 64;
            // e = RU(RU(s0 acc0) + s1 acc1) + floor in FP32 round-up arithmetic: each
            // step rounds toward +inf, so e >= the FP64 expression of the long
            // kernel; the extra over-estimate is < 4 * 2^-23 relative.
#pragma unroll
            for (int h = 0; h < 2; h++) {
                uint32_t v0[32], v1[32];
                TMEM_LD_X32(c0 + 32 * h, v0);
                TMEM_LD_X32(c0 + BN + 32 * h, v1);
                tmem_wait_ld();
                if (h == 1) {  // both halves read: hand the slot back to the MMA warp
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[slot]);
                }
#pragma unroll
                for (int k = 0; k < 32; k++) {
                    float e = __fmaf_ru(g.scale1f, __uint_as_float(v1[k]),
                                        __fmul_ru(g.scale0f, __uint_as_float(v0[k])));
                    if constexpr (FMT == kFmtF16) {
                        const bool rare = __any_sync(0xffffffffu, e <= flag_lim) || !in_range;
                        if (rare)  // warp-uniform, rare: out of line
                            e = short_rare(g, e, k, tb[h], eb[h], ta, ea, bz, mrow,
                                           n0 + half * 64 + 32 * h + k, tiny_tile);
                        else
                            e = __fmul_ru(__fmul_ru(e, rowf), __shfl_sync(0xffffffffu, colf[h], k));
                    }
                    stg[lane * 65 + 32 * h + k] = __fadd_ru(e, g.abs_floorf);
                }
            }
            __syncwarp();
            const int64_t mq = m0 + quarter * 32;
            const int rows = (int)((g.M - mq) < 32 ? (g.M - mq) : 32);
            const int64_t nb = n0 + half * 64 + lane;
            float* crow = static_cast<float*>(g.C) + (int64_t)bz * g.sC + mq * g.ldc + nb;
            const float* yrow = g.Y ? g.Y + (int64_t)bz * g.sC + mq * g.ldc + nb : nullptr;
            const bool ok0 = nb < g.N, ok1 = nb + 32 < g.N;
            for (int r0 = 0; r0 < rows; r0 += 8) {  // y loads of 8 rows before the stores
                float y0[8], y1[8];
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const bool in = yrow && r0 + k < rows;
                    y0[k] = in && ok0 ? __ldg(yrow + (int64_t)(r0 + k) * g.ldc) : 0.0f;
                    y1[k] = in && ok1 ? __ldg(yrow + (int64_t)(r0 + k) * g.ldc + 32) : 0.0f;
                }
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    if (r0 + k >= rows) break;
                    float e0 = stg[(r0 + k) * 65 + lane], e1 = stg[(r0 + k) * 65 + 32 + lane];
                    if (yrow) {
                        e0 = __fmaf_ru(g.uf, fabsf(y0[k]), e0);
                        e1 = __fmaf_ru(g.uf, fabsf(y1[k]), e1);
                    }
                    if (ok0) crow[(int64_t)(r0 + k) * g.ldc] = e0;
                    if (ok1) crow[(int64_t)(r0 + k) * g.ldc + 32] = e1;
                }
            }
            __syncwarp();
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(TMEM_COLS));
    }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x 128 tile with M=256 MMAs issued by the leader CTA.  Each CTA stages its
// own 128 rows of A and HALF (64 rows) of B, so per SM the smem ring holds 96
// instead of 128 rows per k-block and the tensor core reads 6 KB instead of
// 8 KB of smem per MMA -- the single-CTA kernel is smem/L2-feed bound at
// N=128 (tensor pipe ~40 %).  Error model, TMEM layout (acc0 x2 + acc1 per
// CTA, lane = row) and epilogue are identical to k_absgemm_tc.
namespace pair {
constexpr int BM = 128;          // rows of A (and of the output) per CTA
constexpr int BN = 128;          // output columns per pair (= per CTA)
constexpr int BNH = BN / 2;      // rows of B staged per CTA
constexpr int BK = NAO_TC_BK;
constexpr int STAGES = BK == 16 ? 8 : 4;
constexpr int KCHUNK_KB = KCHUNK / BK;
constexpr int A_BYTES = BM * BK * 4;
constexpr int B_BYTES = BNH * BK * 4;
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;   // per CTA
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int NUM_THREADS = 384;
constexpr uint32_t TMEM_COLS = 512;
// kind::tf32, D=F32, K-major A/B, N=128, M=256 (cta_group::2)
constexpr uint32_t kIdesc2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);
constexpr uint32_t kIdesc2F16 = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                ((uint32_t)(256 >> 4) << 24);
}  // namespace pair

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONEC_%=;\n\t"
        "bra WAITC_%=;\n"
        "DONEC_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
// TMA into this CTA's smem, completing bytes on the LEADER CTA's barrier
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map,
                                                 uint32_t bar_cluster, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], m;\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void umma_tf32_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void umma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
template <int FMT>
__device__ __forceinline__ void umma_pair_fmt(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
    if constexpr (FMT == kFmtF16) umma_f16_pair(d, a, b, pair::kIdesc2F16, acc);
    else umma_tf32_pair(d, a, b, pair::kIdesc2, acc);
}

template <int FMT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pair::NUM_THREADS, 1)
    k_absgemm_tc2(const __grid_constant__ CUtensorMap map_ahi,
                  const __grid_constant__ CUtensorMap map_alo,
                  const __grid_constant__ CUtensorMap map_bhi,
                  const __grid_constant__ CUtensorMap map_blo, const __grid_constant__ TcArgs g) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + pair::STAGES * pair::STAGE_BYTES);
    uint64_t* full = bars;                      // [pair::STAGES]  (leader's are used)
    uint64_t* empty = bars + pair::STAGES;            // [pair::STAGES]  (each CTA, multicast commit)
    uint64_t* tfull = bars + 2 * pair::STAGES;        // [2]       (each CTA, multicast commit)
    uint64_t* tempty = bars + 2 * pair::STAGES + 2;   // [2]       (leader's: 16 epilogue warps)
    uint64_t* acc1_full = bars + 2 * pair::STAGES + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * pair::STAGES + 5);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int tiles_m = (int)((g.M + 2 * pair::BM - 1) / (2 * pair::BM)), tiles_n = (int)((g.N + pair::BN - 1) / pair::BN);
    constexpr int GROUP_M = 4;
    const int pid = blockIdx.x >> 1;
    const int group = pid / (GROUP_M * tiles_n);
    const int first_m = group * GROUP_M;
    const int gm = (tiles_m - first_m) < GROUP_M ? (tiles_m - first_m) : GROUP_M;
    const int tm = first_m + (pid % (GROUP_M * tiles_n)) % gm;
    const int tn = (pid % (GROUP_M * tiles_n)) / gm;
    const int n0 = tn * pair::BN, m0 = tm * 2 * pair::BM + (int)rank * pair::BM, bz = blockIdx.z;

    if (threadIdx.x == 0) {
        for (int s = 0; s < pair::STAGES; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; b++) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 16); }
        mbar_init(acc1_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)));
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)));
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(pair::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync_all();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nkb = g.nkb;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer (both CTAs)
            const int za = g.a_batched ? bz : 0, zb = g.b_batched ? bz : 0;
            const int nb = n0 + (int)rank * pair::BNH;
            for (int kb = 0; kb < nkb; kb++) {
                const int s = kb % pair::STAGES;
                const uint32_t ph = (kb / pair::STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* st = smem + s * pair::STAGE_BYTES;
                const uint32_t fb = mapa_rank(smem_u32(&full[s]), 0);
                if (leader) mbar_expect_tx(&full[s], 2 * pair::STAGE_BYTES);
                constexpr int KBE = FmtK<FMT>::kb;
                tma_load_3d_pair(st, &map_ahi, fb, kb * KBE, m0, za);
                tma_load_3d_pair(st + pair::A_BYTES, &map_alo, fb, kb * KBE, m0, za);
                tma_load_3d_pair(st + 2 * pair::A_BYTES, &map_bhi, fb, kb * KBE, nb, zb);
                tma_load_3d_pair(st + 2 * pair::A_BYTES + pair::B_BYTES, &map_blo, fb, kb * KBE, nb, zb);
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && leader) {  // ---------------- MMA issuer (leader only)
            const uint32_t acc1 = tmem + 2 * pair::BN;
            for (int kb = 0; kb < nkb; kb++) {
                const int s = kb % pair::STAGES;
                const uint32_t ph = (kb / pair::STAGES) & 1;
                const int chunk = kb / pair::KCHUNK_KB, buf = chunk & 1;
                const bool first = (kb % pair::KCHUNK_KB) == 0;
                if (first) mbar_wait_cluster(&tempty[buf], ((chunk >> 1) & 1) ^ 1);
                mbar_wait(&full[s], ph);
                fence_after();
                const uint32_t st = smem_u32(smem + s * pair::STAGE_BYTES);
                const uint32_t acc0 = tmem + buf * pair::BN;
#pragma unroll
                for (int j = 0; j < pair::BK / 8; j++) {
                    const uint64_t ahi = make_desc(st + j * 32);
                    const uint64_t alo = make_desc(st + pair::A_BYTES + j * 32);
                    const uint64_t bhi = make_desc(st + 2 * pair::A_BYTES + j * 32);
                    const uint64_t blo = make_desc(st + 2 * pair::A_BYTES + pair::B_BYTES + j * 32);
                    umma_pair_fmt<FMT>(acc0, ahi, bhi, (first && j == 0) ? 0u : 1u);
                    umma_pair_fmt<FMT>(acc1, ahi, blo, (kb == 0 && j == 0) ? 0u : 1u);
                    umma_pair_fmt<FMT>(acc1, alo, bhi, 1u);
                }
                umma_commit_pair(&empty[s]);
                if ((kb % pair::KCHUNK_KB) == pair::KCHUNK_KB - 1 || kb == nkb - 1) umma_commit_pair(&tfull[buf]);
            }
            umma_commit_pair(acc1_full);
        }
    } else if (warp >= 4) {  // ---------------- epilogue (both CTAs, own 128 rows)
        const int ew = warp - 4, quarter = warp & 3, half = ew >> 2;
        const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
        const uint32_t tempty_leader0 = mapa_rank(smem_u32(&tempty[0]), 0);
        const uint32_t tempty_leader1 = mapa_rank(smem_u32(&tempty[1]), 0);
        EpiAcc acc;
        acc.zero();
        const int nchunks = (nkb + pair::KCHUNK_KB - 1) / pair::KCHUNK_KB;
        for (int c = 0; c < nchunks; c++) {
            const int buf = c & 1;
            mbar_wait(&tfull[buf], (c >> 1) & 1);
            fence_after();
            uint32_t v[32];
            const uint32_t col = tmem + lane_addr + buf * pair::BN + half * 64;
            TMEM_LD_X32(col, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; i++) acc.add(i, __uint_as_float(v[i]));
            TMEM_LD_X32(col + 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; i++)
                acc.add(32 + i, __uint_as_float(v[i]));
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(buf ? tempty_leader1 : tempty_leader0);
        }
        mbar_wait(acc1_full, 0);
        fence_after();
        const uint32_t col1 = tmem + lane_addr + 2 * pair::BN + half * 64;
        double* stg = reinterpret_cast<double*>(smem) + ew * (32 * 65);
        tile_epilogue<FMT>(g, acc, col1, stg, lane, quarter, half, m0, n0, bz);
    }
    fence_before();
    cluster_sync_all();
    if (warp == 2) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(pair::TMEM_COLS));
    }
}

// |x| -> (hi, lo) TF32 parts, K-major [rows, Kp] (zero padded), optionally
// reading x transposed (x is [K, rows] row-major when `trans`).
__device__ __forceinline__ void split_one(float x, float& h, float& l) {
    const float a = fabsf(x);
    const uint32_t hb = __float_as_uint(a) & 0xFFFFE000u;  // truncate to TF32: hi <= a
    h = __uint_as_float(hb);
    const uint32_t rb = __float_as_uint(__fsub_rn(a, h));  // exact remainder
    l = __uint_as_float((rb & 0x1FFFu) ? ((rb & 0xFFFFE000u) + 0x2000u) : rb);  // RU to TF32
    if (h != 0.f && h < 1.17549435e-38f) h = 1.17549435e-38f;  // no subnormal operands
    if (l != 0.f && l < 1.17549435e-38f) l = 1.17549435e-38f;
}

// Fast path: x is [batch*rows, K] contiguous with K % 4 == 0 (so Kp == K).
__global__ void k_split_tf32_vec(const float4* __restrict__ x, float4* __restrict__ hi,
                                 float4* __restrict__ lo, int64_t n4) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n4;
         t += (int64_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(x + t);
        float4 h, l;
        split_one(v.x, h.x, l.x); split_one(v.y, h.y, l.y);
        split_one(v.z, h.z, l.z); split_one(v.w, h.w, l.w);
        hi[t] = h;
        lo[t] = l;
    }
}

__global__ void k_split_tf32(const float* __restrict__ x, float* __restrict__ hi,
                             float* __restrict__ lo, int64_t batch, int64_t rows, int64_t K,
                             int64_t Kp, int64_t ld, int64_t sbatch, int trans) {
    const int64_t total = batch * rows * Kp;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = t % Kp, r = (t / Kp) % rows, b = t / (Kp * rows);
        float a = 0.f;
        if (k < K) {
            const float* xb = x + b * sbatch;
            a = fabsf(trans ? __ldg(xb + k * ld + r) : __ldg(xb + r * ld + k));
        }
        uint32_t ab = __float_as_uint(a);
        uint32_t hb = ab & 0xFFFFE000u;                       // truncate to TF32: hi <= a
        float h = __uint_as_float(hb);
        float rem = __fsub_rn(a, h);                          // exact
        uint32_t rb = __float_as_uint(rem);
        uint32_t lb = (rb & 0x1FFFu) ? ((rb & 0xFFFFE000u) + 0x2000u) : rb;  // RU to TF32
        float l = __uint_as_float(lb);
        // tensor cores may flush subnormals: lift non-zero subnormal parts to FLT_MIN
        if (h != 0.f && h < 1.17549435e-38f) h = 1.17549435e-38f;
        if (l != 0.f && l < 1.17549435e-38f) l = 1.17549435e-38f;
        hi[t] = h;
        lo[t] = l;
    }
}

// NAO_TC_PAIR=1 selects the CTA-pair kernel (measured 5-10 % slower than the
// single-CTA kernel at every Qwen3-8B shape: the pair couples two epilogues and
// two TMA streams per MMA while the L2->SM feed per SM drops only 25 %).
static bool tc_use_pair() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("NAO_TC_PAIR");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

// NAO_TC_SHORT=0 disables the persistent short-K kernel (A/B measurements)
static bool tc_no_short() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("NAO_TC_SHORT");
        v = (e && e[0] == '0') ? 1 : 0;
    }
    return v == 1;
}

// host double -> float rounded toward +inf
static float f32_ru(double x) {
    float f = (float)x;
    if ((double)f < x) f = nextafterf(f, INFINITY);
    return f;
}

using EncodeFn = PFN_cuTensorMapEncodeTiled_v12000;

static EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

static int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t Kp, int64_t batch,
                    int box_rows = BM, int fmt = kFmtTF32) {
    EncodeFn enc = get_encode();
    NAO_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
    const int es = fmt == kFmtF16 ? 2 : 4;
    const int bk = 64 / es;  // 64-byte K rows (SWIZZLE_64B)
    cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)batch};
    cuuint64_t strides[2] = {(cuuint64_t)Kp * es, (cuuint64_t)(rows * Kp * es)};
    cuuint32_t box[3] = {(cuuint32_t)(fmt == kFmtF16 ? bk : BK), (cuuint32_t)box_rows, 1};
    cuuint32_t est[3] = {1, 1, 1};
    CUresult r = enc(map, fmt == kFmtF16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                         : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                     3, const_cast<void*>(base), dims, strides, box, est,
                     CU_TENSOR_MAP_INTERLEAVE_NONE,
                     (fmt != kFmtF16 && BK == 32) ? CU_TENSOR_MAP_SWIZZLE_128B
                                                  : CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    NAO_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return NAO_OK;
}

// ------------------------------------------------------------ FP16 split
// |x| -> x_s = |x| * 2^-e (e per row: the row max lands in [2^14, 2^15)), then
//   x_s >= 2^-14 : hi = RZ_f16(x_s),  lo = RU_f16((x_s - hi) * 2^10)
//   x_s <  2^-14 : hi = RU_f16(x_s) (subnormal half),  lo = 0
// so x_s <= hi + 2^-10 lo, with relative excess <= 2^-20 (1.001) for normal
// hi and absolute excess < 2^-24 for the tiny ones; lo <= 2^-10 hi (1.001).
// FP32 arithmetic: the power-of-two scaling is exact (rounded UP when it
// would leave the FP32 range), remainders are exact, the FP16 roundings are
// bit operations, so every part is an exact half.
__device__ __forceinline__ float scale_ru(float a, int t) {  // a * 2^t, rounded up
    const int t1 = t > 126 ? 126 : (t < -126 ? -126 : t);
    int t2 = t - t1;
    t2 = t2 > 126 ? 126 : (t2 < -126 ? -126 : t2);
    a = __fmul_ru(a, pow2f(t1));
    return t2 ? __fmul_ru(a, pow2f(t2)) : a;
}
__device__ __forceinline__ float ru_f16f(float v) {  // v >= 0, finite, < 65504
    if (v >= 0x1p-14f) {
        const uint32_t b = __float_as_uint(v);
        return __uint_as_float((b & 0x1FFFu) ? (b & ~0x1FFFu) + 0x2000u : b);
    }
    return ceilf(v * 0x1p24f) * 0x1p-24f;  // subnormal half grid (exact scalings)
}
// returns 1 when the element is "tiny" (non-zero, below the normal half range)
__device__ __forceinline__ int split16_one(float x, int e, __half& h, __half& l) {
    const float a = scale_ru(fabsf(x), -e);
    float hf, lf = 0.f;
    if (!(a < INFINITY)) { hf = a; }  // inf / nan propagate
    else if (a >= 0x1p-14f) {
        hf = __uint_as_float(__float_as_uint(a) & ~0x1FFFu);  // RZ to 11 significant bits
        lf = ru_f16f(__fmul_rn(__fsub_rn(a, hf), 0x1p10f));    // exact remainder * 2^10
    } else {
        hf = ru_f16f(a);
    }
    h = __float2half_rn(hf);  // exact (representable)
    l = __float2half_rn(lf);
    return (a > 0.f && a < 0x1p-14f) ? 1 : 0;
}
__device__ __forceinline__ int row_scale_exp(float amax) {
    if (!(amax > 0.f) || !(amax < INFINITY)) return 0;
    int e;
    frexpf(amax, &e);  // amax = f 2^e, f in [0.5, 1)
    return e - 15;
}
__device__ __forceinline__ float nan_max(float m, float v) {  // max that keeps NaN
    return (v == v) ? fmaxf(m, v) : v;
}

// x row-major [rows, K] (ld), a warp per row: max pass, then the split pass
// (the row is re-read from L1/L2).  VEC: K % 8 == 0, ld % 4 == 0, 16-byte base.
template <bool VEC>
__global__ void __launch_bounds__(256) k_split_f16_rows(const float* __restrict__ x,
                                                       __half* __restrict__ hi,
                                                       __half* __restrict__ lo,
                                                       int32_t* __restrict__ sexp, int64_t batch,
                                                       int64_t rows, int64_t K, int64_t Kp,
                                                       int64_t ld, int64_t sbatch) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
         t < batch * rows; t += nw) {
        const int64_t b = t / rows, r = t % rows;
        const float* xr = x + b * sbatch + r * ld;
        float m = 0.f;
        if (VEC) {
            const float4* x4 = reinterpret_cast<const float4*>(xr);
            for (int64_t k = lane; k < (K >> 2); k += 32) {
                const float4 v = __ldg(x4 + k);
                m = nan_max(nan_max(nan_max(nan_max(m, fabsf(v.x)), fabsf(v.y)), fabsf(v.z)),
                            fabsf(v.w));
            }
        } else {
            for (int64_t k = lane; k < K; k += 32) m = nan_max(m, fabsf(__ldg(xr + k)));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, o));
        const int e = row_scale_exp(m);
        int tiny = 0;
        __half* hr = hi + t * Kp;
        __half* lr = lo + t * Kp;
        if (VEC) {
            const float4* x4 = reinterpret_cast<const float4*>(xr);
            for (int64_t k = lane; k < (K >> 2); k += 32) {
                const float4 v = __ldg(x4 + k);
                __half h[4], l[4];
                tiny += split16_one(v.x, e, h[0], l[0]) + split16_one(v.y, e, h[1], l[1]) +
                        split16_one(v.z, e, h[2], l[2]) + split16_one(v.w, e, h[3], l[3]);
                reinterpret_cast<uint2*>(hr)[k] = *reinterpret_cast<const uint2*>(h);
                reinterpret_cast<uint2*>(lr)[k] = *reinterpret_cast<const uint2*>(l);
            }
        } else {
            for (int64_t k = lane; k < Kp; k += 32) {
                __half h = __float2half(0.f), l = __float2half(0.f);
                if (k < K) tiny += split16_one(__ldg(xr + k), e, h, l);
                hr[k] = h;
                lr[k] = l;
            }
        }
        tiny = warp_sum(tiny);
        if (lane == 0) {
            sexp[t] = e;
            sexp[batch * rows + t] = tiny;  // second block: tiny-part counts
        }
    }
}

// Single DRAM pass: a CTA per row stages the row in shared memory (float4,
// coalesced), block-reduces the max, then splits from shared memory.
// Needs K % 8 == 0, ld % 4 == 0, 16-byte aligned x, K * 4 <= 96 KB.
constexpr int kSplitThreads = 256;
__global__ void __launch_bounds__(kSplitThreads) k_split_f16_rows_smem(
    const float* __restrict__ x, __half* __restrict__ hi, __half* __restrict__ lo,
    int32_t* __restrict__ sexp, int64_t batch, int64_t rows, int64_t K, int64_t ld,
    int64_t sbatch) {
    extern __shared__ float4 srow[];
    __shared__ float wmax[kSplitThreads / 32];
    __shared__ int wtiny[kSplitThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t K4 = K >> 2;
    for (int64_t t = blockIdx.x; t < batch * rows; t += gridDim.x) {
        const int64_t b = t / rows, r = t % rows;
        const float4* xr = reinterpret_cast<const float4*>(x + b * sbatch + r * ld);
        float m = 0.f;
        for (int64_t k = threadIdx.x; k < K4; k += kSplitThreads) {
            const float4 v = __ldg(xr + k);
            srow[k] = v;
            m = nan_max(nan_max(nan_max(nan_max(m, fabsf(v.x)), fabsf(v.y)), fabsf(v.z)),
                        fabsf(v.w));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) wmax[w] = m;
        __syncthreads();
        m = wmax[0];
#pragma unroll
        for (int i = 1; i < kSplitThreads / 32; i++) m = nan_max(m, wmax[i]);
        const int e = row_scale_exp(m);
        uint2* hr = reinterpret_cast<uint2*>(hi + t * K);
        uint2* lr = reinterpret_cast<uint2*>(lo + t * K);
        int tiny = 0;
        for (int64_t k = threadIdx.x; k < K4; k += kSplitThreads) {
            const float4 v = srow[k];
            __half h[4], l[4];
            tiny += split16_one(v.x, e, h[0], l[0]) + split16_one(v.y, e, h[1], l[1]) +
                    split16_one(v.z, e, h[2], l[2]) + split16_one(v.w, e, h[3], l[3]);
            __stcs(hr + k, *reinterpret_cast<const uint2*>(h));
            __stcs(lr + k, *reinterpret_cast<const uint2*>(l));
        }
        tiny = warp_sum(tiny);
        if (lane == 0) wtiny[w] = tiny;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tt = 0;
            for (int i = 0; i < kSplitThreads / 32; i++) tt += wtiny[i];
            sexp[t] = e;
            sexp[batch * rows + t] = tt;
        }
    }
}

// x is [K, rows] row-major per batch (ld): output row r = input column r.
// A CTA owns 32 output rows: column maxima over K, then 32x32 transposed tiles.
__global__ void __launch_bounds__(256) k_split_f16_cols(const float* __restrict__ x,
                                                       __half* __restrict__ hi,
                                                       __half* __restrict__ lo,
                                                       int32_t* __restrict__ sexp, int64_t batch,
                                                       int64_t rows, int64_t K, int64_t Kp,
                                                       int64_t ld, int64_t sbatch) {
    __shared__ float tile[32][33];
    __shared__ float cmax[8][32];
    __shared__ int cexp[32];
    __shared__ int ctiny[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t ctiles = (rows + 31) / 32;
    for (int64_t bt = blockIdx.x; bt < batch * ctiles; bt += gridDim.x) {
        const int64_t b = bt / ctiles, c0 = (bt % ctiles) * 32;
        const float* xb = x + b * sbatch;
        const int64_t c = c0 + lane;
        float m = 0.f;
        if (c < rows)
            for (int64_t k = w; k < K; k += 8) m = nan_max(m, fabsf(__ldg(xb + k * ld + c)));
        cmax[w][lane] = m;
        __syncthreads();
        if (w == 0) {
            float mm = cmax[0][lane];
            for (int i = 1; i < 8; i++) mm = nan_max(mm, cmax[i][lane]);
            const int e = row_scale_exp(mm);
            if (c < rows) sexp[b * rows + c] = e;
            cexp[lane] = e;
            ctiny[lane] = 0;
        }
        __syncthreads();
        for (int64_t k0 = 0; k0 < Kp; k0 += 32) {
            for (int i = w; i < 32; i += 8) {
                const int64_t k = k0 + i;
                tile[i][lane] = (k < K && c < rows) ? __ldg(xb + k * ld + c) : 0.f;
            }
            __syncthreads();
            for (int j = w; j < 32; j += 8) {  // output row c0 + j, k = k0 + lane
                const int64_t r = c0 + j, k = k0 + lane;
                if (r < rows && k < Kp) {
                    __half h = __float2half(0.f), l = __float2half(0.f);
                    if (k < K && split16_one(tile[lane][j], cexp[j], h, l)) atomicAdd(&ctiny[j], 1);
                    hi[(b * rows + r) * Kp + k] = h;
                    lo[(b * rows + r) * Kp + k] = l;
                }
            }
            __syncthreads();
        }
        if (w == 0 && c < rows) sexp[batch * rows + b * rows + c] = ctiny[lane];
        __syncthreads();
    }
}

// Exact FP64 recompute of flagged outputs (FP16 path): eps = s * sum |a||b|
// (+ u|y|), a warp per element.  count > capacity: every element of a row /
// column with tiny parts is recomputed instead.  Leaves the count at zero.
struct FixArgs {
    const float* A;       // [batch_a, M, K]
    const float* B;       // [batch_b, K, N] or [batch_b, N, K] (trans_b)
    int64_t sA, sB;       // batch strides (0 = broadcast)
    int trans_b;
    int64_t M, N, K, batch;
    void* C;
    const float* Y;
    int64_t ldc, sC;
    int out_f64;
    double s, u;
    const int32_t* a_tiny;
    const int32_t* b_tiny;
    int a_batched, b_batched;
    unsigned long long* count;
    const unsigned long long* list;
    unsigned long long cap;
};

__device__ __forceinline__ void fix_one(const FixArgs& f, int64_t bz, int64_t m, int64_t n,
                                        int lane) {
    const float* a = f.A + bz * f.sA + m * f.K;
    const float* b = f.B + bz * f.sB;
    double acc = 0.0;
    for (int64_t k = lane; k < f.K; k += 32) {
        const double bv = f.trans_b ? (double)__ldg(b + n * f.K + k) : (double)__ldg(b + k * f.N + n);
        acc = __dadd_rn(acc, __dmul_rn(fabs((double)__ldg(a + k)), fabs(bv)));
    }
    acc = warp_sum(acc);
    if (lane == 0) {
        const int64_t o = bz * f.sC + m * f.ldc + n;
        double e = __dmul_rn(f.s, acc);
        if (f.Y) e = __dadd_rn(e, __dmul_rn(f.u, fabs((double)__ldg(f.Y + o))));
        if (f.out_f64) static_cast<double*>(f.C)[o] = e;
        else static_cast<float*>(f.C)[o] = __double2float_ru(e);
    }
}

__global__ void __launch_bounds__(256) k_absgemm_fix(const __grid_constant__ FixArgs f) {
    const unsigned long long cnt = *(volatile unsigned long long*)f.count;
    if (cnt == 0) return;
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t w0 = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (cnt <= f.cap) {
        for (int64_t i = w0; i < (int64_t)cnt; i += nw) {
            const unsigned long long idx = f.list[i];
            const int64_t n = (int64_t)(idx % (unsigned long long)f.N);
            const int64_t m = (int64_t)((idx / (unsigned long long)f.N) % (unsigned long long)f.M);
            const int64_t bz = (int64_t)(idx / ((unsigned long long)f.N * (unsigned long long)f.M));
            fix_one(f, bz, m, n, lane);
        }
    } else {
        const int64_t total = f.batch * f.M * f.N;
        for (int64_t t = w0; t < total; t += nw) {
            const int64_t n = t % f.N, m = (t / f.N) % f.M, bz = t / (f.N * f.M);
            const int ta = __ldg(f.a_tiny + (f.a_batched ? bz * f.M : 0) + m);
            const int tb = __ldg(f.b_tiny + (f.b_batched ? bz * f.N : 0) + n);
            if (ta + tb > 0) fix_one(f, bz, m, n, lane);
        }
    }
}

template <int FMT>
static int launch_tc(const void* a_hi, const void* a_lo, const int32_t* a_exp, const void* b_hi,
                     const void* b_lo, const int32_t* b_exp, void* eps, int eps_f64,
                     int64_t batch, int64_t batch_a, int64_t batch_b, int64_t M, int64_t N,
                     int64_t K, int64_t ldc, int64_t stride_c, double gamma_const,
                     const float* y_or_null, double u, double slack, cudaStream_t stream,
                     const float* A = nullptr, const float* B = nullptr, int trans_b = 0,
                     void* fix_ws = nullptr, size_t fix_ws_bytes = 0) {
    NAO_REQUIRE(a_hi && a_lo && b_hi && b_lo && eps, "abs-gemm tc: null pointer");
    NAO_REQUIRE(FMT == kFmtTF32 || (a_exp && b_exp), "abs-gemm tc f16: exponent arrays missing");
    NAO_REQUIRE(FMT == kFmtTF32 || (A && B && fix_ws && fix_ws_bytes >= 128),
                "abs-gemm tc f16: operands / fix-up workspace missing");
    NAO_REQUIRE(M >= 1 && N >= 1 && K >= 1 && batch >= 1, "abs-gemm tc: bad shape");
    NAO_REQUIRE((batch_a == batch || batch_a == 1) && (batch_b == batch || batch_b == 1),
                "abs-gemm tc: bad batch broadcast");
    NAO_REQUIRE(ceil_div(N, BN) * ceil_div(M, BM) < (1LL << 31) && batch <= 65535,
                "abs-gemm tc: grid too large");
    const int64_t Kp = FMT == kFmtF16 ? (K + 7) / 8 * 8 : (K + 3) / 4 * 4;
    const int bk = FMT == kFmtF16 ? 32 : BK;  // elements per 64-byte k-block
    const bool use_pair = FMT == kFmtTF32 && tc_use_pair();  // pair: TF32 only (slower, kept for A/B)
    CUtensorMap mah, mal, mbh, mbl;
    int rc;
    const int b_box = use_pair ? pair::BNH : BN;
    if ((rc = make_map(&mah, a_hi, M, Kp, batch_a, BM, FMT))) return rc;
    if ((rc = make_map(&mal, a_lo, M, Kp, batch_a, BM, FMT))) return rc;
    if ((rc = make_map(&mbh, b_hi, N, Kp, batch_b, b_box, FMT))) return rc;
    if ((rc = make_map(&mbl, b_lo, N, Kp, batch_b, b_box, FMT))) return rc;
    TcArgs g;
    memset(&g, 0, sizeof g);
    g.M = M; g.N = N; g.K = K;
    g.nkb = (int)((Kp + bk - 1) / bk);
    g.a_batched = batch_a > 1; g.b_batched = batch_b > 1;
    g.C = eps; g.Y = y_or_null; g.ldc = ldc; g.sC = stride_c; g.out_f64 = eps_f64; g.u = u;
    g.a_exp = a_exp; g.b_exp = b_exp;
    if (FMT == kFmtF16) {
        g.a_tiny = a_exp + batch_a * M;  // second block of the split's row info
        g.b_tiny = b_exp + batch_b * N;
        g.fix_count = static_cast<unsigned long long*>(fix_ws);
        g.fix_list = g.fix_count + 8;
        g.fix_cap = (unsigned long long)(fix_ws_bytes / 8 - 8);
    }
    // compensation factors (see header); 2 MMA instructions per 64-byte k-block
    const double mma_rel = 3.0 * 0x1p-23;
    const double j0 = (double)(KCHUNK_KB * 2);
    const double j1 = 2.0 * (double)g.nkb * 2;
    const double comp_split = 1.0 / (1.0 - 1.002 * 0x1p-20);
    const double comp0 = 1.0 / (1.0 - j0 * mma_rel);
    NAO_REQUIRE(j1 * mma_rel < 0.5, "abs-gemm tc: K too large for the acc1 error model");
    const double comp1 = 1.0 / (1.0 - j1 * mma_rel);
    const double s = gamma_const * comp_split * (1.0 + slack) * (1.0 + 0x1p-50);
    g.scale0 = s * comp0;
    g.scale0f = f32_ru(g.scale0);
    // FP16 lo parts carry a 2^10 scale
    g.scale1 = s * comp1 * (FMT == kFmtF16 ? 0x1p-10 : 1.0);
    g.abs_floor = gamma_const * (double)K * 0x1p-120;
    g.scale1f = f32_ru(g.scale1);
    g.abs_floorf = f32_ru(g.abs_floor);
    g.uf = f32_ru(u);
    // excess of the tiny parts <= 2^-24 * 2^15 * 1.001 per tiny element (scaled
    // units); unflagged outputs have it <= 2^-20 of their value
    g.fix_thr = g.scale0 * 0x1p11 * 1.002;
    g.fix_thrf = (float)(g.fix_thr * (1.0 + 0x1p-20));
    int rc_k = NAO_OK;
    if (!eps_f64 && g.nkb <= KCHUNK_KB && !tc_no_short()) {
        static bool attr3_set = false;
        if (!attr3_set) {
            NAO_CHECK_CUDA(cudaFuncSetAttribute(k_absgemm_tc_short<FMT>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                shortk::SMEM_BYTES));
            attr3_set = true;
        }
        const int64_t tiles = ceil_div(N, BN) * ceil_div(M, BM) * batch;
        const unsigned ctas = (unsigned)(tiles < kNumSMs ? tiles : kNumSMs);
        k_absgemm_tc_short<FMT><<<ctas, NUM_THREADS, shortk::SMEM_BYTES, stream>>>(
            mah, mal, mbh, mbl, g, (int)batch);
        NAO_CHECK_LAUNCH();
    } else if (use_pair) {
        static bool attr2_set = false;
        if (!attr2_set) {
            NAO_CHECK_CUDA(cudaFuncSetAttribute(k_absgemm_tc2<FMT>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                pair::SMEM_BYTES));
            attr2_set = true;
        }
        dim3 grid2((unsigned)(2 * ceil_div(N, pair::BN) * ceil_div(M, 2 * pair::BM)), 1,
                   (unsigned)batch);
        k_absgemm_tc2<FMT><<<grid2, pair::NUM_THREADS, pair::SMEM_BYTES, stream>>>(mah, mal, mbh,
                                                                                  mbl, g);
        NAO_CHECK_LAUNCH();
    } else {
    static bool attr_set = false;
    if (!attr_set) {
        NAO_CHECK_CUDA(cudaFuncSetAttribute(k_absgemm_tc<FMT>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            SMEM_BYTES));
#if NAO_TC_REGSPLIT  // the full carveout: room for a commit CTA beside the ring
        NAO_CHECK_CUDA(cudaFuncSetAttribute(k_absgemm_tc<FMT>,
                                            cudaFuncAttributePreferredSharedMemoryCarveout, 100));
#endif
        attr_set = true;
    }
    dim3 grid((unsigned)(ceil_div(N, BN) * ceil_div(M, BM)), 1, (unsigned)batch);
    k_absgemm_tc<FMT><<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(mah, mal, mbh, mbl, g);
    NAO_CHECK_LAUNCH();
    }
    (void)rc_k;
    if (FMT == kFmtF16) {  // exact recompute of flagged outputs, then reset the count
        FixArgs f;
        memset(&f, 0, sizeof f);
        f.A = A; f.B = B;
        f.sA = batch_a > 1 ? M * K : 0;
        f.sB = batch_b > 1 ? N * K : 0;
        f.trans_b = trans_b;
        f.M = M; f.N = N; f.K = K; f.batch = batch;
        f.C = eps; f.Y = y_or_null; f.ldc = ldc; f.sC = stride_c; f.out_f64 = eps_f64;
        f.s = gamma_const * (1.0 + slack) * (1.0 + 0x1p-50);
        f.u = u;
        f.a_tiny = g.a_tiny; f.b_tiny = g.b_tiny;
        f.a_batched = g.a_batched; f.b_batched = g.b_batched;
        f.count = g.fix_count; f.list = g.fix_list; f.cap = g.fix_cap;
        k_absgemm_fix<<<kNumSMs * 4, 256, 0, stream>>>(f);
        NAO_CHECK_LAUNCH();
        NAO_CHECK_CUDA(cudaMemsetAsync(g.fix_count, 0, 8, stream));
    }
    return NAO_OK;
}

}  // namespace tc
}  // namespace nao

using namespace nao;

extern "C" {

int64_t nao_tf32_split_cols(int64_t K) { return (K + 3) / 4 * 4; }

int nao_abs_gemm_tc_kchunk(void) { return nao::tc::KCHUNK; }

int nao_tf32_split(const float* x, float* hi, float* lo, int64_t batch, int64_t rows, int64_t K,
                   int64_t ld, int64_t stride_batch, int transpose, void* stream) {
    NAO_REQUIRE(x && hi && lo, "tf32 split: null pointer");
    NAO_REQUIRE(batch >= 1 && rows >= 0 && K >= 1, "tf32 split: bad shape");
    const int64_t Kp = nao_tf32_split_cols(K);
    const int64_t total = batch * rows * Kp;
    if (total == 0) return NAO_OK;
    if (!transpose && Kp == K && ld == K && stride_batch == rows * K &&
        (reinterpret_cast<uintptr_t>(x) % 16) == 0) {
        const int64_t n4 = total / 4;
        int64_t b4 = (n4 + 255) / 256;
        if (b4 > kNumSMs * 16) b4 = kNumSMs * 16;
        tc::k_split_tf32_vec<<<(unsigned)b4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
            reinterpret_cast<const float4*>(x), reinterpret_cast<float4*>(hi),
            reinterpret_cast<float4*>(lo), n4);
        NAO_CHECK_LAUNCH();
        return NAO_OK;
    }
    int64_t blocks = (total + 255) / 256;
    if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
    tc::k_split_tf32<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        x, hi, lo, batch, rows, K, Kp, ld, stride_batch, transpose);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

// hi/lo operands from nao_tf32_split: A parts [batch_a, M, Kp], B parts [batch_b, N, Kp]
// (batch_a / batch_b either `batch` or 1 = broadcast).
int nao_abs_gemm_tc(const float* a_hi, const float* a_lo, const float* b_hi, const float* b_lo,
                    void* eps, int eps_f64, int64_t batch, int64_t batch_a, int64_t batch_b,
                    int64_t M, int64_t N, int64_t K, int64_t ldc, int64_t stride_c,
                    double gamma_const, const float* y_or_null, double u, double slack,
                    void* stream) {
    return nao::tc::launch_tc<nao::tc::kFmtTF32>(
        a_hi, a_lo, nullptr, b_hi, b_lo, nullptr, eps, eps_f64, batch, batch_a, batch_b, M, N, K,
        ldc, stride_c, gamma_const, y_or_null, u, slack, static_cast<cudaStream_t>(stream));
}

int64_t nao_f16_split_cols(int64_t K) { return (K + 7) / 8 * 8; }

int nao_f16_split(const float* x, void* hi, void* lo, int32_t* row_info, int64_t batch,
                  int64_t rows, int64_t K, int64_t ld, int64_t stride_batch, int transpose,
                  void* stream) {
    NAO_REQUIRE(x && hi && lo && row_info, "f16 split: null pointer");
    int32_t* row_exp = row_info;
    NAO_REQUIRE(batch >= 1 && rows >= 0 && K >= 1, "f16 split: bad shape");
    const int64_t Kp = nao_f16_split_cols(K);
    if (rows == 0) return NAO_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (!transpose) {
        int64_t blocks = ceil_div(batch * rows, 8);
        if (blocks > kNumSMs * 16) blocks = kNumSMs * 16;
        const bool vec = (K % 8) == 0 && (ld % 4) == 0 && (stride_batch % 4) == 0 &&
                         (reinterpret_cast<uintptr_t>(x) % 16) == 0;
        // rows of <= 2048 elements: warp per row (the row stays in L1 for the
        // second pass); longer rows: CTA per row staged in shared memory
        static const int64_t smem_min_k = [] {  // experiment knob
            const char* e = getenv("NAO_SPLIT_SMEM_MIN_K");
            return (int64_t)(e ? atoll(e) : 2049);
        }();
        if (vec && K >= smem_min_k && K * 4 <= 96 * 1024) {
            static bool attr = false;
            if (!attr) {
                NAO_CHECK_CUDA(cudaFuncSetAttribute(tc::k_split_f16_rows_smem,
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    96 * 1024));
                attr = true;
            }
            int64_t nb = batch * rows;
            if (nb > kNumSMs * 32) nb = kNumSMs * 32;
            tc::k_split_f16_rows_smem<<<(unsigned)nb, tc::kSplitThreads, (size_t)K * 4, st>>>(
                x, static_cast<__half*>(hi), static_cast<__half*>(lo), row_exp, batch, rows, K,
                ld, stride_batch);
        } else if (vec)
            tc::k_split_f16_rows<true><<<(unsigned)blocks, 256, 0, st>>>(
                x, static_cast<__half*>(hi), static_cast<__half*>(lo), row_exp, batch, rows, K,
                Kp, ld, stride_batch);
        else
            tc::k_split_f16_rows<false><<<(unsigned)blocks, 256, 0, st>>>(
                x, static_cast<__half*>(hi), static_cast<__half*>(lo), row_exp, batch, rows, K,
                Kp, ld, stride_batch);
    } else {
        int64_t blocks = batch * ceil_div(rows, 32);
        if (blocks > kNumSMs * 8) blocks = kNumSMs * 8;
        tc::k_split_f16_cols<<<(unsigned)blocks, 256, 0, st>>>(
            x, static_cast<__half*>(hi), static_cast<__half*>(lo), row_exp, batch, rows, K, Kp,
            ld, stride_batch);
    }
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

// FP16 parts from nao_f16_split (hi/lo [batch_x, rows, Kp] halves + row exponents)
size_t nao_abs_gemm_tc16_fix_workspace(void) { return (size_t)8 << 20; }

int nao_abs_gemm_tc16(const void* a_hi, const void* a_lo, const int32_t* a_info, const void* b_hi,
                      const void* b_lo, const int32_t* b_info, const float* A, const float* B,
                      int transpose_b, void* eps, int eps_f64, int64_t batch, int64_t batch_a,
                      int64_t batch_b, int64_t M, int64_t N, int64_t K, int64_t ldc,
                      int64_t stride_c, double gamma_const, const float* y_or_null, double u,
                      double slack, void* fix_ws, size_t fix_ws_bytes, void* stream) {
    return nao::tc::launch_tc<nao::tc::kFmtF16>(
        a_hi, a_lo, a_info, b_hi, b_lo, b_info, eps, eps_f64, batch, batch_a, batch_b, M, N, K,
        ldc, stride_c, gamma_const, y_or_null, u, slack, static_cast<cudaStream_t>(stream), A, B,
        transpose_b, fix_ws, fix_ws_bytes);
}

}  // extern "C"
