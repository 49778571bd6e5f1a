// Abs-GEMM bound on the FP32 pipe (north_star (1), FFMA path).
//
//   eps[b,m,n] = c * sum_k |A[b,m,k]| |B[b,k,n]|  (* (1+slack))  [+ u |y[b,m,n]|]
//
// reference: bounds.py:100-111 (FP64 BLAS on |A|,|B|) and the linear branch
// bounds.py:214-217.  Soundness without FP64 FMAs: the inner product runs in
// FP32 with round-toward-+inf FFMA (__fmaf_ru), so every partial sum is >= the
// exact one; each chunk of kFlushK products is then flushed into an FP64
// accumulator.  Over-estimate per chunk <= kFlushK * 2^-23 (3.8e-6 at 32),
// inside the rtol 1e-5 budget, and the FP64 flushes/BLAS differences are
// covered by `slack`.
//
// Also the sequential-profile matmul VALUE kernel (engine.py:157-182) used by
// the bit-exact profile mode: products rounded to FP32, left fold over k (or
// the FP64-fma emulation of the "+fma" profiles).
#include "common.cuh"
#include "profile_fold.cuh"

namespace nao {

constexpr int BM = 128, BN = 128, BK = 16;
constexpr int kFlushK = 32;  // products per FP32 round-up chunk

struct GemmArgs {
    const float* A; const float* B; void* C; const float* Y;
    int64_t M, N, K;
    int64_t lda, ldb, ldc;           // row strides (elements)
    int64_t sA, sB, sC;              // batch strides (0 = broadcast)
    int transpose_b;                 // B stored as [N, K]
    int out_f64;
    double c, slack, u;              // eps = c*acc*(1+slack) [+ u|y|]
};

__global__ void __launch_bounds__(256, 1) k_absgemm_ffma(const __grid_constant__ GemmArgs g) {
    __shared__ __align__(16) float As[2][BK][BM + 4];
    __shared__ __align__(16) float Bs[2][BK][BN + 4];
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    const int64_t b = blockIdx.z;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    const float* A = g.A + b * g.sA;
    const float* B = g.B + b * g.sB;

    float ra[8], rb[8];  // register prefetch of the next tile
    auto load_tile = [&](int64_t k0) {
#pragma unroll
        for (int i = 0; i < 8; i++) {  // A: 128 rows x 16 k
            int idx = t + 256 * i, kk = idx & 15, row = idx >> 4;
            int64_t m = m0 + row, k = k0 + kk;
            ra[i] = (m < g.M && k < g.K) ? fabsf(__ldg(A + m * g.lda + k)) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 8; i++) {
            int idx = t + 256 * i;
            int kk, col;
            if (g.transpose_b) { kk = idx & 15; col = idx >> 4; }
            else { col = idx & 127; kk = idx >> 7; }
            int64_t n = n0 + col, k = k0 + kk;
            float v = 0.f;
            if (n < g.N && k < g.K)
                v = g.transpose_b ? __ldg(B + n * g.ldb + k) : __ldg(B + k * g.ldb + n);
            rb[i] = fabsf(v);
        }
    };
    auto store_tile = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            int idx = t + 256 * i;
            As[buf][idx & 15][idx >> 4] = ra[i];
        }
#pragma unroll
        for (int i = 0; i < 8; i++) {
            int idx = t + 256 * i;
            if (g.transpose_b) Bs[buf][idx & 15][idx >> 4] = rb[i];
            else Bs[buf][idx >> 7][idx & 127] = rb[i];
        }
    };

    float acc[8][8];
    double acc64[8][8];
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) { acc[i][j] = 0.f; acc64[i][j] = 0.0; }

    const int64_t ntiles = (g.K + BK - 1) / BK;
    load_tile(0);
    store_tile(0);
    __syncthreads();
    for (int64_t kt = 0; kt < ntiles; kt++) {
        const int buf = kt & 1;
        if (kt + 1 < ntiles) load_tile((kt + 1) * BK);
#pragma unroll
        for (int kk = 0; kk < BK; kk++) {
            float a[8], bb[8];
            float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8]);
            float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8 + 4]);
            float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 8]);
            float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 8 + 4]);
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
            a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
            bb[0] = b0.x; bb[1] = b0.y; bb[2] = b0.z; bb[3] = b0.w;
            bb[4] = b1.x; bb[5] = b1.y; bb[6] = b1.z; bb[7] = b1.w;
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) acc[i][j] = __fmaf_ru(a[i], bb[j], acc[i][j]);
        }
        if (((kt + 1) * BK) % kFlushK == 0 || kt + 1 == ntiles) {
#pragma unroll
            for (int i = 0; i < 8; i++)
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    acc64[i][j] = __dadd_rn(acc64[i][j], (double)acc[i][j]);
                    acc[i][j] = 0.f;
                }
        }
        if (kt + 1 < ntiles) store_tile(buf ^ 1);
        __syncthreads();
    }
    // epilogue
    const double scale = __dmul_rn(g.c, __dadd_rn(1.0, g.slack));
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int64_t m = m0 + ty * 8 + i;
        if (m >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int64_t n = n0 + tx * 8 + j;
            if (n >= g.N) continue;
            const int64_t o = b * g.sC + m * g.ldc + n;
            double e = __dmul_rn(scale, acc64[i][j]);
            if (g.Y) e = __dadd_rn(e, __dmul_rn(g.u, fabs((double)__ldg(g.Y + o))));
            if (g.out_f64) static_cast<double*>(g.C)[o] = e;
            else static_cast<float*>(g.C)[o] = __double2float_ru(e);
        }
    }
}

// Sequential-profile matmul values: fold_k rn(a*b) (or the FP64-fma emulation).
__global__ void k_matmul_seq(const float* __restrict__ A, const float* __restrict__ B,
                             float* __restrict__ C, int64_t M, int64_t N, int64_t K, int64_t lda,
                             int64_t ldb, int64_t sA, int64_t sB, int64_t sC, int transpose_b,
                             int fma, const Prof prof) {
    const int64_t b = blockIdx.z;
    const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = (int64_t)blockIdx.y;
    if (n >= N || m >= M) return;
    const float* a = A + b * sA + m * lda;
    const float* bp = B + b * sB;
    float acc = 0.f;
    if (!fma && prof.order != NAO_ORDER_SEQUENTIAL) {
        // FP32 products (rounded) reduced over K in the profile's order
        auto at = [&](int64_t k) {
            const float bv = transpose_b ? __ldg(bp + n * ldb + k) : __ldg(bp + k * ldb + n);
            return __fmul_rn(__ldg(a + k), bv);
        };
        C[b * sC + m * N + n] = fold_profile(at, K, prof);
        return;
    }
    for (int64_t k = 0; k < K; k++) {
        const float bv = transpose_b ? __ldg(bp + n * ldb + k) : __ldg(bp + k * ldb + n);
        const float av = __ldg(a + k);
        if (fma) {
            // engine.py:171-180: step = a64*b64 (+ acc64), rounded once to FP32
            const double step = __dmul_rn((double)av, (double)bv);
            acc = (k == 0) ? (float)step : (float)__dadd_rn(step, (double)acc);
        } else {
            const float p = __fmul_rn(av, bv);
            acc = (k == 0) ? p : __fadd_rn(acc, p);
        }
    }
    C[b * sC + m * N + n] = acc;
}

}  // namespace nao

using namespace nao;

extern "C" {

}  // extern "C"

namespace nao {
// NAO_GEMM_FP64: the reference's own arithmetic -- |a||b| exact in FP64, an
// FP64 running sum per output (error <= gamma_K in FP64, ~K 2^-53), then
// const * S * (1 + slack) [+ u|y|].  The API path of matmul_bound / op_bound
// (eps within ~1e-12 of numpy's, reference test tolerances of 1e-9 hold); the
// streaming verifier uses the tensor-core paths.
constexpr int kF64T = 64, kF64K = 16;
__global__ void __launch_bounds__(256) k_absgemm_fp64(const __grid_constant__ GemmArgs g) {
    __shared__ double As[kF64K][kF64T], Bs[kF64K][kF64T];
    const int64_t bz = blockIdx.z;
    const int64_t m0 = (int64_t)blockIdx.y * kF64T, n0 = (int64_t)blockIdx.x * kF64T;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const float* a = g.A + bz * g.sA;
    const float* b = g.B + bz * g.sB;
    double acc[4][4] = {};
    for (int64_t k0 = 0; k0 < g.K; k0 += kF64K) {
        for (int t = threadIdx.x; t < kF64K * kF64T; t += 256) {
            const int kk = t % kF64K, r = t / kF64K;
            const int64_t gm = m0 + r, gk = k0 + kk;
            As[kk][r] = (gm < g.M && gk < g.K) ? fabs((double)__ldg(a + gm * g.lda + gk)) : 0.0;
            const int kb = t / kF64T, c = t % kF64T;
            const int64_t gn = n0 + c, gk2 = k0 + kb;
            float bv = 0.f;
            if (gn < g.N && gk2 < g.K)
                bv = g.transpose_b ? __ldg(b + gn * g.ldb + gk2) : __ldg(b + gk2 * g.ldb + gn);
            Bs[kb][c] = fabs((double)bv);
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < kF64K; kk++) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; i++) { av[i] = As[kk][ty * 4 + i]; bv[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
            for (int i = 0; i < 4; i++)
#pragma unroll
                for (int j = 0; j < 4; j++) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    const double s = __dmul_ru(g.c, 1.0 + g.slack);
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int64_t gm = m0 + ty * 4 + i, gn = n0 + tx * 4 + j;
            if (gm >= g.M || gn >= g.N) continue;
            const int64_t o = bz * g.sC + gm * g.ldc + gn;
            double e = __dmul_ru(s, acc[i][j]);
            if (g.Y) e = __dadd_ru(e, __dmul_rn(g.u, fabs((double)__ldg(g.Y + o))));
            if (g.out_f64) static_cast<double*>(g.C)[o] = e;
            else static_cast<float*>(g.C)[o] = __double2float_ru(e);
        }
}
}  // namespace nao

extern "C" {

int nao_abs_gemm_bound(const float* A, const float* B, void* eps, int eps_f64, int64_t batch,
                       int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                       int64_t stride_a, int64_t stride_b, int64_t stride_c, int transpose_b,
                       double gamma_const, const float* y_or_null, double u, double slack,
                       int path, void* stream) {
    NAO_REQUIRE(A && B && eps, "abs-gemm: null pointer");
    NAO_REQUIRE(batch >= 0 && M >= 0 && N >= 0 && K >= 1, "abs-gemm: bad shape");
    NAO_REQUIRE(path == NAO_GEMM_FFMA_RU || path == NAO_GEMM_FP64,
                "abs-gemm: path %d not available through nao_abs_gemm_bound", path);
    NAO_REQUIRE(batch <= 65535, "abs-gemm: batch too large");
    if (batch == 0 || M == 0 || N == 0) return NAO_OK;
    GemmArgs g;
    g.A = A; g.B = B; g.C = eps; g.Y = y_or_null;
    g.M = M; g.N = N; g.K = K; g.lda = lda; g.ldb = ldb; g.ldc = ldc;
    g.sA = stride_a; g.sB = stride_b; g.sC = stride_c;
    g.transpose_b = transpose_b; g.out_f64 = eps_f64;
    g.c = gamma_const; g.slack = slack; g.u = u;
    if (path == NAO_GEMM_FP64) {
        dim3 grid64((unsigned)ceil_div(N, kF64T), (unsigned)ceil_div(M, kF64T), (unsigned)batch);
        NAO_REQUIRE(grid64.y <= 65535, "abs-gemm: M too large");
        k_absgemm_fp64<<<grid64, 256, 0, static_cast<cudaStream_t>(stream)>>>(g);
        NAO_CHECK_LAUNCH();
        return NAO_OK;
    }
    dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM), (unsigned)batch);
    NAO_REQUIRE(grid.y <= 65535, "abs-gemm: M too large");
    k_absgemm_ffma<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(g);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

int nao_matmul_profile(const float* A, const float* B, float* C, int64_t batch, int64_t M,
                       int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t stride_a,
                       int64_t stride_b, int64_t stride_c, int transpose_b,
                       const nao_profile* profile, void* stream) {
    const int fma = profile ? profile->fma : 0;
    NAO_REQUIRE(A && B && C, "matmul: null pointer");
    NAO_REQUIRE(K >= 1, "cannot reduce an empty axis");
    if (batch == 0 || M == 0 || N == 0) return NAO_OK;
    NAO_REQUIRE(M <= 65535 && batch <= 65535, "matmul_profile: shape too large");
    if (!fma) NAO_CHECK_PROFILE(profile, K);
    dim3 grid((unsigned)ceil_div(N, 128), (unsigned)M, (unsigned)batch);
    k_matmul_seq<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        A, B, C, M, N, K, lda, ldb, stride_a, stride_b, stride_c, transpose_b, fma,
        make_prof(profile));
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

}  // extern "C"
