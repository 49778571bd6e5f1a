// Memory-bound operator values + IEEE-754 bounds (north_star (2)).
//
// FP32 parts follow the reference's default "sequential" DeviceProfile
// bit for bit (engine.py:80-84 left fold per row, engine.py:133-154 FP64
// intrinsic rounded once), and every FP64 bound expression is evaluated in
// the same operation order as bounds.py with explicit __d*_rn intrinsics (no
// FMA contraction).  Only the row sums of the FP64 templates differ in
// association from numpy's pairwise np.sum; the caller's `slack` (>= 4 n 2^-53)
// covers that, so eps_gpu >= eps_ref and eps_gpu <= eps_ref (1 + slack).
//
// Row kernels use one warp per 32 rows: 32x32 tiles are loaded coalesced
// (lane = column), transposed through shared memory, and each lane then
// folds its own row left to right -- 32 independent sequential folds per warp.
#include <cmath>
#include <algorithm>
#include "common.cuh"
#include "unary.cuh"
#include "profile_fold.cuh"

namespace nao {

constexpr int kRowWarps = 4;  // warps per CTA in row kernels

struct RowTile {
    float t[32][33];
};

// eps output: FP64 (API dtype) or FP32 rounded up (streaming pipeline)
__device__ __forceinline__ void store_eps(void* eps, int f64, int64_t i, double v, double slack) {
    double e = __dmul_rn(v, __dadd_rn(1.0, slack));
    if (f64) static_cast<double*>(eps)[i] = e;
    else static_cast<float*>(eps)[i] = __double2float_ru(e);
}

// ----------------------------------------------------------------- softmax

// bounds.py:114-135 over engine.py:185-194 (axis already moved last by the host).
__global__ void __launch_bounds__(32 * kRowWarps) k_softmax(
    const float* __restrict__ x, float* __restrict__ y, void* __restrict__ eps, int eps_f64,
    int64_t rows, int64_t n, double u, double rc, double slack) {
    __shared__ RowTile tiles[kRowWarps][2];
    __shared__ float s_m[kRowWarps][32], s_S[kRowWarps][32];
    __shared__ double s_epsS[kRowWarps][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t r0 = ((int64_t)blockIdx.x * kRowWarps + w) * 32;
    if (r0 >= rows) return;
    const int64_t my_row = r0 + lane;
    const bool row_ok = my_row < rows;
    float (*tx)[33] = tiles[w][0].t;
    float (*te)[33] = tiles[w][1].t;

    // phase 1: row max (order independent, exact)
    float m = -INFINITY;
    for (int64_t c0 = 0; c0 < n; c0 += 32) {
        const int64_t c = c0 + lane;
        for (int rr = 0; rr < 32; rr++) {
            const int64_t r = r0 + rr;
            tx[rr][lane] = (r < rows && c < n) ? __ldg(x + r * n + c) : -INFINITY;
        }
        __syncwarp();
        const int cm = (int)(n - c0 < 32 ? n - c0 : 32);
        for (int cc = 0; cc < cm; cc++) m = fmaxf(m, tx[lane][cc]);
        __syncwarp();
    }
    s_m[w][lane] = m;
    __syncwarp();

    // phase 2: z = x - m, e = fp32(exp64(z)), S = left fold (profile), FP64 sums
    float S = 0.0f;
    double se = 0.0, seps = 0.0;
    const double two_u = __dmul_rn(2.0, u);
    const double m64a = fabs((double)m);
    for (int64_t c0 = 0; c0 < n; c0 += 32) {
        const int64_t c = c0 + lane;
        for (int rr = 0; rr < 32; rr++) {
            const int64_t r = r0 + rr;
            float xv = 0.f, ev = 0.f;
            if (r < rows && c < n) {
                xv = __ldg(x + r * n + c);
                float z = __fsub_rn(xv, s_m[w][rr]);
                ev = (float)exp((double)z);
                y[r * n + c] = ev;  // stash e in the output buffer
            }
            tx[rr][lane] = xv;
            te[rr][lane] = ev;
        }
        __syncwarp();
        const int cm = (int)(n - c0 < 32 ? n - c0 : 32);
        for (int cc = 0; cc < cm; cc++) {
            const float ev = te[lane][cc];
            S = (c0 == 0 && cc == 0) ? ev : __fadd_rn(S, ev);
            const double e64 = (double)ev;
            const double eps_z = __dmul_rn(u, __dadd_rn(fabs((double)tx[lane][cc]), m64a));
            const double eps_e = __dadd_rn(__dmul_rn(e64, eps_z), __dmul_rn(two_u, e64));
            se = __dadd_rn(se, e64);
            seps = __dadd_rn(seps, eps_e);
        }
        __syncwarp();
    }
    s_S[w][lane] = S;
    s_epsS[w][lane] = __dadd_rn(__dmul_rn(rc, se), __dmul_rn(__dadd_rn(rc, 1.0), seps));
    __syncwarp();
    (void)row_ok;

    // phase 3 (coalesced, elementwise): y = e / S ; eps_y
    for (int rr = 0; rr < 32; rr++) {
        const int64_t r = r0 + rr;
        if (r >= rows) break;
        const float Sr = s_S[w][rr];
        const double S64 = (double)Sr, epsS = s_epsS[w][rr];
        const double m64 = fabs((double)s_m[w][rr]);
        const double S2 = __dmul_rn(S64, S64);
        const double invS = __ddiv_rn(1.0, S64), kS2 = __ddiv_rn(epsS, S2);
        for (int64_t c = lane; c < n; c += 32) {
            const int64_t i = r * n + c;
            const float ev = y[i];
            const float xv = __ldg(x + i);
            const float yv = __fdiv_rn(ev, Sr);
            y[i] = yv;
            const double e64 = (double)ev;
            const double eps_z = __dmul_rn(u, __dadd_rn(fabs((double)xv), m64));
            const double eps_e = __dadd_rn(__dmul_rn(e64, eps_z), __dmul_rn(two_u, e64));
            const double t1 = __dmul_rn(eps_e, invS);
            const double t2 = __dmul_rn(e64, kS2);
            const double v = __dadd_rn(__dadd_rn(t1, t2), __dmul_rn(u, fabs((double)yv)));
            store_eps(eps, eps_f64, i, v, slack);
        }
    }
}

// --------------------------------------------------------------- layernorm

// bounds.py:143-169 over engine.py:197-213.
__global__ void __launch_bounds__(32 * kRowWarps) k_layernorm(
    const float* __restrict__ x, float* __restrict__ y, void* __restrict__ eps, int eps_f64,
    int64_t rows, int64_t n, float ln_eps, double u, double rc, double slack) {
    __shared__ RowTile tiles[kRowWarps];
    __shared__ float s_mu[kRowWarps][32], s_sigma[kRowWarps][32];
    __shared__ double s_epsmu[kRowWarps][32], s_epssig[kRowWarps][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t r0 = ((int64_t)blockIdx.x * kRowWarps + w) * 32;
    if (r0 >= rows) return;
    float (*tx)[33] = tiles[w].t;
    const float nf = (float)n;
    const double nd = (double)n;

    // phase 1: mu = fold(x) / float32(n); sum |x| in FP64
    float acc = 0.f;
    double sabs = 0.0;
    for (int64_t c0 = 0; c0 < n; c0 += 32) {
        const int64_t c = c0 + lane;
        for (int rr = 0; rr < 32; rr++) {
            const int64_t r = r0 + rr;
            tx[rr][lane] = (r < rows && c < n) ? __ldg(x + r * n + c) : 0.f;
        }
        __syncwarp();
        const int cm = (int)(n - c0 < 32 ? n - c0 : 32);
        for (int cc = 0; cc < cm; cc++) {
            const float v = tx[lane][cc];
            acc = (c0 == 0 && cc == 0) ? v : __fadd_rn(acc, v);
            sabs = __dadd_rn(sabs, fabs((double)v));
        }
        __syncwarp();
    }
    const float mu = __fdiv_rn(acc, nf);
    const double eps_mu =
        __dadd_rn(__ddiv_rn(__dmul_rn(rc, sabs), nd), __dmul_rn(u, fabs((double)mu)));
    s_mu[w][lane] = mu;
    s_epsmu[w][lane] = eps_mu;
    __syncwarp();

    // phase 2: xc = x - mu, sq = xc*xc, var = fold(sq)/n; FP64 sums of sq and eps_sq
    float acc2 = 0.f;
    double ssq = 0.0, seps = 0.0;
    for (int64_t c0 = 0; c0 < n; c0 += 32) {
        const int64_t c = c0 + lane;
        for (int rr = 0; rr < 32; rr++) {
            const int64_t r = r0 + rr;
            float v = 0.f;
            if (r < rows && c < n) {
                float xc = __fsub_rn(__ldg(x + r * n + c), s_mu[w][rr]);
                v = xc;
            }
            tx[rr][lane] = v;
        }
        __syncwarp();
        const int cm = (int)(n - c0 < 32 ? n - c0 : 32);
        for (int cc = 0; cc < cm; cc++) {
            const float xc = tx[lane][cc];
            const float sq = __fmul_rn(xc, xc);
            acc2 = (c0 == 0 && cc == 0) ? sq : __fadd_rn(acc2, sq);
            const double xc64 = fabs((double)xc), sq64 = (double)sq;
            const double eps_xc = __dadd_rn(eps_mu, __dmul_rn(u, xc64));
            const double eps_sq =
                __dadd_rn(__dmul_rn(__dmul_rn(2.0, xc64), eps_xc), __dmul_rn(u, sq64));
            ssq = __dadd_rn(ssq, sq64);
            seps = __dadd_rn(seps, eps_sq);
        }
        __syncwarp();
    }
    const float var = __fdiv_rn(acc2, nf);
    const float sp = __fadd_rn(var, ln_eps);
    const float sigma = __fsqrt_rn(sp);
    const double eps_ssq = __dadd_rn(__dmul_rn(rc, ssq), __dmul_rn(__dadd_rn(rc, 1.0), seps));
    const double eps_var = __dadd_rn(__ddiv_rn(eps_ssq, nd), __dmul_rn(u, fabs((double)var)));
    const double eps_sp = __dadd_rn(eps_var, __dmul_rn(u, fabs((double)sp)));
    const double sig64 = fabs((double)sigma);
    const double eps_sig = __dadd_rn(__ddiv_rn(eps_sp, __dmul_rn(2.0, sig64)), __dmul_rn(u, sig64));
    s_sigma[w][lane] = sigma;
    s_epssig[w][lane] = eps_sig;
    __syncwarp();

    // phase 3: y = xc / sigma ; eps_y
    for (int rr = 0; rr < 32; rr++) {
        const int64_t r = r0 + rr;
        if (r >= rows) break;
        const float mu_r = s_mu[w][rr], sg = s_sigma[w][rr];
        const double sg64 = fabs((double)sg), sg2 = __dmul_rn(sg64, sg64);
        const double emu = s_epsmu[w][rr], esg = s_epssig[w][rr];
        const double inv_sg = __ddiv_rn(1.0, sg64), k_sg2 = __ddiv_rn(esg, sg2);
        for (int64_t c = lane; c < n; c += 32) {
            const int64_t i = r * n + c;
            const float xc = __fsub_rn(__ldg(x + i), mu_r);
            const float yv = __fdiv_rn(xc, sg);
            y[i] = yv;
            const double xc64 = fabs((double)xc);
            const double eps_xc = __dadd_rn(emu, __dmul_rn(u, xc64));
            const double t1 = __dmul_rn(eps_xc, inv_sg);
            const double t2 = __dmul_rn(xc64, k_sg2);
            const double v = __dadd_rn(__dadd_rn(t1, t2), __dmul_rn(u, fabs((double)yv)));
            store_eps(eps, eps_f64, i, v, slack);
        }
    }
}

// ------------------------------------------------------ sum / mean / max / min

// engine.py:240-251 values, bounds.py:194-208 templates.  kind: 0 sum 1 mean 2 max 3 min
__global__ void __launch_bounds__(32 * kRowWarps) k_reduce_rows(
    const float* __restrict__ x, float* __restrict__ y, void* __restrict__ eps, int eps_f64,
    int64_t rows, int64_t n, int kind, double u, double rc, double slack) {
    __shared__ RowTile tiles[kRowWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t r0 = ((int64_t)blockIdx.x * kRowWarps + w) * 32;
    if (r0 >= rows) return;
    float (*tx)[33] = tiles[w].t;
    float acc = 0.f;
    double sabs = 0.0;
    for (int64_t c0 = 0; c0 < n; c0 += 32) {
        const int64_t c = c0 + lane;
        for (int rr = 0; rr < 32; rr++) {
            const int64_t r = r0 + rr;
            tx[rr][lane] = (r < rows && c < n) ? __ldg(x + r * n + c) : 0.f;
        }
        __syncwarp();
        const int cm = (int)(n - c0 < 32 ? n - c0 : 32);
        for (int cc = 0; cc < cm; cc++) {
            const float v = tx[lane][cc];
            if (c0 == 0 && cc == 0) acc = v;
            else if (kind == 2) acc = fmaxf(acc, v);
            else if (kind == 3) acc = fminf(acc, v);
            else acc = __fadd_rn(acc, v);
            sabs = __dadd_rn(sabs, fabs((double)v));
        }
        __syncwarp();
    }
    const int64_t r = r0 + lane;
    if (r < rows) {
        float out = acc;
        if (kind == 1) out = __fdiv_rn(acc, (float)n);
        y[r] = out;
        double e = 0.0;
        if (kind <= 1) {
            e = __dmul_rn(rc, sabs);
            if (kind == 1) e = __dadd_rn(__ddiv_rn(e, (double)n), __dmul_rn(u, fabs((double)out)));
        }
        if (eps) store_eps(eps, eps_f64, r, e, kind <= 1 ? slack : 0.0);
    }
}

// Thread per row (sum / mean / max / min, sequential profile): the row's
// sequential FP32 fold is the critical path (n dependent FADDs), so every
// row gets its own thread and all rows run at once; the order-free FP64
// sum of |x| for the bound uses four partial accumulators (no dependent
// DADD chain; numpy's own order differs anyway, covered by `slack`).  Rows
// stream through float4 loads (a warp's rows share L1 lines across steps).
__global__ void __launch_bounds__(128) k_reduce_lane(
    const float* __restrict__ x, float* __restrict__ y, void* __restrict__ eps, int eps_f64,
    int64_t rows, int64_t n, int kind, double u, double rc, double slack) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* xr = x + r * n;
    float acc = 0.f;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    auto fold = [&](float v, bool first) {
        if (first) acc = v;
        else if (kind == NAO_RED_MAX) acc = fmaxf(acc, v);
        else if (kind == NAO_RED_MIN) acc = fminf(acc, v);
        else acc = __fadd_rn(acc, v);
    };
    int64_t k = 0;
    if ((n & 3) == 0 && (reinterpret_cast<uintptr_t>(xr) & 15) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(xr);
        const int64_t n4 = n >> 2;
        for (int64_t q = 0; q < n4; q++) {
            const float4 v = __ldg(x4 + q);
            fold(v.x, q == 0); fold(v.y, false); fold(v.z, false); fold(v.w, false);
            s0 = __dadd_rn(s0, fabs((double)v.x)); s1 = __dadd_rn(s1, fabs((double)v.y));
            s2 = __dadd_rn(s2, fabs((double)v.z)); s3 = __dadd_rn(s3, fabs((double)v.w));
        }
        k = n;
    }
    for (; k < n; k++) {
        const float v = __ldg(xr + k);
        fold(v, k == 0);
        s0 = __dadd_rn(s0, fabs((double)v));
    }
    float out = acc;
    if (kind == NAO_RED_MEAN) out = __fdiv_rn(acc, (float)n);
    y[r] = out;
    double e = 0.0;
    if (kind <= NAO_RED_MEAN) {
        const double sabs = __dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3));
        e = __dmul_rn(rc, sabs);
        if (kind == NAO_RED_MEAN) e = __dadd_rn(__ddiv_rn(e, (double)n), __dmul_rn(u, fabs((double)out)));
    }
    if (eps) store_eps(eps, eps_f64, r, e, kind <= NAO_RED_MEAN ? slack : 0.0);
}

// ------------------------------------------------------ elementwise pieces

// engine.py:133-154: FP64 evaluation rounded once to FP32 (csrc/unary.cuh),
// plus the value-ambiguity list and the optional intrinsic bound 2u|y| taken
// at the largest candidate (never below the reference's).
template <int KIND>  // compile-time kind: no per-element switch in the FP64 evaluation
__global__ void k_unary(const float* __restrict__ x, float* __restrict__ y, int64_t n,
                        void* __restrict__ eps, int eps_f64, double eps_scale,
                        unsigned long long* __restrict__ amb, long long amb_cap) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const UnaryOut o = unary_eval(KIND, __ldg(x + i));
        y[i] = o.y;
        if (eps) {
            const double m = fmax(fabs((double)o.lo), fabs((double)o.hi));
            const double e = __dmul_rn(eps_scale, m);
            if (eps_f64) static_cast<double*>(eps)[i] = e;
            else static_cast<float*>(eps)[i] = __double2float_ru(e);
        }
        if (amb && fbits_differ(o.lo, o.hi)) list_push(amb, amb_cap, (unsigned long long)i);
    }
}

// eps = scale * |y|  (single-rounding u|y| / intrinsic 2u|y| templates, bounds.py:196-199)
__global__ void k_scaled_abs(const float* __restrict__ y, void* __restrict__ eps, int eps_f64,
                             int64_t n, double scale) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double e = __dmul_rn(scale, fabs((double)__ldg(y + i)));
        if (eps_f64) static_cast<double*>(eps)[i] = e;
        else static_cast<float*>(eps)[i] = __double2float_ru(e);
    }
}

static int ew_grid(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (int)(b < kNumSMs * 16 ? (b < 1 ? 1 : b) : kNumSMs * 16);
}

static int row_grid(int64_t rows) { return (int)ceil_div(rows, 32 * kRowWarps); }

}  // namespace nao

namespace nao { namespace rowb {
static int launch(const float* x, float* y, void* eps, int eps_f64, int64_t rows, int64_t n,
                  int kind, float ln_eps, double u, double rc, double slack, cudaStream_t st);
static int launch_profile(const float* x, float* y, void* eps, int eps_f64, int64_t rows,
                          int64_t n, int kind, float ln_eps, double u, double rc, double slack,
                          const Prof& prof, cudaStream_t st);
static int softmax_c(const float* x, float* y, void* eps, int eps_f64, int64_t rows, int64_t n,
                     double u, double rc, double slack, cudaStream_t st);
} }

using namespace nao;

extern "C" {

int nao_softmax_bound(const float* x, float* y, void* eps, int eps_f64, int64_t rows, int64_t n,
                      double u, double rc, double slack, const nao_profile* profile,
                      void* stream) {
    NAO_REQUIRE(rows >= 0 && n > 0, "softmax: cannot reduce an empty axis");
    NAO_REQUIRE(x && y && eps, "softmax: null pointer");
    NAO_CHECK_PROFILE(profile, n);
    if (rows == 0) return NAO_OK;
    if (profile && profile->order != NAO_ORDER_SEQUENTIAL)
        return rowb::launch_profile(x, y, eps, eps_f64, rows, n, 0, 0.f, u, rc, slack,
                                    make_prof(profile), static_cast<cudaStream_t>(stream));
    {
        int rc_c = rowb::softmax_c(x, y, eps, eps_f64, rows, n, u, rc, slack,
                                   static_cast<cudaStream_t>(stream));
        if (rc_c >= 0) return rc_c;
        int rc_b = rowb::launch(x, y, eps, eps_f64, rows, n, 0, 0.f, u, rc, slack,
                                static_cast<cudaStream_t>(stream));
        if (rc_b >= 0) return rc_b;
    }
    k_softmax<<<row_grid(rows), 32 * kRowWarps, 0, static_cast<cudaStream_t>(stream)>>>(
        x, y, eps, eps_f64, rows, n, u, rc, slack);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

int nao_layernorm_bound(const float* x, float* y, void* eps, int eps_f64, int64_t rows, int64_t n,
                        float ln_eps, double u, double rc, double slack,
                        const nao_profile* profile, void* stream) {
    NAO_REQUIRE(rows >= 0 && n > 0, "layernorm: cannot reduce an empty axis");
    NAO_REQUIRE(x && y && eps, "layernorm: null pointer");
    NAO_CHECK_PROFILE(profile, n);
    if (rows == 0) return NAO_OK;
    if (profile && profile->order != NAO_ORDER_SEQUENTIAL)
        return rowb::launch_profile(x, y, eps, eps_f64, rows, n, 1, ln_eps, u, rc, slack,
                                    make_prof(profile), static_cast<cudaStream_t>(stream));
    {
        int rc_b = rowb::launch(x, y, eps, eps_f64, rows, n, 1, ln_eps, u, rc, slack,
                                static_cast<cudaStream_t>(stream));
        if (rc_b >= 0) return rc_b;
    }
    k_layernorm<<<row_grid(rows), 32 * kRowWarps, 0, static_cast<cudaStream_t>(stream)>>>(
        x, y, eps, eps_f64, rows, n, ln_eps, u, rc, slack);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

int nao_reduce_bound(const float* x, float* y, void* eps, int eps_f64, int64_t rows, int64_t n,
                     int kind, double u, double rc, double slack, const nao_profile* profile,
                     void* stream) {
    NAO_REQUIRE(rows >= 0 && n > 0, "cannot reduce an empty axis");
    NAO_REQUIRE(kind >= NAO_RED_SUM && kind <= NAO_RED_MIN, "bad reduce kind %d", kind);
    NAO_CHECK_PROFILE(profile, n);
    if (rows == 0) return NAO_OK;
    if (profile && profile->order != NAO_ORDER_SEQUENTIAL && kind <= NAO_RED_MEAN)
        return rowb::launch_profile(x, y, eps, eps_f64, rows, n, 2 + kind, 0.f, u, rc, slack,
                                    make_prof(profile), static_cast<cudaStream_t>(stream));
    // thread per row for many short rows (the q/k RMSNorm means: 65536 / 16384
    // rows of 128, 0.077 / 0.081 -> 0.045 / 0.043 ms); long rows keep the
    // staged-row kernel (a thread per 4096-long row leaves most SMs idle:
    // 0.095 -> 0.205 ms measured)
    if (n <= 1024 && rows >= 4096) {
        k_reduce_lane<<<(unsigned)ceil_div(rows, 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
            x, y, eps, eps_f64, rows, n, kind, u, rc, slack);
        NAO_CHECK_LAUNCH();
        return NAO_OK;
    }
    {
        int rc_b = rowb::launch(x, y, eps, eps_f64, rows, n, 2 + kind, 0.f, u, rc, slack,
                                static_cast<cudaStream_t>(stream));
        if (rc_b >= 0) return rc_b;
    }
    k_reduce_rows<<<row_grid(rows), 32 * kRowWarps, 0, static_cast<cudaStream_t>(stream)>>>(
        x, y, eps, eps_f64, rows, n, kind, u, rc, slack);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

int nao_unary_fp64(const float* x, float* y, int64_t n, int kind, void* eps, int eps_f64,
                   double eps_scale, uint64_t* amb_list, int64_t amb_cap, void* stream) {
    NAO_REQUIRE(kind >= NAO_UN_EXP && kind <= NAO_UN_SILU, "bad unary kind %d", kind);
    NAO_REQUIRE(amb_list == nullptr || amb_cap >= 0, "bad ambiguity list capacity");
    if (n == 0) return NAO_OK;
    auto* amb = reinterpret_cast<unsigned long long*>(amb_list);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int g = ew_grid(n);
    switch (kind) {
        case NAO_UN_EXP: k_unary<NAO_UN_EXP><<<g, 256, 0, st>>>(x, y, n, eps, eps_f64, eps_scale, amb, amb_cap); break;
        case NAO_UN_LOG: k_unary<NAO_UN_LOG><<<g, 256, 0, st>>>(x, y, n, eps, eps_f64, eps_scale, amb, amb_cap); break;
        case NAO_UN_SQRT: k_unary<NAO_UN_SQRT><<<g, 256, 0, st>>>(x, y, n, eps, eps_f64, eps_scale, amb, amb_cap); break;
        case NAO_UN_RSQRT: k_unary<NAO_UN_RSQRT><<<g, 256, 0, st>>>(x, y, n, eps, eps_f64, eps_scale, amb, amb_cap); break;
        case NAO_UN_TANH: k_unary<NAO_UN_TANH><<<g, 256, 0, st>>>(x, y, n, eps, eps_f64, eps_scale, amb, amb_cap); break;
        case NAO_UN_GELU: k_unary<NAO_UN_GELU><<<g, 256, 0, st>>>(x, y, n, eps, eps_f64, eps_scale, amb, amb_cap); break;
        default: k_unary<NAO_UN_SILU><<<g, 256, 0, st>>>(x, y, n, eps, eps_f64, eps_scale, amb, amb_cap); break;
    }
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

int nao_scaled_abs_bound(const float* y, void* eps, int eps_f64, int64_t n, double scale,
                         void* stream) {
    if (n == 0) return NAO_OK;
    k_scaled_abs<<<ew_grid(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(y, eps, eps_f64, n,
                                                                            scale);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

}  // extern "C"

// ------------------------------------------------------------ conv2d lowering
// Patch rows of an NCHW input for the implicit-GEMM conv bound (SURVEY.md 2.3
// extension): col[b, oh*OW + ow, (c*k + kh)*k + kw] = x[b, c, oh*s-p+kh, ow*s-p+kw]
// (0 outside), i.e. torch unfold's K order, written row-major [B, OH*OW, K]
// in one launch (consecutive threads -> consecutive K: coalesced stores; the
// ~k*k-fold re-reads of x hit L1/L2).
namespace nao {
// warp per patch row (oh, ow decoded once), lanes over K; KS = compile-time
// kernel side (1/3/7 cover the configs) so the K decode is multiply-shift
template <int KS>
__global__ void __launch_bounds__(256) k_im2col_rows(const float* __restrict__ x,
                                                     float* __restrict__ col, int C, int H, int W,
                                                     int k_rt, int stride, int pad, int OH, int OW) {
    const int k = KS > 0 ? KS : k_rt;
    const int kk2 = k * k;
    const int b = blockIdx.y;
    const int L = OH * OW, K = C * kk2;
    const float* xb = x + (int64_t)b * C * H * W;
    float* cb = col + (int64_t)b * L * K;
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x >> 5);
    for (int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < L; p += nw) {
        const int oh = p / OW, ow = p - oh * OW;
        const int ih0 = oh * stride - pad, iw0 = ow * stride - pad;
        float* crow = cb + (int64_t)p * K;
        for (int kk = lane; kk < K; kk += 32) {
            const int c = kk / kk2, r = kk - c * kk2;
            const int kh = r / k, kw = r - kh * k;
            const int ih = ih0 + kh, iw = iw0 + kw;
            float v = 0.f;
            if ((unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W)
                v = __ldg(xb + ((int64_t)c * H + ih) * W + iw);
            crow[kk] = v;
        }
    }
}
}  // namespace nao

extern "C" int nao_im2col_rows(const float* x, float* col, int64_t batch, int64_t C, int64_t H,
                               int64_t W, int64_t k, int64_t stride, int64_t pad, void* stream) {
    NAO_REQUIRE(batch >= 0 && C > 0 && H > 0 && W > 0 && k > 0 && stride > 0 && pad >= 0,
                "im2col: bad geometry");
    NAO_REQUIRE(batch <= 65535, "im2col: batch %lld > 65535", (long long)batch);
    const int64_t OH = (H + 2 * pad - k) / stride + 1, OW = (W + 2 * pad - k) / stride + 1;
    NAO_REQUIRE(OH > 0 && OW > 0, "im2col: empty output");
    NAO_REQUIRE(OH * OW * C * k * k < (int64_t)1 << 31, "im2col: per-sample patch matrix too large");
    if (batch == 0) return NAO_OK;
    int64_t gx = (OH * OW + 7) / 8;  // 8 warps (rows) per CTA
    const int64_t cap = (int64_t)nao::kNumSMs * 8 / batch + 1;
    if (gx > cap) gx = cap;
    const dim3 grid((unsigned)gx, (unsigned)batch);
    auto st = static_cast<cudaStream_t>(stream);
#define NAO_IM2COL(KS) nao::k_im2col_rows<KS><<<grid, 256, 0, st>>>( \
        x, col, (int)C, (int)H, (int)W, (int)k, (int)stride, (int)pad, (int)OH, (int)OW)
    if (k == 1) NAO_IM2COL(1);
    else if (k == 3) NAO_IM2COL(3);
    else if (k == 7) NAO_IM2COL(7);
    else NAO_IM2COL(0);
#undef NAO_IM2COL
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

// ------------------------------------------------------------ fault / drift hook
// Mirrors the reference's additive `inject` hook on node outputs
// (engine.py:325-351): the claimed value of element i is y_i moved by
// +-1 ulp with probability ~1/period (hash of (seed, i)) -- honest
// cross-device drift -- plus an optional relative fault `scale` on every
// element with (hash % fault_period == 0).
namespace nao {
__device__ __forceinline__ float drift_one(float v, int64_t i, uint32_t seed, uint32_t period,
                                           float fault_scale, uint32_t fault_period) {
    uint32_t h = (uint32_t)i * 0x9E3779B1u ^ seed;
    h ^= h >> 16; h *= 0x85EBCA6Bu; h ^= h >> 13; h *= 0xC2B2AE35u; h ^= h >> 16;
    // h % period without an integer division when period is a power of two
    const uint32_t hm = (period & (period - 1)) == 0 ? (h & (period - 1)) : (period ? h % period : 1u);
    if (period && hm == 0 && v != 0.0f && isfinite(v))
        v = __int_as_float(__float_as_int(v) + ((h >> 20) & 1 ? 1 : -1));
    if (fault_period && ((h >> 8) % fault_period) == 0) v = v * (1.0f + fault_scale);
    return v;
}

// 4 float4 per thread per step (16-byte aligned y/out; 64 B in flight per
// thread keeps HBM busy), scalar tail.  period = fault_period = 0 is a pure
// copy: the proposer harness's claim of a deterministic node.
template <bool COPY>
__global__ void __launch_bounds__(256) k_inject_drift(const float* __restrict__ y,
                                                      float* __restrict__ out, int64_t n,
                                                      uint32_t seed, uint32_t period,
                                                      float fault_scale, uint32_t fault_period) {
    const int64_t nv = n >> 2;
    const float4* y4 = reinterpret_cast<const float4*>(y);
    float4* o4 = reinterpret_cast<float4*>(out);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; v + 3 * stride < nv; v += 4 * stride) {
        float4 a[4];
#pragma unroll
        for (int u = 0; u < 4; u++) a[u] = __ldg(y4 + v + u * stride);
#pragma unroll
        for (int u = 0; u < 4; u++) {
            if (!COPY) {
                const int64_t i = 4 * (v + u * stride);
                a[u].x = drift_one(a[u].x, i, seed, period, fault_scale, fault_period);
                a[u].y = drift_one(a[u].y, i + 1, seed, period, fault_scale, fault_period);
                a[u].z = drift_one(a[u].z, i + 2, seed, period, fault_scale, fault_period);
                a[u].w = drift_one(a[u].w, i + 3, seed, period, fault_scale, fault_period);
            }
            o4[v + u * stride] = a[u];  // default policy: the claim is read next
        }
    }
    for (; v < nv; v += stride) {
        float4 a = __ldg(y4 + v);
        if (!COPY) {
            const int64_t i = 4 * v;
            a.x = drift_one(a.x, i, seed, period, fault_scale, fault_period);
            a.y = drift_one(a.y, i + 1, seed, period, fault_scale, fault_period);
            a.z = drift_one(a.z, i + 2, seed, period, fault_scale, fault_period);
            a.w = drift_one(a.w, i + 3, seed, period, fault_scale, fault_period);
        }
        o4[v] = a;
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
        const int64_t i = (nv << 2) + threadIdx.x;
        out[i] = drift_one(__ldg(y + i), i, seed, period, fault_scale, fault_period);
    }
}
}  // namespace nao

extern "C" int nao_inject_drift(const float* y, float* out, int64_t n, uint32_t seed,
                                uint32_t period, float fault_scale, uint32_t fault_period,
                                void* stream) {
    if (n == 0) return NAO_OK;
    NAO_REQUIRE((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(out)) % 16 == 0,
                "y/out must be 16-byte aligned");
    // one resident wave (8 CTAs of 256 per SM), 4 float4 in flight per thread
    const int64_t want = ((n >> 2) + 255) / 256;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, nao::kNumSMs * 8));
    if (period == 0 && fault_period == 0)
        nao::k_inject_drift<true><<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
            y, out, n, seed, period, fault_scale, fault_period);
    else
        nao::k_inject_drift<false><<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
            y, out, n, seed, period, fault_scale, fault_period);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

// ------------------------------------------------------------------------
// Row kernels, design B (few rows / long rows): a CTA stages R whole rows in
// shared memory (one DRAM read of x), one thread per row runs the profile's
// left fold (the only serial part), and every order-free piece -- max, FP64
// template sums, the elementwise value/bound epilogue -- is spread over all
// 256 threads.  DRAM traffic = read x + write y + write eps.
namespace nao {
namespace rowb {

constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (kThreads / 32) ? red[threadIdx.x] : 0.0;
        t = warp_sum(t);
    }
    if (threadIdx.x == 0) red[0] = t;
    __syncthreads();
    const double r = red[0];
    __syncthreads();
    return r;
}

// kind: 0 softmax, 1 layernorm, 2 sum, 3 mean, 4 max, 5 min
__global__ void __launch_bounds__(kThreads) k_rows_smem(
    const float* __restrict__ x, float* __restrict__ y, void* __restrict__ eps, int eps_f64,
    int64_t rows, int64_t n, int R, int kind, float ln_eps, double u, double rc, double slack,
    const Prof prof) {
    extern __shared__ __align__(16) float sx[];       // [R][n] x, then [R][n] e (softmax)
    __shared__ double red[kThreads / 32];
    __shared__ float s_a[32], s_b[32];                // per-row FP32 scalars
    __shared__ double s_d0[32], s_d1[32];             // per-row FP64 scalars
    const int64_t r0 = (int64_t)blockIdx.x * R;
    const int nr = (int)((rows - r0) < R ? (rows - r0) : R);
    float* se = sx + (size_t)R * n;
    // stage rows (coalesced, vectorised when aligned)
    const int64_t total = (int64_t)nr * n;
    const float* xb = x + r0 * n;
    if (((reinterpret_cast<uintptr_t>(xb) | (n * 4)) & 15) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(xb);
        float4* s4 = reinterpret_cast<float4*>(sx);
        for (int64_t i = threadIdx.x; i < total / 4; i += kThreads) s4[i] = __ldg(x4 + i);
    } else {
        for (int64_t i = threadIdx.x; i < total; i += kThreads) sx[i] = __ldg(xb + i);
    }
    __syncthreads();
    const double two_u = __dmul_rn(2.0, u);
    for (int r = 0; r < nr; r++) {
        const float* row = sx + (size_t)r * n;
        if (kind == 0) {  // ---- softmax: max (order free), e = fp32(exp64(x-m))
            float m = -INFINITY;
            for (int64_t c = threadIdx.x; c < n; c += kThreads) m = fmaxf(m, row[c]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = (double)m;
            __syncthreads();
            if (threadIdx.x == 0) {
                float mm = -INFINITY;
                for (int i = 0; i < kThreads / 32; i++) mm = fmaxf(mm, (float)red[i]);
                s_a[r] = mm;
                s_b[r] = mm;  // kept for the epilogue (s_a is reused by the fold)
            }
            __syncthreads();
            m = s_a[r];
            const double m64a = fabs((double)m);
            double se_part = 0.0, seps_part = 0.0;
            float* erow = se + (size_t)r * n;
            for (int64_t c = threadIdx.x; c < n; c += kThreads) {
                const float xv = row[c];
                const float ev = (float)exp((double)__fsub_rn(xv, m));
                erow[c] = ev;
                const double e64 = (double)ev;
                const double eps_z = __dmul_rn(u, __dadd_rn(fabs((double)xv), m64a));
                se_part = __dadd_rn(se_part, e64);
                seps_part = __dadd_rn(seps_part, __dadd_rn(__dmul_rn(e64, eps_z), __dmul_rn(two_u, e64)));
            }
            const double s_e = block_sum(se_part, red);
            const double s_eps = block_sum(seps_part, red);
            if (threadIdx.x == 0) s_d0[r] = __dadd_rn(__dmul_rn(rc, s_e), __dmul_rn(__dadd_rn(rc, 1.0), s_eps));
        } else if (kind == 1) {  // ---- layernorm: FP64 sum |x| (order free)
            double sa = 0.0;
            for (int64_t c = threadIdx.x; c < n; c += kThreads) sa = __dadd_rn(sa, fabs((double)row[c]));
            sa = block_sum(sa, red);
            if (threadIdx.x == 0) s_d0[r] = sa;
        } else if (kind <= 3) {  // sum / mean: order-free FP64 sum |x| by the whole CTA
            double sa = 0.0;
            for (int64_t c = threadIdx.x; c < n; c += kThreads) sa = __dadd_rn(sa, fabs((double)row[c]));
            sa = block_sum(sa, red);
            if (threadIdx.x == 0) s_d0[r] = sa;
        }
    }
    __syncthreads();
    // serial profile folds: thread r owns row r
    if (threadIdx.x < nr && prof.order != NAO_ORDER_SEQUENTIAL) {
        // another device profile's order (engine.py:95-113): generic fold
        const int r = threadIdx.x;
        const float* row = (kind == 0 ? se : sx) + (size_t)r * n;
        const float acc = fold_profile([&](int64_t k) { return row[k]; }, n, prof);
        if (kind == 1) {  // mu, then the profile fold over sq = (x - mu)^2
            const float mu = __fdiv_rn(acc, (float)n);
            s_a[r] = mu;
            s_b[r] = fold_profile([&](int64_t k) {
                const float xc = __fsub_rn(row[k], mu);
                return __fmul_rn(xc, xc);
            }, n, prof);
        } else {
            s_a[r] = acc;
        }
    } else if (threadIdx.x < nr) {
        const int r = threadIdx.x;
        const float* row = (kind == 0 ? se : sx) + (size_t)r * n;
        float acc = row[0];
        if (kind == 4) { for (int64_t c = 1; c < n; c++) acc = fmaxf(acc, row[c]); }
        else if (kind == 5) { for (int64_t c = 1; c < n; c++) acc = fminf(acc, row[c]); }
        else if (kind >= 2 && (n & 3) == 0 && n >= 8) {
            // sum / mean left fold from 16-byte smem loads, the next 8 in flight
            const float4* r4 = reinterpret_cast<const float4*>(row);
            const int64_t n4 = n >> 2;
            float4 v = r4[0];
            acc = __fadd_rn(__fadd_rn(__fadd_rn(v.x, v.y), v.z), v.w);
            int64_t c = 1;
            for (; c + 8 <= n4; c += 8) {
                float4 b[8];
#pragma unroll
                for (int k = 0; k < 8; k++) b[k] = r4[c + k];
#pragma unroll
                for (int k = 0; k < 8; k++)
                    acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, b[k].x), b[k].y), b[k].z),
                                    b[k].w);
            }
            for (; c < n4; c++) {
                v = r4[c];
                acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, v.x), v.y), v.z), v.w);
            }
        } else {
#pragma unroll 8
            for (int64_t c = 1; c < n; c++) acc = __fadd_rn(acc, row[c]);
        }
        if (kind == 1) {  // mu, then the second fold over sq = (x - mu)^2
            const float mu = __fdiv_rn(acc, (float)n);
            float xc0 = __fsub_rn(row[0], mu);
            float acc2 = __fmul_rn(xc0, xc0);
#pragma unroll 8
            for (int64_t c = 1; c < n; c++) {
                const float xc = __fsub_rn(row[c], mu);
                acc2 = __fadd_rn(acc2, __fmul_rn(xc, xc));
            }
            s_a[r] = mu;
            s_b[r] = acc2;
        } else {
            s_a[r] = acc;
        }
    }
    __syncthreads();
    if (kind >= 2) {  // reductions: one output per row
        if (threadIdx.x < nr) {
            const int r = threadIdx.x;
            float out = s_a[r];
            if (kind == 3) out = __fdiv_rn(out, (float)n);
            y[r0 + r] = out;
            double e = 0.0;
            if (kind <= 3) {
                e = __dmul_rn(rc, s_d0[r]);
                if (kind == 3) e = __dadd_rn(__ddiv_rn(e, (double)n), __dmul_rn(u, fabs((double)out)));
            }
            if (eps) store_eps(eps, eps_f64, r0 + r, e, kind <= 3 ? slack : 0.0);
        }
        return;
    }
    const double nd = (double)n;
    for (int r = 0; r < nr; r++) {
        const float* row = sx + (size_t)r * n;
        float* yrow = y + (r0 + r) * n;
        const int64_t ob = (r0 + r) * n;
        if (kind == 0) {
            const float S = s_a[r];
            const double S64 = (double)S, S2 = __dmul_rn(S64, S64), epsS = s_d0[r];
            // divisions by per-row constants as reciprocal multiplies: <= 2 ulp FP64,
            // covered by `slack` (>= 2^-50)
            const double invS = __ddiv_rn(1.0, S64), kS2 = __ddiv_rn(epsS, S2);
            const float* erow = se + (size_t)r * n;
            const double m64a = fabs((double)s_b[r]);
            for (int64_t c = threadIdx.x; c < n; c += kThreads) {
                const float ev = erow[c];
                const float yv = __fdiv_rn(ev, S);
                yrow[c] = yv;
                const double e64 = (double)ev;
                const double eps_z = __dmul_rn(u, __dadd_rn(fabs((double)row[c]), m64a));
                const double eps_e = __dadd_rn(__dmul_rn(e64, eps_z), __dmul_rn(two_u, e64));
                const double v = __dadd_rn(__dadd_rn(__dmul_rn(eps_e, invS), __dmul_rn(e64, kS2)),
                                           __dmul_rn(u, fabs((double)yv)));
                store_eps(eps, eps_f64, ob + c, v, slack);
            }
        } else {
            // layernorm: FP64 chain (bounds.py:159-168), order-free sums over sq, eps_sq
            const float mu = s_a[r];
            const double eps_mu = __dadd_rn(__ddiv_rn(__dmul_rn(rc, s_d0[r]), nd),
                                            __dmul_rn(u, fabs((double)mu)));
            double ssq = 0.0, seps = 0.0;
            for (int64_t c = threadIdx.x; c < n; c += kThreads) {
                const float xc = __fsub_rn(row[c], mu);
                const float sq = __fmul_rn(xc, xc);
                const double xc64 = fabs((double)xc), sq64 = (double)sq;
                const double eps_xc = __dadd_rn(eps_mu, __dmul_rn(u, xc64));
                ssq = __dadd_rn(ssq, sq64);
                seps = __dadd_rn(seps, __dadd_rn(__dmul_rn(__dmul_rn(2.0, xc64), eps_xc),
                                                 __dmul_rn(u, sq64)));
            }
            ssq = block_sum(ssq, red);
            seps = block_sum(seps, red);
            const float var = __fdiv_rn(s_b[r], (float)n);
            const float sp = __fadd_rn(var, ln_eps);
            const float sigma = __fsqrt_rn(sp);
            const double eps_ssq = __dadd_rn(__dmul_rn(rc, ssq), __dmul_rn(__dadd_rn(rc, 1.0), seps));
            const double eps_var = __dadd_rn(__ddiv_rn(eps_ssq, nd), __dmul_rn(u, fabs((double)var)));
            const double eps_sp = __dadd_rn(eps_var, __dmul_rn(u, fabs((double)sp)));
            const double sg64 = fabs((double)sigma), sg2 = __dmul_rn(sg64, sg64);
            const double esg = __dadd_rn(__ddiv_rn(eps_sp, __dmul_rn(2.0, sg64)), __dmul_rn(u, sg64));
            const double inv_sg = __ddiv_rn(1.0, sg64), k_sg2 = __ddiv_rn(esg, sg2);
            for (int64_t c = threadIdx.x; c < n; c += kThreads) {
                const float xc = __fsub_rn(row[c], mu);
                const float yv = __fdiv_rn(xc, sigma);
                yrow[c] = yv;
                const double xc64 = fabs((double)xc);
                const double eps_xc = __dadd_rn(eps_mu, __dmul_rn(u, xc64));
                const double v = __dadd_rn(__dadd_rn(__dmul_rn(eps_xc, inv_sg),
                                                     __dmul_rn(xc64, k_sg2)),
                                           __dmul_rn(u, fabs((double)yv)));
                store_eps(eps, eps_f64, ob + c, v, slack);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Rows too long for shared memory (layernorm / sum / mean / max / min with
// n > 24576, e.g. GroupNorm rows C/G*H*W of a 64x64 UNet level): one CTA per
// row streams the row through a double-buffered smem tile.  While thread 0
// runs the profile's serial FP32 fold over tile t (the critical path: one
// dependent FADD per element), warps 1-7 load tile t+1 and accumulate the
// order-free FP64 template sums.  Layernorm makes a second pass for the fold
// over sq = (x - mu)^2 (the loaders write sq into the tile) and a third,
// all-thread elementwise pass for y and eps.  DRAM traffic = 2-3 reads of x +
// writes of y and eps; time ~ passes x n x FADD latency per row, rows in parallel.
constexpr int kStreamTile = 8192;  // floats per tile (2 tiles = 64 KB smem)

__device__ __forceinline__ float fold_tile(float acc, const float* t, int L, bool first, int kind) {
    int c = 0;
    if (first) { acc = t[0]; c = 1; }
    if (kind >= 4) {
        for (; c < L; c++) acc = kind == 4 ? fmaxf(acc, t[c]) : fminf(acc, t[c]);
        return acc;
    }
    for (; c < L && (c & 3); c++) acc = __fadd_rn(acc, t[c]);
    const float4* t4 = reinterpret_cast<const float4*>(t + c);
    const int n4 = (L - c) >> 2;
    int k = 0;
    for (; k + 8 <= n4; k += 8) {
        float4 b[8];
#pragma unroll
        for (int j = 0; j < 8; j++) b[j] = t4[k + j];
#pragma unroll
        for (int j = 0; j < 8; j++)
            acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, b[j].x), b[j].y), b[j].z), b[j].w);
    }
    for (; k < n4; k++) {
        const float4 v = t4[k];
        acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, v.x), v.y), v.z), v.w);
    }
    for (c += 4 * n4; c < L; c++) acc = __fadd_rn(acc, t[c]);
    return acc;
}

// kind: 1 layernorm, 2 sum, 3 mean, 4 max, 5 min
__global__ void __launch_bounds__(kThreads) k_rows_stream(
    const float* __restrict__ x, float* __restrict__ y, void* __restrict__ eps, int eps_f64,
    int64_t rows, int64_t n, int kind, float ln_eps, double u, double rc, double slack) {
    extern __shared__ __align__(16) float sbuf[];     // [2][kStreamTile]
    __shared__ double red[kThreads / 32];
    __shared__ float s_fold;
    const int64_t r = blockIdx.x;
    const float* xr = x + r * n;
    const int ntiles = (int)((n + kStreamTile - 1) / kStreamTile);
    const bool vec = ((reinterpret_cast<uintptr_t>(xr) | (uintptr_t)(n * 4)) & 15) == 0;
    const double nd = (double)n;
    float mu = 0.f;
    double eps_mu = 0.0, ssq = 0.0, seps = 0.0, sabs = 0.0;

    // loader: tile t -> buf, transformed (pass 0: x, pass 1: sq), FP64 sums on the way
    auto load = [&](int t, int pass, int tid0, int nthr) {
        float* b = sbuf + (t & 1) * kStreamTile;
        const int64_t base = (int64_t)t * kStreamTile;
        const int L = (int)(n - base < kStreamTile ? n - base : kStreamTile);
        auto one = [&](float v) -> float {
            if (pass == 0) {
                if (kind <= 3) sabs = __dadd_rn(sabs, fabs((double)v));
                return v;
            }
            const float xc = __fsub_rn(v, mu);
            const float sq = __fmul_rn(xc, xc);
            const double xc64 = fabs((double)xc), sq64 = (double)sq;
            const double eps_xc = __dadd_rn(eps_mu, __dmul_rn(u, xc64));
            ssq = __dadd_rn(ssq, sq64);
            seps = __dadd_rn(seps, __dadd_rn(__dmul_rn(__dmul_rn(2.0, xc64), eps_xc),
                                             __dmul_rn(u, sq64)));
            return sq;
        };
        if (vec) {
            const float4* s4 = reinterpret_cast<const float4*>(xr + base);
            float4* b4 = reinterpret_cast<float4*>(b);
            for (int i = tid0; i < (L >> 2); i += nthr) {
                float4 v = __ldg(s4 + i);
                v.x = one(v.x); v.y = one(v.y); v.z = one(v.z); v.w = one(v.w);
                b4[i] = v;
            }
            for (int i = 4 * (L >> 2) + tid0; i < L; i += nthr) b[i] = one(__ldg(xr + base + i));
        } else {
            for (int i = tid0; i < L; i += nthr) b[i] = one(__ldg(xr + base + i));
        }
    };

    const int passes = kind == 1 ? 2 : 1;
    for (int pass = 0; pass < passes; pass++) {
        float acc = 0.f;
        load(0, pass, threadIdx.x, kThreads);
        __syncthreads();
        for (int t = 0; t < ntiles; t++) {
            if (threadIdx.x == 0) {
                const int64_t base = (int64_t)t * kStreamTile;
                const int L = (int)(n - base < kStreamTile ? n - base : kStreamTile);
                acc = fold_tile(acc, sbuf + (t & 1) * kStreamTile, L, t == 0, kind);
            } else if (threadIdx.x >= 32 && t + 1 < ntiles) {
                load(t + 1, pass, threadIdx.x - 32, kThreads - 32);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) s_fold = acc;
        if (pass == 0) {
            sabs = block_sum(sabs, red);  // (syncs; publishes s_fold)
            if (kind == 1) {
                mu = __fdiv_rn(s_fold, (float)n);
                eps_mu = __dadd_rn(__ddiv_rn(__dmul_rn(rc, sabs), nd), __dmul_rn(u, fabs((double)mu)));
            }
        } else {
            ssq = block_sum(ssq, red);
            seps = block_sum(seps, red);
        }
    }
    if (kind >= 2) {
        if (threadIdx.x == 0) {
            float out = s_fold;
            if (kind == 3) out = __fdiv_rn(out, (float)n);
            y[r] = out;
            double e = 0.0;
            if (kind <= 3) {
                e = __dmul_rn(rc, sabs);
                if (kind == 3) e = __dadd_rn(__ddiv_rn(e, nd), __dmul_rn(u, fabs((double)out)));
            }
            if (eps) store_eps(eps, eps_f64, r, e, kind <= 3 ? slack : 0.0);
        }
        return;
    }
    // layernorm epilogue (bounds.py:159-168), same expressions as k_rows_smem
    const float var = __fdiv_rn(s_fold, (float)n);
    const float sp = __fadd_rn(var, ln_eps);
    const float sigma = __fsqrt_rn(sp);
    const double eps_ssq = __dadd_rn(__dmul_rn(rc, ssq), __dmul_rn(__dadd_rn(rc, 1.0), seps));
    const double eps_var = __dadd_rn(__ddiv_rn(eps_ssq, nd), __dmul_rn(u, fabs((double)var)));
    const double eps_sp = __dadd_rn(eps_var, __dmul_rn(u, fabs((double)sp)));
    const double sg64 = fabs((double)sigma), sg2 = __dmul_rn(sg64, sg64);
    const double esg = __dadd_rn(__ddiv_rn(eps_sp, __dmul_rn(2.0, sg64)), __dmul_rn(u, sg64));
    const double inv_sg = __ddiv_rn(1.0, sg64), k_sg2 = __ddiv_rn(esg, sg2);
    float* yr = y + r * n;
    for (int64_t c = threadIdx.x; c < n; c += kThreads) {
        const float xc = __fsub_rn(__ldg(xr + c), mu);
        const float yv = __fdiv_rn(xc, sigma);
        yr[c] = yv;
        const double xc64 = fabs((double)xc);
        const double eps_xc = __dadd_rn(eps_mu, __dmul_rn(u, xc64));
        const double v = __dadd_rn(__dadd_rn(__dmul_rn(eps_xc, inv_sg), __dmul_rn(xc64, k_sg2)),
                                   __dmul_rn(u, fabs((double)yv)));
        store_eps(eps, eps_f64, r * n + c, v, slack);
    }
}

// ---------------------------------------------------------------------------
// Softmax, design C (many long rows): three launches, each at full occupancy.
//   K1 warp per row : m = max, e = fp32(exp64(x - m)) -> y, FP64 eps sums
//   K2 lane per row : the profile's sequential FP32 fold S of e (32 rows per
//                     warp instruction: the only serial part, no idle CTA)
//   K3 warp per row : y = e / S and the eps epilogue
// Per-row stats (epsS f64, m f32, S f32) live in the first 16 bytes of the
// row's own eps slot until K3 reads them (all lanes, then __syncwarp) and
// overwrites that slot with the bound.
struct RowStats { uint32_t w[4]; };  // [0..1] epsS bits, [2] m bits, [3] S bits
__device__ __forceinline__ uint32_t* stats_ptr(void* eps, int f64, int64_t r, int64_t n) {
    return reinterpret_cast<uint32_t*>(static_cast<char*>(eps) + (size_t)r * n * (f64 ? 8 : 4));
}

template <bool VEC>
__global__ void __launch_bounds__(256) k_smc_rows(const float* __restrict__ x, float* __restrict__ y,
                                                  void* __restrict__ eps, int eps_f64, int64_t rows,
                                                  int64_t n, double u, double rc) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const double two_u = __dmul_rn(2.0, u);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
         r += nwarps) {
        const float* xr = x + r * n;
        float* er = y + r * n;
        float m = -INFINITY;
        if (VEC) {
            const float4* x4 = reinterpret_cast<const float4*>(xr);
            for (int64_t c = lane; c < (n >> 2); c += 32) {
                const float4 v = __ldg(x4 + c);
                m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
            }
        } else {
            for (int64_t c = lane; c < n; c += 32) m = fmaxf(m, __ldg(xr + c));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        // sum eps_e = sum e (u(|x| + |m|) + 2u) = u sum e|x| + (u|m| + 2u) sum e:
        // two order-free FP64 sums (re-association covered by `slack`)
        double se = 0.0, sex = 0.0;
        auto one = [&](float xv) -> float {
            const float ev = (float)exp((double)__fsub_rn(xv, m));
            const double e64 = (double)ev;
            se = __dadd_rn(se, e64);
            sex = __fma_rn(e64, fabs((double)xv), sex);
            return ev;
        };
        if (VEC) {
            const float4* x4 = reinterpret_cast<const float4*>(xr);
            float4* e4 = reinterpret_cast<float4*>(er);
            for (int64_t c = lane; c < (n >> 2); c += 32) {
                const float4 v = __ldg(x4 + c);
                float4 e;
                e.x = one(v.x); e.y = one(v.y); e.z = one(v.z); e.w = one(v.w);
                e4[c] = e;
            }
        } else {
            for (int64_t c = lane; c < n; c += 32) er[c] = one(__ldg(xr + c));
        }
        se = warp_sum(se);
        sex = warp_sum(sex);
        if (lane == 0) {
            const double um2 = __dadd_rn(__dmul_rn(u, fabs((double)m)), two_u);
            const double seps = __dadd_rn(__dmul_rn(u, sex), __dmul_rn(um2, se));
            const double epsS = __dadd_rn(__dmul_rn(rc, se), __dmul_rn(__dadd_rn(rc, 1.0), seps));
            uint32_t* st = stats_ptr(eps, eps_f64, r, n);
            const unsigned long long b = (unsigned long long)__double_as_longlong(epsS);
            st[0] = (uint32_t)b;
            st[1] = (uint32_t)(b >> 32);
            st[2] = __float_as_uint(m);
        }
    }
}

// lane per row: S = (((e0 + e1) + e2) + ...), the sequential profile's left fold
template <bool VEC>
__global__ void __launch_bounds__(128) k_smc_fold(const float* __restrict__ e, void* __restrict__ eps,
                                                  int eps_f64, int64_t rows, int64_t n) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const float* er = e + r * n;
    float acc;
    if (VEC) {
        const float4* e4 = reinterpret_cast<const float4*>(er);
        const int64_t n4 = n >> 2;
        float4 v = e4[0];
        acc = __fadd_rn(__fadd_rn(__fadd_rn(v.x, v.y), v.z), v.w);
        // batches of 8 float4: the next batch is in flight while this one folds
        constexpr int NB = 8;
        float4 cur[NB], nxt[NB];
        int64_t c = 1;
        const int64_t nb = (n4 - 1) / NB;  // full batches after element group 0
#pragma unroll
        for (int k = 0; k < NB; k++) cur[k] = nb > 0 ? e4[c + k] : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t b = 0; b < nb; b++) {
            const int64_t cn = c + NB;
            if (b + 1 < nb) {
#pragma unroll
                for (int k = 0; k < NB; k++) nxt[k] = e4[cn + k];
            }
#pragma unroll
            for (int k = 0; k < NB; k++)
                acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, cur[k].x), cur[k].y), cur[k].z),
                                cur[k].w);
#pragma unroll
            for (int k = 0; k < NB; k++) cur[k] = nxt[k];
            c = cn;
        }
        for (; c < n4; c++) {
            const float4 a = e4[c];
            acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, a.x), a.y), a.z), a.w);
        }
    } else {
        acc = er[0];
        for (int64_t c = 1; c < n; c++) acc = __fadd_rn(acc, er[c]);
    }
    stats_ptr(eps, eps_f64, r, n)[3] = __float_as_uint(acc);
}

template <bool VEC>
__global__ void __launch_bounds__(256) k_smc_epi(const float* __restrict__ x, float* __restrict__ y,
                                                 void* __restrict__ eps, int eps_f64, int64_t rows,
                                                 int64_t n, double u, double slack) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
         r += nwarps) {
        const uint32_t* st = stats_ptr(eps, eps_f64, r, n);
        const double epsS =
            __longlong_as_double((long long)(((unsigned long long)st[1] << 32) | st[0]));
        const float m = __uint_as_float(st[2]), S = __uint_as_float(st[3]);
        __syncwarp();  // every lane holds the stats before the slot is overwritten
        // eps_y = e (u(|x|+|m|) + 2u)/S + e epsS/S^2 + u|y| = e (A|x| + B) + u|y|
        // with A = u/S, B = (u|m| + 2u)/S + epsS/S^2: every term >= 0, a few
        // FP64 ulps from bounds.py's order (covered by `slack` >= 2^-50), and
        // the (1 + slack) factor folded into A, B and u
        const double S64 = (double)S;
        const double sl = __dadd_rn(1.0, slack), two_u = __dmul_rn(2.0, u);
        const double A = __dmul_rn(__ddiv_rn(u, S64), sl);
        const double B = __dmul_rn(__dadd_rn(
            __ddiv_rn(__dadd_rn(__dmul_rn(u, fabs((double)m)), two_u), S64),
            __ddiv_rn(epsS, __dmul_rn(S64, S64))), sl);
        const double us = __dmul_rn(u, sl);
        const float* xr = x + r * n;
        float* yr = y + r * n;
        const int64_t ob = r * n;
        if (VEC) {
            const float4* x4 = reinterpret_cast<const float4*>(xr);
            float4* y4 = reinterpret_cast<float4*>(yr);
            for (int64_t c = lane; c < (n >> 2); c += 32) {
                const float4 xv = __ldg(x4 + c);
                const float4 ev = y4[c];
                const float xs[4] = {xv.x, xv.y, xv.z, xv.w}, es[4] = {ev.x, ev.y, ev.z, ev.w};
                float ys[4];
                double vs[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    ys[k] = __fdiv_rn(es[k], S);
                    const double t = __fma_rn(A, fabs((double)xs[k]), B);
                    vs[k] = __fma_rn((double)es[k], t, __dmul_rn(us, fabs((double)ys[k])));
                }
                y4[c] = make_float4(ys[0], ys[1], ys[2], ys[3]);
                if (eps_f64) {
                    double2* e2 = reinterpret_cast<double2*>(static_cast<double*>(eps) + ob) + 2 * c;
                    e2[0] = make_double2(vs[0], vs[1]);
                    e2[1] = make_double2(vs[2], vs[3]);
                } else {
                    reinterpret_cast<float4*>(static_cast<float*>(eps) + ob)[c] = make_float4(
                        __double2float_ru(vs[0]), __double2float_ru(vs[1]),
                        __double2float_ru(vs[2]), __double2float_ru(vs[3]));
                }
            }
        } else {
            for (int64_t c = lane; c < n; c += 32) {
                const float xv = __ldg(xr + c), ev = yr[c];
                const float yv = __fdiv_rn(ev, S);
                yr[c] = yv;
                const double t = __fma_rn(A, fabs((double)xv), B);
                const double v = __fma_rn((double)ev, t, __dmul_rn(us, fabs((double)yv)));
                if (eps_f64) static_cast<double*>(eps)[ob + c] = v;
                else static_cast<float*>(eps)[ob + c] = __double2float_ru(v);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Softmax, design G (many rows, 16-byte aligned, R rows of e fit in ~64 KB):
// one CTA per group of R rows, persistent over groups, e kept in shared memory
// so HBM sees read x + write y + write eps (12-16 B/element; the epilogue's
// re-read of x hits L2).  Phase 1 warp per row (max, e = fp32(exp64(x-m)) ->
// smem, FP64 eps sums); phase 2 lane r of warp 0 runs row r's sequential fold
// from smem (conflict-free: rows padded to n+4 floats); phase 3 warp per row
// epilogue.  2-3 CTAs per SM overlap one CTA's serial fold with the others'
// memory phases.
constexpr int kSmgBudget = 72 * 1024;

__global__ void __launch_bounds__(256) k_smg(const float* __restrict__ x, float* __restrict__ y,
                                             void* __restrict__ eps, int eps_f64, int64_t rows,
                                             int n, int R, double u, double rc, double slack) {
    extern __shared__ __align__(16) float s_e[];  // [R][n + 4]
    __shared__ float s_m[32], s_S[32];
    __shared__ double s_epsS[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ns = n + 4, n4 = n >> 2;
    const double two_u = __dmul_rn(2.0, u);
    const double sl = __dadd_rn(1.0, slack);
    for (int64_t g0 = (int64_t)blockIdx.x * R; g0 < rows; g0 += (int64_t)gridDim.x * R) {
        const int nr = (int)(rows - g0 < R ? rows - g0 : R);
        // phase 1
        for (int r = w; r < nr; r += 8) {
            const float4* x4 = reinterpret_cast<const float4*>(x + (g0 + r) * n);
            float m = -INFINITY;
            for (int c = lane; c < n4; c += 32) {
                const float4 v = __ldg(x4 + c);
                m = fmaxf(m, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            // sum eps_e = sum e (u(|x| + |m|) + 2u) = u sum e|x| + (u|m| + 2u) sum e:
            // two order-free FP64 sums (re-association covered by `slack`)
            double se = 0.0, sex = 0.0;
            auto one = [&](float xv) -> float {
                const float ev = (float)exp((double)__fsub_rn(xv, m));
                const double e64 = (double)ev;
                se = __dadd_rn(se, e64);
                sex = __fma_rn(e64, fabs((double)xv), sex);
                return ev;
            };
            float4* e4 = reinterpret_cast<float4*>(s_e + (size_t)r * ns);
            for (int c = lane; c < n4; c += 32) {
                const float4 v = __ldg(x4 + c);
                float4 e;
                e.x = one(v.x); e.y = one(v.y); e.z = one(v.z); e.w = one(v.w);
                e4[c] = e;
            }
            se = warp_sum(se);
            sex = warp_sum(sex);
            if (lane == 0) {
                const double um2 = __dadd_rn(__dmul_rn(u, fabs((double)m)), two_u);
                const double seps = __dadd_rn(__dmul_rn(u, sex), __dmul_rn(um2, se));
                s_m[r] = m;
                s_epsS[r] = __dadd_rn(__dmul_rn(rc, se), __dmul_rn(__dadd_rn(rc, 1.0), seps));
            }
        }
        __syncthreads();
        // phase 2: S = (((e0 + e1) + e2) + ...)
        if (threadIdx.x < nr) {
            const float4* e4 = reinterpret_cast<const float4*>(s_e + (size_t)threadIdx.x * ns);
            float4 v = e4[0];
            float acc = __fadd_rn(__fadd_rn(__fadd_rn(v.x, v.y), v.z), v.w);
            int c = 1;
            for (; c + 8 <= n4; c += 8) {
                float4 b[8];
#pragma unroll
                for (int k = 0; k < 8; k++) b[k] = e4[c + k];
#pragma unroll
                for (int k = 0; k < 8; k++)
                    acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, b[k].x), b[k].y), b[k].z),
                                    b[k].w);
            }
            for (; c < n4; c++) {
                v = e4[c];
                acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, v.x), v.y), v.z), v.w);
            }
            s_S[threadIdx.x] = acc;
        }
        __syncthreads();
        // phase 3
        for (int r = w; r < nr; r += 8) {
            // eps_y = e (u(|x|+|m|) + 2u)/S + e epsS/S^2 + u|y| = e (A|x| + B) + u|y|,
            // A = u/S, B = (u|m| + 2u)/S + epsS/S^2, all terms >= 0 (a few FP64
            // ulps from bounds.py's order, covered by `slack`); the (1 + slack)
            // factor is folded into A, B and u
            const float S = s_S[r];
            const double S64 = (double)S;
            const double A = __dmul_rn(__ddiv_rn(u, S64), sl);
            const double B = __dmul_rn(__dadd_rn(
                __ddiv_rn(__dadd_rn(__dmul_rn(u, fabs((double)s_m[r])), two_u), S64),
                __ddiv_rn(s_epsS[r], __dmul_rn(S64, S64))), sl);
            const double us = __dmul_rn(u, sl);
            const int64_t ob = (g0 + r) * n;
            const float4* x4 = reinterpret_cast<const float4*>(x + ob);
            const float4* e4 = reinterpret_cast<const float4*>(s_e + (size_t)r * ns);
            float4* y4 = reinterpret_cast<float4*>(y + ob);
            for (int c = lane; c < n4; c += 32) {
                const float4 xv = __ldg(x4 + c);
                const float4 ev = e4[c];
                const float xs[4] = {xv.x, xv.y, xv.z, xv.w}, es[4] = {ev.x, ev.y, ev.z, ev.w};
                float ys[4];
                double vs[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    ys[k] = __fdiv_rn(es[k], S);
                    const double t = __fma_rn(A, fabs((double)xs[k]), B);
                    vs[k] = __fma_rn((double)es[k], t, __dmul_rn(us, fabs((double)ys[k])));
                }
                __stcs(y4 + c, make_float4(ys[0], ys[1], ys[2], ys[3]));
                if (eps_f64) {
                    double2* e2 = reinterpret_cast<double2*>(static_cast<double*>(eps) + ob) + 2 * c;
                    __stcs(e2, make_double2(vs[0], vs[1]));
                    __stcs(e2 + 1, make_double2(vs[2], vs[3]));
                } else {
                    __stcs(reinterpret_cast<float4*>(static_cast<float*>(eps) + ob) + c, make_float4(
                        __double2float_ru(vs[0]), __double2float_ru(vs[1]),
                        __double2float_ru(vs[2]), __double2float_ru(vs[3])));
                }
            }
        }
        __syncthreads();  // s_e / s_S reused by the next group
    }
}

// design C for many long rows (returns -1 when it does not apply)
static int softmax_c(const float* x, float* y, void* eps, int eps_f64, int64_t rows, int64_t n,
                     double u, double rc, double slack, cudaStream_t st) {
    if (n < 128 || rows < 1024) return -1;
    const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                       reinterpret_cast<uintptr_t>(eps)) & 15) == 0 && (n & 3) == 0;
    // design G (default since round 2): ~25% faster alone; in round 1 its 72 KB
    // CTAs crowded the concurrently running commit out of the SMs, but with
    // FP64 row bounds and the round-2 commit it wins in the overlapped verifier
    // too (bench 76.0 -> 75.5 %, softmax 33.7 -> 26.7 ms per step);
    // NAO_SOFTMAX_DESIGN=C selects design C
    static const int design = [] {
        const char* e = getenv("NAO_SOFTMAX_DESIGN");
        return e && e[0] == 'C' ? 0 : 1;
    }();
    const int64_t row_bytes = (n + 4) * 4;
    static const int budget = [] {
        const char* e = getenv("NAO_SMG_BUDGET");
        const int b = e ? atoi(e) : kSmgBudget;
        return b > 0 && b <= kSmgBudget ? b : kSmgBudget;
    }();
    // G stages whole rows in shared memory: below 8 rows per CTA (n > ~2200)
    // too few sequential folds overlap per SM and design C (e through L2, a
    // fold thread for every row) is faster (SD-UNet n = 4096 rows: 40.7 vs
    // 44.8 ms per step)
    if (vec && design == 1 && 8 * row_bytes <= budget && n < (1 << 30)) {
        int R = (int)(budget / row_bytes);
        if (R > 32) R = 32;
        if (R > 8) R &= ~7;
        const size_t smem = (size_t)R * row_bytes;
        static bool attr = false;
        if (!attr) {
            NAO_CHECK_CUDA(cudaFuncSetAttribute(k_smg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                kSmgBudget));
            attr = true;
        }
        const int64_t groups = ceil_div(rows, (int64_t)R);
        static const int per_sm = [] {
            const char* e = getenv("NAO_SMG_CTAS");
            return e ? atoi(e) : 0;
        }();
        const int64_t cap = per_sm > 0 ? per_sm : (kSmgBudget * 3 / budget);
        const int64_t grid = std::min<int64_t>(groups, (int64_t)kNumSMs * cap);
        k_smg<<<(unsigned)grid, 256, smem, st>>>(x, y, eps, eps_f64, rows, (int)n, R, u, rc, slack);
        NAO_CHECK_LAUNCH();
        return NAO_OK;
    }
    const int64_t wblocks = std::min<int64_t>(ceil_div(rows, 8), (int64_t)kNumSMs * 8);
    if (vec) {
        k_smc_rows<true><<<(unsigned)wblocks, 256, 0, st>>>(x, y, eps, eps_f64, rows, n, u, rc);
        k_smc_fold<true><<<(unsigned)ceil_div(rows, 128), 128, 0, st>>>(y, eps, eps_f64, rows, n);
        k_smc_epi<true><<<(unsigned)wblocks, 256, 0, st>>>(x, y, eps, eps_f64, rows, n, u, slack);
    } else {
        k_smc_rows<false><<<(unsigned)wblocks, 256, 0, st>>>(x, y, eps, eps_f64, rows, n, u, rc);
        k_smc_fold<false><<<(unsigned)ceil_div(rows, 128), 128, 0, st>>>(y, eps, eps_f64, rows, n);
        k_smc_epi<false><<<(unsigned)wblocks, 256, 0, st>>>(x, y, eps, eps_f64, rows, n, u, slack);
    }
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

// rows per CTA for design B (0 = use the transposed-tile kernels)
static int rows_per_cta(int64_t rows, int64_t n, int kind) {
    const int64_t bufs = kind == 0 ? 2 : 1;
    const int64_t per_row = bufs * n * 4;
    const int64_t budget = 96 * 1024;
    if (per_row > budget) return 0;
    // reductions: short rows -> lane-per-row transposed tiles (k_reduce_rows);
    // long rows -> one row per CTA (the serial fold is the critical path, so
    // spread rows over as many SMs / CTAs as possible)
    if (kind >= 2) return n <= 1024 ? 0 : 1;
    int64_t R = budget / per_row;
    if (R > 32) R = 32;
    // transposed-tile kernels win when there are enough rows to fill the GPU with warps
    if (rows >= (int64_t)kNumSMs * 4 * 32 * 8 && n <= 2048 && kind != 1) return 0;
    // keep >= 2 CTAs per SM worth of work when rows are few
    while (R > 1 && ceil_div(rows, R) < 2 * kNumSMs) R >>= 1;
    return (int)R;
}

static int launch(const float* x, float* y, void* eps, int eps_f64, int64_t rows, int64_t n,
                  int kind, float ln_eps, double u, double rc, double slack, cudaStream_t st) {
    const int R = rows_per_cta(rows, n, kind);
    if (R == 0 && kind >= 1 && n * 4 > 96 * 1024) {  // rows beyond shared memory
        const size_t sm = 2 * kStreamTile * sizeof(float);
        static bool attr_s = false;
        if (!attr_s) {
            NAO_CHECK_CUDA(cudaFuncSetAttribute(k_rows_stream,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            attr_s = true;
        }
        k_rows_stream<<<(unsigned)rows, kThreads, sm, st>>>(x, y, eps, eps_f64, rows, n, kind, ln_eps,
                                                            u, rc, slack);
        NAO_CHECK_LAUNCH();
        return NAO_OK;
    }
    if (R == 0) return -1;
    const size_t smem = (size_t)(kind == 0 ? 2 : 1) * R * n * 4;
    static bool attr = false;
    if (!attr) {
        NAO_CHECK_CUDA(cudaFuncSetAttribute(k_rows_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            200 * 1024));
        attr = true;
    }
    k_rows_smem<<<(unsigned)ceil_div(rows, R), kThreads, smem, st>>>(x, y, eps, eps_f64, rows, n, R,
                                                                     kind, ln_eps, u, rc, slack,
                                                                     Prof{NAO_ORDER_SEQUENTIAL, 32,
                                                                          nullptr});
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

// Non-sequential device profiles: always the shared-memory row kernel (the
// fold thread walks the staged row in the profile's order).
static int launch_profile(const float* x, float* y, void* eps, int eps_f64, int64_t rows,
                          int64_t n, int kind, float ln_eps, double u, double rc, double slack,
                          const Prof& prof, cudaStream_t st) {
    const int64_t per_row = (kind == 0 ? 2 : 1) * n * 4;
    NAO_REQUIRE(per_row <= 96 * 1024, "profile-order emulation supports rows of up to %lld "
                "elements", (long long)(96 * 1024 / (kind == 0 ? 8 : 4)));
    int64_t R = (96 * 1024) / per_row;
    if (R > 32) R = 32;
    while (R > 1 && ceil_div(rows, R) < 2 * kNumSMs) R >>= 1;
    static bool attr = false;
    if (!attr) {
        NAO_CHECK_CUDA(cudaFuncSetAttribute(k_rows_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            200 * 1024));
        attr = true;
    }
    const size_t smem = (size_t)(kind == 0 ? 2 : 1) * R * n * 4;
    k_rows_smem<<<(unsigned)ceil_div(rows, R), kThreads, smem, st>>>(
        x, y, eps, eps_f64, rows, n, (int)R, kind, ln_eps, u, rc, slack, prof);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

}  // namespace rowb
}  // namespace nao
