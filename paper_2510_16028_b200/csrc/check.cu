// Acceptance check (north_star (3)).
//
// nao_check: ONE pass over (local y, claimed y', eps) per operator emitting
//   * n_violations  = #{ |y'-y| > eps }      (dispute.py:641-648, strict >)
//   * n_borderline  = #{ eps*lo < |y'-y| <= eps }  (eps is an over-estimate of
//                     the reference bound by at most 1/lo; borderline elements
//                     are where a verdict could differ -> reported, not hidden)
//   * max_ratio     = max |y'-y| / eps
//   * the exact threshold verdict p_max > 1 of observed_p_max
//     (dispute.py:114-141): for every grid point p and array {abs, rel} the
//     percentile exceeds tau iff fewer than k+1 keys are <= tau (k =
//     floor((n-1)p/100)); the pass histograms keys into the intervals between
//     the sorted thresholds, so one read decides all 46 comparisons.  The one
//     undecidable case (exactly k+1 keys <= tau) is settled exactly by a second
//     pass that runs only when that case occurs (max key <= tau, min key > tau,
//     numpy's _lerp).
// nao_error_profiles / nao_percentile_profile: exact numpy-"linear"
//   percentiles (full radix sort of the FP64 keys), used by the API-level
//   percentile_profile / observed_p_max (calibration.py:33-37).
#include <cub/cub.cuh>
#include <cmath>
#include <vector>
#include <algorithm>

#include "common.cuh"

namespace nao {

constexpr int kMaxGrid = 32;

struct CheckAccum {  // device scratch, zeroed per call
    unsigned long long n_viol, n_border, n_nonfinite, n_amb_flag;
    unsigned long long hist_abs[kMaxGrid + 1];
    unsigned long long hist_rel[kMaxGrid + 1];
    unsigned long long max_ratio_bits;       // non-negative double
    unsigned long long amb_lo[2 * kMaxGrid];  // max key <= tau (double bits)
    unsigned long long amb_hi[2 * kMaxGrid];  // min key >  tau (double bits)
    int amb_target[2 * kMaxGrid];             // 1 if target needs pass 2
};

struct CheckParams {
    const float* local;
    const float* claimed;
    const void* eps;
    int64_t n;
    int eps_kind;       // NAO_EPS_*
    double eps_scale;   // NAO_EPS_SCALED_LOCAL: eps = scale*|local|
    double lo_factor;   // borderline band
    double epsilon;     // relative-error guard (calibration.py:19)
    int G;
    double t_abs[kMaxGrid];  // thresholds sorted ascending (host)
    double t_rel[kMaxGrid];
};

struct FinalParams {
    int G;
    int64_t n;
    double grid[kMaxGrid];       // percentile grid (original order)
    double tau_abs[kMaxGrid];    // effective thresholds, original order
    double tau_rel[kMaxGrid];
    int lpos_abs[kMaxGrid];      // #{sorted t < tau_i}
    int lpos_rel[kMaxGrid];
};

__device__ __forceinline__ int bsearch_pos(const double* t, int G, double key) {
    int pos = 0;  // number of thresholds strictly below key
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1)
        if (pos + step <= G && t[pos + step - 1] < key) pos += step;
    return pos;
}
__device__ __forceinline__ int bsearch_pos32(const float* t, int G, float key) {
    int pos = 0;
#pragma unroll
    for (int step = 16; step >= 1; step >>= 1)
        if (pos + step <= G && t[pos + step - 1] < key) pos += step;
    return pos;
}

// Exact FP64 keys of one element (dispute.py:134-138).
__device__ __forceinline__ double abs_key(float y, float yc) {
    return fabs(__dsub_rn((double)y, (double)yc));
}
__device__ __forceinline__ double rel_key(double diff, float y, double epsilon) {
    return __ddiv_rn(diff, __dadd_rn(fabs((double)y), epsilon));
}

struct SmemT {
    double t_abs[kMaxGrid], t_rel[kMaxGrid];
    float f_rel[kMaxGrid];
    float f_rel_lo[kMaxGrid], f_rel_hi[kMaxGrid];  // guard band edges
    unsigned long long hist_abs[kMaxGrid + 1], hist_rel[kMaxGrid + 1];
    unsigned long long viol, border, nonfin;
    double maxr;
};

constexpr float kGuard = 1.0f / 524288.0f;  // 2^-19 relative guard for the FP32 fast path

template <int EPSK>
__device__ __forceinline__ double load_eps(const CheckParams& p, int64_t i, float y) {
    if (EPSK == NAO_EPS_TENSOR_F32) return (double)__ldg(static_cast<const float*>(p.eps) + i);
    if (EPSK == NAO_EPS_TENSOR_F64) return __ldg(static_cast<const double*>(p.eps) + i);
    if (EPSK == NAO_EPS_SCALED_LOCAL) return __dmul_rn(p.eps_scale, fabs((double)y));
    return 0.0;
}

template <int EPSK>
__global__ void __launch_bounds__(256) k_check(const __grid_constant__ CheckParams p,
                                               CheckAccum* __restrict__ acc) {
    __shared__ SmemT sm;
    const int G = p.G;
    if (threadIdx.x < kMaxGrid) {
        int i = threadIdx.x;
        double ta = i < G ? p.t_abs[i] : INFINITY;
        double tr = i < G ? p.t_rel[i] : INFINITY;
        sm.t_abs[i] = ta;
        sm.t_rel[i] = tr;
        float fr = (float)tr;
        sm.f_rel[i] = fr;
        sm.f_rel_lo[i] = fr * (1.0f - kGuard);
        sm.f_rel_hi[i] = fr * (1.0f + kGuard);
    }
    if (threadIdx.x <= kMaxGrid) { sm.hist_abs[threadIdx.x] = 0; sm.hist_rel[threadIdx.x] = 0; }
    if (threadIdx.x == 0) { sm.viol = sm.border = sm.nonfin = 0; sm.maxr = 0.0; }
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // warp-private interval counters (no atomics: one leader per distinct bucket)
    __shared__ uint32_t wc[8][2][kMaxGrid + 1];
    for (int b = lane; b <= kMaxGrid; b += 32) { wc[warp][0][b] = 0; wc[warp][1][b] = 0; }
    __syncwarp();
    unsigned long long viol = 0, border = 0, nonfin = 0;
    double best_num = 0.0, best_den = 1.0;  // max ratio as a fraction
    bool best_inf = false;

    auto process = [&](bool valid, float y, float yc, double eps, int& pa, int& pr) {
        pa = -1; pr = -1;
        if (!valid) return;
        if (!isfinite(y) || !isfinite(yc)) { nonfin++; viol++; pa = G; pr = G; return; }
        const double diff = abs_key(y, yc);
        if (diff > eps) viol++;
        else if (diff > eps * p.lo_factor) border++;
        // running max of diff/eps without a division per element
        if (eps > 0.0) {
            if (!best_inf && diff * best_den > best_num * eps) { best_num = diff; best_den = eps; }
        } else if (diff > 0.0) {
            best_inf = true;
        }
        if (diff == 0.0) { pa = 0; pr = 0; return; }
        pa = bsearch_pos(sm.t_abs, G, diff);
        // relative key: FP32 estimate, exact FP64 only inside the guard band
        const float d32 = (float)diff;
        const float den32 = __fadd_rn(fabsf(y), (float)p.epsilon);
        const float r32 = __fdiv_rn(d32, den32);
        int q = bsearch_pos32(sm.f_rel, G, r32);
        bool safe = (d32 >= 1e-30f) && (r32 >= 1e-30f) && isfinite(r32) &&
                    (q == G || r32 < sm.f_rel_lo[q]) && (q == 0 || r32 > sm.f_rel_hi[q - 1]);
        if (!safe) q = bsearch_pos(sm.t_rel, G, rel_key(diff, y, p.epsilon));
        pr = q;
    };

    auto tally = [&](int pa, int pr) {
        // common case: the whole warp lands in one bucket (e.g. all diffs zero)
        const int a0 = __shfl_sync(0xffffffffu, pa, 0), r0 = __shfl_sync(0xffffffffu, pr, 0);
        if (__all_sync(0xffffffffu, pa == a0 && pr == r0)) {
            if (lane == 0 && a0 >= 0) { wc[warp][0][a0] += 32; wc[warp][1][r0] += 32; }
        } else {
            unsigned ma = __match_any_sync(0xffffffffu, pa);
            unsigned mr = __match_any_sync(0xffffffffu, pr);
            if (pa >= 0 && (__ffs(ma) - 1) == lane) wc[warp][0][pa] += __popc(ma);
            __syncwarp();
            if (pr >= 0 && (__ffs(mr) - 1) == lane) wc[warp][1][pr] += __popc(mr);
            __syncwarp();
        }
        __syncwarp();
    };

    const int64_t n = p.n;
    const int64_t nvec = n >> 2;
    const float4* yl = reinterpret_cast<const float4*>(p.local);
    const float4* yc = reinterpret_cast<const float4*>(p.claimed);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // warp-uniform trip count so every lane joins the ballots
    const int64_t base0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    for (int64_t wb = base0; wb < nvec; wb += stride) {
        const int64_t v = wb + lane;
        const bool ok = v < nvec;
        float4 a = ok ? __ldg(yl + v) : make_float4(0, 0, 0, 0);
        float4 c = ok ? __ldg(yc + v) : make_float4(0, 0, 0, 0);
        double e0 = 0, e1 = 0, e2 = 0, e3 = 0;
        if (ok) {
            if (EPSK == NAO_EPS_TENSOR_F32) {
                float4 e = __ldg(reinterpret_cast<const float4*>(p.eps) + v);
                e0 = e.x; e1 = e.y; e2 = e.z; e3 = e.w;
            } else if (EPSK == NAO_EPS_TENSOR_F64) {
                const double2* ep = reinterpret_cast<const double2*>(p.eps);
                double2 u0 = __ldg(ep + 2 * v), u1 = __ldg(ep + 2 * v + 1);
                e0 = u0.x; e1 = u0.y; e2 = u1.x; e3 = u1.y;
            } else if (EPSK == NAO_EPS_SCALED_LOCAL) {
                e0 = __dmul_rn(p.eps_scale, fabs((double)a.x));
                e1 = __dmul_rn(p.eps_scale, fabs((double)a.y));
                e2 = __dmul_rn(p.eps_scale, fabs((double)a.z));
                e3 = __dmul_rn(p.eps_scale, fabs((double)a.w));
            }
        }
        int pa, pr;
        process(ok, a.x, c.x, e0, pa, pr); tally(pa, pr);
        process(ok, a.y, c.y, e1, pa, pr); tally(pa, pr);
        process(ok, a.z, c.z, e2, pa, pr); tally(pa, pr);
        process(ok, a.w, c.w, e3, pa, pr); tally(pa, pr);
    }
    // scalar tail (n % 4) handled by the first warp of block 0
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        const int64_t i = (nvec << 2) + lane;
        const bool ok = i < n;
        float y = ok ? p.local[i] : 0.f, c = ok ? p.claimed[i] : 0.f;
        double e = ok ? load_eps<EPSK>(p, i, y) : 0.0;
        int pa, pr;
        process(ok, y, c, e, pa, pr);
        tally(pa, pr);
    }
    // reduce
    viol = warp_sum(viol); border = warp_sum(border); nonfin = warp_sum(nonfin);
    double r = best_inf ? INFINITY : (best_num > 0.0 ? best_num / best_den : 0.0);
    r = warp_max(r);
    for (int b = lane; b <= G; b += 32) {
        if (wc[warp][0][b]) atomicAdd(&sm.hist_abs[b], (unsigned long long)wc[warp][0][b]);
        if (wc[warp][1][b]) atomicAdd(&sm.hist_rel[b], (unsigned long long)wc[warp][1][b]);
    }
    if (lane == 0) {
        atomicAdd(&sm.viol, viol);
        atomicAdd(&sm.border, border);
        atomicAdd(&sm.nonfin, nonfin);
        atomic_max_nonneg(&sm.maxr, r);
    }
    __syncthreads();
    if (threadIdx.x <= G) {
        if (sm.hist_abs[threadIdx.x]) atomicAdd(&acc->hist_abs[threadIdx.x], sm.hist_abs[threadIdx.x]);
        if (sm.hist_rel[threadIdx.x]) atomicAdd(&acc->hist_rel[threadIdx.x], sm.hist_rel[threadIdx.x]);
    }
    if (threadIdx.x == 0) {
        if (sm.viol) atomicAdd(&acc->n_viol, sm.viol);
        if (sm.border) atomicAdd(&acc->n_border, sm.border);
        if (sm.nonfin) atomicAdd(&acc->n_nonfinite, sm.nonfin);
        atomicMax(&acc->max_ratio_bits, (unsigned long long)__double_as_longlong(sm.maxr));
    }
}

// numpy _lerp (_function_base_impl.py:4657-4679), no FMA contraction.
__device__ __forceinline__ double np_lerp(double a, double b, double t) {
    double d = __dsub_rn(b, a);
    double r = __dadd_rn(a, __dmul_rn(d, t));
    if (t >= 0.5) r = __dsub_rn(b, __dmul_rn(d, __dsub_rn(1.0, t)));
    return r;
}

// virtual index (n-1)*q, q = p/100 (_function_base_impl.py:126-129, :4277)
struct VIdx { int64_t prev, next; double g; bool last; };
__device__ __forceinline__ VIdx virtual_index(int64_t n, double p) {
    VIdx v;
    double q = __ddiv_rn(p, 100.0);
    double vi = __dmul_rn((double)(n - 1), q);
    if (vi >= (double)(n - 1)) {
        v.prev = v.next = n - 1; v.g = __dadd_rn(vi, 1.0); v.last = true;
    } else {
        double f = floor(vi);
        v.prev = (int64_t)f; v.next = v.prev + 1; v.g = __dsub_rn(vi, f); v.last = false;
    }
    return v;
}

// phase: 0 = after pass 1 (decide / flag ambiguous), 1 = after pass 2.
__global__ void k_check_finalize(const __grid_constant__ FinalParams fp, CheckAccum* acc,
                                 nao_check_result* out, int phase) {
    if (threadIdx.x != 0) return;
    const int G = fp.G;
    int exceeded = 0, first = -1, n_amb = 0;
    for (int arr = 0; arr < 2; arr++) {
        const unsigned long long* hist = arr == 0 ? acc->hist_abs : acc->hist_rel;
        for (int i = 0; i < G; i++) {
            const double tau = arr == 0 ? fp.tau_abs[i] : fp.tau_rel[i];
            const int L = arr == 0 ? fp.lpos_abs[i] : fp.lpos_rel[i];
            unsigned long long cle = 0;
            for (int b = 0; b <= L; b++) cle += hist[b];
            VIdx v = virtual_index(fp.n, fp.grid[i]);
            bool ex;
            if (v.last) {
                ex = cle < (unsigned long long)fp.n;
            } else if (cle <= (unsigned long long)v.prev) {
                ex = true;
            } else if (cle >= (unsigned long long)v.prev + 2) {
                ex = false;
            } else {  // x_(k) <= tau < x_(k+1): interpolate exactly
                const int t = arr * kMaxGrid + i;
                if (phase == 0) {
                    acc->amb_target[t] = 1;
                    acc->amb_lo[t] = 0ull;
                    acc->amb_hi[t] = 0x7ff0000000000000ull;  // +inf
                    n_amb++;
                    ex = false;
                } else {
                    double a = __longlong_as_double((long long)acc->amb_lo[t]);
                    double b = __longlong_as_double((long long)acc->amb_hi[t]);
                    ex = np_lerp(a, b, v.g) > tau;
                }
            }
            if (ex) {
                exceeded = 1;
                if (first < 0) first = arr * G + i;
            }
        }
    }
    if (phase == 0) acc->n_amb_flag = (unsigned long long)n_amb;
    if (phase == 0 && n_amb > 0) return;  // pass 2 + phase-1 finalize complete the result
    out->n = (uint64_t)fp.n;
    out->n_violations = acc->n_viol;
    out->n_borderline = acc->n_border;
    out->n_nonfinite = acc->n_nonfinite;
    out->max_ratio = __longlong_as_double((long long)acc->max_ratio_bits);
    out->threshold_exceeded = exceeded;
    out->first_exceeded = first;
    out->n_ambiguous = (int32_t)acc->n_amb_flag;
}

// Pass 2 (rare): for each ambiguous target, max key <= tau and min key > tau.
__global__ void __launch_bounds__(256) k_check_pass2(const __grid_constant__ CheckParams p,
                                                     const __grid_constant__ FinalParams fp,
                                                     CheckAccum* __restrict__ acc) {
    if (acc->n_amb_flag == 0) return;
    __shared__ int targets[2 * kMaxGrid];
    __shared__ double taus[2 * kMaxGrid];
    __shared__ int nt;
    if (threadIdx.x == 0) {
        int c = 0;
        for (int t = 0; t < 2 * kMaxGrid; t++)
            if (acc->amb_target[t]) {
                targets[c] = t;
                taus[c] = (t < kMaxGrid) ? fp.tau_abs[t] : fp.tau_rel[t - kMaxGrid];
                c++;
            }
        nt = c;
    }
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float y = p.local[i], c = p.claimed[i];
        double diff = abs_key(y, c);
        double rel = rel_key(diff, y, p.epsilon);
        for (int k = 0; k < nt; k++) {
            int t = targets[k];
            double key = t < kMaxGrid ? diff : rel;
            unsigned long long bits = (unsigned long long)__double_as_longlong(key);
            if (key <= taus[k]) atomicMax(&acc->amb_lo[t], bits);
            else atomicMin(&acc->amb_hi[t], bits);
        }
    }
}

// ------------------------------------------------------- exact percentiles

__global__ void k_error_keys(const float* __restrict__ a, const float* __restrict__ b, int64_t n,
                             double epsilon, unsigned long long* __restrict__ kabs,
                             unsigned long long* __restrict__ krel) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float y = a[i];
        double d = abs_key(y, b[i]);
        kabs[i] = (unsigned long long)__double_as_longlong(d);
        krel[i] = (unsigned long long)__double_as_longlong(rel_key(d, y, epsilon));
    }
}

// Order-preserving map of arbitrary doubles to uint64 (NaN counted aside).
__global__ void k_value_keys(const double* __restrict__ v, int64_t n,
                             unsigned long long* __restrict__ keys,
                             unsigned long long* __restrict__ nan_count) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double x = v[i];
        unsigned long long u = (unsigned long long)__double_as_longlong(x);
        if (isnan(x)) atomicAdd(nan_count, 1ull);
        keys[i] = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
    }
}

__device__ __forceinline__ double key_to_value(unsigned long long k, bool signed_map) {
    if (!signed_map) return __longlong_as_double((long long)k);
    unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)u);
}

__global__ void k_profile_from_sorted(const unsigned long long* __restrict__ sorted, int64_t n,
                                      const __grid_constant__ FinalParams fp, bool signed_map,
                                      const unsigned long long* nan_count, double* __restrict__ out) {
    int i = threadIdx.x;
    if (i >= fp.G) return;
    if (nan_count && *nan_count) { out[i] = NAN; return; }
    VIdx v = virtual_index(n, fp.grid[i]);
    double a = key_to_value(sorted[v.prev], signed_map);
    double b = key_to_value(sorted[v.next], signed_map);
    out[i] = np_lerp(a, b, v.g);
}

static int grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, kNumSMs * 8));
}

static size_t sort_temp_bytes(int64_t n) {
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, (unsigned long long*)nullptr,
                                   (unsigned long long*)nullptr, (int)n);
    return tb;
}

static int fill_grid(FinalParams& fp, const double* grid, int G) {
    NAO_REQUIRE(G > 0 && G <= kMaxGrid, "grid size %d out of range (1..%d)", G, kMaxGrid);
    memset(&fp, 0, sizeof fp);
    fp.G = G;
    for (int i = 0; i < G; i++) {
        NAO_REQUIRE(std::isfinite(grid[i]) && grid[i] >= 0.0 && grid[i] <= 100.0,
                    "Percentiles must be in the range [0, 100]");
        fp.grid[i] = grid[i];
    }
    return NAO_OK;
}

}  // namespace nao

using namespace nao;

extern "C" {

size_t nao_check_workspace(void) { return sizeof(CheckAccum) + 256; }

int nao_check(const float* local, const float* claimed, int64_t n, int eps_kind, const void* eps,
              double eps_scale, double lo_factor, const double* grid, const double* tau_abs,
              const double* tau_rel, int n_grid, double epsilon, nao_check_result* result,
              void* workspace, size_t workspace_bytes, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    NAO_REQUIRE(n > 0, "percentile profile of empty input");
    NAO_REQUIRE(local && claimed && result, "null pointer argument");
    NAO_REQUIRE(eps_kind >= NAO_EPS_TENSOR_F32 && eps_kind <= NAO_EPS_ZERO, "bad eps_kind %d",
                eps_kind);
    NAO_REQUIRE(eps_kind == NAO_EPS_SCALED_LOCAL || eps_kind == NAO_EPS_ZERO || eps != nullptr,
                "eps tensor missing");
    NAO_REQUIRE((reinterpret_cast<uintptr_t>(local) | reinterpret_cast<uintptr_t>(claimed)) % 16 == 0,
                "local/claimed must be 16-byte aligned");
    NAO_REQUIRE(eps == nullptr || reinterpret_cast<uintptr_t>(eps) % 16 == 0,
                "eps must be 16-byte aligned");
    Workspace ws(workspace, workspace_bytes);
    CheckAccum* acc = ws.take<CheckAccum>(1);
    NAO_REQUIRE(acc != nullptr, "workspace too small");
    FinalParams fp;
    int rc = fill_grid(fp, grid, n_grid);
    if (rc) return rc;
    fp.n = n;
    CheckParams p;
    memset(&p, 0, sizeof p);
    p.local = local; p.claimed = claimed; p.eps = eps; p.n = n; p.eps_kind = eps_kind;
    p.eps_scale = eps_scale; p.lo_factor = lo_factor; p.epsilon = epsilon; p.G = n_grid;
    // effective thresholds: ratio obs/tau > 1  <=>  obs > tau (tau > 0) or obs > 0 (tau <= 0)
    std::vector<double> ea(n_grid), er(n_grid);
    for (int i = 0; i < n_grid; i++) {
        ea[i] = tau_abs[i] > 0.0 ? tau_abs[i] : 0.0;
        er[i] = tau_rel[i] > 0.0 ? tau_rel[i] : 0.0;
        fp.tau_abs[i] = ea[i];
        fp.tau_rel[i] = er[i];
    }
    std::vector<double> sa = ea, sr = er;
    std::sort(sa.begin(), sa.end());
    std::sort(sr.begin(), sr.end());
    for (int i = 0; i < n_grid; i++) {
        p.t_abs[i] = sa[i];
        p.t_rel[i] = sr[i];
        fp.lpos_abs[i] = (int)(std::lower_bound(sa.begin(), sa.end(), ea[i]) - sa.begin());
        fp.lpos_rel[i] = (int)(std::lower_bound(sr.begin(), sr.end(), er[i]) - sr.begin());
    }
    NAO_CHECK_CUDA(cudaMemsetAsync(acc, 0, sizeof(CheckAccum), st));
    const int threads = 256;
    int64_t warps_needed = ((n >> 2) + 31) / 32;
    int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((warps_needed + 7) / 8, kNumSMs * 8));
    switch (eps_kind) {
        case NAO_EPS_TENSOR_F32: k_check<NAO_EPS_TENSOR_F32><<<blocks, threads, 0, st>>>(p, acc); break;
        case NAO_EPS_TENSOR_F64: k_check<NAO_EPS_TENSOR_F64><<<blocks, threads, 0, st>>>(p, acc); break;
        case NAO_EPS_SCALED_LOCAL: k_check<NAO_EPS_SCALED_LOCAL><<<blocks, threads, 0, st>>>(p, acc); break;
        default: k_check<NAO_EPS_ZERO><<<blocks, threads, 0, st>>>(p, acc); break;
    }
    NAO_CHECK_LAUNCH();
    k_check_finalize<<<1, 32, 0, st>>>(fp, acc, result, 0);
    NAO_CHECK_LAUNCH();
    k_check_pass2<<<grid_for(n, 256), 256, 0, st>>>(p, fp, acc);
    NAO_CHECK_LAUNCH();
    k_check_finalize<<<1, 32, 0, st>>>(fp, acc, result, 1);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

size_t nao_percentile_workspace(int64_t n) {
    if (n <= 0) return 0;
    return (size_t)(4 * 8 * n) + sort_temp_bytes(n) + 4096;
}

int nao_error_profiles(const float* local, const float* claimed, int64_t n, double epsilon,
                       const double* grid, int n_grid, double* abs_prof, double* rel_prof,
                       void* workspace, size_t workspace_bytes, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    NAO_REQUIRE(n > 0, "percentile profile of empty input");
    FinalParams fp;
    int rc = fill_grid(fp, grid, n_grid);
    if (rc) return rc;
    fp.n = n;
    Workspace ws(workspace, workspace_bytes);
    auto* ka = ws.take<unsigned long long>(n);
    auto* kr = ws.take<unsigned long long>(n);
    auto* sa = ws.take<unsigned long long>(n);
    auto* sr = ws.take<unsigned long long>(n);
    size_t tb = sort_temp_bytes(n);
    void* tmp = ws.take<uint8_t>(tb);
    NAO_REQUIRE(ka && kr && sa && sr && tmp, "workspace too small");
    k_error_keys<<<grid_for(n, 256), 256, 0, st>>>(local, claimed, n, epsilon, ka, kr);
    NAO_CHECK_LAUNCH();
    NAO_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, ka, sa, (int)n, 0, 64, st));
    NAO_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, kr, sr, (int)n, 0, 64, st));
    k_profile_from_sorted<<<1, kMaxGrid, 0, st>>>(sa, n, fp, false, nullptr, abs_prof);
    k_profile_from_sorted<<<1, kMaxGrid, 0, st>>>(sr, n, fp, false, nullptr, rel_prof);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

int nao_percentile_profile(const double* values, int64_t n, const double* grid, int n_grid,
                           double* out, void* workspace, size_t workspace_bytes, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    NAO_REQUIRE(n > 0, "percentile profile of empty input");
    FinalParams fp;
    int rc = fill_grid(fp, grid, n_grid);
    if (rc) return rc;
    fp.n = n;
    Workspace ws(workspace, workspace_bytes);
    auto* k = ws.take<unsigned long long>(n);
    auto* s = ws.take<unsigned long long>(n);
    auto* nanc = ws.take<unsigned long long>(1);
    size_t tb = sort_temp_bytes(n);
    void* tmp = ws.take<uint8_t>(tb);
    NAO_REQUIRE(k && s && nanc && tmp, "workspace too small");
    NAO_CHECK_CUDA(cudaMemsetAsync(nanc, 0, 8, st));
    k_value_keys<<<grid_for(n, 256), 256, 0, st>>>(values, n, k, nanc);
    NAO_CHECK_LAUNCH();
    NAO_CHECK_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, k, s, (int)n, 0, 64, st));
    k_profile_from_sorted<<<1, kMaxGrid, 0, st>>>(s, n, fp, true, nanc, out);
    NAO_CHECK_LAUNCH();
    return NAO_OK;
}

}  // extern "C"
