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
#include "check_common.cuh"
#include "unary.cuh"

namespace nao {

struct CheckParams {
    const float* local;
    const float* claimed;
    const void* eps;
    int64_t n;
    int eps_kind;       // NAO_EPS_*
    double eps_scale;   // NAO_EPS_SCALED_LOCAL: eps = scale*|local|
    double lo_factor;   // borderline band
    unsigned long long* border;  // optional borderline list [1 + cap] (include/nao_b200.h)
    long long border_cap;
    VerdictSpec v;      // grid, thresholds, epsilon
};

constexpr int kCheckThreads = 256, kCheckWarps = kCheckThreads / 32, kQ = 64;
constexpr float kGuard = 1.0f / 524288.0f;  // 2^-19 relative guard for the FP32 fast path

struct CheckSmem {
    double t_abs[kMaxGrid], t_rel[kMaxGrid];
    float f_rel[kMaxGrid], f_rel_lo[kMaxGrid], f_rel_hi[kMaxGrid];
    uint32_t wc[kCheckWarps][2][kMaxGrid + 1];   // warp-private interval counters
    float qy[kCheckWarps][kQ], qc[kCheckWarps][kQ];  // warp compaction queue of
    double qe[kCheckWarps][kQ];                      // non-zero differences
    unsigned long long qi[kCheckWarps][kQ];          // and their flat indices
    unsigned long long viol, border, nonfin;
    double maxr;
    int is_last;
    VerdictSmem vs;
};

template <int EPSK>
__device__ __forceinline__ double load_eps(const CheckParams& p, int64_t i, float y) {
    if (EPSK == NAO_EPS_TENSOR_F32) return (double)__ldg(static_cast<const float*>(p.eps) + i);
    if (EPSK == NAO_EPS_TENSOR_F64) return __ldg(static_cast<const double*>(p.eps) + i);
    if (EPSK == NAO_EPS_SCALED_LOCAL) return __dmul_rn(p.eps_scale, fabs((double)y));
    return 0.0;
}

template <int EPSK>
__global__ void __launch_bounds__(kCheckThreads, 3) k_check(const __grid_constant__ CheckParams p,
                                                         CheckAccum* __restrict__ acc,
                                                         nao_check_result* __restrict__ out) {
    __shared__ CheckSmem sm;
    const int G = p.v.G;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x < kMaxGrid) {
        const int i = threadIdx.x;
        const double ta = i < G ? p.v.t_abs[i] : INFINITY;
        const double tr = i < G ? p.v.t_rel[i] : INFINITY;
        sm.t_abs[i] = ta;
        sm.t_rel[i] = tr;
        const float fr = (float)tr;
        sm.f_rel[i] = fr;
        sm.f_rel_lo[i] = fr * (1.0f - kGuard);
        sm.f_rel_hi[i] = fr * (1.0f + kGuard);
    }
    if (threadIdx.x < 2 * kMaxGrid) { sm.vs.amb[threadIdx.x] = 0; }
    for (int b = lane; b <= kMaxGrid; b += 32) { sm.wc[w][0][b] = 0; sm.wc[w][1][b] = 0; }
    if (threadIdx.x == 0) { sm.viol = sm.border = sm.nonfin = 0; sm.maxr = 0.0; sm.is_last = 0; }
    __syncthreads();

    unsigned long long viol = 0, border = 0, nonfin = 0;
    double best_num = 0.0, best_den = 1.0;  // running max of diff/eps as a fraction
    bool best_inf = false;
    uint32_t nzero = 0;  // y' == y exactly: diff 0 -> bucket 0, never a violation

    // exact processing of one non-zero difference (all lanes busy: no divergence)
    auto process = [&](float y, float yc, double eps, unsigned long long idx) {
        if (!isfinite(y) || !isfinite(yc)) {
            nonfin++; viol++;
            atomicAdd(&sm.wc[w][0][G], 1u); atomicAdd(&sm.wc[w][1][G], 1u);
            return;
        }
        const double diff = abs_key(y, yc);
        if (diff > eps) viol++;
        else if (diff > eps * p.lo_factor) {
            border++;
            if (p.border) list_push(p.border, p.border_cap, idx);
        }
        if (eps > 0.0) {
            if (!best_inf && diff * best_den > best_num * eps) { best_num = diff; best_den = eps; }
        } else if (diff > 0.0) {
            best_inf = true;
        }
        int pa = 0, q = 0;
        if (diff != 0.0) {
            pa = bsearch_pos(sm.t_abs, G, diff);
            const float d32 = (float)diff;
            const float r32 = __fdiv_rn(d32, __fadd_rn(fabsf(y), (float)p.v.epsilon));
            q = bsearch_pos32(sm.f_rel, G, r32);
            const bool safe = (d32 >= 1e-30f) && (r32 >= 1e-30f) && isfinite(r32) &&
                              (q == G || r32 < sm.f_rel_lo[q]) &&
                              (q == 0 || r32 > sm.f_rel_hi[q - 1]);
            if (!safe) q = bsearch_pos(sm.t_rel, G, rel_key(diff, y, p.v.epsilon));
        }
        atomicAdd(&sm.wc[w][0][pa], 1u);
        atomicAdd(&sm.wc[w][1][q], 1u);
    };
    int qn = 0;  // warp-uniform queue length
    auto push = [&](bool flag, float y, float yc, double e, unsigned long long idx) {
        const unsigned m = __ballot_sync(0xffffffffu, flag);
        if (m == 0) return;
        if (flag) {
            const int pos = qn + __popc(m & ((1u << lane) - 1u));
            sm.qy[w][pos] = y; sm.qc[w][pos] = yc; sm.qe[w][pos] = e; sm.qi[w][pos] = idx;
        }
        qn += __popc(m);
        if (qn >= 32) {
            __syncwarp();
            process(sm.qy[w][lane], sm.qc[w][lane], sm.qe[w][lane], sm.qi[w][lane]);
            __syncwarp();
            if (lane < qn - 32) {
                sm.qy[w][lane] = sm.qy[w][32 + lane];
                sm.qc[w][lane] = sm.qc[w][32 + lane];
                sm.qe[w][lane] = sm.qe[w][32 + lane];
                sm.qi[w][lane] = sm.qi[w][32 + lane];
            }
            __syncwarp();
            qn -= 32;
        }
    };

    const int64_t n = p.n;
    const int64_t nvec = n >> 2;
    const float4* yl = reinterpret_cast<const float4*>(p.local);
    const float4* ycl = reinterpret_cast<const float4*>(p.claimed);
    // Each warp walks 64 consecutive float4 pairs per step (lanes take v and
    // v + 32) and prefetches the next step's pairs before compacting the
    // current ones, so ~128 B per lane stay in flight while the queue drains.
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
    int64_t wb = (int64_t)blockIdx.x * blockDim.x * 2 + (int64_t)w * 64;
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 na0 = zero4, nc0 = zero4, na1 = zero4, nc1 = zero4;
    if (wb + lane < nvec) { na0 = __ldg(yl + wb + lane); nc0 = __ldg(ycl + wb + lane); }
    if (wb + 32 + lane < nvec) { na1 = __ldg(yl + wb + 32 + lane); nc1 = __ldg(ycl + wb + 32 + lane); }
    auto group = [&](const float4 a, const float4 c, const int64_t v) {
        const bool ok = v < nvec;
        const bool z0 = (a.x == c.x) & isfinite(a.x), z1 = (a.y == c.y) & isfinite(a.y);
        const bool z2 = (a.z == c.z) & isfinite(a.z), z3 = (a.w == c.w) & isfinite(a.w);
        const bool all_eq = z0 & z1 & z2 & z3;
        if (ok && all_eq) nzero += 4;
        if (__all_sync(0xffffffffu, all_eq || !ok)) return;
        double e0 = 0, e1 = 0, e2 = 0, e3 = 0;
        if (ok && !all_eq) {  // eps is only read where a difference exists
            if (EPSK == NAO_EPS_TENSOR_F32) {
                const float4 e = __ldg(reinterpret_cast<const float4*>(p.eps) + v);
                e0 = e.x; e1 = e.y; e2 = e.z; e3 = e.w;
            } else if (EPSK == NAO_EPS_TENSOR_F64) {
                const double2* ep = reinterpret_cast<const double2*>(p.eps);
                const double2 u0 = __ldg(ep + 2 * v), u1 = __ldg(ep + 2 * v + 1);
                e0 = u0.x; e1 = u0.y; e2 = u1.x; e3 = u1.y;
            } else if (EPSK == NAO_EPS_SCALED_LOCAL) {
                e0 = __dmul_rn(p.eps_scale, fabs((double)a.x));
                e1 = __dmul_rn(p.eps_scale, fabs((double)a.y));
                e2 = __dmul_rn(p.eps_scale, fabs((double)a.z));
                e3 = __dmul_rn(p.eps_scale, fabs((double)a.w));
            }
            if (z0) nzero++;
            if (z1) nzero++;
            if (z2) nzero++;
            if (z3) nzero++;
        }
        const bool live = ok && !all_eq;
        const unsigned long long i0 = 4ull * (unsigned long long)v;
        push(live && !z0, a.x, c.x, e0, i0);
        push(live && !z1, a.y, c.y, e1, i0 + 1);
        push(live && !z2, a.z, c.z, e2, i0 + 2);
        push(live && !z3, a.w, c.w, e3, i0 + 3);
    };
    for (; wb < nvec; wb += stride) {  // warp-uniform trip count (ballots)
        const float4 a0 = na0, c0 = nc0, a1 = na1, c1 = nc1;
        const int64_t wn = wb + stride;
        if (wn + lane < nvec) { na0 = __ldg(yl + wn + lane); nc0 = __ldg(ycl + wn + lane); }
        if (wn + 32 + lane < nvec) { na1 = __ldg(yl + wn + 32 + lane); nc1 = __ldg(ycl + wn + 32 + lane); }
        group(a0, c0, wb + lane);
        group(a1, c1, wb + 32 + lane);
    }
    // scalar tail (n % 4): first warp of block 0
    if (blockIdx.x == 0 && w == 0) {
        const int64_t i = (nvec << 2) + lane;
        const bool ok = i < n;
        float y = 0.f, c = 0.f;
        double e = 0.0;
        if (ok) { y = p.local[i]; c = p.claimed[i]; e = load_eps<EPSK>(p, i, y); }
        const bool z = (y == c) && isfinite(y);
        if (ok && z) nzero++;
        push(ok && !z, y, c, e, (unsigned long long)i);
    }
    __syncwarp();
    if (lane < qn) process(sm.qy[w][lane], sm.qc[w][lane], sm.qe[w][lane], sm.qi[w][lane]);
    __syncwarp();
    if (nzero) { atomicAdd(&sm.wc[w][0][0], nzero); atomicAdd(&sm.wc[w][1][0], nzero); }

    // ---- block reduction -> global accumulator
    viol = warp_sum(viol); border = warp_sum(border); nonfin = warp_sum(nonfin);
    double r = best_inf ? INFINITY : (best_num > 0.0 ? best_num / best_den : 0.0);
    r = warp_max(r);
    __syncwarp();
    if (lane == 0) {
        atomicAdd(&sm.viol, viol);
        atomicAdd(&sm.border, border);
        atomicAdd(&sm.nonfin, nonfin);
        atomic_max_nonneg(&sm.maxr, r);
    }
    __syncthreads();
    if (threadIdx.x <= G) {
        unsigned long long ha = 0, hr = 0;
        for (int ww = 0; ww < kCheckWarps; ww++) {
            ha += sm.wc[ww][0][threadIdx.x];
            hr += sm.wc[ww][1][threadIdx.x];
        }
        if (ha) atomicAdd(&acc->hist_abs[threadIdx.x], ha);
        if (hr) atomicAdd(&acc->hist_rel[threadIdx.x], hr);
    }
    if (threadIdx.x == 0) {
        if (sm.viol) atomicAdd(&acc->n_viol, sm.viol);
        if (sm.border) atomicAdd(&acc->n_border, sm.border);
        if (sm.nonfin) atomicAdd(&acc->n_nonfinite, sm.nonfin);
        if (sm.maxr > 0.0)
            atomicMax(&acc->max_ratio_bits, (unsigned long long)__double_as_longlong(sm.maxr));
        __threadfence();
        sm.is_last = atomicAdd(&acc->blocks_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!sm.is_last) return;

    // ---- last block: decide all 2G targets, settle ambiguous ones exactly
    __threadfence();
    decide_targets(p.v, n, acc->hist_abs, acc->hist_rel, sm.vs, false);
    if (sm.vs.n_amb > 0) {
        settle_ambiguous(p.v, p.local, p.claimed, n, sm.vs);
        decide_targets(p.v, n, acc->hist_abs, acc->hist_rel, sm.vs, true);
    }
    if (threadIdx.x == 0) {
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
    // leave the accumulator zeroed for the next call on this stream
    unsigned long long* z = reinterpret_cast<unsigned long long*>(acc);
    for (int i = threadIdx.x; i < (int)(sizeof(CheckAccum) / 8); i += blockDim.x) z[i] = 0ull;
}

// ------------------------------------------------------- exact percentiles

struct FinalParams {
    int G;
    int64_t n;
    double grid[kMaxGrid];
};

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

int fill_verdict_spec(VerdictSpec& v, const double* grid, const double* tau_abs,
                      const double* tau_rel, int n_grid, double epsilon) {
    NAO_REQUIRE(n_grid > 0 && n_grid <= kMaxGrid, "grid size %d out of range (1..%d)", n_grid,
                kMaxGrid);
    NAO_REQUIRE(grid && tau_abs && tau_rel, "null grid/threshold array");
    memset(&v, 0, sizeof v);
    v.G = n_grid;
    v.epsilon = epsilon;
    double sa[kMaxGrid], sr[kMaxGrid];
    for (int i = 0; i < n_grid; i++) {
        NAO_REQUIRE(std::isfinite(grid[i]) && grid[i] >= 0.0 && grid[i] <= 100.0,
                    "Percentiles must be in the range [0, 100]");
        v.grid[i] = grid[i];
        v.tau_abs[i] = sa[i] = tau_abs[i] > 0.0 ? tau_abs[i] : 0.0;
        v.tau_rel[i] = sr[i] = tau_rel[i] > 0.0 ? tau_rel[i] : 0.0;
    }
    std::sort(sa, sa + n_grid);
    std::sort(sr, sr + n_grid);
    for (int i = 0; i < n_grid; i++) {
        v.t_abs[i] = sa[i];
        v.t_rel[i] = sr[i];
        v.lpos_abs[i] = (int)(std::lower_bound(sa, sa + n_grid, v.tau_abs[i]) - sa);
        v.lpos_rel[i] = (int)(std::lower_bound(sr, sr + n_grid, v.tau_rel[i]) - sr);
    }
    return NAO_OK;
}

}  // namespace nao

using namespace nao;

extern "C" {

size_t nao_check_workspace(void) { return sizeof(CheckAccum) + 256; }

size_t nao_verdict_spec_bytes(void) { return sizeof(VerdictSpec); }

int nao_verdict_spec_fill(void* spec_host, const double* grid, const double* tau_abs,
                          const double* tau_rel, int n_grid, double epsilon) {
    NAO_REQUIRE(spec_host != nullptr, "spec buffer is null");
    return fill_verdict_spec(*static_cast<VerdictSpec*>(spec_host), grid, tau_abs, tau_rel,
                             n_grid, epsilon);
}

int nao_check(const float* local, const float* claimed, int64_t n, int eps_kind, const void* eps,
              double eps_scale, double lo_factor, const double* grid, const double* tau_abs,
              const double* tau_rel, int n_grid, double epsilon, nao_check_result* result,
              void* workspace, size_t workspace_bytes, uint64_t* border_list,
              int64_t border_cap, void* stream) {
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
    NAO_REQUIRE(n_grid > 0 && n_grid <= kMaxGrid, "grid size %d out of range (1..%d)", n_grid,
                kMaxGrid);
    Workspace ws(workspace, workspace_bytes);
    CheckAccum* acc = ws.take<CheckAccum>(1);
    NAO_REQUIRE(acc != nullptr, "workspace too small");
    static thread_local CheckParams p;
    memset(&p, 0, sizeof p);
    p.local = local; p.claimed = claimed; p.eps = eps; p.n = n; p.eps_kind = eps_kind;
    p.eps_scale = eps_scale; p.lo_factor = lo_factor;
    NAO_REQUIRE(lo_factor > 0.0 && lo_factor <= 1.0, "lo_factor %g out of (0, 1]", lo_factor);
    NAO_REQUIRE(border_list == nullptr || border_cap >= 0, "bad borderline list capacity");
    p.border = reinterpret_cast<unsigned long long*>(border_list);
    p.border_cap = (long long)border_cap;
    int rc = fill_verdict_spec(p.v, grid, tau_abs, tau_rel, n_grid, epsilon);
    if (rc) return rc;
    // one resident wave: 3 CTAs per SM (launch bounds), each warp 64 float4 per step
    const int64_t warps_needed = ((n >> 2) + 63) / 64;
    const int blocks = (int)std::max<int64_t>(
        1, std::min<int64_t>((warps_needed + kCheckWarps - 1) / kCheckWarps, kNumSMs * 3));
    switch (eps_kind) {
        case NAO_EPS_TENSOR_F32:
            k_check<NAO_EPS_TENSOR_F32><<<blocks, kCheckThreads, 0, st>>>(p, acc, result); break;
        case NAO_EPS_TENSOR_F64:
            k_check<NAO_EPS_TENSOR_F64><<<blocks, kCheckThreads, 0, st>>>(p, acc, result); break;
        case NAO_EPS_SCALED_LOCAL:
            k_check<NAO_EPS_SCALED_LOCAL><<<blocks, kCheckThreads, 0, st>>>(p, acc, result); break;
        default:
            k_check<NAO_EPS_ZERO><<<blocks, kCheckThreads, 0, st>>>(p, acc, result); break;
    }
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
