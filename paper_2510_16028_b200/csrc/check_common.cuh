// Shared pieces of the acceptance check: exact
// FP64 error keys, numpy's "linear" percentile index and _lerp, the per-node
// verdict spec (thresholds on the grid) and the histogram verdict.  Used by
// the standalone check (check.cu) and the check fused into the Merkle commit
// (merkle.cu, nao_commit_check_tensors).
#pragma once
#include "common.cuh"

namespace nao {

constexpr int kMaxGrid = 32;

// Per-node verdict spec (include/nao_b200.h nao_verdict_spec_*): effective
// thresholds in grid order and ascending, for the one-pass histogram verdict.
struct VerdictSpec {
    int32_t G;
    int32_t pad_;
    double epsilon;               // relative-error guard (calibration.py:19)
    double grid[kMaxGrid];
    double tau_abs[kMaxGrid];     // effective thresholds (tau <= 0 -> 0), grid order
    double tau_rel[kMaxGrid];
    double t_abs[kMaxGrid];       // the same, sorted ascending
    double t_rel[kMaxGrid];
    int32_t lpos_abs[kMaxGrid];   // #{sorted t < tau_i}
    int32_t lpos_rel[kMaxGrid];
};

// Device accumulator of one check (zero before use; the finalizing CTA zeroes it again).
struct CheckAccum {
    unsigned long long n_viol, n_border, n_nonfinite;
    unsigned long long hist_abs[kMaxGrid + 1];
    unsigned long long hist_rel[kMaxGrid + 1];
    unsigned long long max_ratio_bits;        // non-negative double
    unsigned long long amb_lo[2 * kMaxGrid];  // max key <= tau (double bits)
    unsigned long long amb_hi[2 * kMaxGrid];  // min key >  tau (double bits)
    // partial mode (combinable records): per-bucket key range; min stored as
    // max of ~bits so that the zero state means "empty"
    unsigned long long bmax[2][kMaxGrid + 1];
    unsigned long long bmin_inv[2][kMaxGrid + 1];
    unsigned int blocks_done;
    unsigned int pad_;
};

// Host: fill a spec from the grid and the node's thresholds (ratio obs/tau > 1
// <=> obs > tau for tau > 0, obs > 0 for tau <= 0: dispute.py:114-127).
int fill_verdict_spec(VerdictSpec& v, const double* grid, const double* tau_abs,
                      const double* tau_rel, int n_grid, double epsilon);

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

// Block-level verdict scratch (shared memory).
struct VerdictSmem {
    int amb[2 * kMaxGrid];
    int n_amb, exceeded, first;
    unsigned long long amb_lo[2 * kMaxGrid], amb_hi[2 * kMaxGrid];
};

// Decide every (array, grid point) from the interval histograms: the
// percentile exceeds tau iff fewer than k+1 keys are <= tau (k = prev index;
// the "last" case: fewer than n).  Exactly k+1 keys <= tau is ambiguous in
// phase 1 (flagged in vs.amb) and settled in phase 2 from amb_lo / amb_hi
// (max key <= tau, min key > tau) with numpy's _lerp.  All threads call.
__device__ inline void decide_targets(const VerdictSpec& v, int64_t n,
                                      const volatile unsigned long long* hist_abs,
                                      const volatile unsigned long long* hist_rel,
                                      VerdictSmem& vs, bool phase2) {
    const int G = v.G;
    const int t = threadIdx.x;
    if (t == 0) { vs.n_amb = 0; vs.exceeded = 0; vs.first = 0x7fffffff; }
    __syncthreads();
    if (t < 2 * G) {
        const int arr = t / G, i = t % G;
        const volatile unsigned long long* hist = arr == 0 ? hist_abs : hist_rel;
        const double tau = arr == 0 ? v.tau_abs[i] : v.tau_rel[i];
        const int L = arr == 0 ? v.lpos_abs[i] : v.lpos_rel[i];
        unsigned long long cle = 0;
        for (int b = 0; b <= L; b++) cle += hist[b];
        const VIdx x = virtual_index(n, v.grid[i]);
        bool ex;
        if (x.last) ex = cle < (unsigned long long)n;
        else if (cle <= (unsigned long long)x.prev) ex = true;
        else if (cle >= (unsigned long long)x.prev + 2) ex = false;
        else if (!phase2) { vs.amb[arr * kMaxGrid + i] = 1; atomicAdd(&vs.n_amb, 1); ex = false; }
        else {
            const double a = __longlong_as_double((long long)vs.amb_lo[arr * kMaxGrid + i]);
            const double b = __longlong_as_double((long long)vs.amb_hi[arr * kMaxGrid + i]);
            ex = np_lerp(a, b, x.g) > tau;
        }
        if (ex) { atomicOr(&vs.exceeded, 1); atomicMin(&vs.first, arr * G + i); }
    }
    __syncthreads();
}

// Phase 2 (rare): one block rescans the tensor for the ambiguous targets.
__device__ inline void settle_ambiguous(const VerdictSpec& v, const float* local,
                                        const float* claimed, int64_t n, VerdictSmem& vs) {
    const int G = v.G;
    if (threadIdx.x < 2 * kMaxGrid) {
        vs.amb_lo[threadIdx.x] = 0ull;
        vs.amb_hi[threadIdx.x] = 0x7ff0000000000000ull;  // +inf
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const float y = local[i], c = claimed[i];
        const double diff = abs_key(y, c);
        const double rel = rel_key(diff, y, v.epsilon);
        for (int t = 0; t < 2 * G; t++) {
            const int arr = t / G, gi = t % G;
            if (!vs.amb[arr * kMaxGrid + gi]) continue;
            const double key = arr == 0 ? diff : rel;
            const double tau = arr == 0 ? v.tau_abs[gi] : v.tau_rel[gi];
            const unsigned long long bits = (unsigned long long)__double_as_longlong(key);
            if (key <= tau) atomicMax(&vs.amb_lo[arr * kMaxGrid + gi], bits);
            else atomicMin(&vs.amb_hi[arr * kMaxGrid + gi], bits);
        }
    }
    __syncthreads();
}

}  // namespace nao
