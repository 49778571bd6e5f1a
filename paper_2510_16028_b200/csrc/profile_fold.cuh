// Device-profile reduction orders (engine.py:75-113).
// fold_profile(at, n, p) sums at(0..n-1) in FP32 (round to nearest, no FMA)
// in exactly the order the reference's reduce_last_axis uses:
//   sequential : (((a0 + a1) + a2) + ...)
//   pairwise   : pw(a[0:n]) = pw(a[0:m]) + pw(a[m:n]), m = ceil(n/2)  (engine.py:87-92)
//   blocked(b) : sequential folds of consecutive b-blocks, then a sequential
//                fold of the block sums                        (engine.py:104-110)
//   permuted   : sequential fold of a[perm[0]], a[perm[1]], ... (engine.py:111-112);
//                perm is the host-computed numpy Philox permutation (:75-77)
#pragma once
#include "common.cuh"

namespace nao {

struct Prof {
    int order;            // NAO_ORDER_*
    int block;            // blocked
    const int64_t* perm;  // permuted (device)
};

__host__ inline Prof make_prof(const nao_profile* p) {
    Prof q{NAO_ORDER_SEQUENTIAL, 32, nullptr};
    if (p) { q.order = p->order; q.block = p->block_size; q.perm = p->perm; }
    return q;
}

// host validation of a descriptor for a reduced length n
#define NAO_CHECK_PROFILE(p, n)                                                               \
    do {                                                                                      \
        if (p) {                                                                              \
            NAO_REQUIRE((p)->order >= NAO_ORDER_SEQUENTIAL && (p)->order <= NAO_ORDER_PERMUTED, \
                        "unknown reduction order %d", (p)->order);                            \
            NAO_REQUIRE((p)->order != NAO_ORDER_PERMUTED ||                                   \
                            ((p)->perm != nullptr && (p)->perm_n == (int64_t)(n)),            \
                        "permuted profile: permutation of length %lld required",              \
                        (long long)(n));                                                      \
        }                                                                                     \
    } while (0)

template <class At>
__device__ float fold_profile(const At& at, int64_t n, const Prof& p) {
    if (p.order == NAO_ORDER_PAIRWISE) {
        // post-order walk of the recursive-halving tree with an explicit stack
        struct Frame { int64_t lo, len; float left; int state; };
        Frame st[64];
        int sp = 0;
        st[sp++] = {0, n, 0.f, 0};
        float ret = 0.f;
        while (sp > 0) {
            Frame& f = st[sp - 1];
            if (f.len == 1) { ret = at(f.lo); sp--; continue; }
            const int64_t mid = (f.len + 1) / 2;
            if (f.state == 0) { f.state = 1; st[sp++] = {f.lo, mid, 0.f, 0}; continue; }
            if (f.state == 1) { f.left = ret; f.state = 2; st[sp++] = {f.lo + mid, f.len - mid, 0.f, 0}; continue; }
            ret = __fadd_rn(f.left, ret);
            sp--;
        }
        return ret;
    }
    if (p.order == NAO_ORDER_BLOCKED) {
        const int64_t b = p.block > 1 ? p.block : 1;
        float acc = 0.f;
        for (int64_t i = 0; i < n; i += b) {
            float part = at(i);
            const int64_t e = i + b < n ? i + b : n;
            for (int64_t k = i + 1; k < e; k++) part = __fadd_rn(part, at(k));
            acc = (i == 0) ? part : __fadd_rn(acc, part);
        }
        return acc;
    }
    if (p.order == NAO_ORDER_PERMUTED) {
        float acc = at(p.perm[0]);
        for (int64_t k = 1; k < n; k++) acc = __fadd_rn(acc, at(p.perm[k]));
        return acc;
    }
    float acc = at(0);
    for (int64_t k = 1; k < n; k++) acc = __fadd_rn(acc, at(k));
    return acc;
}

}  // namespace nao
