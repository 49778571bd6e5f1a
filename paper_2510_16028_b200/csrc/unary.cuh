// FP64 intrinsics of the reference (engine.py:133-154, _unary_intrinsic) and
// the envelope of FP32 results a different faithful libm could give.
//
// The reference evaluates exp/log/tanh/x**3 with numpy's FP64 SIMD loops,
// which are not correctly rounded and differ across CPUs (measured here:
// numpy tanh within 3 ulp of glibc, x**3 off the correctly rounded cube on
// 2.8 % of inputs).  One FP32 rounding hides those differences unless the
// FP64 value sits within a few ulps of an FP32 rounding boundary -- or, for
// gelu, unless 1 + tanh(inner) cancels (x << 0), where the FP64 noise of
// tanh becomes a large relative error of the result.  unary_eval returns
// this GPU's value and the range [lo, hi] of FP32 results reachable by any
// evaluation inside the envelope; lo != hi marks a value-ambiguous element
// (its verdict is settled by nao_refine_borderline, its bound taken at the
// largest candidate).
#pragma once
#include "common.cuh"

namespace nao {

constexpr double kGeluS = 0.7978845608028654;  // math.sqrt(2/pi)  (engine.py:23)
constexpr double kGeluC = 0.044715;            // engine.py:24
// relative envelope of one FP64 libm call (this GPU's <= 2 ulp plus numpy's
// <= 4 ulp, doubled); 1 ulp <= 2^-52 relative
constexpr double kLibmRel = 16.0 * 0x1p-52;

struct UnaryOut {
    double v;        // this GPU's FP64 value
    float y;         // (float)v: the value used
    float lo, hi;    // FP32 results reachable inside the envelope (lo <= hi)
};

// FP32 roundings of every FP64 value within [v - r|v|, v + r|v|]
__device__ __forceinline__ void env_round(double v, double r, float& lo, float& hi) {
    if (!isfinite(v) || v == 0.0) { lo = hi = (float)v; return; }
    const double d = __dmul_ru(r, fabs(v));
    lo = __double2float_rn(__dsub_rd(v, d));
    hi = __double2float_rn(__dadd_ru(v, d));
}

__device__ __forceinline__ UnaryOut unary_eval(int kind, float xf) {
    const double x = (double)xf;
    UnaryOut o;
    switch (kind) {
        case NAO_UN_EXP: o.v = exp(x); env_round(o.v, kLibmRel, o.lo, o.hi); break;
        case NAO_UN_LOG: o.v = log(x); env_round(o.v, kLibmRel, o.lo, o.hi); break;
        case NAO_UN_SQRT:  // IEEE sqrt: correctly rounded everywhere
            o.v = __dsqrt_rn(x); o.lo = o.hi = (float)o.v; break;
        case NAO_UN_RSQRT:  // 1.0 / np.sqrt: two correctly rounded operations
            o.v = __ddiv_rn(1.0, __dsqrt_rn(x)); o.lo = o.hi = (float)o.v; break;
        case NAO_UN_TANH: o.v = tanh(x); env_round(o.v, kLibmRel, o.lo, o.hi); break;
        case NAO_UN_GELU: {
            // 0.5 * x * (1 + tanh(S * (x + C * x**3))); x*x is exact (FP32 x),
            // so x*x*x is the correctly rounded cube; numpy's x**3 is within 2 ulp
            const double x3 = __dmul_rn(__dmul_rn(x, x), x);
            const double inner = __dmul_rn(kGeluS, __dadd_rn(x, __dmul_rn(kGeluC, x3)));
            const double t = tanh(inner);
            const double w = __dadd_rn(1.0, t);
            const double h = __dmul_rn(0.5, x);  // exact
            o.v = __dmul_rn(h, w);
            if (!isfinite(o.v)) { o.lo = o.hi = (float)o.v; break; }
            // inner: x**3 (2 ulp) + 3 roundings -> <= 8 ulp relative; tanh' = 1 - t^2
            // <= 2 (1 - |t|); tanh itself: kLibmRel; 1 + t: one rounding
            const double r_in = 8.0 * 0x1p-52;
            const double dt = __dadd_ru(__dmul_ru(__dmul_ru(2.0, __dsub_ru(1.0, fabs(t))),
                                                  __dmul_ru(fabs(inner), r_in)),
                                        __dmul_ru(kLibmRel, fabs(t)));
            const double dw = __dadd_ru(dt, __dmul_ru(0x1p-52, fabs(w)));
            const double wlo = fmax(0.0, __dsub_rd(w, dw)), whi = __dadd_ru(w, dw);
            // y = h w (one rounding): the extremes over [wlo, whi], widened by 2 ulp
            const double ya = __dmul_rn(h, wlo), yb = __dmul_rn(h, whi);
            const double ymin = fmin(ya, yb), ymax = fmax(ya, yb);
            o.lo = __double2float_rn(__dsub_rd(ymin, __dmul_ru(0x1p-51, fabs(ymin))));
            o.hi = __double2float_rn(__dadd_ru(ymax, __dmul_ru(0x1p-51, fabs(ymax))));
            break;
        }
        default: {  // silu: x / (1 + exp(-x))
            const double e = exp(-x);
            o.v = __ddiv_rn(x, __dadd_rn(1.0, e));
            env_round(o.v, kLibmRel + 4.0 * 0x1p-52, o.lo, o.hi);
            break;
        }
    }
    o.y = (float)o.v;
    // the chosen value always lies in the range
    if (o.y < o.lo) o.lo = o.y;
    if (o.y > o.hi) o.hi = o.y;
    return o;
}

// FP64 result of the reference's fp64=True path (no FP32 rounding)
__device__ __forceinline__ double unary_f64(int kind, double x) {
    switch (kind) {
        case NAO_UN_EXP: return exp(x);
        case NAO_UN_LOG: return log(x);
        case NAO_UN_SQRT: return __dsqrt_rn(x);
        case NAO_UN_RSQRT: return __ddiv_rn(1.0, __dsqrt_rn(x));
        case NAO_UN_TANH: return tanh(x);
        case NAO_UN_GELU: {
            const double x3 = __dmul_rn(__dmul_rn(x, x), x);
            const double inner = __dmul_rn(kGeluS, __dadd_rn(x, __dmul_rn(kGeluC, x3)));
            return __dmul_rn(__dmul_rn(0.5, x), __dadd_rn(1.0, tanh(inner)));
        }
        default: return __ddiv_rn(x, __dadd_rn(1.0, exp(-x)));
    }
}

__device__ __forceinline__ bool fbits_differ(float a, float b) {
    return __float_as_uint(a) != __float_as_uint(b);
}

// append a flat index to a borderline / ambiguity list (count always grows)
__device__ __forceinline__ void list_push(unsigned long long* list, long long cap, unsigned long long idx) {
    const unsigned long long pos = atomicAdd(list, 1ull);
    if (pos < (unsigned long long)cap) list[1 + pos] = idx;
}

}  // namespace nao
