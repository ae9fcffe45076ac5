// One SOV step on the device: Eq. 2 and the factor of Eq. 3,
//   q = Phi(b') - Phi(a'),  y = Phi^{-1}(Phi(a') + w q)
// evaluated tail-aware (reading R9) with CUDA's fp64 erfc / erfcx / log1p and Wichura's
// AS 241 rational Phi^{-1} (the oracle uses Halley iterations on erfc instead: independent paths).
// Alg. 3 lines 4 and 11 print Phi^{-1}[R (Phi(B) - Phi(A))] without "+Phi(A)"; Eq. 2 governs (R4).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

namespace mvn {

constexpr double kFarTail = 35.0;  // |limit| beyond which Phibar underflows toward subnormals
constexpr double kRsqrt2 = 0.70710678118654752440;
constexpr double kSqrt2 = 1.41421356237309504880;

__device__ __forceinline__ double Phi_lo(double x) { return 0.5 * erfc(-x * kRsqrt2); }   // P(Z <= x)
__device__ __forceinline__ double Phi_hi(double x) { return 0.5 * erfc(x * kRsqrt2); }    // P(Z > x)

// log P(Z > x) for x >= kFarTail: P(Z > x) = erfcx(x/sqrt2)/2 * exp(-x^2/2)
static __device__ __noinline__ double log_Phi_hi_far(double x) { return log(0.5 * erfcx(x * kRsqrt2)) - 0.5 * x * x; }

// Solve log P(Z > y) = T for y >= x0 (x0 >= kFarTail, log P(Z > x0) >= T). Newton from the left
// end point; the function is concave decreasing, so after one step the iterates decrease
// monotonically onto the root and stay in the far-tail domain.
static __device__ __noinline__ double Phi_hi_inv_far(double T, double x0) {
    double y = x0;
    for (int it = 0; it < 60; ++it) {
        double g = log_Phi_hi_far(y) - T;
        double gp = -0.79788456080286535588 / erfcx(y * kRsqrt2);  // -sqrt(2/pi)/erfcx
        double step = g / gp;
        y -= step;
        if (fabs(step) <= 1e-17 * y) break;
    }
    return y;
}

static __device__ __noinline__ void sov_step_far_upper(double ap, double bp, double w, double &logq, double &y) {
    double la = log_Phi_hi_far(ap);
    double lb = isinf(bp) ? -CUDART_INF : log_Phi_hi_far(bp);
    logq = isinf(lb) ? la : la + log1p(-exp(lb - la));
    double t = log1p(-w) + logq;                        // log((1-w) q)
    double lp;                                          // log(Phibar(b') + (1-w) q)
    if (isinf(lb)) lp = t;
    else { double m = fmax(lb, t); lp = m + log1p(exp(-fabs(lb - t))); }
    y = Phi_hi_inv_far(lp, ap);
}

// Phi^{-1}(p) for 0 < p <= 1/2 (+ rounding): Wichura's AS 241 (PPND16) rational approximations,
// relative error <= 6.1e-16 on [1e-300, 0.5] (checked against mpmath, tests/test_ppnd16_coeffs.py).
// Straight-line code (one log, one sqrt, one division), far shorter than the general erfcinv.
__device__ __forceinline__ double Phi_inv_lower(double p) {
    const double q = p - 0.5;
    if (fabs(q) <= 0.425) {
        const double r = 0.180625 - q * q;
        const double num = ((((((2.5090809287301226727e+3 * r + 3.3430575583588128105e+4) * r + 6.7265770927008700853e+4) * r +
                               4.5921953931549871457e+4) * r + 1.3731693765509461125e+4) * r + 1.9715909503065514427e+3) * r +
                             1.3314166789178437745e+2) * r + 3.3871328727963666080e0;
        const double den = ((((((5.2264952788528545610e+3 * r + 2.8729085735721942674e+4) * r + 3.9307895800092710610e+4) * r +
                               2.1213794301586595867e+4) * r + 5.3941960214247511077e+3) * r + 6.8718700749205790830e+2) * r +
                             4.2313330701600911252e+1) * r + 1.0;
        return q * num / den;
    }
    double r = sqrt(-log(p));
    double num, den;
    if (r <= 5.0) {
        r -= 1.6;
        num = ((((((7.74545014278341407640e-4 * r + 2.27238449892691845833e-2) * r + 2.41780725177450611770e-1) * r +
                  1.27045825245236838258e0) * r + 3.64784832476320460504e0) * r + 5.76949722146069140550e0) * r +
                4.63033784615654529590e0) * r + 1.42343711074968357734e0;
        den = ((((((1.05075007164441684324e-9 * r + 5.47593808499534494600e-4) * r + 1.51986665636164571966e-2) * r +
                  1.48103976427480074590e-1) * r + 6.89767334985100004550e-1) * r + 1.67638483018380384940e0) * r +
                2.05319162663775882187e0) * r + 1.0;
    } else {
        r -= 5.0;
        num = ((((((2.01033439929228813265e-7 * r + 2.71155556874348757815e-5) * r + 1.24266094738807843860e-3) * r +
                  2.65321895265761230930e-2) * r + 2.96560571828504891230e-1) * r + 1.78482653991729133580e0) * r +
                5.46378491116411436990e0) * r + 6.65790464350110377720e0;
        den = ((((((2.04426310338993978564e-15 * r + 1.42151175831644588870e-7) * r + 1.84631831751005468180e-5) * r +
                  7.86869131145613259100e-4) * r + 1.48753612908506148525e-2) * r + 1.36929880922735805310e-1) * r +
                5.99832206555887937690e-1) * r + 1.0;
    }
    return -num / den;
}

// General limits (finite b allowed). ap/bp may be +-inf.
__device__ __forceinline__ void sov_step(double ap, double bp, double w, double &logq, double &y) {
    if (!(ap < bp)) { logq = -CUDART_INF; y = ap; return; }
    if (ap >= kFarTail) { sov_step_far_upper(ap, bp, w, logq, y); return; }
    if (bp <= -kFarTail) {   // reflection x -> -x, w -> 1-w
        double yr;
        sov_step_far_upper(-bp, -ap, 1.0 - w, logq, yr);
        y = -yr;
        return;
    }
    const double d = isinf(ap) ? 0.0 : Phi_lo(ap);
    const double eb = isinf(bp) ? 0.0 : Phi_hi(bp);
    double q;
    if (ap >= 0.0) {
        q = Phi_hi(ap) - eb;
        logq = log(q);
    } else if (bp <= 0.0) {
        q = Phi_lo(bp) - d;
        logq = log(q);
    } else {
        const double s = d + eb;
        q = 1.0 - s;
        logq = (q > 0.5) ? log1p(-s) : log(q);
    }
    const double plo = d + w * q;
    const double phi = eb + (1.0 - w) * q;
    y = (plo < phi) ? Phi_inv_lower(plo) : -Phi_inv_lower(phi);
}

// Phi^{-1}(p) for 0 < p <= 1/2, the same AS 241 rational approximations as Phi_inv_lower but
// evaluated without branches: the central and the tail forms are both computed and selected, the
// two tail coefficient sets (r <= 5, r > 5) are selected per lane. In a warp whose lanes fall in
// different regions this costs one evaluation of each form instead of a divergent replay, and it
// needs one division instead of two.
__device__ __forceinline__ double Phi_inv_lower_nb(double p) {
    const double q = p - 0.5;
    const double rc = 0.180625 - q * q;
    const double numc = ((((((2.5090809287301226727e+3 * rc + 3.3430575583588128105e+4) * rc + 6.7265770927008700853e+4) * rc +
                            4.5921953931549871457e+4) * rc + 1.3731693765509461125e+4) * rc + 1.9715909503065514427e+3) * rc +
                          1.3314166789178437745e+2) * rc + 3.3871328727963666080e0;
    const double denc = ((((((5.2264952788528545610e+3 * rc + 2.8729085735721942674e+4) * rc + 3.9307895800092710610e+4) * rc +
                            2.1213794301586595867e+4) * rc + 5.3941960214247511077e+3) * rc + 6.8718700749205790830e+2) * rc +
                          4.2313330701600911252e+1) * rc + 1.0;
    const double rt = sqrt(-log(p));
    const bool far = rt > 5.0;
    const double x = rt - (far ? 5.0 : 1.6);
#define MVN_SEL(a2, a3) (far ? (a3) : (a2))
    const double numt =
        ((((((MVN_SEL(7.74545014278341407640e-4, 2.01033439929228813265e-7) * x + MVN_SEL(2.27238449892691845833e-2, 2.71155556874348757815e-5)) * x +
             MVN_SEL(2.41780725177450611770e-1, 1.24266094738807843860e-3)) * x + MVN_SEL(1.27045825245236838258e0, 2.65321895265761230930e-2)) * x +
           MVN_SEL(3.64784832476320460504e0, 2.96560571828504891230e-1)) * x + MVN_SEL(5.76949722146069140550e0, 1.78482653991729133580e0)) * x +
         MVN_SEL(4.63033784615654529590e0, 5.46378491116411436990e0)) * x + MVN_SEL(1.42343711074968357734e0, 6.65790464350110377720e0);
    const double dent =
        ((((((MVN_SEL(1.05075007164441684324e-9, 2.04426310338993978564e-15) * x + MVN_SEL(5.47593808499534494600e-4, 1.42151175831644588870e-7)) * x +
             MVN_SEL(1.51986665636164571966e-2, 1.84631831751005468180e-5)) * x + MVN_SEL(1.48103976427480074590e-1, 7.86869131145613259100e-4)) * x +
           MVN_SEL(6.89767334985100004550e-1, 1.48753612908506148525e-2)) * x + MVN_SEL(1.67638483018380384940e0, 1.36929880922735805310e-1)) * x +
         MVN_SEL(2.05319162663775882187e0, 5.99832206555887937690e-1)) * x + 1.0;
#undef MVN_SEL
    const bool central = fabs(q) <= 0.425;
    return (central ? q * numc : -numt) / (central ? denc : dent);
}

// Upper-exceedance fast path (b = +inf, every BASELINE config): Phibar(b') = 0.
// One erfc for both signs of a' (t = Phibar(|a'|)), one log, one Phi^{-1} call site:
//   a' >= 0: q = t,      log q = log t,             y = -Phi^{-1}((1-w) q)
//   a' <  0: q = 1 - t,  log q = log1p(-t),          y = Phi^{-1}(min(t + w q, (1-w) q)) (signed)
// log1p(-t) is formed as log(v) - delta (2 - v) with v = fl(1 - t) in [1/2, 1) and
// delta = (v - 1) + t the exact rounding error of 1 - t (first-order correction; error <= 2^-55
// absolute), so both signs share one log.
__device__ __forceinline__ void sov_step_upper(double ap, double w, double &logq, double &y, double &q) {
    if (ap >= kFarTail) { sov_step_far_upper(ap, CUDART_INF, w, logq, y); q = exp(logq); return; }
    const bool pos = ap >= 0.0;
    const double t = isinf(ap) ? 0.0 : 0.5 * erfc(fabs(ap) * kRsqrt2);
    const double v = pos ? t : 1.0 - t;                  // q
    const double delta = pos ? 0.0 : (v - 1.0) + t;
    logq = log(v) - delta * (2.0 - v);
    const double phi = (1.0 - w) * v;
    const double plo = pos ? 1.0 : t + w * v;            // a' >= 0: p_lo >= 1/2 >= p_hi
    const bool lower = plo < phi;
    const double r = Phi_inv_lower_nb(lower ? plo : phi);
    y = lower ? r : -r;
    q = v;
}

}  // namespace mvn
