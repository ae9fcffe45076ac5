// One SOV step on the device: Eq. 2 and the factor of Eq. 3,
//   q = Phi(b') - Phi(a'),  y = Phi^{-1}(Phi(a') + w q)
// evaluated tail-aware (reading R9) with CUDA's fp64 erfc / erfcinv / erfcx / log1p.
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
__device__ __noinline__ double log_Phi_hi_far(double x) { return log(0.5 * erfcx(x * kRsqrt2)) - 0.5 * x * x; }

// Solve log P(Z > y) = T for y >= x0 (x0 >= kFarTail, log P(Z > x0) >= T). Newton from the left
// end point; the function is concave decreasing, so after one step the iterates decrease
// monotonically onto the root and stay in the far-tail domain.
__device__ __noinline__ double Phi_hi_inv_far(double T, double x0) {
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

__device__ __noinline__ void sov_step_far_upper(double ap, double bp, double w, double &logq, double &y) {
    double la = log_Phi_hi_far(ap);
    double lb = isinf(bp) ? -CUDART_INF : log_Phi_hi_far(bp);
    logq = isinf(lb) ? la : la + log1p(-exp(lb - la));
    double t = log1p(-w) + logq;                        // log((1-w) q)
    double lp;                                          // log(Phibar(b') + (1-w) q)
    if (isinf(lb)) lp = t;
    else { double m = fmax(lb, t); lp = m + log1p(exp(-fabs(lb - t))); }
    y = Phi_hi_inv_far(lp, ap);
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
    y = (plo < phi) ? -kSqrt2 * erfcinv(2.0 * plo) : kSqrt2 * erfcinv(2.0 * phi);
}

// Upper-exceedance fast path (b = +inf, every BASELINE config): Phibar(b') = 0.
__device__ __forceinline__ void sov_step_upper(double ap, double w, double &logq, double &y) {
    if (ap >= kFarTail) { sov_step_far_upper(ap, CUDART_INF, w, logq, y); return; }
    double q, d;
    if (ap >= 0.0) {
        q = Phi_hi(ap);
        d = 0.0;              // unused: p_lo >= 1/2 > p_hi below
        logq = log(q);
        y = kSqrt2 * erfcinv(2.0 * ((1.0 - w) * q));
        return;
    }
    d = isinf(ap) ? 0.0 : Phi_lo(ap);
    q = 1.0 - d;
    logq = log1p(-d);                                  // q > 1/2 here
    const double plo = d + w * q;
    const double phi = (1.0 - w) * q;
    y = (plo < phi) ? -kSqrt2 * erfcinv(2.0 * plo) : kSqrt2 * erfcinv(2.0 * phi);
}

}  // namespace mvn
