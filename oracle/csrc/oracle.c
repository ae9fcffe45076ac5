/*
 * ORACLE (test infrastructure only) — plain, slow, obviously-correct CPU reference for the
 * hot path of arXiv 2405.14892 ("Parallel Approximations for High-Dimensional Multivariate
 * Normal Probability Computation in Confidence Region Detection Applications").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library. The product path (paper_2405_14892_b200/) never links or calls it, and this
 * file shares no code, header, table or constant generator with the CUDA library.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; R-numbers = the readings listed in DESIGN.md
 * ("Readings of the paper"), which follow SURVEY.md §8(c).
 *
 * Build: gcc -O2 -fno-fast-math -ffp-contract=off -fopenmp -shared -fPIC (see oracle/__init__.py).
 * No BLAS, no intrinsics. Threads only split independent work (rows i of one Cholesky column,
 * independent QMC units); per-element arithmetic order never depends on the thread count.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_SQRT1_2 0.70710678118654752440  /* 1/sqrt(2) */
#define ORC_SQRT2PI 2.50662827463100050242  /* sqrt(2*pi) */
#define ORC_SQRTPI 1.77245385090551602730   /* sqrt(pi) */
/* Far-tail switch of R9: |limit| beyond which Phibar underflows toward subnormals. */
#define ORC_FAR_TAIL 35.0

/* ------------------------------------------------------------------------------------------ */
/* Univariate normal: Phi(x) = P(Z <= x) (Table I, "Univariate normal distribution      */
/* function"); computed from libm erfc, so both tails keep full relative accuracy.            */
/* ------------------------------------------------------------------------------------------ */
double orc_Phi(double x) { return 0.5 * erfc(-x * ORC_SQRT1_2); }
double orc_Phibar(double x) { return 0.5 * erfc(x * ORC_SQRT1_2); }

/* erfcx(z) = exp(z^2) erfc(z) for z >= 24 by the Laplace continued fraction
 *   erfc z = exp(-z^2)/sqrt(pi) * 1/(z + (1/2)/(z + 1/(z + (3/2)/(z + 2/(z + ...)))))
 * evaluated bottom-up with 40 terms (converged to < 1 ulp for z >= 24). Only the far tail of R9
 * (|x| >= 35, i.e. z >= 24.7) uses it. */
double orc_erfcx_far(double z)
{
    double f = z;
    for (int k = 40; k >= 1; --k) f = z + (0.5 * k) / f;
    return 1.0 / (ORC_SQRTPI * f);
}

/* log Phibar(x) for x >= ORC_FAR_TAIL: Phibar(x) = 1/2 erfcx(x/sqrt2) exp(-x^2/2). */
double orc_log_Phibar_far(double x)
{
    return log(0.5 * orc_erfcx_far(x * ORC_SQRT1_2)) - 0.5 * x * x;
}

/* Phi^{-1}(p) for 0 < p <= 1/2 (+ rounding): Abramowitz & Stegun 26.2.23 start (|err|<4.5e-4),
 * then Halley iterations on f(y) = Phi(y) - p, f' = phi(y), f'' = -y phi(y). Cubic convergence:
 * 5 steps reach the fixed point of the erfc-based residual. Independent of any erfcinv. */
double orc_Phiinv_lower(double p)
{
    double t = sqrt(-2.0 * log(p));
    double y = -(t - (2.515517 + 0.802853 * t + 0.010328 * t * t) /
                         (1.0 + 1.432788 * t + 0.189269 * t * t + 0.001308 * t * t * t));
    for (int it = 0; it < 6; ++it) {
        double f = orc_Phi(y) - p;
        double phi = exp(-0.5 * y * y) / ORC_SQRT2PI;
        double u = f / phi;
        y = y - u / (1.0 + 0.5 * y * u);
    }
    return y;
}

/* Far upper tail (R9): the y >= x0 with log Phibar(y) = T, where x0 >= ORC_FAR_TAIL and
 * log Phibar(x0) >= T. Newton on g(y) = log Phibar(y) - T, g'(y) = -sqrt(2/pi)/erfcx(y/sqrt2);
 * g is concave and decreasing, so the iterates approach the root monotonically from the right
 * after the first step and never leave the far-tail domain. */
double orc_Phibar_inv_far(double T, double x0)
{
    double y = x0;
    for (int it = 0; it < 60; ++it) {
        double g = orc_log_Phibar_far(y) - T;
        double gp = -sqrt(2.0 / 3.14159265358979323846) / orc_erfcx_far(y * ORC_SQRT1_2);
        double step = g / gp;
        y = y - step;
        if (fabs(step) <= 1e-17 * y) break;
    }
    return y;
}

static double orc_logaddexp(double x, double y)
{
    if (x == -INFINITY) return y;
    if (y == -INFINITY) return x;
    double m = x > y ? x : y;
    return m + log1p(exp(-fabs(x - y)));
}

/* Upper far tail of one SOV step: a' >= ORC_FAR_TAIL (so b' > a' too). Log-space throughout. */
static void orc_step_far_upper(double ap, double bp, double w, double *logq, double *y)
{
    double la = orc_log_Phibar_far(ap);
    double lb = (bp == INFINITY) ? -INFINITY : orc_log_Phibar_far(bp);
    /* q = Phibar(a') - Phibar(b') */
    *logq = (lb == -INFINITY) ? la : la + log1p(-exp(lb - la));
    /* p_hi = Phibar(b') + (1-w) q ;  y = Phibar^{-1}(p_hi) */
    double lphi = orc_logaddexp(lb, log1p(-w) + *logq);
    *y = orc_Phibar_inv_far(lphi, ap);
}

/* One step of the SOV recursion for one (row, sample): Eq. 2
 *   d = Phi(a'), e = Phi(b'), y = Phi^{-1}[d + w (e - d)], q = e - d   (factor of Eq. 3)
 * evaluated tail-aware as in reading R9: with ebar = Phibar(b'),
 *   a' >= 0: q = Phibar(a') - ebar;  b' <= 0: q = Phi(b') - d;  else q = 1 - (d + ebar);
 *   log q = log1p(-(d + ebar)) when q > 1/2 (middle case), else log(q);
 *   p_lo = d + w q, p_hi = ebar + (1-w) q;  y = Phi^{-1}(p_lo) if p_lo < p_hi else -Phi^{-1}(p_hi).
 * Far tails (a' >= 35 or b' <= -35) are evaluated in log space (upper tail directly, lower tail by
 * the reflection x -> -x, w -> 1-w). Empty interval a' >= b': q = 0, log q = -inf, y = a'. */
void orc_sov_step(double ap, double bp, double w, double *logq, double *y)
{
    if (!(ap < bp)) { *logq = -INFINITY; *y = ap; return; }
    if (ap >= ORC_FAR_TAIL) { orc_step_far_upper(ap, bp, w, logq, y); return; }
    if (bp <= -ORC_FAR_TAIL) {
        double yr;
        orc_step_far_upper(-bp, -ap, 1.0 - w, logq, &yr);
        *y = -yr;
        return;
    }
    double d = (ap == -INFINITY) ? 0.0 : orc_Phi(ap);
    double ebar = (bp == INFINITY) ? 0.0 : orc_Phibar(bp);
    double q, lq;
    if (ap >= 0.0) {
        q = orc_Phibar(ap) - ebar;
        lq = log(q);
    } else if (bp <= 0.0) {
        q = orc_Phi(bp) - d;
        lq = log(q);
    } else {
        double s = d + ebar;
        q = 1.0 - s;
        lq = (q > 0.5) ? log1p(-s) : log(q);
    }
    double plo = d + w * q;
    double phi = ebar + (1.0 - w) * q;
    *logq = lq;
    *y = (plo < phi) ? orc_Phiinv_lower(plo) : -orc_Phiinv_lower(phi);
}

/* ------------------------------------------------------------------------------------------ */
/* Cholesky (Alg. 1 line 8 "L <- dpotrf(Sigma)"; Sigma = L L^T): textbook        */
/* Cholesky-Crout, column by column:                                                           */
/*   L_jj = sqrt(S_jj - sum_{t<j} L_jt^2),  L_ij = (S_ij - sum_{t<j} L_it L_jt) / L_jj          */
/* A: n x n row-major; the lower triangle (i >= j) is read and overwritten with L; the strict  */
/* upper triangle is left untouched. Returns -1 on success, else the 0-based row j of the      */
/* first non-positive (or NaN) pivot (reading R17).                                            */
/* ------------------------------------------------------------------------------------------ */
long long orc_cholesky(long long n, double *A, int nthreads)
{
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    for (long long j = 0; j < n; ++j) {
        double *Aj = A + j * n;
        double d = Aj[j];
        for (long long t = 0; t < j; ++t) d -= Aj[t] * Aj[t];
        if (!(d > 0.0)) return j;
        double ljj = sqrt(d);
        Aj[j] = ljj;
#pragma omp parallel for schedule(static)
        for (long long i = j + 1; i < n; ++i) {
            double *Ai = A + i * n;
            double s = Ai[j];
            for (long long t = 0; t < j; ++t) s -= Ai[t] * Aj[t];
            Ai[j] = s / ljj;
        }
    }
    return -1;
}

/* ------------------------------------------------------------------------------------------ */
/* QMC point (reading R8): Richtmyer lattice with a random shift, exact in 64-bit integers:     */
/*   X = (j * G_k + D_k) mod 2^64,   w = (floor(X / 2^12) + 1/2) * 2^-52                        */
/* G_k = floor(frac(sqrt(p_k)) 2^64), D_k = the shift of row k for this unit's shift r. Both    */
/* are inputs (computed by oracle/lattice.py). w is an odd multiple of 2^-53, so w and 1-w are */
/* exact in fp64.                                                                              */
/* ------------------------------------------------------------------------------------------ */
double orc_lattice_w(uint64_t j, uint64_t G, uint64_t D)
{
    uint64_t X = j * G + D;
    return ((double)(X >> 12) + 0.5) * 0x1p-52;
}

/* ------------------------------------------------------------------------------------------ */
/* SOV sweep for one QMC unit (shift r, lattice indices j = j0 .. j0+J-1):                     */
/* Alg. 2 (PMVN) with Alg. 3 (QMC tile kernel) written out per sample    */
/* without tiling (tiles only reorder the same sums): for k = 0..n-1 (sorted order)            */
/*   s   = sum_{t<k} L_kt y_t            (ascending t; Alg. 2 l.10-13 + Alg. 3 l.10)            */
/*   a'  = (a_k - s)/L_kk, b' = (b_k - s)/L_kk                 (Eq. 2; Alg. 3 l.11)      */
/*   (log q, y_k) = orc_sov_step(a', b', w_{k,j})              (Alg. 3 l.12-13, reading R4/R9)  */
/*   ell_k(j) = ell_{k-1}(j) + log q      (running log of the product p_j, R10)                */
/* One sweep gives every prefix (reading R1): ell_k(j) is the log of sample j's product for the */
/* prefix o(1..k). Per prefix k the unit reports (M_k, S_k) with M_k = max_j ell_k(j) and       */
/* S_k = sum_j exp(ell_k(j) - M_k) (ascending j), i.e. a two-pass log-sum-exp (R10/R11).       */
/*                                                                                             */
/* L: row-major n x n (lower triangle used, ldl = row stride). The sample loop is innermost     */
/* for speed; each sample's own operation order is exactly the per-sample loop above.         */
/* out_MS: [n][2] = (M_k, S_k). ell_out (nullable): [n][J]. y_out (nullable): [n][J].          */
/* ------------------------------------------------------------------------------------------ */
int orc_sov_unit(long long n, const double *L, long long ldl, const double *a, const double *b,
                 const uint64_t *G, const uint64_t *D, long long j0, long long J, double *out_MS,
                 double *ell_out, double *y_out)
{
    double *Y = (double *)malloc(sizeof(double) * (size_t)n * (size_t)J);
    double *s = (double *)malloc(sizeof(double) * (size_t)J);
    double *ell = (double *)malloc(sizeof(double) * (size_t)J);
    double *ellk = (double *)malloc(sizeof(double) * (size_t)J);
    if (!Y || !s || !ell || !ellk) { free(Y); free(s); free(ell); free(ellk); return 1; }
    for (long long j = 0; j < J; ++j) ell[j] = 0.0;
    for (long long k = 0; k < n; ++k) {
        const double *Lk = L + k * ldl;
        for (long long j = 0; j < J; ++j) s[j] = 0.0;
        for (long long t = 0; t < k; ++t) {
            const double lkt = Lk[t];
            const double *Yt = Y + t * J;
            for (long long j = 0; j < J; ++j) s[j] += lkt * Yt[j];
        }
        const double lkk = Lk[k];
        double *Yk = Y + k * J;
        for (long long j = 0; j < J; ++j) {
            double w = orc_lattice_w((uint64_t)(j0 + j), G[k], D[k]);
            double ap = (a[k] - s[j]) / lkk;
            double bp = (b[k] - s[j]) / lkk;
            double lq, y;
            orc_sov_step(ap, bp, w, &lq, &y);
            Yk[j] = y;
            ell[j] += lq;
            ellk[j] = ell[j];
        }
        double M = -INFINITY;
        for (long long j = 0; j < J; ++j) if (ellk[j] > M) M = ellk[j];
        double S = 0.0;
        if (M != -INFINITY)
            for (long long j = 0; j < J; ++j) S += exp(ellk[j] - M);
        out_MS[2 * k] = M;
        out_MS[2 * k + 1] = S;
        if (ell_out) memcpy(ell_out + k * J, ellk, sizeof(double) * (size_t)J);
    }
    if (y_out) memcpy(y_out, Y, sizeof(double) * (size_t)n * (size_t)J);
    free(Y); free(s); free(ell); free(ellk);
    return 0;
}

/* Units u = unit_begin .. unit_end-1, ordered (r, c): shift r = u / C, chunk c = u % C with
 * C = ceil(N / chunk); the unit covers lattice indices j = c*chunk+1 .. min((c+1)*chunk, N).
 * D: [R][n] shifts. out: [unit_end-unit_begin][n][2]. Units are independent (threads split them). */
int orc_sov_units(long long n, const double *L, long long ldl, const double *a, const double *b,
                  const uint64_t *G, const uint64_t *D, long long N, long long R, long long chunk,
                  long long unit_begin, long long unit_end, double *out, int nthreads)
{
    (void)R;
    long long C = (N + chunk - 1) / chunk;
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 1) reduction(| : err)
    for (long long u = unit_begin; u < unit_end; ++u) {
        long long r = u / C, c = u % C;
        long long j0 = c * chunk + 1;
        long long J = (c + 1) * chunk <= N ? chunk : N - c * chunk;
        err |= orc_sov_unit(n, L, ldl, a, b, G, D + r * n, j0, J,
                            out + (u - unit_begin) * n * 2, NULL, NULL);
    }
    return err;
}

/* ------------------------------------------------------------------------------------------ */
/* NEXT-2: Monte-Carlo validation of the confidence regions ("draws N samples from the    */
/* fitted distribution, where N_s represents the number of samples exceeding a given threshold */
/* ... p_hat(alpha) = N_s/N"; supplement P:20-23).                                              */
/* Sample s (global index) draws z_k = Phi^{-1}(w_{k,s}) for k = 0..n-1 with                   */
/*   X = SplitMix64-mix(seed + GAMMA (s 2^32 + k + 1)),  w = (floor(X / 2^12) + 1/2) 2^-52      */
/* (reading R20), forms x_k = sum_{t<=k} L_kt z_t (ascending t; x = L z, so mu + x is a draw of */
/* the field in sorted order) and records its first failing row                                */
/*   first[s - s0] = min{k : x_k <= a_k}  (n if x_k > a_k for every k),                         */
/* i.e. the sample exceeds u on the region o(1..k*) iff first >= k*. If margin is non-NULL it  */
/* receives x_f - a_f at the reported row (0 when first = n) for tie diagnostics.              */
/* ------------------------------------------------------------------------------------------ */
uint64_t orc_mc_mix(uint64_t seed, uint64_t s, uint64_t k)
{
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * ((s << 32) + k + 1ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

double orc_mc_z(uint64_t seed, uint64_t s, uint64_t k)
{
    uint64_t X = orc_mc_mix(seed, s, k);
    double w = ((double)(X >> 12) + 0.5) * 0x1p-52;
    return w <= 0.5 ? orc_Phiinv_lower(w) : -orc_Phiinv_lower(1.0 - w);
}

int orc_mc_first(long long n, const double *L, long long ldl, const double *a, uint64_t seed, long long s0,
                 long long ns, int *first, double *margin, double *min_gap, int nthreads)
{
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 16) reduction(| : err)
    for (long long s = 0; s < ns; ++s) {
        double *z = (double *)malloc(sizeof(double) * (size_t)n);
        if (!z) { err |= 1; continue; }
        int f = (int)n;
        double gap = INFINITY;            /* smallest |x_k - a_k| over rows k <= f */
        double mg = 0.0;
        for (long long k = 0; k < n; ++k) {
            z[k] = orc_mc_z(seed, (uint64_t)(s0 + s), (uint64_t)k);
            const double *Lk = L + k * ldl;
            double x = 0.0;
            for (long long t = 0; t <= k; ++t) x += Lk[t] * z[t];
            double d = fabs(x - a[k]) / (1.0 + fabs(a[k]));
            if (d < gap) gap = d;
            if (!(x > a[k])) { f = (int)k; mg = x - a[k]; break; }
        }
        first[s] = f;
        if (margin) margin[s] = mg;
        if (min_gap) min_gap[s] = gap;
        free(z);
    }
    return err;
}
