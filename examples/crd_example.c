/*
 * Plain-C use of the libmvn C ABI (include/mvn.h), no Python: confidence regions of a small
 * synthetic field end to end on one B200 through mvn_crd (host buffers in and out).
 *
 *   gcc -O2 -std=c11 -I include examples/crd_example.c -L paper_2405_14892_b200 -lmvn \
 *       -Wl,-rpath,'$ORIGIN/../paper_2405_14892_b200' -lm -o examples/crd_example
 *   ./examples/crd_example [grid_side] [N] [R] [dump_file]
 *
 * The field: a jittered g x g grid on [0,1]^2, Matérn (sigma^2 = 1, beta = 0.1, nu = 1/2) with a
 * nugget 1e-8, and a smooth mean mu(x, y) = sin(3x) cos(2y) (inputs only; the method's arithmetic
 * all runs in libmvn). Prints log P_k for the first prefixes and the regions for 1 - alpha in
 * {0.8, 0.9, 0.95, 0.99}. With a dump_file, the inputs and results are also written there (raw
 * little-endian: int64 n, double xy[2n], double mu[n], int64 order[n], double logP[n], int64 k*[4])
 * so a checker can recompute them independently (tests/test_c_example.py runs the oracle on them).
 * Exit status: 0 on success, the mvn_status otherwise.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mvn.h"

static double uniform01(uint64_t *s) {           /* xorshift64*: input jitter only */
    *s ^= *s >> 12; *s ^= *s << 25; *s ^= *s >> 27;
    return (double)((*s * 0x2545F4914F6CDD1Dull) >> 11) * 0x1p-53;
}

int main(int argc, char **argv) {
    const int g = argc > 1 ? atoi(argv[1]) : 20;
    const int64_t N = argc > 2 ? atoll(argv[2]) : 2000;
    const int32_t R = argc > 3 ? atoi(argv[3]) : 4;
    const int64_t n = (int64_t)g * g;
    double *xy = malloc(sizeof(double) * 2 * n), *mu = malloc(sizeof(double) * n), *logP = malloc(sizeof(double) * n);
    int64_t *order = malloc(sizeof(int64_t) * n);
    uint64_t s = 0x1234567ull;
    for (int i = 0; i < g; ++i)
        for (int j = 0; j < g; ++j) {
            const int64_t k = (int64_t)i * g + j;
            xy[2 * k] = (i + 0.5) / g + (uniform01(&s) - 0.5) * 0.8 / g;
            xy[2 * k + 1] = (j + 0.5) / g + (uniform01(&s) - 0.5) * 0.8 / g;
            mu[k] = sin(3.0 * xy[2 * k]) * cos(2.0 * xy[2 * k + 1]);
        }
    const double conf[4] = {0.80, 0.90, 0.95, 0.99};
    int64_t kstar[4];
    int32_t tie[4];
    mvn_ctx *ctx = NULL;
    mvn_status st = mvn_create(0, NULL, &ctx);
    if (st != MVN_OK) { fprintf(stderr, "mvn_create: status %d (needs a B200)\n", (int)st); return (int)st; }
    mvn_crd_problem p = {n, xy, mu, 1.0, 0.1, 0.5, 1e-8, 0.0, N, R, 3001, conf, 4, 0};
    mvn_crd_result r = {order, logP, kstar, tie, -1, {0}};
    st = mvn_crd(ctx, &p, &r);
    if (st != MVN_OK) { fprintf(stderr, "mvn_crd: %s\n", mvn_last_error(ctx)); mvn_destroy(ctx); return (int)st; }
    printf("%s\nn = %lld, N x R = %lld x %d\n", mvn_version(), (long long)n, (long long)N, R);
    for (int64_t k = 0; k < (n < 8 ? n : 8); ++k)
        printf("  P_%lld = %.6f  (site %lld)\n", (long long)(k + 1), exp(logP[k]), (long long)order[k]);
    for (int i = 0; i < 4; ++i) printf("  region for 1-alpha = %.2f: %lld sites\n", conf[i], (long long)kstar[i]);
    printf("  device ms: upload %.3f cov %.3f potrf %.3f sov %.3f finalize %.3f download %.3f\n", r.ms_stage[0],
           r.ms_stage[1], r.ms_stage[2], r.ms_stage[3], r.ms_stage[4], r.ms_stage[5]);
    if (argc > 4) {
        FILE *f = fopen(argv[4], "wb");
        if (!f) { perror(argv[4]); mvn_destroy(ctx); return 3; }
        fwrite(&n, sizeof n, 1, f);
        fwrite(xy, sizeof(double), (size_t)(2 * n), f);
        fwrite(mu, sizeof(double), (size_t)n, f);
        fwrite(order, sizeof(int64_t), (size_t)n, f);
        fwrite(logP, sizeof(double), (size_t)n, f);
        fwrite(kstar, sizeof(int64_t), 4, f);
        fclose(f);
    }
    mvn_destroy(ctx);
    free(xy); free(mu); free(logP); free(order);
    return 0;
}
