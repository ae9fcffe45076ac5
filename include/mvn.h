/*
 * mvn.h — C ABI of libmvn.so, the B200-native (sm_100a) hot path of arXiv 2405.14892:
 * confidence-region detection from high-dimensional multivariate normal (MVN) probabilities.
 *
 *   geometry, theta = (sigma^2, beta, nu), u, 1-alpha            (problem statement)
 *     -> mvn_marginal_order   p_M, descending order, limits      (Alg. 1 l.3-6)
 *     -> mvn_cov_matern       Sigma tiles in sorted order         (Eq. 6; Alg. 1 l.2)
 *     -> mvn_potrf            Sigma = L L^T in place              (Alg. 1 l.8)
 *     -> mvn_sov_prefix       one SOV/QMC sweep -> per-prefix     (Alg. 2-3; Eq. 2-3)
 *                             log-sum-exp partials (M_k, S_k)
 *     -> mvn_prefix_finalize  log P_k                             (Alg. 2 l.19 mean(p))
 *     -> mvn_confidence_region k*(1-alpha)                        (Eq. 4-5)
 *
 * Citations: P:n = PAPER.md line n; R-numbers = readings in DESIGN.md §2.
 *
 * Conventions (all functions):
 *  - Ownership: the caller owns every buffer passed in. "d_" pointers are device pointers (e.g. a
 *    torch tensor's data_ptr()), everything else is host memory. The context owns only its
 *    internal workspace (Y-history scratch, block partials, lattice generators, device scalars).
 *  - Streams: every device operation is enqueued on the context's stream (mvn_create /
 *    mvn_set_stream). Functions returning host values (info, k_out, mvn_crd) synchronise it.
 *  - Errors are returned, never thrown or printed; mvn_last_error() has the message. No CPU
 *    fallback exists: without a usable sm_100a device, mvn_create fails with MVN_E_CUDA.
 *  - Threading: a context is single-threaded; use one context per host thread / device.
 *  - Precision: fp64 throughout.
 */
#ifndef MVN_H
#define MVN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MVN_OK = 0,
    MVN_E_USAGE = 1,    /* invalid argument (sizes, NaN limits, a_k > b_k, conf not in (0,1), ...) */
    MVN_E_NUMERIC = 2,  /* Sigma not positive definite: see info (first failing 0-based row)       */
    MVN_E_IO = 3,       /* reserved (file I/O lives above the ABI)                                  */
    MVN_E_CUDA = 4,     /* CUDA runtime error or no usable device                                   */
    MVN_E_NCCL = 5,     /* reserved: collectives live in the Python layer (torch.distributed)       */
    MVN_E_NOMEM = 6     /* device or host allocation failed                                         */
} mvn_status;

typedef struct mvn_ctx mvn_ctx;

/* Create a context bound to CUDA device `device` and stream `cuda_stream` (a cudaStream_t; NULL =
 * the legacy default stream). Fails with MVN_E_CUDA unless the device is compute capability 10.0
 * (B200, sm_100a — the only architecture this library is built for). */
mvn_status mvn_create(int device, void *cuda_stream, mvn_ctx **out);
/* Free the context and its workspace. Waits for all outstanding work on the context's device (the
 * bound stream itself is not touched: its owner may have destroyed it already). */
void mvn_destroy(mvn_ctx *ctx);
/* Rebind the context to another stream of its device. The new stream first waits (device-side
 * event, no host sync) for everything the context enqueued before, so a context's workspace is
 * never used by two streams at once; calls on the new stream are then ordered after the old ones. */
mvn_status mvn_set_stream(mvn_ctx *ctx, void *cuda_stream);
const char *mvn_last_error(const mvn_ctx *ctx);
const char *mvn_version(void);
/* Release the context's cached workspace (Y history, partials). */
mvn_status mvn_trim(mvn_ctx *ctx);

/* ---------------------------------------------------------------------------------------------
 * Lower tile-packed symmetric storage (Chameleon-style tile descriptor, restated).
 * nt = ceil(n/nb) tiles per side; tile (i,j), i >= j, starts at ((i*(i+1))/2 + j) * nb*nb doubles
 * and is an nb x nb column-major block. The row panel of tile-row i is contiguous. Edge tiles are
 * padded: padded diagonal entries are 1, padded off-diagonal entries 0, so the padded matrix is
 * SPD with L's padding equal to the identity. nb must be 128 in this build (MVN_E_USAGE
 * otherwise).                                                                                   */
typedef struct {
    int64_t n;   /* matrix order, >= 1 */
    int64_t nb;  /* tile size (128) */
} mvn_tiles;

int64_t mvn_tiles_count(mvn_tiles t);   /* nt*(nt+1)/2, or -1 if invalid */
size_t mvn_tiles_bytes(mvn_tiles t);    /* 8 * nb*nb * count, 0 if invalid */

/* dense column-major (leading dimension ld >= n, device) <-> tile-packed (device). pack reads the
 * lower triangle only and writes the padding; unpack writes the lower triangle and zeroes the
 * strict upper triangle of the dense matrix. */
mvn_status mvn_pack_lower(mvn_ctx *ctx, mvn_tiles t, const double *d_dense, int64_t ld, double *d_tiles);
mvn_status mvn_unpack_lower(mvn_ctx *ctx, mvn_tiles t, const double *d_tiles, double *d_dense, int64_t ld);

/* ---------------------------------------------------------------------------------------------
 * a1. Marginal probabilities and order (Alg. 1 l.3-6; readings R2, R13). HOST.
 *   z_i = (mu_i - u)/sqrt(var_i), p_M[i] = Phi(z_i) = P(X_i > u);
 *   order = indices sorted by z descending, ties by ascending index (stable);
 *   a_sorted[k] = u - mu[order[k]]  (lower limit of the k-th sorted location; b = +inf, R2).
 * mu, var_diag: n doubles (var_diag = Sigma_ii = sigma^2 + nugget). order: n int64 (out),
 * a_sorted: n doubles (out), pM: n doubles (out, nullable, original order).
 * MVN_E_USAGE if n < 1, any input is NaN, or any var <= 0.                                      */
mvn_status mvn_marginal_order(int64_t n, const double *mu, const double *var_diag, double u,
                              int64_t *order, double *a_sorted, double *pM);

/* ---------------------------------------------------------------------------------------------
 * a2. Matérn covariance tiles (Eq. 6, as printed: no sqrt(2 nu) scaling, R14):
 *   Sigma_kl = sigma2 * M_nu(h/beta) + nugget * delta_kl,  h = ||x_k - x_l||_2  (Euclidean)
 *   nu = 0.5: e^{-x};  nu = 1.5: (1+x) e^{-x};  nu = 2.5: (1 + x + x^2/3) e^{-x} (closed forms, the
 *   fast kernels); any other 0 < nu <= 50: M_nu(x) = 2^{1-nu}/Gamma(nu) x^nu K_nu(x) with K_nu by
 *   Temme's series (x <= 2) / Steed's continued fraction (x > 2) and the forward recurrence (e.g.
 *   the wind fit's nu = 1.43391); M_nu(0) = 1.
 * d_xy: n x 2 row-major device doubles, ALREADY in sorted order (x_{o(k)}). d_tiles: device,
 * mvn_tiles_bytes(t) bytes, fully written (including padding). Exactly symmetric.
 * MVN_E_USAGE for sigma2 <= 0, beta <= 0, nugget < 0, or nu outside (0, 50].                    */
mvn_status mvn_cov_matern(mvn_ctx *ctx, mvn_tiles t, const double *d_xy, double sigma2, double beta,
                          double nu, double nugget, double *d_tiles);

/* ---------------------------------------------------------------------------------------------
 * a3. Tiled right-looking Cholesky in place (Alg. 1 l.8 "L <- dpotrf(Sigma)"; box (a) of
 * P:319): for k: POTRF(A_kk) -> TRSM(A_ik, i>k) -> SYRK/GEMM(A_ij, i>=j>k) on fp64 DMMA.
 * d_tiles: in Sigma (lower tiles), out L (lower tiles; strict upper part of diagonal tiles
 * zeroed). *info (host, out): -1 on success, else the 0-based global row of the first
 * non-positive pivot, with MVN_E_NUMERIC returned (reading R17; no jitter retry). Synchronises. */
mvn_status mvn_potrf(mvn_ctx *ctx, mvn_tiles t, double *d_tiles, int64_t *info);

/* NEXT-4 for a3: the same factorisation with the trailing updates
 * A_ij -= sum_c L_ic L_jc^T (K = 128 kp per super-step) on the int8 tensor cores (tcgen05), an
 * Ozaki-style split (reading R25): per super-step the panel rows get a power-of-two scale
 * over the panel's columns and 8 signed 7-bit digits; the 36 products with p + q <= 9 are exact
 * int8 GEMMs, combined in fp64. The panel factorisation and the look-ahead update stay on fp64
 * DMMA. MVN_POTRF_FP64 = mvn_potrf. Not bitwise equal to the fp64 factor (the dropped digit products
 * are ~the rounding of an fp64 GEMM: residual ||L L^T - Sigma||_F / ||Sigma||_F stays ~1e-16);
 * info / errors / synchronisation as mvn_potrf. Workspace: the panel's slices (~ one panel of L).   */
#define MVN_POTRF_FP64 0
#define MVN_POTRF_INT8 1
mvn_status mvn_potrf_ex(mvn_ctx *ctx, mvn_tiles t, double *d_tiles, int64_t *info, int32_t method);

/* ---------------------------------------------------------------------------------------------
 * NEXT-1: building blocks of the distributed tiled Cholesky, 1-D
 * block-cyclic over super-panels of kp tile columns (super-panel s = tile columns s*kp ..
 * s*kp+kp-1 is owned by rank s mod W; kp = mvn_potrf_panel_width(n)). The step loop and the
 * NCCL panel broadcasts are in the Python layer (paper_2405_14892_b200/parallel.py,
 * potrf_distributed); the right-looking recurrence is the one of mvn_potrf, which is built from
 * the same two calls (Alg. 1 l.8; the paper runs it distributed on Chameleon/StarPU, P:81,
 * P:609-645), so both produce bit-identical factors. Per super-step s (k = s*kp):
 *   owner(s):  mvn_potrf_panel(k, kp)  -> mvn_panel_pack(k, kp)  -> broadcast
 *   others:    receive                 -> mvn_panel_unpack(k, kp)
 *   all:       mvn_potrf_update(k, kp, own columns >= k+kp)
 * A panel of (k, kp) is the tiles (k+j .. nt-1, k+j), j < kp, stored contiguously (layout at
 * mvn_panel_pack): sum_j (nt-k-j) * nb*nb doubles, device. All calls are asynchronous on the context's
 * stream; pivots are checked on the device and collected by mvn_potrf_info.                    */

/* Tile columns per super-panel (1..8) that mvn_potrf uses for order n (and potrf_distributed must
 * use to produce the same factor); -1 if n < 1. The environment variable MVN_POTRF_KP overrides. */
int64_t mvn_potrf_panel_width(int64_t n);

/* Factor the kp (1..8; clipped at nt) tile columns k .. k+kp-1 in place: POTRF of the diagonal tile
 * and TRSM of the tiles below, column by column, each further column first updated with the
 * previous columns of the super-panel. All updates from columns < k must have been applied. A
 * non-positive pivot records its 0-based global row in the context's device info (first failure
 * only) and leaves its tile.                                                                     */
mvn_status mvn_potrf_panel(mvn_ctx *ctx, mvn_tiles t, double *d_tiles, int64_t k, int64_t kp);

/* Trailing update with the super-panel (k, kp): A_ij -= sum_{c=k}^{k+kp-1} L_ic L_jc^T for every
 * i >= j and every tile column j = col_first + m*col_stride + b (m >= 0, 0 <= b < col_block, j < nt)
 * — blocks of col_block columns every col_stride columns (1, 1: all columns from col_first).
 * Requires k + kp <= col_first, 1 <= col_block <= col_stride. sm_reserve SMs are left free for
 * concurrent panel work (0..nsm-1).                                                              */
mvn_status mvn_potrf_update(mvn_ctx *ctx, mvn_tiles t, double *d_tiles, int64_t k, int64_t kp, int64_t col_first,
                            int64_t col_stride, int64_t col_block, int32_t sm_reserve);

/* Super-panel (k, kp) <-> contiguous panel buffer (device, caller-owned, size above); the buffer
 * holds the super-panel's tiles row after row: tile (i, k+j) at ((m <= kp ? m(m+1)/2 : kp(kp+1)/2 +
 * (m-kp) kp) + j) nb^2 doubles, m = i - k (kp clipped at nt - k), so a row (i, k .. k+kp-1) is
 * contiguous — the operand layout of the trailing update. */
mvn_status mvn_panel_pack(mvn_ctx *ctx, mvn_tiles t, const double *d_tiles, int64_t k, int64_t kp, double *d_panel);
mvn_status mvn_panel_unpack(mvn_ctx *ctx, mvn_tiles t, const double *d_panel, int64_t k, int64_t kp, double *d_tiles);

/* Reads (synchronising the stream) the device info of mvn_potrf_panel: -1 if every pivot so far
 * was positive, else the first failing 0-based row. reset != 0 sets it back to -1 afterwards.  */
mvn_status mvn_potrf_info(mvn_ctx *ctx, int64_t *info, int32_t reset);

/* ---------------------------------------------------------------------------------------------
 * NEXT-1 distributed STORAGE (P:81, P:609-645 — the paper's dense runs keep
 * the tiles distributed over the nodes): a rank holds only the tile columns it owns under the 1-D
 * block-cyclic map (super-panel s = tile columns s*kp .. s*kp+kp-1 owned by rank s mod world), so
 * its memory is ~1/world of the 8 n^2/2 bytes. Local layout: the owned tiles, row after row —
 * tile (i, j), i >= j, j owned, at (owned tiles in rows < i + owned columns < j) * nb*nb doubles.
 * The same recurrence as mvn_potrf (bit-identical factor): per super-step s, owner(s) factors
 * super-panel s in its storage (mvn_dpotrf_panel) and packs it (mvn_dpanel_pack, layout at
 * mvn_panel_pack); the buffer is broadcast (torch.distributed / NCCL, above the ABI); every rank
 * updates its own columns from the BUFFER (mvn_dpotrf_update: no unpack, no full copy).
 * Synchronisation, streams and errors as the calls above; pivots go to the context's device info
 * (mvn_potrf_info). kp = 1..8 (normally mvn_potrf_panel_width(n)).                               */
typedef struct {
    int64_t n, nb;          /* order, tile size (128) */
    int32_t world, rank;    /* ranks, this rank (0 <= rank < world) */
    int32_t kp;             /* tile columns (and rows) per block */
    int32_t prows;          /* 0 or 1: 1-D (column blocks over all ranks); P > 1: 2-D block-cyclic over a
                               P x (world / P) grid, rank = pr * (world / P) + pc: block (I, J) of kp x kp
                               tiles is owned by (I mod P, J mod (world / P)) */
} mvn_dtiles;

/* Bytes of the rank's local storage (0 for invalid d). */
size_t mvn_dtiles_bytes(mvn_dtiles d);
/* Doubles in the broadcast buffer of super-panel s (-1 for invalid arguments). */
int64_t mvn_dpanel_numel(mvn_dtiles d, int64_t s);
/* a2 on the owned tiles only (arguments as mvn_cov_matern; d_xy holds all n sorted locations). */
mvn_status mvn_dcov_matern(mvn_ctx *ctx, mvn_dtiles d, const double *d_xy, double sigma2, double beta, double nu,
                           double nugget, double *d_local);
/* Factor super-panel s in place, on the rank holding its diagonal block (MVN_E_USAGE otherwise):
 * 1-D: the whole super-panel (as mvn_potrf_panel); 2-D: the diagonal block only (kp x kp tiles). */
mvn_status mvn_dpotrf_panel(mvn_ctx *ctx, mvn_dtiles d, double *d_local, int64_t s);
/* 2-D, every rank of super-panel s's process column: after the factored diagonal block arrived in
 * d_panel (its leading kp(kp+1)/2 tiles), solve this rank's rows of the super-panel below it:
 * per column c: update by the columns before c, then L_ic = A_ic L_cc^{-T} (no-op for 1-D). */
mvn_status mvn_dpanel_trsm(mvn_ctx *ctx, mvn_dtiles d, double *d_local, int64_t s, const double *d_panel);
/* This rank's tiles of super-panel s -> their places in the buffer d_panel (mvn_dpanel_numel(d, s)
 * doubles; other places untouched): 1-D the owner packs everything; 2-D each rank of the process
 * column packs its rows (the diagonal block's rank first, for mvn_dpanel_trsm), and the pieces are
 * combined over the ranks (all-gather / broadcasts, above the ABI). */
mvn_status mvn_dpanel_pack(mvn_ctx *ctx, mvn_dtiles d, const double *d_local, int64_t s, double *d_panel);
/* A_ij -= sum_{c in super-panel s} L_ic L_jc^T, operands read from super-panel s's buffer, for every
 * owned tile column j of the super-panels >= sp_first (just_one != 0: super-panel sp_first only,
 * which must then be owned) and every owned i >= j (2-D: this rank's row blocks). Requires
 * sp_first > s. sm_reserve as mvn_potrf_update. */
mvn_status mvn_dpotrf_update(mvn_ctx *ctx, mvn_dtiles d, double *d_local, int64_t s, const double *d_panel,
                             int64_t sp_first, int32_t just_one, int32_t sm_reserve);
/* Copy the owned tiles into their places in a full tile-packed buffer (other tiles untouched). */
mvn_status mvn_dgather(mvn_ctx *ctx, mvn_dtiles d, const double *d_local, double *d_tiles);

/* ---------------------------------------------------------------------------------------------
 * a5. QMC point set (reading R8). The global sample index g in [0, N*R) maps to shift r = g / N
 * and lattice index j = g % N + 1 (1-based). Row k (0-based, sorted order) of sample g uses
 *   X = (j * G_k + D_k^r) mod 2^64,  w = (floor(X / 2^12) + 1/2) * 2^-52,
 *   G_k = floor(frac(sqrt(p_{k+1})) * 2^64)  (p_1 = 2: k-th prime),
 *   D_k^r = SplitMix64_mix(seed + 0x9E3779B97F4A7C15 * (r * 2^32 + k + 1))  (mod 2^64).
 * mvn_lattice_generators: HOST, writes gen[0..n). mvn_lattice_shifts: HOST, D[r*n + k].       */
mvn_status mvn_lattice_generators(int64_t n, uint64_t *gen);
mvn_status mvn_lattice_shifts(uint64_t seed, int32_t R, int64_t n, uint64_t *D);

typedef struct {
    int64_t N;             /* lattice points per shift, >= 1 */
    int32_t R;             /* random shifts, >= 1 */
    uint64_t seed;         /* shift seed */
    int64_t sample_begin;  /* global sample range [begin, end) processed by this call */
    int64_t sample_end;    /*   0 <= begin < end <= N*R  (a rank's shard, or everything) */
    const uint64_t *d_gen; /* nullable (device, n): the lattice generators G_k to use instead of R8's
                              sqrt-prime ones (e.g. a component-by-component rule);
                              w = (floor((j G_k + D_k^r mod 2^64) / 2^12) + 1/2) 2^-52 as in R8.
                              NULL (aggregate initialisers that omit it): the library's table. */
} mvn_qmc;

/* ---------------------------------------------------------------------------------------------
 * a5-a8. One SOV sweep over all n rows for every sample in the range (Alg. 2, with
 * the QMC tile kernel Alg. 3; Eq. 2-3; prefixes collapsed into one sweep,
 * reading R1). Per sample, for k = 0..n-1:
 *   s = sum_{t<k} L_kt y_t;  a' = (a_k - s)/L_kk;  b' = (b_k - s)/L_kk;
 *   (log q, y_k) = tail-aware Phi / Phi^{-1} step of reading R9;  ell_k = ell_{k-1} + log q.
 * Output: for every prefix k, over the samples of the range,
 *   d_M[k] = max_g ell_k(g),  d_S[k] = sum_g exp(ell_k(g) - d_M[k])
 * (M = -inf, S = 0 if every sample has probability 0). Deterministic for a given range, n and
 * device (fixed sample blocking, fixed combine order).
 * d_L: tile-packed L from mvn_potrf. d_a: n device doubles (-inf allowed). d_b: n device doubles
 * or NULL for b = +inf (every BASELINE config). MVN_E_USAGE if the range is empty/out of bounds,
 * n, N, R < 1, or any limit is NaN or a_k > b_k (checked on the device; the call synchronises the
 * stream once for that check before enqueuing the sweep).                                      */
mvn_status mvn_sov_prefix(mvn_ctx *ctx, mvn_tiles t, const double *d_L, const double *d_a,
                          const double *d_b, const mvn_qmc *q, double *d_M, double *d_S);

/* NEXT-4 ("mixed precision ... tensor core execution"): the same sweep
 * with a selectable arithmetic for the GEMM update a6 (s of every row from the rows of earlier row
 * blocks). MVN_SOV_FP64 = mvn_sov_prefix (fp64 DMMA, the default path). MVN_SOV_INT8 = the update
 * on the int8 tensor cores (tcgen05, TMEM) as an Ozaki-style split, reading R24:
 * L_kt = 2^{e_k} sum_p a_p 2^{-7p} and y = 2^7 sum_q b_q 2^{-7q} with 8 signed 7-bit digits each,
 * the 36 products of p + q <= 9 exact in int32, combined in fp64; everything else (in-block part
 * of s, the Phi / Phi^{-1} chain, log-sum-exp) is the fp64 path's. Same inputs, lattice and
 * outputs; results agree with the fp64 path to ~1e-12 in log P (not bitwise). Requirements:
 * d_b == NULL (b = +inf, every BASELINE config) and every sample value |y_k| < 63.5 (|a'| below
 * ~60); a violation of the latter is detected on the device and returned as MVN_E_NUMERIC. The
 * int8 call synchronises the stream at its end (that check). Workspace: the 8 slices of L (as
 * many bytes as L) plus a Y-digit history of ~n KB per pair of SMs.                              */
#define MVN_SOV_FP64 0
#define MVN_SOV_INT8 1
mvn_status mvn_sov_prefix_ex(mvn_ctx *ctx, mvn_tiles t, const double *d_L, const double *d_a,
                             const double *d_b, const mvn_qmc *q, int32_t method, double *d_M, double *d_S);

/* The same sweep as per-UNIT partials (SURVEY §8(b), §8(e)'s bitwise-deterministic combine): unit u
 * = the global samples [128 u, min(128 u + 128, N*R)) (q->sample_begin / end are ignored). For the
 * units [unit_begin, unit_end) it writes d_partial[u - unit_begin][k][2] = (max_g ell_k(g), sum_g
 * exp(ell_k(g) - max)) over the unit's samples (device, caller-owned, n doubles x 2 per unit). A
 * unit's partial does not depend on how the units are split over calls or ranks (its samples always
 * sit on the same lanes of one 128-sample block), so concatenating the ranks' partials (all-gather)
 * and reducing them in unit order with mvn_prefix_reduce gives the same bits on any number of GPUs.
 * Errors as mvn_sov_prefix.                                                                      */
mvn_status mvn_sov_prefix_units(mvn_ctx *ctx, mvn_tiles t, const double *d_L, const double *d_a,
                                const double *d_b, const mvn_qmc *q, int64_t unit_begin, int64_t unit_end,
                                double *d_partial);
/* (M, S) of `units` consecutive unit partials (layout above), combined in unit order (device). */
mvn_status mvn_prefix_reduce(mvn_ctx *ctx, int64_t n, int64_t units, const double *d_partial, double *d_M, double *d_S);

/* ---------------------------------------------------------------------------------------------
 * NEXT-1: the sweep over ROW PHASES, for an L that is not resident in one buffer (P:81, P:609-645:
 * the paper's dense runs keep the tiles distributed). The sweep of mvn_sov_prefix (same samples,
 * same arithmetic, same bits of (M, S)) is cut into consecutive ranges of tile rows; each call
 * brings only the tiles of its rows — the rank's own tiles plus the others' broadcast over NVLink
 * (parallel.sov_distributed), or slices of a full buffer. Between calls the sweep keeps, per sample,
 * its log weight and its Y history (one slot of n_pad x (w + 4) doubles per 128-sample block).
 *
 * mvn_sweep_begin: checks the limits (as mvn_sov_prefix; b may be NULL = +inf), copies a, b and the
 *   lattice generators, allocates the state (stream-ordered, on the context's stream). *out owns it
 *   until mvn_sweep_end / mvn_sweep_free.
 * mvn_sweep_rows: tile rows [tile_row_begin, tile_row_end) of L; tile_row_begin must be where the
 *   previous call stopped (0 first), tile_row_end <= ceil(n / 128). d_rows (device, caller-owned,
 *   read by kernels on the stream: keep it unchanged until they are done) holds the tiles (i, j),
 *   begin <= i < end, j <= i, row after row: tile (i, j) at (i(i+1)/2 + j - begin(begin+1)/2) * nb^2
 *   doubles — the same order as the full tile-packed buffer, so a slice of it can be passed.
 * mvn_sweep_end: after the last row, the block partials -> (M, S) as mvn_sov_prefix; frees the state.
 * mvn_sweep_free: frees the state without results (any time). A sweep must end before its context
 *   is destroyed; the state comes from a context-owned memory pool that keeps the memory for the
 *   next sweep until mvn_trim. Errors: MVN_E_USAGE for calls out of order or bad arguments (the
 *   state stays valid), MVN_E_CUDA.                                  */
typedef struct mvn_sweep mvn_sweep;
mvn_status mvn_sweep_begin(mvn_ctx *ctx, int64_t n, const double *d_a, const double *d_b, const mvn_qmc *q,
                           mvn_sweep **out);
mvn_status mvn_sweep_rows(mvn_sweep *sw, const double *d_rows, int64_t tile_row_begin, int64_t tile_row_end);
mvn_status mvn_sweep_end(mvn_sweep *sw, double *d_M, double *d_S);
void mvn_sweep_free(mvn_sweep *sw);

/* Distributed storage -> row slice: the element offset, in a rank's local buffer (mvn_dtiles
 * layout), of its first tile in tile row i (i = ceil(n/128): the total), so the rank's tiles of rows
 * [b, e) are local[off(b) .. off(e)) — one contiguous piece to broadcast. mvn_drows_unpack places
 * rank d.rank's piece of rows [b, e) (d_piece = that range, device) into the row slice d_rows
 * (layout of mvn_sweep_rows); other tiles untouched. -1 / MVN_E_USAGE for invalid arguments.     */
int64_t mvn_drows_offset(mvn_dtiles d, int64_t tile_row);
mvn_status mvn_drows_unpack(mvn_ctx *ctx, mvn_dtiles d, const double *d_piece, int64_t tile_row_begin,
                            int64_t tile_row_end, double *d_rows);

/* Multi-GPU combine helpers (reading R11): after all_reduce(MAX) of M into d_Mglob,
 *   S <- S * exp(M - Mglob), M <- Mglob  (elementwise, device; S = 0 where M = -inf).
 * Then all_reduce(SUM) of S and mvn_prefix_finalize.                                           */
mvn_status mvn_prefix_rescale(mvn_ctx *ctx, int64_t n, const double *d_Mglob, double *d_M, double *d_S);

/* a8. log P_k = M_k + log S_k - log(NR) (the mean of Alg. 2 l.19 over all NR samples), device. */
mvn_status mvn_prefix_finalize(mvn_ctx *ctx, int64_t n, int64_t NR, const double *d_M,
                               const double *d_S, double *d_logP);

/* Per-shift estimates (reading R11: "mean(p)", over R randomly shifted
 * lattices): row r of d_logP_shift (device, [R][n]) receives log P^(r)_k, the estimate of shift r
 * alone (the sample range [r N, (r + 1) N) of mvn_sov_prefix, one sweep per shift). With
 * mvn_prefix_shift_stats (host) they give the combined log P_k = log mean_r P^(r)_k (= the
 * all-sample estimate, N equal per shift) and the relative standard error across the shifts,
 * rel_se_k = sd_r(P^(r)_k) / (sqrt(R) mean_r P^(r)_k) (sample sd, R - 1; ~ the standard error of
 * log P_k; 0 for R = 1; NaN where every P^(r)_k = 0), evaluated relative to max_r log P^(r)_k so
 * nothing underflows. The QMC error estimate of the regions; not part of the timed path.
 * Errors: USAGE as mvn_sov_prefix.                                                              */
mvn_status mvn_sov_prefix_shifts(mvn_ctx *ctx, mvn_tiles t, const double *d_L, const double *d_a, const double *d_b,
                                 const mvn_qmc *q, double *d_logP_shift);
mvn_status mvn_prefix_shift_stats(int64_t n, int32_t R, const double *logP_shift, double *logP, double *rel_se);

/* ---------------------------------------------------------------------------------------------
 * a10. Confidence regions (Eq. 4-5; readings R12, R16). HOST.
 * logP: n host doubles in sorted order. Running minimum first (ulp guard), then for each level
 * c = conf[i] in (0,1): k_out[i] = max{k : log P_k >= log c} (0 if none); the region is
 * order[0 .. k_out[i]). near_tie[i] (nullable) = 1 if |log P_{k*} - log c| <= 1e-8 or
 * |log P_{k*+1} - log c| <= 1e-8. The confidence function F(o(k)) = P_k (Eq. 5).             */
mvn_status mvn_confidence_region(int64_t n, const double *logP, const double *conf, int64_t nconf,
                                 int64_t *k_out, int32_t *near_tie);

/* ---------------------------------------------------------------------------------------------
 * NEXT-2: Monte-Carlo validation of the confidence regions ("draws
 * N samples from the fitted distribution, where N_s represents the number of samples exceeding a
 * given threshold ... p_hat(alpha) = N_s/N"; supplement P:20-23). Reading R20:
 * sample s (global index, 0-based) draws, for every sorted row k,
 *   z_k = Phi^{-1}(w),  w = (floor(X / 2^12) + 1/2) 2^-52,
 *   X = SplitMix64_mix(seed + 0x9E3779B97F4A7C15 * (s * 2^32 + k + 1))  (mod 2^64),
 * and the field in sorted order is mu + L z. It exceeds u on the region o(1..k*) iff
 * (L z)_k > a_k for all k < k*, so one pass records its first failing row
 *   f_s = min{k : (L z)_k <= a_k}   (n if none),
 * and p_hat(k*) = #{s : f_s >= k*} / N for every level at once.                                 */
typedef struct {
    uint64_t seed;         /* z-generator seed */
    int64_t sample_begin;  /* global sample range [begin, end) of this call (a rank's shard) */
    int64_t sample_end;
    int32_t method;        /* 0: X = L Z on the fp64 tensor path (DMMA); 1: the same product emulated
                              exactly-per-slice on the int8 tensor cores (tcgen05.mma kind::i8, TMEM
                              accumulators; Ozaki split into 8 signed 7-bit slices, absolute error
                              <= ~1e-12 relative to max|L_k.| max|z|, reading R22), M128 N64 per CTA;
                              2: the same arithmetic at the full-rate M128 N128 shape, the 36 products
                              split by level over a 2-CTA cluster (multicast operands, L2 exchange) */
} mvn_mc;

/* d_L: tile-packed L (mvn_potrf), d_a: n device doubles (the limits a_k of the sweep).
 * d_count: n+1 device uint64, ACCUMULATED (count[f] += samples with first failing row f), so
 * chunks and ranks add up (all_reduce SUM across ranks). d_first: nullable, device int32 per
 * sample of the range (f_s). Work: n(n+1) fp64 flops per sample on DMMA (X = L Z, never stored).
 * Internal workspace: the Z block (<= ~8 GB; samples are processed in chunks).
 * MVN_E_USAGE for an empty / negative range.                                                    */
mvn_status mvn_mc_validate(mvn_ctx *ctx, mvn_tiles t, const double *d_L, const double *d_a, const mvn_mc *m,
                           uint64_t *d_count, int32_t *d_first);

/* HOST. p_hat[i] = #{s : f_s >= k_star[i]} / N_total from the histogram count[0..n] (the
 * confidence level the MC draws give the region of size k_star[i]). MVN_E_USAGE if
 * N_total < 1 or a k_star is outside [0, n].                                                   */
mvn_status mvn_mc_levels(int64_t n, const uint64_t *count, int64_t N_total, const int64_t *k_star, int64_t nconf,
                         double *p_hat);

/* ---------------------------------------------------------------------------------------------
 * NEXT-4: posterior conditioning before Alg. 1 (§V-A):
 * m noisy observations y = A x + N(0, tau^2 I) of the field at sites obs give
 *   Sigma_post = (Sigma^{-1} + tau^{-2} A^T A)^{-1}          (Eq. 7)
 *   mu_post    = mu + tau^{-2} Sigma_post A^T (y - A mu)     (Eq. 8)
 * which "can be used as input to Algorithm 1 (line 2) ... to update the a vector".
 * Computed as the Schur complement left by a partial tiled Cholesky of the augmented matrix
 * [[Sigma_oo + tau^2 I, Sigma_{o,:}, r], [Sigma_{:,o}, Sigma, 0], [r^T, 0, 1]], r = y - mu_o
 * (reading R21): the trailing block is Sigma_post, the last row is -(mu_post - mu).
 * Use: mvn_posterior -> mvn_marginal_order(mu_post, var_post, u) -> mvn_posterior_tiles(order)
 * -> mvn_potrf -> mvn_sov_prefix -> ...                                                          */
typedef struct {
    int64_t n;             /* sites */
    const double *xy;      /* host, n x 2 row-major, original order */
    const double *mu;      /* host, n prior mean */
    int64_t m;             /* observations, >= 1 */
    const int64_t *obs;    /* host, m distinct site indices in [0, n) */
    const double *y;       /* host, m observed values */
    double sigma2, beta, nu, nugget;   /* Matérn of the field (Eq. 6, R14) */
    double tau;            /* observation noise standard deviation (> 0; the paper uses 0.5) */
} mvn_posterior_problem;

/* Conditions the field; writes mu_post and var_post = diag(Sigma_post) (host, n each, original
 * order) and keeps Sigma_post in the context's workspace ((m_pad + n + 1)^2 / 2 doubles, m_pad =
 * m rounded up to 128) for mvn_posterior_tiles. *info (host): -1, or the first failing row of the
 * observation block (MVN_E_NUMERIC). MVN_E_USAGE for bad sizes / indices / tau <= 0.            */
mvn_status mvn_posterior(mvn_ctx *ctx, const mvn_posterior_problem *p, double *mu_post, double *var_post, int64_t *info);

/* Writes Sigma_post permuted to `order` (host, n: sorted position -> site, e.g. from
 * mvn_marginal_order) into the tile-packed d_tiles (t.n = the n of the last mvn_posterior).      */
mvn_status mvn_posterior_tiles(mvn_ctx *ctx, mvn_tiles t, const int64_t *order, double *d_tiles);

/* ---------------------------------------------------------------------------------------------
 * NEXT-3 (part): Tile Low-Rank compression at a fixed accuracy (§II-C,
 * P:175-176; Alg. 1 l.7 "pmvn_init() also encompasses the compression of the covariance matrix into
 * the TLR format"). Reading R23: every off-diagonal tile (I, J), I > J, of the tile-packed
 * d_tiles is replaced IN PLACE by its rank-k truncated SVD U_k S_k V_k^T; diagonal tiles stay dense.
 * k follows the accuracy eps: mode MVN_TLR_ABS (0): k = #{sigma_i >= eps}; mode MVN_TLR_REL_FRO (1):
 * the smallest k with ||A - A_k||_F <= eps ||A||_F for that tile (0 <= eps <= 1). The paper does not
 * state its convention; both are offered. The dense POTRF / SOV then run on the compressed
 * covariance unchanged (the TLR arithmetic of the Cholesky is not built: this gives the paper's
 * accuracy study of TLR vs dense, not its speedup). d_ranks: device int32 array of nt(nt-1)/2
 * ranks, tile (I, J) at I(I-1)/2 + J. Asynchronous. USAGE on a bad mode or eps.               */
enum { MVN_TLR_ABS = 0, MVN_TLR_REL_FRO = 1 };
mvn_status mvn_tlr_compress(mvn_ctx *ctx, mvn_tiles t, double *d_tiles, double eps, int32_t mode, int32_t *d_ranks);

/* ---------------------------------------------------------------------------------------------
 * NEXT-3: the TLR Cholesky (Alg. 1 l.7-8: "compression of the covariance matrix into the TLR
 * format"; step (a) "can be performed using both dense and TLR computations. However, (b),
 * (c), and (d) are only performed in dense"). Reading R26 (oracle/tlr.py
 * tlr_cholesky):
 *   1. every off-diagonal tile of Sigma is compressed at eps (mvn_tlr_compress's rule, R23) into
 *      factors U_t V_t^T;
 *   2. tile column j = 0 .. nt-1: T_i = Stilde_ij - sum_{k<j} U_ik (V_ik^T V_jk) U_jk^T (i >= j, the
 *      updates applied in factored form: 4 128 r_ik r_jk + 2 128^2 r_jk flops instead of 2 128^3),
 *      L_jj = chol(T_j), L_ij = T_i L_jj^{-T}, and each L_ij is truncated at eps once (U_t V_t^T);
 *   3. the off-diagonal tiles of d_tiles receive Ltilde = U_t V_t^T reconstructed, so that
 *      mvn_sov_prefix (dense) reads the TLR factor unchanged.
 * d_tiles: in Sigma (tile-packed, sorted order), out the factor: L_jj dense on the diagonal,
 * Ltilde_ij off it. d_U, d_V (device, caller-owned, mvn_tlr_slots_bytes(t, kmax) bytes each): slot
 * t = I(I-1)/2 + J holds U_t, V_t as column-major 128 x kmax blocks at t 128 kmax doubles (first
 * r_t columns used); on return the factors of Ltilde. d_ranks (device int32, nt(nt-1)/2): the ranks
 * r_t of Ltilde; d_ranks_sigma (nullable): Sigma's ranks after step 1. kmax in [1, 128] is the slot
 * width (memory per slot pair = 2 128 kmax doubles; kmax = 64 fits both factors in the bytes of a
 * dense tile). *info (host): -1, or the first failing global row (MVN_E_NUMERIC). MVN_E_NOMEM if a
 * tile needed a rank above kmax (stored truncated to kmax; the factor is then not at accuracy eps;
 * reported before a failing pivot, which the truncation may have caused). MVN_E_USAGE as mvn_tlr_compress, or kmax outside [1, 128]. Synchronises (info).            */
size_t mvn_tlr_slots_bytes(mvn_tiles t, int32_t kmax);

/* The SOV sweep of mvn_sov_prefix with the update in factored form (SURVEY §8(f) rank 3 "factored
 * SOV update A -= U(V^T Y)"): for the rows of tile row T, s = sum_{J<T} U_TJ (V_TJ^T Y_J) from
 * mvn_tlr_potrf's factor slots (d_U, d_V, d_ranks, kmax as returned there) plus the dense diagonal
 * tile L_TT read from d_L (tile-packed; only the diagonal tiles are read). Same samples, lattice,
 * Phi chain and outputs (d_M, d_S) as mvn_sov_prefix on the reconstructed factor, equal to it up to
 * summation order. The paper itself keeps this step dense; the factored form costs
 * 4 128 r_TJ + 256 r_TJ flops per sample and tile instead of 2 128^2, so it pays only for ranks
 * below ~43. USAGE as mvn_sov_prefix, or kmax outside [1, 128], or missing slots for n > 128. */
mvn_status mvn_sov_prefix_tlr(mvn_ctx *ctx, mvn_tiles t, const double *d_L, const double *d_U, const double *d_V,
                              const int32_t *d_ranks, int32_t kmax, const double *d_a, const double *d_b,
                              const mvn_qmc *q, double *d_M, double *d_S);
mvn_status mvn_tlr_potrf(mvn_ctx *ctx, mvn_tiles t, double *d_tiles, double eps, int32_t mode, int32_t kmax,
                         double *d_U, double *d_V, int32_t *d_ranks, int32_t *d_ranks_sigma, int64_t *info);

/* ---------------------------------------------------------------------------------------------
 * End-to-end CRD (Alg. 1) on one GPU with HOST buffers: upload, a1..a10, download.
 * This is the call a user makes; bench.py's "e2e" number times it.                             */
typedef struct {
    int64_t n;
    const double *xy;      /* host, n x 2 row-major, original order */
    const double *mu;      /* host, n, original order */
    double sigma2, beta, nu, nugget, u;
    int64_t N;
    int32_t R;
    uint64_t seed;
    const double *conf;    /* host, nconf levels in (0,1) */
    int64_t nconf;
    int32_t method;        /* 0: fp64 throughout; bit 0 (MVN_CRD_SOV_INT8): the SOV GEMM on the int8 tensor
                              cores (mvn_sov_prefix_ex); bit 1 (MVN_CRD_POTRF_INT8): the Cholesky
                              updates too (mvn_potrf_ex) — NEXT-4 mixed precision; bit 2 (MVN_CRD_TLR):
                              step (a) as the TLR Cholesky at accuracy tlr_eps (mvn_tlr_potrf, mode
                              MVN_TLR_ABS, slots of 128 columns in the context; steps (b)-(d) dense on
                              L~) — NEXT-3; not with bit 1 */
    double tlr_eps;        /* MVN_CRD_TLR: the accuracy eps (>= 0); ignored otherwise */
} mvn_crd_problem;
#define MVN_CRD_SOV_INT8 1
#define MVN_CRD_POTRF_INT8 2
#define MVN_CRD_TLR 4

typedef struct {
    int64_t *order;        /* host out, n: original index of sorted position k */
    double *logP;          /* host out, n: log P_k (sorted order, before running min) */
    int64_t *k_star;       /* host out, nconf */
    int32_t *near_tie;     /* host out, nconf (nullable) */
    int64_t info;          /* -1 or first failing Cholesky row */
    double ms_stage[6];    /* device time per stage: upload, cov, potrf, sov, finalize, download */
} mvn_crd_result;

mvn_status mvn_crd(mvn_ctx *ctx, const mvn_crd_problem *p, mvn_crd_result *out);

#ifdef __cplusplus
}
#endif
#endif /* MVN_H */
