// Internal declarations shared by the libmvn translation units (not part of the ABI).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mvn {

constexpr int kTile = 128;  // storage tile (mvn_tiles.nb)

cudaError_t matern_init();
cudaError_t launch_cov_matern(int64_t n, const double *xy, double sigma2, double beta, double nu, double nugget,
                              double *tiles, cudaStream_t st);
cudaError_t launch_pack(int64_t n, const double *dense, int64_t ld, double *tiles, bool to_tiles, cudaStream_t st);
cudaError_t launch_rescale(int64_t n, const double *Mg, double *M, double *S, cudaStream_t st);
cudaError_t launch_check_limits(int64_t n, const double *a, const double *b, int *flag, cudaStream_t st);
cudaError_t launch_finalize(int64_t n, int64_t NR, const double *M, const double *S, double *logP, cudaStream_t st);

cudaError_t potrf_init();
cudaError_t launch_potrf(int64_t n, double *tiles, int64_t *d_info, cudaStream_t st, int ncols = 0);
// NEXT-4: the trailing updates of the factorisation on the int8 tensor cores (kernels_potrf_oz.cu)
struct PotrfOz {
    int8_t *LAp;             // potrf_oz_lap_bytes(n, kp): the panel's digit slices
    double *rs;              // n_pad doubles: the panel rows' scales
    double *xch;             // potrf_oz_xch_bytes(clusters)
    int clusters;            // 2-CTA clusters of the update kernel
    int clusters_reserved;   // the same while the panel stream runs beside it
};
cudaError_t launch_potrf_ex(int64_t n, double *tiles, int64_t *d_info, cudaStream_t st, int ncols, const PotrfOz *oz);
cudaError_t potrf_oz_init();
int potrf_oz_max_clusters(int nsm);
int potrf_panel_sms();
int64_t potrf_oz_lap_bytes(int64_t n, int kp);
int64_t potrf_oz_xch_bytes(int clusters);
cudaError_t launch_potrf_update_oz(int64_t n, double *tiles, int k, int w, int c0, int cs, int cb, int clusters,
                                   int8_t *LAp, double *rs, double *xch, cudaStream_t st);
// distributed-factorisation building blocks (NEXT-1)
int potrf_panel_width(int64_t n);   // kp: tile columns per super-panel for order n (MVN_POTRF_KP overrides)
cudaError_t launch_potrf_panel(int64_t n, double *tiles, int k, int kp, int64_t *d_info, cudaStream_t st);
cudaError_t launch_potrf_update(int64_t n, double *tiles, int k, int kp, int c0, int cs, int cb, int sm_reserve,
                                cudaStream_t st);
cudaError_t launch_panel_copy(int64_t n, double *tiles, int k, int kp, double *panel, bool to_panel, cudaStream_t st);
// the same on explicit storages (TileMap, common.cuh): a rank's owned columns (NEXT-1 distributed
// storage), the full buffer, or a super-panel broadcast buffer
struct TileMap;
struct RowSel;
cudaError_t launch_potrf_panel_map(int64_t n, const TileMap &tm, int k, int kp, int64_t *d_info, cudaStream_t st,
                                   int row_end);
cudaError_t launch_potrf_update_map(int64_t n, const TileMap &dst, const TileMap &src, int k, int kp, int c0, int cs,
                                    int cb, int sm_reserve, cudaStream_t st);
cudaError_t launch_potrf_update_map(int64_t n, const TileMap &dst, const TileMap &src, const TileMap &srcB, int k, int kp,
                                    int c0, int cs, int cb, int sm_reserve, const RowSel &rs, cudaStream_t st);
cudaError_t launch_panel_trsm_map(int64_t n, const TileMap &tm, const TileMap &pb, int k, int w, const RowSel &rs,
                                  cudaStream_t st);
cudaError_t launch_panel_copy_map(int64_t n, const TileMap &from, const TileMap &to, int k, int kp, cudaStream_t st);
cudaError_t launch_rows_copy_map(const TileMap &from, const TileMap &to, int tb, int te, cudaStream_t st);
cudaError_t launch_cov_matern_map(int64_t n, const double *xy, double sigma2, double beta, double nu, double nugget,
                                  const TileMap &tm, cudaStream_t st);

struct SovLaunch {
    const double *L;
    int64_t n;
    const double *a, *b;
    const uint64_t *G;
    int64_t N;
    uint64_t seed;
    int64_t g_begin, g_end;
    const int64_t *cta;  // device [grid][3]: first sample, count, first block (sov_partition)
    int64_t nblk;        // sample blocks
    int grid;            // persistent CTAs (<= SM count)
    double *Y;           // [grid][ceil(n/64)*64][sov_y_stride()]
    double *part;    // [nblk][ceil(n/64)*64][2]
    double *Mout, *Sout;
    int lag = 0;             // soft grid lockstep distance in row blocks (0 = off)
    int *step_done = nullptr;  // [max_blocks][nrb] counters (zeroed by launch_sov)
    const int *need = nullptr; // [max_blocks]: CTAs with more than b blocks
    int max_blocks = 0;
    int hints = 1;           // L2 cache-policy hints
    int serial_rb = 0;       // row blocks whose GEMM waits for the previous chain (no fp64 contention)
    int unit_mode = 0;       // 1: blocks = global 128-sample units, partials [units][n][2] left in `part`
    // row phases (mvn_sweep_rows): rb1 > 0 runs row blocks [rb0, rb1) only, carrying the log weights
    // in ell[g - g_begin] and the Y histories in per-block slots (yoff: sov_phase_yoff); the
    // partials stay in `part` (no reduce)
    int rb0 = 0, rb1 = 0;
    double *ell = nullptr;
    const int64_t *yoff = nullptr;
    // NEXT-3: the factored SOV update (k_sov_tlr) from mvn_tlr_potrf's factor slots
    const double *tU = nullptr, *tV = nullptr;
    const int *tranks = nullptr;
    int tkmax = 0;
};
int64_t sov_phase_yoff(const int64_t *cta, int grid, int64_t n_pad, int unit_mode, int64_t *yoff);
cudaError_t sov_init();
int sov_block_samples();
int sov_y_stride();
int64_t sov_partition(int64_t g_begin, int64_t g_end, int grid, int64_t *cta);
int64_t sov_partition_units(int64_t u0, int64_t u1, int64_t g_end, int grid, int64_t *cta);
cudaError_t launch_sov(const SovLaunch &L, cudaStream_t st);
cudaError_t launch_reduce_blocks(const double *part, int64_t nblk, int64_t n, int64_t n_pad, double *M, double *S,
                                 cudaStream_t st);
cudaError_t launch_reduce_units(const double *part, int64_t units, int64_t n, double *M, double *S, cudaStream_t st);

// NEXT-4: the SOV GEMM on the int8 tensor cores (kernels_sov_oz.cu)
struct SovOzLaunch {
    const int8_t *LA;        // L slices (launch_mc_oz_prepare)
    const double *rowscale;
    const double *L;
    int64_t n;
    const double *a;
    const uint64_t *G;
    int64_t N;
    uint64_t seed;
    const int64_t *cl;       // device [clusters][3] (sov_oz_partition)
    int clusters;
    int64_t nblk;            // sample blocks of 128 over all clusters
    int8_t *YS;              // sov_oz_ys_bytes
    double *xch;             // sov_oz_xch_bytes
    double *part;            // [2 nblk][n_pad][2]
    double *Mout, *Sout;
    int *flag;               // device int: |y| >= 63.5 seen
    int lag = 0;             // cluster lockstep distance in steps (0 = off)
    int *step_done = nullptr;
    const int *need = nullptr;
    int max_blocks = 0;
};
cudaError_t sov_oz_init();
int sov_oz_max_clusters(int nsm);
int64_t sov_oz_ys_bytes(int64_t n, int clusters);
int64_t sov_oz_xch_bytes(int clusters);
int64_t sov_oz_partition(int64_t g_begin, int64_t g_end, int clusters, int64_t *cl);
cudaError_t launch_sov_oz(const SovOzLaunch &L, cudaStream_t st);

// NEXT-4: posterior conditioning helpers (kernels_post.cu)
cudaError_t launch_add_diag(double *tiles, int64_t begin, int64_t end, double v, cudaStream_t st);
cudaError_t launch_set_row(double *tiles, int64_t row, int64_t col0, int64_t ncols, const double *v, cudaStream_t st);
cudaError_t launch_add_pairs(double *tiles, const int64_t *rows, int64_t col0, int64_t count, double v, cudaStream_t st);
cudaError_t launch_get_row(const double *tiles, int64_t row, int64_t col0, int64_t ncols, double *out, cudaStream_t st);
cudaError_t launch_get_diag(const double *tiles, int64_t begin, int64_t n, double *out, cudaStream_t st);
cudaError_t launch_permute_sym(const double *src, int64_t off, const int64_t *order, int64_t n, double *dst, cudaStream_t st);

// NEXT-3 (part): fixed-accuracy TLR compression of the off-diagonal tiles (kernels_tlr.cu)
cudaError_t tlr_init();
cudaError_t launch_tlr_compress(int64_t n, double *tiles, double eps, int mode, int *ranks, cudaStream_t st);
// NEXT-3: the TLR Cholesky (R26): factor slots, workspace, the column loop
size_t tlr_slot_doubles(int64_t n, int kmax);
size_t tlr_work_doubles(int64_t n, int64_t chunk_slots);
cudaError_t launch_tlr_potrf(int64_t n, double *tiles, double eps, int mode, int kmax, double *U, double *V,
                             int *ranks, int *ranks_sigma, double *work, int64_t chunk_slots, int *overflow,
                             int64_t *d_info, cudaStream_t st);

// NEXT-2: Monte-Carlo validation
cudaError_t mc_init();
int64_t mc_z_doubles(int64_t n, int64_t ns);
cudaError_t launch_mc_chunk(int64_t n, const double *tiles, const double *a, uint64_t seed, int64_t s0, int64_t ns,
                            double *Z, int *first, unsigned long long *count, int nsm, cudaStream_t st);
cudaError_t launch_mc_first_init(int *first, int64_t ns, int n, cudaStream_t st);
cudaError_t launch_mc_count(const int *first, int64_t ns, unsigned long long *count, cudaStream_t st);
// NEXT-2 on the int8 tensor cores (kernels_mc_oz.cu): Ozaki-split X = L Z with tcgen05.mma kind::i8
cudaError_t mc_oz_init();
int64_t mc_oz_la_bytes(int64_t n);
int64_t mc_oz_zb_bytes(int64_t n, int64_t ns);
cudaError_t launch_mc_oz_prepare(int64_t n, const double *tiles, double *rowscale, int8_t *LA, cudaStream_t st);
int64_t mc_oz2_zb_bytes(int64_t n, int64_t ns);
int64_t mc_oz2_xch_bytes(int nsm);
cudaError_t launch_mc_oz2_chunk(int64_t n, const int8_t *LA, const double *rowscale, const double *a, uint64_t seed,
                                int64_t s0, int64_t ns, int8_t *ZB, double *xch, int *first, unsigned long long *count,
                                int nsm, cudaStream_t st);
cudaError_t launch_mc_oz_chunk(int64_t n, const int8_t *LA, const double *rowscale, const double *a, uint64_t seed,
                               int64_t s0, int64_t ns, int8_t *ZB, int *first, unsigned long long *count, int nsm,
                               cudaStream_t st);

}  // namespace mvn
