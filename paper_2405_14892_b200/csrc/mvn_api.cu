// libmvn C ABI (include/mvn.h): argument validation, workspace, lattice tables, host steps
// (a1 marginal order, a10 regions) and launch orchestration. No Python, no CPU fallback.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/mvn.h"
#include "mvn_internal.h"
#include "common.cuh"

struct mvn_ctx {
    int device = 0;
    int nsm = 148;
    cudaStream_t stream = nullptr;
    std::string err;
    // workspace (device)
    void *Y = nullptr; size_t Y_cap = 0;
    void *part = nullptr; size_t part_cap = 0;
    void *cta = nullptr; size_t cta_cap = 0;
    void *sync = nullptr; size_t sync_cap = 0;   // SOV lockstep counters + need[]
    uint64_t *G = nullptr; int64_t G_n = 0;
    int64_t *d_info = nullptr;
    // recorded on the bound stream at the end of every entry point (DevGuard); a stream change
    // makes the new stream wait on it, so work enqueued on two streams never shares the workspace
    // concurrently (the workspace above is per context, not per stream)
    cudaEvent_t done = nullptr;
    // mvn_crd buffers
    void *crd_L = nullptr; size_t crd_L_cap = 0;
    void *crd_vec = nullptr; size_t crd_vec_cap = 0;
    // mvn_posterior: augmented matrix (Schur complement = Sigma_post) and small vectors
    void *post = nullptr; size_t post_cap = 0;
    void *postv = nullptr; size_t postv_cap = 0;
    int64_t post_n = 0, post_off = 0;
    // mvn_mc_validate
    void *mcZ = nullptr; size_t mcZ_cap = 0;
    void *mcLA = nullptr; size_t mcLA_cap = 0;     // int8 slices of L (method 1)
    void *mcRS = nullptr; size_t mcRS_cap = 0;     // per-row scales
    void *mcX = nullptr; size_t mcX_cap = 0;       // method 2: cluster exchange scratch
    void *mcF = nullptr; size_t mcF_cap = 0;
    void *sozX = nullptr; size_t sozX_cap = 0;     // int8 SOV: cluster exchange scratch
    void *pozA = nullptr; size_t pozA_cap = 0;     // int8 POTRF: panel digit slices
    void *pozR = nullptr; size_t pozR_cap = 0;     // int8 POTRF: panel row scales
    void *pozX = nullptr; size_t pozX_cap = 0;     // int8 POTRF: cluster exchange scratch
    void *tlrW = nullptr; size_t tlrW_cap = 0;     // TLR Cholesky: panel + M / Z chunks + overflow flag
    void *tlrS = nullptr; size_t tlrS_cap = 0;     // mvn_crd with MVN_CRD_TLR: the factor slots U, V and ranks
    // mvn_sweep state: stream-ordered allocations from the context's own pool, which keeps the
    // memory between sweeps (no re-mapping per sweep) until mvn_trim / mvn_destroy
    cudaMemPool_t pool = nullptr;
};

namespace {

mvn_status fail(mvn_ctx *c, mvn_status s, const std::string &msg) {
    if (c) c->err = msg;
    return s;
}

mvn_status cuda_fail(mvn_ctx *c, cudaError_t e, const char *where) {
    return fail(c, MVN_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define MVN_CUDA(ctx, call)                                              \
    do {                                                                 \
        cudaError_t _e = (call);                                         \
        if (_e != cudaSuccess) return cuda_fail((ctx), _e, #call);       \
    } while (0)

mvn_status ensure(mvn_ctx *c, void **buf, size_t *cap, size_t bytes) {
    if (*cap >= bytes) return MVN_OK;
    if (*buf) {
        cudaStreamSynchronize(c->stream);
        cudaFree(*buf);
        *buf = nullptr;
        *cap = 0;
    }
    cudaError_t e = cudaMalloc(buf, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(c, MVN_E_NOMEM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed: " + cudaGetErrorString(e));
    }
    *cap = bytes;
    return MVN_OK;
}

// Every entry point runs on the context's device (the caller's current device is restored on
// return), so one process may drive several GPUs through several contexts.
// The guard also records the context's `done` event on its stream when the call returns (the
// ordering point mvn_set_stream hands to a new stream).
struct DevGuard {
    int prev = -1;
    const mvn_ctx *ctx = nullptr;
    explicit DevGuard(const mvn_ctx *c) : ctx(c) {
        int cur = -1;
        if (c && cudaGetDevice(&cur) == cudaSuccess && cur != c->device && cudaSetDevice(c->device) == cudaSuccess) prev = cur;
    }
    ~DevGuard() {
        if (ctx && ctx->done) cudaEventRecord(ctx->done, ctx->stream);
        if (prev >= 0) cudaSetDevice(prev);
    }
    DevGuard(const DevGuard &) = delete;
    DevGuard &operator=(const DevGuard &) = delete;
};

bool tiles_ok(mvn_tiles t) { return t.n >= 1 && t.nb == mvn::kTile; }

// ----------------------------------------------------------------------------- lattice (R8)
std::vector<uint64_t> first_primes(int64_t n) {
    std::vector<uint64_t> out;
    if (n <= 0) return out;
    const double ln = std::log((double)std::max<int64_t>(n, 6));
    const uint64_t bound = n < 6 ? 15 : (uint64_t)(n * (ln + std::log(ln))) + 1;
    std::vector<uint8_t> comp(bound + 1, 0);
    for (uint64_t c = 2; c <= bound && (int64_t)out.size() < n; ++c) {
        if (comp[c]) continue;
        out.push_back(c);
        for (uint64_t m = c * c; m <= bound; m += c) comp[m] = 1;
    }
    return out;
}

// floor(frac(sqrt(p)) * 2^64) = floor(sqrt(p * 2^128)) mod 2^64 by a bitwise search on the fraction
// b: the largest b with (a 2^64 + b)^2 <= p 2^128, a = floor(sqrt p), tested exactly in 128-bit
// integers as 2ab + floor(b^2 / 2^64) + frac <= (p - a^2) 2^64.
uint64_t sqrt_frac64(uint64_t p) {
    uint64_t a = (uint64_t)std::sqrt((double)p);
    while (a * a > p) --a;
    while ((a + 1) * (a + 1) <= p) ++a;
    const unsigned __int128 c = (unsigned __int128)(p - a * a) << 64;
    uint64_t b = 0;
    for (int bit = 63; bit >= 0; --bit) {
        const uint64_t cand = b | (1ull << bit);
        const unsigned __int128 sq = (unsigned __int128)cand * cand;
        const uint64_t hi = (uint64_t)(sq >> 64), lo = (uint64_t)sq;
        const unsigned __int128 X = (unsigned __int128)2 * a * cand + hi;
        const bool ok = X < c || (X == c && lo == 0);
        if (ok) b = cand;
    }
    return b;
}

uint64_t shift64(uint64_t seed, uint64_t r, uint64_t k) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * ((r << 32) + k + 1ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

mvn_status ensure_generators(mvn_ctx *c, int64_t n) {
    if (c->G_n >= n) return MVN_OK;
    std::vector<uint64_t> g((size_t)n);
    mvn_status s = mvn_lattice_generators(n, g.data());
    if (s != MVN_OK) return fail(c, s, "lattice generators");
    if (c->G) { cudaStreamSynchronize(c->stream); cudaFree(c->G); c->G = nullptr; c->G_n = 0; }
    MVN_CUDA(c, cudaMalloc(&c->G, sizeof(uint64_t) * (size_t)n));
    MVN_CUDA(c, cudaMemcpy(c->G, g.data(), sizeof(uint64_t) * (size_t)n, cudaMemcpyHostToDevice));
    c->G_n = n;
    return MVN_OK;
}

}  // namespace

extern "C" {

const char *mvn_version(void) { return "mvn-b200 0.1 (sm_100a, fp64 DMMA)"; }

mvn_status mvn_create(int device, void *cuda_stream, mvn_ctx **out) {
    if (!out) return MVN_E_USAGE;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { cudaGetLastError(); return MVN_E_CUDA; }
    if (device < 0 || device >= ndev) return MVN_E_USAGE;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return MVN_E_CUDA;
    if (prop.major != 10 || prop.minor != 0) return MVN_E_CUDA;   // sm_100a binary only
    mvn_ctx *c = new mvn_ctx();
    c->device = device;
    c->nsm = prop.multiProcessorCount;
    c->stream = (cudaStream_t)cuda_stream;
    {
        DevGuard dev_guard(c);                        // the caller's current device is restored
        const int64_t minus1 = -1;
        if (mvn::potrf_init() != cudaSuccess || mvn::sov_init() != cudaSuccess || mvn::mc_init() != cudaSuccess ||
            mvn::mc_oz_init() != cudaSuccess || mvn::tlr_init() != cudaSuccess || mvn::matern_init() != cudaSuccess || mvn::sov_oz_init() != cudaSuccess || mvn::potrf_oz_init() != cudaSuccess ||
            cudaMalloc(&c->d_info, 2 * sizeof(int64_t)) != cudaSuccess ||
            cudaMemcpy(c->d_info, &minus1, sizeof(int64_t), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            if (c->d_info) cudaFree(c->d_info);
            if (c->done) cudaEventDestroy(c->done);
            c->done = nullptr;
            dev_guard.ctx = nullptr;
            delete c;
            return MVN_E_CUDA;
        }
    }
    *out = c;
    return MVN_OK;
}

void mvn_destroy(mvn_ctx *c) {
    if (!c) return;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    // no stream synchronise: the bound stream may already be destroyed by its owner; cudaFree
    // waits for the device's outstanding work itself
    cudaDeviceSynchronize();
    for (void *p : {c->Y, c->part, c->cta, c->sync, (void *)c->G, (void *)c->d_info, c->crd_L, c->crd_vec, c->mcZ, c->mcF,
                    c->post, c->postv, c->mcLA, c->mcRS, c->mcX, c->sozX, c->pozA, c->pozR, c->pozX, c->tlrW, c->tlrS})
        if (p) cudaFree(p);
    if (c->done) cudaEventDestroy(c->done);
    if (c->pool) cudaMemPoolDestroy(c->pool);
    delete c;
    if (prev >= 0) cudaSetDevice(prev);
}

mvn_status mvn_set_stream(mvn_ctx *c, void *s) {
    if (!c) return MVN_E_USAGE;
    if ((cudaStream_t)s != c->stream && c->done) {
        // everything the context enqueued so far (on the old stream, recorded when each call
        // returned) completes before the new stream's next use of the shared workspace
        int prev = -1;
        cudaGetDevice(&prev);
        if (prev != c->device) cudaSetDevice(c->device);
        const cudaError_t e = cudaStreamWaitEvent((cudaStream_t)s, c->done, 0);
        if (prev >= 0 && prev != c->device) cudaSetDevice(prev);
        if (e != cudaSuccess) return cuda_fail(c, e, "mvn_set_stream: cudaStreamWaitEvent");
    }
    c->stream = (cudaStream_t)s;
    return MVN_OK;
}

const char *mvn_last_error(const mvn_ctx *c) { return c ? c->err.c_str() : "null context"; }

mvn_status mvn_trim(mvn_ctx *c) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    cudaStreamSynchronize(c->stream);
    for (void **p : {&c->Y, &c->part, &c->cta, &c->sync, &c->crd_L, &c->crd_vec, &c->mcZ, &c->mcF, &c->post, &c->postv, &c->mcLA, &c->mcRS, &c->mcX, &c->sozX, &c->pozA, &c->pozR, &c->pozX, &c->tlrW, &c->tlrS})
        if (*p) { cudaFree(*p); *p = nullptr; }
    c->Y_cap = c->part_cap = c->cta_cap = c->sync_cap = c->crd_L_cap = c->crd_vec_cap = c->mcZ_cap = c->mcF_cap = 0;
    c->post_cap = c->postv_cap = c->mcLA_cap = c->mcRS_cap = c->mcX_cap = c->sozX_cap = c->pozA_cap = c->pozR_cap = c->pozX_cap = c->tlrW_cap = c->tlrS_cap = 0;
    c->post_n = c->post_off = 0;
    if (c->pool) cudaMemPoolTrimTo(c->pool, 0);
    return MVN_OK;
}

int64_t mvn_tiles_count(mvn_tiles t) {
    if (!tiles_ok(t)) return -1;
    const int64_t nt = (t.n + t.nb - 1) / t.nb;
    return nt * (nt + 1) / 2;
}

size_t mvn_tiles_bytes(mvn_tiles t) {
    const int64_t c = mvn_tiles_count(t);
    return c < 0 ? 0 : (size_t)c * (size_t)(t.nb * t.nb) * sizeof(double);
}

mvn_status mvn_pack_lower(mvn_ctx *c, mvn_tiles t, const double *d_dense, int64_t ld, double *d_tiles) {
    DevGuard dev_guard(c);
    if (!c || !tiles_ok(t) || !d_dense || !d_tiles || ld < t.n) return fail(c, MVN_E_USAGE, "mvn_pack_lower: bad arguments");
    MVN_CUDA(c, mvn::launch_pack(t.n, d_dense, ld, d_tiles, true, c->stream));
    return MVN_OK;
}

mvn_status mvn_unpack_lower(mvn_ctx *c, mvn_tiles t, const double *d_tiles, double *d_dense, int64_t ld) {
    DevGuard dev_guard(c);
    if (!c || !tiles_ok(t) || !d_dense || !d_tiles || ld < t.n) return fail(c, MVN_E_USAGE, "mvn_unpack_lower: bad arguments");
    MVN_CUDA(c, mvn::launch_pack(t.n, d_dense, ld, const_cast<double *>(d_tiles), false, c->stream));
    return MVN_OK;
}

mvn_status mvn_marginal_order(int64_t n, const double *mu, const double *var, double u, int64_t *order,
                              double *a_sorted, double *pM) {
    if (n < 1 || !mu || !var || !order || !a_sorted || std::isnan(u)) return MVN_E_USAGE;
    std::vector<double> z((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        if (std::isnan(mu[i]) || !(var[i] > 0.0)) return MVN_E_USAGE;
        z[i] = (mu[i] - u) / std::sqrt(var[i]);
    }
    std::vector<int64_t> o((size_t)n);
    std::iota(o.begin(), o.end(), 0);
    std::stable_sort(o.begin(), o.end(), [&](int64_t x, int64_t y) { return z[x] > z[y]; });
    for (int64_t k = 0; k < n; ++k) {
        order[k] = o[k];
        a_sorted[k] = u - mu[o[k]];
    }
    if (pM)
        for (int64_t i = 0; i < n; ++i) pM[i] = 0.5 * std::erfc(-z[i] * 0.70710678118654752440);
    return MVN_OK;
}

mvn_status mvn_cov_matern(mvn_ctx *c, mvn_tiles t, const double *d_xy, double sigma2, double beta, double nu,
                          double nugget, double *d_tiles) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!tiles_ok(t) || !d_xy || !d_tiles || !(sigma2 > 0) || !(beta > 0) || !(nugget >= 0) ||
        !(nu > 0 && nu <= 50))
        return fail(c, MVN_E_USAGE, "mvn_cov_matern: need nb=128, sigma2>0, beta>0, nugget>=0, 0 < nu <= 50");
    MVN_CUDA(c, mvn::launch_cov_matern(t.n, d_xy, sigma2, beta, nu, nugget, d_tiles, c->stream));
    return MVN_OK;
}

mvn_status mvn_potrf(mvn_ctx *c, mvn_tiles t, double *d_tiles, int64_t *info) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!tiles_ok(t) || !d_tiles || !info) return fail(c, MVN_E_USAGE, "mvn_potrf: bad arguments");
    const int64_t minus1 = -1;
    MVN_CUDA(c, cudaMemcpyAsync(c->d_info, &minus1, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    MVN_CUDA(c, mvn::launch_potrf(t.n, d_tiles, c->d_info, c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(info, c->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    MVN_CUDA(c, cudaStreamSynchronize(c->stream));
    if (*info >= 0 && *info < t.n)
        return fail(c, MVN_E_NUMERIC, "mvn_potrf: matrix not positive definite at row " + std::to_string(*info));
    if (*info >= t.n) *info = -1;   // cannot happen (padding is the identity)
    return MVN_OK;
}

mvn_status mvn_potrf_ex(mvn_ctx *c, mvn_tiles t, double *d_tiles, int64_t *info, int32_t method) {
    if (method == MVN_POTRF_FP64) return mvn_potrf(c, t, d_tiles, info);
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (method != MVN_POTRF_INT8) return fail(c, MVN_E_USAGE, "mvn_potrf_ex: method must be MVN_POTRF_FP64 or MVN_POTRF_INT8");
    if (!tiles_ok(t) || !d_tiles || !info) return fail(c, MVN_E_USAGE, "mvn_potrf_ex: bad arguments");
    const int kp = mvn::potrf_panel_width(t.n);
    const int64_t n_pad = (t.n + t.nb - 1) / t.nb * t.nb;
    mvn::PotrfOz oz;
    oz.clusters = mvn::potrf_oz_max_clusters(c->nsm);
    oz.clusters_reserved = std::max(1, std::min(oz.clusters, (c->nsm - mvn::potrf_panel_sms()) / 2));
    mvn_status s;
    if ((s = ensure(c, &c->pozA, &c->pozA_cap, (size_t)mvn::potrf_oz_lap_bytes(t.n, kp))) != MVN_OK) return s;
    if ((s = ensure(c, &c->pozR, &c->pozR_cap, sizeof(double) * (size_t)n_pad)) != MVN_OK) return s;
    if ((s = ensure(c, &c->pozX, &c->pozX_cap, (size_t)mvn::potrf_oz_xch_bytes(oz.clusters))) != MVN_OK) return s;
    oz.LAp = (int8_t *)c->pozA; oz.rs = (double *)c->pozR; oz.xch = (double *)c->pozX;
    const int64_t minus1 = -1;
    MVN_CUDA(c, cudaMemcpyAsync(c->d_info, &minus1, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    MVN_CUDA(c, mvn::launch_potrf_ex(t.n, d_tiles, c->d_info, c->stream, 0, &oz));
    MVN_CUDA(c, cudaMemcpyAsync(info, c->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    MVN_CUDA(c, cudaStreamSynchronize(c->stream));
    if (*info >= 0 && *info < t.n)
        return fail(c, MVN_E_NUMERIC, "mvn_potrf_ex: matrix not positive definite at row " + std::to_string(*info));
    if (*info >= t.n) *info = -1;
    return MVN_OK;
}

mvn_status mvn_potrf_panel(mvn_ctx *c, mvn_tiles t, double *d_tiles, int64_t k, int64_t kp) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    const int64_t nt = tiles_ok(t) ? (t.n + t.nb - 1) / t.nb : 0;
    if (!nt || !d_tiles || k < 0 || k >= nt || kp < 1 || kp > 8) return fail(c, MVN_E_USAGE, "mvn_potrf_panel: bad arguments");
    MVN_CUDA(c, mvn::launch_potrf_panel(t.n, d_tiles, (int)k, (int)kp, c->d_info, c->stream));
    return MVN_OK;
}

mvn_status mvn_potrf_update(mvn_ctx *c, mvn_tiles t, double *d_tiles, int64_t k, int64_t kp, int64_t col_first,
                            int64_t col_stride, int64_t col_block, int32_t sm_reserve) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    const int64_t nt = tiles_ok(t) ? (t.n + t.nb - 1) / t.nb : 0;
    if (!nt || !d_tiles || k < 0 || kp < 1 || kp > 8 || col_first < std::min(k + kp, nt) || col_stride < 1 ||
        col_block < 1 || col_block > col_stride || sm_reserve < 0 || sm_reserve >= c->nsm)
        return fail(c, MVN_E_USAGE, "mvn_potrf_update: bad arguments (need k + kp <= col_first, 1 <= col_block <= col_stride)");
    if (col_first >= nt) return MVN_OK;
    MVN_CUDA(c, mvn::launch_potrf_update(t.n, d_tiles, (int)k, (int)kp, (int)col_first, (int)std::min<int64_t>(col_stride, nt),
                                         (int)std::min<int64_t>(col_block, nt), sm_reserve, c->stream));
    return MVN_OK;
}

int64_t mvn_potrf_panel_width(int64_t n) { return n < 1 ? -1 : mvn::potrf_panel_width(n); }

mvn_status mvn_panel_pack(mvn_ctx *c, mvn_tiles t, const double *d_tiles, int64_t k, int64_t kp, double *d_panel) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    const int64_t nt = tiles_ok(t) ? (t.n + t.nb - 1) / t.nb : 0;
    if (!nt || !d_tiles || !d_panel || k < 0 || k >= nt || kp < 1 || kp > 8)
        return fail(c, MVN_E_USAGE, "mvn_panel_pack: bad arguments");
    MVN_CUDA(c, mvn::launch_panel_copy(t.n, const_cast<double *>(d_tiles), (int)k, (int)kp, d_panel, true, c->stream));
    return MVN_OK;
}

mvn_status mvn_panel_unpack(mvn_ctx *c, mvn_tiles t, const double *d_panel, int64_t k, int64_t kp, double *d_tiles) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    const int64_t nt = tiles_ok(t) ? (t.n + t.nb - 1) / t.nb : 0;
    if (!nt || !d_tiles || !d_panel || k < 0 || k >= nt || kp < 1 || kp > 8)
        return fail(c, MVN_E_USAGE, "mvn_panel_unpack: bad arguments");
    MVN_CUDA(c, mvn::launch_panel_copy(t.n, d_tiles, (int)k, (int)kp, const_cast<double *>(d_panel), false, c->stream));
    return MVN_OK;
}

// ---- NEXT-1 distributed storage: a rank holds only the tiles it owns (TileMap::kDist), 1-D (tile
// columns over all ranks) or 2-D (row blocks over prows process rows x column blocks over the rest)
namespace {
int dP(const mvn_dtiles &d) { return d.prows > 1 ? d.prows : 1; }
int dQ(const mvn_dtiles &d) { return d.world / dP(d); }
int dpr(const mvn_dtiles &d) { return d.rank / dQ(d); }
int dpc(const mvn_dtiles &d) { return d.rank % dQ(d); }
bool dtiles_ok(const mvn_dtiles &d) {
    return d.n >= 1 && d.nb == mvn::kTile && d.world >= 1 && d.rank >= 0 && d.rank < d.world && d.kp >= 1 && d.kp <= 8 &&
           d.prows >= 0 && d.world % dP(d) == 0;
}
int64_t dtiles_nt(const mvn_dtiles &d) { return (d.n + d.nb - 1) / d.nb; }
int64_t dtiles_S(const mvn_dtiles &d) { return (dtiles_nt(d) + d.kp - 1) / d.kp; }
mvn::TileMap dmap(const mvn_dtiles &d, double *local) {
    if (dP(d) == 1) return mvn::TileMap::dist(local, d.world, d.rank, d.kp);
    return mvn::TileMap::dist2(local, dP(d), dpr(d), dQ(d), dpc(d), d.kp);
}
mvn::RowSel drows(const mvn_dtiles &d) {
    mvn::RowSel r;
    r.P = dP(d); r.pr = dpr(d); r.kp = d.kp;
    return r;
}
mvn::TileMap pmap(const mvn_dtiles &d, const double *panel, int64_t s) {
    const int64_t nt = dtiles_nt(d), k = s * d.kp;
    return mvn::TileMap::panel(const_cast<double *>(panel), (int)k, (int)std::min<int64_t>(d.kp, nt - k));
}
}  // namespace

size_t mvn_dtiles_bytes(mvn_dtiles d) {
    if (!dtiles_ok(d)) return 0;
    return (size_t)dmap(d, nullptr).index(dtiles_nt(d), 0) * (size_t)(d.nb * d.nb) * sizeof(double);
}

int64_t mvn_dpanel_numel(mvn_dtiles d, int64_t s) {
    if (!dtiles_ok(d) || s < 0 || s >= dtiles_S(d)) return -1;
    const int64_t nt = dtiles_nt(d), k = s * d.kp, w = std::min<int64_t>(d.kp, nt - k);
    int64_t t = 0;
    for (int64_t j = 0; j < w; ++j) t += nt - k - j;
    return t * d.nb * d.nb;
}

mvn_status mvn_dcov_matern(mvn_ctx *c, mvn_dtiles d, const double *d_xy, double sigma2, double beta, double nu,
                           double nugget, double *d_local) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!dtiles_ok(d) || !d_xy || !d_local || !(sigma2 > 0) || !(beta > 0) || !(nugget >= 0) || !(nu > 0 && nu <= 50))
        return fail(c, MVN_E_USAGE, "mvn_dcov_matern: bad arguments");
    MVN_CUDA(c, mvn::launch_cov_matern_map(d.n, d_xy, sigma2, beta, nu, nugget, dmap(d, d_local), c->stream));
    return MVN_OK;
}

mvn_status mvn_dpotrf_panel(mvn_ctx *c, mvn_dtiles d, double *d_local, int64_t s) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!dtiles_ok(d) || !d_local || s < 0 || s >= dtiles_S(d) || s % dQ(d) != dpc(d) || s % dP(d) != dpr(d))
        return fail(c, MVN_E_USAGE, "mvn_dpotrf_panel: bad arguments (super-panel s's diagonal block must be this rank's)");
    const int64_t k = s * d.kp;
    // 1-D: the whole super-panel; 2-D: its diagonal block only (the rows below: mvn_dpanel_trsm)
    const int row_end = dP(d) == 1 ? 0 : (int)std::min<int64_t>(k + d.kp, dtiles_nt(d));
    MVN_CUDA(c, mvn::launch_potrf_panel_map(d.n, dmap(d, d_local), (int)k, d.kp, c->d_info, c->stream, row_end));
    return MVN_OK;
}

mvn_status mvn_dpanel_trsm(mvn_ctx *c, mvn_dtiles d, double *d_local, int64_t s, const double *d_panel) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!dtiles_ok(d) || !d_local || !d_panel || s < 0 || s >= dtiles_S(d) || s % dQ(d) != dpc(d))
        return fail(c, MVN_E_USAGE, "mvn_dpanel_trsm: bad arguments (super-panel s must be in this rank's process column)");
    if (dP(d) == 1) return MVN_OK;                                                  // 1-D: done by mvn_dpotrf_panel
    MVN_CUDA(c, mvn::launch_panel_trsm_map(d.n, dmap(d, d_local), pmap(d, d_panel, s), (int)(s * d.kp), d.kp, drows(d),
                                           c->stream));
    return MVN_OK;
}

mvn_status mvn_dpanel_pack(mvn_ctx *c, mvn_dtiles d, const double *d_local, int64_t s, double *d_panel) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!dtiles_ok(d) || !d_local || !d_panel || s < 0 || s >= dtiles_S(d) || s % dQ(d) != dpc(d))
        return fail(c, MVN_E_USAGE, "mvn_dpanel_pack: bad arguments (super-panel s must be in this rank's process column)");
    MVN_CUDA(c, mvn::launch_panel_copy_map(d.n, dmap(d, const_cast<double *>(d_local)), pmap(d, d_panel, s),
                                           (int)(s * d.kp), d.kp, c->stream));
    return MVN_OK;
}

mvn_status mvn_dpotrf_update(mvn_ctx *c, mvn_dtiles d, double *d_local, int64_t s, const double *d_panel,
                             int64_t sp_first, int32_t just_one, int32_t sm_reserve) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    const int64_t S = dtiles_S(d);
    if (!dtiles_ok(d) || !d_local || !d_panel || s < 0 || s >= S || sp_first <= s || sm_reserve < 0 || sm_reserve >= c->nsm)
        return fail(c, MVN_E_USAGE, "mvn_dpotrf_update: bad arguments (need 0 <= s < sp_first)");
    // the first super-panel >= sp_first in this rank's process column
    const int Q = dQ(d), pc = dpc(d);
    const int64_t sp0 = sp_first + ((pc - sp_first % Q) % Q + Q) % Q;
    if (sp0 >= S || (just_one && sp0 != sp_first)) return MVN_OK;                 // nothing owned there
    const int64_t nt = dtiles_nt(d);
    const int c0 = (int)(sp0 * d.kp), cs = just_one ? (int)nt : d.kp * Q;
    const mvn::TileMap pm = pmap(d, d_panel, s);
    MVN_CUDA(c, mvn::launch_potrf_update_map(d.n, dmap(d, d_local), pm, pm, (int)(s * d.kp), d.kp, c0, cs, d.kp,
                                             sm_reserve, drows(d), c->stream));
    return MVN_OK;
}

mvn_status mvn_dgather(mvn_ctx *c, mvn_dtiles d, const double *d_local, double *d_tiles) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!dtiles_ok(d) || !d_local || !d_tiles) return fail(c, MVN_E_USAGE, "mvn_dgather: bad arguments");
    const mvn::TileMap from = dmap(d, const_cast<double *>(d_local)), to = mvn::TileMap::full(d_tiles);
    for (int64_t s = dpc(d); s < dtiles_S(d); s += dQ(d))
        MVN_CUDA(c, mvn::launch_panel_copy_map(d.n, from, to, (int)(s * d.kp), d.kp, c->stream));
    return MVN_OK;
}

mvn_status mvn_potrf_info(mvn_ctx *c, int64_t *info, int32_t reset) {
    DevGuard dev_guard(c);
    if (!c || !info) return fail(c, MVN_E_USAGE, "mvn_potrf_info: bad arguments");
    MVN_CUDA(c, cudaMemcpyAsync(info, c->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    if (reset) {
        const int64_t minus1 = -1;
        MVN_CUDA(c, cudaMemcpyAsync(c->d_info, &minus1, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    }
    MVN_CUDA(c, cudaStreamSynchronize(c->stream));
    return MVN_OK;
}

mvn_status mvn_lattice_generators(int64_t n, uint64_t *gen) {
    if (n < 1 || !gen) return MVN_E_USAGE;
    std::vector<uint64_t> p = first_primes(n);
    if ((int64_t)p.size() != n) return MVN_E_USAGE;
    for (int64_t k = 0; k < n; ++k) gen[k] = sqrt_frac64(p[k]);
    return MVN_OK;
}

mvn_status mvn_lattice_shifts(uint64_t seed, int32_t R, int64_t n, uint64_t *D) {
    if (n < 1 || R < 1 || !D) return MVN_E_USAGE;
    for (int64_t r = 0; r < R; ++r)
        for (int64_t k = 0; k < n; ++k) D[r * n + k] = shift64(seed, (uint64_t)r, (uint64_t)k);
    return MVN_OK;
}

namespace {
// The fp64 sweep. Sample mode (u0 < 0): the range [q->sample_begin, q->sample_end), balanced over the
// CTAs, reduced to (M, S). Unit mode: the global 128-sample units [u0, u1), whole units per CTA, the
// per-unit partials left in d_partial ([u1 - u0][n][2]).
struct TlrSlots {
    const double *U = nullptr, *V = nullptr;
    const int *ranks = nullptr;
    int kmax = 0;
};

mvn_status sov_prefix_impl(mvn_ctx *c, mvn_tiles t, const double *d_L, const double *d_a, const double *d_b,
                           const mvn_qmc *q, int64_t u0, int64_t u1, double *d_partial, double *d_M, double *d_S,
                           const TlrSlots *tlr = nullptr) {
    mvn_status s;
    if ((s = ensure_generators(c, t.n)) != MVN_OK) return s;
    {   // NaN limits or a_k > b_k: MVN_E_USAGE (synchronises on a 4-byte flag before the sweep)
        int *d_flag = reinterpret_cast<int *>(c->d_info) + 2;      // spare bytes after the pivot flag
        int h_flag = 0;
        MVN_CUDA(c, mvn::launch_check_limits(t.n, d_a, d_b, d_flag, c->stream));
        MVN_CUDA(c, cudaMemcpyAsync(&h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        MVN_CUDA(c, cudaStreamSynchronize(c->stream));
        if (h_flag) return fail(c, MVN_E_USAGE, "mvn_sov_prefix: a limit is NaN or a_k > b_k");
    }
    const bool units = u0 >= 0;
    const int64_t NR = q->N * (int64_t)q->R;
    const int64_t nsamp = units ? std::min<int64_t>(u1 * 128, NR) - u0 * 128 : q->sample_end - q->sample_begin;
    mvn::SovLaunch L;
    L.L = d_L; L.n = t.n; L.a = d_a; L.b = d_b; L.G = q->d_gen ? q->d_gen : c->G; L.N = q->N; L.seed = q->seed;
    L.g_begin = units ? u0 * 128 : q->sample_begin; L.g_end = units ? std::min<int64_t>(u1 * 128, NR) : q->sample_end;
    L.grid = (int)std::min<int64_t>(units ? u1 - u0 : nsamp, c->nsm);
    std::vector<int64_t> cta((size_t)L.grid * 3);
    L.nblk = units ? mvn::sov_partition_units(u0, u1, L.g_end, L.grid, cta.data())
                   : mvn::sov_partition(q->sample_begin, q->sample_end, L.grid, cta.data());
    L.unit_mode = units ? 1 : 0;
    const int64_t n_pad = (t.n + 63) / 64 * 64;
    const int ys = mvn::sov_y_stride();
    if ((s = ensure(c, &c->Y, &c->Y_cap, (size_t)L.grid * n_pad * ys * sizeof(double))) != MVN_OK) return s;
    if (!units && (s = ensure(c, &c->part, &c->part_cap, (size_t)L.nblk * n_pad * 2 * sizeof(double))) != MVN_OK) return s;
    if ((s = ensure(c, &c->cta, &c->cta_cap, cta.size() * sizeof(int64_t))) != MVN_OK) return s;
    // soft lockstep: need[b] = CTAs with more than b sample blocks; counters [max_blocks][nrb]
    static const int env_lag = [] { const char *e = getenv("MVN_SOV_LAG"); return e ? atoi(e) : 0; }();   // off: measured no gain (r01)
    static const int env_hints = [] { const char *e = getenv("MVN_SOV_HINTS"); return e ? atoi(e) : 1; }();
    const int bs = mvn::sov_block_samples();
    int max_blocks = 0;
    for (int g = 0; g < L.grid; ++g) max_blocks = std::max<int>(max_blocks, (int)((cta[3 * g + 1] + bs - 1) / bs));
    max_blocks = std::max(max_blocks, 1);
    std::vector<int> sync_host((size_t)max_blocks, 0);
    for (int g = 0; g < L.grid; ++g)
        for (int b = 0; b < (int)((cta[3 * g + 1] + bs - 1) / bs); ++b) ++sync_host[(size_t)b];
    const int64_t nrb = (t.n + 63) / 64;
    const size_t sync_bytes = sizeof(int) * ((size_t)max_blocks * nrb + max_blocks);
    if ((s = ensure(c, &c->sync, &c->sync_cap, sync_bytes)) != MVN_OK) return s;
    int *d_sync = (int *)c->sync;
    MVN_CUDA(c, cudaMemcpyAsync(d_sync + (size_t)max_blocks * nrb, sync_host.data(), sizeof(int) * max_blocks,
                                cudaMemcpyHostToDevice, c->stream));
    L.lag = env_lag; L.step_done = d_sync; L.need = d_sync + (size_t)max_blocks * nrb; L.max_blocks = max_blocks;
    L.hints = env_hints;
    static const int env_serial = [] { const char *e = getenv("MVN_SOV_SERIAL"); return e ? atoi(e) : 0; }();   // off: measured no gain (r01, r02)
    L.serial_rb = env_serial;
    MVN_CUDA(c, cudaMemcpyAsync(c->cta, cta.data(), cta.size() * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    L.cta = (const int64_t *)c->cta;
    L.Y = (double *)c->Y; L.part = units ? d_partial : (double *)c->part; L.Mout = d_M; L.Sout = d_S;
    if (tlr) {
        L.tU = tlr->U; L.tV = tlr->V; L.tranks = tlr->ranks; L.tkmax = tlr->kmax;
        L.lag = 0;
    }
    MVN_CUDA(c, mvn::launch_sov(L, c->stream));
    return MVN_OK;
}
}  // namespace

mvn_status mvn_sov_prefix(mvn_ctx *c, mvn_tiles t, const double *d_L, const double *d_a, const double *d_b,
                          const mvn_qmc *q, double *d_M, double *d_S) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!tiles_ok(t) || !d_L || !d_a || !q || !d_M || !d_S || q->N < 1 || q->R < 1 || q->sample_begin < 0 ||
        q->sample_end <= q->sample_begin || q->sample_end > q->N * (int64_t)q->R)
        return fail(c, MVN_E_USAGE, "mvn_sov_prefix: bad arguments (need nb=128, 0 <= begin < end <= N*R)");
    return sov_prefix_impl(c, t, d_L, d_a, d_b, q, -1, -1, nullptr, d_M, d_S);
}

mvn_status mvn_sov_prefix_tlr(mvn_ctx *c, mvn_tiles t, const double *d_L, const double *d_U, const double *d_V,
                              const int32_t *d_ranks, int32_t kmax, const double *d_a, const double *d_b, const mvn_qmc *q,
                              double *d_M, double *d_S) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    const int64_t nt = (t.n + 127) / 128;
    if (!tiles_ok(t) || !d_L || !d_a || !q || !d_M || !d_S || q->N < 1 || q->R < 1 || q->sample_begin < 0 ||
        q->sample_end <= q->sample_begin || q->sample_end > q->N * (int64_t)q->R || kmax < 1 || kmax > 128 ||
        (nt > 1 && (!d_U || !d_V || !d_ranks)))
        return fail(c, MVN_E_USAGE, "mvn_sov_prefix_tlr: bad arguments (need nb=128, 0 <= begin < end <= N*R, 1 <= kmax <= 128, factor slots)");
    TlrSlots ts;
    ts.U = d_U; ts.V = d_V; ts.ranks = d_ranks; ts.kmax = kmax;
    if (nt == 1) { ts.U = ts.V = d_L; }               // no off-diagonal tile: the slots are never read
    return sov_prefix_impl(c, t, d_L, d_a, d_b, q, -1, -1, nullptr, d_M, d_S, &ts);
}

mvn_status mvn_sov_prefix_units(mvn_ctx *c, mvn_tiles t, const double *d_L, const double *d_a, const double *d_b,
                                const mvn_qmc *q, int64_t unit_begin, int64_t unit_end, double *d_partial) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    const int64_t U = q ? (q->N * (int64_t)q->R + 127) / 128 : 0;
    if (!tiles_ok(t) || !d_L || !d_a || !q || !d_partial || q->N < 1 || q->R < 1 || unit_begin < 0 ||
        unit_end <= unit_begin || unit_end > U)
        return fail(c, MVN_E_USAGE, "mvn_sov_prefix_units: bad arguments (need nb=128, 0 <= unit_begin < unit_end <= ceil(N*R/128))");
    return sov_prefix_impl(c, t, d_L, d_a, d_b, q, unit_begin, unit_end, d_partial, nullptr, nullptr);
}

}  // extern "C"

struct mvn_sweep {
    mvn_ctx *c = nullptr;
    int64_t n = 0, nt = 0, n_pad = 0, next = 0, nblk = 0, g_begin = 0, g_end = 0, N = 0;
    uint64_t seed = 0;
    int grid = 0;
    double *a = nullptr, *b = nullptr, *Y = nullptr, *part = nullptr, *ell = nullptr;
    uint64_t *G = nullptr;
    int64_t *cta = nullptr, *yoff = nullptr;
};

namespace {
void sweep_release(mvn_sweep *sw) {
    if (!sw) return;
    cudaStream_t st = sw->c ? sw->c->stream : nullptr;
    for (void *p : {(void *)sw->a, (void *)sw->b, (void *)sw->Y, (void *)sw->part, (void *)sw->ell, (void *)sw->G,
                    (void *)sw->cta, (void *)sw->yoff})
        if (p) cudaFreeAsync(p, st);
    delete sw;
}
template <class T>
cudaError_t sweep_alloc(mvn_ctx *c, T **p, size_t count) {
    if (!c->pool) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = c->device;
        cudaError_t e = cudaMemPoolCreate(&c->pool, &props);
        if (e != cudaSuccess) { c->pool = nullptr; return e; }
        uint64_t keep = UINT64_MAX;
        if ((e = cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess) return e;
    }
    return cudaMallocFromPoolAsync(reinterpret_cast<void **>(p), std::max<size_t>(count, 1) * sizeof(T), c->pool, c->stream);
}
}  // namespace

extern "C" {

mvn_status mvn_sweep_begin(mvn_ctx *c, int64_t n, const double *d_a, const double *d_b, const mvn_qmc *q,
                           mvn_sweep **out) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!out || n < 1 || !d_a || !q || q->N < 1 || q->R < 1 || q->sample_begin < 0 ||
        q->sample_end <= q->sample_begin || q->sample_end > q->N * (int64_t)q->R)
        return fail(c, MVN_E_USAGE, "mvn_sweep_begin: bad arguments (0 <= begin < end <= N*R)");
    *out = nullptr;
    mvn_status s;
    if ((s = ensure_generators(c, n)) != MVN_OK) return s;
    {
        int *d_flag = reinterpret_cast<int *>(c->d_info) + 2;
        int h_flag = 0;
        MVN_CUDA(c, mvn::launch_check_limits(n, d_a, d_b, d_flag, c->stream));
        MVN_CUDA(c, cudaMemcpyAsync(&h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        MVN_CUDA(c, cudaStreamSynchronize(c->stream));
        if (h_flag) return fail(c, MVN_E_USAGE, "mvn_sweep_begin: a limit is NaN or a_k > b_k");
    }
    mvn_sweep *sw = new mvn_sweep;
    sw->c = c; sw->n = n; sw->nt = (n + mvn::kTile - 1) / mvn::kTile; sw->n_pad = (n + 63) / 64 * 64;
    sw->g_begin = q->sample_begin; sw->g_end = q->sample_end; sw->N = q->N; sw->seed = q->seed;
    const int64_t nsamp = sw->g_end - sw->g_begin;
    sw->grid = (int)std::min<int64_t>(nsamp, c->nsm);
    std::vector<int64_t> cta((size_t)sw->grid * 3), yoff((size_t)sw->grid);
    sw->nblk = mvn::sov_partition(sw->g_begin, sw->g_end, sw->grid, cta.data());
    const int64_t ydoubles = mvn::sov_phase_yoff(cta.data(), sw->grid, sw->n_pad, 0, yoff.data());
    cudaStream_t st = c->stream;
    cudaError_t e = cudaSuccess;
    if (!e) e = sweep_alloc(c, &sw->a, (size_t)n);
    if (!e && d_b) e = sweep_alloc(c, &sw->b, (size_t)n);
    if (!e) e = sweep_alloc(c, &sw->G, (size_t)n);
    if (!e) e = sweep_alloc(c, &sw->cta, cta.size());
    if (!e) e = sweep_alloc(c, &sw->yoff, yoff.size());
    if (!e) e = sweep_alloc(c, &sw->Y, (size_t)ydoubles);
    if (!e) e = sweep_alloc(c, &sw->part, (size_t)sw->nblk * sw->n_pad * 2);
    if (!e) e = sweep_alloc(c, &sw->ell, (size_t)nsamp);
    if (!e) e = cudaMemcpyAsync(sw->a, d_a, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
    if (!e && d_b) e = cudaMemcpyAsync(sw->b, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
    if (!e) e = cudaMemcpyAsync(sw->G, q->d_gen ? q->d_gen : c->G, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, st);
    if (!e) e = cudaMemcpyAsync(sw->cta, cta.data(), sizeof(int64_t) * cta.size(), cudaMemcpyHostToDevice, st);
    if (!e) e = cudaMemcpyAsync(sw->yoff, yoff.data(), sizeof(int64_t) * yoff.size(), cudaMemcpyHostToDevice, st);
    if (!e) e = cudaStreamSynchronize(st);               // the host vectors above go out of scope
    if (e) {
        sweep_release(sw);
        return cuda_fail(c, e, "mvn_sweep_begin");
    }
    *out = sw;
    return MVN_OK;
}

mvn_status mvn_sweep_rows(mvn_sweep *sw, const double *d_rows, int64_t tb, int64_t te) {
    if (!sw) return MVN_E_USAGE;
    mvn_ctx *c = sw->c;
    DevGuard dev_guard(c);
    if (!d_rows || tb != sw->next || te <= tb || te > sw->nt)
        return fail(c, MVN_E_USAGE, "mvn_sweep_rows: rows must continue where the previous call stopped (tile_row_begin = " +
                                        std::to_string(sw->next) + ", begin < end <= " + std::to_string(sw->nt) + ")");
    mvn::SovLaunch L;
    // the kernels address tile (i, j) as L + (i(i+1)/2 + j) nb^2; only rows [tb, te) are read
    const int64_t shift = tb * (tb + 1) / 2 * (int64_t)mvn::kTile * mvn::kTile;
    L.L = reinterpret_cast<const double *>(reinterpret_cast<uintptr_t>(d_rows) - (uintptr_t)shift * sizeof(double));
    L.n = sw->n; L.a = sw->a; L.b = sw->b; L.G = sw->G; L.N = sw->N; L.seed = sw->seed;
    L.g_begin = sw->g_begin; L.g_end = sw->g_end; L.cta = sw->cta; L.nblk = sw->nblk; L.grid = sw->grid;
    L.Y = sw->Y; L.part = sw->part; L.lag = 0; L.hints = 1;
    const int64_t nrb = sw->n_pad / 64;
    L.rb0 = (int)(2 * tb); L.rb1 = (int)std::min<int64_t>(2 * te, nrb);
    L.ell = sw->ell; L.yoff = sw->yoff;
    MVN_CUDA(c, mvn::launch_sov(L, c->stream));
    sw->next = te;
    return MVN_OK;
}

mvn_status mvn_sweep_end(mvn_sweep *sw, double *d_M, double *d_S) {
    if (!sw) return MVN_E_USAGE;
    mvn_ctx *c = sw->c;
    DevGuard dev_guard(c);
    if (!d_M || !d_S || sw->next != sw->nt)
        return fail(c, MVN_E_USAGE, "mvn_sweep_end: bad arguments or rows missing (next tile row " + std::to_string(sw->next) +
                                        " of " + std::to_string(sw->nt) + ")");
    MVN_CUDA(c, mvn::launch_reduce_blocks(sw->part, sw->nblk, sw->n, sw->n_pad, d_M, d_S, c->stream));
    sweep_release(sw);
    return MVN_OK;
}

void mvn_sweep_free(mvn_sweep *sw) {
    if (!sw) return;
    DevGuard dev_guard(sw->c);
    sweep_release(sw);
}

int64_t mvn_drows_offset(mvn_dtiles d, int64_t i) {
    if (!dtiles_ok(d) || i < 0 || i > dtiles_nt(d)) return -1;
    return dmap(d, nullptr).index(i, 0) * (int64_t)(d.nb * d.nb);
}

mvn_status mvn_drows_unpack(mvn_ctx *c, mvn_dtiles d, const double *d_piece, int64_t tb, int64_t te, double *d_rows) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!dtiles_ok(d) || !d_piece || !d_rows || tb < 0 || te <= tb || te > dtiles_nt(d))
        return fail(c, MVN_E_USAGE, "mvn_drows_unpack: bad arguments");
    const uintptr_t from_shift = (uintptr_t)mvn_drows_offset(d, tb) * sizeof(double);
    const uintptr_t to_shift = (uintptr_t)(tb * (tb + 1) / 2) * mvn::kTile * mvn::kTile * sizeof(double);
    const mvn::TileMap from = dmap(d, reinterpret_cast<double *>(reinterpret_cast<uintptr_t>(d_piece) - from_shift));
    const mvn::TileMap to = mvn::TileMap::full(reinterpret_cast<double *>(reinterpret_cast<uintptr_t>(d_rows) - to_shift));
    MVN_CUDA(c, mvn::launch_rows_copy_map(from, to, (int)tb, (int)te, c->stream));
    return MVN_OK;
}

mvn_status mvn_prefix_reduce(mvn_ctx *c, int64_t n, int64_t units, const double *d_partial, double *d_M, double *d_S) {
    DevGuard dev_guard(c);
    if (!c || n < 1 || units < 1 || !d_partial || !d_M || !d_S) return fail(c, MVN_E_USAGE, "mvn_prefix_reduce: bad arguments");
    MVN_CUDA(c, mvn::launch_reduce_units(d_partial, units, n, d_M, d_S, c->stream));
    return MVN_OK;
}

mvn_status mvn_sov_prefix_ex(mvn_ctx *c, mvn_tiles t, const double *d_L, const double *d_a, const double *d_b,
                             const mvn_qmc *q, int32_t method, double *d_M, double *d_S) {
    if (method == MVN_SOV_FP64) return mvn_sov_prefix(c, t, d_L, d_a, d_b, q, d_M, d_S);
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (method != MVN_SOV_INT8) return fail(c, MVN_E_USAGE, "mvn_sov_prefix_ex: method must be MVN_SOV_FP64 or MVN_SOV_INT8");
    if (!tiles_ok(t) || !d_L || !d_a || d_b || !q || !d_M || !d_S || q->N < 1 || q->R < 1 || q->sample_begin < 0 ||
        q->sample_end <= q->sample_begin || q->sample_end > q->N * (int64_t)q->R)
        return fail(c, MVN_E_USAGE, "mvn_sov_prefix_ex (int8): bad arguments (need nb=128, b = NULL (+inf), 0 <= begin < end <= N*R)");
    mvn_status s;
    if ((s = ensure_generators(c, t.n)) != MVN_OK) return s;
    int *d_flag = reinterpret_cast<int *>(c->d_info) + 2;
    {
        int h_flag = 0;
        MVN_CUDA(c, mvn::launch_check_limits(t.n, d_a, nullptr, d_flag, c->stream));
        MVN_CUDA(c, cudaMemcpyAsync(&h_flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        MVN_CUDA(c, cudaStreamSynchronize(c->stream));
        if (h_flag) return fail(c, MVN_E_USAGE, "mvn_sov_prefix_ex: a limit is NaN");
    }
    // L -> per-row scales and 8 int8 slices in the tcgen05 operand layout (reading R24)
    const int64_t nt = (t.n + t.nb - 1) / t.nb, n_pad = nt * t.nb;
    if ((s = ensure(c, &c->mcLA, &c->mcLA_cap, (size_t)mvn::mc_oz_la_bytes(t.n))) != MVN_OK) return s;
    if ((s = ensure(c, &c->mcRS, &c->mcRS_cap, sizeof(double) * (size_t)n_pad)) != MVN_OK) return s;
    MVN_CUDA(c, mvn::launch_mc_oz_prepare(t.n, d_L, (double *)c->mcRS, (int8_t *)c->mcLA, c->stream));
    const int64_t nsamp = q->sample_end - q->sample_begin;
    mvn::SovOzLaunch L;
    L.clusters = (int)std::min<int64_t>(mvn::sov_oz_max_clusters(c->nsm), (nsamp + 127) / 128);
    std::vector<int64_t> cl((size_t)L.clusters * 3);
    L.nblk = mvn::sov_oz_partition(q->sample_begin, q->sample_end, L.clusters, cl.data());
    if ((s = ensure(c, &c->Y, &c->Y_cap, (size_t)mvn::sov_oz_ys_bytes(t.n, L.clusters))) != MVN_OK) return s;
    if ((s = ensure(c, &c->sozX, &c->sozX_cap, (size_t)mvn::sov_oz_xch_bytes(L.clusters))) != MVN_OK) return s;
    if ((s = ensure(c, &c->part, &c->part_cap, (size_t)(2 * L.nblk) * n_pad * 2 * sizeof(double))) != MVN_OK) return s;
    if ((s = ensure(c, &c->cta, &c->cta_cap, cl.size() * sizeof(int64_t))) != MVN_OK) return s;
    MVN_CUDA(c, cudaMemcpyAsync(c->cta, cl.data(), cl.size() * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    L.LA = (const int8_t *)c->mcLA; L.rowscale = (const double *)c->mcRS; L.L = d_L; L.n = t.n; L.a = d_a; L.G = q->d_gen ? q->d_gen : c->G;
    L.N = q->N; L.seed = q->seed; L.cl = (const int64_t *)c->cta; L.YS = (int8_t *)c->Y; L.xch = (double *)c->sozX;
    L.part = (double *)c->part; L.Mout = d_M; L.Sout = d_S; L.flag = d_flag;
    // soft cluster lockstep (MVN_SOV_OZ_LAG steps, default 1; 0 = off): clusters stay within `lag` row
    // blocks of each other, so the L-slice chunks they all stream are served from L2 more often.
    // Measured at D: lag 0 / 1 / 3 / 8 -> 5.79-5.84 / 5.45 / 5.56 / 5.67 s (profiles/r02_sov_int8.md).
    static const int env_lag = [] { const char *e = getenv("MVN_SOV_OZ_LAG"); return e ? atoi(e) : 1; }();
    if (env_lag > 0) {
        int max_blocks = 0;
        for (int g = 0; g < L.clusters; ++g) max_blocks = std::max<int>(max_blocks, (int)((cl[3 * g + 1] + 127) / 128));
        std::vector<int> need((size_t)max_blocks, 0);
        for (int g = 0; g < L.clusters; ++g)
            for (int b = 0; b < (int)((cl[3 * g + 1] + 127) / 128); ++b) ++need[(size_t)b];
        const int64_t nrb = (t.n + 127) / 128;
        const size_t bytes = sizeof(int) * ((size_t)max_blocks * std::max<int64_t>(nrb - 1, 1) + max_blocks);
        if ((s = ensure(c, &c->sync, &c->sync_cap, bytes)) != MVN_OK) return s;
        int *d_sync = (int *)c->sync;
        int *d_need = d_sync + (size_t)max_blocks * std::max<int64_t>(nrb - 1, 1);
        MVN_CUDA(c, cudaMemcpyAsync(d_need, need.data(), sizeof(int) * max_blocks, cudaMemcpyHostToDevice, c->stream));
        L.lag = env_lag; L.step_done = d_sync; L.need = d_need; L.max_blocks = max_blocks;
    }
    MVN_CUDA(c, mvn::launch_sov_oz(L, c->stream));
    int h_big = 0;
    MVN_CUDA(c, cudaMemcpyAsync(&h_big, d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    MVN_CUDA(c, cudaStreamSynchronize(c->stream));
    if (h_big) return fail(c, MVN_E_NUMERIC, "mvn_sov_prefix_ex (int8): a sample value |y| >= 63.5 is outside the int8 path's fixed scale; use MVN_SOV_FP64");
    return MVN_OK;
}

mvn_status mvn_prefix_rescale(mvn_ctx *c, int64_t n, const double *d_Mglob, double *d_M, double *d_S) {
    DevGuard dev_guard(c);
    if (!c || n < 1 || !d_Mglob || !d_M || !d_S) return fail(c, MVN_E_USAGE, "mvn_prefix_rescale: bad arguments");
    MVN_CUDA(c, mvn::launch_rescale(n, d_Mglob, d_M, d_S, c->stream));
    return MVN_OK;
}

mvn_status mvn_prefix_finalize(mvn_ctx *c, int64_t n, int64_t NR, const double *d_M, const double *d_S, double *d_logP) {
    DevGuard dev_guard(c);
    if (!c || n < 1 || NR < 1 || !d_M || !d_S || !d_logP) return fail(c, MVN_E_USAGE, "mvn_prefix_finalize: bad arguments");
    MVN_CUDA(c, mvn::launch_finalize(n, NR, d_M, d_S, d_logP, c->stream));
    return MVN_OK;
}

mvn_status mvn_sov_prefix_shifts(mvn_ctx *c, mvn_tiles t, const double *d_L, const double *d_a, const double *d_b,
                                 const mvn_qmc *q, double *d_logP_shift) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!tiles_ok(t) || !d_L || !d_a || !q || !d_logP_shift || q->N < 1 || q->R < 1)
        return fail(c, MVN_E_USAGE, "mvn_sov_prefix_shifts: bad arguments (need nb=128, N >= 1, R >= 1)");
    mvn_status s;
    // (M, S) of one shift in the context's small-vector scratch (n x 2); every shift's sweep is the
    // sample range [r N, (r + 1) N) of mvn_sov_prefix, finalised into row r of d_logP_shift
    if ((s = ensure(c, &c->crd_vec, &c->crd_vec_cap, sizeof(double) * 2 * (size_t)t.n)) != MVN_OK) return s;
    double *dM = (double *)c->crd_vec, *dS = dM + t.n;
    for (int32_t r = 0; r < q->R; ++r) {
        mvn_qmc qr = *q;
        qr.sample_begin = (int64_t)r * q->N;
        qr.sample_end = qr.sample_begin + q->N;
        if ((s = sov_prefix_impl(c, t, d_L, d_a, d_b, &qr, -1, -1, nullptr, dM, dS)) != MVN_OK) return s;
        MVN_CUDA(c, mvn::launch_finalize(t.n, q->N, dM, dS, d_logP_shift + (int64_t)r * t.n, c->stream));
    }
    return MVN_OK;
}

mvn_status mvn_prefix_shift_stats(int64_t n, int32_t R, const double *logP_shift, double *logP, double *rel_se) {
    if (n < 1 || R < 1 || !logP_shift || !logP || !rel_se) return MVN_E_USAGE;
    for (int64_t k = 0; k < n; ++k) {
        double m = -INFINITY;
        for (int32_t r = 0; r < R; ++r) m = std::max(m, logP_shift[(int64_t)r * n + k]);
        if (!(m > -INFINITY)) {
            logP[k] = -INFINITY;
            rel_se[k] = NAN;
            continue;
        }
        double sx = 0.0;
        for (int32_t r = 0; r < R; ++r) sx += std::exp(logP_shift[(int64_t)r * n + k] - m);
        const double xm = sx / R;
        double ss = 0.0;
        for (int32_t r = 0; r < R; ++r) {
            const double d = std::exp(logP_shift[(int64_t)r * n + k] - m) - xm;
            ss += d * d;
        }
        logP[k] = m + std::log(xm);
        rel_se[k] = R > 1 ? std::sqrt(ss / (R - 1)) / (std::sqrt((double)R) * xm) : 0.0;
    }
    return MVN_OK;
}

mvn_status mvn_confidence_region(int64_t n, const double *logP, const double *conf, int64_t nconf, int64_t *k_out,
                                 int32_t *near_tie) {
    if (n < 0 || (n > 0 && !logP) || nconf < 0 || (nconf > 0 && (!conf || !k_out))) return MVN_E_USAGE;
    std::vector<double> lp((size_t)n);
    double run = INFINITY;
    for (int64_t k = 0; k < n; ++k) {
        if (std::isnan(logP[k])) return MVN_E_USAGE;
        run = std::min(run, logP[k]);
        lp[k] = run;
    }
    for (int64_t i = 0; i < nconf; ++i) {
        if (!(conf[i] > 0.0 && conf[i] < 1.0)) return MVN_E_USAGE;
        const double lc = std::log(conf[i]);
        // lp is non-increasing: k* = number of prefixes with log P_k >= log c
        const int64_t k = std::partition_point(lp.begin(), lp.end(), [&](double v) { return v >= lc; }) - lp.begin();
        k_out[i] = k;
        if (near_tie)
            near_tie[i] = ((k > 0 && std::fabs(lp[k - 1] - lc) <= 1e-8) || (k < n && std::fabs(lp[k] - lc) <= 1e-8)) ? 1 : 0;
    }
    return MVN_OK;
}

mvn_status mvn_mc_validate(mvn_ctx *c, mvn_tiles t, const double *d_L, const double *d_a, const mvn_mc *m,
                           uint64_t *d_count, int32_t *d_first) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!tiles_ok(t) || !d_L || !d_a || !m || !d_count || m->sample_begin < 0 || m->sample_end <= m->sample_begin)
        return fail(c, MVN_E_USAGE, "mvn_mc_validate: bad arguments (need nb=128, 0 <= begin < end)");
    const int64_t total = m->sample_end - m->sample_begin;
    if (m->method == 1 || m->method == 2) {
        // int8 tensor-core emulation: slice L once, then chunks of draws (Z slices <= ~8 GB)
        const int64_t nt = (t.n + t.nb - 1) / t.nb;
        mvn_status s;
        if ((s = ensure(c, &c->mcLA, &c->mcLA_cap, (size_t)mvn::mc_oz_la_bytes(t.n))) != MVN_OK) return s;
        if ((s = ensure(c, &c->mcRS, &c->mcRS_cap, sizeof(double) * (size_t)(nt * t.nb))) != MVN_OK) return s;
        MVN_CUDA(c, mvn::launch_mc_oz_prepare(t.n, d_L, (double *)c->mcRS, (int8_t *)c->mcLA, c->stream));
        const int blk = m->method == 1 ? 64 : 128;
        const int64_t perblk = m->method == 1 ? mvn::mc_oz_zb_bytes(t.n, blk) : mvn::mc_oz2_zb_bytes(t.n, blk);
        const int64_t chunk = std::min<int64_t>(total, std::max<int64_t>(1, (int64_t)(8ll << 30) / perblk) * blk);
        const int64_t zb = m->method == 1 ? mvn::mc_oz_zb_bytes(t.n, chunk) : mvn::mc_oz2_zb_bytes(t.n, chunk);
        if ((s = ensure(c, &c->mcZ, &c->mcZ_cap, (size_t)zb)) != MVN_OK) return s;
        if (m->method == 2 && (s = ensure(c, &c->mcX, &c->mcX_cap, (size_t)mvn::mc_oz2_xch_bytes(c->nsm))) != MVN_OK) return s;
        if (!d_first && (s = ensure(c, &c->mcF, &c->mcF_cap, (size_t)chunk * sizeof(int32_t))) != MVN_OK) return s;
        for (int64_t s0 = 0; s0 < total; s0 += chunk) {
            const int64_t ns = std::min(chunk, total - s0);
            int *first = d_first ? (int *)d_first + s0 : (int *)c->mcF;
            if (m->method == 1)
                MVN_CUDA(c, mvn::launch_mc_oz_chunk(t.n, (const int8_t *)c->mcLA, (const double *)c->mcRS, d_a, m->seed,
                                                    m->sample_begin + s0, ns, (int8_t *)c->mcZ, first,
                                                    (unsigned long long *)d_count, c->nsm, c->stream));
            else
                MVN_CUDA(c, mvn::launch_mc_oz2_chunk(t.n, (const int8_t *)c->mcLA, (const double *)c->mcRS, d_a, m->seed,
                                                     m->sample_begin + s0, ns, (int8_t *)c->mcZ, (double *)c->mcX, first,
                                                     (unsigned long long *)d_count, c->nsm, c->stream));
        }
        return MVN_OK;
    }
    if (m->method != 0)
        return fail(c, MVN_E_USAGE, "mvn_mc_validate: method must be 0 (fp64 DMMA), 1 or 2 (int8 tensor cores)");
    const int64_t n_pad = (t.n + t.nb - 1) / t.nb * t.nb;
    // chunk: as many 128-sample blocks as fit ~8 GB of Z, at least one
    const int64_t per_blk = mvn::mc_z_doubles(t.n, 128) * (int64_t)sizeof(double);
    int64_t blocks = std::max<int64_t>(1, (int64_t)(8ll << 30) / per_blk);
    int64_t chunk = std::min<int64_t>(total, blocks * 128);
    (void)n_pad;
    mvn_status s;
    if ((s = ensure(c, &c->mcZ, &c->mcZ_cap, (size_t)mvn::mc_z_doubles(t.n, chunk) * sizeof(double))) != MVN_OK) return s;
    if (!d_first && (s = ensure(c, &c->mcF, &c->mcF_cap, (size_t)chunk * sizeof(int32_t))) != MVN_OK) return s;
    for (int64_t s0 = 0; s0 < total; s0 += chunk) {
        const int64_t ns = std::min(chunk, total - s0);
        int *first = d_first ? (int *)d_first + s0 : (int *)c->mcF;
        MVN_CUDA(c, mvn::launch_mc_chunk(t.n, d_L, d_a, m->seed, m->sample_begin + s0, ns, (double *)c->mcZ, first,
                                         (unsigned long long *)d_count, c->nsm, c->stream));
    }
    return MVN_OK;
}

mvn_status mvn_mc_levels(int64_t n, const uint64_t *count, int64_t N_total, const int64_t *k_star, int64_t nconf,
                         double *p_hat) {
    if (n < 1 || !count || N_total < 1 || nconf < 0 || (nconf > 0 && (!k_star || !p_hat))) return MVN_E_USAGE;
    std::vector<uint64_t> tail((size_t)n + 2, 0);
    for (int64_t k = n; k >= 0; --k) tail[(size_t)k] = tail[(size_t)k + 1] + count[k];
    for (int64_t i = 0; i < nconf; ++i) {
        if (k_star[i] < 0 || k_star[i] > n) return MVN_E_USAGE;
        p_hat[i] = (double)tail[(size_t)k_star[i]] / (double)N_total;
    }
    return MVN_OK;
}

mvn_status mvn_posterior(mvn_ctx *c, const mvn_posterior_problem *p, double *mu_post, double *var_post, int64_t *info) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!p || !mu_post || !var_post || !info || p->n < 1 || p->m < 1 || !p->xy || !p->mu || !p->obs || !p->y ||
        !(p->tau > 0) || !(p->sigma2 > 0) || !(p->beta > 0) || !(p->nugget >= 0) || !(p->nu > 0 && p->nu <= 50))
        return fail(c, MVN_E_USAGE, "mvn_posterior: bad arguments");
    const int64_t n = p->n, m = p->m;
    std::vector<char> seen((size_t)n, 0);
    for (int64_t j = 0; j < m; ++j) {
        if (p->obs[j] < 0 || p->obs[j] >= n || seen[(size_t)p->obs[j]] || std::isnan(p->y[j]))
            return fail(c, MVN_E_USAGE, "mvn_posterior: observation indices must be distinct sites, y finite");
        seen[(size_t)p->obs[j]] = 1;
    }
    const int64_t m_pad = (m + mvn::kTile - 1) / mvn::kTile * mvn::kTile;
    const int64_t N = m_pad + n + 1, extra = m_pad + n;
    mvn_tiles ta{N, mvn::kTile};
    // augmented locations: observed sites, decoupled far points (padding), all sites, far point (r row)
    std::vector<double> xy((size_t)(2 * N)), r((size_t)m);
    std::vector<int64_t> rows((size_t)m);
    for (int64_t j = 0; j < m; ++j) {
        xy[2 * j] = p->xy[2 * p->obs[j]];
        xy[2 * j + 1] = p->xy[2 * p->obs[j] + 1];
        r[(size_t)j] = p->y[j] - p->mu[p->obs[j]];
        rows[(size_t)j] = m_pad + p->obs[j];                      // the site row of observation j
    }
    for (int64_t j = m; j < m_pad; ++j) { xy[2 * j] = 1e9 * (double)(j + 1); xy[2 * j + 1] = 1e9; }
    for (int64_t i = 0; i < n; ++i) { xy[2 * (m_pad + i)] = p->xy[2 * i]; xy[2 * (m_pad + i) + 1] = p->xy[2 * i + 1]; }
    xy[2 * extra] = -1e9;
    xy[2 * extra + 1] = -1e9;
    mvn_status s;
    if ((s = ensure(c, &c->post, &c->post_cap, mvn_tiles_bytes(ta))) != MVN_OK) return s;
    if ((s = ensure(c, &c->postv, &c->postv_cap, sizeof(double) * (size_t)(2 * N + 2 * m + 2 * n))) != MVN_OK) return s;
    double *A = (double *)c->post, *d_xy = (double *)c->postv, *d_r = d_xy + 2 * N, *d_dg = d_r + m, *d_row = d_dg + n;
    int64_t *d_rows = (int64_t *)(d_row + n);
    MVN_CUDA(c, cudaMemcpyAsync(d_xy, xy.data(), sizeof(double) * 2 * N, cudaMemcpyHostToDevice, c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(d_r, r.data(), sizeof(double) * m, cudaMemcpyHostToDevice, c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(d_rows, rows.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice, c->stream));
    if ((s = mvn_cov_matern(c, ta, d_xy, p->sigma2, p->beta, p->nu, p->nugget, A)) != MVN_OK) return s;
    MVN_CUDA(c, mvn::launch_add_diag(A, 0, m, p->tau * p->tau, c->stream));           // Sigma_oo + tau^2 I
    MVN_CUDA(c, mvn::launch_add_pairs(A, d_rows, 0, m, p->nugget, c->stream));        // Cov(x_obs_j, y_j) = Sigma_jj
    MVN_CUDA(c, mvn::launch_set_row(A, extra, 0, m, d_r, c->stream));                 // r^T
    const int64_t minus1 = -1;
    MVN_CUDA(c, cudaMemcpyAsync(c->d_info, &minus1, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    MVN_CUDA(c, mvn::launch_potrf(N, A, c->d_info, c->stream, (int)(m_pad / mvn::kTile)));
    MVN_CUDA(c, mvn::launch_get_diag(A, m_pad, n, d_dg, c->stream));
    MVN_CUDA(c, mvn::launch_get_row(A, extra, m_pad, n, d_row, c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(var_post, d_dg, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(mu_post, d_row, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(info, c->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    MVN_CUDA(c, cudaStreamSynchronize(c->stream));
    if (*info >= 0) {
        if (*info >= m) *info = -1;                       // cannot happen: padding is decoupled and positive
        else return fail(c, MVN_E_NUMERIC, "mvn_posterior: observation covariance not positive definite at row " + std::to_string(*info));
    }
    for (int64_t i = 0; i < n; ++i) mu_post[i] = p->mu[i] - mu_post[i];   // the last row holds -(mu_post - mu)
    c->post_n = n;
    c->post_off = m_pad;
    return MVN_OK;
}

mvn_status mvn_posterior_tiles(mvn_ctx *c, mvn_tiles t, const int64_t *order, double *d_tiles) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!tiles_ok(t) || !order || !d_tiles || c->post_n != t.n || !c->post)
        return fail(c, MVN_E_USAGE, "mvn_posterior_tiles: call mvn_posterior first (same n)");
    const int64_t n = t.n;
    std::vector<char> seen((size_t)n, 0);
    for (int64_t i = 0; i < n; ++i) {
        if (order[i] < 0 || order[i] >= n || seen[(size_t)order[i]]) return fail(c, MVN_E_USAGE, "mvn_posterior_tiles: order is not a permutation");
        seen[(size_t)order[i]] = 1;
    }
    mvn_status s;
    if ((s = ensure(c, &c->cta, &c->cta_cap, sizeof(int64_t) * (size_t)n)) != MVN_OK) return s;
    MVN_CUDA(c, cudaMemcpyAsync(c->cta, order, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream));
    MVN_CUDA(c, mvn::launch_permute_sym((const double *)c->post, c->post_off, (const int64_t *)c->cta, n, d_tiles, c->stream));
    MVN_CUDA(c, cudaStreamSynchronize(c->stream));
    return MVN_OK;
}

mvn_status mvn_tlr_compress(mvn_ctx *c, mvn_tiles t, double *d_tiles, double eps, int32_t mode, int32_t *d_ranks) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!tiles_ok(t) || !d_tiles || !d_ranks || !(eps >= 0.0) || (mode != MVN_TLR_ABS && mode != MVN_TLR_REL_FRO) ||
        (mode == MVN_TLR_REL_FRO && !(eps <= 1.0)))
        return fail(c, MVN_E_USAGE, "mvn_tlr_compress: bad arguments (need nb=128, eps >= 0, mode 0 or 1, eps <= 1 for mode 1)");
    MVN_CUDA(c, mvn::launch_tlr_compress(t.n, d_tiles, eps, mode, d_ranks, c->stream));
    return MVN_OK;
}

size_t mvn_tlr_slots_bytes(mvn_tiles t, int32_t kmax) {
    if (!tiles_ok(t) || kmax < 1 || kmax > (int32_t)mvn::kTile) return 0;
    return sizeof(double) * mvn::tlr_slot_doubles(t.n, kmax);
}

mvn_status mvn_tlr_potrf(mvn_ctx *c, mvn_tiles t, double *d_tiles, double eps, int32_t mode, int32_t kmax, double *d_U,
                         double *d_V, int32_t *d_ranks, int32_t *d_ranks_sigma, int64_t *info) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!tiles_ok(t) || !d_tiles || !info || !(eps >= 0.0) || (mode != MVN_TLR_ABS && mode != MVN_TLR_REL_FRO) ||
        (mode == MVN_TLR_REL_FRO && !(eps <= 1.0)) || kmax < 1 || kmax > (int32_t)mvn::kTile)
        return fail(c, MVN_E_USAGE, "mvn_tlr_potrf: bad arguments (need nb=128, eps >= 0, mode 0 or 1, eps <= 1 for mode 1, 1 <= kmax <= 128)");
    const int64_t nt = (t.n + t.nb - 1) / t.nb;
    if (nt > 1 && (!d_U || !d_V || !d_ranks)) return fail(c, MVN_E_USAGE, "mvn_tlr_potrf: factor slots and ranks required");
    // M / Z chunks: at most 2,048 tiles each (256 MB), at least one tile column's worth
    const int64_t need = std::max<int64_t>(1, (nt / 2) * ((nt + 1) / 2));
    const int64_t chunk = std::max<int64_t>(std::min<int64_t>(need, 2048), nt);
    const size_t wbytes = sizeof(double) * mvn::tlr_work_doubles(t.n, chunk);
    mvn_status s;
    const int64_t noff = nt * (nt - 1) / 2;
    if ((s = ensure(c, &c->tlrW, &c->tlrW_cap, wbytes + 256 + sizeof(int32_t) * (size_t)noff)) != MVN_OK) return s;
    int *overflow = (int *)((char *)c->tlrW + wbytes);
    if (!d_ranks_sigma) d_ranks_sigma = (int32_t *)((char *)c->tlrW + wbytes + 256);   // Sigma's ranks, not returned
    const int64_t minus1 = -1;
    MVN_CUDA(c, cudaMemsetAsync(overflow, 0, sizeof(int), c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(c->d_info, &minus1, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    MVN_CUDA(c, mvn::launch_tlr_potrf(t.n, d_tiles, eps, mode, kmax, d_U, d_V, d_ranks, d_ranks_sigma, (double *)c->tlrW,
                                      chunk, overflow, c->d_info, c->stream));
    int ovf = 0;
    MVN_CUDA(c, cudaMemcpyAsync(info, c->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(&ovf, overflow, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    MVN_CUDA(c, cudaStreamSynchronize(c->stream));
    if (*info >= t.n) *info = -1;
    // a rank above kmax first: the truncation to kmax is not at accuracy eps and may itself be what
    // made a later pivot non-positive
    if (ovf > 0)
        return fail(c, MVN_E_NOMEM, "mvn_tlr_potrf: a tile needs rank " + std::to_string(ovf) + " > kmax = " + std::to_string(kmax));
    if (*info >= 0)
        return fail(c, MVN_E_NUMERIC, "mvn_tlr_potrf: matrix not positive definite at row " + std::to_string(*info));
    return MVN_OK;
}

mvn_status mvn_crd(mvn_ctx *c, const mvn_crd_problem *p, mvn_crd_result *out) {
    DevGuard dev_guard(c);
    if (!c) return MVN_E_USAGE;
    if (!p || !out || p->n < 1 || !p->xy || !p->mu || !out->order || !out->logP || (p->nconf > 0 && !out->k_star))
        return fail(c, MVN_E_USAGE, "mvn_crd: bad arguments");
    const int64_t n = p->n;
    mvn_tiles t{n, mvn::kTile};
    cudaEvent_t ev[7];
    for (auto &e : ev) MVN_CUDA(c, cudaEventCreate(&e));
    struct EvGuard { cudaEvent_t *e; ~EvGuard() { for (int i = 0; i < 7; ++i) cudaEventDestroy(e[i]); } } guard{ev};

    // a1 (host): marginals, order, limits, sorted locations
    std::vector<double> var((size_t)n, p->sigma2 + p->nugget), a((size_t)n), xys((size_t)(2 * n));
    mvn_status s = mvn_marginal_order(n, p->mu, var.data(), p->u, out->order, a.data(), nullptr);
    if (s != MVN_OK) return fail(c, s, "mvn_crd: invalid mu / sigma2 / u");
    for (int64_t k = 0; k < n; ++k) {
        xys[2 * k] = p->xy[2 * out->order[k]];
        xys[2 * k + 1] = p->xy[2 * out->order[k] + 1];
    }
    if ((s = ensure(c, &c->crd_L, &c->crd_L_cap, mvn_tiles_bytes(t))) != MVN_OK) return s;
    if ((s = ensure(c, &c->crd_vec, &c->crd_vec_cap, sizeof(double) * (size_t)n * 6)) != MVN_OK) return s;
    double *dL = (double *)c->crd_L;
    double *dxy = (double *)c->crd_vec, *da = dxy + 2 * n, *dM = da + n, *dS = dM + n, *dlp = dS + n;

    MVN_CUDA(c, cudaEventRecord(ev[0], c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(dxy, xys.data(), sizeof(double) * 2 * n, cudaMemcpyHostToDevice, c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(da, a.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    MVN_CUDA(c, cudaEventRecord(ev[1], c->stream));
    if ((s = mvn_cov_matern(c, t, dxy, p->sigma2, p->beta, p->nu, p->nugget, dL)) != MVN_OK) return s;
    MVN_CUDA(c, cudaEventRecord(ev[2], c->stream));
    int64_t info = -1;
    if (p->method & ~(MVN_CRD_SOV_INT8 | MVN_CRD_POTRF_INT8 | MVN_CRD_TLR)) return fail(c, MVN_E_USAGE, "mvn_crd: unknown method bits");
    if (p->method & MVN_CRD_TLR) {
        if ((p->method & MVN_CRD_POTRF_INT8) || !(p->tlr_eps >= 0.0))
            return fail(c, MVN_E_USAGE, "mvn_crd: MVN_CRD_TLR needs tlr_eps >= 0 and excludes MVN_CRD_POTRF_INT8");
        const size_t slot = mvn_tlr_slots_bytes(t, (int32_t)mvn::kTile);
        const int64_t nt = (n + mvn::kTile - 1) / mvn::kTile, noff = nt * (nt - 1) / 2;
        if ((s = ensure(c, &c->tlrS, &c->tlrS_cap, 2 * slot + sizeof(int32_t) * (size_t)std::max<int64_t>(noff, 1) + 256)) != MVN_OK)
            return s;
        double *U = (double *)c->tlrS, *V = (double *)((char *)c->tlrS + slot);
        int32_t *rk = (int32_t *)((char *)c->tlrS + 2 * slot);
        s = mvn_tlr_potrf(c, t, dL, p->tlr_eps, MVN_TLR_ABS, (int32_t)mvn::kTile, U, V, rk, nullptr, &info);
    } else {
        s = mvn_potrf_ex(c, t, dL, &info, (p->method & MVN_CRD_POTRF_INT8) ? MVN_POTRF_INT8 : MVN_POTRF_FP64);
    }
    out->info = info;
    if (s != MVN_OK) return s;
    MVN_CUDA(c, cudaEventRecord(ev[3], c->stream));
    mvn_qmc q{p->N, p->R, p->seed, 0, p->N * (int64_t)p->R};
    if ((s = mvn_sov_prefix_ex(c, t, dL, da, nullptr, &q, (p->method & MVN_CRD_SOV_INT8) ? MVN_SOV_INT8 : MVN_SOV_FP64,
                               dM, dS)) != MVN_OK)
        return s;
    MVN_CUDA(c, cudaEventRecord(ev[4], c->stream));
    if ((s = mvn_prefix_finalize(c, n, q.N * (int64_t)q.R, dM, dS, dlp)) != MVN_OK) return s;
    MVN_CUDA(c, cudaEventRecord(ev[5], c->stream));
    MVN_CUDA(c, cudaMemcpyAsync(out->logP, dlp, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    MVN_CUDA(c, cudaEventRecord(ev[6], c->stream));
    MVN_CUDA(c, cudaStreamSynchronize(c->stream));
    for (int i = 0; i < 6; ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
        out->ms_stage[i] = ms;
    }
    if (p->nconf > 0)
        if ((s = mvn_confidence_region(n, out->logP, p->conf, p->nconf, out->k_star, out->near_tie)) != MVN_OK)
            return fail(c, s, "mvn_crd: invalid confidence levels");
    return MVN_OK;
}

}  // extern "C"
