#include <stdlib.h>
// A5  Map Gaussians -> G-ICP target Gaussians (the map already holds
// Gaussians, so G-ICP "does not need to compute the covariances of the map"
// C = R Lambda^2 R^T).  Per Gaussian: normalised wxyz quaternion -> R (R22), scales (exp if
// log) -> variances s_i^2 sorted descending with ties by axis index (R5), regularised in
// closed form from (R, s) — no eigensolve — then the means are hashed with their covariances
// (single-level grid, cell-ordered copies) for the correspondence search.
#include "grid.cuh"
#include "host_common.cuh"

namespace gsicp {

namespace {

struct MapArgs {
    const float *means, *quats, *scales;
    int scales_are_log, M, mode;
    double eps;
    float4 *pos, *cov_a, *cov_b;
    double *smid_sum;  // nullable: sum of middle scales (auto cell size)
};

__global__ void k_map_to_target(MapArgs a) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double smid = 0.0;
    if (i < a.M) {
        double w = a.quats[4 * (size_t)i], x = a.quats[4 * (size_t)i + 1], y = a.quats[4 * (size_t)i + 2],
               z = a.quats[4 * (size_t)i + 3];
        const double inq = rsqrt(w * w + x * x + y * y + z * z);
        w *= inq; x *= inq; y *= inq; z *= inq;
        const double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                                {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                                {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
        double s[3];
        for (int k = 0; k < 3; ++k) {
            const double v = a.scales[3 * (size_t)i + k];
            s[k] = a.scales_are_log ? exp(v) : v;
        }
        int o[3] = {0, 1, 2};  // stable descending order of the scales
        if (s[o[1]] > s[o[0]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
        if (s[o[2]] > s[o[1]]) { int t = o[1]; o[1] = o[2]; o[2] = t; }
        if (s[o[1]] > s[o[0]]) { int t = o[0]; o[0] = o[1]; o[1] = t; }
        Eig3 e;
        for (int j = 0; j < 3; ++j) {
            e.lam[j] = s[o[j]] * s[o[j]];
            for (int r = 0; r < 3; ++r) e.v[j][r] = R[r][o[j]];
        }
        double C[6] = {0, 0, 0, 0, 0, 0};
        for (int j = 0; j < 3; ++j) {
            const double *v = e.v[j];
            const double l = e.lam[j];
            C[0] += l * v[0] * v[0]; C[1] += l * v[0] * v[1]; C[2] += l * v[0] * v[2];
            C[3] += l * v[1] * v[1]; C[4] += l * v[1] * v[2]; C[5] += l * v[2] * v[2];
        }
        double out[6];
        const uint32_t flags = regularize(C, e, a.mode, a.eps, out);
        a.pos[i] = make_float4(a.means[3 * (size_t)i], a.means[3 * (size_t)i + 1], a.means[3 * (size_t)i + 2],
                               __int_as_float(i));
        store_cov(a.cov_a, a.cov_b, i, out, e.lam[1], flags);
        smid = s[o[1]];
    }
    if (a.smid_sum) {
        for (int off = 16; off > 0; off >>= 1) smid += __shfl_xor_sync(0xffffffffu, smid, off);
        if ((threadIdx.x & 31) == 0) atomicAdd(a.smid_sum, smid);
    }
}

__global__ void k_set_count(int32_t *d, int v) { *d = v; }

}  // namespace

struct TargetWs {
    float4 *pos, *cov_a, *cov_b;
    int32_t *d_M;
    double *smid_sum;
    void *grid;
    uint2 *dense;
    int32_t *dense_hdr;
    long long dense_budget;
    int32_t *knn_idx;  // [M][kGraphK] input indices (graph build scratch)
    int32_t *inv;      // [M] cell-ordered slot of each input index
    int32_t *nbr;      // [M][kGraphK] neighbour slots of each slot (self first)
    float *nbr_key;    // [M] canonical key of the kGraphK-th neighbour (INFINITY if fewer points)
};

// dense (start, count) cell array budget: 8 cells per Gaussian (>= 1M cells), 8 bytes each
static long long dense_budget(int M) { return M * 8LL > (1LL << 20) ? M * 8LL : (1LL << 20); }

static TargetWs target_carve(Carver &c, int M) {
    TargetWs t;
    t.pos = c.take<float4>(M);
    t.cov_a = c.take<float4>(M);
    t.cov_b = c.take<float4>(M);
    t.d_M = c.take<int32_t>(4);
    t.smid_sum = c.take<double>(4);
    t.grid = c.take<char>(grid_bytes(M, 1, true));
    t.dense_budget = dense_budget(M);
    t.dense = c.take<uint2>((size_t)t.dense_budget);
    t.dense_hdr = c.take<int32_t>(8);
    t.knn_idx = c.take<int32_t>((size_t)M * kGraphK);
    t.inv = c.take<int32_t>(M);
    t.nbr = c.take<int32_t>((size_t)M * kGraphK);
    t.nbr_key = c.take<float>(M);
    return t;
}

size_t target_ws_bytes(int M) {
    Carver c(nullptr);
    target_carve(c, M);
    return c.bytes();
}

namespace {

// header {in_use, lo xyz, dims xyz}: the bbox's cells (same cell_coord as the hash) if they fit
__global__ void k_dense_setup(const int32_t *bbox, float inv_h, long long budget, int32_t *hdr) {
    int lo[3], dim[3];
    long long total = 1;
    for (int k = 0; k < 3; ++k) {
        lo[k] = cell_coord(ordered_to_float(bbox[k]), inv_h);
        const int hi = cell_coord(ordered_to_float(bbox[3 + k]), inv_h);
        dim[k] = hi - lo[k] + 1;
        total *= (long long)(dim[k] > 0 ? dim[k] : 0);
    }
    hdr[0] = (total > 0 && total <= budget) ? 1 : 0;
    for (int k = 0; k < 3; ++k) {
        hdr[1 + k] = lo[k];
        hdr[4 + k] = dim[k];
    }
}

__global__ void k_dense_clear(uint2 *dense, long long budget, const int32_t *hdr) {
    if (!hdr[0]) return;
    const long long total = (long long)hdr[4] * hdr[5] * hdr[6];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
        dense[i] = make_uint2(0u, 0u);
}

__global__ void k_dense_fill(const CellEntry *table, uint32_t slots, uint2 *dense, const int32_t *hdr) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (!hdr[0] || s >= slots) return;
    const CellEntry e = table[s];
    if (e.key == kEmptyKey) return;
    const int x = (int)((e.key >> 40) & 0xFFFFFull) - kCoordOff;
    const int y = (int)((e.key >> 20) & 0xFFFFFull) - kCoordOff;
    const int z = (int)(e.key & 0xFFFFFull) - kCoordOff;
    const long long ix = x - hdr[1], iy = y - hdr[2], iz = z - hdr[3];
    dense[(iz * hdr[5] + iy) * hdr[4] + ix] = make_uint2(e.start, e.count);
}

__global__ void k_graph_inv(const float4 *spos, const int32_t *d_n, int32_t *inv) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < *d_n) inv[__float_as_int(spos[s].w)] = s;
}

__global__ void k_graph_finalize(const float4 *spos, const int32_t *d_n, const int32_t *knn_idx, const int32_t *inv,
                                 int32_t *nbr, float *nbr_key) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= *d_n) return;
    const float4 p = spos[s];
    const int orig = __float_as_int(p.w);
    // the list is the exact kGraphK-NN SET (any order): its radius is the largest key32 in it
    float kmax = 0.f;
    bool short_list = false;
    for (int j = 0; j < kGraphK; ++j) {
        const int o = knn_idx[(size_t)orig * kGraphK + j];
        const int sl = o >= 0 ? inv[o] : -1;
        nbr[(size_t)s * kGraphK + j] = sl;
        if (sl >= 0) {
            const float4 q = spos[sl];
            kmax = fmaxf(kmax, canon_key(p.x, p.y, p.z, q.x, q.y, q.z));
        } else {
            short_list = true;
        }
    }
    nbr_key[s] = short_list ? INFINITY : kmax;  // INFINITY: the list holds the whole cloud
}

}  // namespace

cudaError_t knn_graph_launch(const GridView &g, const float4 *pos, const int32_t *d_n, int cap, int32_t *knn_idx,
                             cudaStream_t s);

// Target kNN graph: for every target point (slot) its kGraphK nearest targets (slots, exact,
// self included) and the key of the farthest.  The align kernel uses it as a certificate: if
// 4 key(q, m_j) < key_K(j) (with rounding slack), every target at least as close to q as m_j
// lies in j's list, so the exact 1-NN of q is the best of that list.
static cudaError_t build_graph(const GridView &g, const TargetWs &t, const float4 *pos, const int32_t *d_n, int M,
                               cudaStream_t s) {
    cudaError_t e = knn_graph_launch(g, pos, d_n, M, t.knn_idx, s);
    if (e != cudaSuccess) return e;
    k_graph_inv<<<blocks_for(M, 256), 256, 0, s>>>(g.spos, d_n, t.inv);
    GSICP_LAUNCH_CHECK("k_graph_inv");
    k_graph_finalize<<<blocks_for(M, 256), 256, 0, s>>>(g.spos, d_n, t.knn_idx, t.inv, t.nbr, t.nbr_key);
    GSICP_LAUNCH_CHECK("k_graph_finalize");
    note_launch(2);
    return cudaSuccess;
}

static cudaError_t build_dense(const GridView &g, const TargetWs &t, cudaStream_t s) {
    k_dense_setup<<<1, 1, 0, s>>>(g.bbox, g.inv_h0, t.dense_budget, t.dense_hdr);
    GSICP_LAUNCH_CHECK("k_dense_setup");
    k_dense_clear<<<num_sms() * 8, 256, 0, s>>>(t.dense, t.dense_budget, t.dense_hdr);
    GSICP_LAUNCH_CHECK("k_dense_clear");
    k_dense_fill<<<blocks_for((long long)g.mask + 1, 256), 256, 0, s>>>(g.table, g.mask + 1, t.dense, t.dense_hdr);
    GSICP_LAUNCH_CHECK("k_dense_fill");
    note_launch(3);
    return cudaSuccess;
}

static void fill_target(const GridView &g, const TargetWs &t, int M, gsicp_target *out) {
    out->pos = reinterpret_cast<const float *>(g.spos);
    out->cov_a = reinterpret_cast<const float *>(g.scov_a);
    out->cov_b = reinterpret_cast<const float *>(g.scov_b);
    out->table = g.table;
    out->bbox = g.bbox;
    out->dense = t.dense;
    out->dense_hdr = t.dense_hdr;
    out->nbr = t.nbr;
    out->nbr_key = t.nbr_key;
    out->table_mask = g.mask;
    out->cell = g.h0;
    out->M = M;
}

// auto cell = kAutoCellMult x mean middle scale (a cost knob only; results are exact at any cell size)
constexpr double kAutoCellMult = 3.0;

cudaError_t build_target_launch(const float *means, const float *quats, const float *scales, int scales_are_log,
                                int M, int mode, float eps, float cell, gsicp_target *out, void *ws,
                                cudaStream_t s) {
    Carver c(ws);
    TargetWs t = target_carve(c, M);
    MapArgs a;
    a.means = means; a.quats = quats; a.scales = scales;
    a.scales_are_log = scales_are_log; a.M = M; a.mode = mode; a.eps = (double)eps;
    a.pos = t.pos; a.cov_a = t.cov_a; a.cov_b = t.cov_b;
    a.smid_sum = nullptr;
    if (!(cell > 0.f)) {
        a.smid_sum = t.smid_sum;
        cudaMemsetAsync(t.smid_sum, 0, sizeof(double), s);
    }
    k_map_to_target<<<blocks_for(M, 256), 256, 0, s>>>(a);
    GSICP_LAUNCH_CHECK("k_map_to_target");
    k_set_count<<<1, 1, 0, s>>>(t.d_M, M);
    GSICP_LAUNCH_CHECK("k_set_count");
    note_launch(2);
    if (!(cell > 0.f)) {
        double sum = 0.0;
        cudaError_t e = cudaMemcpyAsync(&sum, t.smid_sum, sizeof(double), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            set_error("build_target auto cell: %s", cudaGetErrorString(e));
            return e;
        }
        cell = (float)(kAutoCellMult * sum / (double)M);
        if (!(cell > 0.f)) cell = 0.01f;
    }
    GridView g = grid_carve(t.grid, M, 1, true, cell);
    cudaError_t e = grid_build(g, t.pos, t.cov_a, t.cov_b, t.d_M, M, s);
    if (e == cudaSuccess) e = build_dense(g, t, s);
    if (e == cudaSuccess) e = build_graph(g, t, t.pos, t.d_M, M, s);
    if (e != cudaSuccess) return e;
    fill_target(g, t, M, out);
    return cudaSuccess;
}

cudaError_t build_target_cloud_launch(const gsicp_cloud &cl, int M, float cell, gsicp_target *out, void *ws,
                                      cudaStream_t s) {
    Carver c(ws);
    TargetWs t = target_carve(c, M);
    GridView g = grid_carve(t.grid, M, 1, true, cell);
    cudaError_t e = grid_build(g, reinterpret_cast<const float4 *>(cl.pos), reinterpret_cast<const float4 *>(cl.cov_a),
                               reinterpret_cast<const float4 *>(cl.cov_b), cl.d_n, M, s);
    if (e == cudaSuccess) e = build_dense(g, t, s);
    if (e == cudaSuccess) e = build_graph(g, t, reinterpret_cast<const float4 *>(cl.pos), cl.d_n, M, s);
    if (e != cudaSuccess) return e;
    fill_target(g, t, M, out);
    return cudaSuccess;
}

}  // namespace gsicp
