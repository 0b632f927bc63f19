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
};

static TargetWs target_carve(Carver &c, int M) {
    TargetWs t;
    t.pos = c.take<float4>(M);
    t.cov_a = c.take<float4>(M);
    t.cov_b = c.take<float4>(M);
    t.d_M = c.take<int32_t>(4);
    t.smid_sum = c.take<double>(4);
    t.grid = c.take<char>(grid_bytes(M, 1, true));
    return t;
}

size_t target_ws_bytes(int M) {
    Carver c(nullptr);
    target_carve(c, M);
    return c.bytes();
}

static void fill_target(const GridView &g, int M, gsicp_target *out) {
    out->pos = reinterpret_cast<const float *>(g.spos);
    out->cov_a = reinterpret_cast<const float *>(g.scov_a);
    out->cov_b = reinterpret_cast<const float *>(g.scov_b);
    out->table = g.table;
    out->bbox = g.bbox;
    out->table_mask = g.mask;
    out->cell = g.h0;
    out->M = M;
}

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
        cell = (float)(3.0 * sum / (double)M);
        if (!(cell > 0.f)) cell = 0.01f;
    }
    GridView g = grid_carve(t.grid, M, 1, true, cell);
    cudaError_t e = grid_build(g, t.pos, t.cov_a, t.cov_b, t.d_M, M, s);
    if (e != cudaSuccess) return e;
    fill_target(g, M, out);
    return cudaSuccess;
}

cudaError_t build_target_cloud_launch(const gsicp_cloud &cl, int M, float cell, gsicp_target *out, void *ws,
                                      cudaStream_t s) {
    Carver c(ws);
    TargetWs t = target_carve(c, M);
    GridView g = grid_carve(t.grid, M, 1, true, cell);
    cudaError_t e = grid_build(g, reinterpret_cast<const float4 *>(cl.pos), reinterpret_cast<const float4 *>(cl.cov_a),
                               reinterpret_cast<const float4 *>(cl.cov_b), cl.d_n, M, s);
    if (e != cudaSuccess) return e;
    fill_target(g, M, out);
    return cudaSuccess;
}

}  // namespace gsicp
