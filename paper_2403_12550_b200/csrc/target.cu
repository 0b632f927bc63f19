#include <stdlib.h>
// A5  Map Gaussians -> G-ICP target Gaussians (the map already holds
// Gaussians, so G-ICP "does not need to compute the covariances of the map"
// C = R Lambda^2 R^T).  Per Gaussian: normalised wxyz quaternion -> R (R22), scales (exp if
// log) -> variances s_i^2 sorted descending with ties by axis index (R5), regularised in
// closed form from (R, s) — no eigensolve — then the means are hashed with their covariances
// (single-level grid, cell-ordered copies) for the correspondence search.
#include "grid.cuh"
#include "host_common.cuh"
#include "search.cuh"

namespace gsicp {

namespace {

struct MapArgs {
    const float *means, *quats, *scales;
    int scales_are_log, M, mode;
    double eps;
    float4 *pos, *cov_a, *cov_b;
    double *smid_sum;  // nullable: sum of middle scales (auto cell size)
    // nullable (N1 map insertion): only rows [*d_base, *d_base + *d_cnt) (M is then the capacity)
    const int32_t *d_base, *d_cnt;
};

__global__ void k_map_to_target(MapArgs a) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    double smid = 0.0;
    bool in = i < a.M;
    if (a.d_base) {
        in = i < *a.d_cnt;
        i += *a.d_base;
    }
    if (in) {
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
                                 int32_t *nbr, float *nbr_key, float *key_in) {
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
    if (key_in) key_in[orig] = nbr_key[s];      // the same, by input row (incremental maintenance)
}

}  // namespace

cudaError_t knn_graph_launch(const GridView &g, const float4 *pos, const int32_t *d_n, int cap, int32_t *knn_idx,
                             cudaStream_t s);

// Target kNN graph: for every target point (slot) its kGraphK nearest targets (slots, exact,
// self included) and the key of the farthest.  The align kernel uses it as a certificate: if
// 4 key(q, m_j) < key_K(j) (with rounding slack), every target at least as close to q as m_j
// lies in j's list, so the exact 1-NN of q is the best of that list.
static cudaError_t graph_finalize(const GridView &g, const TargetWs &t, const int32_t *d_n, int M, float *key_in,
                                  cudaStream_t s) {
    k_graph_inv<<<blocks_for(M, 256), 256, 0, s>>>(g.spos, d_n, t.inv);
    GSICP_LAUNCH_CHECK("k_graph_inv");
    k_graph_finalize<<<blocks_for(M, 256), 256, 0, s>>>(g.spos, d_n, t.knn_idx, t.inv, t.nbr, t.nbr_key, key_in);
    GSICP_LAUNCH_CHECK("k_graph_finalize");
    note_launch(2);
    return cudaSuccess;
}

static cudaError_t build_graph(const GridView &g, const TargetWs &t, const float4 *pos, const int32_t *d_n, int M,
                               cudaStream_t s, float *key_in = nullptr) {
    cudaError_t e = knn_graph_launch(g, pos, d_n, M, t.knn_idx, s);
    if (e != cudaSuccess) return e;
    return graph_finalize(g, t, d_n, M, key_in, s);
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
    a.d_base = a.d_cnt = nullptr;
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
    if (!(cell > 0.f)) {  // automatic: 3 x the estimated spacing (blocking), as the map auto cell
        float sp = 0.f;
        cudaError_t e = estimate_spacing(reinterpret_cast<const float4 *>(cl.pos), cl.d_n, M, t.grid, &sp, s);
        if (e != cudaSuccess) return e;
        cell = (float)(kAutoCellMult * sp);
    }
    GridView g = grid_carve(t.grid, M, 1, true, cell);
    cudaError_t e = grid_build(g, reinterpret_cast<const float4 *>(cl.pos), reinterpret_cast<const float4 *>(cl.cov_a),
                               reinterpret_cast<const float4 *>(cl.cov_b), cl.d_n, M, s);
    if (e == cudaSuccess) e = build_dense(g, t, s);
    if (e == cudaSuccess) e = build_graph(g, t, reinterpret_cast<const float4 *>(cl.pos), cl.d_n, M, s);
    if (e != cudaSuccess) return e;
    fill_target(g, t, M, out);
    return cudaSuccess;
}


// ---------------------------------------------------------------------------------------------
// N1  Device-resident growing map with incremental target maintenance (P:209-214 keyframes,
// P:237 only non-overlapping Gaussians, P:250-255 scale aligning).  The map owns its Gaussians
// (rows [0, *d_M) of means / quats / scales, linear scales) and a target built over them for a
// fixed capacity.  An insertion appends a keyframe's exported Gaussians and maintains the target
// without rebuilding the kNN graph: only the rows whose exact 16-NN set can change are searched
// again — the new rows, and every old row p with a new point x inside its list's ball
// (key32(p, x) <= band_hi(its largest list key): a new point can enter p's list only then) —
// then the hash (cell order) and the slot lists are rebuilt by the O(M) streaming kernels.
// Every count lives on the device, so an insertion can sit inside a CUDA graph (behind a
// conditional node on a device-side keyframe flag).
size_t export_ws_bytes(int cap);
cudaError_t export_launch(const float4 *pos, const float4 *cov_a, const float4 *cov_b, const int32_t *d_n, int cap,
                          const double *d_T, double p, double c, const int32_t *corr, float *means, float *quats,
                          float *scales, int32_t *d_m, void *ws, cudaStream_t s, const int32_t *d_base);
cudaError_t knn_graph_queue_launch(const GridView &g, const float4 *pos, const int32_t *d_n, int cap,
                                   const uint32_t *queue, const uint32_t *queue_n, int32_t *knn_idx, cudaStream_t s);

struct MapWs {
    float *means, *quats, *scales;  // [cap + max_insert][3], [..][4], [..][3] (an export never writes out of bounds)
    int32_t *ctr;                   // [0] M, [1] m (last insert), [2] M + m, [3] queue length (u32),
                                    // [4] Gaussians dropped because the map was full
    float *key_in;                  // [cap] largest key32 of each row's 16-NN list
    uint32_t *queue;                // [cap] rows whose lists are recomputed
    float4 *dpos;                   // [max_insert] the inserted rows' positions (delta grid input)
    void *dgrid;                    // grid over the inserted rows
    int32_t *export_scratch;
    TargetWs t;
};

static MapWs map_carve(Carver &c, int cap, int max_insert) {
    MapWs w;
    w.means = c.take<float>((size_t)(cap + max_insert) * 3);
    w.quats = c.take<float>((size_t)(cap + max_insert) * 4);
    w.scales = c.take<float>((size_t)(cap + max_insert) * 3);
    w.ctr = c.take<int32_t>(8);
    w.key_in = c.take<float>(cap);
    w.queue = c.take<uint32_t>(cap);
    w.dpos = c.take<float4>(max_insert);
    w.dgrid = c.take<char>(grid_bytes(max_insert, 1, false));
    w.export_scratch = c.take<int32_t>(export_ws_bytes(max_insert) / 4 + 64);
    w.t = target_carve(c, cap);
    return w;
}

size_t map_ws_bytes(int cap, int max_insert) {
    Carver c(nullptr);
    map_carve(c, cap, max_insert);
    return c.bytes();
}

namespace {

// initial rows: copy (log scales -> linear), counters
__global__ void k_map_init_rows(const float *means, const float *quats, const float *scales, int scales_are_log,
                                int M0, MapWs w) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < M0) {
        for (int k = 0; k < 3; ++k) {
            w.means[3 * (size_t)i + k] = means[3 * (size_t)i + k];
            const float sc = scales[3 * (size_t)i + k];
            w.scales[3 * (size_t)i + k] = scales_are_log ? (float)exp((double)sc) : sc;
        }
        for (int k = 0; k < 4; ++k) w.quats[4 * (size_t)i + k] = quats[4 * (size_t)i + k];
    }
    if (i == 0) {
        w.ctr[0] = M0;
        w.ctr[1] = 0;
        w.ctr[2] = M0;
        w.ctr[3] = 0;
        w.ctr[4] = 0;
    }
}

// after the export: clamp m to the capacity left (the rows beyond are dropped and counted), M + m,
// queue length 0
__global__ void k_map_clamp(MapWs w, int cap) {
    const int M = w.ctr[0], m = w.ctr[1];
    const int keep = max(min(m, cap - M), 0);
    w.ctr[1] = keep;
    w.ctr[2] = M + keep;
    w.ctr[3] = 0;
    w.ctr[4] += m - keep;
}
// the inserted rows' positions into the delta buffer (the delta grid's input)
__global__ void k_map_stage(MapWs w) {
    const int M = w.ctr[0], m = w.ctr[1];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) w.dpos[i] = w.t.pos[M + i];
}

// rows whose 16-NN list can change: the new rows, and every old row p with a new point inside
// band_hi(key_in[p]) (ball search over the delta grid; rows whose ball misses the delta bbox are
// rejected without a lookup)
__global__ void k_map_mark(MapWs w, GridView dg, int cap) {
    const int M = w.ctr[0], m = w.ctr[1];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (m <= 0) return;
    if (i >= M + m) return;
    bool mark = i >= M;
    if (!mark) {
        const float4 p = w.t.pos[i];
        const float bound = band_hi(w.key_in[i]);
        // squared distance from p to the delta bbox (binary32, a lower bound with margin)
        float gap2 = 0.f;
        const float pc[3] = {p.x, p.y, p.z};
        for (int a = 0; a < 3; ++a) {
            const float lo = ordered_to_float(dg.bbox[a]), hi = ordered_to_float(dg.bbox[3 + a]);
            const float d = fmaxf(fmaxf(lo - pc[a], pc[a] - hi), 0.f) * (1.f - 1e-5f);
            gap2 += d * d;
        }
        if (gap2 <= bound && bound > 16.f * dg.h0 * dg.h0) {
            mark = true;  // a wide list ball (an isolated point): recompute instead of searching it
        } else if (gap2 <= bound) {
            const QueryCell qc(p.x, p.y, p.z, dg.h0, dg.inv_h0);
            int blo[3], bhi[3];
            grid_cell_bbox(dg, 0, blo, bhi);
            CellIndex idx;
            idx.table = dg.table;
            idx.mask = dg.mask;
            idx.level = 0;
            idx.dense = nullptr;
            idx.use_dense = false;
            bool hit = false;
            ball_search(
                qc, idx, blo, bhi, [](int, int, int) { return false; },
                [&](uint2 se) {
                    for (uint32_t j = se.x; j < se.x + se.y && !hit; ++j) {
                        const float4 x = __ldg(dg.spos + j);
                        hit = canon_key(p.x, p.y, p.z, x.x, x.y, x.z) <= bound;
                    }
                },
                [&]() { return hit ? -1.f : bound; });
            mark = hit;
        }
    }
    if (mark) w.queue[atomicAdd(reinterpret_cast<uint32_t *>(w.ctr + 3), 1u)] = (uint32_t)i;
}

__global__ void k_map_commit(int32_t *ctr) { ctr[0] = ctr[2]; }

// conditional-node switch: run the insertion body only for a keyframe
__global__ void k_map_cond(const int32_t *flag, cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, *flag ? 1u : 0u); }

// P:209-214 keyframe decision on the device (R29): fitness (the correspondence proportion of the
// frame's final linearisation) below min_fitness, or max_gap frames since the last keyframe.
// state[0] frames since the last keyframe, state[1] the decision for this frame.
__global__ void k_keyframe(const gsicp_align_stats *st, int32_t *state, float min_fitness, int max_gap) {
    const int since = state[0] + 1;
    const bool kf = st->status != GSICP_ERR_TRACKING_LOST && st->status != GSICP_ERR_DEGENERATE_FRAME &&
                    (st->fitness < (double)min_fitness || since >= max_gap);
    state[1] = kf ? 1 : 0;
    state[0] = kf ? 0 : since;
}

}  // namespace

static GridView map_grid(const MapWs &w, int cap, float cell) { return grid_carve(w.t.grid, cap, 1, true, cell); }

static void fill_map(const MapWs &w, int cap, int max_insert, float cell, int mode, float eps, gsicp_map *out) {
    fill_target(map_grid(w, cap, cell), w.t, cap, &out->target);
    out->means = w.means;
    out->quats = w.quats;
    out->scales = w.scales;
    out->d_M = w.ctr;
    out->capacity = cap;
    out->max_insert = max_insert;
    out->cell = cell;
    out->mode = mode;
    out->eps_var = eps;
    out->ws = w.means;
}

cudaError_t map_init_launch(const float *means, const float *quats, const float *scales, int scales_are_log, int M0,
                            int cap, int max_insert, int mode, float eps, float cell, gsicp_map *out, void *ws,
                            cudaStream_t s) {
    Carver c(ws);
    MapWs w = map_carve(c, cap, max_insert);
    k_map_init_rows<<<blocks_for(M0 > 0 ? M0 : 1, 256), 256, 0, s>>>(means, quats, scales, scales_are_log, M0, w);
    GSICP_LAUNCH_CHECK("k_map_init_rows");
    MapArgs a{};
    a.means = w.means; a.quats = w.quats; a.scales = w.scales;
    a.scales_are_log = 0; a.M = M0; a.mode = mode; a.eps = (double)eps;
    a.pos = w.t.pos; a.cov_a = w.t.cov_a; a.cov_b = w.t.cov_b;
    a.smid_sum = nullptr;
    a.d_base = a.d_cnt = nullptr;
    if (!(cell > 0.f)) {
        a.smid_sum = w.t.smid_sum;
        cudaMemsetAsync(w.t.smid_sum, 0, sizeof(double), s);
    }
    k_map_to_target<<<blocks_for(M0 > 0 ? M0 : 1, 256), 256, 0, s>>>(a);
    GSICP_LAUNCH_CHECK("k_map_to_target");
    note_launch(2);
    if (!(cell > 0.f)) {
        double sum = 0.0;
        cudaError_t e = cudaMemcpyAsync(&sum, w.t.smid_sum, sizeof(double), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            set_error("map_init auto cell: %s", cudaGetErrorString(e));
            return e;
        }
        cell = M0 > 0 ? (float)(kAutoCellMult * sum / (double)M0) : 0.01f;
        if (!(cell > 0.f)) cell = 0.01f;
    }
    GridView g = map_grid(w, cap, cell);
    cudaError_t e = grid_build(g, w.t.pos, w.t.cov_a, w.t.cov_b, w.ctr, cap, s);
    if (e == cudaSuccess) e = build_dense(g, w.t, s);
    if (e == cudaSuccess) e = build_graph(g, w.t, w.t.pos, w.ctr, cap, s, w.key_in);
    if (e != cudaSuccess) return e;
    fill_map(w, cap, max_insert, cell, mode, eps, out);
    return cudaSuccess;
}

// The insertion body: export (appending at *d_M), target rows of the new Gaussians, the delta grid,
// the affected rows, the hash / dense / slot lists over M + m rows, the affected rows' lists.
static cudaError_t map_insert_body(const gsicp_map &mp, const gsicp_cloud &kf, const double *d_T,
                                   const int32_t *corr, double p, double c, cudaStream_t s) {
    const int cap = mp.capacity, mi = mp.max_insert;
    Carver cv(mp.ws);
    MapWs w = map_carve(cv, cap, mi);
    cudaError_t e = export_launch(reinterpret_cast<const float4 *>(kf.pos), reinterpret_cast<const float4 *>(kf.cov_a),
                                  reinterpret_cast<const float4 *>(kf.cov_b), kf.d_n, kf.cap, d_T, p, c, corr, w.means,
                                  w.quats, w.scales, w.ctr + 1, w.export_scratch, s, w.ctr);
    if (e != cudaSuccess) {
        set_error("map_insert export: %s", cudaGetErrorString(e));
        return e;
    }
    k_map_clamp<<<1, 1, 0, s>>>(w, cap);
    GSICP_LAUNCH_CHECK("k_map_clamp");
    MapArgs a{};
    a.means = w.means; a.quats = w.quats; a.scales = w.scales;
    a.scales_are_log = 0; a.M = cap; a.mode = mp.mode; a.eps = (double)mp.eps_var;
    a.pos = w.t.pos; a.cov_a = w.t.cov_a; a.cov_b = w.t.cov_b;
    a.smid_sum = nullptr;
    a.d_base = w.ctr;
    a.d_cnt = w.ctr + 1;
    k_map_to_target<<<blocks_for(mi, 256), 256, 0, s>>>(a);
    GSICP_LAUNCH_CHECK("k_map_to_target (insert)");
    k_map_stage<<<blocks_for(mi, 256), 256, 0, s>>>(w);
    GSICP_LAUNCH_CHECK("k_map_stage");
    note_launch(3);
    GridView dg = grid_carve(w.dgrid, mi, 1, false, mp.cell);
    if ((e = grid_build(dg, w.dpos, nullptr, nullptr, w.ctr + 1, mi, s)) != cudaSuccess) return e;
    k_map_mark<<<blocks_for(cap, 256), 256, 0, s>>>(w, dg, cap);
    GSICP_LAUNCH_CHECK("k_map_mark");
    note_launch();
    GridView g = map_grid(w, cap, mp.cell);
    if ((e = grid_build(g, w.t.pos, w.t.cov_a, w.t.cov_b, w.ctr + 2, cap, s)) != cudaSuccess) return e;
    if ((e = build_dense(g, w.t, s)) != cudaSuccess) return e;
    if ((e = knn_graph_queue_launch(g, w.t.pos, w.ctr + 2, cap, w.queue, reinterpret_cast<const uint32_t *>(w.ctr + 3),
                                    w.t.knn_idx, s)) != cudaSuccess)
        return e;
    if ((e = graph_finalize(g, w.t, w.ctr + 2, cap, w.key_in, s)) != cudaSuccess) return e;
    k_map_commit<<<1, 1, 0, s>>>(w.ctr);
    GSICP_LAUNCH_CHECK("k_map_commit");
    note_launch();
    return cudaSuccess;
}

static cudaStream_t map_body_stream() {
    static thread_local cudaStream_t bs = nullptr;
    static thread_local int dev = -1;
    int d = 0;
    cudaGetDevice(&d);
    if (!bs || dev != d) {
        if (cudaStreamCreateWithFlags(&bs, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        dev = d;
    }
    return bs;
}

cudaError_t map_insert_launch(const gsicp_map &mp, const gsicp_cloud &kf, const double *d_T, const int32_t *corr,
                              double p, double c, const int32_t *d_flag, cudaStream_t s) {
    if (!d_flag) return map_insert_body(mp, kf, d_T, corr, p, c, s);
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cst);
    if (cst != cudaStreamCaptureStatusActive) {  // eager: read the flag (blocking), run or skip
        int32_t f = 0;
        cudaError_t e = cudaMemcpyAsync(&f, d_flag, sizeof(f), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            set_error("map_insert flag: %s", cudaGetErrorString(e));
            return e;
        }
        return f ? map_insert_body(mp, kf, d_T, corr, p, c, s) : cudaSuccess;
    }
    // inside a capture: the body behind a conditional (IF) node switched by the device flag
    cudaGraph_t graph = nullptr;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    unsigned long long cid = 0;
    cudaError_t e;
    if ((e = cudaStreamGetCaptureInfo(s, &cst, &cid, &graph, &deps, &nd)) != cudaSuccess) return e;
    cudaGraphConditionalHandle h;
    if ((e = cudaGraphConditionalHandleCreate(&h, graph, 0, 0)) != cudaSuccess) return e;
    k_map_cond<<<1, 1, 0, s>>>(d_flag, h);
    GSICP_LAUNCH_CHECK("k_map_cond");
    note_launch();
    if ((e = cudaStreamGetCaptureInfo(s, &cst, &cid, &graph, &deps, &nd)) != cudaSuccess) return e;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    if ((e = cudaGraphAddNode(&cnode, graph, deps, nd, &cp)) != cudaSuccess) return e;
    cudaStream_t bs = map_body_stream();
    if (!bs) return cudaErrorInvalidResourceHandle;
    if ((e = cudaStreamBeginCaptureToGraph(bs, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                           cudaStreamCaptureModeRelaxed)) != cudaSuccess)
        return e;
    pdl_suspended() = true;  // no programmatic edges inside the conditional body
    cudaError_t eb = map_insert_body(mp, kf, d_T, corr, p, c, bs);
    pdl_suspended() = false;
    cudaGraph_t body_out = nullptr;
    e = cudaStreamEndCapture(bs, &body_out);
    if (eb != cudaSuccess) return eb;
    if (e != cudaSuccess) return e;
    return cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies);
}

cudaError_t keyframe_launch(const gsicp_align_stats *d_stats, int32_t *d_state, float min_fitness, int max_gap,
                            cudaStream_t s) {
    k_keyframe<<<1, 1, 0, s>>>(d_stats, d_state, min_fitness, max_gap);
    GSICP_LAUNCH_CHECK("k_keyframe");
    note_launch();
    return cudaSuccess;
}

}  // namespace gsicp
