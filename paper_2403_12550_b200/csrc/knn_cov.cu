// A3 + A4  Exact kNN (k <= 32) + covariance + closed-form eigen + regularisation, fused.
// P:92 "The covariance C of one 3D point x is given by computing covariance matrix of
// k-nearest neighbors of x"; Eq. 3-4 for the regularisation (R4-R8).
//
// One thread per query; the query's top-K list lives in registers as packed (key, index) u64
// (sorted ascending).  Search = certified expanding rings on one level of the multi-level
// hash: ring m visits the Chebyshev shell m, skipping cells whose box distance exceeds the
// current K-th key; after ring m every unvisited point is at least m*h + delta_q away
// (delta_q = distance from q to its own cell's nearest face), so the list is exact once the
// K-th key is below that bound (with a conservative rounding margin), or once the ring block
// covers the cloud's bbox.  Level = finest level whose own cell holds >= kMinCell points;
// if rings 0..2 do not certify, the query restarts one level coarser.
#include "grid.cuh"
#include "host_common.cuh"

namespace gsicp {

namespace {

constexpr int kMinCell = 4;
constexpr int kKnnThreads = 128;
constexpr float kRelMargin = 1e-5f;

struct KnnArgs {
    GridView g;
    const float4 *pos;
    const int32_t *d_n;
    int k;
    int mode;
    double eps;
    float4 *cov_a, *cov_b;
    int32_t *knn_idx;
};

template <int K>
__device__ __forceinline__ void topk_insert(unsigned long long (&L)[K], unsigned long long v) {
    if (v >= L[K - 1]) return;
    L[K - 1] = v;
#pragma unroll
    for (int j = K - 1; j > 0; --j) {
        const unsigned long long a = L[j - 1], b = L[j];
        const bool sw = b < a;
        L[j - 1] = sw ? b : a;
        L[j] = sw ? a : b;
    }
}

template <int K>
__device__ __forceinline__ void scan_cell(const GridView &g, uint2 se, float qx, float qy, float qz,
                                          unsigned long long (&L)[K]) {
    for (uint32_t j = se.x; j < se.x + se.y; ++j) {
        const float4 p = __ldg(g.spos + j);
        const float key = canon_key(qx, qy, qz, p.x, p.y, p.z);
        topk_insert<K>(L, pack_ki(key, (uint32_t)__float_as_int(p.w)));
    }
}

// Returns true when the list is certified exact.
template <int K>
__device__ bool knn_search(const GridView &g, int level, int ring_limit, float qx, float qy, float qz,
                           unsigned long long (&L)[K]) {
#pragma unroll
    for (int j = 0; j < K; ++j) L[j] = kEmptyKey;
    const float inv_h = ldexpf(g.inv_h0, -level);
    const float h = ldexpf(g.h0, level);
    const int c[3] = {cell_coord(qx, inv_h), cell_coord(qy, inv_h), cell_coord(qz, inv_h)};
    const float q[3] = {qx, qy, qz};
    float dlo[3], dhi[3];
    float dq = INFINITY;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        dlo[a] = fmaxf(q[a] - (float)c[a] * h, 0.f);
        dhi[a] = fmaxf((float)(c[a] + 1) * h - q[a], 0.f);
        dq = fminf(dq, fminf(dlo[a], dhi[a]));
    }
    int blo[3], bhi[3];
    grid_cell_bbox(g, level, blo, bhi);
    // absolute slack for binary32 cell assignment / box-face rounding
    const float margin = 2e-6f * (fabsf(qx) + fabsf(qy) + fabsf(qz)) + h * kRelMargin;
    for (int m = 0;; ++m) {
        if (m == 0) {
            scan_cell<K>(g, cell_lookup(g.table, g.mask, cell_key(level, c[0], c[1], c[2])), qx, qy, qz, L);
        } else {
            const int cnt = shell_count(m);
            for (int t = 0; t < cnt; ++t) {
                int dx, dy, dz;
                shell_offset(m, t, dx, dy, dz);
                const int x = c[0] + dx, y = c[1] + dy, z = c[2] + dz;
                if (x < blo[0] || x > bhi[0] || y < blo[1] || y > bhi[1] || z < blo[2] || z > bhi[2]) continue;
                const float gx = fmaxf(axis_gap(dx, dlo[0], dhi[0], h) - margin, 0.f);
                const float gy = fmaxf(axis_gap(dy, dlo[1], dhi[1], h) - margin, 0.f);
                const float gz = fmaxf(axis_gap(dz, dlo[2], dhi[2], h) - margin, 0.f);
                const float lb = (gx * gx + gy * gy + gz * gz) * (1.f - kRelMargin);
                if (L[K - 1] != kEmptyKey && lb > ki_key(L[K - 1])) continue;
                scan_cell<K>(g, cell_lookup(g.table, g.mask, cell_key(level, x, y, z)), qx, qy, qz, L);
            }
        }
        const float B = fmaxf((float)m * h + dq - margin, 0.f);
        if (L[K - 1] != kEmptyKey && ki_key(L[K - 1]) < B * B * (1.f - kRelMargin)) return true;
        if (c[0] - m <= blo[0] && c[0] + m >= bhi[0] && c[1] - m <= blo[1] && c[1] + m >= bhi[1] &&
            c[2] - m <= blo[2] && c[2] + m >= bhi[2])
            return true;
        if (m >= ring_limit) return false;
    }
}

template <int K>
__global__ void __launch_bounds__(kKnnThreads) k_knn_cov(KnnArgs a) {
    const int n = *a.d_n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 q = __ldg(a.pos + i);
    const GridView &g = a.g;
    int level = g.levels - 1;
    for (int l = 0; l < g.levels - 1; ++l) {
        const float inv_h = ldexpf(g.inv_h0, -l);
        const uint2 se = cell_lookup(
            g.table, g.mask, cell_key(l, cell_coord(q.x, inv_h), cell_coord(q.y, inv_h), cell_coord(q.z, inv_h)));
        if (se.y >= (uint32_t)kMinCell) {
            level = l;
            break;
        }
    }
    unsigned long long L[K];
    for (; level < g.levels; ++level)
        if (knn_search<K>(g, level, level == g.levels - 1 ? 0x7fffffff : 2, q.x, q.y, q.z, L)) break;

    // query-centred binary64 moments over the k nearest (normalised by the count)
    double s1[3] = {0, 0, 0}, s2[6] = {0, 0, 0, 0, 0, 0};
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (j < a.k && L[j] != kEmptyKey) {
            const float4 p = __ldg(a.pos + ki_idx(L[j]));
            const double d0 = (double)p.x - (double)q.x, d1 = (double)p.y - (double)q.y, d2 = (double)p.z - (double)q.z;
            s1[0] += d0; s1[1] += d1; s1[2] += d2;
            s2[0] += d0 * d0; s2[1] += d0 * d1; s2[2] += d0 * d2;
            s2[3] += d1 * d1; s2[4] += d1 * d2; s2[5] += d2 * d2;
            ++cnt;
        }
        if (a.knn_idx && j < a.k) a.knn_idx[(size_t)i * a.k + j] = L[j] != kEmptyKey ? (int32_t)ki_idx(L[j]) : -1;
    }
    const double inv = 1.0 / (double)cnt;
    const double mu[3] = {s1[0] * inv, s1[1] * inv, s1[2] * inv};
    double C[6] = {s2[0] * inv - mu[0] * mu[0], s2[1] * inv - mu[0] * mu[1], s2[2] * inv - mu[0] * mu[2],
                   s2[3] * inv - mu[1] * mu[1], s2[4] * inv - mu[1] * mu[2], s2[5] * inv - mu[2] * mu[2]};
    const Eig3 e = eig3_sym(C);
    double R[6];
    uint32_t flags = regularize(C, e, a.mode, a.eps, R);
    if (n < a.k) flags |= GSICP_FLAG_LOW_SUPPORT;
    store_cov(a.cov_a, a.cov_b, i, R, e.lam[1], flags);
}

template <int K>
cudaError_t launch_k(const KnnArgs &a, int cap, cudaStream_t s) {
    k_knn_cov<K><<<blocks_for(cap, kKnnThreads), kKnnThreads, 0, s>>>(a);
    GSICP_LAUNCH_CHECK("k_knn_cov");
    note_launch();
    return cudaSuccess;
}

}  // namespace

size_t covariances_ws_bytes(int cap, int levels) { return grid_bytes(cap, levels, false); }

cudaError_t covariances_launch(const float *pos, const int32_t *d_n, int cap, int k, int mode, float eps,
                               float cell0, int levels, float *cov_a, float *cov_b, int32_t *knn_idx, void *ws,
                               cudaStream_t s) {
    KnnArgs a;
    a.g = grid_carve(ws, cap, levels, false, cell0);
    a.pos = reinterpret_cast<const float4 *>(pos);
    a.d_n = d_n;
    a.k = k;
    a.mode = mode;
    a.eps = (double)eps;
    a.cov_a = reinterpret_cast<float4 *>(cov_a);
    a.cov_b = reinterpret_cast<float4 *>(cov_b);
    a.knn_idx = knn_idx;
    cudaError_t e = grid_build(a.g, a.pos, nullptr, nullptr, d_n, cap, s);
    if (e != cudaSuccess) return e;
    if (k <= 4) return launch_k<4>(a, cap, s);
    if (k <= 8) return launch_k<8>(a, cap, s);
    if (k <= 12) return launch_k<12>(a, cap, s);
    if (k <= 16) return launch_k<16>(a, cap, s);
    if (k <= 20) return launch_k<20>(a, cap, s);
    if (k <= 24) return launch_k<24>(a, cap, s);
    return launch_k<32>(a, cap, s);
}

}  // namespace gsicp
