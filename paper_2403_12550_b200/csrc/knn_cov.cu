// A3 + A4  Exact kNN (k <= 32) + covariance + closed-form eigen + regularisation, fused.
// P:92 "The covariance C of one 3D point x is given by computing covariance matrix of
// k-nearest neighbors of x"; Eq. 3-4 for the regularisation (R4-R8).
//
// One thread per query; the query's best-K candidates live in registers as packed (key, index)
// u64 words (unordered, with the current worst tracked).  Search = certified expanding rings
// (search.cuh) on one level of the multi-level hash: own cell, whole shells until K candidates
// are held, then the ball traversal bounded by the current K-th key (exact at any level; the
// level only sets the cost).  Level = finest level whose own cell holds >= kMinCell points.
// Queries are processed in the coarsest level's cell order so a warp's queries are spatial
// neighbours (shared cells, L1 hits, uniform loop trip counts); results scatter to input order.
#include "grid.cuh"
#include "host_common.cuh"
#include "search.cuh"

namespace gsicp {

namespace {

constexpr int kMinCell = 3;
constexpr int kKnnThreads = 128;

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
struct TopK {
    unsigned long long L[K];
    unsigned long long worst;

    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int j = 0; j < K; ++j) L[j] = kEmptyKey;
        worst = kEmptyKey;
    }
    __device__ __forceinline__ bool full() const { return worst != kEmptyKey; }
    __device__ __forceinline__ void insert(unsigned long long v) {
        if (v >= worst) return;
        bool done = false;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const bool hit = !done && L[j] == worst;
            L[j] = hit ? v : L[j];
            done |= hit;
        }
        unsigned long long w = L[0];
#pragma unroll
        for (int j = 1; j < K; ++j) w = L[j] > w ? L[j] : w;
        worst = w;
    }
    // ascending (key, index) order: odd-even transposition network
    __device__ __forceinline__ void sort() {
#pragma unroll
        for (int p = 0; p < K; ++p)
#pragma unroll
            for (int j = p & 1; j + 1 < K; j += 2) {
                const unsigned long long a = L[j], b = L[j + 1];
                L[j] = a < b ? a : b;
                L[j + 1] = a < b ? b : a;
            }
    }
};

template <int K>
__device__ __forceinline__ void scan_cell(const GridView &g, uint2 se, float qx, float qy, float qz, TopK<K> &T) {
    for (uint32_t j = se.x; j < se.x + se.y; ++j) {
        const float4 p = __ldg(g.spos + j);
        T.insert(pack_ki(canon_key(qx, qy, qz, p.x, p.y, p.z), (uint32_t)__float_as_int(p.w)));
    }
}

// Exact best-K of the query on one level: own cell, whole shells until K candidates are held
// (or the cloud is exhausted), then the ball traversal bounded by the current K-th key.
// Returns false (list reset) when K candidates are not found within shell 1 and a coarser level
// exists: sparse neighbourhoods (outliers, far depth points) restart one level up instead of
// growing many shells of small cells.
template <int K>
__device__ bool knn_search(const GridView &g, int level, float qx, float qy, float qz, TopK<K> &T) {
    T.reset();
    const float inv_h = ldexpf(g.inv_h0, -level);
    const QueryCell qc(qx, qy, qz, ldexpf(g.h0, level), inv_h);
    int blo[3], bhi[3];
    grid_cell_bbox(g, level, blo, bhi);
    auto scan = [&](int x, int y, int z) {
        scan_cell<K>(g, cell_lookup(g.table, g.mask, cell_key(level, x, y, z)), qx, qy, qz, T);
    };
    scan(qc.c[0], qc.c[1], qc.c[2]);
    int m_done = 0;
    while (!T.full()) {
        if (qc.covers(m_done, blo, bhi)) return true;  // fewer than K points in the whole cloud
        if (m_done == 1 && level + 1 < g.levels) return false;
        ++m_done;
        const int cnt = shell_count(m_done);
        for (int t = 0; t < cnt; ++t) {
            int dx, dy, dz;
            shell_cell(m_done, t, dx, dy, dz);
            const int x = qc.c[0] + dx, y = qc.c[1] + dy, z = qc.c[2] + dz;
            if (x < blo[0] || x > bhi[0] || y < blo[1] || y > bhi[1] || z < blo[2] || z > bhi[2]) continue;
            scan(x, y, z);
        }
    }
    ball_search(
        qc, g.table, g.mask, blo, bhi, m_done, [&](int x, int y, int z) { return cell_key(level, x, y, z); },
        [&](uint2 se) { scan_cell<K>(g, se, qx, qy, qz, T); }, [&]() { return ki_key(T.worst); });
    return true;
}

template <int K>
__global__ void __launch_bounds__(kKnnThreads) k_knn_cov(KnnArgs a) {
    const int n = *a.d_n;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const GridView &g = a.g;
    const float4 e = __ldg(g.spos + (size_t)(g.levels - 1) * g.cap + t);
    const int i = __float_as_int(e.w);
    const float qx = e.x, qy = e.y, qz = e.z;
    int level = g.levels - 1;
    for (int l = 0; l < g.levels - 1; ++l) {
        const float inv_h = ldexpf(g.inv_h0, -l);
        const uint2 se = cell_lookup(
            g.table, g.mask, cell_key(l, cell_coord(qx, inv_h), cell_coord(qy, inv_h), cell_coord(qz, inv_h)));
        if (se.y >= (uint32_t)kMinCell) {
            level = l;
            break;
        }
    }
    TopK<K> T;
    while (!knn_search<K>(g, level, qx, qy, qz, T)) ++level;
    if (a.knn_idx || a.k != K) T.sort();

    // query-centred binary64 moments over the k nearest (normalised by the count)
    double s1[3] = {0, 0, 0}, s2[6] = {0, 0, 0, 0, 0, 0};
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (j < a.k && T.L[j] != kEmptyKey) {
            const float4 p = __ldg(a.pos + ki_idx(T.L[j]));
            const double d0 = (double)p.x - (double)qx, d1 = (double)p.y - (double)qy, d2 = (double)p.z - (double)qz;
            s1[0] += d0; s1[1] += d1; s1[2] += d2;
            s2[0] += d0 * d0; s2[1] += d0 * d1; s2[2] += d0 * d2;
            s2[3] += d1 * d1; s2[4] += d1 * d2; s2[5] += d2 * d2;
            ++cnt;
        }
        if (a.knn_idx && j < a.k) a.knn_idx[(size_t)i * a.k + j] = T.L[j] != kEmptyKey ? (int32_t)ki_idx(T.L[j]) : -1;
    }
    const double inv = 1.0 / (double)cnt;
    const double mu[3] = {s1[0] * inv, s1[1] * inv, s1[2] * inv};
    double C[6] = {s2[0] * inv - mu[0] * mu[0], s2[1] * inv - mu[0] * mu[1], s2[2] * inv - mu[0] * mu[2],
                   s2[3] * inv - mu[1] * mu[1], s2[4] * inv - mu[1] * mu[2], s2[5] * inv - mu[2] * mu[2]};
    const Eig3 ev = eig3_sym(C);
    double R[6];
    uint32_t flags = regularize(C, ev, a.mode, a.eps, R);
    if (n < a.k) flags |= GSICP_FLAG_LOW_SUPPORT;
    store_cov(a.cov_a, a.cov_b, i, R, ev.lam[1], flags);
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
