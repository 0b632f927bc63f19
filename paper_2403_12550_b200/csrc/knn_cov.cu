// A3 + A4  Exact kNN (k <= 32) + covariance + closed-form eigen + regularisation, fused.
// P:92 "The covariance C of one 3D point x is given by computing covariance matrix of
// k-nearest neighbors of x"; Eq. 3-4 for the regularisation (R4-R8).
//
// Warp-cooperative: a warp takes 32 consecutive queries (coarsest-level cell order, so they are
// spatial neighbours) and searches them one after the other with all 32 lanes:
//   * the query's best-K list is distributed over the lanes (lane j holds the j-th smallest packed
//     (key, index) u64), so an insertion is one ballot + one shuffle, not a K-long register walk;
//   * cells are probed 32 at a time (lane = cell of the current Chebyshev shell, nearest shells
//     first; cells whose box lower bound exceeds the K-th key are skipped), and the points of the
//     non-empty cells are scanned as one flattened, coalesced range (lane = candidate);
//   * after shell m every unscanned point is >= m*h + delta_q away, so the list is exact once its
//     K-th key is below that bound (conservative rounding margin), or once the shell block covers
//     the cloud's bbox.  A query that cannot fill its list within shell 1 restarts one level
//     coarser (multi-level hash: depth-image density varies as z^2).
// The moments of each query are warp-reduced into the lane that owns it; then every lane runs the
// binary64 eigen-decomposition and regularisation of its own query in parallel.
#include <stdlib.h>

#include <algorithm>
#include <string.h>

#include "grid.cuh"
#include "host_common.cuh"
#include "search.cuh"

namespace gsicp {

// per-query diagnostics (tests / profiling only): level, cells probed, candidates, insertions
thread_local int32_t *g_knn_debug = nullptr;

namespace {

constexpr int kMinCell = 3;
constexpr int kKnnThreads = 128;
constexpr int kQueriesPerWarp = 8;  // queries a warp searches one after the other (one work batch)
constexpr int kKnnMinBlocks = 8;    // resident blocks per SM the register budget is sized for
constexpr int kMergeThreshold = 4;  // more passing candidates than this: sort-merge the batch
constexpr unsigned kFull = 0xffffffffu;
constexpr int kKnnBatch = 4;
constexpr int kMaxK = 32;  // hash probes in flight per thread (thread variant)

struct KnnArgs {
    GridView g;
    const float4 *pos;
    const int32_t *d_n;
    int k;
    int mode;
    double eps;
    float4 *cov_a, *cov_b;
    int32_t *knn_idx;
    int4 *debug;
    int32_t *nbr_t;   // [cap][kMaxK]: the k neighbours (input indices, sorted, -1 pad) per query in search order
};

__device__ __forceinline__ unsigned long long shfl_u64(unsigned long long v, int src) {
    return ((unsigned long long)__shfl_sync(kFull, (unsigned)(v >> 32), src) << 32) |
           __shfl_sync(kFull, (unsigned)v, src);
}
__device__ __forceinline__ unsigned long long shfl_xor_u64(unsigned long long v, int m) {
    return ((unsigned long long)__shfl_xor_sync(kFull, (unsigned)(v >> 32), m) << 32) |
           __shfl_xor_sync(kFull, (unsigned)v, m);
}
__device__ __forceinline__ unsigned long long shfl_up_u64(unsigned long long v, int d) {
    return ((unsigned long long)__shfl_up_sync(kFull, (unsigned)(v >> 32), d) << 32) |
           __shfl_up_sync(kFull, (unsigned)v, d);
}

// Warp-distributed sorted best-K list.
template <int K>
struct WarpTopK {
    unsigned long long L;  // lane j < K: j-th smallest (kEmptyKey if fewer); lanes >= K: kEmptyKey
    unsigned long long worst;  // = list[K-1] (warp-uniform)
    int inserts;

    __device__ __forceinline__ void reset() {
        L = kEmptyKey;
        worst = kEmptyKey;
    }
    __device__ __forceinline__ bool full() const { return worst != kEmptyKey; }
    // insert the candidates of all lanes (cand = kEmptyKey for none): a few by ballot + shuffle,
    // many by a warp bitonic sort of the batch merged into the list (fixed ~40 shuffles)
    // bitonic sort (ascending) of the values of lanes [0, W) (other lanes: don't care)
    template <int W>
    __device__ __forceinline__ static unsigned long long sort_w(unsigned long long c, int lane) {
#pragma unroll
        for (int k = 2; k <= W; k <<= 1)
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const unsigned long long o = shfl_xor_u64(c, j);
                const bool up = ((lane & k) == 0) == ((lane & j) == 0);  // keep the min here?
                c = up ? (o < c ? o : c) : (o > c ? o : c);
            }
        return c;
    }
    // bitonic merge of a bitonic 32-sequence to ascending
    __device__ __forceinline__ static unsigned long long merge32(unsigned long long m, int lane) {
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
            const unsigned long long o = shfl_xor_u64(m, j);
            m = ((lane & j) == 0) ? (o < m ? o : m) : (o > m ? o : m);
        }
        return m;
    }
    __device__ __forceinline__ void insert_all(unsigned long long cand, int lane, unsigned long long *wbuf) {
        unsigned pass = __ballot_sync(kFull, cand < worst);
        const int np = __popc(pass);
        if (np > kMergeThreshold && np <= 8 && K <= 24) {
            // few: compact the passing candidates to lanes 0..np-1 (warp scratch), sort those 8,
            // place them descending in lanes 24..31 after the ascending list (a bitonic sequence)
            // and merge — 6 + 5 shuffle stages instead of 15 + 5
            inserts += np;
            if (cand < worst) wbuf[__popc(pass & ((1u << lane) - 1u))] = cand;
            __syncwarp();
            unsigned long long c = lane < np ? wbuf[lane] : kEmptyKey;
            __syncwarp();
            c = sort_w<8>(c, lane);
            const unsigned long long rev = shfl_u64(c, (31 - lane) & 7);
            const unsigned long long m = merge32(lane < K ? L : (lane >= 24 ? rev : kEmptyKey), lane);
            L = lane < K ? m : kEmptyKey;
            worst = shfl_u64(L, K - 1);
            return;
        }
        if (np > kMergeThreshold) {
            inserts += np;
            unsigned long long c = cand < worst ? cand : kEmptyKey;
            c = sort_w<32>(c, lane);
            if (shfl_u64(L, 0) == kEmptyKey) {  // empty list: the sorted batch is the list
                L = lane < K ? c : kEmptyKey;
                worst = shfl_u64(L, K - 1);
                return;
            }
            // list ascending (lanes >= K empty) vs batch descending: lane-wise min = the 32 smallest
            const unsigned long long rev = shfl_u64(c, 31 - lane);
            unsigned long long m = L < rev ? L : rev;
            m = merge32(m, lane);
            L = lane < K ? m : kEmptyKey;
            worst = shfl_u64(L, K - 1);
            return;
        }
        while (pass) {
            const int src = __ffs(pass) - 1;
            pass &= pass - 1;
            const unsigned long long v = shfl_u64(cand, src);
            if (!(v < worst)) continue;  // worst shrank since the ballot
            ++inserts;
            const int p = __popc(__ballot_sync(kFull, lane < K && L < v));
            const unsigned long long up = shfl_up_u64(L, 1);
            if (lane < K) L = lane < p ? L : (lane == p ? v : up);
            worst = shfl_u64(L, K - 1);
        }
    }
};

struct Counters {
    int probes = 0, cands = 0;
};

// Probe the cells one per lane (valid lanes only), then scan all their points as one flattened
// range, 32 candidates per round, inserting into the list.  The owning cell of a candidate is
// found without a search: the non-empty cells are compacted into the warp's cell table (spos
// start, first item), the cell starts falling into a round are OR-reduced into a bit mask, and a
// lane's cell is (cells started before the round) + popc(starts at or below the lane) - 1.
template <int K>
__device__ __forceinline__ void scan_cells(const GridView &g, bool valid, unsigned long long key, float qx, float qy,
                                           float qz, WarpTopK<K> &T, Counters &cn, int lane, unsigned long long *wbuf,
                                           uint2 *wcell) {
    const uint2 se = valid ? cell_lookup(g.table, g.mask, key) : make_uint2(0u, 0u);
    cn.probes += __popc(__ballot_sync(kFull, valid));
    uint32_t incl = se.y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    cn.cands += (int)total;
    const uint32_t excl = incl - se.y;
    const unsigned ne = __ballot_sync(kFull, se.y != 0u);
    if (se.y) wcell[__popc(ne & ((1u << lane) - 1u))] = make_uint2(se.x, excl);
    __syncwarp();
    int before = 0;
    for (uint32_t base = 0; base < total; base += 32) {
        const bool here = se.y != 0u && excl >= base && excl < base + 32u;
        const unsigned P = __reduce_or_sync(kFull, here ? 1u << (excl - base) : 0u);
        const uint32_t item = base + lane;
        unsigned long long cand = kEmptyKey;
        if (item < total) {
            const uint2 c = wcell[before + __popc(P & (0xffffffffu >> (31 - lane))) - 1];
            const float4 p = __ldg(g.spos + c.x + (item - c.y));
            cand = pack_ki(canon_key(qx, qy, qz, p.x, p.y, p.z), (uint32_t)__float_as_int(p.w));
        }
        before += __popc(P);
        T.insert_all(cand, lane, wbuf);
    }
    __syncwarp();
}

// Exact best-K of one query on one level.  Returns false (list reset) if shell 1 does not fill
// the list and a coarser level exists.
template <int K>
__device__ bool knn_search_warp(const GridView &g, int level, float qx, float qy, float qz, WarpTopK<K> &T,
                                Counters &cn, int lane, unsigned long long *wbuf, uint2 *wcell, const int *sbox) {
    T.reset();
    const float inv_h = ldexpf(g.inv_h0, -level);
    const QueryCell qc(qx, qy, qz, ldexpf(g.h0, level), inv_h);
    const int *blo = sbox + 6 * level, *bhi = sbox + 6 * level + 3;
    for (int m = 0;; ++m) {
        // shell 0 and 1 together: lane 0 = own cell, lanes 1..26 = shell 1
        if (m == 1) continue;
        const int cnt = m == 0 ? 27 : shell_count(m);
        for (int t0 = 0; t0 < cnt; t0 += 32) {
            const int t = t0 + lane;
            int dx = 0, dy = 0, dz = 0;
            if (t < cnt) {
                if (m == 0) {
                    if (t > 0) shell_cell(1, t - 1, dx, dy, dz);
                } else {
                    shell_cell(m, t, dx, dy, dz);
                }
            }
            const int x = qc.c[0] + dx, y = qc.c[1] + dy, z = qc.c[2] + dz;
            bool valid = t < cnt && x >= blo[0] && x <= bhi[0] && y >= blo[1] && y <= bhi[1] && z >= blo[2] && z <= bhi[2];
            if (valid && T.full()) {
                const float lb = qc.gap2(dx, 0) + qc.gap2(dy, 1) + qc.gap2(dz, 2);
                valid = !(lb > ki_key(T.worst));
            }
            if (!__any_sync(kFull, valid)) continue;
            scan_cells<K>(g, valid, cell_key(level, x, y, z), qx, qy, qz, T, cn, lane, wbuf, wcell);
        }
        const int mm = m == 0 ? 1 : m;  // shells 0..mm are complete
        if (T.full() && ki_key(T.worst) < qc.certified_key(mm)) return true;
        if (qc.covers(mm, blo, bhi)) return true;  // whole cloud scanned (fewer than K points)
        if (mm == 1 && !T.full() && level + 1 < g.levels) return false;
    }
}

template <int K>
__global__ void __launch_bounds__(kKnnThreads, kKnnMinBlocks) k_knn_search(KnnArgs a) {
    const int n = *a.d_n;
    const GridView &g = a.g;
    const int lane = threadIdx.x & 31;
    __shared__ unsigned long long sBuf[kKnnThreads];
    __shared__ uint2 sCell[kKnnThreads];
    __shared__ int sBox[kMaxLevels * 6];
    if (threadIdx.x < g.levels) grid_cell_bbox(g, threadIdx.x, sBox + 6 * threadIdx.x, sBox + 6 * threadIdx.x + 3);
    __syncthreads();
    unsigned long long *wbuf = sBuf + (threadIdx.x & ~31);
    uint2 *wcell = sCell + (threadIdx.x & ~31);
    // dynamic scheduling: warps take batches of kQueriesPerWarp queries until none are left
    unsigned int *work = g.counters + kMaxLevels;
    for (;;) {
    int wbase = 0;
    if (lane == 0) wbase = (int)atomicAdd(work, 1u) * kQueriesPerWarp;
    wbase = __shfl_sync(kFull, wbase, 0);
    if (wbase >= n) return;
    const int tq = wbase + lane;
    float4 e = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lane < kQueriesPerWarp && tq < n) e = __ldg(g.spos + (size_t)(g.levels - 1) * g.cap + tq);
    const int nq = min(kQueriesPerWarp, n - wbase);
    for (int qi = 0; qi < nq; ++qi) {
        const float qx = __shfl_sync(kFull, e.x, qi), qy = __shfl_sync(kFull, e.y, qi), qz = __shfl_sync(kFull, e.z, qi);
        const int i = __shfl_sync(kFull, __float_as_int(e.w), qi);
        // level: finest whose own cell holds >= kMinCell points (lane l probes level l)
        int level = g.levels - 1;
        {
            bool ok = false;
            if (lane < g.levels - 1) {
                const float inv_h = ldexpf(g.inv_h0, -lane);
                const uint2 se = cell_lookup(
                    g.table, g.mask, cell_key(lane, cell_coord(qx, inv_h), cell_coord(qy, inv_h), cell_coord(qz, inv_h)));
                ok = se.y >= (uint32_t)kMinCell;
            }
            const unsigned b = __ballot_sync(kFull, ok);
            if (b) level = __ffs(b) - 1;
        }
        WarpTopK<K> T;
        T.inserts = 0;
        Counters cn;
        while (!knn_search_warp<K>(g, level, qx, qy, qz, T, cn, lane, wbuf, wcell, sBox)) ++level;
        if (a.debug && lane == 0) a.debug[i] = make_int4(level, cn.probes, cn.cands, T.inserts);
        // moments over the k nearest: lane j < k holds neighbour j (sorted by (key, index))
        const bool have = lane < a.k && T.L != kEmptyKey;
        if (a.knn_idx && lane < a.k) a.knn_idx[(size_t)i * a.k + lane] = have ? (int32_t)ki_idx(T.L) : -1;
        if (a.nbr_t && lane < a.k) a.nbr_t[(size_t)(wbase + qi) * kMaxK + lane] = have ? (int32_t)ki_idx(T.L) : -1;
    }
    }
}

// ---------------------------------------------------------------------------------------------
// Thread-per-query variant.  A query's neighbourhood is small (tens to ~150 candidates), so one
// thread per query with its best-K list in registers issues far fewer warp instructions than a
// warp per query; queries run in coarsest-level cell order, so the 32 threads of a warp scan
// mostly the same cells (broadcast loads).
//   fill : own cell + shell 1 (27 cells, hash probes batched); if the list is not full and a
//          coarser level exists, restart there; else widen whole shells until full
//   ball : every other cell whose conservative lower bound is <= the K-th key (ball_search)
// Exact for the same reason as the warp variant: a cell is skipped only when no point in it can
// beat the current K-th (key, index).
template <int K>
struct ThreadTopK {
    unsigned long long L[K];  // ascending; kEmptyKey pads
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int j = 0; j < K; ++j) L[j] = kEmptyKey;
    }
    __device__ __forceinline__ unsigned long long worst() const { return L[K - 1]; }
    // c < worst(): all compares first (independent), then the shift — no serial chain
    __device__ __forceinline__ void insert(unsigned long long c) {
        bool b[K];
#pragma unroll
        for (int j = 0; j < K; ++j) b[j] = L[j] < c;
#pragma unroll
        for (int j = K - 1; j > 0; --j) L[j] = b[j] ? L[j] : (b[j - 1] ? c : L[j - 1]);
        L[0] = b[0] ? L[0] : c;
    }
};

template <int K>
__device__ __forceinline__ void scan_cell_thread(const float4 *__restrict__ spos, uint2 se, float qx, float qy,
                                                 float qz, ThreadTopK<K> &T, int &cands, int &inserts) {
    cands += (int)se.y;
#pragma unroll 2
    for (uint32_t p = 0; p < se.y; ++p) {
        const float4 P = __ldg(spos + se.x + p);
        const unsigned long long c = pack_ki(canon_key(qx, qy, qz, P.x, P.y, P.z), (uint32_t)__float_as_int(P.w));
        if (c < T.worst()) {
            T.insert(c);
            ++inserts;
        }
    }
}

template <int K>
__device__ bool knn_search_thread(const GridView &g, int level, float qx, float qy, float qz, ThreadTopK<K> &T,
                                  int &probes, int &cands, int &inserts) {
    T.reset();
    const float inv_h = ldexpf(g.inv_h0, -level);
    const QueryCell qc(qx, qy, qz, ldexpf(g.h0, level), inv_h);
    int blo[3], bhi[3];
    grid_cell_bbox(g, level, blo, bhi);
    CellIndex idx;
    idx.table = g.table;
    idx.mask = g.mask;
    idx.level = level;
    idx.dense = nullptr;
    idx.use_dense = false;
    // own cell + shell 1, nearest-first, kKnnBatch probes in flight
    for (int t0 = 0; t0 < 27; t0 += kKnnBatch) {
        int xs[kKnnBatch], ys[kKnnBatch], zs[kKnnBatch];
        bool valid[kKnnBatch];
        float lb[kKnnBatch];
        const float bound = ki_key(T.worst());
#pragma unroll
        for (int j = 0; j < kKnnBatch; ++j) {
            const int t = t0 + j;
            int dx = 0, dy = 0, dz = 0;
            if (t > 0 && t < 27) shell_cell(1, t - 1, dx, dy, dz);
            xs[j] = qc.c[0] + dx;
            ys[j] = qc.c[1] + dy;
            zs[j] = qc.c[2] + dz;
            lb[j] = qc.gap2(dx, 0) + qc.gap2(dy, 1) + qc.gap2(dz, 2);
            valid[j] = t < 27 && xs[j] >= blo[0] && xs[j] <= bhi[0] && ys[j] >= blo[1] && ys[j] <= bhi[1] &&
                       zs[j] >= blo[2] && zs[j] <= bhi[2] && !(lb[j] > bound);
            probes += valid[j];
        }
        uint2 se[kKnnBatch];
        idx.batch(xs, ys, zs, valid, se);
        uint32_t live = 0;
#pragma unroll
        for (int j = 0; j < kKnnBatch; ++j) live |= (se[j].y ? 1u : 0u) << j;
        while (live) {  // one copy of the scan (select the j-th entry without dynamic indexing)
            const int j = __ffs(live) - 1;
            live &= live - 1;
            uint2 sj = se[0];
            float lj = lb[0];
#pragma unroll
            for (int r = 1; r < kKnnBatch; ++r)
                if (r == j) {
                    sj = se[r];
                    lj = lb[r];
                }
            if (!(lj > ki_key(T.worst()))) scan_cell_thread<K>(g.spos, sj, qx, qy, qz, T, cands, inserts);
        }
    }
    int m = 1;
    if (T.worst() == kEmptyKey) {
        if (level + 1 < g.levels) return false;
        // finest-possible level exhausted: widen whole shells until the list is full
        while (T.worst() == kEmptyKey && !qc.covers(m, blo, bhi)) {
            ++m;
            const int cnt = shell_count(m);
            for (int t = 0; t < cnt; ++t) {
                int dx, dy, dz;
                shell_cell(m, t, dx, dy, dz);
                const int x = qc.c[0] + dx, y = qc.c[1] + dy, z = qc.c[2] + dz;
                if (x < blo[0] || x > bhi[0] || y < blo[1] || y > bhi[1] || z < blo[2] || z > bhi[2]) continue;
                const float lb = qc.gap2(dx, 0) + qc.gap2(dy, 1) + qc.gap2(dz, 2);
                if (lb > ki_key(T.worst())) continue;
                ++probes;
                const uint2 se = idx.one(x, y, z);
                if (se.y) scan_cell_thread<K>(g.spos, se, qx, qy, qz, T, cands, inserts);
            }
        }
        if (T.worst() == kEmptyKey) return true;  // fewer than K points in the whole cloud
    }
    if (ki_key(T.worst()) < qc.certified_key(m) || qc.covers(m, blo, bhi)) return true;
    const int mm = m;
    ball_search<true, kKnnBatch>(
        qc, idx, blo, bhi,
        [&](int dx, int dy, int dz) { return max(abs(dx), max(abs(dy), abs(dz))) <= mm; },
        [&](uint2 se) {
            ++probes;
            scan_cell_thread<K>(g.spos, se, qx, qy, qz, T, cands, inserts);
        },
        [&]() { return ki_key(T.worst()); });
    return true;
}

template <int K>
__global__ void __launch_bounds__(kKnnThreads) k_knn_thread(KnnArgs a) {
    const int n = *a.d_n;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const GridView &g = a.g;
    const float4 e = __ldg(g.spos + (size_t)(g.levels - 1) * g.cap + t);
    const float qx = e.x, qy = e.y, qz = e.z;
    const int i = __float_as_int(e.w);
    int level = g.levels - 1;
    for (int l = 0; l < g.levels - 1; ++l) {
        const float inv_h = ldexpf(g.inv_h0, -l);
        const uint2 se =
            cell_lookup(g.table, g.mask, cell_key(l, cell_coord(qx, inv_h), cell_coord(qy, inv_h), cell_coord(qz, inv_h)));
        if (se.y >= (uint32_t)kMinCell) {
            level = l;
            break;
        }
    }
    ThreadTopK<K> T;
    int probes = 0, cands = 0, inserts = 0;
    while (!knn_search_thread<K>(g, level, qx, qy, qz, T, probes, cands, inserts)) ++level;
    if (a.debug) a.debug[i] = make_int4(level, probes, cands, inserts);
    if (a.knn_idx) {
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (j < a.k) a.knn_idx[(size_t)i * a.k + j] = T.L[j] == kEmptyKey ? -1 : (int32_t)ki_idx(T.L[j]);
    }
    if (!a.nbr_t) return;
#pragma unroll
    for (int j = 0; j < K; ++j)
        if (j < a.k) a.nbr_t[(size_t)t * kMaxK + j] = T.L[j] == kEmptyKey ? -1 : (int32_t)ki_idx(T.L[j]);
}

// per-query epilogue (thread per query): covariance (normalised by the count), eigen,
// regularisation, scattered to input order
__global__ void __launch_bounds__(kKnnThreads) k_knn_epilogue(KnnArgs a) {
    const int n = *a.d_n;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const GridView &g = a.g;
    const int i = __float_as_int(__ldg(g.spos + (size_t)(g.levels - 1) * g.cap + t).w);
    const float4 q = __ldg(a.pos + i);
    // moments of the k neighbours about the query (binary64), in list order
    const int4 *lst = reinterpret_cast<const int4 *>(a.nbr_t + (size_t)t * kMaxK);
    double s1[3] = {0, 0, 0}, s2[6] = {0, 0, 0, 0, 0, 0};
    int cnt = 0;
    for (int j4 = 0; j4 < (a.k + 3) / 4; ++j4) {
        const int4 w = __ldg(lst + j4);
        const int ids[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (4 * j4 + u >= a.k || ids[u] < 0) continue;
            const float4 p = __ldg(a.pos + ids[u]);
            const double d0 = (double)p.x - (double)q.x, d1 = (double)p.y - (double)q.y, d2 = (double)p.z - (double)q.z;
            s1[0] += d0;
            s1[1] += d1;
            s1[2] += d2;
            s2[0] += d0 * d0;
            s2[1] += d0 * d1;
            s2[2] += d0 * d2;
            s2[3] += d1 * d1;
            s2[4] += d1 * d2;
            s2[5] += d2 * d2;
            ++cnt;
        }
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

// kNN kernel variant: warp per query (default) or thread per query (GSICP_KNN=thread, A/B only)
bool knn_use_warp() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("GSICP_KNN");
        v = (e && strcmp(e, "thread") == 0) ? 0 : 1;
    }
    return v == 1;
}

template <int K>
cudaError_t launch_search(const KnnArgs &a, int cap, cudaStream_t s) {
    const bool timed = a.nbr_t != nullptr;  // the covariance search (not the target graph build)
    if (timed) ktimer_mark(KT_KNN_SEARCH, false, s);
    if (knn_use_warp()) {
        // a resident grid (one wave) pulling work batches; never more warps than batches
        const long long warps = (cap + kQueriesPerWarp - 1) / kQueriesPerWarp;
        const long long blocks = std::min<long long>(blocks_for(warps * 32, kKnnThreads), (long long)num_sms() * kKnnMinBlocks);
        k_knn_search<K><<<(unsigned)std::max<long long>(blocks, 1), kKnnThreads, 0, s>>>(a);
    } else {
        k_knn_thread<K><<<blocks_for(cap, kKnnThreads), kKnnThreads, 0, s>>>(a);
    }
    GSICP_LAUNCH_CHECK("k_knn_search");
    if (timed) ktimer_mark(KT_KNN_SEARCH, true, s);
    return cudaSuccess;
}

template <int K>
cudaError_t launch_k(const KnnArgs &a, int cap, cudaStream_t s) {
    cudaError_t e = launch_search<K>(a, cap, s);
    if (e != cudaSuccess) return e;
    k_knn_epilogue<<<blocks_for(cap, kKnnThreads), kKnnThreads, 0, s>>>(a);
    GSICP_LAUNCH_CHECK("k_knn_epilogue");
    note_launch(2);
    return cudaSuccess;
}

}  // namespace

size_t covariances_ws_bytes(int cap, int levels) {
    return grid_bytes(cap, levels, false) + align_up((size_t)cap * kMaxK * sizeof(int32_t));
}

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
    a.debug = reinterpret_cast<int4 *>(g_knn_debug);
    a.nbr_t = reinterpret_cast<int32_t *>(static_cast<char *>(ws) + grid_bytes(cap, levels, false));
    cudaError_t e = grid_build(a.g, a.pos, nullptr, nullptr, d_n, cap, s);
    if (e != cudaSuccess) return e;
    if (k <= 4) return launch_k<4>(a, cap, s);
    if (k <= 8) return launch_k<8>(a, cap, s);
    if (k <= 16) return launch_k<16>(a, cap, s);
    if (k <= 20) return launch_k<20>(a, cap, s);
    if (k <= 24) return launch_k<24>(a, cap, s);
    return launch_k<32>(a, cap, s);
}

// Exact kGraphK-NN lists (input indices, sorted by (key, index), self included) of the points of
// an already built single-level grid — the target kNN graph behind the align kernel's certified
// warm start.  No covariances.
cudaError_t knn_graph_launch(const GridView &g, const float4 *pos, const int32_t *d_n, int cap, int32_t *knn_idx,
                             cudaStream_t s) {
    KnnArgs a{};
    a.g = g;
    a.pos = pos;
    a.d_n = d_n;
    a.k = kGraphK;
    a.knn_idx = knn_idx;
    a.nbr_t = nullptr;
    a.debug = nullptr;
    cudaError_t e = launch_search<kGraphK>(a, cap, s);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaSuccess;
}

}  // namespace gsicp
