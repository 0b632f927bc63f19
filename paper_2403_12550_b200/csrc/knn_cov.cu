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

#include <cooperative_groups.h>

#include "grid.cuh"
#include "host_common.cuh"
#include "search.cuh"

namespace cg = cooperative_groups;

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
constexpr int kMaxK = 32;  // neighbour-list stride of the warp search's nbr_t rows

struct KnnArgs {
    GridView g;
    const float4 *pos;
    const int32_t *d_n;
    int k;
    int mode;
    double eps;
    float4 *cov_a, *cov_b;
    int32_t *knn_idx;
    int sort_out;     // knn_idx rows sorted by (key64, index) (API output); else any order (graph)
    int4 *debug;
    int32_t *nbr_t;   // [cap][kMaxK]: the k neighbours (input indices, -1 pad) per query in search order
    // queue mode (fallback of the image-window kernel): the queries are queue[0 .. *queue_n) (input
    // indices) instead of every point; query t of the search is queue[t]
    const uint32_t *queue;
    const uint32_t *queue_n;
    uint32_t *work;   // dynamic work counter of k_knn_search
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
__device__ __forceinline__ double shfl_f64(double v, int src) {
    return __hiloint2double(__shfl_sync(kFull, __double2hiint(v), src), __shfl_sync(kFull, __double2loint(v), src));
}

// Position of this lane's entry (sel: taking part) in the (key64, index) order of all selected
// lanes' entries (the key64 of each computed once, then compared by shuffles).
__device__ __forceinline__ int warp_rank64(bool sel, uint32_t id, double qx, double qy, double qz,
                                           const float4 *__restrict__ pos) {
    double k64 = INFINITY;
    if (sel) {
        const float4 p = __ldg(pos + id);
        k64 = key64(qx, qy, qz, p.x, p.y, p.z);
    }
    int r = 0;
    for (unsigned m = __ballot_sync(kFull, sel); m; m &= m - 1) {
        const int l = __ffs(m) - 1;
        const double ok = shfl_f64(k64, l);
        const uint32_t oi = __shfl_sync(kFull, id, l);
        r += (ok < k64 || (ok == k64 && oi < id)) ? 1 : 0;
    }
    return r;
}

// Exact k nearest by (key64, index) from the candidates of the calling warp, given
// as A (lane j: the j-th smallest packed (key32, index), kEmptyKey past the end) holding every
// candidate of key32 <= band_hi(t), t the k-th key32 — unless `capped` (more candidates than the 32
// lanes existed) and lane 31 still lies in the band: then false (the band may be incomplete).
// On success `pos_out` is this lane's output position (0..k-1, in (key64, index) order if SORT,
// else in list order) or -1 if its entry is not among the k nearest.
template <bool SORT>
__device__ __forceinline__ bool warp_exact_select(unsigned long long A, int k, bool capped, double qx, double qy,
                                                  double qz, const float4 *__restrict__ pos, int lane, int &pos_out) {
    const unsigned long long At = shfl_u64(A, k - 1);
    bool sel;
    if (At == kEmptyKey) {  // fewer than k candidates: all of them
        sel = A != kEmptyKey;
    } else {
        const float t = ki_key(At), hi = band_hi(t), lo = band_lo(t);
        if (capped && ki_key(shfl_u64(A, 31)) <= hi) return false;
        const float kk = ki_key(A);
        const bool inS = A != kEmptyKey && kk < lo;
        const bool inB = A != kEmptyKey && kk >= lo && kk <= hi;
        const int s = __popc(__ballot_sync(kFull, inS)), nb = __popc(__ballot_sync(kFull, inB));
        if (s + nb == k) {
            sel = inS || inB;
        } else {  // a tie band: rank its members by key64
            const int r = warp_rank64(inB, ki_idx(A), qx, qy, qz, pos);
            sel = inS || (inB && r < k - s);
        }
    }
    if (SORT) {
        const int r = warp_rank64(sel, ki_idx(A), qx, qy, qz, pos);
        pos_out = sel ? r : -1;
    } else {
        const unsigned sm = __ballot_sync(kFull, sel);  // (all lanes: not inside the conditional)
        pos_out = sel ? __popc(sm & ((1u << lane) - 1u)) : -1;
    }
    return true;
}

// ids[j] (every lane) = the index of the entry at output position j, -1 if none
template <int K>
__device__ __forceinline__ void collect_ids(int outpos, uint32_t id, int lane, int (&ids)[K]) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const unsigned b = __ballot_sync(kFull, outpos == j);
        const int v = (int)__shfl_sync(kFull, id, b ? __ffs(b) - 1 : 0);
        ids[j] = b ? v : -1;
    }
}

// Warp-distributed sorted list of the 32 smallest candidates (lane j holds the j-th smallest packed
// value, kEmptyKey if fewer).  Candidates are accepted below thr = min(list[31], band_hi of the
// K-th key32), so every candidate within the binary64 resolution band of the K-th is retained as
// long as the 32 lanes hold it (warp_exact_select detects the rare overflow).
// BAND: the values are band-packed (key64, index) pairs of one band (band pass): thr = list[31].
template <int K, bool BAND = false>
struct WarpTopK {
    unsigned long long L;    // this lane's entry
    unsigned long long thr;  // acceptance threshold (warp-uniform)
    unsigned long long kth;  // list[K-1] (warp-uniform)
    int inserts;

    __device__ __forceinline__ void reset() {
        L = kEmptyKey;
        thr = kEmptyKey;
        kth = kEmptyKey;
    }
    __device__ __forceinline__ bool full() const { return kth != kEmptyKey; }
    __device__ __forceinline__ float bound() const { return ki_key(thr); }  // prune / certify against this
    __device__ __forceinline__ void update() {
        kth = shfl_u64(L, K - 1);
        const unsigned long long l31 = shfl_u64(L, 31);
        const unsigned long long b =
            (BAND || kth == kEmptyKey) ? kEmptyKey : pack_ki(band_hi(ki_key(kth)), 0xffffffffu);
        thr = l31 < b ? l31 : b;
    }
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
    // insert the candidates of all lanes (cand = kEmptyKey for none): a few by ballot + shuffle,
    // many by a warp bitonic sort of the batch merged into the list
    __device__ __forceinline__ void insert_all(unsigned long long cand, int lane) {
        unsigned pass = __ballot_sync(kFull, cand < thr);
        const int np = __popc(pass);
        if (np > kMergeThreshold) {
            inserts += np;
            unsigned long long c = cand < thr ? cand : kEmptyKey;
            c = sort_w<32>(c, lane);
            if (shfl_u64(L, 0) == kEmptyKey) {  // empty list: the sorted batch is the list
                L = c;
                update();
                return;
            }
            // list ascending vs batch descending: lane-wise min = the 32 smallest (bitonic)
            const unsigned long long rev = shfl_u64(c, 31 - lane);
            L = merge32(L < rev ? L : rev, lane);
            update();
            return;
        }
        while (pass) {
            const int src = __ffs(pass) - 1;
            pass &= pass - 1;
            const unsigned long long v = shfl_u64(cand, src);
            if (!(v < thr)) continue;  // thr shrank since the ballot
            ++inserts;
            const int p = __popc(__ballot_sync(kFull, L < v));
            const unsigned long long up = shfl_up_u64(L, 1);
            L = lane < p ? L : (lane == p ? v : up);
            update();
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
// make(p) -> the packed candidate value of record p (kEmptyKey: not a candidate).
template <class TopK, class Make>
__device__ __forceinline__ void scan_cells(const GridView &g, bool valid, unsigned long long key, TopK &T,
                                           Counters &cn, int lane, uint2 *wcell, Make make) {
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
            cand = make(__ldg(g.spos + c.x + (item - c.y)));
        }
        before += __popc(P);
        T.insert_all(cand, lane);
    }
    __syncwarp();
}

// Shell-ordered exact search of one query on one level: every cell whose box lower bound is <=
// bound() (binary32 key; +inf: none yet) is scanned (nearest shells first); stops once bound() is
// below the certified key of the shells done, or the shells cover the cloud.  Returns false (list
// reset) if shell 1 does not fill the list and a coarser level exists (only when `escalate`).
// bound(T) is a stateless function of the list (no captured references: keeps T in registers).
template <class TopK, class Make, class Bound>
__device__ __forceinline__ bool knn_shells_warp(const GridView &g, int level, float qx, float qy, float qz, TopK &T,
                                                Counters &cn, int lane, uint2 *wcell, const int *sbox, bool escalate,
                                                Make make, Bound bound) {
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
            const float bd = bound(T);
            if (valid && bd < INFINITY) {
                const float lb = qc.gap2(dx, 0) + qc.gap2(dy, 1) + qc.gap2(dz, 2);
                valid = !(lb > bd);
            }
            if (!__any_sync(kFull, valid)) continue;
            scan_cells(g, valid, cell_key(level, x, y, z), T, cn, lane, wcell, make);
        }
        const int mm = m == 0 ? 1 : m;  // shells 0..mm are complete
        if (bound(T) < qc.certified_key(mm)) return true;
        if (qc.covers(mm, blo, bhi)) return true;  // whole cloud scanned
        if (escalate && mm == 1 && !T.full() && level + 1 < g.levels) return false;
    }
}

template <int K, bool SORT>
__global__ void __launch_bounds__(kKnnThreads, kKnnMinBlocks) k_knn_search(KnnArgs a) {
    pdl_wait();
    pdl_launch_dependents();
    if (a.queue && *a.queue_n == 0u) return;  // empty fallback queue (block-uniform)
    const int n = *a.d_n;
    const GridView &g = a.g;
    const int lane = threadIdx.x & 31;
    __shared__ uint2 sCell[kKnnThreads];
    __shared__ int sBox[kMaxLevels * 6];
    if (threadIdx.x < g.levels) grid_cell_bbox(g, threadIdx.x, sBox + 6 * threadIdx.x, sBox + 6 * threadIdx.x + 3);
    __syncthreads();
    uint2 *wcell = sCell + (threadIdx.x & ~31);
    // dynamic scheduling: warps take batches of kQueriesPerWarp queries until none are left
    const int nq_all = a.queue ? (int)*a.queue_n : n;
    for (;;) {
    int wbase = 0;
    // queue mode: one (hard) query per batch, so the few queued queries spread over all warps
    const int qpw = a.queue ? 1 : kQueriesPerWarp;
    if (lane == 0) wbase = (int)atomicAdd(a.work, 1u) * qpw;
    wbase = __shfl_sync(kFull, wbase, 0);
    if (wbase >= nq_all) return;
    const int tq = wbase + lane;
    float4 e = make_float4(0.f, 0.f, 0.f, 0.f);
    if (lane < qpw && tq < nq_all) {
        if (a.queue) {
            const uint32_t qi = __ldg(a.queue + tq);
            e = __ldg(a.pos + qi);
            e.w = __int_as_float((int)qi);
        } else {
            e = __ldg(g.spos + (size_t)(g.levels - 1) * g.cap + tq);
        }
    }
    const int nq = min(qpw, nq_all - wbase);
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
        auto by_key32 = [&](const float4 &p) {
            return pack_ki(canon_key(qx, qy, qz, p.x, p.y, p.z), (uint32_t)__float_as_int(p.w));
        };
        auto t_bound = [](const WarpTopK<K> &L) { return L.thr != kEmptyKey ? L.bound() : INFINITY; };
        while (!knn_shells_warp(g, level, qx, qy, qz, T, cn, lane, wcell, sBox, true, by_key32, t_bound)) ++level;
        // exact k nearest by (key64, index): the binary32 list resolved in binary64
        int outpos = -1;
        uint32_t myid = ki_idx(T.L);
        if (!warp_exact_select<SORT>(T.L, a.k, shfl_u64(T.L, 31) != kEmptyKey, qx, qy, qz, a.pos, lane, outpos)) {
            // band overflow (more than the list's spare lanes tie with the k-th): a second pass
            // collects exactly the band's members in the exact (key64, index) order
            const float t = ki_key(T.kth), lo = band_lo(t), hi = band_hi(t);
            const bool inS = T.L != kEmptyKey && ki_key(T.L) < lo;
            const int s = __popc(__ballot_sync(kFull, inS));
            const unsigned long long fl = band_floor_bits(t);
            const double dqx = qx, dqy = qy, dqz = qz;
            auto in_band = [&](const float4 &p) {
                const float k32 = canon_key(qx, qy, qz, p.x, p.y, p.z);
                return (k32 >= lo && k32 <= hi)
                           ? band_pack(key64(dqx, dqy, dqz, p.x, p.y, p.z), (uint32_t)__float_as_int(p.w), fl)
                           : kEmptyKey;
            };
            WarpTopK<32, true> B;
            B.inserts = 0;
            knn_shells_warp(g, level, qx, qy, qz, B, cn, lane, wcell, sBox, false, in_band,
                            [hi](const WarpTopK<32, true> &) { return hi; });
            const unsigned long long b = shfl_u64(B.L, (lane - s) & 31);
            const bool takeB = lane >= s && lane < a.k && b != kEmptyKey;
            myid = inS ? ki_idx(T.L) : (takeB ? band_idx(b) : 0u);
            const bool sel = inS || takeB;
            if (SORT) {
                const int r = warp_rank64(sel, myid, dqx, dqy, dqz, a.pos);
                outpos = sel ? r : -1;
            } else {
                outpos = sel ? lane : -1;  // S occupies lanes [0, s), the band's best [s, k)
            }
        }
        if (a.debug && lane == 0 && !a.queue) a.debug[i] = make_int4(level, cn.probes, cn.cands, T.inserts);
        // every selected lane writes its entry at its output position; the rest of the row is -1
        const int cnt = __popc(__ballot_sync(kFull, outpos >= 0));
        if (a.knn_idx) {
            if (outpos >= 0) a.knn_idx[(size_t)i * a.k + outpos] = (int32_t)myid;
            if (lane >= cnt && lane < a.k) a.knn_idx[(size_t)i * a.k + lane] = -1;
        }
        if (a.nbr_t) {
            int32_t *row = a.nbr_t + (size_t)(wbase + qi) * kMaxK;
            if (outpos >= 0) row[outpos] = (int32_t)myid;
            if (lane >= cnt && lane < a.k) row[lane] = -1;
        }
    }
    }
}

// ---------------------------------------------------------------------------------------------
constexpr int pow2ceil(int x) { return x <= 1 ? 1 : 2 * pow2ceil((x + 1) / 2); }

__device__ __forceinline__ void cswap(unsigned long long &a, unsigned long long &b) {
    const unsigned long long lo = a < b ? a : b, hi = a < b ? b : a;
    a = lo;
    b = hi;
}

// Batcher odd-even merge sort of L[0..K) ascending.  The comparator list is built at compile
// time (pads above K stay +inf, so comparators that touch them are dropped) and applied by
// template recursion, so every index is a constant and L stays in registers.
template <int K>
struct BatcherNet {
    static constexpr int N = pow2ceil(K);
    int a[N * 8 * 8], b[N * 8 * 8], count;
    constexpr BatcherNet() : a(), b(), count(0) {
        for (int p = 1; p < N; p <<= 1)
            for (int kk = p; kk >= 1; kk >>= 1)
                for (int j = kk % p; j + kk < N; j += 2 * kk)
                    for (int i = 0; i < kk && i < N - j - kk; ++i) {
                        const int x = i + j, y = i + j + kk;
                        if (y < K && (x / (2 * p)) == (y / (2 * p))) {
                            a[count] = x;
                            b[count] = y;
                            ++count;
                        }
                    }
    }
};
template <int K>
inline constexpr BatcherNet<K> kBatcherNet{};
template <int K, int I>
__device__ __forceinline__ void sort_net_step(unsigned long long (&L)[K]) {
    if constexpr (I < kBatcherNet<K>.count) {
        constexpr int x = kBatcherNet<K>.a[I], y = kBatcherNet<K>.b[I];
        cswap(L[x], L[y]);
        sort_net_step<K, I + 1>(L);
    }
}
template <int K>
__device__ __forceinline__ void sort_net(unsigned long long (&L)[K]) {
    sort_net_step<K, 0>(L);
}

// moments of the query's neighbours (binary64, in the given order) -> covariance -> eigen ->
// regularisation -> store (shared by the image-window kernel and the epilogue of the warp search)
// moments (sum of d, sum of d d^T over the cnt neighbours, d = p - q) -> covariance (/cnt)
// -> eigen -> regularisation -> store
__device__ __forceinline__ void finish_moments(const KnnArgs &a, int n, int i, const double (&s1)[3],
                                               const double (&s2)[6], int cnt) {
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
__device__ __forceinline__ void finish_query(const KnnArgs &a, int n, int i, float4 q, int k, const int (&ids)[K]) {
    double s1[3] = {0, 0, 0}, s2[6] = {0, 0, 0, 0, 0, 0};
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (j >= k || ids[j] < 0) continue;
        const float4 p = __ldg(a.pos + ids[j]);
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
    finish_moments(a, n, i, s1, s2, cnt);
}

// per-query epilogue of the warp search (thread per query, grid-stride): covariance
// (normalised by the count), eigen, regularisation, scattered to input order.  Query t is
// the t-th point in coarsest-cell order, or queue[t] in queue mode.
template <int K>
__global__ void __launch_bounds__(kKnnThreads) k_knn_epilogue(KnnArgs a) {
    pdl_wait();
    pdl_launch_dependents();
    const int n = *a.d_n;
    const int nq = a.queue ? (int)*a.queue_n : n;
    const GridView &g = a.g;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nq; t += gridDim.x * blockDim.x) {
        const int i = a.queue ? (int)__ldg(a.queue + t)
                              : __float_as_int(__ldg(g.spos + (size_t)(g.levels - 1) * g.cap + t).w);
        const int *lst = a.nbr_t + (size_t)t * kMaxK;
        int ids[K];
#pragma unroll
        for (int j = 0; j < K; ++j) ids[j] = j < a.k ? __ldg(lst + j) : -1;
        finish_query<K>(a, n, i, __ldg(a.pos + i), a.k, ids);
    }
}

// ---------------------------------------------------------------------------------------------
// Image-window kNN for depth-frame clouds (A1 output: point i <-> lattice pixel (u/s, v/s) of the
// sampled depth image, pos.w = v*W + u).  A ball B(q, rho) with q_z > rho projects inside the
// pixel box |u - u_q| <= fx rho (q_z + |q_x|) / (q_z (q_z - rho)) (and likewise in v), because
// |x/z - x_q/z_q| = |(x - x_q) z_q - x_q (z - z_q)| / (z z_q) <= rho (z_q + |x_q|) / ((z_q - rho) z_q).
// Sampled pixels differ by multiples of s, so when that bound is < (M+1) s every point within rho
// of q lies in the (2M+1)^2 lattice window around q's pixel: the window is an exact candidate set
// for any query whose k-th radius (with rounding margins) passes the bound.
//   * a block stages a 32x4 tile of lattice pixels plus an M-pixel halo (the points, by a
//     lattice -> point map) in shared memory; a thread owns one pixel's query and reads its
//     window as a stencil — no hashing, no divergence;
//   * exact, insertion-free selection in two passes: pass 1 builds a per-thread histogram of
//     the window's keys over 32 quarter-octave buckets (float exponent + 2 mantissa bits, offset
//     so that bucket 16 is (2 * point spacing)^2; shared-memory atomics, one column per thread)
//     and finds b*, the first bucket whose cumulative count reaches k; pass 2 collects the
//     m = cum(b*) <= 32 candidates at or below b* and sorts them by (key, index) with a Batcher
//     network in registers — the first k are the k nearest of the window;
//   * queries that fail the projection certificate (k-th radius too large for the window: depth
//     edges, grazing surfaces, image periphery), or whose m exceeds the list, go to a queue that
//     the grid search finishes (the hash is only built for them).
// 16 byte counters in two registers (buckets 0-7, 8-15): add one to bucket b
struct Hist16 {
    unsigned long long lo = 0ull, hi = 0ull;
    __device__ __forceinline__ void add(int b) {
        const unsigned long long one = 1ull << (8 * (b & 7));
        if (b < 8) lo += one; else hi += one;
    }
    // first bucket whose cumulative count reaches k (16 if none); *below = the count before it
    __device__ __forceinline__ int select(int k, int &below) const {
        constexpr unsigned long long C = 0x0101010101010101ull;  // byte prefix sums (< 256: no carries)
        const unsigned long long pl = lo * C;
        const unsigned long long ph = hi * C + (pl >> 56) * C;
        const uint32_t w0 = (uint32_t)pl, w1 = (uint32_t)(pl >> 32), w2 = (uint32_t)ph, w3 = (uint32_t)(ph >> 32);
        const uint32_t kk = (uint32_t)k * 0x01010101u;
        const int ge = __popc(__vcmpgeu4(w0, kk)) + __popc(__vcmpgeu4(w1, kk)) + __popc(__vcmpgeu4(w2, kk)) +
                       __popc(__vcmpgeu4(w3, kk));
        const int bs = 16 - ge / 8;  // prefix sums are monotone: the bytes >= k are a suffix
        const int bb = bs - 1;
        const uint32_t wd = bb < 4 ? w0 : (bb < 8 ? w1 : (bb < 12 ? w2 : w3));
        below = bs == 0 ? 0 : (int)((wd >> (8 * (bb & 3))) & 0xFFu);
        return bs;
    }
};
#ifndef GSICP_IMG_SUBRANK
#define GSICP_IMG_SUBRANK 1  // boundary-group rank within a 1/32-octave sub-bucket
#endif
constexpr int kImgTX = 32, kImgTY = 4, kImgThreads = kImgTX * kImgTY;
constexpr int kImgList = 32;
constexpr int kImgBuckets = 32;
constexpr int kImgBucketRef = 16;  // bucket of key = (2 * spacing)^2
constexpr float kImgFar = 1e30f;   // empty lattice pixel: keys overflow to +inf
// image counters (zeroed by k_img_map_clear): window queue, warp-search work, map conflict flag,
// hash queue (what the wide window could not certify), wide-pass work, hash point count
constexpr int kImgCtrQueue = 0, kImgCtrWork = 1, kImgCtrBad = 2, kImgCtrQueue2 = 3,
              kImgCtrHashN = 5, kImgCtrHashQ = 6, kImgCtrQueue3 = 7, kImgCounters = 8;
constexpr uint32_t kBruteMax = 256;  // a last queue up to this size is searched by brute force
constexpr int kImgWideM = 12;  // half-width of the wide window (warp per query)

struct ImgArgs {
    int32_t *map;  // [Hs][Ws] point index of each lattice pixel, -1 if none
    int map_given;  // the map came from A1 (gsicp_backproject_lattice): not rebuilt here
    uint32_t *queue2;
    int H, W, Hs, Ws, stride;
    float fx, fy;
    uint32_t *ctr;
    uint32_t *queue;
};

__global__ void k_img_map_clear(ImgArgs im, int clear_map) {
    pdl_wait();
    pdl_launch_dependents();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (clear_map && j < im.Hs * im.Ws) im.map[j] = -1;
    if (j < kImgCounters) im.ctr[j] = 0u;
}

// lattice -> point map; a point whose pixel id is not a lattice pixel of this image, or two
// points on one pixel, flag the cloud as not a depth-frame cloud (then every query is queued)
__global__ void k_img_map_fill(ImgArgs im, const float4 *__restrict__ pos, const int32_t *__restrict__ d_n) {
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= *d_n) return;
    const int pix = __float_as_int(__ldg(pos + i).w);
    const int v = pix / im.W, u = pix - v * im.W;
    bool ok = pix >= 0 && v < im.H && u % im.stride == 0 && v % im.stride == 0;
    if (ok) ok = atomicCAS(im.map + (v / im.stride) * im.Ws + u / im.stride, -1, i) == -1;
    if (!ok) {
        atomicExch(im.ctr + kImgCtrBad, 1u);
        im.queue[atomicAdd(im.ctr + kImgCtrQueue, 1u)] = (uint32_t)i;
    }
}

// Largest |x'/z' - x/z| over the points (x', z') of the disk of radius rho around (x, z) in the
// xz-plane (the projection of the 3-D ball on it), +inf if the disk reaches z <= 0: the disk spans
// the view angles alpha +- beta, tan(alpha) = x/z, sin(beta) = rho/|(x, z)|, and tan is increasing.
__device__ __forceinline__ double proj_extent(double x, double z, double rho) {
    const double d = sqrt(x * x + z * z);
    if (!(z > 0.0) || !(rho < d)) return INFINITY;
    const double sb = rho / d, cb = sqrt(fmax(1.0 - sb * sb, 0.0));
    const double sa = x / d, ca = z / d;
    // tan(alpha +- beta) = (sa cb +- ca sb) / (ca cb -+ sa sb); a non-positive denominator means
    // the disk reaches the image plane's horizon
    const double dp = ca * cb - sa * sb, dm = ca * cb + sa * sb;
    if (!(dp > 0.0) || !(dm > 0.0)) return INFINITY;
    const double t0 = x / z, tp = (sa * cb + ca * sb) / dp, tm = (sa * cb - ca * sb) / dm;
    return fmax(tp - t0, t0 - tm) * (1.0 + 1e-9) + 1e-12;
}

constexpr int kImgM = 5;  // tile-kernel window half-width (lattice pixels)

// certificate: every point within sqrt(key) of q lies inside the lattice window of half-width w
__device__ __forceinline__ bool img_cert(const ImgArgs &im, float4 q, float key, int w) {
    const double rho = sqrt((double)key) * (1.0 + 1e-5) + 1e-9;
    const double bu = proj_extent((double)q.x, (double)q.z, rho) * (double)im.fx;
    const double bv = proj_extent((double)q.y, (double)q.z, rho) * (double)im.fy;
    const double win = (double)((w + 1) * im.stride) - 1e-3;
    return bu < win && bv < win;
}

template <int K, int M>
__global__ void __launch_bounds__(kImgThreads, 4) k_knn_image(KnnArgs a, ImgArgs im) {
    pdl_wait();
    pdl_launch_dependents();
    constexpr int SW = kImgTX + 2 * M, SH = kImgTY + 2 * M;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4(*tile)[SW] = reinterpret_cast<float4(*)[SW]>(smem_raw);
    uint32_t(*hist)[kImgThreads] = reinterpret_cast<uint32_t(*)[kImgThreads]>(smem_raw + sizeof(float4) * SW * SH);
    unsigned long long(*list)[kImgThreads] = reinterpret_cast<unsigned long long(*)[kImgThreads]>(
        smem_raw + sizeof(float4) * SW * SH + sizeof(uint32_t) * (kImgBuckets / 2) * kImgThreads);
    const int tid = threadIdx.x;
    const int gx0 = blockIdx.x * kImgTX - M, gy0 = blockIdx.y * kImgTY - M;
    const bool bad = __ldg(im.ctr + kImgCtrBad) != 0u;
    for (int t = tid; t < SW * SH; t += kImgThreads) {
        const int ty = t / SW, tx = t - ty * SW;
        const int gx = gx0 + tx, gy = gy0 + ty;
        float4 p = make_float4(kImgFar, kImgFar, kImgFar, __int_as_float(-1));
        if (gx >= 0 && gx < im.Ws && gy >= 0 && gy < im.Hs) {
            const int i = __ldg(im.map + gy * im.Ws + gx);
            if (i >= 0) {
                p = __ldg(a.pos + i);
                p.w = __int_as_float(i);
            }
        }
        tile[ty][tx] = p;
    }
#pragma unroll
    for (int b = 0; b < kImgBuckets / 2; ++b) hist[b][tid] = 0u;
    __syncthreads();
    const int lx = tid % kImgTX, ly = tid / kImgTX;
    const float4 q = tile[ly + M][lx + M];
    const int i = __float_as_int(q.w);
    if (i < 0) return;  // no point on this pixel (no block-wide sync follows)
    if (bad) {
        im.queue[atomicAdd(im.ctr + kImgCtrQueue, 1u)] = (uint32_t)i;
        return;
    }
    const int k = a.k;
    // bucket kImgBucketRef <-> key (2 * spacing)^2, spacing = s z / fx
    const float sp = 2.f * (float)im.stride * q.z / im.fx;
    const int base = (int)(__float_as_uint(fmaxf(sp * sp, 1e-30f)) >> 21) - kImgBucketRef;
    uint32_t *hcol = &hist[0][tid];
    // ---- pass 1: histogram of the window's keys (rows not unrolled: keeps the code in i-cache)
#pragma unroll 1
    for (int dy = 0; dy <= 2 * M; ++dy) {
        const float4 *row = &tile[ly + dy][lx];
#pragma unroll
        for (int dx = 0; dx <= 2 * M; ++dx) {
            const float4 P = row[dx];
            const float key = canon_key(q.x, q.y, q.z, P.x, P.y, P.z);
            const int bk = min(max((int)(__float_as_uint(key) >> 21) - base, 0), kImgBuckets - 1);
            atomicAdd(hcol + (bk >> 1) * kImgThreads, 1u << ((bk & 1) * 16));
        }
    }
    int bstar = -1;
    uint32_t cum = 0, m = 0, below = 0;
#pragma unroll
    for (int b = 0; b < kImgBuckets / 2; ++b) {
        const uint32_t wd = hist[b][tid];
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
            const uint32_t c = (wd >> (16 * hb)) & 0xFFFFu;
            if (bstar < 0 && cum + c >= (uint32_t)k) {
                bstar = 2 * b + hb;
                below = cum;
                m = cum + c;
            }
            cum += c;
        }
    }
    bool ok = bstar >= 0 && m <= (uint32_t)kImgList;
    if (ok) {
        // ---- pass 2: the candidates below b*'s lower edge (shrunk by the binary64 resolution
        // band) are all among the k nearest ("sure", from the bottom of the list); those
        // up to b*'s upper edge (widened by the band) form the boundary group (from the top); in
        // stencil order
        const float lo_edge = __uint_as_float((uint32_t)(base + bstar) << 21);
        const float lo_lim = bstar > 0 ? band_lo(lo_edge) : -1.f;
        const float lim = bstar >= kImgBuckets - 1 ? INFINITY : band_hi(__uint_as_float((uint32_t)(base + bstar + 1) << 21));
        int nlo = 0, nbd = 0;
#pragma unroll 1
        for (int dy = 0; dy <= 2 * M; ++dy) {
            const float4 *row = &tile[ly + dy][lx];
#pragma unroll
            for (int dx = 0; dx <= 2 * M; ++dx) {
                const float4 P = row[dx];
                const float key = canon_key(q.x, q.y, q.z, P.x, P.y, P.z);
                if (key <= lim && key < INFINITY) {
                    const unsigned long long e = pack_ki(key, (uint32_t)__float_as_int(P.w));
                    const bool lo = key < lo_lim;
                    const int slot = lo ? nlo : kImgList - 1 - nbd;  // boundary entries from the top
                    if (nlo + nbd < kImgList) list[slot][tid] = e;
                    nlo += lo ? 1 : 0;
                    nbd += lo ? 0 : 1;
                }
            }
        }
        ok = nlo + nbd <= kImgList && nlo < k && nlo + nbd >= k;
        if (ok) {
            // t = the k-th smallest key32 = the (k - nlo)-th of the boundary group (rank by packed
            // (key32, index)); then over all filled slots: key32 < band_lo(t) is in, > band_hi(t)
            // out, and a tie band around t is ranked by (key64, index).  Masks are over list slots
            // (filled: [0, nlo) and [kImgList - nbd, kImgList)).
            const int r = k - nlo;
            float t = 0.f;
#if GSICP_IMG_SUBRANK
            // the boundary group split by the next 3 mantissa bits (sub-buckets monotone in the
            // key; 0 / 9: band entries below / above b*): the r-th key lies in the first sub-bucket
            // whose cumulative count reaches r, and is ranked among that sub-bucket's few entries
            const int sub0 = ((base + bstar) << 3) - 1;
            auto sub_of = [&](float key) { return min(max((int)(__float_as_uint(key) >> 18) - sub0, 0), 9); };
            Hist16 hs;
            for (int j = kImgList - nbd; j < kImgList; ++j) hs.add(sub_of(ki_key(list[j][tid])));
            int sbelow;
            const int sb = hs.select(r, sbelow);
            const int r2 = r - sbelow;
            for (int j = kImgList - nbd; j < kImgList; ++j) {
                const unsigned long long e = list[j][tid];
                if (sub_of(ki_key(e)) != sb) continue;
                int rank = 0;
                for (int l = kImgList - nbd; l < kImgList; ++l) {
                    const unsigned long long o = list[l][tid];
                    rank += (o < e && sub_of(ki_key(o)) == sb) ? 1 : 0;
                }
                if (rank == r2 - 1) t = ki_key(e);
            }
#else
            for (int j = kImgList - nbd; j < kImgList; ++j) {
                const unsigned long long e = list[j][tid];
                int rank = 0;
                for (int l = kImgList - nbd; l < kImgList; ++l) rank += list[l][tid] < e ? 1 : 0;
                if (rank == r - 1) t = ki_key(e);
            }
#endif
            const float blo = band_lo(t), bhi = band_hi(t);
            const uint32_t filled = (nlo >= 32 ? ~0u : ((1u << nlo) - 1u)) | (nbd == 0 ? 0u : ~0u << (kImgList - nbd));
            uint32_t sel = 0u, band = 0u;
            for (uint32_t f = filled; f; f &= f - 1) {
                const int j = __ffs(f) - 1;
                const float kj = ki_key(list[j][tid]);
                sel |= (kj < blo ? 1u : 0u) << j;
                band |= (kj >= blo && kj <= bhi ? 1u : 0u) << j;
            }
            const int need = k - __popc(sel);
            const double qx = q.x, qy = q.y, qz = q.z;
            // key64 of the entry in slot j, and its rank by (key64, index) among the slots of mask
            auto key_of = [&](int j, uint32_t &id) {
                id = ki_idx(list[j][tid]);
                const float4 p = __ldg(a.pos + id);
                return key64(qx, qy, qz, p.x, p.y, p.z);
            };
            auto rank_in = [&](int j, uint32_t mask) {
                uint32_t ij;
                const double kj = key_of(j, ij);
                int rank = 0;
                for (uint32_t bl = mask; bl; bl &= bl - 1) {
                    uint32_t il;
                    const double kl = key_of(__ffs(bl) - 1, il);
                    rank += (kl < kj || (kl == kj && il < ij)) ? 1 : 0;
                }
                return rank;
            };
            if (__popc(band) == need) {
                sel |= band;
            } else {  // equal-key32 ties across the band
                uint32_t add = 0u;
                for (uint32_t bj = band; bj; bj &= bj - 1)
                    if (rank_in(__ffs(bj) - 1, band) < need) add |= 1u << (__ffs(bj) - 1);
                sel |= add;
            }
            ok = img_cert(im, q, bhi, M);
            if (a.debug) a.debug[i] = make_int4(ok ? -1 : -2, M, (int)m, 0);
            if (ok) {
                if (a.knn_idx)  // the k nearest in (key64, index) order (API output only)
                    for (uint32_t f = sel; f; f &= f - 1)
                        a.knn_idx[(size_t)i * k + rank_in(__ffs(f) - 1, sel)] = (int32_t)ki_idx(list[__ffs(f) - 1][tid]);
                // moments over the selected slots in slot order (deterministic), then the A4 epilogue
                double s1[3] = {0, 0, 0}, s2[6] = {0, 0, 0, 0, 0, 0};
                for (uint32_t f = sel; f; f &= f - 1) {
                    const float4 p = __ldg(a.pos + ki_idx(list[__ffs(f) - 1][tid]));
                    const double d0 = (double)p.x - (double)q.x, d1 = (double)p.y - (double)q.y,
                                 d2 = (double)p.z - (double)q.z;
                    s1[0] += d0;
                    s1[1] += d1;
                    s1[2] += d2;
                    s2[0] += d0 * d0;
                    s2[1] += d0 * d1;
                    s2[2] += d0 * d2;
                    s2[3] += d1 * d1;
                    s2[4] += d1 * d2;
                    s2[5] += d2 * d2;
                }
                finish_moments(a, *a.d_n, i, s1, s2, __popc(sel));
            }
        }
    }
    if (!ok) im.queue[atomicAdd(im.ctr + kImgCtrQueue, 1u)] = (uint32_t)i;
}

// Wide window for the queries the tile kernel could not certify: warp per query, lanes split the
// (2 kImgWideM + 1)^2 window (lattice -> point map and positions read through L1/L2), per-lane
// histogram columns summed across the warp, the m <= 32 candidates at or below b* compacted one
// per lane and sorted by a warp bitonic network; same certificate.  Misses go to the hash queue.
// One wide-window attempt of half-width M2 for query q (pixel us, vs) by the calling warp.
// CACHE: the lane's window keys stay in registers across the histogram passes (small windows);
// otherwise they are recomputed from the map each pass.  Returns true (and finishes the query) if
// the k nearest of the window certify.  `fail` = 1: certificate failed (try a wider window),
// 2: no usable boundary bucket (too few points, or more than 64 at or below b*).
template <int K, int M2, bool CACHE>
__device__ bool wide_attempt(const KnnArgs &a, const ImgArgs &im, int i, float4 q, int us, int vs, int lane,
                             uint32_t (*hist)[32], unsigned long long *lst, int &fail) {
    constexpr int SIDE = 2 * M2 + 1, CELLS = SIDE * SIDE, PER = (CELLS + 31) / 32;
    const int k = a.k;
    int cidx[CACHE ? PER : 1];
    float ckey[CACHE ? PER : 1];
    auto cell_key_of = [&](int j, int &idx) -> float {
        const int c = lane + 32 * j;
        const int x = us + c % SIDE - M2, y = vs + c / SIDE - M2;
        idx = (c < CELLS && x >= 0 && x < im.Ws && y >= 0 && y < im.Hs) ? __ldg(im.map + y * im.Ws + x) : -1;
        if (idx < 0) return INFINITY;
        const float4 P = __ldg(a.pos + idx);
        return canon_key(q.x, q.y, q.z, P.x, P.y, P.z);
    };
    if (CACHE) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int c = lane + 32 * j;
            const int x = us + c % SIDE - M2, y = vs + c / SIDE - M2;
            cidx[j] = (c < CELLS && x >= 0 && x < im.Ws && y >= 0 && y < im.Hs) ? __ldg(im.map + y * im.Ws + x) : -1;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            ckey[j] = INFINITY;
            if (cidx[j] >= 0) {
                const float4 P = __ldg(a.pos + cidx[j]);
                ckey[j] = canon_key(q.x, q.y, q.z, P.x, P.y, P.z);
            }
        }
    }
    auto get = [&](int j, int &idx) -> float {
        if (CACHE) {
            float kk = ckey[0];
            idx = cidx[0];
#pragma unroll
            for (int r = 1; r < (CACHE ? PER : 1); ++r)
                if (r == j) {
                    kk = ckey[r];
                    idx = cidx[r];
                }
            return kk;
        }
        return cell_key_of(j, idx);
    };
    // histogram over 32 quarter-octave buckets; if the k-th falls in the open top bucket, shift
    // the scale up 16 buckets (4 octaves in key) and count again
    const float sp = 2.f * (float)im.stride * q.z / im.fx;
    int base = (int)(__float_as_uint(fmaxf(sp * sp, 1e-30f)) >> 21) - kImgBucketRef;
    int bstar = -1;
    uint32_t m = 0;
    for (int attempt = 0; attempt < 3; ++attempt) {
#pragma unroll
        for (int b = 0; b < kImgBuckets / 2; ++b) hist[b][lane] = 0u;
#pragma unroll(CACHE ? PER : 4)
        for (int j = 0; j < PER; ++j) {
            int idx;
            const float key = get(j, idx);
            if (key < INFINITY) {
                const int bk = min(max((int)(__float_as_uint(key) >> 21) - base, 0), kImgBuckets - 1);
                atomicAdd(&hist[bk >> 1][lane], 1u << ((bk & 1) * 16));
            }
        }
        __syncwarp();
        bstar = -1;
        uint32_t cum = 0;
#pragma unroll
        for (int b = 0; b < kImgBuckets / 2; ++b) {
            const uint32_t wd = __reduce_add_sync(kFull, hist[b][lane]);
#pragma unroll
            for (int hb = 0; hb < 2; ++hb) {
                cum += (wd >> (16 * hb)) & 0xFFFFu;
                if (bstar < 0 && cum >= (uint32_t)k) {
                    bstar = 2 * b + hb;
                    m = cum;
                }
            }
        }
        __syncwarp();
        if (bstar != kImgBuckets - 1) break;
        base += 16;
    }
    if (bstar < 0 || m > 64u) {
        fail = 2;
        return false;
    }
    // the m <= 64 candidates at or below b* (its upper edge widened by the binary64 resolution
    // band), two per lane, sorted: the 32 smallest end up in order across the lanes (lane j: j-th)
    const float lim = bstar >= kImgBuckets - 1 ? INFINITY : band_hi(__uint_as_float((uint32_t)(base + bstar + 1) << 21));
    int nl = 0;
#pragma unroll(CACHE ? PER : 4)
    for (int j = 0; j < PER; ++j) {
        int idx;
        const float key = get(j, idx);
        const bool take = key <= lim && key < INFINITY;
        const unsigned bb = __ballot_sync(kFull, take);
        const int slot = nl + __popc(bb & ((1u << lane) - 1u));
        if (take && slot < 64) lst[slot] = pack_ki(key, (uint32_t)idx);
        nl += __popc(bb);
    }
    __syncwarp();
    if (nl < k || nl > 64) {
        fail = 2;
        return false;
    }
    unsigned long long A = lane < nl ? lst[lane] : kEmptyKey;
    unsigned long long B = lane + 32 < nl ? lst[lane + 32] : kEmptyKey;
    __syncwarp();
    A = WarpTopK<32>::sort_w<32>(A, lane);
    if (nl > 32) {
        B = WarpTopK<32>::sort_w<32>(B, lane);
        const unsigned long long Br = shfl_u64(B, 31 - lane);  // descending
        A = WarpTopK<32>::merge32(A < Br ? A : Br, lane);      // the 32 smallest, a bitonic merge
    }
    const float t = ki_key(shfl_u64(A, k - 1));
    if (!img_cert(im, q, band_hi(t), M2)) {
        fail = 1;
        return false;
    }
    int outpos = -1;
    const bool ok = a.knn_idx ? warp_exact_select<true>(A, k, nl > 32, q.x, q.y, q.z, a.pos, lane, outpos)
                              : warp_exact_select<false>(A, k, nl > 32, q.x, q.y, q.z, a.pos, lane, outpos);
    if (!ok) {
        fail = 2;
        return false;
    }
    if (a.knn_idx && outpos >= 0) a.knn_idx[(size_t)i * k + outpos] = (int32_t)ki_idx(A);
    int ids[K];
    collect_ids<K>(outpos, ki_idx(A), lane, ids);
    if (a.debug && lane == 0) a.debug[i] = make_int4(-3, M2, (int)m, 0);
    if (lane == 0) finish_query<K>(a, *a.d_n, i, q, k, ids);
    return true;
}

// Wide window for the queries the tile kernel could not certify: warp per query, half-width
// kImgWideM (keys cached in registers).  Misses go to the last queue.
template <int K>
__global__ void __launch_bounds__(128) k_knn_image_wide(KnnArgs a, ImgArgs im) {
    pdl_wait();
    pdl_launch_dependents();
    __shared__ uint32_t hist[4][kImgBuckets / 2][32];
    __shared__ unsigned long long lst[4][64];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nq = (int)*(im.ctr + kImgCtrQueue);
    const bool bad = __ldg(im.ctr + kImgCtrBad) != 0u;
    // static warp-strided assignment (a shared work counter serialises thousands of warps on
    // one atomic for a queue of ~1e3)
    const int gw = (int)(blockIdx.x * 4 + wib), nw = (int)gridDim.x * 4;
    for (int t = gw; t < nq; t += nw) {
        const int i = (int)__ldg(im.queue + t);
        const float4 q = __ldg(a.pos + i);
        bool ok = false;
        if (!bad) {
            const int pix = __float_as_int(q.w);
            const int v = pix / im.W, u = pix - v * im.W;
            const int us = u / im.stride, vs = v / im.stride;
            int fail = 0;
            ok = wide_attempt<K, kImgWideM, true>(a, im, i, q, us, vs, lane, hist[wib], lst[wib], fail);
            if (!ok && a.debug && lane == 0) a.debug[i] = make_int4(fail == 1 ? -4 : -5, 0, 0, 0);
        }
        if (!ok && lane == 0) im.queue2[atomicAdd(im.ctr + kImgCtrQueue2, 1u)] = (uint32_t)i;
        __syncwarp();
    }
}

// The last queue: up to kBruteMax queries are searched by brute force over the whole cloud
// (exact by definition — no certificate); a longer queue (e.g. a cloud that is not a depth frame)
// goes to the hash search.  Brute force: a 1024-bin histogram of all keys (octave x 32
// sub-buckets) gives the boundary bin, a second pass collects the keys below it and the bin's
// own, and the k smallest of those are the k nearest.
constexpr int kBruteThreads = 512;

// A cluster of kBruteCluster CTAs per query (thread-block cluster): the CTAs split the cloud and
// merge their histograms / candidate lists through distributed shared memory.
constexpr int kBruteCluster = 8;

// key -> one of 1024 bins: 32 octaves of the key (2^-20 .. 2^11 m^2, the end octaves open) x 32
// sub-buckets (top 5 mantissa bits); bins are ordered like the keys
__device__ __forceinline__ int brute_bin(uint32_t kb) {
    const int o = (int)(kb >> 23) - (127 - 20);
    if (o <= 0) return 0;
    if (o >= 31) return 1023;
    return o * 32 + (int)((kb >> 18) & 31u);
}
// key range [lo, hi) of a bin (as key bits)
__device__ __forceinline__ void brute_bin_range(int bin, uint32_t &lo, uint32_t &hi) {
    if (bin == 0) {
        lo = 0u;
        hi = (uint32_t)(127 - 20 + 1) << 23;
    } else if (bin == 1023) {
        lo = (uint32_t)(127 - 20 + 31) << 23;
        hi = 0x7F800000u;
    } else {
        lo = ((uint32_t)(bin / 32 + 127 - 20) << 23) | ((uint32_t)(bin & 31) << 18);
        hi = lo + (1u << 18);
    }
}

template <int K>
__global__ void __cluster_dims__(kBruteCluster, 1, 1) __launch_bounds__(kBruteThreads, 2)
    k_knn_brute(KnnArgs a, ImgArgs im) {
    pdl_wait();
    pdl_launch_dependents();
    __shared__ uint32_t bins[1024], gbins[1024];
    __shared__ unsigned long long lst[64];
    __shared__ int s_nl, s_nb, s_bin;
    __shared__ uint32_t s_below, s_m;
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t nq = *(im.ctr + kImgCtrQueue2);
    if (nq == 0u || nq > kBruteMax) return;  // uniform over the grid: no cluster barrier is skipped alone
    const int crank = (int)cl.block_rank();
    const int n = *a.d_n, k = a.k, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j0 = crank * kBruteThreads + tid, js = kBruteCluster * kBruteThreads;
    const uint32_t nclusters = gridDim.x / kBruteCluster;
    for (uint32_t t = blockIdx.x / kBruteCluster; t < nq; t += nclusters) {
        const int i = (int)__ldg(im.queue2 + t);
        const float4 q = __ldg(a.pos + i);
        // pass 1: 1024-bin histogram of this CTA's share of the keys
        for (int b = tid; b < 1024; b += kBruteThreads) bins[b] = 0u;
        __syncthreads();
#pragma unroll 4
        for (int j = j0; j < n; j += js) {
            const float4 P = __ldg(a.pos + j);
            atomicAdd(&bins[brute_bin(__float_as_uint(canon_key(q.x, q.y, q.z, P.x, P.y, P.z)))], 1u);
        }
        cl.sync();
        // the cluster's histogram (every CTA sums it: two bins per thread), then the boundary bin
        for (int b = tid; b < 1024; b += kBruteThreads) {
            uint32_t c = 0;
#pragma unroll
            for (int r = 0; r < kBruteCluster; ++r) c += cl.map_shared_rank(bins, r)[b];
            gbins[b] = c;
        }
        __syncthreads();
        if (warp == 0) {  // lane l owns bins [32 l, 32 l + 32): warp prefix of the lane sums
            uint32_t sl = 0;
            for (int b = 0; b < 32; ++b) sl += gbins[32 * lane + b];
            uint32_t incl = sl;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t excl = incl - sl;
            const unsigned hit = __ballot_sync(kFull, incl >= (uint32_t)k);
            // exactly one lane writes s_bin / s_below / s_m: the first lane whose prefix reaches k
            // (its own 32 bins then contain the boundary bin), else lane 31
            if (hit) {
                const int L = __ffs(hit) - 1;
                if (lane == L) {
                    uint32_t cum = excl;
                    for (int b = 0; b < 32; ++b) {
                        const uint32_t c = gbins[32 * lane + b];
                        if (cum + c >= (uint32_t)k) {
                            s_bin = 32 * lane + b;
                            s_below = cum;
                            s_m = cum + c;
                            break;
                        }
                        cum += c;
                    }
                }
            } else if (lane == 31) {  // fewer than k points: all of them
                s_bin = 1024;
                s_below = 0u;
                s_m = incl;
            }
        }
        __syncthreads();
        const int bin = s_bin;
        const uint32_t below = s_below, m = s_m;
        uint32_t klo = 0u, khi = 0x7F800000u;  // boundary range [klo, khi) of key bits
        if (bin < 1024) brute_bin_range(bin, klo, khi);
        (void)below;
        (void)m;
        // pass 2: keys below the boundary bin (shrunk by the binary64 resolution band) are among
        // the k nearest; the boundary group runs up to the bin's top widened by the band
        const float lo_lim = band_lo(__uint_as_float(klo));
        const float hi_lim = khi >= 0x7F800000u ? INFINITY : band_hi(__uint_as_float(khi));
        if (tid == 0) {
            s_nl = 0;
            s_nb = 0;
        }
        __syncthreads();
#pragma unroll 4
        for (int j = j0; j < n; j += js) {
            const float4 P = __ldg(a.pos + j);
            const float key = canon_key(q.x, q.y, q.z, P.x, P.y, P.z);
            if (key <= hi_lim && key < INFINITY) {
                const bool lo = key < lo_lim;
                const int slot = atomicAdd(lo ? &s_nl : &s_nb, 1);
                if (slot < 32) lst[(lo ? 0 : 32) + slot] = pack_ki(key, (uint32_t)j);
            }
        }
        cl.sync();
        if (crank == 0 && warp == 0) {
            // gather the CTAs' lists (at most 32 + 32 entries in all): lane j fetches entry j
            unsigned long long L = kEmptyKey, Bd = kEmptyKey;
            int nl = 0, nb = 0;
            bool over = false;
            for (int r = 0; r < kBruteCluster; ++r) {
                const int cl_l = *cl.map_shared_rank(&s_nl, r), cl_b = *cl.map_shared_rank(&s_nb, r);
                over = over || cl_l > 32 || cl_b > 32;
                const unsigned long long *rl = cl.map_shared_rank(lst, r);
                if (lane >= nl && lane < nl + cl_l) L = rl[lane - nl];
                if (lane >= nb && lane < nb + cl_b) Bd = rl[32 + lane - nb];
                nl += cl_l;
                nb += cl_b;
            }
            over = over || nl > 32 || nb > 32;
            int outpos = -1;
            unsigned long long A = kEmptyKey;
            if (!over) {
                L = WarpTopK<32>::sort_w<32>(L, lane);
                Bd = WarpTopK<32>::sort_w<32>(Bd, lane);
                const unsigned long long Bsh = shfl_u64(Bd, (lane - nl) & 31);
                A = lane < nl ? L : Bsh;  // every sure key32 < every boundary key32
                over = !(a.knn_idx ? warp_exact_select<true>(A, k, nl + nb > 32, q.x, q.y, q.z, a.pos, lane, outpos)
                                   : warp_exact_select<false>(A, k, nl + nb > 32, q.x, q.y, q.z, a.pos, lane, outpos));
            }
            if (over) {  // > 32 near-equal keys at the boundary: hand over to the hash
                if (lane == 0) im.queue[atomicAdd(im.ctr + kImgCtrQueue3, 1u)] = (uint32_t)i;
            } else {
                if (a.knn_idx) {
                    if (outpos >= 0) a.knn_idx[(size_t)i * k + outpos] = (int32_t)ki_idx(A);
                    const int cnt = __popc(__ballot_sync(kFull, outpos >= 0));
                    if (lane >= cnt && lane < k) a.knn_idx[(size_t)i * k + lane] = -1;
                }
                int ids[K];
                collect_ids<K>(outpos, ki_idx(A), lane, ids);
                if (a.debug && lane == 0) a.debug[i] = make_int4(-6, 0, (int)m, 0);
                if (lane == 0) finish_query<K>(a, n, i, q, k, ids);
            }
        }
        cl.sync();  // the lists are read remotely before the next query overwrites them
    }
}

// the hash path takes the last queue when it is longer than kBruteMax, else whatever brute force
// handed over (moved to the front of queue 2)
__global__ void k_img_hash_n(ImgArgs im, const int32_t *__restrict__ d_n, cudaGraphConditionalHandle cond,
                             int use_cond) {
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t q2 = im.ctr[kImgCtrQueue2], q3 = im.ctr[kImgCtrQueue3];
    uint32_t hq = 0u;
    if (q2 > kBruteMax) {
        hq = q2;
    } else if (q3 > 0u) {
        for (uint32_t j = 0; j < q3; ++j) im.queue2[j] = im.queue[j];
        hq = q3;
    }
    im.ctr[kImgCtrHashN] = hq ? (uint32_t)*d_n : 0u;
    im.ctr[kImgCtrHashQ] = hq;
    if (use_cond) cudaGraphSetConditional(cond, hq ? 1u : 0u);  // the graph runs the hash tail only if needed
}

// ---------------------------------------------------------------------------------------------
// Brick kNN for general clouds (maps, voxel clouds; A3+A4 of gsicp_covariances): the grid's
// level-0 cells are "bricks" of edge H (~3.7 point spacings).  A brick's candidates are the
// points of its 27-brick neighbourhood inside the brick's box expanded by R = 0.95 H; the result
// is exact when the query's k-th ball lies inside that box (every point within it was staged).
// A warp takes a contiguous range of the brick list and stages bricks back to back in shared memory
// while their queries fit one 32-lane round (bricks hold ~10 points; a group of ~3 fills the warp), then
// runs the round: a lane per query, each scanning its own brick's candidates (a few distinct
// shared-memory addresses per load), with ONE pass of selection (each key computed once).  The
// screen key here is key32 with its 9 low mantissa bits cleared (key32t: within 2^-14 below key32,
// so |key32t - key64| <= 6.2e-5 key64 and the band of §7.0 widens to kBrickBand = 2e-4); the 9
// bits carry the candidate's slot.  A lane appends every candidate with key32t <= its bound tau
// to a per-lane list (one 32-bit store); when some lane's list nears its capacity the warp
// compacts — each lane with >= k entries buckets them (quarter-octave buckets below tau or its
// largest key, byte counters in one register), takes b*, the bucket holding its k-th entry, lowers tau to
// band_hi(upper edge of b*) and drops the entries above it.  tau never falls below band_hi(k-th
// key32t of all its candidates), so at the end the list holds every candidate the exact selection
// needs: the k-th key32t t, the entries below band_lo(t), and the band resolved in binary64.
// Queries that fail the certificate (and bricks whose neighbourhood overflows the staging buffer)
// go to a queue that the warp search finishes.
#ifndef GSICP_BRICK_SUBRANK
#define GSICP_BRICK_SUBRANK 1  // boundary-bucket rank within a 1/64-octave sub-bucket
#endif
#ifndef GSICP_BRICK_TAU0
#define GSICP_BRICK_TAU0 1  // the list bound starts at the certificate's limit, not +inf
#endif
constexpr int kBrickWarps = 4;
#ifndef GSICP_BRICK_CAP
#define GSICP_BRICK_CAP 448
#endif
#ifndef GSICP_BRICK_L
#define GSICP_BRICK_L 48
#endif
#ifndef GSICP_BRICK_BPS
#define GSICP_BRICK_BPS 4
#endif
constexpr int kBrickCap = GSICP_BRICK_CAP;     // staged candidates per warp (a group of bricks, + a sentinel each)
constexpr float kBrickHalo = 0.95f;  // R / H (< 1: the box stays inside the 27 bricks with margin)
constexpr int kBrickL = GSICP_BRICK_L;        // per-lane list capacity
constexpr int kBrickLx = 32;       // list entries of the final selection (a 32-bit mask)
constexpr int kBrickU = 4;         // candidates between two capacity checks (the list keeps U free)
constexpr uint32_t kBrickSlotMask = 0x1FFu;  // staged-candidate slot in the low bits of a list entry
static_assert(kBrickCap < (int)kBrickSlotMask, "slot field");
// per warp: staged candidates, packed list, 27-brick cell table (13.6 KB: 4 blocks / SM)
constexpr int kBrickSmemPerWarp = kBrickCap * 16 + kBrickL * 32 * 4 + 32 * 8;
constexpr int kBrickBlocksPerSm = GSICP_BRICK_BPS;
constexpr uint32_t kBrickKeyMask = ~kBrickSlotMask;
constexpr float kBrickBand = 2e-4f;  // > 3 x (11 u + 2^-14)
__device__ __forceinline__ float brick_band_hi(float t) { return __fadd_ru(__fmul_ru(t, 1.f + kBrickBand), 1e-36f); }
__device__ __forceinline__ float brick_band_lo(float t) { return __fsub_rd(__fmul_rd(t, 1.f - kBrickBand), 1e-36f); }
// the 27 bricks around a brick, nearest first (own, 6 faces, 12 edges, 8 corners): early
// candidates are close, so the bounds tighten sooner
__constant__ int8_t c_brick_nb[27][3] = {
    {0, 0, 0}, {-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1},
    {-1, -1, 0}, {-1, 1, 0}, {1, -1, 0}, {1, 1, 0}, {-1, 0, -1}, {-1, 0, 1}, {1, 0, -1}, {1, 0, 1},
    {0, -1, -1}, {0, -1, 1}, {0, 1, -1}, {0, 1, 1},
    {-1, -1, -1}, {-1, -1, 1}, {-1, 1, -1}, {-1, 1, 1}, {1, -1, -1}, {1, -1, 1}, {1, 1, -1}, {1, 1, 1}};

// The brick kernel's screen key: the binary32 squared distance with fused multiply-adds.  Every
// operand is positive, so its relative error is <= 5u like canon_key's (DESIGN §7.0's band bound
// holds); it is used consistently inside the kernel (scan and final ranking).
__device__ __forceinline__ float brick_key(float ax, float ay, float az, float bx, float by, float bz) {
    const float dx = ax - bx, dy = ay - by, dz = az - bz;
    return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}
// 8 byte counters in one register (the list compaction: quarter-octave buckets, 2 octaves)
struct Hist8 {
    unsigned long long c = 0ull;
    __device__ __forceinline__ void add(int b) { c += 1ull << (8 * b); }
    __device__ __forceinline__ int select(int k) const {
        const unsigned long long p = c * 0x0101010101010101ull;
        const uint32_t kk = (uint32_t)k * 0x01010101u;
        return 8 - (__popc(__vcmpgeu4((uint32_t)p, kk)) + __popc(__vcmpgeu4((uint32_t)(p >> 32), kk))) / 8;
    }
};
__device__ __forceinline__ int bucket8(uint32_t kb, uint32_t tb) {
    return min(max((int)(kb >> 21) - (int)(tb >> 21) + 7, 0), 7);
}
__device__ __forceinline__ uint32_t bucket8_edge(int b, uint32_t tb) {
    return (uint32_t)max((int)(tb >> 21) - 7 + b + 1, 1) << 21;
}
// 1/8-octave bucket of key bits kb in the 16 buckets whose top (15) holds the key bits tb
__device__ __forceinline__ int bucket16(uint32_t kb, uint32_t tb) {
    return min(max((int)(kb >> 20) - (int)(tb >> 20) + 15, 0), 15);
}
// smallest key bits above bucket b of that scale
__device__ __forceinline__ uint32_t bucket16_edge(int b, uint32_t tb) {
    return (uint32_t)max((int)(tb >> 20) - 15 + b + 1, 1) << 20;
}

struct BrickArgs {
    const uint4 *bricks;     // (start, count, key lo, key hi) of the occupied level-0 cells
    const uint32_t *n_bricks;
    uint32_t *queue;         // queries left to the warp search (input indices)
    uint32_t *queue_n;
};

template <int K, bool SORT>
__global__ void __launch_bounds__(kBrickWarps * 32, kBrickBlocksPerSm) k_knn_brick(KnnArgs a, BrickArgs b) {
    static_assert(K + kBrickU < kBrickLx, "list capacity");
    pdl_wait();
    pdl_launch_dependents();
    extern __shared__ __align__(16) unsigned char brick_smem[];  // kBrickSmemPerWarp per warp
    const GridView &g = a.g;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned char *wsm = brick_smem + (size_t)wid * kBrickSmemPerWarp;
    float4 *cand = reinterpret_cast<float4 *>(wsm);
    uint32_t(*lpk)[32] = reinterpret_cast<uint32_t(*)[32]>(wsm + kBrickCap * 16);
    uint2 *scell = reinterpret_cast<uint2 *>(wsm + kBrickCap * 16 + kBrickL * 32 * 4);
    const int k = a.k, n = *a.d_n;
    const uint32_t nb = *b.n_bricks;
    const float H = g.h0, R = kBrickHalo * g.h0;
    const float4 kSentinel = make_float4(__int_as_float(0x7fc00000), 0.f, 0.f, 0.f);  // NaN: never listed
    // a contiguous range of the brick list per warp (no work counter: a fetch would be one more
    // dependent round trip per brick), taken through a window of 32 records (one per lane): each
    // group picks, among the untaken, the first brick whose queries still fit the round (bin
    // packing: ~31 of 32 lanes busy instead of ~25 in list order); the first hash probe of the
    // next likely brick's 27 neighbour cells is issued ahead, so it overlaps the staging / round
    const uint32_t W = gridDim.x * kBrickWarps, wg = blockIdx.x * kBrickWarps + wid;
    const uint32_t p1 = (uint32_t)((unsigned long long)nb * (wg + 1) / W);
    uint32_t wb = (uint32_t)((unsigned long long)nb * wg / W);
    const uint4 zero4 = make_uint4(0u, 0u, 0u, 0u);
    auto nb_key = [&](const uint4 &r) {  // this lane's neighbour cell of brick r (own cell: lane 0)
        const unsigned long long key = ((unsigned long long)r.w << 32) | r.z;
        const int l = lane < 27 ? lane : 0;
        const int dx = c_brick_nb[l][0], dy = c_brick_nb[l][1], dz = c_brick_nb[l][2];
        return cell_key(0, (int)((key >> 40) & 0xFFFFFull) - kCoordOff + dx, (int)((key >> 20) & 0xFFFFFull) - kCoordOff + dy,
                        (int)(key & 0xFFFFFull) - kCoordOff + dz);
    };
    auto probe_first = [&](const uint4 &r) {
        return lane < 27 ? __ldg(reinterpret_cast<const uint4 *>(g.table + hash_slot(nb_key(r), g.mask))) : zero4;
    };
    auto probe_finish = [&](const uint4 &e, const uint4 &r) {  // (start, count) of the lane's cell
        if (lane >= 27) return make_uint2(0u, 0u);
        const unsigned long long want = nb_key(r);
        const unsigned long long k0 = ((unsigned long long)e.y << 32) | e.x;
        if (k0 == want) return make_uint2(e.z, e.w);
        if (k0 == kEmptyKey) return make_uint2(0u, 0u);
        return cell_lookup(g.table, g.mask, want);  // (collision: probe on; the scan restarts at the home slot)
    };
    auto wrec_of = [&](const uint4 &wr, int c) {
        return make_uint4(__shfl_sync(kFull, wr.x, c), __shfl_sync(kFull, wr.y, c), __shfl_sync(kFull, wr.z, c),
                          __shfl_sync(kFull, wr.w, c));
    };
    uint4 wrec = wb + lane < p1 ? __ldg(b.bricks + wb + lane) : zero4;
    unsigned avail = __ballot_sync(kFull, wb + lane < p1);
    uint4 probe = zero4;
    int probe_for = -1;  // window slot whose first probe is in flight
    if (avail) {
        probe_for = 0;
        probe = probe_first(wrec_of(wrec, 0));
    }
    // at least one untaken brick in the window, reloading it when used up (false: range done)
    auto ensure = [&]() {
        while (avail == 0u && wb + 32u < p1) {
            wb += 32u;
            wrec = wb + lane < p1 ? __ldg(b.bricks + wb + lane) : zero4;
            avail = __ballot_sync(kFull, wb + lane < p1);
            probe_for = -1;
        }
        return avail != 0u;
    };
    bool have_se = false;
    int se_for = -1;
    uint2 se = make_uint2(0u, 0u);
    uint32_t incl = 0u, total = 0u;
    while (ensure()) {
        // ---- a group: bricks staged back to back while their queries fit one round.  Lane j
        // keeps brick j's record: first point, first query lane, candidate offset and count, cell
        int nbr = 0, gq = 0, gnc = 0;
        uint32_t qmask = 0u;
        uint32_t my_start = 0u;
        int my_qs = 0, my_off = 0, my_nc = 0, my_c0 = 0, my_c1 = 0, my_c2 = 0;
        while (ensure()) {
            const int room = 32 - gq;
            const unsigned fit = __ballot_sync(kFull, ((avail >> lane) & 1u) && (nbr == 0 || (int)wrec.y <= room));
            if (!fit) break;
            const int c = __ffs(fit) - 1;
            const uint4 rec = wrec_of(wrec, c);
            const int cnt = (int)rec.y;
            if (!(have_se && se_for == c)) {
                // the 27 bricks (own first): (start, count) one per lane, their prefix and total
                se = probe_finish(probe_for == c ? probe : probe_first(rec), rec);
                incl = se.y;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += y;
                }
                total = __shfl_sync(kFull, incl, 31);
                have_se = true;
                se_for = c;
            }
            if (nbr > 0 && gnc + (int)total + 1 > kBrickCap) break;  // (total bounds the staged count)
            have_se = false;
            avail &= ~(1u << c);
            const unsigned long long key = ((unsigned long long)rec.w << 32) | rec.z;
            const int c0 = (int)((key >> 40) & 0xFFFFFull) - kCoordOff, c1 = (int)((key >> 20) & 0xFFFFFull) - kCoordOff,
                      c2 = (int)(key & 0xFFFFFull) - kCoordOff;
            const uint32_t excl = incl - se.y;
            const unsigned ne = __ballot_sync(kFull, se.y != 0u);
            __syncwarp();
            if (se.y) scell[__popc(ne & ((1u << lane) - 1u))] = make_uint2(se.x, excl);
            __syncwarp();
            // the next likely brick (the first untaken): its probe goes out now
            if (avail) {
                probe_for = __ffs(avail) - 1;
                probe = probe_first(wrec_of(wrec, probe_for));
            } else {
                probe_for = -1;
            }
            const float elo0 = (float)c0 * H - R, elo1 = (float)c1 * H - R, elo2 = (float)c2 * H - R;
            const float ehi0 = (float)(c0 + 1) * H + R, ehi1 = (float)(c1 + 1) * H + R, ehi2 = (float)(c2 + 1) * H + R;
            // records of the 27 cells scanned as one flattened range, 4 x 32 loads in flight at once
            constexpr int kStageB = 4;
            int nc = 0, before = 0;
            for (uint32_t rb0 = 0; rb0 < total; rb0 += 32 * kStageB) {
                float4 pv[kStageB];
#pragma unroll
                for (int u = 0; u < kStageB; ++u) {
                    const uint32_t rb = rb0 + 32u * u;
                    const bool here = se.y != 0u && excl >= rb && excl < rb + 32u;
                    const unsigned P = __reduce_or_sync(kFull, here ? 1u << (excl - rb) : 0u);
                    const uint32_t item = rb + lane;
                    pv[u] = kSentinel;
                    if (item < total) {
                        const uint2 ce = scell[before + __popc(P & (0xffffffffu >> (31 - lane))) - 1];
                        pv[u] = __ldg(g.spos + ce.x + (item - ce.y));
                    }
                    before += __popc(P);
                }
#pragma unroll
                for (int u = 0; u < kStageB; ++u) {
                    const float4 pp = pv[u];
                    const bool in = pp.x >= elo0 && pp.x <= ehi0 && pp.y >= elo1 && pp.y <= ehi1 && pp.z >= elo2 && pp.z <= ehi2;
                    const unsigned bi = __ballot_sync(kFull, in);
                    const int slot = gnc + nc + __popc(bi & ((1u << lane) - 1u));
                    if (in && slot < kBrickCap) cand[slot] = pp;
                    nc += __popc(bi);
                }
            }
            const bool over = gnc + nc + 1 > kBrickCap;  // (only a brick staged alone can overflow)
            if (!over && lane == 0) cand[gnc + nc] = kSentinel;
            if (lane == nbr) {
                my_start = rec.x;
                my_qs = gq;
                my_off = over ? -1 : gnc;
                my_nc = nc;
                my_c0 = c0;
                my_c1 = c1;
                my_c2 = c2;
            }
            if (gq < 32) qmask |= 1u << gq;
            gq += cnt;
            gnc += over ? 0 : nc + 1;
            ++nbr;
            if (cnt > 32 || over) break;  // a big brick runs alone (several rounds)
        }
        if (nbr == 0) break;
        __syncwarp();
        // ---- the group's queries, one per lane (several rounds only for a lone big brick)
        for (int r0 = 0; r0 < gq; r0 += 32) {
            const int L = r0 + lane;
            const bool has = L < gq;
            const int bb = __popc(qmask & (0xffffffffu >> (31 - lane))) - 1;  // (lone brick: 0)
            const uint32_t start = __shfl_sync(kFull, my_start, bb);
            const int qs = __shfl_sync(kFull, my_qs, bb), off = __shfl_sync(kFull, my_off, bb),
                      bnc = __shfl_sync(kFull, my_nc, bb);
            const int c0 = __shfl_sync(kFull, my_c0, bb), c1 = __shfl_sync(kFull, my_c1, bb),
                      c2 = __shfl_sync(kFull, my_c2, bb);
            const float4 q = has ? __ldg(g.spos + start + (L - qs)) : make_float4(0.f, 0.f, 0.f, 0.f);
            const int i = __float_as_int(q.w);
            bool ok = has && off >= 0;
            const int base = ok ? off : 0, nc = ok ? bnc : 0;  // candidates [base, base + nc), sentinel at base + nc
            const int maxnc = __reduce_max_sync(kFull, (unsigned)nc);
            // ---- one pass: list every candidate with key <= tau (lanes without a query: none)
            // tau and the list in the key32t domain (bit patterns: unsigned order == float order)
            uint32_t tau = ok ? 0x7f800000u : 0u, lmax = 0u;
#if GSICP_BRICK_TAU0
            if (ok) {
                // the certificate below needs the k-th ball inside the expanded box: a k-th key above
                // D^2 (D = the query's distance to the box faces) fails it whatever else is listed,
                // so no candidate beyond band_hi(D^2) can matter — start the bound there (D rounded
                // up generously: its binary64 test has margins of ~1e-5 relative)
                const float qv[3] = {q.x, q.y, q.z};
                const int cv[3] = {c0, c1, c2};
                float D = INFINITY;
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                    const float lo_ = (float)cv[ax] * H - R, hi_ = (float)(cv[ax] + 1) * H + R;
                    D = fminf(D, fminf(qv[ax] - lo_, hi_ - qv[ax]));
                }
                const float Du = __fadd_ru(__fmul_ru(fmaxf(D, 0.f), 1.0001f), 1e-6f);
                tau = __float_as_uint(brick_band_hi(__fmul_ru(Du, Du))) & kBrickKeyMask;
            }
#endif
            int m = 0, n_events = 0;
            // compaction of this lane's list: quarter-octave buckets below tau (or, while tau is open,
            // below the largest listed key), b* = the bucket of the k-th entry, tau lowered to
            // band_hi(b*'s upper edge), the entries above it dropped
            auto compact = [&]() {
                const uint32_t top = tau < 0x7f800000u ? tau : lmax;
                Hist8 h;
                for (int s = 0; s < m; ++s) h.add(bucket8(lpk[s][lane], top));
                const int bs = h.select(k);
                tau = min(tau, __float_as_uint(brick_band_hi(__uint_as_float(bucket8_edge(bs, top)))) & kBrickKeyMask);
                int wr = 0;
                for (int s = 0; s < m; ++s) {
                    const uint32_t v = lpk[s][lane];
                    if ((v & kBrickKeyMask) <= tau) lpk[wr++][lane] = v;
                }
                m = wr;
            };
            for (int j0 = 0; j0 <= maxnc; j0 += kBrickU) {
                if (__any_sync(kFull, m > kBrickL - kBrickU)) {
                    // (whole warp: every lane with >= k entries tightens its bound)
                    ++n_events;
                    if (m >= k) compact();
                    if (m > kBrickL - kBrickU) {  // ties crowd one bucket: give the query to the search
                        ok = false;
                        tau = 0u;
                        m = 0;
                    }
                }
#pragma unroll
                for (int u = 0; u < kBrickU; ++u) {
                    const int idx = base + min(j0 + u, nc);
                    const float4 P = cand[idx];
                    const uint32_t kt = __float_as_uint(brick_key(q.x, q.y, q.z, P.x, P.y, P.z)) & kBrickKeyMask;
                    if (kt <= tau && ok) {  // (NaN sentinel: 0x7fc00000 > any finite tau or +inf; no query: tau 0, ok false)
                        lpk[m][lane] = kt | (uint32_t)idx;
                        lmax = max(lmax, kt);
                        ++m;
                    }
                }
            }
            int why = !has ? 0 : (off < 0 ? 1 : (!ok ? 2 : (m < k ? 3 : 0)));
            ok = ok && m >= k;
            // ---- exact selection: tighten once more, t = the k-th key32t, band resolved in binary64
            if (ok) {
                compact();
                ok = m <= kBrickLx;
                if (!ok) why = 4;
            }
            uint32_t sel = 0u;
            if (ok) {
                const double qx = q.x, qy = q.y, qz = q.z;
                Hist16 h;
                for (int s = 0; s < m; ++s) h.add(bucket16(lpk[s][lane], tau));
                int nlo;
                const int bs = h.select(k, nlo);
                uint32_t bd = 0u;  // the boundary bucket's entries
                for (int s = 0; s < m; ++s) bd |= (bucket16(lpk[s][lane], tau) == bs ? 1u : 0u) << s;
                const int r = k - nlo;  // t: the r-th smallest (key32t, slot) of the boundary bucket
                uint32_t t = 0u;
#if GSICP_BRICK_SUBRANK
                {   // split by the next 3 mantissa bits (monotone; clamped ends), rank inside the
                    // sub-bucket holding the r-th entry only (cf. the image kernel)
                    const int sub0 = (((int)(tau >> 20) - 15 + bs) << 3) - 1;
                    auto sub_of = [&](uint32_t v) { return min(max((int)(v >> 17) - sub0, 0), 9); };
                    Hist16 hs;
                    for (uint32_t f = bd; f; f &= f - 1) hs.add(sub_of(lpk[__ffs(f) - 1][lane]));
                    int sbelow;
                    const int sb = hs.select(r, sbelow);
                    const int r2 = r - sbelow;
                    uint32_t bs2 = 0u;
                    for (uint32_t f = bd; f; f &= f - 1)
                        bs2 |= (sub_of(lpk[__ffs(f) - 1][lane]) == sb ? 1u : 0u) << (__ffs(f) - 1);
                    for (uint32_t f = bs2; f; f &= f - 1) {
                        const uint32_t vs = lpk[__ffs(f) - 1][lane];
                        int rank = 0;
                        for (uint32_t f2 = bs2; f2; f2 &= f2 - 1) rank += lpk[__ffs(f2) - 1][lane] < vs ? 1 : 0;
                        if (rank == r2 - 1) t = vs & kBrickKeyMask;
                    }
                }
#else
                for (uint32_t f = bd; f; f &= f - 1) {
                    const uint32_t vs = lpk[__ffs(f) - 1][lane];
                    int rank = 0;
                    for (uint32_t f2 = bd; f2; f2 &= f2 - 1) rank += lpk[__ffs(f2) - 1][lane] < vs ? 1 : 0;
                    if (rank == r - 1) t = vs & kBrickKeyMask;
                }
#endif
                const float blo = brick_band_lo(__uint_as_float(t)), bhi = brick_band_hi(__uint_as_float(t));
                ok = (__float_as_uint(bhi) & kBrickKeyMask) <= tau;  // every candidate up to band_hi(t) is listed
                if (!ok) why = 5;
                uint32_t band = 0u;
                for (int s = 0; s < m; ++s) {
                    const float ks = __uint_as_float(lpk[s][lane] & kBrickKeyMask);
                    sel |= (ks < blo ? 1u : 0u) << s;
                    band |= (ks >= blo && ks <= bhi ? 1u : 0u) << s;
                }
                auto key64_of = [&](int s, uint32_t &id) {
                    const float4 P = cand[lpk[s][lane] & kBrickSlotMask];
                    id = (uint32_t)__float_as_int(P.w);
                    return key64(qx, qy, qz, P.x, P.y, P.z);
                };
                auto rank_in = [&](int s, uint32_t mask) {
                    uint32_t ij;
                    const double kj = key64_of(s, ij);
                    int rank = 0;
                    for (uint32_t bl = mask; bl; bl &= bl - 1) {
                        uint32_t il;
                        const double kl = key64_of(__ffs(bl) - 1, il);
                        rank += (kl < kj || (kl == kj && il < ij)) ? 1 : 0;
                    }
                    return rank;
                };
                const int need = k - __popc(sel);
                if (__popc(band) == need) {
                    sel |= band;
                } else {
                    uint32_t add = 0u;
                    for (uint32_t bj = band; bj; bj &= bj - 1)
                        if (rank_in(__ffs(bj) - 1, band) < need) add |= 1u << (__ffs(bj) - 1);
                    sel |= add;
                }
                // certificate: the k-th ball (binary64 radius with margin) inside the expanded box
                const double rho = sqrt((double)bhi) * (1.0 + 1e-5) + 1e-9;
                const double qc[3] = {qx, qy, qz};
                const int cc[3] = {c0, c1, c2};
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) {
                    const double mg = 1e-7 * fabs(qc[ax]);
                    const float lo_ = (float)cc[ax] * H - R, hi_ = (float)(cc[ax] + 1) * H + R;
                    ok = ok && qc[ax] - rho - mg >= (double)lo_ && qc[ax] + rho + mg <= (double)hi_;
                }
                if (!ok && why == 0) why = 6;
                if (ok) {
                    if (a.knn_idx) {
                        for (uint32_t f = sel; f; f &= f - 1) {
                            const int s = __ffs(f) - 1;
                            const int rk = SORT ? rank_in(s, sel) : __popc(sel & ((1u << s) - 1u));
                            a.knn_idx[(size_t)i * k + rk] = __float_as_int(cand[lpk[s][lane] & kBrickSlotMask].w);
                        }
                    }
                    double s1[3] = {0, 0, 0}, s2[6] = {0, 0, 0, 0, 0, 0};
                    for (uint32_t f = sel; f; f &= f - 1) {
                        const float4 P = cand[lpk[__ffs(f) - 1][lane] & kBrickSlotMask];
                        const double d0 = (double)P.x - qx, d1 = (double)P.y - qy, d2 = (double)P.z - qz;
                        s1[0] += d0;
                        s1[1] += d1;
                        s1[2] += d2;
                        s2[0] += d0 * d0;
                        s2[1] += d0 * d1;
                        s2[2] += d0 * d2;
                        s2[3] += d1 * d1;
                        s2[4] += d1 * d2;
                        s2[5] += d2 * d2;
                    }
                    finish_moments(a, n, i, s1, s2, __popc(sel));
                    if (a.debug) a.debug[i] = make_int4(-7, bnc, m, nbr * 256 + n_events * 65536 + __popc(__ballot_sync(__activemask(), true)));
                }
            }
            {  // the queries left to the warp search (one atomic per warp)
                const bool qd = has && !ok;
                const unsigned qb = __ballot_sync(kFull, qd);
                uint32_t qbase = 0u;
                if (lane == 0 && qb) qbase = atomicAdd(b.queue_n, (uint32_t)__popc(qb));
                qbase = __shfl_sync(kFull, qbase, 0);
                if (qd) {
                    b.queue[qbase + __popc(qb & ((1u << lane) - 1u))] = (uint32_t)i;
                    if (a.debug) a.debug[i] = make_int4(-8, why, bnc, m);
                }
            }
            __syncwarp();  // the list columns are reused by the next round
        }
        __syncwarp();  // the staged candidates are reused by the next group
    }
}

template <int K>
cudaError_t launch_search(const KnnArgs &a, int cap, cudaStream_t s);
template <int K>
cudaError_t launch_epilogue(const KnnArgs &a, int cap, cudaStream_t s);

template <int K, int M>
cudaError_t launch_tile_m(const KnnArgs &a, const ImgArgs &im, cudaStream_t s) {
    constexpr int SW = kImgTX + 2 * M, SH = kImgTY + 2 * M;
    const int smem = (int)(sizeof(float4) * SW * SH + sizeof(uint32_t) * (kImgBuckets / 2) * kImgThreads +
                           sizeof(unsigned long long) * kImgList * kImgThreads);
    static PerDevice<int> attr;  // the opt-in shared memory size, set once per device
    attr.get([&](int) { return (int)cudaFuncSetAttribute(k_knn_image<K, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
    const dim3 grid((unsigned)((im.Ws + kImgTX - 1) / kImgTX), (unsigned)((im.Hs + kImgTY - 1) / kImgTY));
    launch_pdl(k_knn_image<K, M>, grid, dim3(kImgThreads), (size_t)smem, s, a, im);
    GSICP_LAUNCH_CHECK("k_knn_image");
    return cudaSuccess;
}

// window half-width kImgM (4 and 6 measured slower in round 1)
template <int K>
cudaError_t launch_tile(const KnnArgs &a, const ImgArgs &im, cudaStream_t s) {
    return launch_tile_m<K, kImgM>(a, im, s);
}

// stream used to capture conditional-node bodies (per host thread)
cudaStream_t body_stream() {
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

template <int K>
cudaError_t launch_image(KnnArgs a, const ImgArgs &im, int cap, const float4 *pos, const int32_t *d_n, cudaStream_t s,
                         cudaEvent_t window_done) {
    cudaError_t e = cudaSuccess;
    ktimer_mark(KT_COVS, false, s);
    ktimer_mark(KT_KNN_SEARCH, false, s);
    const int L = im.Hs * im.Ws;
    if (im.map_given) {  // the map came with the points: only the counters are reset
        launch_pdl(k_img_map_clear, dim3(1), dim3(32), 0, s, im, 0);
        GSICP_LAUNCH_CHECK("k_img_map_clear");
    } else {
        launch_pdl(k_img_map_clear, dim3(blocks_for(std::max(L, kImgCounters), 256)), dim3(256), 0, s, im, 1);
        GSICP_LAUNCH_CHECK("k_img_map_clear");
        launch_pdl(k_img_map_fill, dim3(blocks_for(cap, 256)), dim3(256), 0, s, im, pos, d_n);
        GSICP_LAUNCH_CHECK("k_img_map_fill");
    }
    e = launch_tile<K>(a, im, s);
    if (e != cudaSuccess) return e;
    ktimer_mark(KT_KNN_SEARCH, true, s);
    if (window_done && (e = cudaEventRecord(window_done, s)) != cudaSuccess) return e;
    ktimer_mark(KT_WIDE, false, s);
    // wide window over the queue (a resident grid pulling queries)
    launch_pdl(k_knn_image_wide<K>, dim3((unsigned)num_sms() * 8), dim3(128), 0, s, a, im);
    GSICP_LAUNCH_CHECK("k_knn_image_wide");
    // the rest: brute force (a short queue), else the hash search + epilogue (long queue)
    launch_pdl(k_knn_brute<K>, dim3((unsigned)(2 * (num_sms() / kBruteCluster) * kBruteCluster)), dim3(kBruteThreads), 0,
               s, a, im);
    GSICP_LAUNCH_CHECK("k_knn_brute");
    // the hash tail (hash the cloud, warp search, epilogue) only for a non-empty hash queue: inside
    // a stream capture as the body of a conditional (IF) graph node whose condition k_img_hash_n
    // sets on the device; otherwise launched directly, each kernel returning at once when idle
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cst);
    if (cst == cudaStreamCaptureStatusActive) {
        cudaGraph_t graph = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t nd = 0;
        unsigned long long cid = 0;
        if ((e = cudaStreamGetCaptureInfo(s, &cst, &cid, &graph, &deps, &nd)) != cudaSuccess) return e;
        cudaGraphConditionalHandle h;
        if ((e = cudaGraphConditionalHandleCreate(&h, graph, 0, 0)) != cudaSuccess) return e;
        launch_pdl(k_img_hash_n, dim3(1), dim3(1), 0, s, im, d_n, h, 1);
        GSICP_LAUNCH_CHECK("k_img_hash_n");
        ktimer_mark(KT_WIDE, true, s);
        ktimer_mark(KT_TAIL, false, s);
        if ((e = cudaStreamGetCaptureInfo(s, &cst, &cid, &graph, &deps, &nd)) != cudaSuccess) return e;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        if ((e = cudaGraphAddNode(&cnode, graph, deps, nd, &cp)) != cudaSuccess) return e;
        cudaStream_t bs = body_stream();
        if (!bs) return cudaErrorInvalidResourceHandle;
        if ((e = cudaStreamBeginCaptureToGraph(bs, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                               cudaStreamCaptureModeRelaxed)) != cudaSuccess)
            return e;
        pdl_suspended() = true;  // no programmatic edges inside the conditional body
        const int32_t *hn = reinterpret_cast<const int32_t *>(im.ctr + kImgCtrHashN);
        cudaError_t eb = grid_build(a.g, pos, nullptr, nullptr, hn, cap, bs);
        a.queue = im.queue2;
        a.queue_n = im.ctr + kImgCtrHashQ;
        a.work = im.ctr + kImgCtrWork;
        if (eb == cudaSuccess) eb = launch_search<K>(a, cap, bs);
        if (eb == cudaSuccess) eb = launch_epilogue<K>(a, cap, bs);
        pdl_suspended() = false;
        cudaGraph_t body_out = nullptr;
        e = cudaStreamEndCapture(bs, &body_out);
        if (eb != cudaSuccess) return eb;
        if (e != cudaSuccess) return e;
        if ((e = cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess)
            return e;
    } else {
        launch_pdl(k_img_hash_n, dim3(1), dim3(1), 0, s, im, d_n, cudaGraphConditionalHandle{}, 0);
        GSICP_LAUNCH_CHECK("k_img_hash_n");
        ktimer_mark(KT_WIDE, true, s);
        ktimer_mark(KT_TAIL, false, s);
        {  // inline, only for a non-empty hash queue (the build kernels return at once otherwise)
            const int32_t *hn = reinterpret_cast<const int32_t *>(im.ctr + kImgCtrHashN);
            e = grid_build(a.g, pos, nullptr, nullptr, hn, cap, s);
            if (e != cudaSuccess) return e;
        }
        a.queue = im.queue2;
        a.queue_n = im.ctr + kImgCtrHashQ;
        a.work = im.ctr + kImgCtrWork;
        e = launch_search<K>(a, cap, s);
        if (e != cudaSuccess) return e;
        e = launch_epilogue<K>(a, cap, s);
        if (e != cudaSuccess) return e;
    }
    ktimer_mark(KT_TAIL, true, s);
    ktimer_mark(KT_COVS, true, s);
    note_launch(8);
    return cudaSuccess;
}

template <int K>
cudaError_t launch_search(const KnnArgs &a, int cap, cudaStream_t s) {
    // a resident grid (one wave) pulling work batches; never more warps than batches
    const long long warps = (cap + kQueriesPerWarp - 1) / kQueriesPerWarp;
    const long long blocks = std::min<long long>(blocks_for(warps * 32, kKnnThreads), (long long)num_sms() * kKnnMinBlocks);
    const dim3 grid((unsigned)std::max<long long>(blocks, 1));
    if (a.sort_out)
        launch_pdl(k_knn_search<K, true>, grid, dim3(kKnnThreads), 0, s, a);
    else
        launch_pdl(k_knn_search<K, false>, grid, dim3(kKnnThreads), 0, s, a);
    GSICP_LAUNCH_CHECK("k_knn_search");
    return cudaSuccess;
}

template <int K>
cudaError_t launch_epilogue(const KnnArgs &a, int cap, cudaStream_t s) {
    const long long blocks = std::min<long long>(blocks_for(cap, kKnnThreads), (long long)num_sms() * 16);
    launch_pdl(k_knn_epilogue<K>, dim3((unsigned)std::max<long long>(blocks, 1)), dim3(kKnnThreads), 0, s, a);
    GSICP_LAUNCH_CHECK("k_knn_epilogue");
    return cudaSuccess;
}

template <int K>
cudaError_t launch_k(const KnnArgs &a, int cap, cudaStream_t s) {
    ktimer_mark(KT_KNN_SEARCH, false, s);
    cudaError_t e = launch_search<K>(a, cap, s);
    if (e != cudaSuccess) return e;
    ktimer_mark(KT_KNN_SEARCH, true, s);
    e = launch_epilogue<K>(a, cap, s);
    if (e != cudaSuccess) return e;
    note_launch(2);
    return cudaSuccess;
}

// General clouds: bricks (k_knn_brick) then the warp search over the queue they leave
template <int K>
cudaError_t launch_brick(KnnArgs a, const BrickArgs &b, int cap, cudaStream_t s) {
    const GridView &g = a.g;
    ktimer_mark(KT_KNN_SEARCH, false, s);
    (void)g;  // (the brick list comes from the grid build's alloc step)
    const dim3 grid((unsigned)num_sms() * kBrickBlocksPerSm);  // one resident wave (by shared memory)
    constexpr int smem = kBrickWarps * kBrickSmemPerWarp;
    static PerDevice<int> attr;  // opt-in dynamic shared memory, once per device
    attr.get([&](int) {
        cudaFuncSetAttribute(k_knn_brick<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        return (int)cudaFuncSetAttribute(k_knn_brick<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    });
    if (a.sort_out)
        launch_pdl(k_knn_brick<K, true>, grid, dim3(kBrickWarps * 32), (size_t)smem, s, a, b);
    else
        launch_pdl(k_knn_brick<K, false>, grid, dim3(kBrickWarps * 32), (size_t)smem, s, a, b);
    GSICP_LAUNCH_CHECK("k_knn_brick");
    ktimer_mark(KT_KNN_SEARCH, true, s);
    a.queue = b.queue;
    a.queue_n = b.queue_n;
    a.work = g.counters + kMaxLevels + 4;
    cudaError_t e = launch_search<K>(a, cap, s);
    if (e == cudaSuccess) e = launch_epilogue<K>(a, cap, s);
    if (e != cudaSuccess) return e;
    note_launch(3);
    return cudaSuccess;
}

}  // namespace

// automatic cell sizes (cell0 <= 0): multiples of the estimated point spacing (the brick kernel
// wants level-0 cells of ~3.7 spacings: ~10 queries and ~120 candidates per brick, the k = 20
// ball inside the brick's box expanded by 0.95 H for > 99.9% of the queries of a surface)
constexpr float kAutoCellMult = 3.5f;
constexpr float kAutoCellMultiLevel = 3.5f;

size_t covariances_ws_bytes(int cap, int levels) {
    return grid_bytes(cap, levels, false) + align_up((size_t)cap * kMaxK * sizeof(int32_t)) +
           align_up((size_t)cap * sizeof(uint4)) + align_up((size_t)cap * sizeof(uint32_t));
}

cudaError_t covariances_launch(const float *pos, const int32_t *d_n, int cap, int k, int mode, float eps,
                               float cell0, int levels, float *cov_a, float *cov_b, int32_t *knn_idx, void *ws,
                               cudaStream_t s) {
    KnnArgs a{};
    if (!(cell0 > 0.f)) {  // automatic: ~k-neighbourhood-sized finest cells (blocking estimate)
        float sp = 0.f;
        cudaError_t e = estimate_spacing(reinterpret_cast<const float4 *>(pos), d_n, cap, ws, &sp, s);
        if (e != cudaSuccess) return e;
        cell0 = (levels > 1 ? kAutoCellMultiLevel : kAutoCellMult) * sp;
    }
    a.g = grid_carve(ws, cap, levels, false, cell0);
    a.pos = reinterpret_cast<const float4 *>(pos);
    a.d_n = d_n;
    a.k = k;
    a.mode = mode;
    a.eps = (double)eps;
    a.cov_a = reinterpret_cast<float4 *>(cov_a);
    a.cov_b = reinterpret_cast<float4 *>(cov_b);
    a.knn_idx = knn_idx;
    a.sort_out = knn_idx != nullptr;
    a.debug = reinterpret_cast<int4 *>(g_knn_debug);
    char *wp = static_cast<char *>(ws) + grid_bytes(cap, levels, false);
    a.nbr_t = reinterpret_cast<int32_t *>(wp);
    wp += align_up((size_t)cap * kMaxK * sizeof(int32_t));
    BrickArgs b{};
    b.bricks = reinterpret_cast<const uint4 *>(wp);
    wp += align_up((size_t)cap * sizeof(uint4));
    b.queue = reinterpret_cast<uint32_t *>(wp);
    b.n_bricks = a.g.counters + kMaxLevels + 2;  // zeroed by the grid build
    b.queue_n = a.g.counters + kMaxLevels + 3;
    a.work = a.g.counters + kMaxLevels;
    if (k <= 24) {  // the alloc step lists the bricks
        a.g.bricks = const_cast<uint4 *>(b.bricks);
        a.g.n_bricks = const_cast<uint32_t *>(b.n_bricks);
    }
    cudaError_t e = grid_build(a.g, a.pos, nullptr, nullptr, d_n, cap, s);
    if (e != cudaSuccess) return e;
    if (k <= 4) return launch_brick<4>(a, b, cap, s);
    if (k <= 8) return launch_brick<8>(a, b, cap, s);
    if (k <= 16) return launch_brick<16>(a, b, cap, s);
    if (k <= 20) return launch_brick<20>(a, b, cap, s);
    if (k <= 24) return launch_brick<24>(a, b, cap, s);
    return launch_k<32>(a, cap, s);  // (the brick list keeps k + 4 < 32 entries: larger k take the warp search)
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
    a.sort_out = 0;  // the graph needs the neighbour set only (k_graph_finalize takes the max key)
    a.nbr_t = nullptr;
    a.debug = nullptr;
    a.work = g.counters + kMaxLevels;
    cudaError_t e = launch_search<kGraphK>(a, cap, s);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaSuccess;
}

// The same for the queued points only (incremental maintenance of a growing map's graph, N1):
// rows queue[0 .. *queue_n) get their exact kGraphK-NN lists over the grid's points.
cudaError_t knn_graph_queue_launch(const GridView &g, const float4 *pos, const int32_t *d_n, int cap,
                                   const uint32_t *queue, const uint32_t *queue_n, int32_t *knn_idx, cudaStream_t s) {
    KnnArgs a{};
    a.g = g;
    a.pos = pos;
    a.d_n = d_n;
    a.k = kGraphK;
    a.knn_idx = knn_idx;
    a.sort_out = 0;
    a.queue = queue;
    a.queue_n = queue_n;
    a.work = g.counters + kMaxLevels;
    cudaError_t e = launch_search<kGraphK>(a, cap, s);
    if (e != cudaSuccess) return e;
    note_launch();
    return cudaSuccess;
}

size_t covariances_image_ws_bytes(int cap, int levels, int H, int W, int stride) {
    const size_t L = (size_t)((H + stride - 1) / stride) * (size_t)((W + stride - 1) / stride);
    return covariances_ws_bytes(cap, levels) + align_up(L * sizeof(int32_t)) +
           2 * align_up((size_t)cap * sizeof(uint32_t)) + align_up(kImgCounters * sizeof(uint32_t));
}

cudaError_t covariances_image_launch(const float *pos, const int32_t *d_n, int cap, int H, int W, int stride,
                                     gsicp_intrinsics Kin, int k, int mode, float eps, float cell0, int levels,
                                     float *cov_a, float *cov_b, int32_t *knn_idx, const int32_t *lattice_map,
                                     void *ws, cudaStream_t s, void *window_done) {
    KnnArgs a{};
    a.g = grid_carve(ws, cap, levels, false, cell0);
    a.pos = reinterpret_cast<const float4 *>(pos);
    a.d_n = d_n;
    a.k = k;
    a.mode = mode;
    a.eps = (double)eps;
    a.cov_a = reinterpret_cast<float4 *>(cov_a);
    a.cov_b = reinterpret_cast<float4 *>(cov_b);
    a.knn_idx = knn_idx;
    a.sort_out = knn_idx != nullptr;
    a.debug = reinterpret_cast<int4 *>(g_knn_debug);
    char *p = static_cast<char *>(ws) + grid_bytes(cap, levels, false);
    a.nbr_t = reinterpret_cast<int32_t *>(p);
    p += align_up((size_t)cap * kMaxK * sizeof(int32_t));
    ImgArgs im{};
    im.H = H;
    im.W = W;
    im.stride = stride;
    im.Hs = (H + stride - 1) / stride;
    im.Ws = (W + stride - 1) / stride;
    im.fx = Kin.fx;
    im.fy = Kin.fy;
    im.map = lattice_map ? const_cast<int32_t *>(lattice_map) : reinterpret_cast<int32_t *>(p);
    im.map_given = lattice_map != nullptr;
    p += align_up((size_t)im.Hs * im.Ws * sizeof(int32_t));
    im.queue = reinterpret_cast<uint32_t *>(p);
    p += align_up((size_t)cap * sizeof(uint32_t));
    im.queue2 = reinterpret_cast<uint32_t *>(p);
    p += align_up((size_t)cap * sizeof(uint32_t));
    im.ctr = reinterpret_cast<uint32_t *>(p);
    const float4 *p4 = a.pos;
    if (k <= 4) return launch_image<4>(a, im, cap, p4, d_n, s, (cudaEvent_t)window_done);
    if (k <= 8) return launch_image<8>(a, im, cap, p4, d_n, s, (cudaEvent_t)window_done);
    if (k <= 16) return launch_image<16>(a, im, cap, p4, d_n, s, (cudaEvent_t)window_done);
    if (k <= 20) return launch_image<20>(a, im, cap, p4, d_n, s, (cudaEvent_t)window_done);
    if (k <= 24) return launch_image<24>(a, im, cap, p4, d_n, s, (cudaEvent_t)window_done);
    return launch_image<32>(a, im, cap, p4, d_n, s, (cudaEvent_t)window_done);
}

}  // namespace gsicp
