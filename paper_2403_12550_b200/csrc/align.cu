// A6-A9  G-ICP alignment in ONE persistent cooperative kernel.
//
// Per Gauss-Newton iteration, every thread takes source points i (grid-stride) and
//   A6  q = K3(T, x_i) in binary64 (no FMA), exact 1-NN of q among the target means by the
//       canonical binary64 (K2 key, index) order (R1, R15), grid search warm-started with
//       the previous iteration's match; valid iff key < r^2 (R15);
//   A7  Sigma = C^t_j + R C^s_i R^T, M = Sigma^{-1} (adjugate, binary64), d = x^t_j - q,
//       J = [[q]x, -I]: accumulates the 21 unique H = J^T M J terms, b = J^T M d, d^T M d and
//       the inlier count (Eq. 1; R1-R3, R16);
// then warp shuffles + shared memory reduce the 29 terms per block into a per-block partial,
// one grid barrier publishes the partials, and EVERY block reduces all partials in the same
// fixed order (so all blocks hold bit-identical H, b), solves the 6x6 system by Cholesky
// (A8), applies the left update T <- [Exp(w) | v] T and evaluates the convergence test —
// identical decisions in every block, no second barrier, no host round trip (A9 at the end).
//
// Latency design: the grid is sized so every thread owns (at most) one "resident" point whose
// source data, current match (position + covariance) and own target cell stay in registers for
// the whole GN loop; an iteration's dependent memory chain is then: scan the own cell (usually
// cached), rarely a neighbour cell, and reload the match covariance only when the match changes.
// Points beyond one per thread (clouds larger than the resident grid) take the generic path.
#include <math.h>

#include "gsicp_internal.cuh"
#include "host_common.cuh"
#include "search.cuh"

namespace gsicp {

// diagnostic timeline hook (gsicp_debug_align_timeline); thread-local like the error string
thread_local long long *g_align_timeline = nullptr;
thread_local long long g_align_timeline_cap = 0;
thread_local int32_t *g_align_debug = nullptr;
// per-iteration linearisation record hook (gsicp_debug_align_iterations)
thread_local double *g_align_iter_rec = nullptr;
thread_local int32_t *g_align_iter_corr = nullptr;
thread_local int g_align_iter_cap = 0;

namespace {

constexpr int kT = kAlignThreads;
constexpr int kWarps = kT / 32;
constexpr int kPad = 32;  // partial record stride (doubles)

struct AlignArgs {
    const float4 *spos, *scov_a, *scov_b;
    const int32_t *d_n;
    int cap;
    const CellEntry *table;
    uint32_t mask;
    float h, inv_h;
    const float4 *tpos, *tcov_a, *tcov_b;
    const int32_t *tbbox;
    const uint2 *dense;       // dense cell array (used iff dense_hdr[0])
    const int32_t *dense_hdr; // {in_use, lo xyz, dims xyz}
    const int32_t *nbr;       // nullable: target kNN graph, [M][kGraphK] slots
    const float *nbr_key;     // [M] key of the kGraphK-th neighbour
    int max_iters;
    float r;                  // max_corr_dist
    double r2;                // (double)r * (double)r: valid iff key64 < r2 (R15)
    float r2f;                // binary32 upper bound of r2 (cell pruning)
    double eps_rot, eps_trans;
    int min_pairs;
    int solver;               // 0 GN, 1 LM (R30)
    double lm_lambda0;
    int linearize_only;
    double *d_T;              // [16] in/out (row-major 4x4)
    gsicp_align_stats *d_stats;
    double *d_lin;            // [44] linearize-only output: H[36], b[6], cost, n
    double *partials;         // [2][grid][kPad]
    unsigned int *barrier;
    int32_t *corr_ws;         // [cap] previous match (cell-ordered slot), -2-slot if gated out, -1 none
    float4 *reuse_ws;         // [cap] non-resident points' reuse state: (query of the last search, d2lb)
    int32_t *corr_out;        // nullable [cap] original target index or -1
    long long *timeline;      // diagnostic (nullable): [0] start, then per iteration G arrivals + pass
    long long timeline_cap;
    int4 *debug;              // diagnostic (nullable): per point bitmasks over iterations (queued, reused,
                              // graph-certified) and the iteration count
    int32_t *seed_slot;       // [cap] iteration-0 matches from k_align_seed (target slot or -1)
    double *seed_hdr;         // [16]: pose the seeds were computed at (12), ticket at [12]
    double seed_ticket;       // k_align_seed: ticket to write; k_align: ticket expected (0: none)
    int32_t *seed_queue;      // [cap] hard queries of the seed pass
    int2 *flat_queue;         // [cap] hard queries of the flat GN path (point, warm-start slot)
    int32_t *rset;            // [cap][kSetCap] the flat path's neighbourhood sets (-1 pads)
    float4 *rset_hdr;         // [cap] (query the set was taken at, rho_cert); rho_cert 0: none
    int32_t *seed_qn;         // [1] their count
    // diagnostic (nullable): per GN iteration it < iter_cap, iter_rec[it * kIterRec + ..] = the pose
    // T_it the iteration linearised at (12, row-major 3x4) then its 29 reduced terms (21 H upper,
    // 6 b, cost, n); iter_corr[it * cap + i] = point i's correspondence (original index or -1)
    double *iter_rec;
    int32_t *iter_corr;
    int iter_cap;
};
constexpr int kIterRec = 48;

__device__ __forceinline__ long long globaltimer_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ float ordered_to_float_(int32_t i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

// The query of a correspondence search: the binary64 K3 transform q (the definition, R15) and its
// binary32 rounding (cell geometry, pruning and the binary32 screen; QueryCell's margin covers
// |q - fl32(q)|).
struct Qry {
    double d0, d1, d2;
    float x, y, z;
    __device__ __forceinline__ Qry(double a, double b, double c)
        : d0(a), d1(b), d2(c), x((float)a), y((float)b), z((float)c) {}
    // >= |q - fl32(q)| (each coordinate within 2^-24 |q_i|: 2 u |fl32(q)|_1 with margin)
    __device__ __forceinline__ float E() const { return 1.2e-7f * (fabsf(x) + fabsf(y) + fabsf(z)) + 1e-30f; }
    __device__ __forceinline__ double key(const float4 &p) const { return key64(d0, d1, d2, p.x, p.y, p.z); }
    __device__ __forceinline__ float key32(const float4 &p) const { return canon_key(x, y, z, p.x, p.y, p.z); }
};

// running 1-NN state of one query: the best (K2 key, original index) so far
struct NN {
    double bk = INFINITY;                 // key64 of best
    uint32_t bi = 0xffffffffu;            // original index of best (= p.w's bits)
    int slot = -1;                        // cell-ordered target slot of best (-1: none yet)
    float4 p;                             // target record of best
    int probes = 0, cands = 0, slow = 0;  // diagnostics
    __device__ __forceinline__ void offer(double k, uint32_t i, int s, const float4 &rec) {
        if (k < bk || (k == bk && i < bi)) {
            bk = k;
            bi = i;
            slot = s;
            p = rec;
        }
    }
    __device__ __forceinline__ void set(double k, int s, const float4 &rec) {
        bk = k;
        bi = (uint32_t)__float_as_int(rec.w);
        slot = s;
        p = rec;
    }
    // Binary32 screen: a candidate c can beat (or tie) the best only if key32(fl32(q), c) <= screen:
    // |q - c| <= |q - best| and |fl32(q) - c| <= |q - c| + E, key32 within 5u of |fl32(q) - c|^2.
    // Only such candidates get the binary64 key (usually just the best itself).
    __device__ __forceinline__ float screen(const Qry &q) const {
        if (slot < 0) return INFINITY;
        const float s = __fmul_ru(__fadd_ru(__fsqrt_ru(__double2float_ru(bk)), q.E()), 1.000002f);
        return __fmul_ru(s, s);
    }
};

constexpr int kCandBatch = 4;   // candidate records loaded together (one latency per batch)
constexpr int kNbBatch = 4;     // neighbour-cell lookups in flight together (fast path)

__device__ __forceinline__ void scan_target_cell(const AlignArgs &a, uint2 se, const Qry &q, NN &nn) {
    ++nn.probes;
    nn.cands += (int)se.y;
    const uint32_t end = se.x + se.y;
    for (uint32_t j0 = se.x; j0 < end; j0 += kCandBatch) {
        float4 p[kCandBatch];
#pragma unroll
        for (int u = 0; u < kCandBatch; ++u) p[u] = j0 + u < end ? __ldg(a.tpos + j0 + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < kCandBatch; ++u) {
            if (j0 + u >= end) break;
            if (q.key32(p[u]) <= nn.screen(q)) nn.offer(q.key(p[u]), (uint32_t)__float_as_int(p[u].w), (int)(j0 + u), p[u]);
        }
    }
}

// binary32 upper bound on min(best key, r^2) for cell pruning (the gaps are binary32 lower bounds)
__device__ __forceinline__ float nn_bound(const AlignArgs &a, const NN &nn) {
    return nn.slot >= 0 ? fminf(__double2float_ru(nn.bk), a.r2f) : a.r2f;
}

// Certified graph step: nn holds a candidate slot j with key k_j.  Every target k that could beat
// it satisfies |m_j - m_k| <= 2 |q - m_j| (triangle inequality), so if 4 k_j < key_K(j) (with
// slack for the binary32 rounding of the graph's key) all of them are in j's K-NN list and the 1-NN
// of q is the best of that list (self included).
// Greedy descent on the graph until a certified step: each step scans the list of the current
// candidate j (which can only improve nn); if j was certified the result is exact.  If the list
// holds nothing better and j is not certified, or after kGraphSteps steps, returns false (nn
// holds the best point seen, a valid upper bound for the grid search).
constexpr int kGraphSteps = 4;
constexpr float kReuseMargin = 1e-5f;  // relative slack on every distance of the reuse test
// the warp path bounds the second neighbour only from this iteration on (earlier pose updates
// are too large for the bound to survive the next step)
#ifndef GSICP_D2_FROM_ITER
#define GSICP_D2_FROM_ITER 2
#endif
#ifndef GSICP_D2_SKIP_REPEAT
#define GSICP_D2_SKIP_REPEAT 1
#endif
constexpr int kD2FromIter = GSICP_D2_FROM_ITER;
// ... and only for queries within this many cells of their match: farther off the surface (noisy
// depth) the second neighbour is nearly as close as the first, the reuse margin d2 - d1 vanishes
// and the second search would be wasted
constexpr float kD2MaxD1 = 0.8f;

// On a certified step the list also bounds the SECOND nearest target: list members have their
// exact distances, every other target k has |q - m_k| >= |m_j - m_k| - |q - m_j| >=
// sqrt(key_K(j)) - sqrt(k_j).  d2lb receives that lower bound on the distance from q to any
// target other than the 1-NN (conservatively rounded), for the motion-bounded reuse in k_align.
__device__ __forceinline__ bool graph_nn(const AlignArgs &a, const Qry &q, NN &nn, float &d2lb) {
    for (int step = 0; step < kGraphSteps; ++step) {
        const int j = nn.slot;
        const float kj = __double2float_ru(nn.bk);
        const int4 *lst = reinterpret_cast<const int4 *>(a.nbr + (size_t)j * kGraphK);
        const float kk = __ldg(a.nbr_key + j);
        int sl[kGraphK];
#pragma unroll
        for (int v = 0; v < kGraphK / 4; ++v) {
            const int4 w = __ldg(lst + v);
            sl[4 * v] = w.x; sl[4 * v + 1] = w.y; sl[4 * v + 2] = w.z; sl[4 * v + 3] = w.w;
        }
        const bool certified = 4.f * kj * (1.f + 4e-5f) < kk * (1.f - 4e-5f);
        // binary32 screen of the list (records in flight together), then the binary64 keys of the
        // few that can beat the best (records reloaded through L1: keeps the doubles out of the
        // 16-wide unrolled section)
        float k32[kGraphK];
        {
            float4 p[kGraphK];
#pragma unroll
            for (int u = 0; u < kGraphK; ++u)
                p[u] = sl[u] >= 0 ? __ldg(a.tpos + sl[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < kGraphK; ++u) k32[u] = sl[u] >= 0 ? q.key32(p[u]) : INFINITY;
        }
        ++nn.probes;
        nn.cands += kGraphK;
        float l1 = INFINITY, l2 = INFINITY;  // the two smallest screen keys of this list
        uint32_t cand = 0u;
        const float scr = nn.screen(q);
#pragma unroll
        for (int u = 0; u < kGraphK; ++u) {
            cand |= (k32[u] <= scr ? 1u : 0u) << u;
            l2 = k32[u] < l1 ? l1 : (k32[u] < l2 ? k32[u] : l2);
            l1 = k32[u] < l1 ? k32[u] : l1;
        }
        while (cand) {
            const int u = __ffs(cand) - 1;
            cand &= cand - 1;
            int su = sl[0];
#pragma unroll
            for (int v = 1; v < kGraphK; ++v) su = v == u ? sl[v] : su;
            const float4 rec = __ldg(a.tpos + su);
            if (q.key32(rec) <= nn.screen(q)) nn.offer(q.key(rec), (uint32_t)__float_as_int(rec.w), su, rec);
        }
        if (certified) {
            const float rc = sqrtf(kk) * (1.f - kReuseMargin) - sqrtf(kj) * (1.f + kReuseMargin);
            // every list member other than the 1-NN: |q - m| >= |fl32(q) - m| - E
            const float d2 = l2 < INFINITY ? fmaxf(sqrtf(__fmul_rd(l2, 0.999999f)) - q.E(), 0.f) : INFINITY;
            d2lb = fmaxf(fminf(d2, rc), 0.f) * (1.f - kReuseMargin);
            return true;
        }
        if (nn.slot == j) return false;  // local minimum without a certificate
    }
    return false;
}

constexpr int kMaxCells = 4;   // cells gathered for one flattened candidate scan (own + 3 neighbours)
constexpr int kFlatBatch = 8;  // candidate records loaded per round trip in the flattened scan

// Candidates of up to kMaxCells cells scanned as one flattened range, kFlatBatch records per
// round trip (instead of one chain of round trips per cell); a cell's records are skipped once
// its lower bound exceeds the shrinking bound.
__device__ __forceinline__ void scan_cells_flat(const AlignArgs &a, const uint2 (&se)[kMaxCells],
                                                const float (&lbs)[kMaxCells], const Qry &q, NN &nn) {
    uint32_t pre[kMaxCells + 1];
    pre[0] = 0;
#pragma unroll
    for (int k = 0; k < kMaxCells; ++k) {
        pre[k + 1] = pre[k] + se[k].y;
        nn.probes += se[k].y ? 1 : 0;
    }
    const uint32_t tot = pre[kMaxCells];
    nn.cands += (int)tot;
    for (uint32_t base = 0; base < tot; base += kFlatBatch) {
        const float bnd = nn_bound(a, nn);
        float4 p[kFlatBatch];
        uint32_t slot[kFlatBatch];
        bool ok[kFlatBatch];
#pragma unroll
        for (int u = 0; u < kFlatBatch; ++u) {
            const uint32_t item = base + u;
            uint32_t s = 0;
            bool v = false;
#pragma unroll
            for (int k = 0; k < kMaxCells; ++k) {
                const bool in = item >= pre[k] && item < pre[k + 1];
                s = in ? se[k].x + (item - pre[k]) : s;
                v = in ? lbs[k] <= bnd : v;
            }
            ok[u] = v;
            slot[u] = s;
            p[u] = v ? __ldg(a.tpos + s) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        uint32_t cand = 0u;
#pragma unroll
        for (int u = 0; u < kFlatBatch; ++u) cand |= (ok[u] && q.key32(p[u]) <= nn.screen(q) ? 1u : 0u) << u;
        while (cand) {  // binary64 keys of the screened few (records reloaded: no doubles in the unrolled part)
            const int u = __ffs(cand) - 1;
            cand &= cand - 1;
            uint32_t su = slot[0];
#pragma unroll
            for (int v = 1; v < kFlatBatch; ++v) su = v == u ? slot[v] : su;
            const float4 rec = __ldg(a.tpos + su);
            if (q.key32(rec) <= nn.screen(q)) nn.offer(q.key(rec), (uint32_t)__float_as_int(rec.w), (int)su, rec);
        }
    }
}

// General exact search after the own cell: grow shells while an ungated search has found
// nothing, then the ball traversal bounded by min(best, r^2).  Out of line so that the
// common fast path keeps its registers.
__device__ __forceinline__ void nn_slow(const AlignArgs &a, const CellIndex &idx, const int *sb, const Qry &q, NN &nn) {
    const QueryCell qc(q.x, q.y, q.z, a.h, a.inv_h);
    const int *blo = sb, *bhi = sb + 3;
    int m_done = 0;
    if (nn.slot < 0 && !(a.r2 < INFINITY)) {
        while (nn.slot < 0 && !qc.covers(m_done, blo, bhi)) {
            ++m_done;
            const int cnt = shell_count(m_done);
            for (int t = 0; t < cnt; ++t) {
                int dx, dy, dz;
                shell_cell(m_done, t, dx, dy, dz);
                const int x = qc.c[0] + dx, y = qc.c[1] + dy, z = qc.c[2] + dz;
                if (x < blo[0] || x > bhi[0] || y < blo[1] || y > bhi[1] || z < blo[2] || z > bhi[2]) continue;
                scan_target_cell(a, idx.one(x, y, z), q, nn);
            }
        }
    }
    ball_search(
        qc, idx, blo, bhi, [&](int dx, int dy, int dz) { return max(max(abs(dx), abs(dy)), abs(dz)) <= m_done; },
        [&](uint2 se) { scan_target_cell(a, se, q, nn); }, [&]() { return nn_bound(a, nn); });
}

// Exact 1-NN given the query's cell geometry and its own cell's (start, count) (already known).
// Fast path: when the ball of the current bound cannot reach offset +-2 on any axis, only the 26
// neighbours can qualify; they are tested by their gaps alone — and none at all when the ball
// stays inside the own cell (the common, warm-started case).
// Returns true when nn is the exact answer; false (only with defer) when the general search is
// still needed — nn then holds the best point seen.
__device__ __forceinline__ bool nn_search(const AlignArgs &a, const CellIndex &idx, const int *sb,
                                          const QueryCell &qc, uint2 own, const Qry &q, NN &nn, bool defer) {
    float glo[3], ghi[3], glo2[3], ghi2[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        glo[k] = qc.gap2(-1, k);
        ghi[k] = qc.gap2(1, k);
        glo2[k] = qc.gap2(-2, k);
        ghi2[k] = qc.gap2(2, k);
    }
    auto fits = [&](float b) {
        return glo2[0] > b && ghi2[0] > b && glo2[1] > b && ghi2[1] > b && glo2[2] > b && ghi2[2] > b;
    };
    // bound from the warm start; without one (or too loose) scan the own cell first
    float b = nn_bound(a, nn);
    bool own_pending = true;
    if (!fits(b)) {
        scan_target_cell(a, own, q, nn);
        own_pending = false;
        b = nn_bound(a, nn);
        if (!fits(b)) {
            ++nn.slow;
            if (defer) return false;  // the block's warps run it cooperatively (warp_nn)
            NN tmp = nn;  // a copy: taking nn's address would pin it to local memory
            nn_slow(a, idx, sb, q, tmp);
            nn = tmp;
            return true;
        }
    }
    const int *blo = sb, *bhi = sb + 3;
    auto nb_lb = [&](int dx, int dy, int dz) {
        return (dx ? (dx < 0 ? glo[0] : ghi[0]) : 0.f) + (dy ? (dy < 0 ? glo[1] : ghi[1]) : 0.f) +
               (dz ? (dz < 0 ? glo[2] : ghi[2]) : 0.f);
    };
    // the ball of bound b reaches at most the 26 neighbours: pick them by their gaps (no loads)
    unsigned todo = 0;
    if (glo[0] <= b || ghi[0] <= b || glo[1] <= b || ghi[1] <= b || glo[2] <= b || ghi[2] <= b) {
        for (int t = 0; t < 26; ++t) {
            int dx, dy, dz;
            shell_cell(1, t, dx, dy, dz);
            const int x = qc.c[0] + dx, y = qc.c[1] + dy, z = qc.c[2] + dz;
            if (nb_lb(dx, dy, dz) <= b && x >= blo[0] && x <= bhi[0] && y >= blo[1] && y <= bhi[1] && z >= blo[2] &&
                z <= bhi[2])
                todo |= 1u << t;
        }
    }
    // own cell (if pending) + up to kMaxCells-1 neighbours per round: one batch of lookups, then
    // all their candidates as one flattened range
    while (own_pending || todo) {
        int xs[kMaxCells], ys[kMaxCells], zs[kMaxCells];
        bool valid[kMaxCells];
        float lbs[kMaxCells];
        valid[0] = false;
        xs[0] = ys[0] = zs[0] = 0;
        lbs[0] = 0.f;
#pragma unroll
        for (int u = 1; u < kMaxCells; ++u) {
            valid[u] = todo != 0;
            const int t = valid[u] ? __ffs(todo) - 1 : 0;
            todo &= todo - 1;
            int dx, dy, dz;
            shell_cell(1, t, dx, dy, dz);
            xs[u] = qc.c[0] + dx;
            ys[u] = qc.c[1] + dy;
            zs[u] = qc.c[2] + dz;
            lbs[u] = nb_lb(dx, dy, dz);
        }
        uint2 se[kMaxCells];
        idx.batch(xs, ys, zs, valid, se);
        se[0] = own_pending ? own : make_uint2(0u, 0u);
        own_pending = false;
        scan_cells_flat(a, se, lbs, q, nn);
    }
    return true;
}

__device__ __forceinline__ double shfl_f64(double v, int src) {
    return __hiloint2double(__shfl_sync(0xffffffffu, __double2hiint(v), src), __shfl_sync(0xffffffffu, __double2loint(v), src));
}

// Warp-cooperative exact 1-NN for one query (all lanes call it with the same arguments; nn is
// uniform on entry and exit).  Cells are visited in Chebyshev shells around the query cell,
// nearest first (shell 0+1 = 27 cells in the first round, then shell m in rounds of 32, lane =
// cell), skipping cells whose lower bound exceeds the current bound; the points of the probed
// cells are scanned as one flattened range (lane = candidate) and the batch minimum by (key64,
// index) is taken by shuffles.  After shell m every unvisited point is >= certified_key(m) away,
// so the search stops as soon as the bound is below that (or the shells cover the target bbox).
// Used for the queries whose per-thread fast path failed, so a few hard queries do not serialise
// a warp.  With fixed_b2 >= 0 it instead finds the best target with key <= fixed_b2 other than
// slot `excl` (the second-neighbour bound of the motion-bounded reuse); the r gate does not apply.
__device__ __forceinline__ void warp_scan_cells(const AlignArgs &a, const CellIndex &idx, const QueryCell &qc, bool valid,
                                                int dx, int dy, int dz, const Qry &q, NN &nn, int lane, int excl) {
    const uint2 se = valid ? idx.one(qc.c[0] + dx, qc.c[1] + dy, qc.c[2] + dz) : make_uint2(0u, 0u);
    uint32_t incl = se.y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t ctot = __shfl_sync(0xffffffffu, incl, 31);
    nn.probes += __popc(__ballot_sync(0xffffffffu, se.y != 0));
    nn.cands += (int)ctot;
    for (uint32_t base = 0; base < ctot; base += 32) {
        const uint32_t item = base + lane;
        int l0 = 0, l1 = 31;
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            const int mid = (l0 + l1) >> 1;
            if (__shfl_sync(0xffffffffu, incl, mid) > item) l1 = mid; else l0 = mid + 1;
        }
        const uint32_t c_incl = __shfl_sync(0xffffffffu, incl, l0);
        const uint32_t c_start = __shfl_sync(0xffffffffu, se.x, l0);
        const uint32_t c_cnt = __shfl_sync(0xffffffffu, se.y, l0);
        double ck = INFINITY;
        uint32_t ci = 0xffffffffu;
        float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
        uint32_t slot = 0;
        if (item < ctot) {
            slot = c_start + (item - (c_incl - c_cnt));
            p = __ldg(a.tpos + slot);
            if ((int)slot != excl) {
                ck = q.key(p);
                ci = (uint32_t)__float_as_int(p.w);
            }
        }
        double mk = ck;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mk = fmin(mk, shfl_f64(mk, lane ^ o));
        const uint32_t mi = __reduce_min_sync(0xffffffffu, ck == mk ? ci : 0xffffffffu);
        if (mk < nn.bk || (mk == nn.bk && mi < nn.bi)) {
            const int src = __ffs(__ballot_sync(0xffffffffu, ck == mk && ci == mi)) - 1;
            nn.bk = mk;
            nn.bi = mi;
            nn.slot = (int)__shfl_sync(0xffffffffu, slot, src);
            nn.p.x = __shfl_sync(0xffffffffu, p.x, src);
            nn.p.y = __shfl_sync(0xffffffffu, p.y, src);
            nn.p.z = __shfl_sync(0xffffffffu, p.z, src);
            nn.p.w = __shfl_sync(0xffffffffu, p.w, src);
        }
    }
}

constexpr int kWarpShells = 3;  // shells visited nearest-first before the box traversal

__device__ void warp_nn(const AlignArgs &a, const CellIndex &idx, const int *sb, const Qry &q, NN &nn, int lane,
                        float fixed_b2 = -1.f, int excl = -1) {
    const QueryCell qc(q.x, q.y, q.z, a.h, a.inv_h);
    const int *blo = sb, *bhi = sb + 3;
    auto bound = [&]() {
        return fixed_b2 >= 0.f ? fminf(nn.slot >= 0 ? __double2float_ru(nn.bk) : INFINITY, fixed_b2) : nn_bound(a, nn);
    };
    auto in_box = [&](int dx, int dy, int dz) {
        const int x = qc.c[0] + dx, y = qc.c[1] + dy, z = qc.c[2] + dz;
        return x >= blo[0] && x <= bhi[0] && y >= blo[1] && y <= bhi[1] && z >= blo[2] && z <= bhi[2];
    };
    // shells 0..kWarpShells, nearest first
    for (int m = 1; m <= kWarpShells; ++m) {
        const int cnt = m == 1 ? 27 : shell_count(m);
        for (int t0 = 0; t0 < cnt; t0 += 32) {
            const float b = bound();
            const int t = t0 + lane;
            int dx = 0, dy = 0, dz = 0;
            bool valid = t < cnt;
            if (valid) {
                if (m == 1) {
                    if (t > 0) shell_cell(1, t - 1, dx, dy, dz);
                } else {
                    shell_cell(m, t, dx, dy, dz);
                }
                valid = in_box(dx, dy, dz) && qc.gap2(dx, 0) + qc.gap2(dy, 1) + qc.gap2(dz, 2) <= b;
            }
            if (!__any_sync(0xffffffffu, valid)) continue;
            warp_scan_cells(a, idx, qc, valid, dx, dy, dz, q, nn, lane, excl);
        }
        // shells 0..m done: every unvisited point is >= certified_key(m) away
        if (bound() < qc.certified_key(m) || qc.covers(m, blo, bhi)) return;
    }
    // the rest of the ball: the box of offsets whose gaps fit the bound, outside the shells
    const float b0 = bound();
    int lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) axis_range(qc, k, b0, blo[k], bhi[k], lo[k], hi[k]);
    const int nx = max(hi[0] - lo[0] + 1, 0), ny = max(hi[1] - lo[1] + 1, 0), nz = max(hi[2] - lo[2] + 1, 0);
    const long long total = (long long)nx * ny * nz;
    for (long long t0 = 0; t0 < total; t0 += 32) {
        const float b = bound();
        const long long t = t0 + lane;
        int dx = 0, dy = 0, dz = 0;
        bool valid = t < total;
        if (valid) {
            dx = lo[0] + (int)(t % nx);
            dy = lo[1] + (int)((t / nx) % ny);
            dz = lo[2] + (int)(t / ((long long)nx * ny));
            valid = max(abs(dx), max(abs(dy), abs(dz))) > kWarpShells &&
                    qc.gap2(dx, 0) + qc.gap2(dy, 1) + qc.gap2(dz, 2) <= b;
        }
        if (!__any_sync(0xffffffffu, valid)) continue;
        warp_scan_cells(a, idx, qc, valid, dx, dy, dz, q, nn, lane, excl);
    }
}

#ifndef GSICP_ALIGN_FUSED
#define GSICP_ALIGN_FUSED 1  // k_align's queue: one traversal for the 1-NN and the second-neighbour bound
#endif
// Fused 1-NN + second neighbour for a queued point whose warm start lies inside r (k_align's
// late iterations: near-ties, the warm start is (almost) the 1-NN): ONE traversal of the cells
// within sqrt(Bw) of q, Bw = rho_w^2 with rho_w the reuse radius of the warm start (>= that of the
// 1-NN: the radius is monotone in the key), every target there ranked by (key64, index) with the
// lane's best and second-best key kept in registers and one warp reduction at the end.  The best
// is the exact 1-NN (closer than the warm start, so inside rho_w); k2, the second-best key, is
// the nearest other target whenever that lies within rho_w — so min(sqrt(k2), rho) equals
// warp_nn(rho^2, excl = 1-NN)'s bound.  nn in: the warm start; out: the 1-NN.
__device__ __forceinline__ void warp_nn_top2(const AlignArgs &a, const CellIndex &idx, const int *sb, const Qry &q,
                                             NN &nn, int lane, float Bw, double &k2) {
    const QueryCell qc(q.x, q.y, q.z, a.h, a.inv_h);
    const int *blo = sb, *bhi = sb + 3;
    double lk1 = INFINITY, lk2 = INFINITY;
    uint32_t li1 = 0xffffffffu, ls1 = 0;
    float4 lp1 = make_float4(0.f, 0.f, 0.f, 0.f);
    auto scan = [&](bool valid, int dx, int dy, int dz) {
        const uint2 se = valid ? idx.one(qc.c[0] + dx, qc.c[1] + dy, qc.c[2] + dz) : make_uint2(0u, 0u);
        uint32_t incl = se.y;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t ctot = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t base = 0; base < ctot; base += 32) {
            const uint32_t item = base + lane;
            int l0 = 0, l1 = 31;
#pragma unroll
            for (int s = 0; s < 5; ++s) {
                const int mid = (l0 + l1) >> 1;
                if (__shfl_sync(0xffffffffu, incl, mid) > item) l1 = mid; else l0 = mid + 1;
            }
            const uint32_t c_incl = __shfl_sync(0xffffffffu, incl, l0);
            const uint32_t c_start = __shfl_sync(0xffffffffu, se.x, l0);
            const uint32_t c_cnt = __shfl_sync(0xffffffffu, se.y, l0);
            if (item < ctot) {
                const uint32_t slot = c_start + (item - (c_incl - c_cnt));
                const float4 p = __ldg(a.tpos + slot);
                const double ck = q.key(p);
                const uint32_t ci = (uint32_t)__float_as_int(p.w);
                if (ck < lk1 || (ck == lk1 && ci < li1)) {
                    lk2 = lk1;
                    lk1 = ck;
                    li1 = ci;
                    ls1 = slot;
                    lp1 = p;
                } else if (ck < lk2) {
                    lk2 = ck;
                }
            }
        }
    };
    auto in_box = [&](int dx, int dy, int dz) {
        const int x = qc.c[0] + dx, y = qc.c[1] + dy, z = qc.c[2] + dz;
        return x >= blo[0] && x <= bhi[0] && y >= blo[1] && y <= bhi[1] && z >= blo[2] && z <= bhi[2];
    };
    bool done = false;
    for (int m = 1; m <= kWarpShells && !done; ++m) {
        const int cnt = m == 1 ? 27 : shell_count(m);
        for (int t0 = 0; t0 < cnt; t0 += 32) {
            const int t = t0 + lane;
            int dx = 0, dy = 0, dz = 0;
            bool valid = t < cnt;
            if (valid) {
                if (m == 1) {
                    if (t > 0) shell_cell(1, t - 1, dx, dy, dz);
                } else {
                    shell_cell(m, t, dx, dy, dz);
                }
                valid = in_box(dx, dy, dz) && qc.gap2(dx, 0) + qc.gap2(dy, 1) + qc.gap2(dz, 2) <= Bw;
            }
            if (!__any_sync(0xffffffffu, valid)) continue;
            scan(valid, dx, dy, dz);
        }
        done = Bw < qc.certified_key(m) || qc.covers(m, blo, bhi);
    }
    if (!done) {  // the rest of the ball: the box of offsets whose gaps fit Bw, outside the shells
        int lo[3], hi[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) axis_range(qc, k, Bw, blo[k], bhi[k], lo[k], hi[k]);
        const int nx = max(hi[0] - lo[0] + 1, 0), ny = max(hi[1] - lo[1] + 1, 0), nz = max(hi[2] - lo[2] + 1, 0);
        const long long total = (long long)nx * ny * nz;
        for (long long t0 = 0; t0 < total; t0 += 32) {
            const long long t = t0 + lane;
            int dx = 0, dy = 0, dz = 0;
            bool valid = t < total;
            if (valid) {
                dx = lo[0] + (int)(t % nx);
                dy = lo[1] + (int)((t / nx) % ny);
                dz = lo[2] + (int)(t / ((long long)nx * ny));
                valid = max(abs(dx), max(abs(dy), abs(dz))) > kWarpShells &&
                        qc.gap2(dx, 0) + qc.gap2(dy, 1) + qc.gap2(dz, 2) <= Bw;
            }
            if (!__any_sync(0xffffffffu, valid)) continue;
            scan(valid, dx, dy, dz);
        }
    }
    double mk = lk1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mk = fmin(mk, shfl_f64(mk, lane ^ o));
    const uint32_t mi = __reduce_min_sync(0xffffffffu, lk1 == mk ? li1 : 0xffffffffu);
    const int src = __ffs(__ballot_sync(0xffffffffu, lk1 == mk && li1 == mi)) - 1;
    double o2 = lane == src ? lk2 : lk1;  // every lane's best is "another target" except the winner's
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) o2 = fmin(o2, shfl_f64(o2, lane ^ o));
    k2 = o2;
    if (mk < INFINITY) {
        nn.bk = mk;
        nn.bi = mi;
        nn.slot = (int)__shfl_sync(0xffffffffu, ls1, src);
        nn.p.x = __shfl_sync(0xffffffffu, lp1.x, src);
        nn.p.y = __shfl_sync(0xffffffffu, lp1.y, src);
        nn.p.z = __shfl_sync(0xffffffffu, lp1.z, src);
        nn.p.w = __shfl_sync(0xffffffffu, lp1.w, src);
    }
}

// K3 transform: q_r = ((R_r0 x + R_r1 y) + R_r2 z) + t_r, binary64, no contraction (R15)
__device__ __forceinline__ void k3(const double *T, float x, float y, float z, double &q0, double &q1, double &q2) {
    const double xd = x, yd = y, zd = z;
    q0 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(T[0], xd), __dmul_rn(T[1], yd)), __dmul_rn(T[2], zd)), T[3]);
    q1 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(T[4], xd), __dmul_rn(T[5], yd)), __dmul_rn(T[6], zd)), T[7]);
    q2 = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(T[8], xd), __dmul_rn(T[9], yd)), __dmul_rn(T[10], zd)), T[11]);
}

#ifndef GSICP_TERMS_STRUCTURED
#define GSICP_TERMS_STRUCTURED 1
#endif
// Eq. 1 terms of one valid pair (binary64).  Returns false if Sigma is not positive definite.
__device__ __forceinline__ bool pair_terms(const double *T, double q0, double q1, double q2, float4 ca, float4 cb,
                                           float4 m, float4 ta, float4 tb, double *acc) {
    const double Cs[3][3] = {{ca.x, ca.y, ca.z}, {ca.y, ca.w, cb.x}, {ca.z, cb.x, cb.y}};
    const double R[3][3] = {{T[0], T[1], T[2]}, {T[4], T[5], T[6]}, {T[8], T[9], T[10]}};
    double RC[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) RC[r][c] = R[r][0] * Cs[0][c] + R[r][1] * Cs[1][c] + R[r][2] * Cs[2][c];
    double S[6];
    const int ri[6] = {0, 0, 0, 1, 1, 2}, ci[6] = {0, 1, 2, 1, 2, 2};
    const double Ct[6] = {ta.x, ta.y, ta.z, ta.w, tb.x, tb.y};
#pragma unroll
    for (int e = 0; e < 6; ++e)
        S[e] = Ct[e] + RC[ri[e]][0] * R[ci[e]][0] + RC[ri[e]][1] * R[ci[e]][1] + RC[ri[e]][2] * R[ci[e]][2];
    // M = S^{-1} by the adjugate
    const double A00 = S[3] * S[5] - S[4] * S[4];
    const double A01 = S[2] * S[4] - S[1] * S[5];
    const double A02 = S[1] * S[4] - S[2] * S[3];
    const double A11 = S[0] * S[5] - S[2] * S[2];
    const double A12 = S[1] * S[2] - S[0] * S[4];
    const double A22 = S[0] * S[3] - S[1] * S[1];
    const double det = S[0] * A00 + S[1] * A01 + S[2] * A02;
    if (!(det > 0.0)) return false;
    const double id = 1.0 / det;
    const double M[3][3] = {{A00 * id, A01 * id, A02 * id}, {A01 * id, A11 * id, A12 * id}, {A02 * id, A12 * id, A22 * id}};
    const double d[3] = {(double)m.x - q0, (double)m.y - q1, (double)m.z - q2};
#if GSICP_TERMS_STRUCTURED
    // J = [A | -I] with A = -[q]x (columns (0, q2, -q1), (-q2, 0, q0), (q1, -q0, 0)): the products
    // with J's literal zeros and -1 written out (IEEE arithmetic cannot drop x * 0.0 by itself),
    // H = [[A^T M A, -A^T M], [-M A, M]], b = [A^T M d; -M d] — the same sums without the zero terms
    double MA[3][3], AtM[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        MA[r][0] = M[r][1] * q2 - M[r][2] * q1;
        MA[r][1] = M[r][2] * q0 - M[r][0] * q2;
        MA[r][2] = M[r][0] * q1 - M[r][1] * q0;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {  // (A^T M)[r][c] = sum_k A[k][r] M[k][c]
        AtM[0][c] = q2 * M[1][c] - q1 * M[2][c];
        AtM[1][c] = q0 * M[2][c] - q2 * M[0][c];
        AtM[2][c] = q1 * M[0][c] - q0 * M[1][c];
    }
    double AtMA[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        AtMA[0][c] = q2 * MA[1][c] - q1 * MA[2][c];
        AtMA[1][c] = q0 * MA[2][c] - q2 * MA[0][c];
        AtMA[2][c] = q1 * MA[0][c] - q0 * MA[1][c];
    }
    const double Md[3] = {M[0][0] * d[0] + M[0][1] * d[1] + M[0][2] * d[2], M[1][0] * d[0] + M[1][1] * d[1] + M[1][2] * d[2],
                          M[2][0] * d[0] + M[2][1] * d[1] + M[2][2] * d[2]};
    int t = 0;
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = r; c < 6; ++c)
            acc[t++] += r < 3 ? (c < 3 ? AtMA[r][c] : -AtM[r][c - 3]) : M[r - 3][c - 3];
    acc[21] += q2 * Md[1] - q1 * Md[2];
    acc[22] += q0 * Md[2] - q2 * Md[0];
    acc[23] += q1 * Md[0] - q0 * Md[1];
    acc[24] -= Md[0];
    acc[25] -= Md[1];
    acc[26] -= Md[2];
    acc[27] += d[0] * Md[0] + d[1] * Md[1] + d[2] * Md[2];
#else
    const double J[3][6] = {{0.0, -q2, q1, -1.0, 0.0, 0.0}, {q2, 0.0, -q0, 0.0, -1.0, 0.0}, {-q1, q0, 0.0, 0.0, 0.0, -1.0}};
    double MJ[3][6], Md[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
        for (int c = 0; c < 6; ++c) MJ[r][c] = M[r][0] * J[0][c] + M[r][1] * J[1][c] + M[r][2] * J[2][c];
        Md[r] = M[r][0] * d[0] + M[r][1] * d[1] + M[r][2] * d[2];
    }
    int t = 0;
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = r; c < 6; ++c) acc[t++] += J[0][r] * MJ[0][c] + J[1][r] * MJ[1][c] + J[2][r] * MJ[2][c];
#pragma unroll
    for (int r = 0; r < 6; ++r) acc[21 + r] += J[0][r] * Md[0] + J[1][r] * Md[1] + J[2][r] * Md[2];
    acc[27] += d[0] * Md[0] + d[1] * Md[1] + d[2] * Md[2];
#endif
    acc[28] += 1.0;
    return true;
}

__device__ __forceinline__ void so3_exp(const double *w, double *R) {
    const double th2 = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
    const double th = sqrt(th2);
    double A, B;
    if (th < 1e-8) {
        A = 1.0;
        B = 0.5;
    } else {
        double sn, cs;
        sincos(th, &sn, &cs);  // one shared range reduction on the solve's serial path
        A = sn / th;
        B = (1.0 - cs) / th2;
    }
    const double K[9] = {0, -w[2], w[1], w[2], 0, -w[0], -w[1], w[0], 0};
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            const double k2 = K[3 * r] * K[c] + K[3 * r + 1] * K[3 + c] + K[3 * r + 2] * K[6 + c];
            R[3 * r + c] = (r == c ? 1.0 : 0.0) + A * K[3 * r + c] + B * k2;
        }
}

// 6x6 Cholesky solve with one reciprocal square root per pivot (the serial latency of the solve
// sits on every GN iteration's critical path); fully unrolled so L stays in registers.
__device__ __forceinline__ bool chol6_solve(const double *H, const double *rhs, double *x) {
    double L[6][6], inv_d[6];
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double s = H[6 * i + j];
#pragma unroll
            for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
            if (i == j) {
                ok = ok && s > 0.0;
                inv_d[i] = rsqrt(s);
                L[i][i] = s * inv_d[i];
            } else {
                L[i][j] = s * inv_d[j];
            }
        }
    if (!ok) return false;
    double y[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        double s = rhs[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s -= L[i][k] * y[k];
        y[i] = s * inv_d[i];
    }
#pragma unroll
    for (int i = 5; i >= 0; --i) {
        double s = y[i];
#pragma unroll
        for (int k = i + 1; k < 6; ++k) s -= L[k][i] * x[k];
        x[i] = s * inv_d[i];
    }
    return true;
}

// A8 for one block (thread 0): solve H delta = -b, update the shared pose, convergence test.
// Out of line: its ~150 live doubles must not raise the register pressure of the point loop.
// Returns 1 when the loop is done (status set).
// LM state kept by every block (identical): [0,12) kept pose, [12,41) its linearisation terms
// (sAcc layout), [41] lambda, [42] 1 once a pose was kept
constexpr int kLmState = 44;

template <bool LM>
__device__ __forceinline__ int solve_step_t(const AlignArgs &a, const double *sAcc, double *sT, int it, int n,
                                         int &status, int &iters, int &converged, double *sLM) {
    double H[36], b[6];
    int t = 0;
    for (int r = 0; r < 6; ++r)
        for (int c = r; c < 6; ++c) H[6 * r + c] = H[6 * c + r] = sAcc[t++];
    for (int r = 0; r < 6; ++r) b[r] = sAcc[21 + r];
    const double n_in = sAcc[28];
    if (a.linearize_only) {
        if (blockIdx.x == 0) {
            for (int k = 0; k < 36; ++k) a.d_lin[k] = H[k];
            for (int k = 0; k < 6; ++k) a.d_lin[36 + k] = b[k];
            a.d_lin[42] = sAcc[27];
            a.d_lin[43] = n_in;
        }
        status = GSICP_OK;
        return 1;
    }
    if (n == 0) {
        status = GSICP_ERR_DEGENERATE_FRAME;
        return 1;
    }
    if constexpr (LM) {
        // Levenberg-Marquardt (R30): keep the trial pose iff its cost beats the kept one
        const bool enough = n_in >= (double)a.min_pairs;
        const bool accept = it == 0 ? enough : (enough && sAcc[27] < sLM[12 + 27]);
        if (it == 0 && !accept) {
            status = GSICP_ERR_TRACKING_LOST;
            return 1;
        }
        if (accept) {
            for (int k = 0; k < 12; ++k) sLM[k] = sT[k];
            for (int k = 0; k < 29; ++k) sLM[12 + k] = sAcc[k];
            sLM[41] = it == 0 ? a.lm_lambda0 : sLM[41] / 10.0;
            sLM[42] = 1.0;
        } else {
            sLM[41] = sLM[41] * 10.0;
        }
        t = 0;
        for (int r = 0; r < 6; ++r)
            for (int c = r; c < 6; ++c) H[6 * r + c] = H[6 * c + r] = sLM[12 + t++];
        for (int r = 0; r < 6; ++r) b[r] = sLM[12 + 21 + r];
        for (int k = 0; k < 6; ++k) H[7 * k] = H[7 * k] + sLM[41] * H[7 * k];
        for (int k = 0; k < 12; ++k) sT[k] = sLM[k];  // the step starts from the kept pose
    } else if (n_in < (double)a.min_pairs) {
        status = GSICP_ERR_TRACKING_LOST;
        return 1;
    }
    double nb[6], delta[6];
    for (int k = 0; k < 6; ++k) nb[k] = -b[k];
    bool ok = chol6_solve(H, nb, delta);
    if (!ok) {
        double tr = 0.0;
        for (int k = 0; k < 6; ++k) tr += H[7 * k];
        for (int k = 0; k < 6; ++k) H[7 * k] += 1e-6 * tr / 6.0;
        ok = chol6_solve(H, nb, delta);
    }
    if (!ok) {
        status = GSICP_ERR_TRACKING_LOST;
        return 1;  // (LM: sT already holds the kept pose)
    }
    double E[9];
    so3_exp(delta, E);
    double Tn[12];
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) Tn[4 * r + c] = E[3 * r] * sT[c] + E[3 * r + 1] * sT[4 + c] + E[3 * r + 2] * sT[8 + c];
        Tn[4 * r + 3] = E[3 * r] * sT[3] + E[3 * r + 1] * sT[7] + E[3 * r + 2] * sT[11] + delta[3 + r];
    }
    for (int k = 0; k < 12; ++k) sT[k] = Tn[k];
    iters = it + 1;
    const double nw = sqrt(delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2]);
    const double nv = sqrt(delta[3] * delta[3] + delta[4] * delta[4] + delta[5] * delta[5]);
    if (nw < a.eps_rot && nv < a.eps_trans) {
        converged = 1;
        status = GSICP_OK;
        return 1;
    }
    if (iters >= a.max_iters) {
        status = GSICP_WARN_MAX_ITERS;
        if constexpr (LM)
            for (int k = 0; k < 12; ++k) sT[k] = sLM[k];  // the best kept iterate
        return 1;
    }
    return 0;
}

// No warm start: the own cell's best becomes the candidate; an empty own cell is seeded from
// the 6 face neighbours (the graph step then needs some candidate to start from).
__device__ __forceinline__ void nn_cold_start(const AlignArgs &a, const CellIndex &idx, const QueryCell &qc, uint2 own,
                                              const Qry &q, NN &nn) {
    scan_target_cell(a, own, q, nn);
    for (int f0 = 0; f0 < 6 && nn.slot < 0; f0 += kMaxCells) {
        int xs[kMaxCells], ys[kMaxCells], zs[kMaxCells];
        bool valid[kMaxCells];
        float lbs[kMaxCells];
#pragma unroll
        for (int u = 0; u < kMaxCells; ++u) {
            int dx = 0, dy = 0, dz = 0;
            valid[u] = f0 + u < 6;
            if (valid[u]) shell_cell(1, f0 + u, dx, dy, dz);
            xs[u] = qc.c[0] + dx;
            ys[u] = qc.c[1] + dy;
            zs[u] = qc.c[2] + dz;
            lbs[u] = 0.f;
        }
        uint2 se[kMaxCells];
        idx.batch(xs, ys, zs, valid, se);
        scan_cells_flat(a, se, lbs, q, nn);
    }
}

__device__ __forceinline__ void load_cell_index(const AlignArgs &a, CellIndex &idx, int *box) {
    idx.table = a.table;
    idx.mask = a.mask;
    idx.level = 0;
    idx.dense = a.dense;
    idx.use_dense = a.dense != nullptr && a.dense_hdr[0] != 0;
    for (int k = 0; k < 3; ++k) {
        idx.lo[k] = a.dense_hdr ? a.dense_hdr[1 + k] : 0;
        idx.dim[k] = a.dense_hdr ? a.dense_hdr[4 + k] : 0;
    }
    for (int k = 0; k < 6; ++k) box[k] = cell_coord(ordered_to_float_(a.tbbox[k]), a.inv_h);
}

// Iteration-0 correspondences ahead of the GN loop (gsicp_align_seed): exact 1-NN of
// K3(T0, x_i) (binary64, R15) for every source point, by the same search as k_align's first iteration
// (cold start, certified graph descent, fast path, block queue solved by whole warps).  It needs
// only the source positions, so it can run concurrently with the source covariances (A2-A4).
constexpr int kSeedT = 256;
constexpr int kSeedHardT = 128;
__global__ void __launch_bounds__(kSeedT) k_align_seed(AlignArgs a) {
    __shared__ double sT[12];
    __shared__ int sBox[6];
    __shared__ CellIndex sIdx;
    const int tid = threadIdx.x;
    const int n = *a.d_n;
    if (tid < 12) sT[tid] = a.d_T[tid];
    if (tid == 0) load_cell_index(a, sIdx, sBox);
    __syncthreads();
    const int i = blockIdx.x * kSeedT + tid;
    if (i < n) {
        const float4 x = __ldg(a.spos + i);
        double q0, q1, q2;
        k3(sT, x.x, x.y, x.z, q0, q1, q2);
        const Qry q(q0, q1, q2);
        const QueryCell qc(q.x, q.y, q.z, a.h, a.inv_h);
        const uint2 own = sIdx.one(qc.c[0], qc.c[1], qc.c[2]);
        NN nn;
        uint2 own_left = own;
        if (a.nbr) {
            nn_cold_start(a, sIdx, qc, own, q, nn);
            own_left = make_uint2(0u, 0u);
        }
        float d2 = 0.f;
        // per thread only the cheap certified case (own cell, then the graph); everything else
        // goes to the warp-cooperative pass (no divergent per-thread grid walks here)
        bool exact = nn.slot >= 0 && a.nbr && graph_nn(a, q, nn, d2);
        if (!exact && !a.nbr) exact = nn_search(a, sIdx, sBox, qc, own_left, q, nn, true);
        a.seed_slot[i] = nn.slot;  // exact, or the best seen (an upper bound for the hard pass)
        if (!exact) a.seed_queue[atomicAdd(a.seed_qn, 1)] = i;
    }
    if (blockIdx.x == 0 && tid < 12) a.seed_hdr[tid] = sT[tid];
    if (blockIdx.x == 0 && tid == 12) a.seed_hdr[12] = a.seed_ticket;
}

// The hard queries of the seed pass, spread over the whole GPU: each warp takes queue entries
// (one query each) and runs the warp-cooperative exact search from the best seen so far.
__global__ void __launch_bounds__(kSeedHardT) k_align_seed_hard(AlignArgs a) {
    __shared__ double sT[12];
    __shared__ int sBox[6];
    __shared__ CellIndex sIdx;
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid < 12) sT[tid] = a.d_T[tid];
    if (tid == 0) load_cell_index(a, sIdx, sBox);
    __syncthreads();
    const int qn = *a.seed_qn;
    const int warps = gridDim.x * (kSeedHardT / 32);
    for (int k = blockIdx.x * (kSeedHardT / 32) + (tid >> 5); k < qn; k += warps) {
        const int i = a.seed_queue[k];
        const float4 x = __ldg(a.spos + i);
        double q0, q1, q2;
        k3(sT, x.x, x.y, x.z, q0, q1, q2);
        const Qry q(q0, q1, q2);
        NN nn;
        const int sl = a.seed_slot[i];
        if (sl >= 0) {
            const float4 rec = __ldg(a.tpos + sl);
            nn.set(q.key(rec), sl, rec);
        }
        warp_nn(a, sIdx, sBox, q, nn, lane);
        if (lane == 0) a.seed_slot[i] = nn.slot;
    }
}

__global__ void k_align_init(int32_t *corr_ws, float4 *reuse_ws, int cap, unsigned int *barrier) {
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cap) {
        corr_ws[i] = -1;
        reuse_ws[i] = make_float4(0.f, 0.f, 0.f, 0.f);  // d2lb = 0: no reuse
    }
    if (i == 0) *barrier = 0u;
}

// The GN loop of one frame on blocks [0, G) of its own (bid = this block's index among them):
// k_align runs one frame on the whole grid, k_align_batch several frames side by side.
// LM: the solver is a template parameter, so the GN kernel carries no LM code (measured: an
// inlined run-time branch cost the GN loop ~3 us per frame through register allocation)
template <bool LM>
__device__ __forceinline__ void align_body(const AlignArgs &a, const int bid, const int G) {
    __shared__ double sT[12];
    __shared__ double sRed[kWarps][kPad];
    __shared__ double sAcc[kPad];
    __shared__ int sDone;
    __shared__ double sLM[kLmState];
    __shared__ int sBox[6];
    __shared__ CellIndex sIdx;
    // per-block queue of queries needing the general search (handled by whole warps)
    __shared__ int sQn, sQn2;
    __shared__ int sQtid[kT];
    __shared__ double4 sQq[kT];
    __shared__ double sQbk[kT];
    __shared__ int sQslot[kT];
    __shared__ float4 sQp[kT];
    __shared__ float sQd2[kT];
    __shared__ unsigned char sQrep[kT];  // the point was queued in the previous iteration too
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = *a.d_n;
    if (tid < 12) sT[tid] = a.d_T[tid];
    if (a.timeline && bid == 0 && tid == 0 && a.timeline_cap > 0) a.timeline[0] = globaltimer_ns();
    __shared__ int sSeeded;
    if (tid == 0) {
        load_cell_index(a, sIdx, sBox);
        // seeds are used only if they were computed at exactly this pose (and not consumed yet)
        bool ok = a.seed_ticket > 0.0 && a.seed_hdr[12] == a.seed_ticket;
        for (int k = 0; k < 12; ++k) ok = ok && __double_as_longlong(a.seed_hdr[k]) == __double_as_longlong(a.d_T[k]);
        sSeeded = ok;
    }
    if (tid == 0) sDone = 0;
    if (tid == 0) sLM[42] = 0.0;
    if (tid == 0) sQn = 0;
    // resident point of this thread: source data, current match and own target cell in registers
    // resident points: block b owns the contiguous chunk [b P, b P + P), P = ceil(n / G) (at most
    // kT): the whole co-resident grid shares the points — and the hard queries each block's warps
    // search — however small the frame is (one block per kT points left most SMs idle and piled
    // the warp searches of a noisy frame onto a few blocks)
    const int P = min(kT, (n + G - 1) / G);
    const int i0 = P == kT ? bid * kT + tid : bid * P + tid;
    const bool has0 = tid < P && i0 < n;
    float4 x0 = make_float4(0.f, 0.f, 0.f, 0.f), ca0 = x0, cb0 = x0;
    if (has0) {
        x0 = __ldg(a.spos + i0);
        ca0 = __ldg(a.scov_a + i0);
        cb0 = __ldg(a.scov_b + i0);
    }
    NN m0;                                // warm start carried across iterations
    float4 ta0 = x0, tb0 = x0;            // covariance of m0.slot (valid iff cov_slot == m0.slot)
    int cov_slot = -1;
    int own_c[3] = {INT_MIN, INT_MIN, INT_MIN};
    uint2 own_se = make_uint2(0u, 0u);
    bool valid0 = false;
    float d2lb = 0.f, qp0 = 0.f, qp1 = 0.f, qp2 = 0.f;  // reuse state: 2nd-NN distance bound at qp
    int dbg_slow = 0, dbg_reuse = 0, dbg_graph = 0, dbg_its = 0;
    __syncthreads();
    int status = GSICP_WARN_MAX_ITERS, iters = 0, converged = 0;
    double n_in = 0.0, cost_last = 0.0;
    for (int it = 0;; ++it) {
        // diagnostic phase stamps of block 0 (only when a timeline is attached; uniform branch)
        auto stamp = [&](int p) {
            if (a.timeline) {
                __syncthreads();
                const long long idx = 1 + (long long)a.max_iters * (G + 1) + (long long)it * 8 + p;
                if (bid == 0 && tid == 0 && idx < a.timeline_cap) a.timeline[idx] = globaltimer_ns();
            }
        };
        stamp(0);
        const double *T = sT;  // read from shared memory at each use (keeps registers for the search)
        // ------------------------------------------------------------ A6: correspondences
        double q0r = 0.0, q1r = 0.0, q2r = 0.0;
        // diagnostic sub-phase clocks of warp 0 of block 0 (SM cycles)
        const bool sub = a.timeline && bid == 0 && tid == 0;
        const long long sub_base = 1 + (long long)a.max_iters * (G + 9) + (long long)it * 8;
        auto sub_stamp = [&](int k) {
            if (sub && sub_base + k < a.timeline_cap) a.timeline[sub_base + k] = clock64();
        };
        const long long lane_t0 = a.timeline && bid == 0 ? clock64() : 0;
        int path_code = 0;
        if (has0) {
            sub_stamp(0);
            k3(T, x0.x, x0.y, x0.z, q0r, q1r, q2r);
            const Qry q(q0r, q1r, q2r);
            const QueryCell qc(q.x, q.y, q.z, a.h, a.inv_h);
            if (qc.c[0] != own_c[0] || qc.c[1] != own_c[1] || qc.c[2] != own_c[2]) {
                own_c[0] = qc.c[0]; own_c[1] = qc.c[1]; own_c[2] = qc.c[2];
                own_se = sIdx.one(qc.c[0], qc.c[1], qc.c[2]);
            }
            if (sub) own_se.x += 0 * (uint32_t)clock();  // keep ordering of the stamp below
            sub_stamp(1);
            NN nn;
            const bool seeded0 = it == 0 && sSeeded;
            if (seeded0) {  // exact match at this pose computed ahead by k_align_seed
                const int sl = __ldg(a.seed_slot + i0);
                if (sl >= 0) {
                    const float4 rec = __ldg(a.tpos + sl);
                    nn.set(q.key(rec), sl, rec);
                }
            } else if (m0.slot >= 0) {  // warm start from the previous match (record kept in registers)
                nn.set(q.key(m0.p), m0.slot, m0.p);
            }
            bool exact = seeded0;
            // motion-bounded reuse: the query moved by delta since the match was proven, with
            // every other target >= d2lb away then, so |q' - m_k| >= d2lb - delta for all k != m;
            // if |q' - m| < d2lb - delta the match stands (no loads).  delta is measured between the
            // binary32 roundings of the two binary64 queries, plus their rounding (2 E)
            if (!exact && d2lb > 0.f) {
                const float ex = q.x - qp0, ey = q.y - qp1, ez = q.z - qp2;
                const float delta = sqrtf(ex * ex + ey * ey + ez * ez) * (1.f + kReuseMargin) + 2.f * q.E();
                // d2lb bounds every target other than the candidate: beating d1 proves the
                // candidate is the 1-NN, or (candidate absent or beyond r) that the point stays gated
                const float d1 = nn.slot >= 0 ? fminf(sqrtf(__double2float_ru(nn.bk)), a.r) : a.r;
                if ((d2lb - delta) * (1.f - kReuseMargin) > d1 * (1.f + kReuseMargin)) {
                    exact = true;
                    d2lb -= delta;
                    dbg_reuse |= 1 << (it & 31);
                }
            }
            if (!exact) d2lb = 0.f;
            sub_stamp(2);
            uint2 own_left = own_se;
            if (!exact && nn.slot < 0 && a.nbr) {  // no warm start: the own cell's best becomes the candidate
                nn_cold_start(a, sIdx, qc, own_se, q, nn);
                own_left = make_uint2(0u, 0u);
            } else if (!exact && a.nbr && nn.bk > 0.25 * (double)a.h * (double)a.h) {
                // the query moved more than half a cell from its previous match (the large early
                // pose updates): start the graph descent from the best of the own cell as well
                // (one cached lookup, one cell of records) instead of walking from the far match
                scan_target_cell(a, own_se, q, nn);
                own_left = make_uint2(0u, 0u);
            }
            path_code = exact ? (seeded0 ? 4 : 0) : 1;
            if (!exact && nn.slot >= 0 && a.nbr) {
                exact = graph_nn(a, q, nn, d2lb);
                dbg_graph |= (exact ? 1 : 0) << (it & 31);
                path_code = exact ? 1 : 2;
            }
            // after iteration 0 a point the graph cannot certify goes straight to the block queue:
            // the warp path also bounds its second neighbour, so the next iterations can reuse
            // (measured: the per-thread cell path here instead is slower, 227 -> 267 us, because
            // the points then lose the second-neighbour bound and fail the reuse test later)
            if (!exact && (it == 0 || !a.nbr)) {
                exact = nn_search(a, sIdx, sBox, qc, own_left, q, nn, true);
                path_code = exact ? 2 : 3;
            }
            if (!exact) path_code = 3;
            qp0 = q.x;
            qp1 = q.y;
            qp2 = q.z;
            if (sub) a.timeline[sub_base + 4] = nn.slot < 0 ? 1 : 0;
            sub_stamp(3);
            if (!exact) {  // hand over to the block's warps (warp_nn below)
                const int k = atomicAdd(&sQn, 1);
                sQtid[k] = tid;
                sQq[k] = make_double4(q0r, q1r, q2r, 0.0);
                sQbk[k] = nn.bk;
                sQslot[k] = nn.slot;
                sQp[k] = nn.p;
                sQrep[k] = it > 0 && it <= 32 ? (unsigned char)((dbg_slow >> ((it - 1) & 31)) & 1) : 0;
            }
            dbg_slow |= (exact ? 0 : 1) << (it & 31);
            ++dbg_its;
            m0 = nn;
        }
        if (a.timeline && bid == 0) {  // diagnostic: slowest lane of each warp of block 0
            long long d = has0 ? clock64() - lane_t0 : 0;
            int code = path_code;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const long long od = __shfl_xor_sync(0xffffffffu, d, o);
                const int oc = __shfl_xor_sync(0xffffffffu, code, o);
                if (od > d) {
                    d = od;
                    code = oc;
                }
            }
            const long long wb = 1 + (long long)a.max_iters * (G + 17) + ((long long)it * kWarps + warp) * 2;
            if (lane == 0 && wb + 1 < a.timeline_cap) {
                a.timeline[wb] = d;
                a.timeline[wb + 1] = code;
            }
        }
        // queries whose fast path failed: one warp each, all lanes cooperating
        __syncthreads();
        for (int k = warp; k < sQn; k += kWarps) {
            const double4 qq = sQq[k];
            const Qry q(qq.x, qq.y, qq.z);
            NN nn;
            nn.slot = sQslot[k];
            if (nn.slot >= 0) nn.set(sQbk[k], nn.slot, sQp[k]);
            float d2 = 0.f;
            // (a point queued again — a near-tie whose bound did not hold — gets the second-neighbour
            // bound every other iteration only: its next reuse test is then unlikely to pass anyway)
            const bool skip_d2 = GSICP_D2_SKIP_REPEAT && sQrep[k] && (it & 1);
            // (only for warm starts within one cell of the query: a far one makes the single ball
            // much larger than warp_nn's shrinking one — measured on the noisy C3 frames)
            const bool fuse_ok = GSICP_ALIGN_FUSED && nn.bk < (double)a.h * (double)a.h;
            if (fuse_ok && it >= kD2FromIter && !skip_d2 && nn.slot >= 0 && nn.bk < a.r2) {
                // the 1-NN and the bound from one traversal around the warm start (inside r, so the
                // 1-NN is too: rho below is the same as after a separate warp_nn)
                const float rw = sqrtf(__double2float_ru(nn.bk)) * 1.25f + 0.25f * a.h;
                double k2;
                warp_nn_top2(a, sIdx, sBox, q, nn, lane, rw * rw, k2);
                const float rho = sqrtf(__double2float_ru(nn.bk)) * 1.25f + 0.25f * a.h;
                d2 = fminf(k2 < INFINITY ? sqrtf(__double2float_rd(k2)) : INFINITY, rho) * (1.f - kReuseMargin);
            } else {
                warp_nn(a, sIdx, sBox, q, nn, lane);
                // a lower bound on every other target's distance (exact within rho), so that the
                // following iterations can keep this answer while the query moves little
                const bool in_r = nn.slot >= 0 && nn.bk < a.r2;
                const float base = in_r ? sqrtf(__double2float_ru(nn.bk)) : a.r;
                if (base < INFINITY && it >= kD2FromIter && !skip_d2) {
                    const float rho = base * 1.25f + 0.25f * a.h;
                    NN n2;
                    warp_nn(a, sIdx, sBox, q, n2, lane, rho * rho, nn.slot);
                    d2 = fminf(n2.slot >= 0 ? sqrtf(__double2float_rd(n2.bk)) : INFINITY, rho) * (1.f - kReuseMargin);
                }
            }
            __syncwarp();  // every lane has read entry k (above) before lane 0 overwrites it
            if (lane == 0) {
                sQbk[k] = nn.bk;
                sQslot[k] = nn.slot;
                sQp[k] = nn.p;
                sQd2[k] = d2;
            }
        }
        __syncthreads();
        if (has0) {
            for (int k = 0; k < sQn; ++k)
                if (sQtid[k] == tid) {
                    if (sQslot[k] >= 0) m0.set(sQbk[k], sQslot[k], sQp[k]); else m0.slot = -1;
                    d2lb = sQd2[k];
                }
            valid0 = m0.slot >= 0 && m0.bk < a.r2;
        }
        // non-resident points (clouds larger than the co-resident grid's threads): rounds of one
        // point per thread over this block's chunks, the cheap certified paths per thread and the
        // rest through the same block queue, solved by whole warps
        __syncthreads();  // the resident readback of the queue (above) is done before its reuse
        for (int r = 1;; ++r) {
            const long long cb = ((long long)r * G + bid) * kT;  // this block's chunk (block-uniform)
            if (P < kT || cb >= n) break;
            if (tid == 0) sQn2 = 0;
            __syncthreads();
            const int i = (int)cb + tid;
            if (i < n) {
                const float4 x = __ldg(a.spos + i);
                double q0, q1, q2;
                k3(T, x.x, x.y, x.z, q0, q1, q2);
                const Qry q(q0, q1, q2);
                const QueryCell qc(q.x, q.y, q.z, a.h, a.inv_h);
                NN nn;
                const bool seeded = it == 0 && sSeeded;
                int slot = seeded ? a.seed_slot[i] : a.corr_ws[i];
                if (slot <= -2) slot = -2 - slot;
                if (slot >= 0) {
                    const float4 rec = __ldg(a.tpos + slot);
                    nn.set(q.key(rec), slot, rec);
                }
                bool exact = seeded;
                // the motion-bounded reuse of the resident path, with its state kept in memory
                const float4 ru = seeded ? make_float4(0.f, 0.f, 0.f, 0.f) : a.reuse_ws[i];
                float d2lb = ru.w;
                if (!exact && d2lb > 0.f) {
                    const float ex = q.x - ru.x, ey = q.y - ru.y, ez = q.z - ru.z;
                    const float delta = sqrtf(ex * ex + ey * ey + ez * ez) * (1.f + kReuseMargin) + 2.f * q.E();
                    const float d1 = nn.slot >= 0 ? fminf(sqrtf(__double2float_ru(nn.bk)), a.r) : a.r;
                    if ((d2lb - delta) * (1.f - kReuseMargin) > d1 * (1.f + kReuseMargin)) {
                        exact = true;
                        d2lb -= delta;
                    }
                }
                if (!exact) d2lb = 0.f;
                const uint2 own = exact ? make_uint2(0u, 0u) : sIdx.one(qc.c[0], qc.c[1], qc.c[2]);
                uint2 own_left = own;
                if (!exact && a.nbr && (nn.slot < 0 || nn.bk > 0.25 * (double)a.h * (double)a.h)) {
                    scan_target_cell(a, own, q, nn);  // (as the resident path: a far or absent warm start)
                    own_left = make_uint2(0u, 0u);
                }
                if (!exact && nn.slot >= 0 && a.nbr) exact = graph_nn(a, q, nn, d2lb);
                if (!exact && !a.nbr) exact = nn_search(a, sIdx, sBox, qc, own_left, q, nn, true);
                if (exact) {
                    a.corr_ws[i] = (nn.slot >= 0 && nn.bk < a.r2) ? nn.slot : -2 - nn.slot;
                    a.reuse_ws[i] = make_float4(q.x, q.y, q.z, seeded ? 0.f : d2lb);
                } else {
                    const int k = atomicAdd(&sQn2, 1);
                    sQtid[k] = i;
                    sQq[k] = make_double4(q0, q1, q2, 0.0);
                    sQbk[k] = nn.bk;
                    sQslot[k] = nn.slot;
                    sQp[k] = nn.p;
                }
            }
            __syncthreads();
            for (int k = warp; k < sQn2; k += kWarps) {
                const double4 qq = sQq[k];
                const Qry q(qq.x, qq.y, qq.z);
                NN nn;
                nn.slot = sQslot[k];
                if (nn.slot >= 0) nn.set(sQbk[k], nn.slot, sQp[k]);
                // the second-neighbour bound for the reuse of the next iterations (as resident
                // points, the fused traversal for a near warm start inside r included)
                float d2 = 0.f;
                if (GSICP_ALIGN_FUSED && it >= kD2FromIter && nn.slot >= 0 && nn.bk < a.r2 &&
                    nn.bk < (double)a.h * (double)a.h) {
                    const float rw = sqrtf(__double2float_ru(nn.bk)) * 1.25f + 0.25f * a.h;
                    double k2;
                    warp_nn_top2(a, sIdx, sBox, q, nn, lane, rw * rw, k2);
                    const float rho = sqrtf(__double2float_ru(nn.bk)) * 1.25f + 0.25f * a.h;
                    d2 = fminf(k2 < INFINITY ? sqrtf(__double2float_rd(k2)) : INFINITY, rho) * (1.f - kReuseMargin);
                } else {
                    warp_nn(a, sIdx, sBox, q, nn, lane);
                    const bool in_r0 = nn.slot >= 0 && nn.bk < a.r2;
                    const float base = in_r0 ? sqrtf(__double2float_ru(nn.bk)) : a.r;
                    if (base < INFINITY && it >= kD2FromIter) {
                        const float rho = base * 1.25f + 0.25f * a.h;
                        NN n2;
                        warp_nn(a, sIdx, sBox, q, n2, lane, rho * rho, nn.slot);
                        d2 = fminf(n2.slot >= 0 ? sqrtf(__double2float_rd(n2.bk)) : INFINITY, rho) * (1.f - kReuseMargin);
                    }
                }
                const bool in_r = nn.slot >= 0 && nn.bk < a.r2;
                if (lane == 0) {
                    a.corr_ws[sQtid[k]] = in_r ? nn.slot : -2 - nn.slot;
                    a.reuse_ws[sQtid[k]] = make_float4(q.x, q.y, q.z, d2);
                }
            }
            __syncthreads();  // the queue entries are read before the next round refills them
        }
        sub_stamp(5);
        stamp(1);
        // ------------------------------------------------------------ A7: Eq. 1 terms
        double acc[kAlignTerms];
#pragma unroll
        for (int k = 0; k < kAlignTerms; ++k) acc[k] = 0.0;
        if (has0) {
            int32_t corr_val = -1;
            sub_stamp(6);
            if (valid0) {
                if (cov_slot != m0.slot) {
                    ta0 = __ldg(a.tcov_a + m0.slot);
                    tb0 = __ldg(a.tcov_b + m0.slot);
                    cov_slot = m0.slot;
                }
                if (pair_terms(T, q0r, q1r, q2r, ca0, cb0, m0.p, ta0, tb0, acc)) corr_val = __float_as_int(m0.p.w);
            }
            if (sub) acc[0] += 0.0 * (double)clock();
            sub_stamp(7);
            if (a.corr_out) a.corr_out[i0] = corr_val;
            if (a.iter_corr && it < a.iter_cap) a.iter_corr[(size_t)it * a.cap + i0] = corr_val;
        }
        for (int i = i0 + G * kT; i < n; i += G * kT) {
            const int slot = a.corr_ws[i];
            int32_t corr_val = -1;
            if (slot >= 0) {
                const float4 x = __ldg(a.spos + i);
                double q0, q1, q2;
                k3(T, x.x, x.y, x.z, q0, q1, q2);
                const float4 m = __ldg(a.tpos + slot);
                if (pair_terms(T, q0, q1, q2, __ldg(a.scov_a + i), __ldg(a.scov_b + i), m, __ldg(a.tcov_a + slot),
                               __ldg(a.tcov_b + slot), acc))
                    corr_val = __float_as_int(m.w);
            }
            if (a.corr_out) a.corr_out[i] = corr_val;
            if (a.iter_corr && it < a.iter_cap) a.iter_corr[(size_t)it * a.cap + i] = corr_val;
        }
        stamp(2);
        // ------------------------------------------------------------ block reduction
#pragma unroll
        for (int k = 0; k < kAlignTerms; ++k)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < kAlignTerms; ++k) sRed[warp][k] = acc[k];
        }
        __syncthreads();
        // every thread's reads of the block queue (sQn, above) happened before this barrier
        if (tid == 0) sQn = 0;
        double *part = a.partials + (size_t)(it & 1) * G * kPad;
        if (tid < kAlignTerms) {
            double s = 0.0;
            for (int w = 0; w < kWarps; ++w) s += sRed[w][tid];
            part[(size_t)bid * kPad + tid] = s;
        }
        // ------------------------------------------------------------ grid barrier
        __syncthreads();
        if (tid == 0) {
            const long long rec = 1 + (long long)it * (G + 1);
            if (a.timeline && rec + G < a.timeline_cap) a.timeline[rec + bid] = globaltimer_ns();
            __threadfence();
            atomicAdd(a.barrier, 1u);
            const unsigned int target = (unsigned int)(it + 1) * (unsigned int)G;
            while (ld_acquire(a.barrier) < target) {
            }
            __threadfence();
            if (a.timeline && bid == 0 && rec + G < a.timeline_cap) a.timeline[rec + G] = globaltimer_ns();
        }
        __syncthreads();
        stamp(3);
        // ------------------------------------------------------------ fixed-order final reduction (every block)
        {
            const int grp = tid >> 5;  // kWarps groups stride over the blocks' partials
            double s = 0.0;
            if (lane < kAlignTerms) {
                // all loads of a chunk in flight at once, then summed in block order
                constexpr int kChunk = 16;
                for (int gb0 = grp; gb0 < G; gb0 += kChunk * kWarps) {
                    double v[kChunk];
#pragma unroll
                    for (int j = 0; j < kChunk; ++j) {
                        const int gb = gb0 + j * kWarps;
                        v[j] = gb < G ? __ldcg(part + (size_t)gb * kPad + lane) : 0.0;
                    }
#pragma unroll
                    for (int j = 0; j < kChunk; ++j) s += v[j];
                }
            }
            sRed[grp][lane] = s;
            __syncthreads();
            if (tid < kAlignTerms) {
                double t = 0.0;
                for (int w = 0; w < kWarps; ++w) t += sRed[w][tid];
                sAcc[tid] = t;
            }
            __syncthreads();
        }
        stamp(4);
        if (a.iter_rec && it < a.iter_cap && bid == 0 && tid < 12 + kAlignTerms) {
            double *rec = a.iter_rec + (size_t)it * kIterRec;
            rec[tid] = tid < 12 ? sT[tid] : sAcc[tid - 12];
        }
        __syncthreads();
        // ------------------------------------------------------------ A8 solve / update / test
        if (tid == 0) {
            n_in = sAcc[28];
            cost_last = sAcc[27];
            int st_ = status, it_ = iters, cv_ = converged;
            sDone = solve_step_t<LM>(a, sAcc, sT, it, n, st_, it_, cv_, sLM);
            if (LM && !a.linearize_only && sLM[42] != 0.0) {  // stats of the kept linearisation
                n_in = sLM[12 + 28];
                cost_last = sLM[12 + 27];
            }
            status = st_;
            iters = it_;
            converged = cv_;
        }
        __syncthreads();
        stamp(5);
        if (sDone) break;
    }
    if (a.debug && has0) a.debug[i0] = make_int4(dbg_slow, dbg_reuse, dbg_graph, dbg_its);
    if (bid == 0 && tid == 0) {
        if (!a.linearize_only) {
            for (int k = 0; k < 12; ++k) a.d_T[k] = sT[k];
            a.d_T[12] = 0.0; a.d_T[13] = 0.0; a.d_T[14] = 0.0; a.d_T[15] = 1.0;
        }
        gsicp_align_stats st;
        st.fitness = n > 0 ? n_in / (double)n : 0.0;
        st.mean_cost = n_in > 0.0 ? cost_last / n_in : 0.0;
        st.n_inliers = (int32_t)n_in;
        st.iters = iters;
        st.converged = converged;
        st.status = status;
        *a.d_stats = st;
    }
}

template <bool LM>
__global__ void __launch_bounds__(kT, 1) k_align(AlignArgs a) {
    pdl_wait();  // (no early launch of dependents: they must not take SMs from this cooperative grid)
    align_body<LM>(a, blockIdx.x, gridDim.x);
}

// N2 frame batch: frame f = blockIdx.x / Gf runs on blocks [f Gf, (f+1) Gf) with its own
// workspace (partials, barrier, match cache), pose and stats; the target is shared.  The frames'
// arguments travel in the launch's parameter space (graph-capturable, no host->device copy).
constexpr int kMaxAlignBatch = 16;
struct AlignBatch {
    AlignArgs f[kMaxAlignBatch];
};

template <bool LM>
__global__ void __launch_bounds__(kT, 1) k_align_batch(const __grid_constant__ AlignBatch b, int Gf) {
    pdl_wait();
    const int f = blockIdx.x / Gf;
    align_body<LM>(b.f[f], blockIdx.x - f * Gf, Gf);
}

__global__ void k_align_init_batch(const __grid_constant__ AlignBatch b) {
    const AlignArgs &a = b.f[blockIdx.y];
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < a.cap) {
        a.corr_ws[i] = -1;
        a.reuse_ws[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (i == 0) *a.barrier = 0u;
}

// ---------------------------------------------------------------------------------------------
// Large clouds (cap above the co-resident grid's threads, e.g. a stride-1 TUM frame): the GN loop
// as ordinary kernels per iteration instead of one persistent cooperative kernel —
//   k_flat_corr : thread per point, the cheap certified paths of k_align (seeds, motion-bounded
//                 reuse, certified graph step, own-cell search), the rest to a global queue;
//   k_flat_hard : a warp per queued point, spread over the whole GPU (warp_nn and the
//                 second-neighbour bound of the reuse test);
//   k_flat_terms: thread per point, the Eq. 1 terms (binary64) and block partials; the last block
//                 to arrive reduces the partials in block order (deterministic) and runs the same
//                 solve step as k_align, then publishes the pose, the iteration and the stop flag.
// In a captured graph the three kernels are the body of a conditional WHILE node (k_flat_terms
// sets its condition); otherwise they are launched max_iters times and return at once after the
// stop.  k_align's persistent grid holds one point per thread for 1 block / SM (168 registers):
// a 205k-point frame then runs its hard queries as 12 warps per block in turn; here they spread
// over every warp slot of the GPU.
// Neighbourhood sets (the flat path's near-tie reuse): a point whose 1-NN stays
// ambiguous — a near-tie with its second neighbour, e.g. noisy depth 1-3 cm off a surface sampled
// at ~1.2 cm — fails both the motion-bounded reuse and the graph certificate every iteration.
// When the warp search solves such a point it also collects every target whose binary32 key from
// fl32(q) is <= rho^2 (rho as the second-neighbour bound's) and keeps the kSetCap nearest: every
// other target is then at least rho_cert from q (rho_cert = the (kSetCap+1)-th member's distance,
// or sqrt(rho^2 / (1 + 6u)) - E when all fit).  At a later query q' with |q' - q| <= delta the
// best member (binary64 keys, ties by index) is the exact 1-NN whenever its distance is below
// rho_cert - delta: one gather of <= kSetCap records per thread instead of a warp search.
constexpr int kSetCap = 16;

// the targets of the cells selected by `valid` with key32(fl32 q) <= B appended to the warp list
// (lane j holds the j-th; cnt may exceed 32: overflow)
__device__ __forceinline__ void warp_collect_cells(const AlignArgs &a, const CellIndex &idx, const QueryCell &qc,
                                                   bool valid, int dx, int dy, int dz, const Qry &q, float B, int lane,
                                                   int &cnt, int &mine) {
    const uint2 se = valid ? idx.one(qc.c[0] + dx, qc.c[1] + dy, qc.c[2] + dz) : make_uint2(0u, 0u);
    uint32_t incl = se.y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t ctot = __shfl_sync(0xffffffffu, incl, 31);
    for (uint32_t base = 0; base < ctot; base += 32) {
        const uint32_t item = base + lane;
        int l0 = 0, l1 = 31;
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            const int mid = (l0 + l1) >> 1;
            if (__shfl_sync(0xffffffffu, incl, mid) > item) l1 = mid; else l0 = mid + 1;
        }
        const uint32_t c_incl = __shfl_sync(0xffffffffu, incl, l0);
        const uint32_t c_start = __shfl_sync(0xffffffffu, se.x, l0);
        const uint32_t c_cnt = __shfl_sync(0xffffffffu, se.y, l0);
        int slot = -1;
        bool in = false;
        if (item < ctot) {
            slot = (int)(c_start + (item - (c_incl - c_cnt)));
            in = q.key32(__ldg(a.tpos + slot)) <= B;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        const int k = lane - cnt, nb = __popc(bal);
        const bool take = k >= 0 && k < nb;
        const int got = __shfl_sync(0xffffffffu, slot, take ? (int)__fns(bal, 0u, k + 1) : lane);
        if (take) mine = got;
        cnt += nb;
    }
}

// every target with key32(fl32 q) <= B (warp_nn's traversal with a fixed bound); stops early
// once more than 32 are found
__device__ void warp_range(const AlignArgs &a, const CellIndex &idx, const int *sb, const Qry &q, float B, int lane,
                           int &cnt, int &mine) {
    const QueryCell qc(q.x, q.y, q.z, a.h, a.inv_h);
    const int *blo = sb, *bhi = sb + 3;
    cnt = 0;
    mine = -1;
    auto in_box = [&](int dx, int dy, int dz) {
        const int x = qc.c[0] + dx, y = qc.c[1] + dy, z = qc.c[2] + dz;
        return x >= blo[0] && x <= bhi[0] && y >= blo[1] && y <= bhi[1] && z >= blo[2] && z <= bhi[2];
    };
    for (int m = 1; m <= kWarpShells; ++m) {
        const int sc = m == 1 ? 27 : shell_count(m);
        for (int t0 = 0; t0 < sc; t0 += 32) {
            const int t = t0 + lane;
            int dx = 0, dy = 0, dz = 0;
            bool valid = t < sc;
            if (valid) {
                if (m == 1) {
                    if (t > 0) shell_cell(1, t - 1, dx, dy, dz);
                } else {
                    shell_cell(m, t, dx, dy, dz);
                }
                valid = in_box(dx, dy, dz) && qc.gap2(dx, 0) + qc.gap2(dy, 1) + qc.gap2(dz, 2) <= B;
            }
            if (!__any_sync(0xffffffffu, valid)) continue;
            warp_collect_cells(a, idx, qc, valid, dx, dy, dz, q, B, lane, cnt, mine);
            if (cnt > 32) return;
        }
        if (B < qc.certified_key(m) || qc.covers(m, blo, bhi)) return;
    }
    int lo[3], hi[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) axis_range(qc, k, B, blo[k], bhi[k], lo[k], hi[k]);
    const int nx = max(hi[0] - lo[0] + 1, 0), ny = max(hi[1] - lo[1] + 1, 0), nz = max(hi[2] - lo[2] + 1, 0);
    const long long total = (long long)nx * ny * nz;
    for (long long t0 = 0; t0 < total; t0 += 32) {
        const long long t = t0 + lane;
        int dx = 0, dy = 0, dz = 0;
        bool valid = t < total;
        if (valid) {
            dx = lo[0] + (int)(t % nx);
            dy = lo[1] + (int)((t / nx) % ny);
            dz = lo[2] + (int)(t / ((long long)nx * ny));
            valid = max(abs(dx), max(abs(dy), abs(dz))) > kWarpShells &&
                    qc.gap2(dx, 0) + qc.gap2(dy, 1) + qc.gap2(dz, 2) <= B;
        }
        if (!__any_sync(0xffffffffu, valid)) continue;
        warp_collect_cells(a, idx, qc, valid, dx, dy, dz, q, B, lane, cnt, mine);
        if (cnt > 32) return;
    }
}

// After the warp search of point i (nn: its exact 1-NN at q): the second-neighbour bound d2 of
// the motion-bounded reuse and, when at most 32 targets lie within rho, the point's
// neighbourhood set (the kSetCap nearest of them).  Returns d2.
__device__ float warp_reuse_state(const AlignArgs &a, const CellIndex &idx, const int *sb, const Qry &q, const NN &nn,
                                  int i, int lane) {
    const bool in_r = nn.slot >= 0 && nn.bk < a.r2;
    const float base = in_r ? sqrtf(__double2float_ru(nn.bk)) : a.r;
    if (!(base < INFINITY)) return 0.f;
    const float rho = base * 1.25f + 0.25f * a.h;
    const float B = rho * rho;
    const float rc_all = fmaxf(__fsub_rd(__fsqrt_rd(__fmul_rd(B, 0.9999994f)), q.E()), 0.f);
    int cnt, mine;
    warp_range(a, idx, sb, q, B, lane, cnt, mine);
    if (cnt <= 32) {
        // binary64 keys of the members, a warp bitonic sort, the kSetCap nearest kept
        const double kk = lane < cnt ? q.key(__ldg(a.tpos + mine)) : INFINITY;
        double sk = kk;
        int ss = lane < cnt ? mine : -1;
#pragma unroll
        for (int kb = 2; kb <= 32; kb <<= 1) {
#pragma unroll
            for (int j = kb >> 1; j > 0; j >>= 1) {
                const double ok = shfl_f64(sk, lane ^ j);
                const int os = __shfl_xor_sync(0xffffffffu, ss, j);
                const bool low = ((lane & kb) == 0) == ((lane & j) == 0);  // this lane keeps the smaller
                if (low ? (ok < sk) : (ok > sk)) {
                    sk = ok;
                    ss = os;
                }
            }
        }
        float rc = rc_all;
        const double k17 = shfl_f64(sk, kSetCap);  // the (kSetCap+1)-th nearest
        if (cnt > kSetCap) rc = fminf(rc, sqrtf(__double2float_rd(k17)));
        rc *= (1.f - kReuseMargin);
        if (lane < kSetCap) a.rset[(size_t)i * kSetCap + lane] = lane < cnt ? ss : -1;
        if (lane == 0) a.rset_hdr[i] = make_float4(q.x, q.y, q.z, rc);
        // the second neighbour: the nearest member other than the 1-NN
        double k2 = lane < cnt && mine != nn.slot ? kk : INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) k2 = fmin(k2, shfl_f64(k2, lane ^ o));
        const float d2s = k2 < INFINITY ? sqrtf(__double2float_rd(k2)) : INFINITY;
        return fminf(fminf(d2s, rho), rc_all) * (1.f - kReuseMargin);
    }
    if (lane == 0) a.rset_hdr[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    NN n2;
    warp_nn(a, idx, sb, q, n2, lane, B, nn.slot);
    return fminf(n2.slot >= 0 ? sqrtf(__double2float_rd(n2.bk)) : INFINITY, rho) * (1.f - kReuseMargin);
}

// The neighbourhood-set test of point i at its new query q: true if the set proves the exact
// 1-NN (nn = it, or the point stays gated); false if there is no set or the query moved too far.
__device__ __forceinline__ bool set_nn(const AlignArgs &a, const Qry &q, int i, NN &nn) {
    const float4 h = __ldcg(a.rset_hdr + i);  // (written during this loop: no read-only path)
    if (!(h.w > 0.f)) return false;
    const float ex = q.x - h.x, ey = q.y - h.y, ez = q.z - h.z;
    const float delta = sqrtf(ex * ex + ey * ey + ez * ez) * (1.f + kReuseMargin) + 2.f * q.E();
    const float L = h.w - delta;
    if (!(L > 0.f)) return false;
    const int4 *ls = reinterpret_cast<const int4 *>(a.rset + (size_t)i * kSetCap);
    int sl[kSetCap];
#pragma unroll
    for (int v = 0; v < kSetCap / 4; ++v) {
        const int4 w = __ldcg(ls + v);
        sl[4 * v] = w.x; sl[4 * v + 1] = w.y; sl[4 * v + 2] = w.z; sl[4 * v + 3] = w.w;
    }
    NN ns;
    float k32[kSetCap];
    {
        float4 p[kSetCap];
#pragma unroll
        for (int u = 0; u < kSetCap; ++u) p[u] = sl[u] >= 0 ? __ldg(a.tpos + sl[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < kSetCap; ++u) k32[u] = sl[u] >= 0 ? q.key32(p[u]) : INFINITY;
    }
    float m32 = INFINITY;
#pragma unroll
    for (int u = 0; u < kSetCap; ++u) m32 = fminf(m32, k32[u]);
    if (m32 < INFINITY) {
        // binary64 keys of the members that can beat or tie the best binary32 one
        const float s0 = __fmul_ru(__fadd_ru(__fsqrt_ru(m32), 2.f * q.E()), 1.000004f);
        const float scr = __fmul_ru(s0, s0);
#pragma unroll
        for (int u = 0; u < kSetCap; ++u) {
            if (k32[u] <= scr) {
                const float4 rec = __ldg(a.tpos + sl[u]);
                ns.offer(q.key(rec), (uint32_t)__float_as_int(rec.w), sl[u], rec);
            }
        }
    }
    const float d1 = ns.slot >= 0 ? fminf(sqrtf(__double2float_ru(ns.bk)), a.r) : a.r;
    if (!(L * (1.f - kReuseMargin) > d1 * (1.f + kReuseMargin))) return false;
    nn = ns;
    return true;
}

struct FlatState {
    int it, stop, status, iters, converged;
    unsigned int active;  // (frame 0 of a batch: the frames still iterating)
    unsigned int qn, arrive;
    double n_in, cost;
    double T[12];
    double lm[kLmState];
};
#ifndef GSICP_FLAT_D2_FROM_ITER
#define GSICP_FLAT_D2_FROM_ITER 2
#endif
constexpr int kFlatD2FromIter = GSICP_FLAT_D2_FROM_ITER;
  // reuse bound + neighbourhood set from this iteration
#ifndef GSICP_FLAT_BATCH
#define GSICP_FLAT_BATCH 6  // frame batches of at least this many frames through the flat loop
#endif                      // (measured: B = 4 7% slower, B = 8 10% and B = 16 32% faster than k_align_batch)
#ifndef GSICP_FLAT_DIV
#define GSICP_FLAT_DIV 1  // clouds above (co-resident threads) / this take the flat path
#endif
constexpr int kFlatT = 256;
constexpr int kFlatHardT = 128;
constexpr int kFlatTermsPerSm = 2;  // k_flat_terms blocks per SM (partials reduced by the last one)

// The flat kernels' parameter: NB frames (blockIdx.y = frame), each with its own arguments,
// workspace and loop state; `active` counts the frames still iterating (the WHILE condition
// drops when it reaches 0).  NB = 1: a single large cloud; kMaxAlignBatch: a frame batch (N2).
template <int NB>
struct FlatBatch {
    AlignArgs f[NB];
    FlatState *fs[NB];
    unsigned int *active;
};

template <int NB>
__global__ void k_flat_init(const __grid_constant__ FlatBatch<NB> fb) {
    const AlignArgs &a = fb.f[blockIdx.y];
    FlatState *fs = fb.fs[blockIdx.y];
    pdl_wait();
    pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (blockIdx.y == 0 && i == 0) *fb.active = gridDim.y;
    if (i < a.cap) {
        a.corr_ws[i] = -1;
        a.reuse_ws[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        a.rset_hdr[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (i == 0) {
        fs->it = 0;
        fs->stop = 0;
        fs->status = GSICP_WARN_MAX_ITERS;
        fs->iters = 0;
        fs->converged = 0;
        fs->qn = 0u;
        fs->arrive = 0u;
        fs->n_in = 0.0;
        fs->cost = 0.0;
        for (int k = 0; k < 12; ++k) fs->T[k] = a.d_T[k];
        fs->lm[42] = 0.0;
    }
}

template <int NB>
__global__ void __launch_bounds__(kFlatT) k_flat_corr(const __grid_constant__ FlatBatch<NB> fb) {
    const AlignArgs &a = fb.f[blockIdx.y];
    FlatState *fs = fb.fs[blockIdx.y];
    __shared__ double sT[12];
    __shared__ int sBox[6];
    __shared__ CellIndex sIdx;
    __shared__ int sIt, sStop, sSeeded;
    pdl_wait();
    pdl_launch_dependents();
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        sStop = fs->stop;
        sIt = fs->it;
        load_cell_index(a, sIdx, sBox);
        // seeds only at the pose they were computed at (iteration 0, the caller's pose)
        bool ok = a.seed_ticket > 0.0 && a.seed_hdr[12] == a.seed_ticket;
        for (int k = 0; k < 12; ++k) ok = ok && __double_as_longlong(a.seed_hdr[k]) == __double_as_longlong(a.d_T[k]);
        sSeeded = ok;
    }
    if (tid < 12) sT[tid] = fs->T[tid];
    __syncthreads();
    if (sStop) return;
    const int it = sIt, n = *a.d_n;
    for (int i0 = blockIdx.x * kFlatT; i0 < n; i0 += gridDim.x * kFlatT) {  // (warp-uniform trip count)
        const int i = i0 + tid;
        bool queued = false;
        int qslot = -1;
        if (i < n) {
            const float4 x = __ldg(a.spos + i);
            double q0, q1, q2;
            k3(sT, x.x, x.y, x.z, q0, q1, q2);
            const Qry q(q0, q1, q2);
            const QueryCell qc(q.x, q.y, q.z, a.h, a.inv_h);
            NN nn;
            const bool seeded = it == 0 && sSeeded;
            int slot = seeded ? a.seed_slot[i] : a.corr_ws[i];
            if (slot <= -2) slot = -2 - slot;
            if (slot >= 0) {
                const float4 rec = __ldg(a.tpos + slot);
                nn.set(q.key(rec), slot, rec);
            }
            bool exact = seeded;
            const float4 ru = seeded ? make_float4(0.f, 0.f, 0.f, 0.f) : a.reuse_ws[i];
            float d2lb = ru.w;
            if (!exact && d2lb > 0.f) {  // the motion-bounded reuse (k_align)
                const float ex = q.x - ru.x, ey = q.y - ru.y, ez = q.z - ru.z;
                const float delta = sqrtf(ex * ex + ey * ey + ez * ez) * (1.f + kReuseMargin) + 2.f * q.E();
                const float d1 = nn.slot >= 0 ? fminf(sqrtf(__double2float_ru(nn.bk)), a.r) : a.r;
                if ((d2lb - delta) * (1.f - kReuseMargin) > d1 * (1.f + kReuseMargin)) {
                    exact = true;
                    d2lb -= delta;
                }
            }
            const bool by_reuse = exact && !seeded;
            if (!exact) d2lb = 0.f;
            bool by_set = false;
            if (!exact && !seeded) by_set = exact = set_nn(a, q, i, nn);  // near-tie points: the neighbourhood set
            const uint2 own = exact ? make_uint2(0u, 0u) : sIdx.one(qc.c[0], qc.c[1], qc.c[2]);
            uint2 own_left = own;
            if (!exact && a.nbr && (nn.slot < 0 || nn.bk > 0.25 * (double)a.h * (double)a.h)) {
                scan_target_cell(a, own, q, nn);  // a far or absent warm start: from the own cell
                own_left = make_uint2(0u, 0u);
            }
            const bool pre = exact;
            if (!exact && nn.slot >= 0 && a.nbr) exact = graph_nn(a, q, nn, d2lb);
            const bool by_graph = exact && !pre;
            if (!exact && !a.nbr) exact = nn_search(a, sIdx, sBox, qc, own_left, q, nn, true);
            if (a.debug && it < 32) {  // diagnostic: per point bitmasks over iterations (queued, reuse, set, graph)
                int4 d = it == 0 ? make_int4(0, 0, 0, 0) : a.debug[i];
                const int bit = 1 << it;
                d.x |= exact ? 0 : bit;
                d.y |= by_reuse ? bit : 0;
                d.z |= by_set ? bit : 0;
                d.w |= by_graph ? bit : 0;
                a.debug[i] = d;
            }
            if (exact) {
                a.corr_ws[i] = (nn.slot >= 0 && nn.bk < a.r2) ? nn.slot : -2 - nn.slot;
                a.reuse_ws[i] = make_float4(q.x, q.y, q.z, seeded ? 0.f : d2lb);
            } else {
                queued = true;
                qslot = nn.slot;
            }
        }
        // the rest to the global queue (one atomic per warp); the warm start travels along
        const unsigned qb = __ballot_sync(0xffffffffu, queued);
        unsigned int base = 0u;
        if (lane == 0 && qb) base = atomicAdd(&fs->qn, (unsigned)__popc(qb));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (queued) a.flat_queue[base + __popc(qb & ((1u << lane) - 1u))] = make_int2(i, qslot);
    }
}

template <int NB>
__global__ void __launch_bounds__(kFlatHardT) k_flat_hard(const __grid_constant__ FlatBatch<NB> fb) {
    const AlignArgs &a = fb.f[blockIdx.y];
    FlatState *fs = fb.fs[blockIdx.y];
    __shared__ double sT[12];
    __shared__ int sBox[6];
    __shared__ CellIndex sIdx;
    __shared__ int sIt, sStop;
    pdl_wait();
    pdl_launch_dependents();
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        sStop = fs->stop;
        sIt = fs->it;
        load_cell_index(a, sIdx, sBox);
    }
    if (tid < 12) sT[tid] = fs->T[tid];
    __syncthreads();
    if (sStop) return;
    const int it = sIt;
    const int qn = (int)fs->qn;
    const int warps = gridDim.x * (kFlatHardT / 32);
    for (int k = blockIdx.x * (kFlatHardT / 32) + (tid >> 5); k < qn; k += warps) {
        const int2 qe = a.flat_queue[k];
        const int i = qe.x, sl = qe.y;
        const float4 x = __ldg(a.spos + i);
        double q0, q1, q2;
        k3(sT, x.x, x.y, x.z, q0, q1, q2);
        const Qry q(q0, q1, q2);
        NN nn;
        if (sl >= 0) {
            const float4 rec = __ldg(a.tpos + sl);
            nn.set(q.key(rec), sl, rec);
        }
        warp_nn(a, sIdx, sBox, q, nn, lane);
        // the second-neighbour bound and the neighbourhood set for the next iterations
        const bool in_r = nn.slot >= 0 && nn.bk < a.r2;
        const float d2 = it >= kFlatD2FromIter ? warp_reuse_state(a, sIdx, sBox, q, nn, i, lane) : 0.f;
        if (lane == 0) {
            a.corr_ws[i] = in_r ? nn.slot : -2 - nn.slot;
            a.reuse_ws[i] = make_float4(q.x, q.y, q.z, d2);
        }
    }
}

template <bool LM, int NB>
__global__ void __launch_bounds__(kFlatT) k_flat_terms(const __grid_constant__ FlatBatch<NB> fb,
                                                      cudaGraphConditionalHandle cond, int use_cond) {
    const AlignArgs &a = fb.f[blockIdx.y];
    FlatState *fs = fb.fs[blockIdx.y];
    constexpr int kW = kFlatT / 32;
    __shared__ double sT[12];
    __shared__ double sRed[kW][kPad];
    __shared__ double sAcc[kPad];
    __shared__ int sIt, sStop, sLast;
    pdl_wait();
    pdl_launch_dependents();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        sStop = fs->stop;
        sIt = fs->it;
    }
    if (tid < 12) sT[tid] = fs->T[tid];
    __syncthreads();
    if (sStop) return;
    const int it = sIt, n = *a.d_n;
    double acc[kAlignTerms];
#pragma unroll
    for (int k = 0; k < kAlignTerms; ++k) acc[k] = 0.0;
    for (int i = blockIdx.x * kFlatT + tid; i < n; i += gridDim.x * kFlatT) {
        const int slot = a.corr_ws[i];
        int32_t corr_val = -1;
        if (slot >= 0) {
            const float4 x = __ldg(a.spos + i);
            double q0, q1, q2;
            k3(sT, x.x, x.y, x.z, q0, q1, q2);
            const float4 m = __ldg(a.tpos + slot);
            if (pair_terms(sT, q0, q1, q2, __ldg(a.scov_a + i), __ldg(a.scov_b + i), m, __ldg(a.tcov_a + slot),
                           __ldg(a.tcov_b + slot), acc))
                corr_val = __float_as_int(m.w);
        }
        if (a.corr_out) a.corr_out[i] = corr_val;
        if (a.iter_corr && it < a.iter_cap) a.iter_corr[(size_t)it * a.cap + i] = corr_val;
    }
#pragma unroll
    for (int k = 0; k < kAlignTerms; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < kAlignTerms; ++k) sRed[warp][k] = acc[k];
    }
    __syncthreads();
    if (tid < kAlignTerms) {
        double t = 0.0;
        for (int w = 0; w < kW; ++w) t += sRed[w][tid];
        a.partials[(size_t)blockIdx.x * kPad + tid] = t;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) sLast = atomicAdd(&fs->arrive, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!sLast) return;
    __threadfence();
    // the last block: every partial in block order (8 chunks per term, then the chunks in order)
    {
        constexpr int kChunks = kFlatT / 32;
        const int term = tid & 31, chunk = tid >> 5;
        const int G = gridDim.x, per = (G + kChunks - 1) / kChunks;
        double sum = 0.0;
        if (term < kAlignTerms) {
            const int b0 = chunk * per, b1 = min(G, b0 + per);
            int b = b0;
            for (; b + 4 <= b1; b += 4) {
                const double v0 = __ldcg(a.partials + (size_t)b * kPad + term);
                const double v1 = __ldcg(a.partials + (size_t)(b + 1) * kPad + term);
                const double v2 = __ldcg(a.partials + (size_t)(b + 2) * kPad + term);
                const double v3 = __ldcg(a.partials + (size_t)(b + 3) * kPad + term);
                sum += v0;
                sum += v1;
                sum += v2;
                sum += v3;
            }
            for (; b < b1; ++b) sum += __ldcg(a.partials + (size_t)b * kPad + term);
        }
        sRed[chunk][term] = sum;
        __syncthreads();
        if (tid < kAlignTerms) {
            double t = 0.0;
            for (int c = 0; c < kChunks; ++c) t += sRed[c][tid];
            sAcc[tid] = t;
        }
        __syncthreads();
    }
    if (a.iter_rec && it < a.iter_cap && tid < 12 + kAlignTerms) {
        double *rec = a.iter_rec + (size_t)it * kIterRec;
        rec[tid] = tid < 12 ? sT[tid] : sAcc[tid - 12];
    }
    if (tid == 0) {
        double n_in = sAcc[28], cost = sAcc[27];
        int st = fs->status, its = fs->iters, cv = fs->converged;
        int done;
        if (a.linearize_only) {
            int t = 0;
            for (int r = 0; r < 6; ++r)
                for (int c = r; c < 6; ++c) a.d_lin[6 * r + c] = a.d_lin[6 * c + r] = sAcc[t++];
            for (int k = 0; k < 6; ++k) a.d_lin[36 + k] = sAcc[21 + k];
            a.d_lin[42] = sAcc[27];
            a.d_lin[43] = sAcc[28];
            st = GSICP_OK;
            done = 1;
        } else {
            done = solve_step_t<LM>(a, sAcc, sT, it, n, st, its, cv, fs->lm);
            if (LM && fs->lm[42] != 0.0) {  // stats of the kept linearisation
                n_in = fs->lm[12 + 28];
                cost = fs->lm[12 + 27];
            }
        }
        fs->status = st;
        fs->iters = its;
        fs->converged = cv;
        fs->n_in = n_in;
        fs->cost = cost;
        for (int k = 0; k < 12; ++k) fs->T[k] = sT[k];
        fs->it = it + 1;
        fs->qn = 0u;
        fs->arrive = 0u;
        if (done) {
            fs->stop = 1;
            if (!a.linearize_only) {
                for (int k = 0; k < 12; ++k) a.d_T[k] = sT[k];
                a.d_T[12] = 0.0; a.d_T[13] = 0.0; a.d_T[14] = 0.0; a.d_T[15] = 1.0;
            }
            gsicp_align_stats sts;
            sts.fitness = n > 0 ? n_in / (double)n : 0.0;
            sts.mean_cost = n_in > 0.0 ? cost / n_in : 0.0;
            sts.n_inliers = (int32_t)n_in;
            sts.iters = its;
            sts.converged = cv;
            sts.status = st;
            *a.d_stats = sts;
            // the last frame to finish ends the loop
            const unsigned int left = atomicSub(fb.active, 1u) - 1u;
            if (use_cond && left == 0u) cudaGraphSetConditional(cond, 0u);
        }
    }
}

// Co-resident grid for the cooperative launch (0 if the kernel cannot be resident at all).
constexpr int kMaxAlignGrid = 2048;  // partial records reserved in the workspace (>= SMs x blocks/SM)

// blocks per SM of the GN kernels (the smaller residency of the GN and LM variants), per device
template <class F1, class F2>
static int coresident_per_sm(F1 k_gn, F2 k_lm) {
    int v = 0, v1 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_gn, kT, 0) != cudaSuccess) v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v1, k_lm, kT, 0) != cudaSuccess) v1 = 0;
    return v < v1 ? v : v1;
}

int align_grid_blocks(int cap, int *per_sm_out) {
    static PerDevice<int> cache;
    const int per_sm = cache.get([](int) { return coresident_per_sm(k_align<false>, k_align<true>); });
    *per_sm_out = per_sm;
    (void)cap;
    const int g = per_sm * num_sms();  // the full co-resident grid; k_align splits the points over it
    return g < kMaxAlignGrid ? g : kMaxAlignGrid;
}

}  // namespace

struct AlignWs {
    double *d_T;
    gsicp_align_stats *d_stats;
    double *d_lin;
    unsigned int *barrier;
    double *partials;
    int32_t *corr_ws;
    float4 *reuse_ws;
    int32_t *seed_slot;
    double *seed_hdr;
    int32_t *seed_queue;
    int32_t *seed_qn;
    FlatState *flat;
    int2 *flat_queue;
    int32_t *rset;
    float4 *rset_hdr;
};

static AlignWs align_carve(Carver &c, int cap) {
    AlignWs w;
    w.d_T = c.take<double>(16);
    w.d_stats = c.take<gsicp_align_stats>(1);
    w.d_lin = c.take<double>(48);
    w.barrier = c.take<unsigned int>(4);
    (void)cap;
    w.partials = c.take<double>((size_t)2 * kMaxAlignGrid * kPad);  // the grid is the co-resident one
    w.corr_ws = c.take<int32_t>(cap);
    w.reuse_ws = c.take<float4>(cap);
    w.seed_slot = c.take<int32_t>(cap);
    w.seed_hdr = c.take<double>(16);
    w.seed_queue = c.take<int32_t>(cap);
    w.seed_qn = c.take<int32_t>(4);
    w.flat = c.take<FlatState>(1);
    w.flat_queue = c.take<int2>(cap);
    w.rset = c.take<int32_t>((size_t)cap * kSetCap);
    w.rset_hdr = c.take<float4>(cap);
    return w;
}
static AlignWs align_carve(void *base, int cap) {
    Carver c(base);
    return align_carve(c, cap);
}

size_t align_ws_bytes(int cap) {
    Carver c(nullptr);
    align_carve(c, cap);
    return c.bytes();
}

double *align_ws_T(void *ws) { return align_carve(ws, 0).d_T; }
gsicp_align_stats *align_ws_stats(void *ws) { return align_carve(ws, 0).d_stats; }
double *align_ws_lin(void *ws) { return align_carve(ws, 0).d_lin; }

// d_T_inout: device pose (may equal the workspace pose); d_stats: device stats destination.
static AlignArgs make_args(const gsicp_cloud &src, const gsicp_target &tgt, double *d_T_inout,
                           const gsicp_align_params &p, gsicp_align_stats *d_stats, int32_t *corr_out,
                           int linearize_only, float r_lin, const AlignWs &w) {
    AlignArgs a;
    a.spos = reinterpret_cast<const float4 *>(src.pos);
    a.scov_a = reinterpret_cast<const float4 *>(src.cov_a);
    a.scov_b = reinterpret_cast<const float4 *>(src.cov_b);
    a.d_n = src.d_n;
    a.cap = src.cap;
    a.table = static_cast<const CellEntry *>(tgt.table);
    a.mask = tgt.table_mask;
    a.h = tgt.cell;
    a.inv_h = 1.0f / tgt.cell;
    a.tpos = reinterpret_cast<const float4 *>(tgt.pos);
    a.tcov_a = reinterpret_cast<const float4 *>(tgt.cov_a);
    a.tcov_b = reinterpret_cast<const float4 *>(tgt.cov_b);
    a.tbbox = tgt.bbox;
    a.dense = static_cast<const uint2 *>(tgt.dense);
    a.dense_hdr = tgt.dense_hdr;
    a.nbr = tgt.nbr;
    a.nbr_key = tgt.nbr_key;
    a.max_iters = p.max_iters;
    a.r = linearize_only ? r_lin : p.max_corr_dist;
    a.r2 = (double)a.r * (double)a.r;
    a.r2f = (float)a.r2;
    if ((double)a.r2f < a.r2) a.r2f = nextafterf(a.r2f, INFINITY);
    a.eps_rot = p.eps_rot;
    a.eps_trans = p.eps_trans;
    a.min_pairs = p.min_pairs;
    a.solver = p.solver;
    a.lm_lambda0 = p.lm_lambda0;
    a.linearize_only = linearize_only;
    a.d_T = d_T_inout;
    a.d_stats = d_stats;
    a.d_lin = w.d_lin;
    a.partials = w.partials;
    a.barrier = w.barrier;
    a.corr_ws = w.corr_ws;
    a.reuse_ws = w.reuse_ws;
    a.corr_out = corr_out;
    a.timeline = g_align_timeline;
    a.timeline_cap = g_align_timeline_cap;
    a.debug = reinterpret_cast<int4 *>(g_align_debug);
    a.seed_slot = w.seed_slot;
    a.seed_hdr = w.seed_hdr;
    a.seed_ticket = 0.0;
    a.seed_queue = w.seed_queue;
    a.seed_qn = w.seed_qn;
    a.flat_queue = w.flat_queue;
    a.rset = w.rset;
    a.rset_hdr = w.rset_hdr;
    a.iter_rec = g_align_iter_rec;
    a.iter_corr = g_align_iter_corr;
    a.iter_cap = g_align_iter_rec ? g_align_iter_cap : 0;
    return a;
}

// Seeds are single-use and bound to the workspace and the host thread: gsicp_align_seed records a
// ticket here, the next align / linearize launch on the same workspace expects it (and clears it),
// so stale seeds (another cloud, pose or workspace) are never used.
// One entry per workspace with pending seeds (a frame batch seeds several workspaces).
struct SeedTicket {
    void *ws = nullptr;
    const void *src = nullptr, *tgt = nullptr;
    double ticket = 0.0;
};
constexpr int kSeedTickets = 32;
thread_local SeedTicket g_seed[kSeedTickets];
thread_local double g_seed_counter = 0.0;

static void seed_record(void *ws, const void *src, const void *tgt, double ticket) {
    int slot = -1;
    for (int k = 0; k < kSeedTickets && slot < 0; ++k)
        if (g_seed[k].ws == ws) slot = k;
    for (int k = 0; k < kSeedTickets && slot < 0; ++k)
        if (g_seed[k].ws == nullptr) slot = k;
    if (slot < 0) {  // table full: evict the oldest ticket (its seeds are then simply not used)
        slot = 0;
        for (int k = 1; k < kSeedTickets; ++k)
            if (g_seed[k].ticket < g_seed[slot].ticket) slot = k;
    }
    g_seed[slot] = SeedTicket{ws, src, tgt, ticket};
}

// the ticket the next launch on `ws` expects (0: none), consumed
static double seed_take(void *ws, const void *src, const void *tgt) {
    for (int k = 0; k < kSeedTickets; ++k)
        if (g_seed[k].ws == ws) {
            const double t = (g_seed[k].src == src && g_seed[k].tgt == tgt) ? g_seed[k].ticket : 0.0;
            g_seed[k] = SeedTicket{};
            return t;
        }
    return 0.0;
}

cudaError_t align_seed_launch(const gsicp_cloud &src, const gsicp_target &tgt, const double *d_T,
                              const gsicp_align_params &p, void *ws, cudaStream_t s) {
    AlignWs w = align_carve(ws, src.cap);
    AlignArgs a = make_args(src, tgt, const_cast<double *>(d_T), p, nullptr, nullptr, 0, 0.f, w);
    g_seed_counter += 1.0;
    a.seed_ticket = g_seed_counter;
    seed_record(ws, src.pos, tgt.pos, a.seed_ticket);
    cudaError_t e = cudaMemsetAsync(w.seed_qn, 0, sizeof(int32_t), s);
    if (e != cudaSuccess) {
        set_error("align_seed memset: %s", cudaGetErrorString(e));
        return e;
    }
    ktimer_mark(KT_SEED, false, s);
    launch_low(k_align_seed, dim3(blocks_for(src.cap > 0 ? src.cap : 1, kSeedT)), dim3(kSeedT), 0, s, a);
    GSICP_LAUNCH_CHECK("k_align_seed");
    constexpr int kSeedHardPerSm = 8;  // resident blocks per SM of the hard pass (measured best, round 1)
    launch_low(k_align_seed_hard, dim3(num_sms() * kSeedHardPerSm), dim3(kSeedHardT), 0, s, a);
    GSICP_LAUNCH_CHECK("k_align_seed_hard");
    ktimer_mark(KT_SEED, true, s);
    note_launch(2);
    return cudaSuccess;
}

// stream used to capture the flat loop's WHILE body (per host thread)
static cudaStream_t flat_body_stream() {
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

template <int NB>
static cudaError_t flat_iteration(const FlatBatch<NB> &fb, int B, int cap_max, bool lm, cudaGraphConditionalHandle h,
                                  int use_cond, cudaStream_t s) {
    const unsigned sm = (unsigned)num_sms();
    const unsigned g1 = std::max(1u, std::min<unsigned>(blocks_for(cap_max > 0 ? cap_max : 1, kFlatT), sm * 16 / B));
    launch_pdl(k_flat_corr<NB>, dim3(g1, B), dim3(kFlatT), 0, s, fb);
    GSICP_LAUNCH_CHECK("k_flat_corr");
    launch_pdl(k_flat_hard<NB>, dim3(std::max(8u, sm * 8 / B), B), dim3(kFlatHardT), 0, s, fb);
    GSICP_LAUNCH_CHECK("k_flat_hard");
    const dim3 g3(std::max(8u, sm * kFlatTermsPerSm / B), B);
    if (lm)
        launch_pdl(k_flat_terms<true, NB>, g3, dim3(kFlatT), 0, s, fb, h, use_cond);
    else
        launch_pdl(k_flat_terms<false, NB>, g3, dim3(kFlatT), 0, s, fb, h, use_cond);
    GSICP_LAUNCH_CHECK("k_flat_terms");
    return cudaSuccess;
}

// The flat GN loop of B frames: init, then the three kernels per iteration — the body of a
// conditional WHILE node inside a stream capture, else max_iters launches (idle after the stop).
template <int NB>
static cudaError_t align_flat_run(const FlatBatch<NB> &fb, int B, int cap_max, int max_iters, bool lm, cudaStream_t s) {
    ktimer_mark(KT_ALIGN, false, s);
    launch_pdl(k_flat_init<NB>, dim3(blocks_for(cap_max > 0 ? cap_max : 1, 256), B), dim3(256), 0, s, fb);
    GSICP_LAUNCH_CHECK("k_flat_init");
    cudaError_t e = cudaSuccess;
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cst);
    if (cst == cudaStreamCaptureStatusActive) {
        cudaGraph_t graph = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t nd = 0;
        unsigned long long cid = 0;
        if ((e = cudaStreamGetCaptureInfo(s, &cst, &cid, &graph, &deps, &nd)) != cudaSuccess) return e;
        cudaGraphConditionalHandle h;
        if ((e = cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault)) != cudaSuccess) return e;
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        if ((e = cudaGraphAddNode(&cnode, graph, deps, nd, &cp)) != cudaSuccess) return e;
        cudaStream_t bs = flat_body_stream();
        if (!bs) return cudaErrorInvalidResourceHandle;
        if ((e = cudaStreamBeginCaptureToGraph(bs, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                               cudaStreamCaptureModeRelaxed)) != cudaSuccess)
            return e;
        const bool was = pdl_suspended();
        pdl_suspended() = true;  // no programmatic edges inside the conditional body
        const cudaError_t eb = flat_iteration(fb, B, cap_max, lm, h, 1, bs);
        pdl_suspended() = was;
        cudaGraph_t body_out = nullptr;
        e = cudaStreamEndCapture(bs, &body_out);
        if (eb != cudaSuccess) return eb;
        if (e != cudaSuccess) return e;
        if ((e = cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies)) != cudaSuccess)
            return e;
    } else {
        for (int k = 0; k < std::max(1, max_iters) && e == cudaSuccess; ++k)
            e = flat_iteration(fb, B, cap_max, lm, cudaGraphConditionalHandle{}, 0, s);
        if (e != cudaSuccess) return e;
    }
    ktimer_mark(KT_ALIGN, true, s);
    note_launch(4);
    return cudaSuccess;
}

static cudaError_t align_flat_launch(const AlignArgs &a, const AlignWs &w, int cap, bool lm, cudaStream_t s) {
    FlatBatch<1> fb;
    fb.f[0] = a;
    fb.fs[0] = w.flat;
    fb.active = &w.flat->active;
    return align_flat_run(fb, 1, cap, a.linearize_only ? 1 : a.max_iters, lm, s);
}

cudaError_t align_launch(const gsicp_cloud &src, const gsicp_target &tgt, double *d_T_inout,
                         const gsicp_align_params &p, gsicp_align_stats *d_stats, int32_t *corr_out,
                         int linearize_only, float r_lin, void *ws, cudaStream_t s) {
    AlignWs w = align_carve(ws, src.cap);
    AlignArgs a = make_args(src, tgt, d_T_inout, p, d_stats, corr_out, linearize_only, r_lin, w);
    a.seed_ticket = seed_take(ws, src.pos, tgt.pos);
    int per_sm = 0;
    const int G = align_grid_blocks(src.cap, &per_sm);
    if (G >= 1 && src.cap > G * kT / GSICP_FLAT_DIV) return align_flat_launch(a, w, src.cap, p.solver == 1, s);
    launch_pdl(k_align_init, dim3(blocks_for(src.cap > 0 ? src.cap : 1, 256)), dim3(256), 0, s, w.corr_ws, w.reuse_ws, src.cap,
               w.barrier);
    GSICP_LAUNCH_CHECK("k_align_init");
    if (G < 1) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k_align<false>);
        set_error("k_align cannot be co-resident: occupancy %d blocks/SM (regs %d, local %zu B, max threads %d)",
                  per_sm, fa.numRegs, fa.localSizeBytes, fa.maxThreadsPerBlock);
        return cudaErrorCooperativeLaunchTooLarge;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributePriority;
    at[1].val.priority = launch_priority(true);
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(kT);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    ktimer_mark(KT_ALIGN, false, s);
    cudaError_t e = p.solver == 1 ? cudaLaunchKernelEx(&cfg, k_align<true>, a) : cudaLaunchKernelEx(&cfg, k_align<false>, a);
    ktimer_mark(KT_ALIGN, true, s);
    if (e != cudaSuccess) {
        set_error("k_align launch: %s", cudaGetErrorString(e));
        return e;
    }
    note_launch(2);
    return cudaSuccess;
}

int align_batch_max() { return kMaxAlignBatch; }

// N2: B frames against one target in one cooperative launch (G / B co-resident blocks per frame).
cudaError_t align_batch_launch(const gsicp_cloud *srcs, int B, const gsicp_target &tgt, double *d_T,
                               const gsicp_align_params &p, gsicp_align_stats *d_stats, int32_t *const *corr_out,
                               void *const *ws, cudaStream_t s) {
    static thread_local AlignBatch hb;  // host staging of the launch parameter (copied at launch)
    int cap_max = 1;
    for (int f = 0; f < B; ++f) {
        AlignWs w = align_carve(ws[f], srcs[f].cap);
        hb.f[f] = make_args(srcs[f], tgt, d_T + 16 * (size_t)f, p, d_stats + f, corr_out ? corr_out[f] : nullptr, 0,
                            0.f, w);
        hb.f[f].timeline = nullptr;  // the diagnostics describe single-frame launches
        hb.f[f].timeline_cap = 0;
        hb.f[f].debug = nullptr;
        if (f > 0) {  // the per-iteration record hook follows frame 0 of a batch
            hb.f[f].iter_rec = nullptr;
            hb.f[f].iter_corr = nullptr;
            hb.f[f].iter_cap = 0;
        }
        hb.f[f].seed_ticket = seed_take(ws[f], srcs[f].pos, tgt.pos);
        if (srcs[f].cap > cap_max) cap_max = srcs[f].cap;
    }
    if (B >= GSICP_FLAT_BATCH) {  // the flat loop over the B frames (blockIdx.y = frame)
        static thread_local FlatBatch<kMaxAlignBatch> fb;
        for (int f = 0; f < B; ++f) {
            fb.f[f] = hb.f[f];
            fb.fs[f] = align_carve(ws[f], srcs[f].cap).flat;
        }
        fb.active = &fb.fs[0]->active;
        return align_flat_run(fb, B, cap_max, p.max_iters, p.solver == 1, s);
    }
    launch_pdl(k_align_init_batch, dim3(blocks_for(cap_max, 256), B), dim3(256), 0, s, hb);
    GSICP_LAUNCH_CHECK("k_align_init_batch");
    static PerDevice<int> cache;
    const int per_sm = cache.get([](int) { return coresident_per_sm(k_align_batch<false>, k_align_batch<true>); });
    int G = per_sm * num_sms();
    if (G > kMaxAlignGrid) G = kMaxAlignGrid;
    const int Gf = G / B;
    if (Gf < 1) {
        set_error("k_align_batch: %d frames do not fit the co-resident grid (%d blocks)", B, G);
        return cudaErrorCooperativeLaunchTooLarge;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributePriority;
    at[1].val.priority = launch_priority(true);
    cfg.gridDim = dim3(Gf * B);
    cfg.blockDim = dim3(kT);
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    ktimer_mark(KT_ALIGN, false, s);
    cudaError_t e = p.solver == 1 ? cudaLaunchKernelEx(&cfg, k_align_batch<true>, hb, Gf)
                                  : cudaLaunchKernelEx(&cfg, k_align_batch<false>, hb, Gf);
    ktimer_mark(KT_ALIGN, true, s);
    if (e != cudaSuccess) {
        set_error("k_align_batch launch: %s", cudaGetErrorString(e));
        return e;
    }
    note_launch(2);
    return cudaSuccess;
}

}  // namespace gsicp
