// Device spatial hash build (see grid.cuh).
#include <string.h>

#include <algorithm>
#include <cmath>

#include "grid.cuh"
#include "host_common.cuh"

namespace gsicp {

namespace {

__global__ void k_grid_init(CellEntry *table, uint32_t slots, uint32_t *counters, int32_t *bbox, uint32_t *mark,
                            const int32_t *__restrict__ d_n) {
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (*d_n <= 0) {  // nothing to hash (e.g. an empty fallback queue): leave the table alone
        if (i < kGridCounters) counters[i] = 0;
        return;
    }
    if (i < slots) {
        CellEntry e;
        e.key = kEmptyKey;
        e.start = 0;
        e.count = 0;
        table[i] = e;
    }
    if (mark && i < (slots + 31) / 32) mark[i] = 0u;
    if (i < kGridCounters) counters[i] = 0;  // per-level allocation + the search work / queue counters
    if (i == 0) {
        for (int a = 0; a < 3; ++a) {
            bbox[a] = float_to_ordered(INFINITY);
            bbox[3 + a] = float_to_ordered(-INFINITY);
        }
    }
}

constexpr int kInsertThreads = 256;
constexpr int kCellCtr = kMaxLevels + 7;  // counters[kCellCtr]: length of g.cells

// Levels [lev_lo, lev_hi): thread t = level * cap + i.  Level 0 reads the caller's points; the
// coarser levels (second phase of a two-phase build) read level 0's cell-ordered records instead,
// so the lanes of a warp mostly share their coarse cell (one probe + one atomic per cell and warp)
// and the scatter writes land in few cells — from a randomly ordered cloud every lane of every
// level would otherwise hit its own cell.
template <bool FROM_L0>
__global__ void __launch_bounds__(kInsertThreads) k_grid_insert(GridView g, const float4 *__restrict__ pos,
                                                               const int32_t *__restrict__ d_n, int lev_lo,
                                                               int lev_hi) {
    __shared__ uint32_t s_nc, s_cbase;
    pdl_wait();
    pdl_launch_dependents();
    const int n = *d_n;
    if (n <= 0) return;  // nothing to hash (block-uniform)
    if (threadIdx.x == 0) s_nc = 0u;
    const long long t = (long long)lev_lo * g.cap + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int level = (int)(t / g.cap);
    const int i = (int)(t - (long long)level * g.cap);
    const bool active = level < lev_hi && i < n;
    float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
    unsigned long long key = kEmptyKey;
    if (active) {
        p = FROM_L0 ? g.spos[i] : __ldg(pos + i);
        const float inv_h = ldexpf(g.inv_h0, -level);
        key = cell_key(level, cell_coord(p.x, inv_h), cell_coord(p.y, inv_h), cell_coord(p.z, inv_h));
    }
    // warp aggregation: lanes of the same cell (spatially coherent inputs share cells, most of all
    // on coarse levels) insert once and take their ranks with a single atomicAdd of the leader
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    uint32_t s = 0, base = 0;
    bool created = false;
    if (active && lane == leader) {
        s = hash_slot(key, g.mask);
        while (true) {
            // a plain read first: once a cell exists (most inserts) no CAS is issued
            const unsigned long long cur = *reinterpret_cast<volatile unsigned long long *>(&g.table[s].key);
            if (cur == key) break;
            if (cur == kEmptyKey) {
                const unsigned long long prev = atomicCAS(&g.table[s].key, kEmptyKey, key);
                if (FROM_L0 && prev == kEmptyKey) created = true;
                if (prev == kEmptyKey || prev == key) break;
            }
            s = (s + 1) & g.mask;
        }
        base = atomicAdd(&g.table[s].count, (uint32_t)__popc(peers));
    }
    s = __shfl_sync(0xffffffffu, s, leader);
    base = __shfl_sync(0xffffffffu, base, leader);
    if (active) g.slot_rank[t] = make_uint2(s, base + __popc(peers & ((1u << lane) - 1u)));
    // (second phase) the new cells join the occupied-cell list, which the alloc step walks instead
    // of the table: offsets aggregated per warp and per block, one global atomic per block
    const unsigned cb = __ballot_sync(0xffffffffu, created);
    __syncthreads();  // s_nc initialised
    uint32_t woff = 0;
    if (lane == 0 && cb) woff = atomicAdd(&s_nc, (uint32_t)__popc(cb));
    woff = __shfl_sync(0xffffffffu, woff, 0);
    // bbox of the points (level 0 lanes only), warp-reduced then one atomic per warp
    const bool bb = active && level == 0;
    float v[6] = {bb ? p.x : INFINITY, bb ? p.y : INFINITY, bb ? p.z : INFINITY,
                  bb ? p.x : -INFINITY, bb ? p.y : -INFINITY, bb ? p.z : -INFINITY};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            v[a] = fminf(v[a], __shfl_xor_sync(0xffffffffu, v[a], o));
            v[3 + a] = fmaxf(v[3 + a], __shfl_xor_sync(0xffffffffu, v[3 + a], o));
        }
    // block reduction, then one atomic per bound per block (same-address atomics serialise in L2:
    // one per warp made the bbox the bottleneck of large builds)
    __shared__ float sbb[6][kInsertThreads / 32];
    const int wid = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int a = 0; a < 6; ++a) sbb[a][wid] = v[a];
    __syncthreads();
    if (threadIdx.x == 0) s_cbase = s_nc ? atomicAdd(g.counters + kCellCtr, s_nc) : 0u;
    if (!FROM_L0 && threadIdx.x < 6) {
        const int a = threadIdx.x;
        float r = sbb[a][0];
        for (int w = 1; w < kInsertThreads / 32; ++w) r = a < 3 ? fminf(r, sbb[a][w]) : fmaxf(r, sbb[a][w]);
        if (isfinite(r)) {
            if (a < 3)
                atomicMin(g.bbox + a, float_to_ordered(r));
            else
                atomicMax(g.bbox + a, float_to_ordered(r));
        }
    }
    __syncthreads();
    if (created) g.cells[s_cbase + woff + __popc(cb & ((1u << lane) - 1u))] = s;
}

// Each level's points get the contiguous range [level*cap, level*cap + n) of spos, cells in
// allocation order.  The occupied cells of levels [lev_lo, lev_hi) are found by a scan of the
// table (table-slot order), or (from_list: the coarse levels of a two-phase build) in the cell
// list of their insert step — the table is sized for one cell per point and level, mostly empty.
// (Level 0 keeps the table order: the list's creation order front-loads the large cells, which
// measured 14% slower in the brick kernel.)  Reservations are aggregated per warp (shuffle scan) and per block (shared
// atomics), so a block issues one global atomicAdd per level for kAllocPerThread*256 cells.
constexpr int kAllocThreads = 256;
constexpr int kAllocPerThread = 4;
constexpr int kAllocChunk = kAllocThreads * kAllocPerThread;

__global__ void __launch_bounds__(kAllocThreads) k_grid_alloc(GridView g, const int32_t *__restrict__ d_n, int lev_lo,
                                                              int lev_hi, int from_list) {
    pdl_wait();
    pdl_launch_dependents();
    __shared__ uint32_t s_tot[kMaxLevels], s_base[kMaxLevels], s_bn, s_bbase;
    if (*d_n <= 0) return;
    const uint32_t nc = from_list ? g.counters[kCellCtr] : g.mask + 1;
    const int lane = threadIdx.x & 31;
    for (uint32_t c0 = blockIdx.x * kAllocChunk; c0 < nc; c0 += gridDim.x * kAllocChunk) {  // block-uniform
        if (threadIdx.x < kMaxLevels) s_tot[threadIdx.x] = 0;
        if (threadIdx.x == 0) s_bn = 0;
        __syncthreads();
        uint32_t slot[kAllocPerThread], cnt[kAllocPerThread], off[kAllocPerThread];
        unsigned long long keys[kAllocPerThread];
        int lev[kAllocPerThread];
#pragma unroll
        for (int r = 0; r < kAllocPerThread; ++r) {
            const uint32_t e = c0 + r * kAllocThreads + threadIdx.x;
            slot[r] = e < nc ? (from_list ? g.cells[e] : e) : 0u;
            keys[r] = kEmptyKey;
            cnt[r] = 0;
            lev[r] = -1;
            if (e < nc) {
                keys[r] = g.table[slot[r]].key;
                const int l = (int)(keys[r] >> 60);
                if (l >= lev_lo && l < lev_hi) {
                    lev[r] = l;
                    cnt[r] = g.table[slot[r]].count;
                }
            }
            off[r] = 0;
            for (int l = lev_lo; l < lev_hi; ++l) {
                const bool mine = lev[r] == l;
                if (!__any_sync(0xffffffffu, mine)) continue;
                const uint32_t c = mine ? cnt[r] : 0u;
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
                uint32_t wbase = 0;
                if (lane == 31) wbase = atomicAdd(s_tot + l, total);
                wbase = __shfl_sync(0xffffffffu, wbase, 31);
                if (mine) off[r] = wbase + incl - c;
            }
        }
        __syncthreads();
        if (threadIdx.x >= lev_lo && threadIdx.x < lev_hi)
            s_base[threadIdx.x] = s_tot[threadIdx.x] ? atomicAdd(g.counters + threadIdx.x, s_tot[threadIdx.x]) : 0u;
        __syncthreads();
        uint32_t start[kAllocPerThread];
#pragma unroll
        for (int r = 0; r < kAllocPerThread; ++r) {
            start[r] = lev[r] >= 0 ? (uint32_t)lev[r] * (uint32_t)g.cap + s_base[lev[r]] + off[r] : 0u;
            if (lev[r] >= 0) g.table[slot[r]].start = start[r];
        }
        if (g.bricks && lev_lo == 0) {
            // the occupied level-0 cells as a compact list: offsets aggregated per warp and per
            // block (one global atomic per block: same-address atomics per warp were the bottleneck)
            unsigned bal[kAllocPerThread];
            uint32_t wtot = 0;
#pragma unroll
            for (int r = 0; r < kAllocPerThread; ++r) {
                bal[r] = __ballot_sync(0xffffffffu, lev[r] == 0 && cnt[r] > 0);
                wtot += __popc(bal[r]);
            }
            uint32_t woff = 0;
            if (lane == 0 && wtot) woff = atomicAdd(&s_bn, wtot);
            woff = __shfl_sync(0xffffffffu, woff, 0);
            __syncthreads();
            if (threadIdx.x == 0) s_bbase = s_bn ? atomicAdd(g.n_bricks, s_bn) : 0u;
            __syncthreads();
            uint32_t pos = s_bbase + woff;
#pragma unroll
            for (int r = 0; r < kAllocPerThread; ++r) {
                if (bal[r] >> lane & 1u)
                    g.bricks[pos + __popc(bal[r] & ((1u << lane) - 1u))] =
                        make_uint4(start[r], cnt[r], (uint32_t)keys[r], (uint32_t)(keys[r] >> 32));
                pos += __popc(bal[r]);
            }
        }
        __syncthreads();  // the shared totals are read before the next chunk resets them
    }
}

// FROM_L0: levels >= 1 of a two-phase build, records copied from level 0's cell-ordered array
template <bool WITH_COV, bool FROM_L0>
__global__ void k_grid_scatter(GridView g, const float4 *__restrict__ pos, const float4 *__restrict__ cov_a,
                               const float4 *__restrict__ cov_b, const int32_t *__restrict__ d_n, int lev_lo,
                               int lev_hi) {
    pdl_wait();
    pdl_launch_dependents();
    const int n = *d_n;
    const long long t = (long long)lev_lo * g.cap + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int level = (int)(t / g.cap);
    const int i = (int)(t - (long long)level * g.cap);
    if (level >= lev_hi || i >= n) return;
    const uint2 sr = g.slot_rank[t];
    const uint32_t dst = g.table[sr.x].start + sr.y;
    if (FROM_L0) {
        g.spos[dst] = g.spos[i];
    } else {
        const float4 p = __ldg(pos + i);
        g.spos[dst] = make_float4(p.x, p.y, p.z, __int_as_float(i));
        if (WITH_COV && level == 0) {
            g.scov_a[dst] = __ldg(cov_a + i);
            g.scov_b[dst] = __ldg(cov_b + i);
        }
    }
}

// ---- spacing estimate of a cloud (the automatic cell size; a cost knob only — every search is
// exact at any cell size): occupancy of a kSpG^3 trial grid over the bbox.  For points sampled on
// surfaces at spacing l, each occupied trial cell (edge h) holds ~(h / l)^2 points, so
// l ~= h sqrt(occupied / n).
constexpr int kSpG = 32;
constexpr int kSpWords = kSpG * kSpG * kSpG / 32;  // occupancy bitmap

__global__ void k_sp_init(uint32_t *scr) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < kSpWords) scr[i] = 0u;
    if (i < 3) {
        reinterpret_cast<int32_t *>(scr + kSpWords)[i] = float_to_ordered(INFINITY);
        reinterpret_cast<int32_t *>(scr + kSpWords)[3 + i] = float_to_ordered(-INFINITY);
    }
    if (i == 0) scr[kSpWords + 6] = scr[kSpWords + 7] = 0u;
}

__global__ void k_sp_bbox(const float4 *__restrict__ pos, const int32_t *__restrict__ d_n, uint32_t *scr) {
    const int n = *d_n;
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 p = __ldg(pos + i);
        const float c[3] = {p.x, p.y, p.z};
        for (int a = 0; a < 3; ++a)
            if (isfinite(c[a])) {
                lo[a] = fminf(lo[a], c[a]);
                hi[a] = fmaxf(hi[a], c[a]);
            }
    }
    int32_t *bb = reinterpret_cast<int32_t *>(scr + kSpWords);
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(bb + a, float_to_ordered(lo[a]));
            atomicMax(bb + 3 + a, float_to_ordered(hi[a]));
        }
    }
}

__global__ void k_sp_mark(const float4 *__restrict__ pos, const int32_t *__restrict__ d_n, uint32_t *scr) {
    const int n = *d_n;
    const int32_t *bb = reinterpret_cast<const int32_t *>(scr + kSpWords);
    float lo[3], ext = 0.f;
    for (int a = 0; a < 3; ++a) {
        lo[a] = ordered_to_float(bb[a]);
        ext = fmaxf(ext, ordered_to_float(bb[3 + a]) - lo[a]);
    }
    const float inv = ext > 0.f ? (float)kSpG / ext : 0.f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 p = __ldg(pos + i);
        if (!isfinite(p.x) || !isfinite(p.y) || !isfinite(p.z)) continue;
        const int x = min(max((int)((p.x - lo[0]) * inv), 0), kSpG - 1);
        const int y = min(max((int)((p.y - lo[1]) * inv), 0), kSpG - 1);
        const int z = min(max((int)((p.z - lo[2]) * inv), 0), kSpG - 1);
        const int c = (z * kSpG + y) * kSpG + x;
        atomicOr(scr + (c >> 5), 1u << (c & 31));
    }
}

__global__ void k_sp_count(uint32_t *scr) {
    uint32_t c = 0;
    for (int i = threadIdx.x; i < kSpWords; i += blockDim.x) c += __popc(scr[i]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(scr + kSpWords + 6, c);
}

}  // namespace

size_t spacing_scratch_bytes() { return (size_t)(kSpWords + 8) * sizeof(uint32_t); }

// Blocking: reads the estimate back to the host.  scratch: >= spacing_scratch_bytes() of device memory.
cudaError_t estimate_spacing(const float4 *pos, const int32_t *d_n, int cap, void *scratch, float *spacing,
                             cudaStream_t s) {
    uint32_t *scr = static_cast<uint32_t *>(scratch);
    k_sp_init<<<blocks_for(kSpWords + 8, 256), 256, 0, s>>>(scr);
    const unsigned gb = std::min<unsigned>(blocks_for(cap, 256), (unsigned)num_sms() * 8);
    k_sp_bbox<<<gb, 256, 0, s>>>(pos, d_n, scr);
    k_sp_mark<<<gb, 256, 0, s>>>(pos, d_n, scr);
    k_sp_count<<<1, 1024, 0, s>>>(scr);
    GSICP_LAUNCH_CHECK("estimate_spacing");
    note_launch(4);
    uint32_t host[8];
    int32_t n = 0;
    cudaError_t e = cudaMemcpyAsync(host, scr + kSpWords, sizeof(host), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&n, d_n, sizeof(n), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        set_error("estimate_spacing: %s", cudaGetErrorString(e));
        return e;
    }
    auto of = [](uint32_t v) {
        const int32_t i = (int32_t)v;
        float f;
        const int32_t b = i >= 0 ? i : i ^ 0x7FFFFFFF;
        memcpy(&f, &b, sizeof f);
        return f;
    };
    float ext = 0.f;
    for (int a = 0; a < 3; ++a) ext = std::max(ext, of(host[3 + a]) - of(host[a]));
    const double occ = (double)host[6];
    double sp = 0.01;
    if (n > 1 && ext > 0.f && std::isfinite(ext) && occ > 0.0) sp = (double)ext / kSpG * std::sqrt(occ / (double)n);
    *spacing = (float)sp;
    return cudaSuccess;
}

uint32_t grid_table_slots(int cap, int levels) {
    // >= 1.25 slots per (point, level): the load factor stays <= 80% even if every point sits in
    // its own cell on every level (linear probing terminates), while real clouds (many points
    // per cell) use a small, more cache-friendly table
    uint64_t want = (5ull * (uint64_t)cap * (uint64_t)levels + 3) / 4;
    uint64_t s = 1024;
    while (s < want) s <<= 1;
    return (uint32_t)s;
}

static GridView carve(Carver &c, int cap, int levels, bool with_cov, float h0, bool with_mark) {
    GridView g{};
    const uint32_t slots = grid_table_slots(cap, levels);
    g.table = c.take<CellEntry>(slots);
    g.mask = slots - 1;
    g.levels = levels;
    g.bricks = nullptr;
    g.n_bricks = nullptr;
    g.h0 = h0;
    g.inv_h0 = h0 > 0.f ? 1.0f / h0 : 0.f;
    g.spos = c.take<float4>((size_t)levels * cap);
    g.scov_a = with_cov ? c.take<float4>(cap) : nullptr;
    g.scov_b = with_cov ? c.take<float4>(cap) : nullptr;
    g.slot_rank = c.take<uint2>((size_t)levels * cap);
    g.cells = c.take<uint32_t>((size_t)levels * cap);
    g.counters = c.take<uint32_t>(kGridCounters);
    g.mark = with_mark ? c.take<uint32_t>((slots + 31) / 32) : nullptr;
    g.bbox = c.take<int32_t>(8);
    g.cap = cap;
    return g;
}

size_t grid_bytes(int cap, int levels, bool with_cov, bool with_mark) {
    Carver c(nullptr);
    carve(c, cap, levels, with_cov, 1.f, with_mark);
    return c.bytes();
}

GridView grid_carve(void *base, int cap, int levels, bool with_cov, float h0, bool with_mark) {
    Carver c(base);
    return carve(c, cap, levels, with_cov, h0, with_mark);
}

cudaError_t grid_build(const GridView &g, const float4 *pos, const float4 *cov_a, const float4 *cov_b,
                       const int32_t *d_n, int n_host_max, cudaStream_t s) {
    const int T = 256;
    const uint32_t slots = g.mask + 1;
    // two phases (level 0 from the caller's points, then the coarser levels from level 0's
    // cell-ordered records) for large clouds; small ones (frames, already in image order) in one
    const bool two = g.levels > 1 && n_host_max >= kTwoPhaseMin;
    const int hi0 = two ? 1 : g.levels;
    const unsigned ab_list = std::min<unsigned>(blocks_for((long long)g.levels * g.cap, kAllocChunk), (unsigned)num_sms() * 4);
    launch_pdl(k_grid_init, dim3(blocks_for(slots, T)), dim3(T), 0, s, g.table, slots, g.counters, g.bbox, g.mark, d_n);
    GSICP_LAUNCH_CHECK("k_grid_init");
    int nl = 1;
    for (int ph = 0; ph < (two ? 2 : 1); ++ph) {
        const int lo = ph == 0 ? 0 : 1, hi = ph == 0 ? hi0 : g.levels;
        const long long work = (long long)(hi - lo) * g.cap;
        if (ph == 0)
            launch_pdl(k_grid_insert<false>, dim3(blocks_for(work, kInsertThreads)), dim3(kInsertThreads), 0, s, g, pos,
                       d_n, lo, hi);
        else
            launch_pdl(k_grid_insert<true>, dim3(blocks_for(work, kInsertThreads)), dim3(kInsertThreads), 0, s, g, pos,
                       d_n, lo, hi);
        GSICP_LAUNCH_CHECK("k_grid_insert");
        launch_pdl(k_grid_alloc, dim3(ph ? ab_list : blocks_for(slots, kAllocChunk)), dim3(kAllocThreads), 0, s, g, d_n, lo,
                   hi, ph);
        GSICP_LAUNCH_CHECK("k_grid_alloc");
        if (ph == 1)
            launch_pdl(k_grid_scatter<false, true>, dim3(blocks_for(work, T)), dim3(T), 0, s, g, pos, cov_a, cov_b, d_n,
                       lo, hi);
        else if (g.scov_a)
            launch_pdl(k_grid_scatter<true, false>, dim3(blocks_for(work, T)), dim3(T), 0, s, g, pos, cov_a, cov_b, d_n,
                       lo, hi);
        else
            launch_pdl(k_grid_scatter<false, false>, dim3(blocks_for(work, T)), dim3(T), 0, s, g, pos, cov_a, cov_b, d_n,
                       lo, hi);
        GSICP_LAUNCH_CHECK("k_grid_scatter");
        nl += 3;
    }
    note_launch(nl);
    return cudaSuccess;
}

}  // namespace gsicp
