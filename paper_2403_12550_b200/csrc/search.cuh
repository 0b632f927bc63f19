// Exact grid search helpers shared by the kNN (A3) and correspondence (A6) kernels.
//
// A query q in cell c (edge h) first scans its own cell, then whole Chebyshev shells only while
// it holds too few candidates (shells 1..3 come from a constant table ordered nearest-first),
// then runs a ball traversal: every remaining cell whose conservative box lower bound is <= the
// current bound (the K-th key, or min(best, r^2) for the gated 1-NN) is scanned.  That is
// exactly the set of cells that can hold a better candidate, so the result is exact at any cell
// size; the cell size only sets the cost.  Binary32 rounding of the cell assignment and of the
// keys is absorbed by a conservative margin on every bound.
#pragma once
#include "gsicp_internal.cuh"
#include "shell_offsets.inc"

namespace gsicp {

constexpr float kRelMargin = 1e-5f;
constexpr int kLookupBatch = 8;  // independent hash probes in flight per thread

__device__ __forceinline__ void shell_cell(int m, int t, int &dx, int &dy, int &dz) {
    if (m <= 3) {
        const char4 o = kShellOffsets[(m == 1 ? 0 : (m == 2 ? 26 : 124)) + t];
        dx = o.x;
        dy = o.y;
        dz = o.z;
    } else {
        shell_offset(m, t, dx, dy, dz);
    }
}

// Query-side geometry for one level.
struct QueryCell {
    int c[3];
    float dlo[3], dhi[3];
    float dq;      // distance to the nearest own-cell face
    float margin;  // absolute slack for rounding
    float h;

    __device__ __forceinline__ QueryCell(float qx, float qy, float qz, float h_, float inv_h) {
        h = h_;
        const float q[3] = {qx, qy, qz};
        c[0] = cell_coord(qx, inv_h);
        c[1] = cell_coord(qy, inv_h);
        c[2] = cell_coord(qz, inv_h);
        dq = INFINITY;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            dlo[a] = fmaxf(q[a] - (float)c[a] * h, 0.f);
            dhi[a] = fmaxf((float)(c[a] + 1) * h - q[a], 0.f);
            dq = fminf(dq, fminf(dlo[a], dhi[a]));
        }
        margin = 2e-6f * (fabsf(qx) + fabsf(qy) + fabsf(qz)) + h * kRelMargin;
    }
    // after shells 0..m are scanned, every unscanned point has key >= certified_key(m)
    __device__ __forceinline__ float certified_key(int m) const {
        const float B = fmaxf((float)m * h + dq - margin, 0.f);
        return B * B * (1.f - kRelMargin);
    }
    __device__ __forceinline__ bool covers(int m, const int *blo, const int *bhi) const {
        return c[0] - m <= blo[0] && c[0] + m >= bhi[0] && c[1] - m <= blo[1] && c[1] + m >= bhi[1] &&
               c[2] - m <= blo[2] && c[2] + m >= bhi[2];
    }
    // conservative squared gap along axis a to the cells at offset o
    __device__ __forceinline__ float gap2(int o, int a) const {
        const float g = fmaxf(axis_gap(o, dlo[a], dhi[a], h) - margin, 0.f);
        return g * g * (1.f - kRelMargin);
    }
};

// Offsets along one axis whose squared gap stays <= room, clipped to the cells [blo, bhi]:
// returns [lo, hi] (empty if lo > hi).
__device__ __forceinline__ void axis_range(const QueryCell &qc, int a, float room, int blo, int bhi, int &lo,
                                           int &hi) {
    int p = 0;
    while (qc.c[a] + p < bhi && qc.gap2(p + 1, a) <= room) ++p;
    int q = 0;
    while (qc.c[a] + q > blo && qc.gap2(q - 1, a) <= room) --q;
    lo = max(q, blo - qc.c[a]);
    hi = min(p, bhi - qc.c[a]);
}

// 0, -1, 1, -2, 2, ...
__device__ __forceinline__ int zigzag(int k) { return (k & 1) ? -((k + 1) >> 1) : (k >> 1); }


// Cell index of a grid: the open-addressing hash table always, plus (targets only) a dense
// (start, count) array over the bbox when it fits its budget — then a lookup is one load with
// no hashing or probing, and neighbouring cells along x are adjacent in memory.
struct CellIndex {
    const CellEntry *table;
    uint32_t mask;
    int level;
    const uint2 *dense;  // nullable
    int lo[3], dim[3];
    bool use_dense;

    __device__ __forceinline__ uint2 one(int x, int y, int z) const {
        if (use_dense) {
            const int ix = x - lo[0], iy = y - lo[1], iz = z - lo[2];
            if ((unsigned)ix >= (unsigned)dim[0] || (unsigned)iy >= (unsigned)dim[1] || (unsigned)iz >= (unsigned)dim[2])
                return make_uint2(0u, 0u);
            return __ldg(dense + ((size_t)iz * dim[1] + iy) * dim[0] + ix);
        }
        return cell_lookup(table, mask, cell_key(level, x, y, z));
    }

    // B lookups with all first loads in flight together; invalid entries give (0, 0)
    template <int B>
    __device__ __forceinline__ void batch(const int (&xs)[B], const int (&ys)[B], const int (&zs)[B],
                                          const bool (&valid)[B], uint2 (&se)[B]) const {
        if (use_dense) {
#pragma unroll
            for (int j = 0; j < B; ++j) se[j] = valid[j] ? one(xs[j], ys[j], zs[j]) : make_uint2(0u, 0u);
            return;
        }
        unsigned long long keys[B];
        uint4 e[B];
        uint32_t s[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
            keys[j] = cell_key(level, xs[j], ys[j], zs[j]);
            s[j] = hash_slot(keys[j], mask);
            e[j] = valid[j] ? __ldg(reinterpret_cast<const uint4 *>(table + s[j])) : make_uint4(0xffffffffu, 0xffffffffu, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < B; ++j) {
            se[j] = make_uint2(0u, 0u);
            if (!valid[j]) continue;
            while (true) {
                const unsigned long long k = ((unsigned long long)e[j].y << 32) | e[j].x;
                if (k == keys[j]) {
                    se[j] = make_uint2(e[j].z, e[j].w);
                    break;
                }
                if (k == kEmptyKey) break;
                s[j] = (s[j] + 1) & mask;
                e[j] = __ldg(reinterpret_cast<const uint4 *>(table + s[j]));
            }
        }
    }
};

// Ball traversal over the cells not yet scanned (skip(dx, dy, dz) is true for those already done).
// Rows (fixed y, z) are pruned by their gap; inside a row the x-extent is computed from the gaps
// alone (no loads), then cells are looked up kLookupBatch at a time, nearest first, and a cell is
// scanned only if its lower bound is still <= bound() (which may shrink while scanning).
//   scan(uint2 start_count);  bound() -> float
// kCompact: one (non-unrolled) copy of scan() per batch instead of kLookupBatch inlined copies —
// for callers whose scan() is large (register-resident best-K lists).
template <bool kCompact = false, int B = kLookupBatch, class Skip, class Scan, class Bound>
__device__ __forceinline__ void ball_search(const QueryCell &qc, const CellIndex &idx, const int *blo, const int *bhi,
                                            Skip skip, Scan scan, Bound bound) {
    int zlo, zhi;
    axis_range(qc, 2, bound(), blo[2], bhi[2], zlo, zhi);
    for (int kz = 0; kz <= 2 * max(-zlo, zhi); ++kz) {
        const int dz = zigzag(kz);
        if (dz < zlo || dz > zhi) continue;
        const float gz = qc.gap2(dz, 2);
        if (gz > bound()) continue;
        int ylo, yhi;
        axis_range(qc, 1, bound() - gz, blo[1], bhi[1], ylo, yhi);
        for (int ky = 0; ky <= 2 * max(-ylo, yhi); ++ky) {
            const int dy = zigzag(ky);
            if (dy < ylo || dy > yhi) continue;
            const float gzy = gz + qc.gap2(dy, 1);
            if (gzy > bound()) continue;
            int xlo, xhi;
            axis_range(qc, 0, bound() - gzy, blo[0], bhi[0], xlo, xhi);
            const int kxmax = 2 * max(-xlo, xhi);
            for (int kx0 = 0; kx0 <= kxmax; kx0 += B) {
                int xs[B], ys[B], zs[B];
                bool valid[B];
                float lb[B];
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int dx = zigzag(kx0 + j);
                    valid[j] = kx0 + j <= kxmax && dx >= xlo && dx <= xhi && !skip(dx, dy, dz);
                    lb[j] = gzy + qc.gap2(dx, 0);
                    xs[j] = qc.c[0] + dx;
                    ys[j] = qc.c[1] + dy;
                    zs[j] = qc.c[2] + dz;
                }
                uint2 se[B];
                idx.batch(xs, ys, zs, valid, se);
                if (kCompact) {
                    uint32_t live = 0;
#pragma unroll
                    for (int j = 0; j < B; ++j) live |= (se[j].y ? 1u : 0u) << j;
                    while (live) {
                        const int j = __ffs(live) - 1;
                        live &= live - 1;
                        uint2 sj = se[0];
                        float lj = lb[0];
#pragma unroll
                        for (int r = 1; r < B; ++r)
                            if (r == j) {
                                sj = se[r];
                                lj = lb[r];
                            }
                        if (lj <= bound()) scan(sj);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < B; ++j)
                        if (se[j].y && lb[j] <= bound()) scan(se[j]);
                }
            }
        }
    }
}

}  // namespace gsicp
