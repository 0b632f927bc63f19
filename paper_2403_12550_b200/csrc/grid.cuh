// Device spatial hash: counting-sort of points into voxel cells keyed by a
// 64-bit (level, cell) key in an open-addressing table.  Build = 4 kernels, O(n):
//   init  : clear the table, counters and bbox
//   insert: per (point, level) insert the cell key (atomicCAS probing), take a rank in the cell
//           (atomicAdd on its count) and fold the point into the bbox
//   alloc : per occupied slot reserve a contiguous range (warp-aggregated atomicAdd)
//   scatter: write point (and covariance) records into their cell range
// Multi-level grids of large clouds (capacity >= kTwoPhaseMin) are built in two phases: level 0
// from the caller's points, then insert / alloc / scatter of the coarser levels from level 0's
// cell-ordered records (a randomly ordered map otherwise gives every lane its own cell on every
// level: no warp aggregation, scattered writes), their alloc walking the list of cells the
// second insert created instead of the whole table (7 kernels).
// The order of cells in memory and of points inside a cell is not deterministic, but every
// consumer orders candidates by the canonical (key, index) pair, so results are.
#pragma once
#include "gsicp_internal.cuh"

namespace gsicp {

constexpr int kGridCounters = kMaxLevels + 8;
constexpr int kTwoPhaseMin = 1 << 18;  // clouds of >= this capacity: two-phase multi-level build (grid.cu)

struct GridView {
    CellEntry *table;
    uint32_t mask;
    int levels;
    float h0, inv_h0;
    float4 *spos;            // [levels * cap]: level l's points, cell-ordered, in [l*cap, l*cap + n)
                             // as (x, y, z, original index bits)
    float4 *scov_a, *scov_b; // nullable: cell-ordered covariances (target grids)
    uint2 *slot_rank;        // [levels * cap]
    uint32_t *cells;         // [levels * cap] occupied table slots in creation order (length in counters[kMaxLevels + 7])
    uint32_t *counters;      // [kMaxLevels] points allocated per level, then kGridCounters - kMaxLevels
                             // work / queue counters of the search kernels (all zeroed by the build)
    uint32_t *mark;          // nullable: one bit per table slot, zeroed by the build (tile kNN units)
    int32_t *bbox;           // [6] ordered-int encoded float min xyz / max xyz
    int cap;
    uint4 *bricks;           // nullable: the alloc step also lists the occupied level-0 cells here
    uint32_t *n_bricks;      //   as (start, count, key lo, key hi), count in *n_bricks (zeroed by init)
};

__device__ __forceinline__ int32_t float_to_ordered(float f) {
    int32_t i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float ordered_to_float(int32_t i) { return __int_as_float(i >= 0 ? i : i ^ 0x7FFFFFFF); }

// host helpers (defined in grid.cu)
size_t grid_bytes(int cap, int levels, bool with_cov, bool with_mark = false);
uint32_t grid_table_slots(int cap, int levels);
GridView grid_carve(void *base, int cap, int levels, bool with_cov, float h0, bool with_mark = false);
cudaError_t grid_build(const GridView &g, const float4 *pos, const float4 *cov_a, const float4 *cov_b,
                       const int32_t *d_n, int n_host_max, cudaStream_t s);
// automatic cell size: mean point spacing of a surface-sampled cloud (blocking; scratch >=
// spacing_scratch_bytes() device bytes, e.g. the head of a grid workspace before its build)
size_t spacing_scratch_bytes();
cudaError_t estimate_spacing(const float4 *pos, const int32_t *d_n, int cap, void *scratch, float *spacing,
                             cudaStream_t s);

// bbox of level-0 cell coordinates at level l
__device__ __forceinline__ void grid_cell_bbox(const GridView &g, int level, int lo[3], int hi[3]) {
    const float inv_h = ldexpf(g.inv_h0, -level);
    for (int a = 0; a < 3; ++a) {
        lo[a] = cell_coord(ordered_to_float(__ldg(g.bbox + a)), inv_h);
        hi[a] = cell_coord(ordered_to_float(__ldg(g.bbox + 3 + a)), inv_h);
    }
}

}  // namespace gsicp
