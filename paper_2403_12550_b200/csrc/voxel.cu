// N4 voxel downsampling (at most one output point per occupied voxel, the centroid
// of its members; reading R31): voxel = (floor(x/h), floor(y/h), floor(z/h)) with binary64
// division; centroid = binary64 sum of the members / count, rounded to binary32; outputs in the
// order of each voxel's smallest input index (stable), w = member count (int bits).
// Kernels: clear the open-addressing voxel table; insert every point (atomicCAS on the packed
// voxel key, binary64 atomicAdd of the coordinates — exact for members of one voxel, whose
// coordinates share their binary exponents up to a few bits, so the order of the adds does not
// change the sum —, atomicAdd of the count, atomicMin of the first index); mark the points that
// are their voxel's first member; tile counts + prefix + in-tile ballot rank (as k_export) write
// the centroids compactly.  HBM traffic ~ 16 B in + (16 B out per voxel) + the table.
#include "gsicp_internal.cuh"
#include "host_common.cuh"

namespace gsicp {

namespace {

constexpr int kVoxThreads = 256;
constexpr unsigned long long kVoxEmpty = ~0ull;

struct VoxWs {
    unsigned long long *keys;
    double *sum;  // [slots][3]
    uint32_t *cnt, *first;
    int32_t *slot;  // [cap] voxel slot of each point (-1: skipped)
    int32_t *tile_count;
    uint32_t mask;
};

static uint32_t vox_slots(int cap) {
    uint32_t s = 1024;
    while (s < (uint32_t)cap + (uint32_t)cap / 4u) s <<= 1;  // load <= 0.8 even if every point is its own voxel
    return s;
}

static VoxWs vox_carve(Carver &c, int cap) {
    VoxWs w;
    const uint32_t slots = vox_slots(cap);
    w.mask = slots - 1;
    w.keys = c.take<unsigned long long>(slots);
    w.sum = c.take<double>((size_t)slots * 3);
    w.cnt = c.take<uint32_t>(slots);
    w.first = c.take<uint32_t>(slots);
    w.slot = c.take<int32_t>(cap);
    w.tile_count = c.take<int32_t>((cap + kVoxThreads - 1) / kVoxThreads);
    return w;
}

__device__ __forceinline__ uint32_t vox_hash(unsigned long long k, uint32_t mask) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    return (uint32_t)k & mask;
}

__global__ void k_vox_clear(VoxWs w) {
    pdl_wait();
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s <= w.mask; s += gridDim.x * blockDim.x) {
        w.keys[s] = kVoxEmpty;
        w.sum[3 * (size_t)s] = 0.0;
        w.sum[3 * (size_t)s + 1] = 0.0;
        w.sum[3 * (size_t)s + 2] = 0.0;
        w.cnt[s] = 0u;
        w.first[s] = 0xffffffffu;
    }
}

// Warp-aggregated insert: the lanes of a warp holding points of the same voxel (adjacent pixels
// mostly) elect their lowest lane — also their smallest index — which inserts the key and adds the
// group's binary64 sums (exact, so the grouping does not change them) with one set of atomics.
__global__ void k_vox_insert(VoxWs w, const float4 *__restrict__ pos, const int32_t *__restrict__ d_n, double h) {
    pdl_wait();
    const int n = *d_n;
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < n; base += warps * 32) {
        const int i = base + lane;
        float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
        bool valid = i < n;
        if (valid) {
            p = pos[i];
            valid = isfinite(p.x) && isfinite(p.y) && isfinite(p.z);
            if (!valid) w.slot[i] = -1;
        }
        unsigned long long key = kVoxEmpty;  // (never a real key: bit 63 is clear in every packed key)
        if (valid) {
            const long long ix = (long long)floor(__ddiv_rn((double)p.x, h));
            const long long iy = (long long)floor(__ddiv_rn((double)p.y, h));
            const long long iz = (long long)floor(__ddiv_rn((double)p.z, h));
            // 21 bits per axis (two's complement, masked): voxels within +-2^20 of the origin
            key = ((unsigned long long)(ix & 0x1fffff) << 42) | ((unsigned long long)(iy & 0x1fffff) << 21) |
                  (unsigned long long)(iz & 0x1fffff);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(peers) - 1;
        double sx = 0.0, sy = 0.0, sz = 0.0;
        for (int src = 0; src < 32; ++src) {  // the group's sums at its leader (all lanes shuffle)
            const float vx = __shfl_sync(0xffffffffu, p.x, src), vy = __shfl_sync(0xffffffffu, p.y, src),
                        vz = __shfl_sync(0xffffffffu, p.z, src);
            if ((peers >> src) & 1u) {
                sx += (double)vx;
                sy += (double)vy;
                sz += (double)vz;
            }
        }
        int s = -1;
        if (valid && lane == leader) {
            uint32_t t = vox_hash(key, w.mask);
            while (true) {
                const unsigned long long prev = atomicCAS(&w.keys[t], kVoxEmpty, key);
                if (prev == kVoxEmpty || prev == key) break;
                t = (t + 1) & w.mask;
            }
            s = (int)t;
            atomicAdd(&w.sum[3 * (size_t)t], sx);
            atomicAdd(&w.sum[3 * (size_t)t + 1], sy);
            atomicAdd(&w.sum[3 * (size_t)t + 2], sz);
            atomicAdd(&w.cnt[t], (uint32_t)__popc(peers));
            atomicMin(&w.first[t], (uint32_t)i);
        }
        s = __shfl_sync(0xffffffffu, s, leader);
        if (valid) w.slot[i] = s;
    }
}

__device__ __forceinline__ bool vox_is_first(const VoxWs &w, int i, int n) {
    if (i >= n) return false;
    const int s = w.slot[i];
    return s >= 0 && w.first[s] == (uint32_t)i;
}

__global__ void __launch_bounds__(kVoxThreads) k_vox_count(VoxWs w, const int32_t *__restrict__ d_n, int tiles) {
    pdl_wait();
    const int n = *d_n;
    for (int b = blockIdx.x; b < tiles; b += gridDim.x) {
        const int c = __syncthreads_count(vox_is_first(w, b * kVoxThreads + threadIdx.x, n));
        if (threadIdx.x == 0) w.tile_count[b] = c;
    }
}

__global__ void __launch_bounds__(kVoxThreads) k_vox_emit(VoxWs w, const int32_t *__restrict__ d_n, int tiles,
                                                          float4 *__restrict__ out, int32_t *__restrict__ d_m) {
    __shared__ int sWarp[kVoxThreads / 32];
    __shared__ int sBase;
    pdl_wait();
    const int n = *d_n;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int b = blockIdx.x; b < tiles; b += gridDim.x) {
        int part = 0;
        for (int t = threadIdx.x; t < b; t += kVoxThreads) part += w.tile_count[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) sWarp[wid] = part;
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int k = 0; k < kVoxThreads / 32; ++k) s += sWarp[k];
            sBase = s;
        }
        __syncthreads();
        const int i = b * kVoxThreads + threadIdx.x;
        const bool take = vox_is_first(w, i, n);
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if (lane == 0) sWarp[wid] = __popc(bal);
        __syncthreads();
        int before = sBase;
        for (int k = 0; k < wid; ++k) before += sWarp[k];
        if (take) {
            const int s = w.slot[i];
            const double c = (double)w.cnt[s];
            out[before + __popc(bal & ((1u << lane) - 1u))] =
                make_float4((float)(w.sum[3 * (size_t)s] / c), (float)(w.sum[3 * (size_t)s + 1] / c),
                            (float)(w.sum[3 * (size_t)s + 2] / c), __int_as_float((int)w.cnt[s]));
        }
        if (b == tiles - 1 && threadIdx.x == kVoxThreads - 1) *d_m = before + __popc(bal);
        __syncthreads();
    }
}

}  // namespace

size_t voxel_ws_bytes(int cap) {
    Carver c(nullptr);
    vox_carve(c, cap);
    return c.bytes();
}

cudaError_t voxel_launch(const float4 *pos, const int32_t *d_n, int cap, float voxel, float4 *out, int32_t *d_m,
                         void *ws, cudaStream_t s) {
    Carver c(ws);
    VoxWs w = vox_carve(c, cap);
    const int tiles = (cap + kVoxThreads - 1) / kVoxThreads;
    const int grid = tiles < 8 * num_sms() ? tiles : 8 * num_sms();
    const int cgrid = (int)((w.mask + 1 + 255) / 256) < 8 * num_sms() ? (int)((w.mask + 1 + 255) / 256) : 8 * num_sms();
    cudaError_t e;
    if ((e = launch_pdl(k_vox_clear, dim3(cgrid), dim3(256), 0, s, w)) != cudaSuccess) return e;
    if ((e = launch_pdl(k_vox_insert, dim3(grid), dim3(kVoxThreads), 0, s, w, pos, d_n, (double)voxel)) != cudaSuccess)
        return e;
    if ((e = launch_pdl(k_vox_count, dim3(grid), dim3(kVoxThreads), 0, s, w, d_n, tiles)) != cudaSuccess) return e;
    if ((e = launch_pdl(k_vox_emit, dim3(grid), dim3(kVoxThreads), 0, s, w, d_n, tiles, out, d_m)) != cudaSuccess)
        return e;
    note_launch(4);
    return cudaSuccess;
}

}  // namespace gsicp
