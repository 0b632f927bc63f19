// A1  Depth back-projection + uniform stride downsampling (Fig. 2; pinhole S:46).
// Two kernels: per-tile valid counts, then each tile sums the counts before it (a few hundred
// ints at most), block-scans its own flags and writes the stable row-major compaction.
// K1 (R13): x = (float)(((double)u - (double)cx) * (double)z / (double)fx), binary64, no FMA.
#include "gsicp_internal.cuh"
#include "host_common.cuh"

namespace gsicp {

namespace {

constexpr int kBpThreads = 256;
constexpr int kBpPerThread = 4;
constexpr int kBpTile = kBpThreads * kBpPerThread;

struct BpArgs {
    const float *depth;
    int H, W, pitch, stride, Ws, Hs;  // Ws, Hs: sampled lattice size
    int rows_sampled;                 // depth holds only the sampled rows (row r = image row r*stride)
    int32_t *map;                     // nullable [Hs*Ws]: output index of each sampled pixel, -1 if invalid
    float fx, fy, cx, cy, zmin, zmax;
    float4 *out;
    int32_t *d_n;
    uint32_t *tile_counts;
    int tiles;
};

__device__ __forceinline__ bool bp_valid(const BpArgs &a, int j, float &z, int &u, int &v) {
    if (j >= a.Ws * a.Hs) return false;
    const int vs = j / a.Ws, us = j - vs * a.Ws;
    u = us * a.stride;
    v = vs * a.stride;
    z = __ldg(a.depth + (size_t)(a.rows_sampled ? vs : v) * a.pitch + u);
    return isfinite(z) && z >= a.zmin && z <= a.zmax;
}

__global__ void k_bp_count(BpArgs a) {
    pdl_wait();
    pdl_launch_dependents();
    __shared__ uint32_t warp_tot[kBpThreads / 32];
    const int base = blockIdx.x * kBpTile + threadIdx.x * kBpPerThread;
    uint32_t c = 0;
#pragma unroll
    for (int e = 0; e < kBpPerThread; ++e) {
        float z;
        int u, v;
        c += bp_valid(a, base + e, z, u, v) ? 1u : 0u;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kBpThreads / 32; ++w) t += warp_tot[w];
        a.tile_counts[blockIdx.x] = t;
    }
}

__global__ void k_bp_emit(BpArgs a) {
    pdl_wait();
    pdl_launch_dependents();
    __shared__ uint32_t red[kBpThreads / 32];
    __shared__ uint32_t warp_excl[kBpThreads / 32];
    __shared__ uint32_t s_prefix;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // exclusive prefix of this tile = sum of earlier tile counts
    uint32_t acc = 0;
    for (int t = threadIdx.x; t < blockIdx.x; t += kBpThreads) acc += a.tile_counts[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    // local flags
    const int base = blockIdx.x * kBpTile + threadIdx.x * kBpPerThread;
    float z[kBpPerThread];
    int u[kBpPerThread], v[kBpPerThread];
    bool ok[kBpPerThread];
    uint32_t mine = 0;
#pragma unroll
    for (int e = 0; e < kBpPerThread; ++e) {
        ok[e] = bp_valid(a, base + e, z[e], u[e], v[e]);
        mine += ok[e] ? 1u : 0u;
    }
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_excl[warp] = incl;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t p = 0;
        for (int w = 0; w < kBpThreads / 32; ++w) p += red[w];
        s_prefix = p;
        uint32_t run = 0;
        for (int w = 0; w < kBpThreads / 32; ++w) {
            const uint32_t t = warp_excl[w];
            warp_excl[w] = run;
            run += t;
        }
        if (blockIdx.x == a.tiles - 1) *a.d_n = (int32_t)(p + run);
    }
    __syncthreads();
    uint32_t dst = s_prefix + warp_excl[warp] + incl - mine;
    if (a.map) {
        uint32_t d2 = dst;
#pragma unroll
        for (int e = 0; e < kBpPerThread; ++e)
            if (base + e < a.Ws * a.Hs) a.map[base + e] = ok[e] ? (int32_t)(d2++) : -1;
    }
#pragma unroll
    for (int e = 0; e < kBpPerThread; ++e) {
        if (!ok[e]) continue;
        const double zd = (double)z[e];
        const double x = __ddiv_rn(__dmul_rn(__dsub_rn((double)u[e], (double)a.cx), zd), (double)a.fx);
        const double y = __ddiv_rn(__dmul_rn(__dsub_rn((double)v[e], (double)a.cy), zd), (double)a.fy);
        a.out[dst++] = make_float4(__double2float_rn(x), __double2float_rn(y), z[e], __int_as_float(v[e] * a.W + u[e]));
    }
}

}  // namespace

size_t backproject_ws_bytes(int H, int W, int stride) {
    const long long Ws = (W + stride - 1) / stride, Hs = (H + stride - 1) / stride;
    const long long tiles = (Ws * Hs + kBpTile - 1) / kBpTile;
    return align_up((size_t)(tiles > 0 ? tiles : 1) * sizeof(uint32_t));
}

cudaError_t backproject_launch(const float *depth, int H, int W, int pitch, gsicp_intrinsics K, int stride,
                               float zmin, float zmax, float *pos_out, int32_t *d_n, void *ws, cudaStream_t s,
                               int rows_sampled, int32_t *map) {
    BpArgs a;
    a.rows_sampled = rows_sampled;
    a.map = map;
    a.depth = depth;
    a.H = H; a.W = W; a.pitch = pitch; a.stride = stride;
    a.Ws = (W + stride - 1) / stride;
    a.Hs = (H + stride - 1) / stride;
    a.fx = K.fx; a.fy = K.fy; a.cx = K.cx; a.cy = K.cy;
    a.zmin = zmin; a.zmax = zmax;
    a.out = reinterpret_cast<float4 *>(pos_out);
    a.d_n = d_n;
    a.tile_counts = static_cast<uint32_t *>(ws);
    a.tiles = (int)(((long long)a.Ws * a.Hs + kBpTile - 1) / kBpTile);
    ktimer_mark(KT_BP, false, s);
    launch_pdl(k_bp_count, dim3(a.tiles), dim3(kBpThreads), 0, s, a);
    GSICP_LAUNCH_CHECK("k_bp_count");
    launch_pdl(k_bp_emit, dim3(a.tiles), dim3(kBpThreads), 0, s, a);
    GSICP_LAUNCH_CHECK("k_bp_emit");
    ktimer_mark(KT_BP, true, s);
    note_launch(2);
    return cudaSuccess;
}

}  // namespace gsicp
