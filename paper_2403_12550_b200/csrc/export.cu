// A4 export: source points -> 3DGS Gaussians for map insertion (ALG-12).
//   Eq. 3 C = R Lambda^2 R^T; Eq. 4 Lambda' = Lambda / median(S);
//   scale aligning Lambda'' = Lambda' / z^p, with the absolute factor c (R21).
// The stored regularised covariance (cov_a/cov_b, written by gsicp_covariances*) IS
// sum_i var'_i v_i v_i^T with the mode's regularised variances var' (R6-R8: ELLIPSE
// max(lam_i/lam_1, eps), PLANE (1, 1, eps), NONE max(lam_i, 1e-6), degenerate I or
// v2v2^T + eps(I - v2v2^T)), so its eigen-decomposition gives Lambda'^2 and the frame
// directly: the export reads 48 B per point and writes 40 B, runs only for the frames that
// become keyframes, and leaves the per-frame kNN kernels untouched.
// Per point: closed-form binary64 eigen (eig3_sym) of the stored covariance; scales
// c * sqrt(var'_j) / z^p (z = the camera-frame depth pos.z; z <= 0 -> scales 0); frame
// (v2, v1, v0) made right-handed, rotated into the world by T's rotation, as a unit wxyz
// quaternion with w >= 0; mean K3(T, x) rounded to binary32 (T null: identity).
// Overlap filter ("only Gaussians that do not overlap with the existing current map are
// considered as target Gaussians"; R28): with a correspondence array, only the points WITHOUT a
// valid correspondence in the final linearisation (corr < 0: no map mean within the distance
// threshold, the same test that gives the keyframe proportion) are exported,
// compacted stably in index order: tile counts (k_export_count, __syncthreads_count), then each
// tile's offset = the sum of the earlier tiles' counts and the rank inside the tile from warp
// ballots.
#include "gsicp_internal.cuh"
#include "host_common.cuh"

namespace gsicp {

namespace {

constexpr int kExportThreads = 256;  // = one tile of points per block

struct ExportArgs {
    const float4 *pos, *cov_a, *cov_b;
    const int32_t *d_n;
    const double *T;  // device, row-major 4x4, nullable
    double p, c;
    float *means, *quats, *scales;
    const int32_t *corr;  // nullable: export only corr < 0, compacted
    int32_t *tile_count;  // [tiles] (corr only)
    int32_t *d_m;         // nullable: rows written
    const int32_t *d_base;  // nullable: rows are written at *d_base + row (appending to a map, N1)
};

__global__ void __launch_bounds__(kExportThreads) k_export_count(const int32_t *__restrict__ corr,
                                                                   const int32_t *__restrict__ d_n,
                                                                   int32_t *__restrict__ tile_count, int tiles) {
    pdl_wait();
    const int n = *d_n;
    for (int b = blockIdx.x; b < tiles; b += gridDim.x) {
        const int i = b * kExportThreads + threadIdx.x;
        const int c = __syncthreads_count(i < n && corr[i] < 0);
        if (threadIdx.x == 0) tile_count[b] = c;
    }
}

// unit quaternion (w >= 0) of a rotation matrix: the largest of 4w^2-1 = tr, 4x^2-1 = 2R00 - tr, ...
// selects the division-safe formula (Shepperd)
__device__ __forceinline__ void rot_to_quat(const double (&R)[3][3], double (&q)[4]) {
    const double tr = R[0][0] + R[1][1] + R[2][2];
    if (tr >= R[0][0] && tr >= R[1][1] && tr >= R[2][2]) {
        const double s = 2.0 * sqrt(1.0 + tr);
        q[0] = 0.25 * s; q[1] = (R[2][1] - R[1][2]) / s; q[2] = (R[0][2] - R[2][0]) / s; q[3] = (R[1][0] - R[0][1]) / s;
    } else if (R[0][0] >= R[1][1] && R[0][0] >= R[2][2]) {
        const double s = 2.0 * sqrt(1.0 + R[0][0] - R[1][1] - R[2][2]);
        q[0] = (R[2][1] - R[1][2]) / s; q[1] = 0.25 * s; q[2] = (R[0][1] + R[1][0]) / s; q[3] = (R[0][2] + R[2][0]) / s;
    } else if (R[1][1] >= R[2][2]) {
        const double s = 2.0 * sqrt(1.0 + R[1][1] - R[0][0] - R[2][2]);
        q[0] = (R[0][2] - R[2][0]) / s; q[1] = (R[0][1] + R[1][0]) / s; q[2] = 0.25 * s; q[3] = (R[1][2] + R[2][1]) / s;
    } else {
        const double s = 2.0 * sqrt(1.0 + R[2][2] - R[0][0] - R[1][1]);
        q[0] = (R[1][0] - R[0][1]) / s; q[1] = (R[0][2] + R[2][0]) / s; q[2] = (R[1][2] + R[2][1]) / s; q[3] = 0.25 * s;
    }
    const double inv = (q[0] < 0.0 ? -1.0 : 1.0) * gs_rsqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] *= inv;
}

__global__ void __launch_bounds__(kExportThreads) k_export(ExportArgs a, int tiles) {
    __shared__ int sWarp[kExportThreads / 32];
    __shared__ int sBase;
    pdl_wait();
    const int n = *a.d_n;
    double T[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) T[k] = a.T ? a.T[k] : ((k == 0 || k == 5 || k == 10) ? 1.0 : 0.0);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int b = blockIdx.x; b < tiles; b += gridDim.x) {
        const int i = b * kExportThreads + threadIdx.x;
        int row = i;
        bool take = i < n;
        if (a.corr) {
            // tile offset = sum of the earlier tiles' counts (block-strided sum + warp reductions)
            int part = 0;
            for (int t = threadIdx.x; t < b; t += kExportThreads) part += a.tile_count[t];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            if (lane == 0) sWarp[wid] = part;
            __syncthreads();
            if (threadIdx.x == 0) {
                int s = 0;
                for (int w = 0; w < kExportThreads / 32; ++w) s += sWarp[w];
                sBase = s;
            }
            __syncthreads();
            take = take && a.corr[i] < 0;
            const unsigned bal = __ballot_sync(0xffffffffu, take);
            if (lane == 0) sWarp[wid] = __popc(bal);
            __syncthreads();
            int before = sBase;
            for (int w = 0; w < wid; ++w) before += sWarp[w];
            row = before + __popc(bal & ((1u << lane) - 1u));
            if (b == tiles - 1 && threadIdx.x == kExportThreads - 1 && a.d_m) *a.d_m = before + __popc(bal);
            __syncthreads();  // sWarp / sBase reused by the next tile
        } else if (b == 0 && threadIdx.x == 0 && a.d_m) {
            *a.d_m = n;
        }
        if (!take) continue;
        const float4 x = a.pos[i], ca = a.cov_a[i], cb = a.cov_b[i];
        const double C[6] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y};
        const Eig3 e = eig3_sym(C);
        const double z = x.z;
        const double f = z > 0.0 ? a.c / pow(z, a.p) : 0.0;
        // frame columns (v2, v1, v0) = e.v[0..2]; right-handed: v0 <- -v0 if det < 0
        double F[3][3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int j = 0; j < 3; ++j) F[r][j] = e.v[j][r];
        double cr[3];
        cross3(e.v[0], e.v[1], cr);
        if (dot3(cr, e.v[2]) < 0.0)
#pragma unroll
            for (int r = 0; r < 3; ++r) F[r][2] = -F[r][2];
        double Rw[3][3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int j = 0; j < 3; ++j) Rw[r][j] = T[4 * r] * F[0][j] + T[4 * r + 1] * F[1][j] + T[4 * r + 2] * F[2][j];
        double q[4];
        rot_to_quat(Rw, q);
        // K3 (R15): ((R_r0 x + R_r1 y) + R_r2 z) + t_r, no contraction
        const double xd = x.x, yd = x.y, zd = x.z;
        float m[3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
            m[r] = (float)__dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(T[4 * r], xd), __dmul_rn(T[4 * r + 1], yd)),
                                              __dmul_rn(T[4 * r + 2], zd)),
                                    T[4 * r + 3]);
        if (a.d_base) row += *a.d_base;
        const size_t i3 = 3 * (size_t)row, i4 = 4 * (size_t)row;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            a.means[i3 + r] = m[r];
            a.scales[i3 + r] = (float)(f * sqrt(e.lam[r]));
        }
        *reinterpret_cast<float4 *>(a.quats + i4) = make_float4((float)q[0], (float)q[1], (float)q[2], (float)q[3]);
    }
}

}  // namespace

size_t export_ws_bytes(int cap) { return (size_t)((cap + kExportThreads - 1) / kExportThreads) * 4 + 256; }

cudaError_t export_launch(const float4 *pos, const float4 *cov_a, const float4 *cov_b, const int32_t *d_n, int cap,
                          const double *d_T, double p, double c, const int32_t *corr, float *means, float *quats,
                          float *scales, int32_t *d_m, void *ws, cudaStream_t s, const int32_t *d_base) {
    const int tiles = (cap + kExportThreads - 1) / kExportThreads;
    ExportArgs a{pos, cov_a, cov_b, d_n, d_T, p, c, means, quats, scales, corr, (int32_t *)ws, d_m, d_base};
    const int blocks = tiles < 8 * num_sms() ? tiles : 8 * num_sms();
    if (corr) {
        const cudaError_t e = launch_pdl(k_export_count, dim3(blocks), dim3(kExportThreads), 0, s, corr, d_n,
                                         a.tile_count, tiles);
        note_launch();
        if (e != cudaSuccess) return e;
    }
    note_launch();
    return launch_pdl(k_export, dim3(blocks), dim3(kExportThreads), 0, s, a, tiles);
}

}  // namespace gsicp
