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
#include "gsicp_internal.cuh"
#include "host_common.cuh"

namespace gsicp {

namespace {

struct ExportArgs {
    const float4 *pos, *cov_a, *cov_b;
    const int32_t *d_n;
    const double *T;  // device, row-major 4x4, nullable
    double p, c;
    float *means, *quats, *scales;
};

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

__global__ void __launch_bounds__(256) k_export(ExportArgs a) {
    pdl_wait();
    const int n = *a.d_n;
    double T[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) T[k] = a.T ? a.T[k] : ((k == 0 || k == 5 || k == 10) ? 1.0 : 0.0);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
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
        const size_t i3 = 3 * (size_t)i, i4 = 4 * (size_t)i;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            a.means[i3 + r] = m[r];
            a.scales[i3 + r] = (float)(f * sqrt(e.lam[r]));
        }
        *reinterpret_cast<float4 *>(a.quats + i4) = make_float4((float)q[0], (float)q[1], (float)q[2], (float)q[3]);
    }
}

}  // namespace

cudaError_t export_launch(const float4 *pos, const float4 *cov_a, const float4 *cov_b, const int32_t *d_n, int cap,
                          const double *d_T, double p, double c, float *means, float *quats, float *scales,
                          cudaStream_t s) {
    ExportArgs a{pos, cov_a, cov_b, d_n, d_T, p, c, means, quats, scales};
    const int blocks = (cap + 255) / 256 < 8 * num_sms() ? (cap + 255) / 256 : 8 * num_sms();
    note_launch();
    return launch_pdl(k_export, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, s, a);
}

}  // namespace gsicp
