// C ABI of libgsicp (include/gsicp.h): argument validation, workspace carving, status mapping.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include "gsicp_internal.cuh"
#include "host_common.cuh"

namespace gsicp {

static thread_local char g_err[512] = "";
static thread_local uint64_t g_launches = 0;
extern thread_local int32_t *g_knn_debug;  // knn_cov.cu
extern thread_local long long *g_align_timeline;  // align.cu
extern thread_local long long g_align_timeline_cap;
extern thread_local int32_t *g_align_debug;
extern thread_local double *g_align_iter_rec;
extern thread_local int32_t *g_align_iter_corr;
extern thread_local int g_align_iter_cap;

// (launches captured into a conditional graph node's body are not counted: they run only when the
// device switches the node on — the hash tail of the image-window kNN, which a frame rarely needs)
void note_launch(int n) {
    if (!pdl_suspended()) g_launches += (uint64_t)n;
}

static thread_local int g_ktimer_on = 0;
static thread_local cudaEvent_t g_kt_ev[KT_COUNT][2] = {};
static thread_local bool g_kt_used[KT_COUNT] = {};

void ktimer_mark(int id, bool stop, cudaStream_t s) {
    if (!g_ktimer_on || id < 0 || id >= KT_COUNT) return;
    if (id >= KT_BP && g_ktimer_on < 2) return;  // stage spans only at level 2
    cudaEvent_t &ev = g_kt_ev[id][stop ? 1 : 0];
    if (!ev && cudaEventCreate(&ev) != cudaSuccess) {
        ev = nullptr;
        return;
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
    else
        cudaEventRecord(ev, s);
    if (stop) g_kt_used[id] = true;
}
void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// defined in the kernel translation units
size_t backproject_ws_bytes(int H, int W, int stride);
cudaError_t backproject_launch(const float *depth, int H, int W, int pitch, gsicp_intrinsics K, int stride,
                               float zmin, float zmax, float *pos_out, int32_t *d_n, void *ws, cudaStream_t s,
                               int rows_sampled, int32_t *map);
size_t covariances_ws_bytes(int cap, int levels);
cudaError_t covariances_launch(const float *pos, const int32_t *d_n, int cap, int k, int mode, float eps,
                               float cell0, int levels, float *cov_a, float *cov_b, int32_t *knn_idx, void *ws,
                               cudaStream_t s);
size_t covariances_image_ws_bytes(int cap, int levels, int H, int W, int stride);
cudaError_t covariances_image_launch(const float *pos, const int32_t *d_n, int cap, int H, int W, int stride,
                                     gsicp_intrinsics K, int k, int mode, float eps, float cell0, int levels,
                                     float *cov_a, float *cov_b, int32_t *knn_idx, const int32_t *lattice_map,
                                     void *ws, cudaStream_t s, void *window_done);
size_t target_ws_bytes(int M);
cudaError_t build_target_launch(const float *means, const float *quats, const float *scales, int scales_are_log,
                                int M, int mode, float eps, float cell, gsicp_target *out, void *ws,
                                cudaStream_t s);
cudaError_t build_target_cloud_launch(const gsicp_cloud &cl, int M, float cell, gsicp_target *out, void *ws,
                                      cudaStream_t s);
size_t voxel_ws_bytes(int cap);
cudaError_t voxel_launch(const float4 *pos, const int32_t *d_n, int cap, float voxel, float4 *out, int32_t *d_m,
                         void *ws, cudaStream_t s);
size_t export_ws_bytes(int cap);
cudaError_t export_launch(const float4 *pos, const float4 *cov_a, const float4 *cov_b, const int32_t *d_n, int cap,
                          const double *d_T, double p, double c, const int32_t *corr, float *means, float *quats,
                          float *scales, int32_t *d_m, void *ws, cudaStream_t s, const int32_t *d_base = nullptr);
size_t map_ws_bytes(int cap, int max_insert);
cudaError_t map_init_launch(const float *means, const float *quats, const float *scales, int scales_are_log, int M0,
                            int cap, int max_insert, int mode, float eps, float cell, gsicp_map *out, void *ws,
                            cudaStream_t s);
cudaError_t map_insert_launch(const gsicp_map &mp, const gsicp_cloud &kf, const double *d_T, const int32_t *corr,
                              double p, double c, const int32_t *d_flag, cudaStream_t s);
cudaError_t keyframe_launch(const gsicp_align_stats *d_stats, int32_t *d_state, float min_fitness, int max_gap,
                            cudaStream_t s);
size_t align_ws_bytes(int cap);
int align_batch_max();
cudaError_t align_batch_launch(const gsicp_cloud *srcs, int B, const gsicp_target &tgt, double *d_T,
                               const gsicp_align_params &p, gsicp_align_stats *d_stats, int32_t *const *corr_out,
                               void *const *ws, cudaStream_t s);
double *align_ws_T(void *ws);
gsicp_align_stats *align_ws_stats(void *ws);
double *align_ws_lin(void *ws);
cudaError_t align_seed_launch(const gsicp_cloud &src, const gsicp_target &tgt, const double *d_T,
                              const gsicp_align_params &p, void *ws, cudaStream_t s);
cudaError_t align_launch(const gsicp_cloud &src, const gsicp_target &tgt, double *d_T_inout,
                         const gsicp_align_params &p, gsicp_align_stats *d_stats, int32_t *corr_out,
                         int linearize_only, float r_lin, void *ws, cudaStream_t s);

}  // namespace gsicp

using namespace gsicp;

#define BAD(...)                                  \
    do {                                          \
        set_error(__VA_ARGS__);                   \
        return GSICP_ERR_INVALID_ARGUMENT;        \
    } while (0)

static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }
static bool aligned256(const void *p) { return ((uintptr_t)p & 255u) == 0; }

static gsicp_status cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return GSICP_OK;
    if (g_err[0] == 0) set_error("%s: %s", what, cudaGetErrorString(e));
    return GSICP_ERR_CUDA;
}

static gsicp_status check_ws(void *ws, size_t have, size_t need) {
    if (!ws || !aligned256(ws)) BAD("workspace must be non-null and 256-byte aligned");
    if (have < need) {
        set_error("workspace too small: %zu < %zu bytes", have, need);
        return GSICP_ERR_WORKSPACE_TOO_SMALL;
    }
    return GSICP_OK;
}

static gsicp_status check_cloud(const gsicp_cloud *c, const char *name) {
    if (!c) BAD("%s: null cloud", name);
    if (c->cap < 1) BAD("%s: cap must be >= 1", name);
    if (!c->pos || !c->cov_a || !c->cov_b || !c->d_n) BAD("%s: null array", name);
    if (!aligned16(c->pos) || !aligned16(c->cov_a) || !aligned16(c->cov_b)) BAD("%s: arrays must be 16-byte aligned", name);
    return GSICP_OK;
}

static gsicp_status check_target(const gsicp_target *t) {
    if (!t || !t->pos || !t->cov_a || !t->cov_b || !t->table || !t->bbox) BAD("target: not built");
    if (!(t->cell > 0.f) || t->M < 1) BAD("target: invalid");
    return GSICP_OK;
}

extern "C" {

int32_t gsicp_abi_version(void) { return 1; }

const char *gsicp_status_string(gsicp_status s) {
    switch (s) {
        case GSICP_OK: return "ok";
        case GSICP_ERR_INVALID_ARGUMENT: return "invalid argument";
        case GSICP_ERR_WORKSPACE_TOO_SMALL: return "workspace too small";
        case GSICP_ERR_CUDA: return "cuda error";
        case GSICP_ERR_DEGENERATE_FRAME: return "degenerate frame (no valid points)";
        case GSICP_ERR_TRACKING_LOST: return "tracking lost (too few correspondences)";
        case GSICP_WARN_MAX_ITERS: return "max iterations reached";
        case GSICP_WARN_LOW_SUPPORT: return "low support (fewer than k points)";
    }
    return "unknown status";
}

const char *gsicp_last_error(void) { return g_err; }
void gsicp_debug_knn_counters(int32_t *d_out) { gsicp::g_knn_debug = d_out; }
void gsicp_debug_align_counters(int32_t *d_out) { gsicp::g_align_debug = d_out; }
void gsicp_debug_align_iterations(double *d_rec, int32_t *d_corr, int32_t max_iters) {
    gsicp::g_align_iter_rec = max_iters > 0 ? d_rec : nullptr;
    gsicp::g_align_iter_corr = max_iters > 0 ? d_corr : nullptr;
    gsicp::g_align_iter_cap = d_rec && max_iters > 0 ? max_iters : 0;
}

// ---------------------------------------------------------------------------------------------
// Sequence tracking helpers: constant-velocity initial pose and the pose history.
namespace gsicp {
namespace {
// T_out = T1 (T0^-1 T1): the last relative motion applied once more (rigid 4x4, row-major)
__global__ void k_pose_predict(const double *__restrict__ hist, double *__restrict__ T_out) {
    const double *A = hist, *B = hist + 16;  // T_{t-2}, T_{t-1}
    double Ai[12];  // inverse of A: [R^T | -R^T t]
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) Ai[4 * r + c] = A[4 * c + r];
        Ai[4 * r + 3] = -(A[r] * A[3] + A[4 + r] * A[7] + A[8 + r] * A[11]);
    }
    double D[12];  // A^-1 B
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 4; ++c)
            D[4 * r + c] = Ai[4 * r] * B[c] + Ai[4 * r + 1] * B[4 + c] + Ai[4 * r + 2] * B[8 + c] + (c == 3 ? Ai[4 * r + 3] : 0.0);
    double P[12];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 4; ++c)
            P[4 * r + c] = B[4 * r] * D[c] + B[4 * r + 1] * D[4 + c] + B[4 * r + 2] * D[8 + c] + (c == 3 ? B[4 * r + 3] : 0.0);
    // re-orthonormalise the rotation (Gram-Schmidt on the rows): the poses carry rounding-level
    // departures from SO(3), which the transpose-inverse above would compound from frame to frame
    double r0[3] = {P[0], P[1], P[2]}, r1[3] = {P[4], P[5], P[6]};
    const double n0 = 1.0 / sqrt(r0[0] * r0[0] + r0[1] * r0[1] + r0[2] * r0[2]);
    for (int k = 0; k < 3; ++k) r0[k] *= n0;
    const double d01 = r0[0] * r1[0] + r0[1] * r1[1] + r0[2] * r1[2];
    for (int k = 0; k < 3; ++k) r1[k] -= d01 * r0[k];
    const double n1 = 1.0 / sqrt(r1[0] * r1[0] + r1[1] * r1[1] + r1[2] * r1[2]);
    for (int k = 0; k < 3; ++k) r1[k] *= n1;
    const double r2[3] = {r0[1] * r1[2] - r0[2] * r1[1], r0[2] * r1[0] - r0[0] * r1[2], r0[0] * r1[1] - r0[1] * r1[0]};
    for (int k = 0; k < 3; ++k) {
        T_out[k] = r0[k];
        T_out[4 + k] = r1[k];
        T_out[8 + k] = r2[k];
    }
    T_out[3] = P[3]; T_out[7] = P[7]; T_out[11] = P[11];
    T_out[12] = 0.0; T_out[13] = 0.0; T_out[14] = 0.0; T_out[15] = 1.0;
}
// history <- (T_{t-1}, T_t); the trajectory (if any) records T_t at its running counter
__global__ void k_pose_push(double *__restrict__ hist, const double *__restrict__ T, double *__restrict__ traj,
                            int32_t *__restrict__ counter, int32_t cap) {
    const int k = threadIdx.x;
    if (k < 16) {
        const double t = T[k];
        hist[k] = hist[16 + k];
        hist[16 + k] = t;
        if (traj && counter) {
            const int32_t c = *counter;
            if (c < cap) traj[(size_t)c * 16 + k] = t;
        }
    }
    __syncthreads();
    if (k == 0 && counter) *counter += 1;
}
}  // namespace
}  // namespace gsicp

gsicp_status gsicp_pose_predict(const double *d_hist, double *d_T_out, void *stream) {
    g_err[0] = 0;
    if (!d_hist || !d_T_out) BAD("pose_predict: null pointer");
    gsicp::k_pose_predict<<<1, 1, 0, (cudaStream_t)stream>>>(d_hist, d_T_out);
    gsicp::note_launch();
    return cuda_status(cudaGetLastError(), "pose_predict");
}

gsicp_status gsicp_pose_push(double *d_hist, const double *d_T, double *d_traj, int32_t *d_counter, int32_t traj_cap,
                             void *stream) {
    g_err[0] = 0;
    if (!d_hist || !d_T) BAD("pose_push: null pointer");
    if ((d_traj == nullptr) != (d_counter == nullptr)) BAD("pose_push: trajectory and counter go together");
    gsicp::k_pose_push<<<1, 32, 0, (cudaStream_t)stream>>>(d_hist, d_T, d_traj, d_counter, traj_cap);
    gsicp::note_launch();
    return cuda_status(cudaGetLastError(), "pose_push");
}

size_t gsicp_voxel_downsample_workspace_size(int32_t cap) { return cap < 1 ? 0 : voxel_ws_bytes(cap); }

gsicp_status gsicp_voxel_downsample(const float *pos, const int32_t *d_n, int32_t cap, float voxel, float *pos_out,
                                    int32_t *d_m_out, void *ws, size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    if (!pos || !d_n || !pos_out || !d_m_out) BAD("voxel_downsample: null pointer");
    if (!aligned16(pos) || !aligned16(pos_out)) BAD("voxel_downsample: pos and pos_out must be 16-byte aligned");
    if (cap < 1) BAD("voxel_downsample: cap must be >= 1");
    if (!(voxel > 0.f) || !isfinite(voxel)) BAD("voxel_downsample: voxel must be > 0");
    gsicp_status st = check_ws(ws, ws_bytes, voxel_ws_bytes(cap));
    if (st != GSICP_OK) return st;
    return cuda_status(voxel_launch((const float4 *)pos, d_n, cap, voxel, (float4 *)pos_out, d_m_out, ws,
                                    (cudaStream_t)stream),
                       "voxel_downsample");
}

size_t gsicp_export_workspace_size(int32_t cap) { return cap < 1 ? 0 : export_ws_bytes(cap); }

gsicp_status gsicp_export_gaussians(const float *pos, const float *cov_a, const float *cov_b, const int32_t *d_n,
                                    int32_t cap, const double *d_T, double p, double c, const int32_t *corr,
                                    float *means_out, float *quats_out, float *scales_out, int32_t *d_m_out,
                                    void *ws, size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    if (!pos || !cov_a || !cov_b || !d_n || !means_out || !quats_out || !scales_out)
        BAD("export_gaussians: null pointer");
    if (!aligned16(pos) || !aligned16(cov_a) || !aligned16(cov_b) || !aligned16(quats_out))
        BAD("export_gaussians: pos, cov_a, cov_b and quats_out must be 16-byte aligned");
    if (cap < 1) BAD("export_gaussians: cap must be >= 1");
    if (!isfinite(p) || !isfinite(c) || !(c > 0.0)) BAD("export_gaussians: p must be finite and c > 0");
    if (corr) {
        if (!d_m_out) BAD("export_gaussians: a correspondence filter needs d_m_out");
        gsicp_status st = check_ws(ws, ws_bytes, export_ws_bytes(cap));
        if (st != GSICP_OK) return st;
    }
    return cuda_status(export_launch((const float4 *)pos, (const float4 *)cov_a, (const float4 *)cov_b, d_n, cap, d_T,
                                     p, c, corr, means_out, quats_out, scales_out, d_m_out, ws, (cudaStream_t)stream),
                       "export_gaussians");
}

gsicp_status gsicp_graph_instantiate(void *graph, void **exec_out) {
    g_err[0] = 0;
    if (!graph || !exec_out) BAD("graph_instantiate: null pointer");
    cudaGraphExec_t ex = nullptr;
    const cudaError_t e = cudaGraphInstantiateWithFlags(&ex, (cudaGraph_t)graph, cudaGraphInstantiateFlagUseNodePriority);
    *exec_out = ex;
    return cuda_status(e, "graph_instantiate");
}
gsicp_status gsicp_graph_launch(void *exec, void *stream) {
    g_err[0] = 0;
    if (!exec) BAD("graph_launch: null exec");
    return cuda_status(cudaGraphLaunch((cudaGraphExec_t)exec, (cudaStream_t)stream), "graph_launch");
}
gsicp_status gsicp_graph_destroy(void *exec) {
    g_err[0] = 0;
    if (!exec) return GSICP_OK;
    return cuda_status(cudaGraphExecDestroy((cudaGraphExec_t)exec), "graph_destroy");
}

void gsicp_debug_kernel_timer(int enable) { gsicp::g_ktimer_on = enable < 0 ? 0 : enable; }

int gsicp_debug_kernel_time(int kernel, float *ms) {
    using namespace gsicp;
    if (!ms || kernel < 0 || kernel >= KT_COUNT || !g_kt_used[kernel]) return 0;
    *ms = 0.f;
    return cudaEventElapsedTime(ms, g_kt_ev[kernel][0], g_kt_ev[kernel][1]) == cudaSuccess ? 1 : 0;
}
void gsicp_debug_align_timeline(int64_t *d_out, int64_t capacity) {
    gsicp::g_align_timeline = reinterpret_cast<long long *>(d_out);
    gsicp::g_align_timeline_cap = d_out ? capacity : 0;
}
uint64_t gsicp_kernel_launch_count(void) { return g_launches; }

size_t gsicp_backproject_workspace_size(int32_t H, int32_t W, int32_t stride) {
    if (H < 1 || W < 1 || stride < 1) return 0;
    return backproject_ws_bytes(H, W, stride);
}

static gsicp_status backproject_common(const float *depth_m, int32_t H, int32_t W, int32_t row_pitch_elems,
                                       gsicp_intrinsics K, int32_t stride, float z_min, float z_max, float *pos_out,
                                       int32_t cap, int32_t *d_n_out, void *ws, size_t ws_bytes, void *stream,
                                       int rows_sampled, int32_t *map) {
    g_err[0] = 0;
    if (!depth_m || !pos_out || !d_n_out) BAD("backproject: null pointer");
    if (H < 1 || W < 1 || stride < 1 || row_pitch_elems < W) BAD("backproject: bad image geometry");
    if (!(K.fx > 0.f) || !(K.fy > 0.f) || !isfinite(K.cx) || !isfinite(K.cy)) BAD("backproject: bad intrinsics");
    if (!(z_min <= z_max)) BAD("backproject: z_min > z_max");
    if (!aligned16(pos_out)) BAD("backproject: pos_out must be 16-byte aligned");
    const long long need = (long long)((H + stride - 1) / stride) * ((W + stride - 1) / stride);
    if (cap < need) BAD("backproject: cap %d < %lld sampled pixels", cap, need);
    gsicp_status st = check_ws(ws, ws_bytes, backproject_ws_bytes(H, W, stride));
    if (st != GSICP_OK) return st;
    return cuda_status(backproject_launch(depth_m, H, W, row_pitch_elems, K, stride, z_min, z_max, pos_out, d_n_out, ws,
                                          (cudaStream_t)stream, rows_sampled, map),
                       "backproject");
}

gsicp_status gsicp_backproject_downsample(const float *depth_m, int32_t H, int32_t W, int32_t row_pitch_elems,
                                          gsicp_intrinsics K, int32_t stride, float z_min, float z_max,
                                          float *pos_out, int32_t cap, int32_t *d_n_out, void *ws, size_t ws_bytes,
                                          void *stream) {
    return backproject_common(depth_m, H, W, row_pitch_elems, K, stride, z_min, z_max, pos_out, cap, d_n_out, ws,
                              ws_bytes, stream, 0, nullptr);
}

gsicp_status gsicp_backproject_lattice(const float *depth, int32_t rows_sampled, int32_t H, int32_t W,
                                       int32_t row_pitch_elems, gsicp_intrinsics K, int32_t stride, float z_min,
                                       float z_max, float *pos_out, int32_t cap, int32_t *d_n_out,
                                       int32_t *lattice_map_out, void *ws, size_t ws_bytes, void *stream) {
    if (rows_sampled != 0 && rows_sampled != 1) {
        g_err[0] = 0;
        BAD("backproject_lattice: rows_sampled must be 0 or 1");
    }
    return backproject_common(depth, H, W, row_pitch_elems, K, stride, z_min, z_max, pos_out, cap, d_n_out, ws,
                              ws_bytes, stream, rows_sampled, lattice_map_out);
}

gsicp_status gsicp_backproject_sampled_rows(const float *depth_rows, int32_t H, int32_t W, int32_t row_pitch_elems,
                                            gsicp_intrinsics K, int32_t stride, float z_min, float z_max,
                                            float *pos_out, int32_t cap, int32_t *d_n_out, void *ws, size_t ws_bytes,
                                            void *stream) {
    return backproject_common(depth_rows, H, W, row_pitch_elems, K, stride, z_min, z_max, pos_out, cap, d_n_out, ws,
                              ws_bytes, stream, 1, nullptr);
}

gsicp_status gsicp_upload_sampled_rows(float *dst_rows, const float *src_host, int32_t H, int32_t W,
                                       int32_t src_pitch_elems, int32_t stride, void *stream) {
    g_err[0] = 0;
    if (!dst_rows || !src_host) BAD("upload_sampled_rows: null pointer");
    if (H < 1 || W < 1 || stride < 1 || src_pitch_elems < W) BAD("upload_sampled_rows: bad image geometry");
    const int rows = (H + stride - 1) / stride;
    return cuda_status(cudaMemcpy2DAsync(dst_rows, (size_t)W * sizeof(float), src_host,
                                         (size_t)stride * src_pitch_elems * sizeof(float), (size_t)W * sizeof(float),
                                         (size_t)rows, cudaMemcpyHostToDevice, (cudaStream_t)stream),
                       "upload_sampled_rows");
}

size_t gsicp_covariances_workspace_size(int32_t cap, int32_t levels) {
    if (cap < 1 || levels < 1 || levels > kMaxLevels) return 0;
    return covariances_ws_bytes(cap, levels);
}

gsicp_status gsicp_covariances(const float *pos, const int32_t *d_n, int32_t cap, int32_t k, gsicp_reg_mode mode,
                               float eps_var, float cell0, int32_t levels, float *cov_a, float *cov_b,
                               int32_t *knn_idx, void *ws, size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    if (!pos || !d_n || !cov_a || !cov_b) BAD("covariances: null pointer");
    if (!aligned16(pos) || !aligned16(cov_a) || !aligned16(cov_b)) BAD("covariances: arrays must be 16-byte aligned");
    if (cap < 1 || (uint32_t)cap > kMaxBandIndex) BAD("covariances: cap must be in [1, 2^27)");
    if (k < 1 || k > 32) BAD("covariances: k must be in [1, 32]");
    if (mode != GSICP_REG_NONE && mode != GSICP_REG_PLANE && mode != GSICP_REG_ELLIPSE) BAD("covariances: bad mode");
    if (!(eps_var > 0.f) || !(eps_var <= 1.f)) BAD("covariances: eps_var must be in (0, 1]");
    if (!isfinite(cell0)) BAD("covariances: cell0 must be finite (<= 0: automatic)");
    if (levels < 1 || levels > kMaxLevels) BAD("covariances: levels must be in [1, %d]", kMaxLevels);
    gsicp_status st = check_ws(ws, ws_bytes, covariances_ws_bytes(cap, levels));
    if (st != GSICP_OK) return st;
    return cuda_status(covariances_launch(pos, d_n, cap, k, (int)mode, eps_var, cell0, levels, cov_a, cov_b, knn_idx, ws,
                                          (cudaStream_t)stream),
                       "covariances");
}

size_t gsicp_covariances_image_workspace_size(int32_t cap, int32_t levels, int32_t H, int32_t W, int32_t stride) {
    if (cap < 1 || levels < 1 || levels > kMaxLevels || H < 1 || W < 1 || stride < 1) return 0;
    return covariances_image_ws_bytes(cap, levels, H, W, stride);
}

gsicp_status gsicp_covariances_image(const float *pos, const int32_t *d_n, int32_t cap, int32_t H, int32_t W,
                                     int32_t stride, gsicp_intrinsics K, int32_t k, gsicp_reg_mode mode, float eps_var,
                                     float cell0, int32_t levels, float *cov_a, float *cov_b, int32_t *knn_idx,
                                     const int32_t *lattice_map, void *ws, size_t ws_bytes, void *stream,
                                     void *window_done_event) {
    g_err[0] = 0;
    if (!pos || !d_n || !cov_a || !cov_b) BAD("covariances_image: null pointer");
    if (!aligned16(pos) || !aligned16(cov_a) || !aligned16(cov_b)) BAD("covariances_image: arrays must be 16-byte aligned");
    if (cap < 1 || (uint32_t)cap > kMaxBandIndex) BAD("covariances_image: cap must be in [1, 2^27)");
    if (H < 1 || W < 1 || stride < 1) BAD("covariances_image: bad image geometry");
    if ((long long)H * W >= (1ll << 31)) BAD("covariances_image: image too large for 32-bit pixel ids");
    if (!(K.fx > 0.f) || !(K.fy > 0.f) || !isfinite(K.fx) || !isfinite(K.fy)) BAD("covariances_image: bad intrinsics");
    if (k < 1 || k > 32) BAD("covariances_image: k must be in [1, 32]");
    if (mode != GSICP_REG_NONE && mode != GSICP_REG_PLANE && mode != GSICP_REG_ELLIPSE) BAD("covariances_image: bad mode");
    if (!(eps_var > 0.f) || !(eps_var <= 1.f)) BAD("covariances_image: eps_var must be in (0, 1]");
    if (!(cell0 > 0.f) || !isfinite(cell0)) BAD("covariances_image: cell0 must be > 0");
    if (levels < 1 || levels > kMaxLevels) BAD("covariances_image: levels must be in [1, %d]", kMaxLevels);
    gsicp_status st = check_ws(ws, ws_bytes, covariances_image_ws_bytes(cap, levels, H, W, stride));
    if (st != GSICP_OK) return st;
    return cuda_status(covariances_image_launch(pos, d_n, cap, H, W, stride, K, k, (int)mode, eps_var, cell0, levels,
                                                cov_a, cov_b, knn_idx, lattice_map, ws, (cudaStream_t)stream,
                                                window_done_event),
                       "covariances_image");
}

size_t gsicp_map_workspace_size(int32_t capacity, int32_t max_insert) {
    if (capacity < 1 || (uint32_t)capacity > kMaxBandIndex || max_insert < 1) return 0;
    return map_ws_bytes(capacity, max_insert);
}

gsicp_status gsicp_map_init(const float *means, const float *quats_wxyz, const float *scales, int32_t scales_are_log,
                            int32_t M0, int32_t capacity, int32_t max_insert, gsicp_reg_mode mode, float eps_var,
                            float cell, gsicp_map *out, void *ws, size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    if (!out || (M0 > 0 && (!means || !quats_wxyz || !scales))) BAD("map_init: null pointer");
    if (capacity < 1 || (uint32_t)capacity > kMaxBandIndex) BAD("map_init: capacity must be in [1, 2^27)");
    if (max_insert < 1) BAD("map_init: max_insert must be >= 1");
    if (M0 < 0 || M0 > capacity) BAD("map_init: M0 must be in [0, capacity]");
    if (mode != GSICP_REG_NONE && mode != GSICP_REG_PLANE && mode != GSICP_REG_ELLIPSE) BAD("map_init: bad mode");
    if (!(eps_var > 0.f) || !(eps_var <= 1.f)) BAD("map_init: eps_var must be in (0, 1]");
    if (!isfinite(cell)) BAD("map_init: cell must be finite");
    if (M0 == 0 && !(cell > 0.f)) BAD("map_init: an empty map needs an explicit cell > 0");
    gsicp_status st = check_ws(ws, ws_bytes, map_ws_bytes(capacity, max_insert));
    if (st != GSICP_OK) return st;
    return cuda_status(map_init_launch(means, quats_wxyz, scales, scales_are_log, M0, capacity, max_insert, (int)mode,
                                       eps_var, cell, out, ws, (cudaStream_t)stream),
                       "map_init");
}

gsicp_status gsicp_map_insert(const gsicp_map *map, const gsicp_cloud *kf, const double *d_T, const int32_t *corr,
                              double p, double c, const int32_t *d_flag, void *stream) {
    g_err[0] = 0;
    if (!map || !map->ws) BAD("map_insert: null map");
    gsicp_status st = check_cloud(kf, "map_insert");
    if (st != GSICP_OK) return st;
    if (kf->cap > map->max_insert) BAD("map_insert: keyframe cap %d > max_insert %d", kf->cap, map->max_insert);
    if (!isfinite(p) || !isfinite(c) || !(c > 0.0)) BAD("map_insert: p must be finite and c > 0");
    return cuda_status(map_insert_launch(*map, *kf, d_T, corr, p, c, d_flag, (cudaStream_t)stream), "map_insert");
}

gsicp_status gsicp_keyframe_decide(const gsicp_align_stats *d_stats, int32_t *d_state, float min_fitness,
                                   int32_t max_gap, void *stream) {
    g_err[0] = 0;
    if (!d_stats || !d_state) BAD("keyframe_decide: null pointer");
    if (max_gap < 1) BAD("keyframe_decide: max_gap must be >= 1");
    return cuda_status(keyframe_launch(d_stats, d_state, min_fitness, max_gap, (cudaStream_t)stream), "keyframe_decide");
}

size_t gsicp_build_target_workspace_size(int32_t M) {
    if (M < 1) return 0;
    return target_ws_bytes(M);
}

gsicp_status gsicp_build_target(const float *means, const float *quats_wxyz, const float *scales,
                                int32_t scales_are_log, int32_t M, gsicp_reg_mode mode, float eps_var, float cell,
                                gsicp_target *out, void *target_ws, size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    if (!means || !quats_wxyz || !scales || !out) BAD("build_target: null pointer");
    if (M < 1 || (uint32_t)M > kMaxBandIndex) BAD("build_target: M must be in [1, 2^27)");
    if (mode != GSICP_REG_NONE && mode != GSICP_REG_PLANE && mode != GSICP_REG_ELLIPSE) BAD("build_target: bad mode");
    if (!(eps_var > 0.f) || !(eps_var <= 1.f)) BAD("build_target: eps_var must be in (0, 1]");
    if (!isfinite(cell)) BAD("build_target: cell must be finite");
    gsicp_status st = check_ws(target_ws, ws_bytes, target_ws_bytes(M));
    if (st != GSICP_OK) return st;
    return cuda_status(build_target_launch(means, quats_wxyz, scales, scales_are_log, M, (int)mode, eps_var, cell, out,
                                           target_ws, (cudaStream_t)stream),
                       "build_target");
}

gsicp_status gsicp_build_target_cloud(const gsicp_cloud *cloud, int32_t M, float cell, gsicp_target *out,
                                      void *target_ws, size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    gsicp_status st = check_cloud(cloud, "build_target_cloud");
    if (st != GSICP_OK) return st;
    if (!out) BAD("build_target_cloud: null out");
    if (M < 1 || M > cloud->cap || (uint32_t)M > kMaxBandIndex) BAD("build_target_cloud: M must be in [1, min(cap, 2^27))");
    if (!isfinite(cell)) BAD("build_target_cloud: cell must be finite (<= 0: automatic)");
    st = check_ws(target_ws, ws_bytes, target_ws_bytes(M));
    if (st != GSICP_OK) return st;
    return cuda_status(build_target_cloud_launch(*cloud, M, cell, out, target_ws, (cudaStream_t)stream),
                       "build_target_cloud");
}

size_t gsicp_align_workspace_size(int32_t src_cap) {
    if (src_cap < 1) return 0;
    return align_ws_bytes(src_cap);
}

static gsicp_status check_params(const gsicp_align_params *p) {
    if (!p) BAD("align: null params");
    if (p->max_iters < 1 || p->max_iters > 10000) BAD("align: max_iters must be in [1, 10000]");
    if (!(p->max_corr_dist > 0.f)) BAD("align: max_corr_dist must be > 0 (INFINITY allowed)");
    if (!(p->eps_rot >= 0.0) || !(p->eps_trans >= 0.0)) BAD("align: eps must be >= 0");
    if (p->min_pairs < 0) BAD("align: min_pairs must be >= 0");
    if (p->solver != 0 && p->solver != 1) BAD("align: solver must be 0 (GN) or 1 (LM)");
    if (p->solver == 1 && !(p->lm_lambda0 > 0.0 && p->lm_lambda0 < 1e30)) BAD("align: lm_lambda0 must be > 0");
    return GSICP_OK;
}

gsicp_status gsicp_align_async(const gsicp_cloud *src, const gsicp_target *tgt, double *d_T_inout,
                               const gsicp_align_params *prm, gsicp_align_stats *d_stats, int32_t *corr_out,
                               void *ws, size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    gsicp_status st = check_cloud(src, "align src");
    if (st != GSICP_OK) return st;
    if ((st = check_target(tgt)) != GSICP_OK) return st;
    if ((st = check_params(prm)) != GSICP_OK) return st;
    if (!d_T_inout || !d_stats) BAD("align_async: null device pose / stats");
    if ((st = check_ws(ws, ws_bytes, align_ws_bytes(src->cap))) != GSICP_OK) return st;
    return cuda_status(align_launch(*src, *tgt, d_T_inout, *prm, d_stats, corr_out, 0, 0.f, ws, (cudaStream_t)stream),
                       "align");
}

int32_t gsicp_align_batch_max(void) { return align_batch_max(); }

gsicp_status gsicp_align_batch_async(const gsicp_cloud *srcs, int32_t B, const gsicp_target *tgt, double *d_T,
                                     const gsicp_align_params *prm, gsicp_align_stats *d_stats,
                                     int32_t *const *corr_out, void *const *ws, size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    if (!srcs || !ws || !d_T || !d_stats) BAD("align_batch: null pointer");
    if (B < 1 || B > align_batch_max()) BAD("align_batch: B must be in [1, %d]", align_batch_max());
    gsicp_status st = check_target(tgt);
    if (st != GSICP_OK) return st;
    if ((st = check_params(prm)) != GSICP_OK) return st;
    for (int f = 0; f < B; ++f) {
        if ((st = check_cloud(srcs + f, "align_batch src")) != GSICP_OK) return st;
        if ((st = check_ws(ws[f], ws_bytes, align_ws_bytes(srcs[f].cap))) != GSICP_OK) return st;
        for (int g2 = 0; g2 < f; ++g2)
            if (ws[g2] == ws[f]) BAD("align_batch: every frame needs its own workspace");
    }
    return cuda_status(align_batch_launch(srcs, B, *tgt, d_T, *prm, d_stats, corr_out, ws, (cudaStream_t)stream),
                       "align_batch");
}


gsicp_status gsicp_align_seed(const gsicp_cloud *src, const gsicp_target *tgt, const double *d_T,
                              const gsicp_align_params *prm, void *ws, size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    gsicp_status st = check_cloud(src, "align_seed src");
    if (st != GSICP_OK) return st;
    if ((st = check_target(tgt)) != GSICP_OK) return st;
    if ((st = check_params(prm)) != GSICP_OK) return st;
    if (!d_T) BAD("align_seed: null device pose");
    if ((st = check_ws(ws, ws_bytes, align_ws_bytes(src->cap))) != GSICP_OK) return st;
    return cuda_status(align_seed_launch(*src, *tgt, d_T, *prm, ws, (cudaStream_t)stream), "align_seed");
}

gsicp_status gsicp_align(const gsicp_cloud *src, const gsicp_target *tgt, const double *init_T,
                         const gsicp_align_params *prm, double *out_T, gsicp_align_stats *out_stats, void *ws,
                         size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    gsicp_status st = check_cloud(src, "align src");
    if (st != GSICP_OK) return st;
    if ((st = check_target(tgt)) != GSICP_OK) return st;
    if ((st = check_params(prm)) != GSICP_OK) return st;
    if (!init_T || !out_T || !out_stats) BAD("align: null host pointer");
    if ((st = check_ws(ws, ws_bytes, align_ws_bytes(src->cap))) != GSICP_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    double *dT = align_ws_T(ws);
    gsicp_align_stats *dS = align_ws_stats(ws);
    cudaError_t e = cudaMemcpyAsync(dT, init_T, 16 * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "align H2D");
    e = align_launch(*src, *tgt, dT, *prm, dS, nullptr, 0, 0.f, ws, s);
    if (e != cudaSuccess) return cuda_status(e, "align");
    e = cudaMemcpyAsync(out_T, dT, 16 * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_stats, dS, sizeof(gsicp_align_stats), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "align D2H");
    return (gsicp_status)out_stats->status;
}

gsicp_status gsicp_linearize(const gsicp_cloud *src, const gsicp_target *tgt, const double *T, float max_corr_dist,
                             double *H, double *b, double *cost, int32_t *n_inliers, int32_t *corr_opt, void *ws,
                             size_t ws_bytes, void *stream) {
    g_err[0] = 0;
    gsicp_status st = check_cloud(src, "linearize src");
    if (st != GSICP_OK) return st;
    if ((st = check_target(tgt)) != GSICP_OK) return st;
    if (!T || !H || !b || !cost || !n_inliers) BAD("linearize: null host pointer");
    if (!(max_corr_dist > 0.f)) BAD("linearize: max_corr_dist must be > 0");
    if ((st = check_ws(ws, ws_bytes, align_ws_bytes(src->cap))) != GSICP_OK) return st;
    cudaStream_t s = (cudaStream_t)stream;
    double *dT = align_ws_T(ws);
    gsicp_align_stats *dS = align_ws_stats(ws);
    double *dL = align_ws_lin(ws);
    gsicp_align_params p = {1, max_corr_dist, 0.0, 0.0, 0};
    cudaError_t e = cudaMemcpyAsync(dT, T, 16 * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "linearize H2D");
    e = align_launch(*src, *tgt, dT, p, dS, corr_opt, 1, max_corr_dist, ws, s);
    if (e != cudaSuccess) return cuda_status(e, "linearize");
    double lin[44];
    e = cudaMemcpyAsync(lin, dL, sizeof(lin), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_status(e, "linearize D2H");
    memcpy(H, lin, 36 * sizeof(double));
    memcpy(b, lin + 36, 6 * sizeof(double));
    *cost = lin[42];
    *n_inliers = (int32_t)lin[43];
    return GSICP_OK;
}

}  // extern "C"
