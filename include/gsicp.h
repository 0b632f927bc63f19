/*
 * gsicp.h — C ABI of the B200-native G-ICP tracking hot path of GS-ICP SLAM
 * (arXiv 2403.12550).  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n,
 * Rn = reading n in DESIGN.md §3.  Library: paper_2403_12550_b200/libgsicp.so.
 *
 * Conventions (all entry points):
 *  - Array pointers marked [dev] are CUDA device pointers OWNED BY THE CALLER; the
 *    library never allocates device memory.  Each call takes a caller workspace sized by
 *    the matching *_workspace_size() query (256-byte aligned base required).
 *  - `stream` is a cudaStream_t passed as void*.  All work is stream-ordered on it; calls are
 *    reentrant, so independent calls on different streams / devices may run concurrently (S:84,
 *    S:163).  gsicp_align and gsicp_linearize synchronise `stream` (they return host results),
 *    and so do the automatic cell sizes (cell <= 0) of gsicp_covariances / gsicp_build_target*.
 *  - State: the library keeps per-device caches of device properties and kernel occupancies
 *    (filled once per device under std::call_once, immutable after) and thread-local state only
 *    (error string, launch counter, diagnostic hooks, a per-thread capture stream for
 *    conditional graph nodes).  It reads no environment variables.
 *  - Keys (DESIGN R1): every nearest-neighbour decision follows the binary64 K2
 *    order (key = (dx*dx + dy*dy) + dz*dz with dx = (double)b.x - q.x, ties by lower index); the
 *    kernels screen in binary32 and resolve the candidates near the k-th / best key in binary64.
 *  - Host-side argument errors return GSICP_ERR_INVALID_ARGUMENT before anything is launched.
 *    CUDA launch errors return GSICP_ERR_CUDA (detail in gsicp_last_error()).
 *  - Point layout (SoA, binary32, 16-byte aligned float4 records):
 *      pos[i]   = (x, y, z, w)              metres; w = int32 payload bits
 *      cov_a[i] = (c00, c01, c02, c11)      regularised covariance, m^2 (or unitless after
 *      cov_b[i] = (c12, c22, lam_mid, flags)  ELLIPSE/PLANE regularisation); flags int32 bits
 *  - Counts that kernels produce live on the device (int32 *d_n) so a whole frame can be
 *    captured in one CUDA graph without host round trips.
 */
#ifndef GSICP_H
#define GSICP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library is built with -fvisibility=hidden */
#endif

typedef enum {
    GSICP_OK = 0,
    GSICP_ERR_INVALID_ARGUMENT = 1,
    GSICP_ERR_WORKSPACE_TOO_SMALL = 2,
    GSICP_ERR_CUDA = 3,
    GSICP_ERR_DEGENERATE_FRAME = 4, /* 0 valid points                                   */
    GSICP_ERR_TRACKING_LOST = 5,    /* inliers < min_pairs; out_T = last valid pose     */
    GSICP_WARN_MAX_ITERS = 6,       /* not converged within max_iters; out_T = last iterate     */
    GSICP_WARN_LOW_SUPPORT = 7      /* some cloud had fewer than k points                */
} gsicp_status;

typedef enum { GSICP_REG_NONE = 0, GSICP_REG_PLANE = 1, GSICP_REG_ELLIPSE = 2 } gsicp_reg_mode;

/* per-point flags stored in cov_b.w */
#define GSICP_FLAG_LOW_SUPPORT 1u /* fewer than k points in the cloud                     */
#define GSICP_FLAG_DEGENERATE 2u  /* lam_2 <= 1e-12 m^2, or lam_1 <= 1e-12 (PLANE/ELLIPSE), R8 */

typedef struct { float fx, fy, cx, cy; } gsicp_intrinsics;

/* A Gaussian cloud G = {X, C} in device memory. */
typedef struct {
    const float *pos;   /* [dev] float4[cap]                                  */
    const float *cov_a; /* [dev] float4[cap]                                  */
    const float *cov_b; /* [dev] float4[cap]                                  */
    const int32_t *d_n; /* [dev] number of valid points n <= cap              */
    int32_t cap;
} gsicp_cloud;

/* Target Gaussians G^t: a spatially hashed copy of a cloud, built by
 * gsicp_build_target / gsicp_build_target_cloud.  Every pointer is a view into the caller's
 * target workspace and stays valid (and must stay unmodified) while that buffer lives.
 * Treat the fields as opaque. */
typedef struct {
    const float *pos;     /* [dev] float4[M], cell order, w = original index bits */
    const float *cov_a;   /* [dev] float4[M], cell order                          */
    const float *cov_b;   /* [dev] float4[M], cell order                          */
    const void *table;    /* [dev] open-addressing cell table                     */
    const int32_t *bbox;  /* [dev] int32[6] ordered-int float bbox of the means   */
    const void *dense;    /* [dev] dense (start, count) cell array over the bbox, */
    const int32_t *dense_hdr; /* [dev] {in_use, lo xyz, dims xyz}: used when it fits */
    const int32_t *nbr;   /* [dev] int32[M][16] exact 16-NN slots of each slot (kNN graph) */
    const float *nbr_key; /* [dev] float[M] key of the 16th neighbour                     */
    uint32_t table_mask;  /* table slots - 1                                      */
    float cell;           /* cell edge h (m)                                      */
    int32_t M;
} gsicp_target;

typedef struct {
    int32_t max_iters;     /* GN iterations cap, default 30                          */
    float max_corr_dist;   /* r (m): pair valid iff key < r*r (R15); INFINITY = no gate      */
    double eps_rot;        /* converged iff |omega| < eps_rot and |v| < eps_trans     */
    double eps_trans;
    int32_t min_pairs;     /* fewer inliers -> TRACKING_LOST, default 50       */
    int32_t solver;        /* 0 = Gauss-Newton (default); 1 = Levenberg-Marquardt (R30): a trial
                              pose is kept iff its Eq. 1 cost is below the last kept one, step
                              (H + lambda diag H) delta = -b, lambda / 10 on accept, x 10 on reject;
                              at the cap the best kept pose is returned                */
    double lm_lambda0;     /* initial lambda (solver 1), > 0                                  */
} gsicp_align_params;

typedef struct {
    double fitness;        /* n_inliers / N_s of the final linearisation (R19)   */
    double mean_cost;      /* cost / n_inliers, cost = sum d^T M d (Eq. 1)                   */
    int32_t n_inliers;
    int32_t iters;         /* GN updates applied                                             */
    int32_t converged;
    int32_t status;        /* gsicp_status of the loop                                       */
} gsicp_align_stats;

/* ---------------------------------------------------------------------------------------
 * A1  Back-projection + uniform stride downsampling (Fig. 2 "downsampling and
 * reprojecting the current depth image"; pinhole S:46).  For v = 0, s, 2s, ... < H and
 * u = 0, s, ... < W, keep pixel (u, v) iff z = depth[v*row_pitch + u] is finite and
 * z_min <= z <= z_max; emit pos = (x, y, z, v*W+u) with x = (float)(((double)u - cx) * z / fx)
 * evaluated in binary64 (R13, R14).  Output is compacted in row-major pixel order (stable)
 * into pos_out[0 .. n) and n is written to *d_n_out.
 *  depth_m  [dev] binary32 metres, H rows of row_pitch_elems floats
 *  pos_out  [dev] float4[cap]; cap >= ceil(H/s)*ceil(W/s) is required
 *  Errors: INVALID_ARGUMENT (H, W, s < 1, pitch < W, cap too small, z_min > z_max, bad intrinsics).
 *  A frame with 0 valid points is not an error here; *d_n_out = 0 and gsicp_align reports
 *  GSICP_ERR_DEGENERATE_FRAME. */
size_t gsicp_backproject_workspace_size(int32_t H, int32_t W, int32_t stride);
gsicp_status gsicp_backproject_downsample(const float *depth_m, int32_t H, int32_t W, int32_t row_pitch_elems,
                                          gsicp_intrinsics K, int32_t stride, float z_min, float z_max,
                                          float *pos_out, int32_t cap, int32_t *d_n_out, void *ws, size_t ws_bytes,
                                          void *stream);

/* Same output (bit-identical) from only the rows A1 reads: depth_rows holds ceil(H/stride)
 * rows of row_pitch_elems floats, row r being image row r*stride — what a caller uploads when
 * the frame arrives in host memory (1/stride of the bytes).  Errors as above. */
gsicp_status gsicp_backproject_sampled_rows(const float *depth_rows, int32_t H, int32_t W, int32_t row_pitch_elems,
                                            gsicp_intrinsics K, int32_t stride, float z_min, float z_max,
                                            float *pos_out, int32_t cap, int32_t *d_n_out, void *ws, size_t ws_bytes,
                                            void *stream);
/* A1 that also writes the lattice map lattice_map_out [dev] int32[ceil(H/s)*ceil(W/s)]: the output
 * index of each sampled pixel (row-major lattice), -1 where the pixel is invalid — the index the
 * image-window kNN uses (gsicp_covariances_image), built here for free.  rows_sampled = 0: depth is
 * the full image (as gsicp_backproject_downsample); 1: only the sampled rows (as
 * gsicp_backproject_sampled_rows).  Errors as above. */
gsicp_status gsicp_backproject_lattice(const float *depth, int32_t rows_sampled, int32_t H, int32_t W,
                                       int32_t row_pitch_elems, gsicp_intrinsics K, int32_t stride, float z_min,
                                       float z_max, float *pos_out, int32_t cap, int32_t *d_n_out,
                                       int32_t *lattice_map_out, void *ws, size_t ws_bytes, void *stream);

/* Host -> device staging for it: copies rows 0, stride, 2*stride, ... of a host depth image
 * (src_pitch_elems floats per row; pinned memory for an asynchronous copy) into dst_rows
 * [dev] (ceil(H/stride) rows of W floats), stream-ordered.  Errors: INVALID_ARGUMENT, CUDA. */
gsicp_status gsicp_upload_sampled_rows(float *dst_rows, const float *src_host, int32_t H, int32_t W,
                                       int32_t src_pitch_elems, int32_t stride, void *stream);

/* ---------------------------------------------------------------------------------------
 * A2-A4  Per-point covariance of the exact k nearest neighbours ("computing covariance
 * matrix of k-nearest neighbors of x"; self included, ties by lower index),
 * normalised by k, followed by regularisation (Eq. 3-4; R6-R8):
 *   NONE    sum_i max(lam_i, 1e-6) v_i v_i^T
 *   PLANE   v2 v2^T + v1 v1^T + eps_var v0 v0^T            (S = [1, 1, eps])
 *   ELLIPSE sum_i max(lam_i / lam_1, eps_var) v_i v_i^T     (Lambda' = Lambda/median(S), Eq. 4)
 * The neighbour order is the binary64 K2 key (R1) then index.  A device spatial hash with
 * `levels` cell sizes cell0 * 2^l is built in the workspace; every query picks the finest level
 * whose own cell holds >= 3 points and runs a certified expanding-ring search (exact result).
 *  pos      [dev] float4[cap] (w ignored), d_n [dev] count; cap < 2^27
 *  k        1..32 neighbours.  If n < k all n points are used and GSICP_FLAG_LOW_SUPPORT set.
 *  cell0    finest cell edge (m); <= 0: automatic (2 x the estimated point spacing for several
 *           levels, 3 x for one; estimated on the device from a 32^3 occupancy grid; blocking);
 *           levels 1..8.  (Performance knobs only: results are exact at any cell size.)
 *  cov_a, cov_b [dev] float4[cap] outputs in input order (cov_b.z = raw lam_1, cov_b.w = flags)
 *  knn_idx  [dev] nullable int32[cap*k]: neighbours sorted by (K2 key, index), -1 padded
 *  Errors: INVALID_ARGUMENT. */
size_t gsicp_covariances_workspace_size(int32_t cap, int32_t levels);
gsicp_status gsicp_covariances(const float *pos, const int32_t *d_n, int32_t cap, int32_t k, gsicp_reg_mode mode,
                               float eps_var, float cell0, int32_t levels, float *cov_a, float *cov_b,
                               int32_t *knn_idx, void *ws, size_t ws_bytes, void *stream);

/* Same result as gsicp_covariances (bit-identical neighbour lists and covariances), for a
 * depth-frame cloud: pos/d_n exactly as written by gsicp_backproject_downsample with the same
 * (H, W, stride) and fx, fy of K (pos.w = pixel id v*W + u).  Candidates come from the
 * (2M+1)^2 lattice-pixel window around each query's pixel (M = 5), exact whenever the k-th
 * radius rho satisfies the projection bound f rho (z + |x|) / (z (z - rho)) < (M+1) s in both
 * image axes (every point within rho then lies in the window); the remaining queries are
 * finished by the hash search of gsicp_covariances (cell0 > 0, levels as there).  A cloud that is
 * not a depth-frame cloud (a pixel id off the lattice, two points on one pixel) is detected on
 * the device and handled entirely by the hash search, so the result is exact for any input.
 *  lattice_map [dev] nullable: the map gsicp_backproject_lattice wrote for exactly these points
 *  (then it is used as is, not rebuilt or validated); NULL: built and validated here.
 *  window_done_event nullable cudaEvent_t: recorded on `stream` right after the window kernel
 *  (before the latency-bound wide-window / brute-force stages), so that independent work on
 *  another stream can start there instead of competing with the window kernel for the SMs.
 *  Errors: INVALID_ARGUMENT. */
size_t gsicp_covariances_image_workspace_size(int32_t cap, int32_t levels, int32_t H, int32_t W, int32_t stride);
gsicp_status gsicp_covariances_image(const float *pos, const int32_t *d_n, int32_t cap, int32_t H, int32_t W,
                                     int32_t stride, gsicp_intrinsics K, int32_t k, gsicp_reg_mode mode,
                                     float eps_var, float cell0, int32_t levels, float *cov_a, float *cov_b,
                                     int32_t *knn_idx, const int32_t *lattice_map, void *ws, size_t ws_bytes,
                                     void *stream, void *window_done_event);

/* ---------------------------------------------------------------------------------------
 * A5  Map Gaussians -> G-ICP targets (the map's Gaussians are reused as
 * targets with no covariance recomputation; P:189-191 C = R Lambda^2 R^T).  Quaternion wxyz,
 * normalised before use; scales linear, or log if scales_are_log (R22); the regularised
 * covariance is formed in closed form from (R, s) (no eigensolve), then the means are hashed
 * with cell edge `cell` (<= 0: 3 x mean middle scale; a performance knob only — results are exact).
 *  means [dev] float[M][3], quats_wxyz [dev] float[M][4], scales [dev] float[M][3]
 *  target_ws: caller buffer holding the target for as long as it is used
 *  out: host struct filled with views into target_ws.  Synchronises `stream` only if cell <= 0. */
size_t gsicp_build_target_workspace_size(int32_t M);
gsicp_status gsicp_build_target(const float *means, const float *quats_wxyz, const float *scales,
                                int32_t scales_are_log, int32_t M, gsicp_reg_mode mode, float eps_var, float cell,
                                gsicp_target *out, void *target_ws, size_t ws_bytes, void *stream);

/* Same, from a cloud that already carries G-ICP covariances (e.g. gsicp_covariances output;
 * used for frame-to-frame tracking and the C1 configuration).  cell <= 0: automatic (3 x the
 * estimated point spacing; blocking).  M < 2^27. */
gsicp_status gsicp_build_target_cloud(const gsicp_cloud *cloud, int32_t M, float cell, gsicp_target *out,
                                      void *target_ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * A6-A9  G-ICP alignment: T* = argmin_T sum_i d_i^T (C^t_i + R C^s_i R^T)^{-1} d_i (Eq. 1,
 * P:103-131; R1-R3), d_i = x^t_j - T x^s_i with j the exact nearest target mean of T x^s_i
 * (P:95), by Gauss-Newton on a left twist (omega, v) with J = [[q]x, -I] (R16), 6x6 Cholesky
 * solve, Exp(omega) update, and a device-side convergence test, all inside ONE persistent
 * kernel (grid barrier per iteration) — no host round trip between iterations.
 *  init_T   host double[16] row-major, maps source (camera) coordinates to target (map).
 *  out_T    host double[16]; out_stats host.  Blocking: synchronises `stream`.
 *  Returns OK / WARN_MAX_ITERS / ERR_TRACKING_LOST / ERR_DEGENERATE_FRAME (n == 0). */
size_t gsicp_align_workspace_size(int32_t src_cap);
gsicp_status gsicp_align(const gsicp_cloud *src, const gsicp_target *tgt, const double *init_T,
                         const gsicp_align_params *prm, double *out_T, gsicp_align_stats *out_stats, void *ws,
                         size_t ws_bytes, void *stream);

/* Non-blocking / graph-capturable variant: the pose is read from and written to device memory
 * (d_T_inout [dev] double[16]) and the stats go to d_stats [dev]; nothing is synchronised.
 * corr_out [dev] nullable int32[cap]: final correspondence (original target index or -1). */
gsicp_status gsicp_align_async(const gsicp_cloud *src, const gsicp_target *tgt, double *d_T_inout,
                               const gsicp_align_params *prm, gsicp_align_stats *d_stats, int32_t *corr_out,
                               void *ws, size_t ws_bytes, void *stream);

/* N2 frame batch (the throughput mode): B independent frames aligned against the same target in
 * ONE cooperative launch — each frame runs the GN loop of gsicp_align_async on G/B co-resident
 * blocks with its own grid barrier, partials and convergence test, so the per-iteration latency
 * (barrier, reduction, solve) is paid once for the batch.  Per-frame results equal
 * gsicp_align_async's up to the summation grouping of the H/b partials (the block count differs).
 *  srcs    host array [B] of clouds;  B in [1, gsicp_align_batch_max()];
 *  d_T     [dev] double[B*16]: frame f's pose (row-major 4x4) at d_T + 16 f, read and updated;
 *  d_stats [dev] gsicp_align_stats[B];
 *  corr_out NULL or host array [B] of nullable [dev] int32[cap_f] (final correspondences);
 *  ws      host array [B] of distinct align workspaces (gsicp_align_workspace_size(cap_f) each,
 *          ws_bytes = the smallest of their sizes).  Seeds (gsicp_align_seed) computed on a
 *          frame's workspace at its current pose are used as in gsicp_align_async.
 *  Errors: INVALID_ARGUMENT, WORKSPACE_TOO_SMALL, CUDA.  Asynchronous, graph-capturable. */
int32_t gsicp_align_batch_max(void);
gsicp_status gsicp_align_batch_async(const gsicp_cloud *srcs, int32_t B, const gsicp_target *tgt, double *d_T,
                                     const gsicp_align_params *prm, gsicp_align_stats *d_stats,
                                     int32_t *const *corr_out, void *const *ws, size_t ws_bytes, void *stream);

/* Iteration-0 correspondences ahead of the GN loop (A6 at the initial pose, P:95 / R15): for
 * every source point the exact 1-NN of fl32(K3(T0, x_i)) among the target means, written into
 * the align workspace `ws`.  Reads only src->pos / src->d_n (not the covariances), the target and
 * the device pose d_T (double[16], T0), so it may run on a second stream concurrently with
 * gsicp_covariances of the same cloud; the caller orders it before the align call (event join).
 * The seeds are consumed by the NEXT gsicp_align / gsicp_align_async / gsicp_linearize issued
 * FROM THE SAME HOST THREAD on the same workspace with the same src->pos and tgt->pos, and only
 * if that call starts from exactly the
 * pose d_T held when the seed kernel ran (checked bitwise on the device); otherwise they are
 * ignored and the search runs as usual.  Results are identical with or without seeding.
 * Errors: as gsicp_align_async.  Asynchronous. */
gsicp_status gsicp_align_seed(const gsicp_cloud *src, const gsicp_target *tgt, const double *d_T,
                              const gsicp_align_params *prm, void *ws, size_t ws_bytes, void *stream);

/* TEST / DIAGNOSTIC export: one linearisation of Eq. 1 at pose T (host double[16]) without any
 * update — H (host double[36], row-major, twist order (omega, v)), b (host double[6]),
 * cost and inlier count; corr_opt [dev] nullable int32[cap] (original target index or -1).
 * Uses gsicp_align_workspace_size(src->cap).  Blocking. */
gsicp_status gsicp_linearize(const gsicp_cloud *src, const gsicp_target *tgt, const double *T, float max_corr_dist,
                             double *H, double *b, double *cost, int32_t *n_inliers, int32_t *corr_opt, void *ws,
                             size_t ws_bytes, void *stream);

/* DIAGNOSTIC: while set (non-NULL) on the calling thread, every gsicp_covariances call also writes
 * per query i: d_out[4*i + 0..3] = (grid level searched, cells probed, candidates scanned,
 * list insertions), int32, device memory of at least 4*cap entries.  NULL switches it off. */
void gsicp_debug_knn_counters(int32_t *d_out);

/* DIAGNOSTIC: while set, every align / linearize launch on the calling thread records device
 * globaltimer stamps (ns) into d_out (int64, device, `capacity` entries): [0] kernel start, then
 * per GN iteration `it` at [1 + it*(G+1) + b] the barrier arrival of block b and at
 * [1 + it*(G+1) + G] the barrier release seen by block 0 (G = grid size).  NULL switches it off. */
void gsicp_debug_align_timeline(int64_t *d_out, int64_t capacity);

/* DIAGNOSTIC: while set, align / linearize launches write per resident source point i
 * d_out[4*i + 0..3] = bitmasks over the GN iterations (bit it) of: search handed to the
 * warp-cooperative path, motion-bounded reuse, kNN-graph certificate; then the iteration count,
 * summed over the GN iterations (int32, device, >= 4*cap entries).  NULL switches it off. */
void gsicp_debug_align_counters(int32_t *d_out);

/* DIAGNOSTIC (per-iteration parity, SURVEY §8(c).5 "per-iteration H/b"): while set (d_rec
 * non-NULL, max_iters > 0) on the calling thread, every align launch (and frame 0 of a batch)
 * records, for each Gauss-Newton iteration it < max_iters that runs, d_rec[48*it + 0..11] = the
 * pose T_it the iteration linearised at (row-major 3x4, binary64) and d_rec[48*it + 12..40] = its
 * reduced Eq. 1 terms (21 upper-triangular H entries row by row, b[6], cost, inlier count);
 * d_corr (nullable, int32[max_iters * src cap]) gets d_corr[it*cap + i] = point i's
 * correspondence in that iteration (original target index, -1 none).  Device memory of the caller;
 * the pointers are baked into CUDA graphs captured while set.  NULL switches it off. */
void gsicp_debug_align_iterations(double *d_rec, int32_t *d_corr, int32_t max_iters);

/* DIAGNOSTIC: kernel timer.  While enabled (1: spans 0-2 below; 2: all spans) on the calling
 * thread, the launches of the hot kernels record a CUDA event pair around themselves on their stream (also inside a
 * stream capture: the events then record at every graph replay).  gsicp_debug_kernel_time
 * returns 1 and the elapsed ms of the LAST recorded span `kernel`: 0 = the kNN search kernel
 * (k_knn_search of gsicp_covariances; the 11x11 window kernel of gsicp_covariances_image),
 * 1 = k_align of the align calls, 2 = the two seed kernels of gsicp_align_seed, 3 = A1,
 * 4 = gsicp_covariances_image on the caller's stream (all of it), 5 = its wide-window + brute
 * force stage, 6 = its hash tail (join + search + epilogue); the caller synchronises first.
 * Returns 0 if none was recorded. */
void gsicp_debug_kernel_timer(int enable);
int gsicp_debug_kernel_time(int kernel, float *ms);

/* ---------------------------------------------------------------------------------------
 * Sequence tracking (C5): the initial pose of frame t is the constant-velocity extrapolation
 * T_{t-1} (T_{t-2}^-1 T_{t-1}) (binary64; the rotation re-orthonormalised), computed on
 * the device so that a whole sequence runs without host round trips.
 *  gsicp_pose_predict: d_hist [dev] double[32] = (T_{t-2}, T_{t-1}) row-major 4x4; writes d_T_out.
 *  gsicp_pose_push: d_hist <- (T_{t-1}, d_T); if d_traj [dev] double[traj_cap*16] and d_counter
 *  [dev] int32 are given, d_traj[*d_counter] = d_T and ++*d_counter (while < traj_cap).
 *  Errors: INVALID_ARGUMENT, CUDA. */
gsicp_status gsicp_pose_predict(const double *d_hist, double *d_T_out, void *stream);
gsicp_status gsicp_pose_push(double *d_hist, const double *d_T, double *d_traj, int32_t *d_counter, int32_t traj_cap,
                             void *stream);

/* N4 voxel downsampling (reading R31): at most one output point per occupied voxel,
 * the centroid of its members.  Voxel = (floor(x/h), floor(y/h), floor(z/h)), binary64 division;
 * centroid = binary64 mean of the members rounded to binary32; outputs ordered by each voxel's
 * smallest input index; non-finite points skipped; voxels within +-2^20 h of the origin.
 *  pos [dev] float4[cap] (x, y, z, payload), d_n [dev] int32 (<= cap);
 *  pos_out [dev] float4[cap]: rows [0, *d_m_out) = (centroid, member count as int bits) — a
 *      general cloud: search it with gsicp_covariances, not the image-window path;
 *  ws: gsicp_voxel_downsample_workspace_size(cap) bytes, 256-byte aligned.
 *  Errors: INVALID_ARGUMENT, WORKSPACE_TOO_SMALL, CUDA. */
size_t gsicp_voxel_downsample_workspace_size(int32_t cap);
gsicp_status gsicp_voxel_downsample(const float *pos, const int32_t *d_n, int32_t cap, float voxel, float *pos_out,
                                    int32_t *d_m_out, void *ws, size_t ws_bytes, void *stream);

/* A4 export: source points -> 3DGS Gaussians for keyframe insertion into the map (ALG-12).
 * P:187-191 Eq. 3 C = R Lambda^2 R^T, Eq. 4 Lambda' = Lambda / median(S)
 * Lambda'' = Lambda' / z^p (p = 1.5 best) with the absolute factor c (R21).
 *  pos, cov_a, cov_b [dev]: a source cloud and the covariances gsicp_covariances* wrote for it
 *      (the regularised covariance: its spectrum is the mode's Lambda'^2, its eigenvectors R);
 *  d_n [dev] int32: the number of points (<= cap); d_T [dev] double[16] row-major or NULL
 *      (identity): the pose mapping the camera frame into the world (the tracked pose);
 *  p, c: the scale-aligning exponent and factor.
 *  means_out [dev] float[cap*3] = K3(T, x) rounded to binary32; quats_out [dev] float[cap*4]
 *      (16-byte aligned) unit wxyz quaternion (w >= 0) of T_R * (v2, v1, v0) made right-handed;
 *  scales_out [dev] float[cap*3] = c * sqrt(var'_j) / z^p, descending, z = the point's camera
 *      depth (z <= 0: scales 0).  Exactly the layout gsicp_build_target reads (scales linear).
 *  corr [dev] nullable int32[cap]: the overlap filter (R28) — if given, only the points
 *      with corr[i] < 0 (no valid correspondence in the final linearisation: gsicp_align_async's
 *      corr_out, or gsicp_linearize's) are exported, compacted in index order into rows
 *      [0, *d_m_out); then d_m_out is required and ws must hold gsicp_export_workspace_size(cap)
 *      bytes (256-byte aligned).  Without corr, row i is point i and *d_m_out (if given) = *d_n.
 *  Rows beyond the exported count are not written.  Errors: INVALID_ARGUMENT (null, misaligned,
 *  cap < 1, p or c not finite, c <= 0, corr without d_m_out), WORKSPACE_TOO_SMALL, CUDA. */
size_t gsicp_export_workspace_size(int32_t cap);
gsicp_status gsicp_export_gaussians(const float *pos, const float *cov_a, const float *cov_b, const int32_t *d_n,
                                    int32_t cap, const double *d_T, double p, double c, const int32_t *corr,
                                    float *means_out, float *quats_out, float *scales_out, int32_t *d_m_out,
                                    void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * N1  Keyframes and a device-resident growing map with incremental target maintenance
 * (P:209-214 keyframe selection by the correspondence proportion, P:237 only Gaussians that do
 * not overlap the current map, P:250-255 scale aligning, P:262-266 forced keyframe; R28, R29).
 * The map owns its Gaussians (rows [0, *d_M) of means / quats wxyz / scales (linear), capacity
 * rows) and the G-ICP target over them (`target`, usable by every align call).  An insertion
 * appends a keyframe's exported Gaussians (gsicp_export_gaussians with the overlap filter) and
 * maintains the target incrementally: the exact 16-NN lists are recomputed only for the new
 * rows and the old rows whose list ball contains a new point; hash, dense cell
 * array and slot lists are rebuilt by streaming kernels.  The result equals a from-scratch
 * gsicp_build_target of the same rows (same neighbour sets, same covariances).  All counts stay
 * on the device: an insertion (and the keyframe decision) can be captured in a CUDA graph. */
typedef struct {
    gsicp_target target;   /* views into the map workspace (target.M = capacity)       */
    float *means;          /* [dev] float[capacity][3]                                 */
    float *quats;          /* [dev] float[capacity][4] wxyz                            */
    float *scales;         /* [dev] float[capacity][3] linear                          */
    int32_t *d_M;          /* [dev] d_M[0] current rows, d_M[1] rows added by the last insert,
                              d_M[4] Gaussians dropped because the map was full            */
    int32_t capacity, max_insert, mode;
    float cell, eps_var;
    void *ws;              /* the map workspace (opaque)                                */
} gsicp_map;

/* capacity >= 1 rows (< 2^27), max_insert >= 1: the largest keyframe cloud cap inserted. */
size_t gsicp_map_workspace_size(int32_t capacity, int32_t max_insert);
/* Copies M0 (<= capacity) initial Gaussians (scales linear or log) into the map and builds its
 * target with cell edge `cell` (<= 0: 3 x mean middle scale, blocking), kept for the map's life.
 * mode / eps_var: the regularisation of the target covariances (as gsicp_build_target). */
gsicp_status gsicp_map_init(const float *means, const float *quats_wxyz, const float *scales, int32_t scales_are_log,
                            int32_t M0, int32_t capacity, int32_t max_insert, gsicp_reg_mode mode, float eps_var,
                            float cell, gsicp_map *out, void *ws, size_t ws_bytes, void *stream);
/* Appends the keyframe cloud's Gaussians (kf->cap <= max_insert; d_T [dev] double[16] its
 * camera->world pose; corr [dev] nullable: the overlap filter, as gsicp_export_gaussians; p, c
 * scale aligning) and maintains the target.  d_flag [dev] nullable int32: insert only if
 * *d_flag != 0 — inside a stream capture this becomes a conditional graph node switched on the
 * device; eagerly it is read back (blocking).  Rows beyond the capacity are dropped and counted
 * in d_M[4].  Errors: INVALID_ARGUMENT, CUDA. */
gsicp_status gsicp_map_insert(const gsicp_map *map, const gsicp_cloud *kf, const double *d_T, const int32_t *corr,
                              double p, double c, const int32_t *d_flag, void *stream);
/* P:209-214 / P:262-266 keyframe decision on the device (R29): d_state [dev] int32[2] =
 * (frames since the last keyframe, decision); the frame is a keyframe iff it was tracked (status
 * not TRACKING_LOST / DEGENERATE_FRAME) and fitness < min_fitness or max_gap frames have passed;
 * then d_state = (0, 1), else (since + 1, 0).  d_stats [dev]: the frame's align stats. */
gsicp_status gsicp_keyframe_decide(const gsicp_align_stats *d_stats, int32_t *d_state, float min_fitness,
                                   int32_t max_gap, void *stream);

/* CUDA-graph helpers for callers that capture a whole frame (host pointers; stream-ordered).
 * gsicp_graph_instantiate: instantiates a captured graph (cudaGraph_t) so that kernel nodes keep
 * their launch priorities (cudaGraphInstantiateFlagUseNodePriority): the frame's critical path
 * runs at high priority and the side-stream work (iteration-0 seeds) at low priority.
 * gsicp_graph_launch / gsicp_graph_destroy: launch on a stream / destroy the executable graph. */
gsicp_status gsicp_graph_instantiate(void *graph, void **exec_out);
gsicp_status gsicp_graph_launch(void *exec, void *stream);
gsicp_status gsicp_graph_destroy(void *exec);

/* Misc */
const char *gsicp_status_string(gsicp_status s);
const char *gsicp_last_error(void);         /* thread-local detail of the last error           */
uint64_t gsicp_kernel_launch_count(void);   /* kernels launched by this thread (diagnostics)   */
int32_t gsicp_abi_version(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* GSICP_H */
