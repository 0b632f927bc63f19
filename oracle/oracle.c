/*
 * ORACLE — plain, slow, obviously-correct CPU implementation of the GS-ICP SLAM
 * G-ICP tracking hot path (arXiv 2403.12550).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares no code, header, table or constant generator
 * with the CUDA path (paper_2403_12550_b200/csrc) and never reads its outputs.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * Rn = reading n listed in DESIGN.md §3 (Rn = SURVEY.md §8(c).3 Qn for n >= 3).
 *
 * Precision: all arithmetic in IEEE binary64.  Where a floating-point value decides an
 * integer (kNN / NN membership) the decision is taken on SURVEY §8(c).1's canonical binary64
 * keys (DESIGN.md §3 R1): K2 key = (dx*dx + dy*dy) + dz*dz with dx = (double)a.x - (double)b.x,
 * and for correspondences the query is the binary64 K3 transform itself (R15, no rounding of
 * T x to binary32).  -ffp-contract=off: no FMA contraction changes the rounding.
 * Storage format: points and covariances are stored as binary32 (the hot path's
 * SoA format); the oracle rounds its binary64 results to binary32 where the format
 * stores them (DESIGN.md §3 R2).
 *
 * Parity pins (tests/test_oracle_*.py) — every function below is pinned to
 * something other than itself; see DESIGN.md §4 for the table.
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fopenmp -shared -fPIC oracle.c -lm
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORA_FLAG_LOW_SUPPORT 1
#define ORA_FLAG_DEGENERATE 2

enum { ORA_NONE = 0, ORA_PLANE = 1, ORA_ELLIPSE = 2 };
enum { ORA_OK = 0, ORA_DEGENERATE_FRAME = 4, ORA_TRACKING_LOST = 5, ORA_MAX_ITERS = 6 };

static const double ORA_TAU = 1e-12;      /* degenerate-eigenvalue threshold, m^2 (R8) */
static const double ORA_NONE_FLOOR = 1e-6; /* NONE-mode eigenvalue floor, m^2 */

/* ------------------------------------------------------------------------- */
/* O1  Back-projection + uniform stride downsampling.
 * P:163 (Fig. 2 caption): "We generate a point cloud by downsampling and
 * reprojecting the current depth image"; pinhole model S:46:
 * point = ((u-cx) d/fx, (v-cy) d/fy, d); invalid / out-of-window pixels skipped
 * (S:46).  Stride from (0,0), integer pixel coordinates (R13, R14).
 * K1: x = (float)(((double)u - (double)cx) * (double)z / (double)fx).
 * Output in row-major pixel order; out_pix = v*W + u.  Returns n, or -1 if n > cap.
 */
int ora_backproject(const float *depth, int H, int W, int pitch, float fx, float fy, float cx, float cy,
                    int stride, float zmin, float zmax, float *out_xyz, int32_t *out_pix, int cap) {
    int n = 0;
    for (int v = 0; v < H; v += stride) {
        for (int u = 0; u < W; u += stride) {
            float z = depth[(int64_t)v * pitch + u];
            if (!isfinite(z) || !(z >= zmin && z <= zmax)) continue;
            if (n >= cap) return -1;
            double zd = (double)z;
            double x = (((double)u - (double)cx) * zd) / (double)fx;
            double y = (((double)v - (double)cy) * zd) / (double)fy;
            out_xyz[3 * n + 0] = (float)x;
            out_xyz[3 * n + 1] = (float)y;
            out_xyz[3 * n + 2] = z;
            out_pix[n] = v * W + u;
            ++n;
        }
    }
    return n;
}

/* ------------------------------------------------------------------------- */
/* Canonical binary64 squared-distance key K2: the query q in binary64
 * (a binary32 cloud point widened exactly, or the binary64 K3 transform of one), b a binary32
 * point widened exactly; dx = b.x - q.x (the sign is irrelevant: squares of negations are
 * bit-identical), key = (dx*dx + dy*dy) + dz*dz, every op rounded separately, left to right. */
static inline double ora_keyd(const double *q, const float *b) {
    double dx = (double)b[0] - q[0];
    double dy = (double)b[1] - q[1];
    double dz = (double)b[2] - q[2];
    double s = dx * dx;
    s = s + dy * dy;
    s = s + dz * dz;
    return s;
}
static inline double ora_key(const float *a, const float *b) {
    double q[3] = {(double)a[0], (double)a[1], (double)a[2]};
    return ora_keyd(q, b);
}

/* (key, idx) lexicographic "less than" — the kNN / NN order (R12). */
static inline int ora_less(double ka, int ia, double kb, int ib) {
    return ka < kb || (ka == kb && ia < ib);
}

/* insert (key, idx) into the sorted list of length *len (capacity k) */
static inline void ora_topk_insert(double *keys, int32_t *ids, int *len, int k, double key, int id) {
    int m = *len;
    if (m == k) {
        if (!ora_less(key, id, keys[k - 1], ids[k - 1])) return;
        m = k - 1;
    }
    int p = m;
    while (p > 0 && ora_less(key, id, keys[p - 1], ids[p - 1])) {
        keys[p] = keys[p - 1];
        ids[p] = ids[p - 1];
        --p;
    }
    keys[p] = key;
    ids[p] = id;
    if (*len < k) ++*len;
}

/* O2  Exact kNN by brute force: the definition ("k-nearest neighbors of x";
 * S:64 self included; S:39 min(k,n) sorted; S:82 ties by lower index).
 * For each query q in qidx[0..nq): out_idx[q*k + j] = j-th neighbour, -1 pads when n<k.
 * out_key (nullable) gets the keys. */
void ora_knn_brute(const float *xyz, int n, const int32_t *qidx, int nq, int k, int32_t *out_idx, double *out_key) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int qi = 0; qi < nq; ++qi) {
        double keys[256];
        int32_t ids[256];
        int len = 0;
        const float *q = xyz + 3 * (int64_t)qidx[qi];
        for (int j = 0; j < n; ++j) ora_topk_insert(keys, ids, &len, k, ora_key(q, xyz + 3 * (int64_t)j), j);
        for (int j = 0; j < k; ++j) {
            out_idx[(int64_t)qi * k + j] = j < len ? ids[j] : -1;
            if (out_key) out_key[(int64_t)qi * k + j] = j < len ? keys[j] : INFINITY;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* Exact kd-tree over binary32 points (speed-up for large clouds; validated against
 * ora_knn_brute and scipy's cKDTree in tests).  Split values are point coordinates,
 * so a subtree across a split plane s can be skipped iff the binary64 plane key
 * fl(fl(q_a - s)^2) exceeds the current k-th key: rounding is monotone and every K2 key is
 * a rounded sum of non-negative terms, so every point p behind the plane has
 * key(q, p) >= fl((q_a - p_a)^2) >= that plane key. */
typedef struct {
    int32_t *perm;   /* point ids in tree order */
    int32_t *lo, *hi; /* node range */
    int32_t *left, *right;
    int8_t *axis;
    float *split;
    int nnodes;
    const float *xyz;
} ora_kdtree;

static const float *g_sort_xyz;
static int g_sort_axis;
static int ora_cmp_axis(const void *a, const void *b) {
    int ia = *(const int32_t *)a, ib = *(const int32_t *)b;
    float va = g_sort_xyz[3 * (int64_t)ia + g_sort_axis], vb = g_sort_xyz[3 * (int64_t)ib + g_sort_axis];
    if (va < vb) return -1;
    if (va > vb) return 1;
    return (ia > ib) - (ia < ib);
}

static int ora_kd_build_rec(ora_kdtree *t, int lo, int hi) {
    int node = t->nnodes++;
    t->lo[node] = lo;
    t->hi[node] = hi;
    t->left[node] = t->right[node] = -1;
    t->axis[node] = -1;
    if (hi - lo <= 8) return node;
    float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = lo; i < hi; ++i)
        for (int a = 0; a < 3; ++a) {
            float v = t->xyz[3 * (int64_t)t->perm[i] + a];
            if (v < mn[a]) mn[a] = v;
            if (v > mx[a]) mx[a] = v;
        }
    int ax = 0;
    for (int a = 1; a < 3; ++a)
        if (mx[a] - mn[a] > mx[ax] - mn[ax]) ax = a;
    if (!(mx[ax] > mn[ax])) return node; /* all coincident: leaf */
    g_sort_xyz = t->xyz;
    g_sort_axis = ax;
    qsort(t->perm + lo, hi - lo, sizeof(int32_t), ora_cmp_axis);
    int mid = (lo + hi) / 2;
    t->axis[node] = (int8_t)ax;
    t->split[node] = t->xyz[3 * (int64_t)t->perm[mid] + ax];
    /* left: [lo,mid) all <= split ; right: [mid,hi) all >= split */
    int l = ora_kd_build_rec(t, lo, mid);
    int r = ora_kd_build_rec(t, mid, hi);
    t->left[node] = l;
    t->right[node] = r;
    return node;
}

void *ora_kdtree_build(const float *xyz, int n) {
    ora_kdtree *t = (ora_kdtree *)calloc(1, sizeof(ora_kdtree));
    int cap = 2 * (n / 4 + 1) + 16;
    t->perm = (int32_t *)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
    t->lo = (int32_t *)malloc(sizeof(int32_t) * cap);
    t->hi = (int32_t *)malloc(sizeof(int32_t) * cap);
    t->left = (int32_t *)malloc(sizeof(int32_t) * cap);
    t->right = (int32_t *)malloc(sizeof(int32_t) * cap);
    t->axis = (int8_t *)malloc(cap);
    t->split = (float *)malloc(sizeof(float) * cap);
    t->xyz = xyz;
    for (int i = 0; i < n; ++i) t->perm[i] = i;
    if (n > 0) ora_kd_build_rec(t, 0, n);
    return t;
}

void ora_kdtree_free(void *p) {
    ora_kdtree *t = (ora_kdtree *)p;
    if (!t) return;
    free(t->perm); free(t->lo); free(t->hi); free(t->left); free(t->right); free(t->axis); free(t->split);
    free(t);
}

static void ora_kd_search(const ora_kdtree *t, int node, const double *q, int k, double *keys, int32_t *ids, int *len) {
    if (t->axis[node] < 0) {
        for (int i = t->lo[node]; i < t->hi[node]; ++i) {
            int id = t->perm[i];
            ora_topk_insert(keys, ids, len, k, ora_keyd(q, t->xyz + 3 * (int64_t)id), id);
        }
        return;
    }
    int ax = t->axis[node];
    double d = q[ax] - (double)t->split[node];
    int first = d <= 0 ? t->left[node] : t->right[node];
    int second = d <= 0 ? t->right[node] : t->left[node];
    ora_kd_search(t, first, q, k, keys, ids, len);
    double pk = d * d;
    if (*len < k || !(pk > keys[*len - 1])) ora_kd_search(t, second, q, k, keys, ids, len);
}

/* kNN of arbitrary binary32 query positions q[nq][3] against the tree's points (same order/ties
 * as brute force). */
void ora_kdtree_knn(const void *tree, const float *q, int nq, int k, int32_t *out_idx, double *out_key) {
    const ora_kdtree *t = (const ora_kdtree *)tree;
#pragma omp parallel for schedule(dynamic, 256)
    for (int i = 0; i < nq; ++i) {
        double keys[256];
        int32_t ids[256];
        int len = 0;
        double qd[3] = {(double)q[3 * (int64_t)i], (double)q[3 * (int64_t)i + 1], (double)q[3 * (int64_t)i + 2]};
        if (t->nnodes > 0) ora_kd_search(t, 0, qd, k, keys, ids, &len);
        for (int j = 0; j < k; ++j) {
            out_idx[(int64_t)i * k + j] = j < len ? ids[j] : -1;
            if (out_key) out_key[(int64_t)i * k + j] = j < len ? keys[j] : INFINITY;
        }
    }
}

/* 1-NN of binary64 queries (the K3 transforms of O7) by (K2, index); -1 / inf if the tree is empty. */
void ora_kdtree_nn_d(const void *tree, const double *q, int nq, int32_t *out_idx, double *out_key) {
    const ora_kdtree *t = (const ora_kdtree *)tree;
#pragma omp parallel for schedule(dynamic, 256)
    for (int i = 0; i < nq; ++i) {
        double key = INFINITY;
        int32_t id = -1;
        int len = 0;
        if (t->nnodes > 0) ora_kd_search(t, 0, q + 3 * (int64_t)i, 1, &key, &id, &len);
        out_idx[i] = len ? id : -1;
        out_key[i] = len ? key : INFINITY;
    }
}

/* ------------------------------------------------------------------------- */
/* O3  Covariance of the neighbour set (sample covariance normalised by k,
 * two-pass in binary64).  C packed as (c00,c01,c02,c11,c12,c22). */
void ora_covariance(const float *xyz, const int32_t *nbr, int m, double *C) {
    double mu[3] = {0, 0, 0};
    int cnt = 0;
    for (int j = 0; j < m; ++j) {
        if (nbr[j] < 0) continue;
        for (int a = 0; a < 3; ++a) mu[a] += (double)xyz[3 * (int64_t)nbr[j] + a];
        ++cnt;
    }
    for (int a = 0; a < 3; ++a) mu[a] /= (double)cnt;
    double S[3][3] = {{0}};
    for (int j = 0; j < m; ++j) {
        if (nbr[j] < 0) continue;
        double d[3];
        for (int a = 0; a < 3; ++a) d[a] = (double)xyz[3 * (int64_t)nbr[j] + a] - mu[a];
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) S[a][b] += d[a] * d[b];
    }
    C[0] = S[0][0] / cnt; C[1] = S[0][1] / cnt; C[2] = S[0][2] / cnt;
    C[3] = S[1][1] / cnt; C[4] = S[1][2] / cnt; C[5] = S[2][2] / cnt;
}

/* O4  Symmetric eigen-decomposition (Eq. 3: C = R Lambda^2 R^T, read as the
 * eigen-decomposition of the PSD covariance, R4) by the cyclic Jacobi method in binary64,
 * until off(A) <= 1e-15 ||A||_F (max 50 sweeps).  Output lam[0] >= lam[1] >= lam[2]
 * (= lambda_2, lambda_1, lambda_0 in the paper's s2>s1>s0 order, R5), clamped at 0;
 * V column-major: V[3*j + r] is component r of the eigenvector of lam[j]. */
void ora_eigen_jacobi(const double *Cp, double *lam, double *V) {
    double A[3][3] = {{Cp[0], Cp[1], Cp[2]}, {Cp[1], Cp[3], Cp[4]}, {Cp[2], Cp[4], Cp[5]}};
    double Q[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    double fro = 0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) fro += A[i][j] * A[i][j];
    fro = sqrt(fro);
    for (int sweep = 0; sweep < 50; ++sweep) {
        double off = sqrt(2.0 * (A[0][1] * A[0][1] + A[0][2] * A[0][2] + A[1][2] * A[1][2]));
        if (off <= 1e-15 * fro) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                if (A[p][q] == 0.0) continue;
                /* Golub & Van Loan Alg. 8.4.1 (symmetric Schur 2x2) */
                double tau = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
                double t = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
                for (int k = 0; k < 3; ++k) { /* A <- A J */
                    double akp = A[k][p], akq = A[k][q];
                    A[k][p] = c * akp - s * akq;
                    A[k][q] = s * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) { /* A <- J^T A */
                    double apk = A[p][k], aqk = A[q][k];
                    A[p][k] = c * apk - s * aqk;
                    A[q][k] = s * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) { /* Q <- Q J */
                    double qkp = Q[k][p], qkq = Q[k][q];
                    Q[k][p] = c * qkp - s * qkq;
                    Q[k][q] = s * qkp + c * qkq;
                }
            }
    }
    int ord[3] = {0, 1, 2};
    double d[3] = {A[0][0], A[1][1], A[2][2]};
    /* sort descending, stable by index */
    for (int i = 0; i < 3; ++i)
        for (int j = i + 1; j < 3; ++j)
            if (d[ord[j]] > d[ord[i]]) { int tmp = ord[i]; ord[i] = ord[j]; ord[j] = tmp; }
    for (int j = 0; j < 3; ++j) {
        lam[j] = d[ord[j]] > 0 ? d[ord[j]] : 0.0;
        for (int r = 0; r < 3; ++r) V[3 * j + r] = Q[r][ord[j]];
    }
}

static void ora_add_outer(double *Cp, double w, const double *v) {
    Cp[0] += w * v[0] * v[0]; Cp[1] += w * v[0] * v[1]; Cp[2] += w * v[0] * v[2];
    Cp[3] += w * v[1] * v[1]; Cp[4] += w * v[1] * v[2]; Cp[5] += w * v[2] * v[2];
}

/* O5  Regularisation from an eigen-decomposition (lam descending, V columns).
 *  NONE    : sum max(lam_i, 1e-6) v v^T
 *  PLANE   : S = [1, 1, eps] as variances: v2v2^T + v1v1^T + eps v0v0^T   (R6)
 *  ELLIPSE : Lambda' = Lambda / median(S)  (Eq. 4) => variances lam_i/lam_mid,
 *            floored at eps (R7):  sum max(lam_i/lam_1, eps) v v^T
 *  Degenerate (R8): lam_2 <= tau -> I (NONE: 1e-6 I), flag; lam_1 <= tau < lam_2 (line) ->
 *            v2v2^T + eps (I - v2v2^T) for PLANE/ELLIPSE, flag.
 * Returns flags. */
int ora_regularize_eig(const double *lam, const double *V, int mode, double eps, double *out) {
    for (int i = 0; i < 6; ++i) out[i] = 0.0;
    const double *v2 = V, *v1 = V + 3, *v0 = V + 6;
    if (mode == ORA_NONE) {
        for (int j = 0; j < 3; ++j) ora_add_outer(out, lam[j] > ORA_NONE_FLOOR ? lam[j] : ORA_NONE_FLOOR, V + 3 * j);
        return lam[0] <= ORA_TAU ? ORA_FLAG_DEGENERATE : 0;
    }
    if (lam[0] <= ORA_TAU) {
        out[0] = out[3] = out[5] = 1.0;
        return ORA_FLAG_DEGENERATE;
    }
    if (lam[1] <= ORA_TAU) {
        double I[6] = {1, 0, 0, 1, 0, 1};
        for (int i = 0; i < 6; ++i) out[i] = eps * I[i];
        ora_add_outer(out, 1.0 - eps, v2);
        return ORA_FLAG_DEGENERATE;
    }
    if (mode == ORA_PLANE) {
        ora_add_outer(out, 1.0, v2);
        ora_add_outer(out, 1.0, v1);
        ora_add_outer(out, eps, v0);
        return 0;
    }
    /* ELLIPSE */
    for (int j = 0; j < 3; ++j) {
        double w = lam[j] / lam[1];
        ora_add_outer(out, w > eps ? w : eps, V + 3 * j);
    }
    return 0;
}

int ora_regularize(const double *C, int mode, double eps, double *out) {
    double lam[3], V[9];
    ora_eigen_jacobi(C, lam, V);
    return ora_regularize_eig(lam, V, mode, eps, out);
}

/* A2-A4 composed: kNN (brute force if n <= brute_max, else kd-tree) -> covariance ->
 * regularise.  cov_out: n*6 binary32 (stored format), raw_out (nullable): n*6 binary64
 * raw covariances, lam_mid_out (nullable): binary64 lambda_1, flags_out: n int32. */
void ora_covariances(const float *xyz, int n, int k, int mode, double eps, int brute_max,
                     float *cov_out, double *raw_out, double *lam_mid_out, int32_t *flags_out) {
    int32_t *nbr = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1) * k);
    if (n <= brute_max) {
        int32_t *q = (int32_t *)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
        for (int i = 0; i < n; ++i) q[i] = i;
        ora_knn_brute(xyz, n, q, n, k, nbr, NULL);
        free(q);
    } else {
        void *t = ora_kdtree_build(xyz, n);
        ora_kdtree_knn(t, xyz, n, k, nbr, NULL);
        ora_kdtree_free(t);
    }
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        double C[6], lam[3], V[9], R[6];
        ora_covariance(xyz, nbr + (int64_t)i * k, k, C);
        ora_eigen_jacobi(C, lam, V);
        int fl = ora_regularize_eig(lam, V, mode, eps, R);
        if (n < k) fl |= ORA_FLAG_LOW_SUPPORT;
        for (int j = 0; j < 6; ++j) cov_out[6 * (int64_t)i + j] = (float)R[j];
        if (raw_out)
            for (int j = 0; j < 6; ++j) raw_out[6 * (int64_t)i + j] = C[j];
        if (lam_mid_out) lam_mid_out[i] = lam[1];
        flags_out[i] = fl;
    }
    free(nbr);
}

/* ------------------------------------------------------------------------- */
/* O6  Map Gaussian -> G-ICP target covariance (the map's Gaussians are
 * reused as targets without recomputing covariances; P:189-191 C = R Lambda^2 R^T).
 * q = wxyz normalised (R22); scales linear or log (exp); variances s_i^2 sorted descending,
 * ties by axis index (R5); then O5. */
void ora_target_from_map(const float *quats, const float *scales, int scales_are_log, int M, int mode,
                         double eps, float *cov_out, int32_t *flags_out) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < M; ++i) {
        double w = quats[4 * (int64_t)i], x = quats[4 * (int64_t)i + 1], y = quats[4 * (int64_t)i + 2],
               z = quats[4 * (int64_t)i + 3];
        double nq = sqrt(w * w + x * x + y * y + z * z);
        w /= nq; x /= nq; y /= nq; z /= nq;
        double R[3][3] = {{1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
                          {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
                          {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)}};
        double s[3];
        for (int a = 0; a < 3; ++a) {
            double v = (double)scales[3 * (int64_t)i + a];
            s[a] = scales_are_log ? exp(v) : v;
        }
        int ord[3] = {0, 1, 2};
        for (int a = 0; a < 3; ++a)
            for (int b = a + 1; b < 3; ++b)
                if (s[ord[b]] > s[ord[a]]) { int t = ord[a]; ord[a] = ord[b]; ord[b] = t; }
        double lam[3], V[9], out[6];
        for (int j = 0; j < 3; ++j) {
            lam[j] = s[ord[j]] * s[ord[j]];
            for (int r = 0; r < 3; ++r) V[3 * j + r] = R[r][ord[j]];
        }
        flags_out[i] = ora_regularize_eig(lam, V, mode, eps, out);
        for (int j = 0; j < 6; ++j) cov_out[6 * (int64_t)i + j] = (float)out[j];
    }
}

/* ------------------------------------------------------------------------- */
/* K3 transform of a binary32 point by the binary64 pose: q_r = ((R_r0 x + R_r1 y) + R_r2 z) + t_r */
static inline void ora_transform(const double *T, const float *p, double *q) {
    double x = p[0], y = p[1], z = p[2];
    for (int r = 0; r < 3; ++r) {
        double a = T[4 * r + 0] * x;
        a = a + T[4 * r + 1] * y;
        a = a + T[4 * r + 2] * z;
        q[r] = a + T[4 * r + 3];
    }
}

static void ora_sym_unpack(const float *c, double A[3][3]) {
    A[0][0] = c[0]; A[0][1] = A[1][0] = c[1]; A[0][2] = A[2][0] = c[2];
    A[1][1] = c[3]; A[1][2] = A[2][1] = c[4]; A[2][2] = c[5];
}

/* Cholesky inverse of an SPD 3x3 (returns 0 if not PD). */
static int ora_inv_spd3(double S[3][3], double Mi[3][3]) {
    double L[3][3] = {{0}};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = S[i][j];
            for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
            if (i == j) {
                if (!(s > 0)) return 0;
                L[i][i] = sqrt(s);
            } else
                L[i][j] = s / L[j][j];
        }
    for (int c = 0; c < 3; ++c) {
        double e[3] = {c == 0, c == 1, c == 2}, y[3], x[3];
        for (int i = 0; i < 3; ++i) {
            double s = e[i];
            for (int k = 0; k < i; ++k) s -= L[i][k] * y[k];
            y[i] = s / L[i][i];
        }
        for (int i = 2; i >= 0; --i) {
            double s = y[i];
            for (int k = i + 1; k < 3; ++k) s -= L[k][i] * x[k];
            x[i] = s / L[i][i];
        }
        for (int r = 0; r < 3; ++r) Mi[r][c] = x[r];
    }
    return 1;
}

/* O7 + O8: correspondences and linearisation of Eq. 1 at pose T.
 * O7: q_i = K3(T, x_i) in binary64; j* = argmin over (K2(q_i, m_j), j) ("nearest neighbor",
 *     R15); valid iff key < r^2 with r^2 = (double)r * (double)r (strict, R15).
 * O8: Sigma_i = C^t_j + R C^s_i R^T (R3), M_i = Sigma_i^{-1}, d_i = m_j - q_i,
 *     J_i = [[q_i]x, -I] (left twist (omega, v), R16), H = sum J^T M J, b = sum J^T M d,
 *     cost = sum d^T M d (Eq. 1), summed in index order in binary64.  A pair whose Sigma is not
 *     positive definite is skipped (after R31).
 * tree: kd-tree over tgt_xyz or NULL (brute force).  H row-major 36, b 6.  corr (nullable).
 * Returns the inlier count. */
/* bsum (nullable): sum over the valid pairs of |J_i^T M_i d_i| — the scale of SURVEY §8(c).5's
 * per-iteration b tolerance (b itself -> 0 at the optimum). */
int ora_linearize_ex(const float *src_xyz, const float *src_cov, int n, const float *tgt_xyz, const float *tgt_cov,
                     int M, const void *tree, const double *T, float max_corr_dist, double *H, double *b,
                     double *cost, int32_t *corr, double *bsum);
int ora_linearize(const float *src_xyz, const float *src_cov, int n, const float *tgt_xyz, const float *tgt_cov,
                  int M, const void *tree, const double *T, float max_corr_dist, double *H, double *b,
                  double *cost, int32_t *corr) {
    return ora_linearize_ex(src_xyz, src_cov, n, tgt_xyz, tgt_cov, M, tree, T, max_corr_dist, H, b, cost, corr, NULL);
}
int ora_linearize_ex(const float *src_xyz, const float *src_cov, int n, const float *tgt_xyz, const float *tgt_cov,
                     int M, const void *tree, const double *T, float max_corr_dist, double *H, double *b,
                     double *cost, int32_t *corr, double *bsum) {
    double r2 = (double)max_corr_dist * (double)max_corr_dist;
    double *contrib = (double *)calloc((size_t)(n > 0 ? n : 1) * 28, sizeof(double));
    int32_t *cj = (int32_t *)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
#pragma omp parallel for schedule(dynamic, 256)
    for (int i = 0; i < n; ++i) {
        double q[3];
        ora_transform(T, src_xyz + 3 * (int64_t)i, q);
        int best = -1;
        double bk = INFINITY;
        if (tree) {
            ora_kdtree_nn_d(tree, q, 1, &best, &bk);
        } else {
            for (int j = 0; j < M; ++j) {
                double kk = ora_keyd(q, tgt_xyz + 3 * (int64_t)j);
                if (best < 0 || ora_less(kk, j, bk, best)) { bk = kk; best = j; }
            }
        }
        if (!(best >= 0 && bk < r2)) { cj[i] = -1; continue; }
        cj[i] = best;
        double Cs[3][3], Ct[3][3], S[3][3], Mi[3][3], RC[3][3];
        ora_sym_unpack(src_cov + 6 * (int64_t)i, Cs);
        ora_sym_unpack(tgt_cov + 6 * (int64_t)best, Ct);
        for (int a = 0; a < 3; ++a)
            for (int c = 0; c < 3; ++c) {
                double s = 0;
                for (int k = 0; k < 3; ++k) s += T[4 * a + k] * Cs[k][c];
                RC[a][c] = s;
            }
        for (int a = 0; a < 3; ++a)
            for (int c = 0; c < 3; ++c) {
                double s = 0;
                for (int k = 0; k < 3; ++k) s += RC[a][k] * T[4 * c + k];
                S[a][c] = Ct[a][c] + s;
            }
        if (!ora_inv_spd3(S, Mi)) { cj[i] = -1; continue; }
        double d[3];
        for (int a = 0; a < 3; ++a) d[a] = (double)tgt_xyz[3 * (int64_t)best + a] - q[a];
        /* J = [[q]x, -I] (3x6) */
        double J[3][6] = {{0, -q[2], q[1], -1, 0, 0}, {q[2], 0, -q[0], 0, -1, 0}, {-q[1], q[0], 0, 0, 0, -1}};
        double MJ[3][6], Md[3];
        for (int a = 0; a < 3; ++a) {
            for (int c = 0; c < 6; ++c) {
                double s = 0;
                for (int k = 0; k < 3; ++k) s += Mi[a][k] * J[k][c];
                MJ[a][c] = s;
            }
            Md[a] = Mi[a][0] * d[0] + Mi[a][1] * d[1] + Mi[a][2] * d[2];
        }
        double *o = contrib + (int64_t)i * 28;
        int t = 0;
        for (int r = 0; r < 6; ++r)
            for (int c = r; c < 6; ++c) {
                double s = 0;
                for (int k = 0; k < 3; ++k) s += J[k][r] * MJ[k][c];
                o[t++] = s; /* 21 upper-triangular H terms */
            }
        for (int r = 0; r < 6; ++r) o[21 + r] = J[0][r] * Md[0] + J[1][r] * Md[1] + J[2][r] * Md[2];
        o[27] = d[0] * Md[0] + d[1] * Md[1] + d[2] * Md[2];
    }
    double acc[28] = {0}, bs = 0.0;
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
        if (corr) corr[i] = cj[i];
        if (cj[i] < 0) continue;
        ++cnt;
        for (int t = 0; t < 28; ++t) acc[t] += contrib[(int64_t)i * 28 + t];
        const double *bi = contrib + (int64_t)i * 28 + 21;
        bs += sqrt(bi[0] * bi[0] + bi[1] * bi[1] + bi[2] * bi[2] + bi[3] * bi[3] + bi[4] * bi[4] + bi[5] * bi[5]);
    }
    if (bsum) *bsum = bs;
    int t = 0;
    for (int r = 0; r < 6; ++r)
        for (int c = r; c < 6; ++c) { H[6 * r + c] = H[6 * c + r] = acc[t++]; }
    for (int r = 0; r < 6; ++r) b[r] = acc[21 + r];
    *cost = acc[27];
    free(contrib);
    free(cj);
    return cnt;
}

/* 6x6 Cholesky solve H x = rhs (returns 0 if not PD). */
static int ora_chol6(const double *H, const double *rhs, double *x) {
    double L[6][6] = {{0}};
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = H[6 * i + j];
            for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
            if (i == j) {
                if (!(s > 0)) return 0;
                L[i][i] = sqrt(s);
            } else
                L[i][j] = s / L[j][j];
        }
    double y[6];
    for (int i = 0; i < 6; ++i) {
        double s = rhs[i];
        for (int k = 0; k < i; ++k) s -= L[i][k] * y[k];
        y[i] = s / L[i][i];
    }
    for (int i = 5; i >= 0; --i) {
        double s = y[i];
        for (int k = i + 1; k < 6; ++k) s -= L[k][i] * x[k];
        x[i] = s / L[i][i];
    }
    return 1;
}

/* O9  delta = -H^{-1} b by 6x6 Cholesky; if H is not PD add 1e-6 tr(H)/6 I and retry.
 * Returns 0 if both attempts fail. */
int ora_solve(const double *H, const double *b, double *delta) {
    double nb[6];
    for (int i = 0; i < 6; ++i) nb[i] = -b[i];
    if (ora_chol6(H, nb, delta)) return 1;
    double Hd[36], tr = 0;
    memcpy(Hd, H, sizeof(Hd));
    for (int i = 0; i < 6; ++i) tr += H[7 * i];
    for (int i = 0; i < 6; ++i) Hd[7 * i] += 1e-6 * tr / 6.0;
    return ora_chol6(Hd, nb, delta);
}

/* Exp map of so(3) by Rodrigues; 2nd-order Taylor below theta = 1e-8. */
void ora_so3_exp(const double *w, double *R) {
    double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    double K[3][3] = {{0, -w[2], w[1]}, {w[2], 0, -w[0]}, {-w[1], w[0], 0}};
    double K2[3][3];
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) K2[a][c] = K[a][0] * K[0][c] + K[a][1] * K[1][c] + K[a][2] * K[2][c];
    double A, B;
    if (th < 1e-8) { A = 1.0; B = 0.5; }
    else { A = sin(th) / th; B = (1.0 - cos(th)) / (th * th); }
    for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) R[3 * a + c] = (a == c ? 1.0 : 0.0) + A * K[a][c] + B * K2[a][c];
}

/* Left update T <- [Exp(omega) | v] T (R16). */
void ora_update(double *T, const double *delta) {
    double E[9], Rn[9], tn[3];
    ora_so3_exp(delta, E);
    for (int a = 0; a < 3; ++a) {
        for (int c = 0; c < 3; ++c) Rn[3 * a + c] = E[3 * a] * T[c] + E[3 * a + 1] * T[4 + c] + E[3 * a + 2] * T[8 + c];
        tn[a] = E[3 * a] * T[3] + E[3 * a + 1] * T[7] + E[3 * a + 2] * T[11] + delta[3 + a];
    }
    for (int a = 0; a < 3; ++a) {
        for (int c = 0; c < 3; ++c) T[4 * a + c] = Rn[3 * a + c];
        T[4 * a + 3] = tn[a];
    }
    T[12] = T[13] = T[14] = 0.0;
    T[15] = 1.0;
}

/* O10/O11  Gauss-Newton loop (R16-R20).  stats: [fitness, mean_cost, n_inliers,
 * iters, converged, status].  NN: prebuilt kd-tree over tgt_xyz if given, else a tree built here
 * (use_tree) or brute force.  Returns status. */
/* O10 with the solver option.  solver 0: Gauss-Newton (O9 each iteration).  solver 1:
 * Levenberg-Marquardt (R30; the paper is silent, SPEC S:151/S:157 ask for a damped fallback):
 * iteration k linearises at the trial pose T_k; T_k is accepted iff k == 0 or its Eq. 1 cost is
 * below the last accepted cost (a trial with fewer than min_pairs inliers is rejected); accept:
 * lambda <- k == 0 ? lambda0 : lambda / 10, keep (T_a, H_a, b_a, cost_a, n_a); reject: lambda <-
 * 10 lambda.  Step: (H_a + lambda diag(H_a)) delta = -b_a (O9's Cholesky with its PD fallback),
 * T_{k+1} = Exp(delta) T_a (left update).  Converged iff |omega| < eps_rot and |v| < eps_trans
 * (the pose returned is then T_{k+1}, as for GN); at the cap the best accepted pose T_a is returned
 * ("max-iters, best iterate").  Stats from the accepted linearisation. */
int ora_align2(const float *src_xyz, const float *src_cov, int n, const float *tgt_xyz, const float *tgt_cov,
               int M, int use_tree, const void *prebuilt, const double *T0, int max_iters, float max_corr_dist,
               double eps_rot, double eps_trans, int min_pairs, int solver, double lambda0, double *T_out,
               double *stats) {
    void *own = (!prebuilt && use_tree) ? ora_kdtree_build(tgt_xyz, M) : NULL;
    const void *tree = prebuilt ? prebuilt : own;
    double T[16], Ta[16], Ha[36], ba[6], cost_a = 0, lambda = lambda0;
    memcpy(T, T0, sizeof(T));
    memcpy(Ta, T0, sizeof(Ta));
    int status = ORA_MAX_ITERS, iters = 0, conv = 0, ninl = 0, n_a = 0;
    double cost = 0;
    for (int it = 0; it < max_iters; ++it) {
        double H[36], b[6], delta[6];
        ninl = ora_linearize(src_xyz, src_cov, n, tgt_xyz, tgt_cov, M, tree, T, max_corr_dist, H, b, &cost, NULL);
        if (solver == 0) {
            if (ninl < min_pairs) { status = ORA_TRACKING_LOST; break; }
            if (!ora_solve(H, b, delta)) { status = ORA_TRACKING_LOST; break; }
            ora_update(T, delta);
        } else {
            int accept = it == 0 ? ninl >= min_pairs : (ninl >= min_pairs && cost < cost_a);
            if (it == 0 && !accept) { status = ORA_TRACKING_LOST; break; }
            if (accept) {
                memcpy(Ta, T, sizeof(Ta));
                memcpy(Ha, H, sizeof(Ha));
                memcpy(ba, b, sizeof(ba));
                cost_a = cost;
                n_a = ninl;
                if (it > 0) lambda = lambda / 10.0;
            } else {
                lambda = lambda * 10.0;
            }
            double D[36];
            memcpy(D, Ha, sizeof(D));
            for (int k = 0; k < 6; ++k) D[7 * k] = Ha[7 * k] + lambda * Ha[7 * k];
            if (!ora_solve(D, ba, delta)) { status = ORA_TRACKING_LOST; break; }
            memcpy(T, Ta, sizeof(T));
            ora_update(T, delta);
        }
        iters = it + 1;
        double nw = sqrt(delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2]);
        double nv = sqrt(delta[3] * delta[3] + delta[4] * delta[4] + delta[5] * delta[5]);
        if (nw < eps_rot && nv < eps_trans) { conv = 1; status = ORA_OK; break; }
    }
    if (solver != 0) {
        if (status == ORA_MAX_ITERS) memcpy(T, Ta, sizeof(T));  /* best (accepted) iterate */
        if (status == ORA_TRACKING_LOST && iters > 0) memcpy(T, Ta, sizeof(T));
        ninl = n_a;
        cost = cost_a;
    }
    if (own) ora_kdtree_free(own);
    memcpy(T_out, T, sizeof(T));
    stats[0] = n > 0 ? (double)ninl / n : 0.0;
    stats[1] = ninl > 0 ? cost / ninl : 0.0;
    stats[2] = ninl;
    stats[3] = iters;
    stats[4] = conv;
    stats[5] = status;
    return status;
}

int ora_align(const float *src_xyz, const float *src_cov, int n, const float *tgt_xyz, const float *tgt_cov,
              int M, int use_tree, const void *prebuilt, const double *T0, int max_iters, float max_corr_dist,
              double eps_rot, double eps_trans, int min_pairs, double *T_out, double *stats) {
    return ora_align2(src_xyz, src_cov, n, tgt_xyz, tgt_cov, M, use_tree, prebuilt, T0, max_iters, max_corr_dist,
                      eps_rot, eps_trans, min_pairs, 0, 0.0, T_out, stats);
}

int ora_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* thread count of the OpenMP loops (the bench's baseline uses every host core even under a
 * launcher that sets OMP_NUM_THREADS=1) */
void ora_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* O12  Scale aligning for map insertion (Lambda'' = Lambda' / z^p, p empirically
 * 1.5).  scales_out = c * scales_in / z^p (c: absolute factor, R21).  z <= 0 -> -1. */
int ora_scale_align(const double *scales_in, double z, double p, double c, double *scales_out) {
    if (!(z > 0)) return -1;
    double f = c / pow(z, p);
    for (int a = 0; a < 3; ++a) scales_out[a] = scales_in[a] * f;
    return 0;
}

/* O12' 3DGS export of one source point (ALG-12; Eq. 3-4):
 *  1. C = R Lambda^2 R^T (Eq. 3) by O4 (Jacobi): variances lam_2 >= lam_1 >= lam_0, frame (v2, v1, v0);
 *  2. the mode's regularised variances (the spectrum of O5's output, R6-R8):
 *       ELLIPSE  max(lam_i / lam_1, eps)   (Lambda' = Lambda / median(S), Eq. 4, floored, R7)
 *       PLANE    (1, 1, eps)               (R6)
 *       NONE     max(lam_i, 1e-6)
 *       degenerate (R8): lam_2 <= tau -> (1, 1, 1) (NONE: 1e-6 each); lam_1 <= tau -> (1, eps, eps);
 *  3. Lambda'' = Lambda' / z^p with the absolute factor c (R21): scales_i = c * sqrt(var_i) / z^p,
 *     z = the point's depth in the camera frame (p_cam[2]); z <= 0 -> scales 0 and return -1;
 *  4. the Gaussian's orientation: the frame (v2, v1, v0) made right-handed (v0 <- -v0 if det < 0),
 *     rotated into the world by T (R_w = T_R * frame), as a unit quaternion wxyz with w >= 0
 *     (Shepperd's method: the largest of 1 + trace, 1 + 2 R_aa - trace picks the stable formula);
 *  5. the mean: K3(T, p_cam).
 * T: row-major 4x4 binary64 (NULL = identity). */
static void ora_quat_from_rot(double R[3][3], double *q) {
    double tr = R[0][0] + R[1][1] + R[2][2];
    double w, x, y, z;
    if (tr >= R[0][0] && tr >= R[1][1] && tr >= R[2][2]) {
        double s = 2.0 * sqrt(1.0 + tr);
        w = 0.25 * s; x = (R[2][1] - R[1][2]) / s; y = (R[0][2] - R[2][0]) / s; z = (R[1][0] - R[0][1]) / s;
    } else if (R[0][0] >= R[1][1] && R[0][0] >= R[2][2]) {
        double s = 2.0 * sqrt(1.0 + R[0][0] - R[1][1] - R[2][2]);
        w = (R[2][1] - R[1][2]) / s; x = 0.25 * s; y = (R[0][1] + R[1][0]) / s; z = (R[0][2] + R[2][0]) / s;
    } else if (R[1][1] >= R[2][2]) {
        double s = 2.0 * sqrt(1.0 + R[1][1] - R[0][0] - R[2][2]);
        w = (R[0][2] - R[2][0]) / s; x = (R[0][1] + R[1][0]) / s; y = 0.25 * s; z = (R[1][2] + R[2][1]) / s;
    } else {
        double s = 2.0 * sqrt(1.0 + R[2][2] - R[0][0] - R[1][1]);
        w = (R[1][0] - R[0][1]) / s; x = (R[0][2] + R[2][0]) / s; y = (R[1][2] + R[2][1]) / s; z = 0.25 * s;
    }
    double n = sqrt(w * w + x * x + y * y + z * z);
    double sg = w < 0 ? -1.0 : 1.0;
    q[0] = sg * w / n; q[1] = sg * x / n; q[2] = sg * y / n; q[3] = sg * z / n;
}

int ora_export_gaussian(const double *C, const float *p_cam, const double *T, int mode, double eps, double p,
                        double c, double *mean_out, double *quat_out, double *scale_out) {
    double lam[3], V[9], var[3];
    ora_eigen_jacobi(C, lam, V);
    if (mode == ORA_NONE) {
        for (int j = 0; j < 3; ++j) var[j] = lam[j] > ORA_NONE_FLOOR ? lam[j] : ORA_NONE_FLOOR;
    } else if (lam[0] <= ORA_TAU) {
        var[0] = var[1] = var[2] = 1.0;
    } else if (lam[1] <= ORA_TAU) {
        var[0] = 1.0; var[1] = var[2] = eps;
    } else if (mode == ORA_PLANE) {
        var[0] = var[1] = 1.0; var[2] = eps;
    } else {
        for (int j = 0; j < 3; ++j) {
            double w = lam[j] / lam[1];
            var[j] = w > eps ? w : eps;
        }
    }
    double z = (double)p_cam[2];
    int rc = 0;
    double f = 0.0;
    if (z > 0) f = c / pow(z, p); else rc = -1;
    for (int j = 0; j < 3; ++j) scale_out[j] = f * sqrt(var[j]);
    /* right-handed frame: columns v2, v1, v0 */
    double F[3][3];
    for (int r = 0; r < 3; ++r)
        for (int j = 0; j < 3; ++j) F[r][j] = V[3 * j + r];
    double det = F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) - F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
                 F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
    if (det < 0)
        for (int r = 0; r < 3; ++r) F[r][2] = -F[r][2];
    double Rw[3][3];
    for (int r = 0; r < 3; ++r)
        for (int j = 0; j < 3; ++j)
            Rw[r][j] = T ? T[4 * r + 0] * F[0][j] + T[4 * r + 1] * F[1][j] + T[4 * r + 2] * F[2][j] : F[r][j];
    ora_quat_from_rot(Rw, quat_out);
    if (T) {
        ora_transform(T, p_cam, mean_out);
    } else {
        for (int r = 0; r < 3; ++r) mean_out[r] = (double)p_cam[r];
    }
    return rc;
}

/* O12' over a cloud: raw covariances (n*6 binary64, from ora_covariances' raw_out). */
void ora_export_gaussians(const float *xyz, const double *raw, int n, const double *T, int mode, double eps,
                          double p, double c, double *means, double *quats, double *scales) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i)
        ora_export_gaussian(raw + 6 * (int64_t)i, xyz + 3 * (int64_t)i, T, mode, eps, p, c, means + 3 * (int64_t)i,
                            quats + 4 * (int64_t)i, scales + 3 * (int64_t)i);
}

/* N4 voxel downsampling ("at most one output point per occupied voxel; output point
 * = centroid of members"; R31): voxel of a point = (floor(x / h), floor(y / h), floor(z / h)) with
 * binary64 division; output point = the binary64 mean of the members' coordinates (summed in index
 * order), rounded to binary32; outputs ordered by the smallest input index of each voxel; cnt_out =
 * members.  Non-finite points are skipped.  Returns m.  O(n log n): (key, index) pairs sorted. */
typedef struct { int64_t k[3]; int32_t i; } ora_vkey;
static int ora_vkey_cmp(const void *pa, const void *pb) {
    const ora_vkey *a = (const ora_vkey *)pa, *b = (const ora_vkey *)pb;
    for (int d = 0; d < 3; ++d)
        if (a->k[d] != b->k[d]) return a->k[d] < b->k[d] ? -1 : 1;
    return a->i < b->i ? -1 : (a->i > b->i);
}
typedef struct { int32_t first; float p[3]; int32_t cnt; } ora_vout;
static int ora_vout_cmp(const void *pa, const void *pb) {
    const ora_vout *a = (const ora_vout *)pa, *b = (const ora_vout *)pb;
    return a->first < b->first ? -1 : (a->first > b->first);
}
int ora_voxel_downsample(const float *xyz, int n, float voxel, float *out_xyz, int32_t *cnt_out) {
    ora_vkey *v = (ora_vkey *)malloc(sizeof(ora_vkey) * (size_t)(n > 0 ? n : 1));
    int nv = 0;
    for (int i = 0; i < n; ++i) {
        const float *p = xyz + 3 * (int64_t)i;
        if (!isfinite(p[0]) || !isfinite(p[1]) || !isfinite(p[2])) continue;
        for (int d = 0; d < 3; ++d) v[nv].k[d] = (int64_t)floor((double)p[d] / (double)voxel);
        v[nv].i = i;
        ++nv;
    }
    qsort(v, (size_t)nv, sizeof(ora_vkey), ora_vkey_cmp);
    ora_vout *o = (ora_vout *)malloc(sizeof(ora_vout) * (size_t)(nv > 0 ? nv : 1));
    int m = 0;
    for (int a = 0; a < nv;) {
        int b = a;
        double s[3] = {0, 0, 0};
        while (b < nv && v[b].k[0] == v[a].k[0] && v[b].k[1] == v[a].k[1] && v[b].k[2] == v[a].k[2]) {
            for (int d = 0; d < 3; ++d) s[d] += (double)xyz[3 * (int64_t)v[b].i + d];  /* index order */
            ++b;
        }
        o[m].first = v[a].i;
        o[m].cnt = b - a;
        for (int d = 0; d < 3; ++d) o[m].p[d] = (float)(s[d] / (double)(b - a));
        ++m;
        a = b;
    }
    qsort(o, (size_t)m, sizeof(ora_vout), ora_vout_cmp);
    for (int j = 0; j < m; ++j) {
        for (int d = 0; d < 3; ++d) out_xyz[3 * (int64_t)j + d] = o[j].p[d];
        cnt_out[j] = o[j].cnt;
    }
    free(v);
    free(o);
    return m;
}
