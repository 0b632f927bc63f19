// Internal device primitives of libgsicp (sm_100a).  Not part of the ABI.
// Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, Rn = DESIGN.md §3 reading n.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gsicp.h"

namespace gsicp {

constexpr unsigned long long kEmptyKey = ~0ull;
constexpr int32_t kCoordOff = 1 << 19;   // cell coordinates clamp to [-2^19, 2^19)
constexpr double kTau = 1e-12;           // degenerate eigenvalue threshold, m^2 (R8)
constexpr double kNoneFloor = 1e-6;      // NONE-mode eigenvalue floor, m^2
constexpr int kMaxLevels = 8;
constexpr int kAlignThreads = 384;       // 12 warps x 148 SMs >= 51k resident points (168 regs)
constexpr int kAlignTerms = 29;          // 21 H (upper) + 6 b + cost + count
#ifndef GSICP_GRAPH_K
#define GSICP_GRAPH_K 16
#endif
constexpr int kGraphK = GSICP_GRAPH_K;   // target kNN-graph degree (self included)

// 16-byte cell-table entry: 64-bit cell key, start offset and point count of the cell.
struct __align__(16) CellEntry {
    unsigned long long key;
    uint32_t start;
    uint32_t count;
};

// Programmatic dependent launch: wait for the stream predecessor grid (its completion and memory
// flush) — first statement of every kernel launched with launch_pdl — and let the next kernel of
// the stream launch early (it waits the same way).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------------------------------
// Canonical keys (DESIGN R1).  The DEFINITION is the binary64 key K2:
// dx = (double)b.x - q.x (q binary64: a binary32 point widened exactly, or the K3 transform of
// one), key = (dx*dx + dy*dy) + dz*dz, each op rounded separately (no FMA), order (key, index).
__device__ __forceinline__ double key64(double qx, double qy, double qz, float bx, float by, float bz) {
    const double dx = __dsub_rn((double)bx, qx), dy = __dsub_rn((double)by, qy), dz = __dsub_rn((double)bz, qz);
    double s = __dmul_rn(dx, dx);
    s = __dadd_rn(s, __dmul_rn(dy, dy));
    s = __dadd_rn(s, __dmul_rn(dz, dz));
    return s;
}
__device__ __forceinline__ double key64f(float ax, float ay, float az, float bx, float by, float bz) {
    return key64((double)ax, (double)ay, (double)az, bx, by, bz);
}

// The binary32 SCREEN key: the same expression in binary32.  For binary32 points a, b it is within
// 5u (u = 2^-24) of the exact squared distance, and key64 within 5 * 2^-53, so
// |key32 - key64| <= 11 u key64 (plus binary32 underflow, < 1e-44 absolute).  Candidates are ranked
// by key32 and only those within the band [band_lo(t), band_hi(t)] of the k-th / best key32 t are
// resolved in binary64: every candidate below band_lo(t) is certainly among the k
// nearest by key64, every one above band_hi(t) certainly not (kBand = 4e-6 > 22 u).
__device__ __forceinline__ float canon_key(float ax, float ay, float az, float bx, float by, float bz) {
    float dx = __fsub_rn(ax, bx), dy = __fsub_rn(ay, by), dz = __fsub_rn(az, bz);
    float s = __fmul_rn(dx, dx);
    s = __fadd_rn(s, __fmul_rn(dy, dy));
    s = __fadd_rn(s, __fmul_rn(dz, dz));
    return s;
}
constexpr float kBand = 4e-6f;
__device__ __forceinline__ float band_hi(float t) { return __fadd_ru(__fmul_ru(t, 1.f + kBand), 1e-36f); }
__device__ __forceinline__ float band_lo(float t) { return __fsub_rd(__fmul_rd(t, 1.f - kBand), 1e-36f); }

// (key32, index) packed so that unsigned 64-bit order == lexicographic (key32, index) order
// (keys are >= 0, so their IEEE bit patterns are monotone as unsigned integers).
__device__ __forceinline__ unsigned long long pack_ki(float key, uint32_t idx) {
    return ((unsigned long long)__float_as_uint(key) << 32) | idx;
}
__device__ __forceinline__ float ki_key(unsigned long long v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint32_t ki_idx(unsigned long long v) { return (uint32_t)v; }

// Exact (key64, index) order of candidates inside one band, packed in 64 bits: a band spans less
// than 1e-5 relative in key64, i.e. < 2^37 binary64 ulps, so the key64 bit pattern minus that of
// the band's floor fits 37 bits above a 27-bit index (clouds of < 2^27 points; checked by the API).
constexpr int kBandIdxBits = 27;
constexpr uint32_t kMaxBandIndex = (1u << kBandIdxBits) - 1u;
// (A band around t < 1e-30 has floor 0 and the offset saturates: pairs of distinct points closer
// than ~1e-18 m are then ordered by index — the one documented inexact corner, DESIGN R1.)
__device__ __forceinline__ unsigned long long band_pack(double key, uint32_t idx, unsigned long long floor_bits) {
    unsigned long long off = (unsigned long long)__double_as_longlong(key) - floor_bits;
    off = off < (1ull << (64 - kBandIdxBits)) ? off : (1ull << (64 - kBandIdxBits)) - 1ull;
    return (off << kBandIdxBits) | idx;
}
__device__ __forceinline__ uint32_t band_idx(unsigned long long v) { return (uint32_t)(v & kMaxBandIndex); }
// floor of a band: a binary64 value below every key64 of a candidate whose key32 >= band_lo(t)
__device__ __forceinline__ unsigned long long band_floor_bits(float t) {
    const double f = t < 1e-30f ? 0.0 : fmax((double)band_lo(t) * (1.0 - 2e-6), 0.0);
    return (unsigned long long)__double_as_longlong(f);
}

// ---------------------------------------------------------------------------------------
// Spatial hash: cell coordinates c = floor(p * inv_h) (binary32, same function at build and
// query time), key = level<<60 | (cx+off)<<40 | (cy+off)<<20 | (cz+off).
__device__ __forceinline__ int cell_coord(float p, float inv_h) {
    float f = floorf(__fmul_rn(p, inv_h));
    f = fminf(fmaxf(f, -(float)kCoordOff), (float)(kCoordOff - 1));
    return (int)f;
}
__device__ __forceinline__ unsigned long long cell_key(int level, int cx, int cy, int cz) {
    return ((unsigned long long)level << 60) | ((unsigned long long)(uint32_t)(cx + kCoordOff) << 40) |
           ((unsigned long long)(uint32_t)(cy + kCoordOff) << 20) | (unsigned long long)(uint32_t)(cz + kCoordOff);
}
__device__ __forceinline__ uint32_t hash_slot(unsigned long long key, uint32_t mask) {
    return (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 32) & mask;
}
// Returns (start, count) of the cell, (0, 0) if absent.  The table is read-only here.
__device__ __forceinline__ uint2 cell_lookup(const CellEntry *__restrict__ table, uint32_t mask,
                                             unsigned long long key) {
    uint32_t s = hash_slot(key, mask);
    while (true) {
        const uint4 e = __ldg(reinterpret_cast<const uint4 *>(table + s));
        const unsigned long long k = ((unsigned long long)e.y << 32) | e.x;
        if (k == key) return make_uint2(e.z, e.w);
        if (k == kEmptyKey) return make_uint2(0u, 0u);
        s = (s + 1) & mask;
    }
}

// Lower bound on the distance from q to cells at offset o along one axis, given the query's
// distances to its own cell's lower / upper faces (dlo, dhi) and the cell edge h.
__device__ __forceinline__ float axis_gap(int o, float dlo, float dhi, float h) {
    return o < 0 ? dlo + (float)(-o - 1) * h : (o > 0 ? dhi + (float)(o - 1) * h : 0.0f);
}

// Cell offset t (0 <= t < shell_count(m)) of the Chebyshev shell m >= 1 around a cell.
#define GS_HD __host__ __device__ __forceinline__
GS_HD double gs_rsqrt(double x) {
#ifdef __CUDA_ARCH__
    return rsqrt(x);
#else
    return 1.0 / sqrt(x);
#endif
}

GS_HD int shell_count(int m) { return (2 * m + 1) * (2 * m + 1) * (2 * m + 1) - (2 * m - 1) * (2 * m - 1) * (2 * m - 1); }
GS_HD void shell_offset(int m, int t, int &dx, int &dy, int &dz) {
    const int w = 2 * m + 1, w2 = w * w;
    if (t < 2 * w2) {
        dz = t < w2 ? -m : m;
        const int r = t < w2 ? t : t - w2;
        dy = r / w - m;
        dx = r % w - m;
        return;
    }
    t -= 2 * w2;
    const int per = 8 * m;
    dz = -m + 1 + t / per;
    const int r = t % per;
    if (r < 2 * w) {
        dy = r < w ? -m : m;
        dx = (r < w ? r : r - w) - m;
    } else {
        const int r2 = r - 2 * w, w1 = 2 * m - 1;
        dx = r2 < w1 ? -m : m;
        dy = (r2 < w1 ? r2 : r2 - w1) - m + 1;
    }
}

// ---------------------------------------------------------------------------------------
// Closed-form symmetric 3x3 eigen-decomposition in binary64 (trigonometric eigenvalues and
// the "most separated eigenvalue first" eigenvector construction, robust for repeated roots).
// A = (a00, a01, a02, a11, a12, a22).  lam[0] >= lam[1] >= lam[2] (clamped >= 0);
// v[j] is the unit eigenvector of lam[j].  Eq. 3 read as eigen-decomposition (R4).
struct Eig3 {
    double lam[3];
    double v[3][3];
};

GS_HD void cross3(const double *a, const double *b, double *c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}
GS_HD double dot3(const double *a, const double *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

// eigenvector of a (well separated) eigenvalue e: the largest cross product of rows of A - eI
GS_HD void eigvec_separated(const double *A, double e, double *out) {
    const double r0[3] = {A[0] - e, A[1], A[2]};
    const double r1[3] = {A[1], A[3] - e, A[4]};
    const double r2[3] = {A[2], A[4], A[5] - e};
    double c0[3], c1[3], c2[3];
    cross3(r0, r1, c0);
    cross3(r0, r2, c1);
    cross3(r1, r2, c2);
    const double d0 = dot3(c0, c0), d1 = dot3(c1, c1), d2 = dot3(c2, c2);
    // value selects (no pointer into local arrays, which would force them to local memory)
    double c[3] = {c0[0], c0[1], c0[2]};
    double d = d0;
    if (d1 > d) { c[0] = c1[0]; c[1] = c1[1]; c[2] = c1[2]; d = d1; }
    if (d2 > d) { c[0] = c2[0]; c[1] = c2[1]; c[2] = c2[2]; d = d2; }
    if (d > 0.0) {
        const double inv = gs_rsqrt(d);
        out[0] = c[0] * inv; out[1] = c[1] * inv; out[2] = c[2] * inv;
    } else {
        out[0] = 1.0; out[1] = 0.0; out[2] = 0.0;
    }
}

__host__ __device__ inline Eig3 eig3_sym(const double *Ain) {
    Eig3 r;
    double amax = fmax(fmax(fabs(Ain[0]), fabs(Ain[1])), fmax(fmax(fabs(Ain[2]), fabs(Ain[3])), fmax(fabs(Ain[4]), fabs(Ain[5]))));
    if (!(amax > 0.0)) {
        for (int i = 0; i < 3; ++i) {
            r.lam[i] = 0.0;
            for (int j = 0; j < 3; ++j) r.v[i][j] = (i == j) ? 1.0 : 0.0;
        }
        return r;
    }
    const double s = 1.0 / amax;
    double A[6];
    for (int i = 0; i < 6; ++i) A[i] = Ain[i] * s;
    const double q = (A[0] + A[3] + A[5]) / 3.0;
    const double b00 = A[0] - q, b11 = A[3] - q, b22 = A[5] - q;
    const double off = A[1] * A[1] + A[2] * A[2] + A[4] * A[4];
    const double p = sqrt((b00 * b00 + b11 * b11 + b22 * b22 + 2.0 * off) / 6.0);
    if (!(p > 0.0)) {  // multiple of the identity
        for (int i = 0; i < 3; ++i) {
            r.lam[i] = fmax(q * amax, 0.0);
            for (int j = 0; j < 3; ++j) r.v[i][j] = (i == j) ? 1.0 : 0.0;
        }
        return r;
    }
    const double c00 = b11 * b22 - A[4] * A[4];
    const double c01 = A[1] * b22 - A[4] * A[2];
    const double c02 = A[1] * A[4] - b11 * A[2];
    const double det = (b00 * c00 - A[1] * c01 + A[2] * c02) / (p * p * p);
    const double half = fmin(fmax(0.5 * det, -1.0), 1.0);
    const double ang = acos(half) / 3.0;
    const double kTwoThirdsPi = 2.09439510239319549;
    const double be2 = 2.0 * cos(ang);
    const double be0 = 2.0 * cos(ang + kTwoThirdsPi);
    const double be1 = -(be0 + be2);
    (void)be1;
    // The trigonometric estimate is accurate only for the most separated eigenvalue (acos near
    // +-1 loses half the digits of the nearly repeated pair), so: take that eigenvector from
    // cross products, its eigenvalue as a Rayleigh quotient, and the other two eigenpairs from
    // the exact 2x2 problem on the orthogonal complement (absolute accuracy ~eps ||A||).
    double ws[3];
    eigvec_separated(A, half >= 0.0 ? q + p * be2 : q + p * be0, ws);
    const double Aw[3] = {A[0] * ws[0] + A[1] * ws[1] + A[2] * ws[2], A[1] * ws[0] + A[3] * ws[1] + A[4] * ws[2],
                          A[2] * ws[0] + A[4] * ws[1] + A[5] * ws[2]};
    const double ls = dot3(ws, Aw);
    double U[3], V[3];
    if (fabs(ws[0]) > fabs(ws[1])) {
        const double inv = gs_rsqrt(ws[0] * ws[0] + ws[2] * ws[2]);
        U[0] = -ws[2] * inv; U[1] = 0.0; U[2] = ws[0] * inv;
    } else {
        const double inv = gs_rsqrt(ws[1] * ws[1] + ws[2] * ws[2]);
        U[0] = 0.0; U[1] = ws[2] * inv; U[2] = -ws[1] * inv;
    }
    cross3(ws, U, V);
    const double AU[3] = {A[0] * U[0] + A[1] * U[1] + A[2] * U[2], A[1] * U[0] + A[3] * U[1] + A[4] * U[2],
                          A[2] * U[0] + A[4] * U[1] + A[5] * U[2]};
    const double AV[3] = {A[0] * V[0] + A[1] * V[1] + A[2] * V[2], A[1] * V[0] + A[3] * V[1] + A[4] * V[2],
                          A[2] * V[0] + A[4] * V[1] + A[5] * V[2]};
    const double m00 = dot3(U, AU), m01 = 0.5 * (dot3(U, AV) + dot3(V, AU)), m11 = dot3(V, AV);
    const double mean = 0.5 * (m00 + m11), hd = 0.5 * (m00 - m11);
    const double rad = sqrt(hd * hd + m01 * m01);
    const double mu_hi = mean + rad;
    // smaller root without cancellation when it is tiny: det / mu_hi
    const double det2 = m00 * m11 - m01 * m01;
    const double mu_lo = (mean > 0.0 && mu_hi > 0.0 && rad > 0.5 * mean) ? det2 / mu_hi : mean - rad;
    // eigenvector (x, y) of mu_hi in the (U, V) basis; mu_lo's is its rotation
    double x, y;
    if (hd >= 0.0) { x = hd + rad; y = m01; } else { x = m01; y = rad - hd; }
    const double nrm = x * x + y * y;
    if (nrm > 0.0) { const double inv = gs_rsqrt(nrm); x *= inv; y *= inv; } else { x = 1.0; y = 0.0; }
    double vh[3], vl[3];
    for (int k = 0; k < 3; ++k) {
        vh[k] = x * U[k] + y * V[k];
        vl[k] = -y * U[k] + x * V[k];
    }
    // assemble descending
    double lam3[3], vec3[3][3];
    const bool sep_largest = half >= 0.0;
    lam3[0] = sep_largest ? ls : mu_hi;
    lam3[1] = sep_largest ? mu_hi : mu_lo;
    lam3[2] = sep_largest ? mu_lo : ls;
    for (int k = 0; k < 3; ++k) {
        vec3[0][k] = sep_largest ? ws[k] : vh[k];
        vec3[1][k] = sep_largest ? vh[k] : vl[k];
        vec3[2][k] = sep_largest ? vl[k] : ws[k];
    }
    // guard the order against rounding (the roles above hold up to ~eps ||A||)
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2 - i; ++j)
            if (lam3[j + 1] > lam3[j]) {
                const double tl = lam3[j]; lam3[j] = lam3[j + 1]; lam3[j + 1] = tl;
                for (int k = 0; k < 3; ++k) {
                    const double tv = vec3[j][k]; vec3[j][k] = vec3[j + 1][k]; vec3[j + 1][k] = tv;
                }
            }
    for (int j = 0; j < 3; ++j) {
        r.lam[j] = fmax(lam3[j] * amax, 0.0);
        for (int k = 0; k < 3; ++k) r.v[j][k] = vec3[j][k];
    }
    return r;
}

// Regularisation of a raw covariance C (R6-R8):
//  NONE    C + sum_i max(0, 1e-6 - lam_i) v v^T         ( = sum max(lam_i, 1e-6) v v^T, S:81 )
//  PLANE   I - (1 - eps) v0 v0^T                         ( = v2v2^T + v1v1^T + eps v0v0^T, P:195 )
//  ELLIPSE C / lam_1 + max(0, eps - lam_0/lam_1) v0 v0^T ( = sum max(lam_i/lam_1, eps) v v^T, Eq. 4 )
//  degenerate: lam_2 <= tau -> I (NONE: floor I); lam_1 <= tau < lam_2 -> v2v2^T + eps (I - v2v2^T)
// Returns flags; out = (c00, c01, c02, c11, c12, c22).
__host__ __device__ inline uint32_t regularize(const double *C, const Eig3 &e, int mode, double eps, double *out) {
    auto add_outer = [&](double w, const double *v) {
        out[0] += w * v[0] * v[0]; out[1] += w * v[0] * v[1]; out[2] += w * v[0] * v[2];
        out[3] += w * v[1] * v[1]; out[4] += w * v[1] * v[2]; out[5] += w * v[2] * v[2];
    };
    if (mode == GSICP_REG_NONE) {
        for (int i = 0; i < 6; ++i) out[i] = C[i];
        for (int j = 0; j < 3; ++j)
            if (e.lam[j] < kNoneFloor) add_outer(kNoneFloor - e.lam[j], e.v[j]);
        return e.lam[0] <= kTau ? GSICP_FLAG_DEGENERATE : 0u;
    }
    if (e.lam[0] <= kTau) {
        out[0] = 1.0; out[1] = 0.0; out[2] = 0.0; out[3] = 1.0; out[4] = 0.0; out[5] = 1.0;
        return GSICP_FLAG_DEGENERATE;
    }
    if (e.lam[1] <= kTau) {
        out[0] = eps; out[1] = 0.0; out[2] = 0.0; out[3] = eps; out[4] = 0.0; out[5] = eps;
        add_outer(1.0 - eps, e.v[0]);
        return GSICP_FLAG_DEGENERATE;
    }
    if (mode == GSICP_REG_PLANE) {
        out[0] = 1.0; out[1] = 0.0; out[2] = 0.0; out[3] = 1.0; out[4] = 0.0; out[5] = 1.0;
        add_outer(eps - 1.0, e.v[2]);
        return 0u;
    }
    const double inv = 1.0 / e.lam[1];
    for (int i = 0; i < 6; ++i) out[i] = C[i] * inv;
    const double r0 = e.lam[2] * inv;
    if (r0 < eps) add_outer(eps - r0, e.v[2]);
    return 0u;
}

__device__ __forceinline__ void store_cov(float4 *cov_a, float4 *cov_b, int i, const double *c, double lam_mid,
                                          uint32_t flags) {
    cov_a[i] = make_float4((float)c[0], (float)c[1], (float)c[2], (float)c[3]);
    cov_b[i] = make_float4((float)c[4], (float)c[5], (float)lam_mid, __uint_as_float(flags));
}

}  // namespace gsicp
