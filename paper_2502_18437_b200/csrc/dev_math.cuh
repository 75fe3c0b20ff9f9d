// dev_math.cuh — device-side math, SDF, contact and constitutive functions of the
// B200 MPM hot path.  Each function names the reference definition it reproduces
// (CRESSim-MPM CPU reference, proj/include/mpm/*.hpp).  Arithmetic is FP32 with
// FMA contraction allowed (tolerance-checked against the oracle) EXCEPT the
// stencil-base arithmetic, which uses explicit round-to-nearest intrinsics so the
// binning keys are bit-identical to the reference (math.hpp:219-223).
#pragma once
#include <cstdint>
#include <cfloat>

#include "dev_types.h"

namespace mpmb {

struct V3 { float x, y, z; };
struct M3 { float m[9]; };   // row-major, math.hpp:46-48
struct Q4 { float x, y, z, w; };

// Reference arithmetic: the contact / SDF / push-out / free-body path is evaluated
// without FMA contraction and in the reference's operation order (the x86-64 reference
// build has no FMA).  Rigid motions that are exactly tangential to a needle make the
// contact test v_n < 0 a rounding-level decision (tests/test_gpu_parity.py); matching
// the reference's rounding there is what keeps the device on the reference trajectory.
// The P2G/G2P transfer sums keep FMA: their order already differs (atomics).
#define FA __fadd_rn
#define FS __fsub_rn
#define FM __fmul_rn
#define FD __fdiv_rn

__device__ __forceinline__ V3 mk(float x, float y, float z) { return V3{x, y, z}; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return V3{FA(a.x, b.x), FA(a.y, b.y), FA(a.z, b.z)}; }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return V3{FS(a.x, b.x), FS(a.y, b.y), FS(a.z, b.z)}; }
__device__ __forceinline__ V3 operator-(V3 a) { return V3{-a.x, -a.y, -a.z}; }
__device__ __forceinline__ V3 operator*(V3 a, float s) { return V3{FM(a.x, s), FM(a.y, s), FM(a.z, s)}; }
__device__ __forceinline__ V3 vdiv(V3 a, float s) { return V3{FD(a.x, s), FD(a.y, s), FD(a.z, s)}; }
__device__ __forceinline__ float dot(V3 a, V3 b) {  // math.hpp:29
    return FA(FA(FM(a.x, b.x), FM(a.y, b.y)), FM(a.z, b.z));
}
__device__ __forceinline__ V3 cross(V3 a, V3 b) {  // math.hpp:30-32
    return V3{FS(FM(a.y, b.z), FM(a.z, b.y)), FS(FM(a.z, b.x), FM(a.x, b.z)),
              FS(FM(a.x, b.y), FM(a.y, b.x))};
}
__device__ __forceinline__ float norm2(V3 a) { return dot(a, a); }
__device__ __forceinline__ float norm(V3 a) { return __fsqrt_rn(norm2(a)); }
// float trig evaluated in FP64 and rounded once (matches glibc's float results except
// where glibc itself is not correctly rounded)
__device__ __forceinline__ float sin_ref(float x) { return static_cast<float>(sin(static_cast<double>(x))); }
__device__ __forceinline__ float cos_ref(float x) { return static_cast<float>(cos(static_cast<double>(x))); }
__device__ __forceinline__ float atan2_ref(float y, float x) {
    return static_cast<float>(atan2(static_cast<double>(y), static_cast<double>(x)));
}
// math.hpp:35-38
__device__ __forceinline__ V3 normalized(V3 a) {
    float n = norm(a);
    return n > 0.f ? vdiv(a, n) : V3{1.f, 0.f, 0.f};
}

// math.hpp:157-162
__device__ __forceinline__ V3 qrotate(Q4 q, V3 v) {
    V3 u{q.x, q.y, q.z};
    V3 t = cross(u, v) * 2.f;
    return v + t * q.w + cross(u, t);
}
__device__ __forceinline__ V3 qrotate_inv(Q4 q, V3 v) { return qrotate(Q4{-q.x, -q.y, -q.z, q.w}, v); }
// math.hpp:151-156
__device__ __forceinline__ Q4 qmul(Q4 a, Q4 o) {
    return Q4{FS(FA(FA(FM(a.w, o.x), FM(a.x, o.w)), FM(a.y, o.z)), FM(a.z, o.y)),
              FA(FA(FS(FM(a.w, o.y), FM(a.x, o.z)), FM(a.y, o.w)), FM(a.z, o.x)),
              FA(FS(FA(FM(a.w, o.z), FM(a.x, o.y)), FM(a.y, o.x)), FM(a.z, o.w)),
              FS(FS(FS(FM(a.w, o.w), FM(a.x, o.x)), FM(a.y, o.y)), FM(a.z, o.z))};
}
// math.hpp:144-149
__device__ __forceinline__ Q4 qnormalized(Q4 q) {
    float n = __fsqrt_rn(FA(FA(FA(FM(q.x, q.x), FM(q.y, q.y)), FM(q.z, q.z)), FM(q.w, q.w)));
    if (n <= 0.f) return Q4{0.f, 0.f, 0.f, 1.f};
    return Q4{FD(q.x, n), FD(q.y, n), FD(q.z, n), FD(q.w, n)};
}

// ---------------------------------------------------------------- spline (math.hpp)
// Stencil base and fractional coordinate, exactly the reference's P2G arithmetic
// (math.hpp:219-224): inv_dx = 1/dx (host-computed), p = (x - o) * inv_dx,
// base = (int)floor(p - 0.5), fx = p - base.  No contraction: bit-exact keys.
__device__ __forceinline__ int stencil_base(float x, float o, float inv_dx, float& fx) {
    float p = __fmul_rn(__fsub_rn(x, o), inv_dx);
    int base = static_cast<int>(floorf(__fsub_rn(p, 0.5f)));
    fx = __fsub_rn(p, static_cast<float>(base));
    return base;
}
// Quadratic B-spline weights (math.hpp:226-228).
__device__ __forceinline__ void bspline_w(float fx, float w[3]) {
    float a = 1.5f - fx, b = fx - 1.f, c = fx - 0.5f;
    w[0] = 0.5f * a * a;
    w[1] = 0.75f - b * b;
    w[2] = 0.5f * c * c;
}
// Interior band test, DIVIDING by dx (math.hpp:203-213) as deactivation does.
// in domain <=> 0.5 <= p < dims - 1.5 per axis; a multiply by 1/dx decides every particle
// farther than a safe margin from both thresholds, the exact division the rest.
template <class SceneT>
__device__ __forceinline__ bool spline_in_domain(V3 pos, const SceneT& S) {
    {
        const float d[3] = {__fsub_rn(pos.x, S.origin[0]), __fsub_rn(pos.y, S.origin[1]),
                            __fsub_rn(pos.z, S.origin[2])};
        bool inside = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float q = d[a] * S.inv_dx;
            const float eps = 1e-3f + 1e-5f * static_cast<float>(S.dims[a]);
            inside = inside && q > 0.5f + eps && q < static_cast<float>(S.dims[a]) - 1.5f - eps;
        }
        if (inside) return true;
    }
    const float p[3] = {__fdiv_rn(__fsub_rn(pos.x, S.origin[0]), S.dx),
                        __fdiv_rn(__fsub_rn(pos.y, S.origin[1]), S.dx),
                        __fdiv_rn(__fsub_rn(pos.z, S.origin[2]), S.dx)};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        int base = static_cast<int>(floorf(__fsub_rn(p[a], 0.5f)));
        if (base < 0 || base + 2 > S.dims[a] - 1) return false;
    }
    return true;
}

// ------------------------------------------------------------- matrices
__device__ __forceinline__ float det3(const float a[9]) {  // math.hpp:273-277
    return FA(FA(FM(a[0], FS(FM(a[4], a[8]), FM(a[5], a[7]))),
                 FM(a[1], FS(FM(a[5], a[6]), FM(a[3], a[8])))),
              FM(a[2], FS(FM(a[3], a[7]), FM(a[4], a[6]))));
}

// Cauchy stress (materials.hpp:35-54), FP64 internally, J clamped >= 1e-6.
// b = F F^T is symmetric; the 6 unique entries are computed once.
__device__ __forceinline__ void neo_hookean(const float F[9], float mu, float lambda, float s[9]) {
    // the reference's own operation order, every FP64 op round-to-nearest and unfused, and a
    // true division by Jc: bit-identical to the cached stress of solvers.hpp:69-74
    double f[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) f[i] = static_cast<double>(F[i]);
    const double J = __dadd_rn(
        __dsub_rn(__dmul_rn(f[0], __dsub_rn(__dmul_rn(f[4], f[8]), __dmul_rn(f[5], f[7]))),
                  __dmul_rn(f[1], __dsub_rn(__dmul_rn(f[3], f[8]), __dmul_rn(f[5], f[6])))),
        __dmul_rn(f[2], __dsub_rn(__dmul_rn(f[3], f[7]), __dmul_rn(f[4], f[6]))));
    const double Jc = J < 1e-6 ? 1e-6 : J;
    const double d = __dmul_rn(static_cast<double>(lambda), log(Jc));
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double b = __dadd_rn(__dadd_rn(__dmul_rn(f[3 * i], f[3 * j]), __dmul_rn(f[3 * i + 1], f[3 * j + 1])),
                                       __dmul_rn(f[3 * i + 2], f[3 * j + 2]));
            double v = __dmul_rn(static_cast<double>(mu), __dsub_rn(b, i == j ? 1.0 : 0.0));
            if (i == j) v = __dadd_rn(v, d);
            s[3 * i + j] = static_cast<float>(__ddiv_rn(v, Jc));
        }
}

// The same Cauchy stress in FP32 without cancellation, for the P2G hot loop:
//   F F^T - I = H + H^T + H H^T   and   J - 1 = tr H + (principal 2x2 minors of H) + det H
// with H = F - I (exact for F near I), ln J = log1p(J - 1).  The reference evaluates in
// FP64 because the float difference F F^T - I cancels (materials.hpp:29-34); this form
// has no such difference, and agrees with the FP64 value to a few float ulps.  Away from
// F = I (|J - 1| >= 0.5) J is the cofactor determinant of F, clamped at 1e-6 exactly as the
// reference (materials.hpp:42); tests/test_gpu_stress_kat.py pins both branches.
// Far from F = I the H-expansion sums O(1) terms of opposite sign (F = 0.01 I: tr H + minors +
// det H = -2.97 + 2.94 - 0.97), which loses J near the 1e-6 clamp; the cofactor determinant of
// F itself is exact there (products of the small entries).
// (by value both ways: the out-of-line call stays in registers)
static __device__ __noinline__ float3 neo_hookean_far(float f0, float f1, float f2, float f3, float f4, float f5, float f6,
                                               float f7, float f8) {
    const float J = fmaf(f0, fmaf(f4, f8, -f5 * f7), fmaf(-f1, fmaf(f3, f8, -f5 * f6), f2 * fmaf(f3, f7, -f4 * f6)));
    const float Jc = J < 1e-6f ? 1e-6f : J;  // materials.hpp:42
    return make_float3(J, logf(Jc), 1.f / Jc);
}

__device__ __forceinline__ float neo_hookean_f32(const float F[9], float mu, float lambda, float s[9]) {
    const float h0 = F[0] - 1.f, h1 = F[1], h2 = F[2];
    const float h3 = F[3], h4 = F[4] - 1.f, h5 = F[5];
    const float h6 = F[6], h7 = F[7], h8 = F[8] - 1.f;
    const float m2 = fmaf(h0, h4, -h1 * h3) + fmaf(h0, h8, -h2 * h6) + fmaf(h4, h8, -h5 * h7);
    const float dh = h0 * fmaf(h4, h8, -h5 * h7) + h1 * fmaf(h5, h6, -h3 * h8) + h2 * fmaf(h3, h7, -h4 * h6);
    const float j1 = (h0 + h4 + h8) + m2 + dh;
    float J, lnJ, invJ;
#ifndef MPMB_STRESS_FAR_OUTLINE
#define MPMB_STRESS_FAR_OUTLINE 1
#endif
    if (__builtin_expect(fabsf(j1) < 0.5f, 1)) {  // near F = I: J - 1 without cancellation
        J = 1.f + j1;
        lnJ = log1pf(j1);
        invJ = 1.f / J;
    } else {
        // out of line: the hot loop keeps one branch
        float3 r;
        if (MPMB_STRESS_FAR_OUTLINE) {
            r = neo_hookean_far(F[0], F[1], F[2], F[3], F[4], F[5], F[6], F[7], F[8]);
        } else {
            const float Jd = fmaf(F[0], fmaf(F[4], F[8], -F[5] * F[7]),
                                  fmaf(-F[1], fmaf(F[3], F[8], -F[5] * F[6]), F[2] * fmaf(F[3], F[7], -F[4] * F[6])));
            const float Jc = Jd < 1e-6f ? 1e-6f : Jd;
            r = make_float3(Jd, logf(Jc), 1.f / Jc);
        }
        J = r.x;
        lnJ = r.y;
        invJ = r.z;
    }
    const float d = lambda * lnJ;
    // (b - I)_ij = h_ij + h_ji + sum_k h_ik h_jk
    const float b00 = 2.f * h0 + fmaf(h0, h0, fmaf(h1, h1, h2 * h2));
    const float b11 = 2.f * h4 + fmaf(h3, h3, fmaf(h4, h4, h5 * h5));
    const float b22 = 2.f * h8 + fmaf(h6, h6, fmaf(h7, h7, h8 * h8));
    const float b01 = (h1 + h3) + fmaf(h0, h3, fmaf(h1, h4, h2 * h5));
    const float b02 = (h2 + h6) + fmaf(h0, h6, fmaf(h1, h7, h2 * h8));
    const float b12 = (h5 + h7) + fmaf(h3, h6, fmaf(h4, h7, h5 * h8));
    s[0] = fmaf(mu, b00, d) * invJ;
    s[4] = fmaf(mu, b11, d) * invJ;
    s[8] = fmaf(mu, b22, d) * invJ;
    s[1] = s[3] = mu * b01 * invJ;
    s[2] = s[6] = mu * b02 * invJ;
    s[5] = s[7] = mu * b12 * invJ;
    return J;
}

// Scaled-Newton polar decomposition in FP64 (math.hpp:286-340); returns R only
// (U is not used by the projection).  false on failure.
__device__ __forceinline__ bool polar_R(const float m[9], float R[9]) {
#pragma unroll
    for (int i = 0; i < 9; ++i)
        if (!isfinite(m[i])) return false;
    if (det3(m) <= 0.f) return false;
    double x[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) x[i] = m[i];
    for (int iter = 0; iter < 50; ++iter) {
        double d = x[0] * (x[4] * x[8] - x[5] * x[7]) + x[1] * (x[5] * x[6] - x[3] * x[8]) +
                   x[2] * (x[3] * x[7] - x[4] * x[6]);
        if (!(d > 0.0) || !isfinite(d)) return false;
        double id = 1.0 / d;
        double it[9];
        it[0] = (x[4] * x[8] - x[5] * x[7]) * id;
        it[1] = (x[5] * x[6] - x[3] * x[8]) * id;
        it[2] = (x[3] * x[7] - x[4] * x[6]) * id;
        it[3] = (x[2] * x[7] - x[1] * x[8]) * id;
        it[4] = (x[0] * x[8] - x[2] * x[6]) * id;
        it[5] = (x[1] * x[6] - x[0] * x[7]) * id;
        it[6] = (x[1] * x[5] - x[2] * x[4]) * id;
        it[7] = (x[2] * x[3] - x[0] * x[5]) * id;
        it[8] = (x[0] * x[4] - x[1] * x[3]) * id;
        double nx = 0.0, ni = 0.0;
#pragma unroll
        for (int i = 0; i < 9; ++i) {
            nx += x[i] * x[i];
            ni += it[i] * it[i];
        }
        double gamma = sqrt(sqrt(ni / nx));
        double ig = 1.0 / gamma;
        double delta = 0.0;
#pragma unroll
        for (int i = 0; i < 9; ++i) {
            double next = 0.5 * (gamma * x[i] + it[i] * ig);
            double diff = next - x[i];
            delta += diff * diff;
            x[i] = next;
        }
        if (delta < 1e-16) break;  // sqrt(delta) < 1e-8
    }
#pragma unroll
    for (int i = 0; i < 9; ++i) R[i] = static_cast<float>(x[i]);
    return true;
}

// Co-rotational projection (materials.hpp:59-72).
__device__ __forceinline__ bool corotational_project(const float Fp[9], const float Cc[9], float dt,
                                                     float beta, float out[9]) {
    if (dt <= 0.f) return false;
    float A[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) A[i] = Cc[i] * dt + ((i % 4) == 0 ? 1.f : 0.f);
    float Ft[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            Ft[3 * i + j] = A[3 * i] * Fp[j] + A[3 * i + 1] * Fp[3 + j] + A[3 * i + 2] * Fp[6 + j];
    float R[9];
    if (!polar_R(Ft, R)) return false;
    float dtr = det3(Ft);
    if (!(dtr > 0.f)) return false;
    float s = (1.f - beta) / dtr;
    float Fq[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) Fq[i] = R[i] * beta + Ft[i] * s;
    // inverse of F_prev (math.hpp:252-271)
    const float c00 = Fp[4] * Fp[8] - Fp[5] * Fp[7];
    const float c01 = Fp[5] * Fp[6] - Fp[3] * Fp[8];
    const float c02 = Fp[3] * Fp[7] - Fp[4] * Fp[6];
    float det = Fp[0] * c00 + Fp[1] * c01 + Fp[2] * c02;
    if (fabsf(det) <= 1e-12f) return false;
    float idt = 1.f / det;
    float inv[9];
    inv[0] = c00 * idt;
    inv[3] = c01 * idt;
    inv[6] = c02 * idt;
    inv[1] = (Fp[2] * Fp[7] - Fp[1] * Fp[8]) * idt;
    inv[4] = (Fp[0] * Fp[8] - Fp[2] * Fp[6]) * idt;
    inv[7] = (Fp[1] * Fp[6] - Fp[0] * Fp[7]) * idt;
    inv[2] = (Fp[1] * Fp[5] - Fp[2] * Fp[4]) * idt;
    inv[5] = (Fp[2] * Fp[3] - Fp[0] * Fp[5]) * idt;
    inv[8] = (Fp[0] * Fp[4] - Fp[1] * Fp[3]) * idt;
    float idtt = 1.f / dt;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            float v = Fq[3 * i] * inv[j] + Fq[3 * i + 1] * inv[3 + j] + Fq[3 * i + 2] * inv[6 + j];
            out[3 * i + j] = (v - (i == j ? 1.f : 0.f)) * idtt;
        }
    return true;
}

// ------------------------------------------------------------------- SDF (geometry.hpp)
struct Sdf {
    float distance;
    V3 normal;
    V3 tangent;
    int region;
};

__device__ __forceinline__ float clampf(float v, float lo, float hi) {
    return v < lo ? lo : (hi < v ? hi : v);
}

// geometry.hpp:204-213
__device__ __forceinline__ V3 closest_on_segment(V3 a, V3 b, V3 p, float& t) {
    V3 ab = b - a;
    float len2 = norm2(ab);
    t = len2 > 1e-18f ? clampf(FD(dot(p - a, ab), len2), 0.f, 1.f) : 0.f;
    return a + ab * t;
}

// geometry.hpp:217-242
__device__ __forceinline__ V3 closest_on_triangle(V3 a, V3 b, V3 c, V3 p) {
    V3 ab = b - a, ac = c - a, ap = p - a;
    float d1 = dot(ab, ap), d2 = dot(ac, ap);
    if (d1 <= 0.f && d2 <= 0.f) return a;
    V3 bp = p - b;
    float d3 = dot(ab, bp), d4 = dot(ac, bp);
    if (d3 >= 0.f && d4 <= d3) return b;
    float vc = FS(FM(d1, d4), FM(d3, d2));
    if (vc <= 0.f && d1 >= 0.f && d3 <= 0.f) return a + ab * FD(d1, d1 - d3);
    V3 cp = p - c;
    float d5 = dot(ab, cp), d6 = dot(ac, cp);
    if (d6 >= 0.f && d5 <= d6) return c;
    float vb = FS(FM(d5, d2), FM(d1, d6));
    if (vb <= 0.f && d2 >= 0.f && d6 <= 0.f) return a + ac * FD(d2, d2 - d6);
    float va = FS(FM(d3, d6), FM(d5, d4));
    if (va <= 0.f && (d4 - d3) >= 0.f && (d5 - d6) >= 0.f) {
        float w = FD(d4 - d3, FA(d4 - d3, d5 - d6));
        return b + (c - b) * w;
    }
    float denom = FD(1.f, FA(FA(va, vb), vc));
    return a + ab * FM(vb, denom) + ac * FM(vc, denom);
}

// False when the point is provably outside every contact / push-out band of the shape
// (DevShape::lbox, tested in the shape's frame); the reference's query would return no
// effect there.  The substep pipeline uses the precomputed world boxes (cull_may_touch).
__device__ __forceinline__ bool shape_may_touch(const DevShape& g, const DevPose& pose, V3 point) {
    if (g.lbox_h[0] < 0.f) return true;
    Q4 q{pose.rot[0], pose.rot[1], pose.rot[2], pose.rot[3]};
    const V3 p = qrotate_inv(q, point - mk(pose.pos[0], pose.pos[1], pose.pos[2]));
    const float m = 1.001f;
    return fabsf(p.x - g.lbox_c[0]) <= g.lbox_h[0] * m + 1e-5f && fabsf(p.y - g.lbox_c[1]) <= g.lbox_h[1] * m + 1e-5f &&
           fabsf(p.z - g.lbox_c[2]) <= g.lbox_h[2] * m + 1e-5f;
}

// World-space SDF query (geometry.hpp:370-395) against one device shape.
__device__ inline Sdf sdf_query(const DevShape& g, const DevPose& pose, const float* verts,
                                const int* ints, V3 point) {
    Q4 q{pose.rot[0], pose.rot[1], pose.rot[2], pose.rot[3]};
    V3 p = qrotate_inv(q, point - mk(pose.pos[0], pose.pos[1], pose.pos[2]));
    Sdf s;
    s.distance = 0.f;
    s.normal = mk(1.f, 0.f, 0.f);
    s.tangent = mk(0.f, 1.f, 0.f);
    s.region = REGION_BULK;
    switch (g.geom) {
        case GEOM_PLANE:  // geometry.hpp:136-142
            s.distance = p.y;
            s.normal = mk(0.f, 1.f, 0.f);
            s.region = REGION_SURFACE;
            break;
        case GEOM_SPHERE: {  // geometry.hpp:144-151
            float r = norm(p);
            s.distance = r - g.gp[0];
            s.normal = r > 1e-9f ? vdiv(p, r) : mk(1.f, 0.f, 0.f);
            s.region = REGION_SURFACE;
            break;
        }
        case GEOM_BOX: {  // geometry.hpp:153-176
            s.region = REGION_SURFACE;
            V3 h = mk(g.gp[0], g.gp[1], g.gp[2]);
            V3 qv = mk(fabsf(p.x) - h.x, fabsf(p.y) - h.y, fabsf(p.z) - h.z);
            float qmax = qv.x;
            if (qmax < qv.y) qmax = qv.y;
            if (qmax < qv.z) qmax = qv.z;
            if (qmax <= 0.f) {
                s.distance = qmax;
                if (qv.x >= qv.y && qv.x >= qv.z)
                    s.normal = mk(p.x >= 0.f ? 1.f : -1.f, 0.f, 0.f);
                else if (qv.y >= qv.z)
                    s.normal = mk(0.f, p.y >= 0.f ? 1.f : -1.f, 0.f);
                else
                    s.normal = mk(0.f, 0.f, p.z >= 0.f ? 1.f : -1.f);
            } else {
                V3 cl = mk(clampf(p.x, -h.x, h.x), clampf(p.y, -h.y, h.y), clampf(p.z, -h.z, h.z));
                V3 d = p - cl;
                s.distance = norm(d);
                s.normal = s.distance > 1e-9f ? vdiv(d, s.distance) : mk(1.f, 0.f, 0.f);
            }
            break;
        }
        case GEOM_QUAD_SLICER: {  // geometry.hpp:178-202
            const float hl = g.gp[0], hh = g.gp[1], sr = g.gp[2];
            if (p.y >= hh) {
                V3 axis = mk(clampf(p.x, -hl, hl), hh, 0.f);
                V3 d = p - axis;
                float r = norm(d);
                s.distance = r - sr;
                s.normal = r > 1e-9f ? vdiv(d, r) : mk(0.f, 1.f, 0.f);
                s.region = REGION_SPINE;
            } else if (fabsf(p.x) <= hl && p.y >= -hh) {
                s.distance = p.z;
                s.normal = mk(0.f, 0.f, p.z >= 0.f ? 1.f : -1.f);
                s.region = REGION_EDGE;
            } else {
                s.region = REGION_BULK;
                s.distance = FLT_MAX;
            }
            break;
        }
        case GEOM_TRI_MESH_SLICER: {  // geometry.hpp:244-293
            const V3* vt = reinterpret_cast<const V3*>(verts) + g.vtx_begin;
            const int* sp = ints + g.spine_begin;
            const int* ix = ints + g.idx_begin;
            float best_spine = FLT_MAX;
            V3 spine_pt = mk(0.f, 0.f, 0.f);
            for (int e = 0; e + 1 < g.n_spine; e += 2) {
                float t;
                V3 qq = closest_on_segment(vt[sp[e]], vt[sp[e + 1]], p, t);
                float d = norm(p - qq);
                if (d < best_spine) { best_spine = d; spine_pt = qq; }
            }
            float best_surf = FLT_MAX;
            V3 surf_pt = mk(0.f, 0.f, 0.f), surf_n = mk(0.f, 0.f, 0.f);
            for (int t = 0; t + 2 < g.n_idx; t += 3) {
                V3 a = vt[ix[t]], b = vt[ix[t + 1]], c = vt[ix[t + 2]];
                V3 qq = closest_on_triangle(a, b, c, p);
                float d = norm(p - qq);
                if (d < best_surf) {
                    best_surf = d;
                    surf_pt = qq;
                    surf_n = normalized(cross(b - a, c - a));
                }
            }
            if (best_spine <= best_surf + 1e-9f && best_spine < FLT_MAX) {
                V3 d = p - spine_pt;
                float r = norm(d);
                s.distance = r - g.gp[0];
                s.normal = r > 1e-9f ? vdiv(d, r) : mk(0.f, 1.f, 0.f);
                s.region = REGION_SPINE;
            } else {
                float side = dot(p - surf_pt, surf_n) >= 0.f ? 1.f : -1.f;
                s.distance = FM(side, best_surf);
                s.normal = surf_n * side;
                s.region = REGION_EDGE;
            }
            break;
        }
        case GEOM_ARC: {  // geometry.hpp:295-327
            const float kTwoPi = 6.28318548f;  // float(2*pi), as Real(2*3.14159...)
            float t;
            if (norm(mk(p.x, p.y, 0.f)) < 1e-9f) {
                t = 0.f;
            } else {
                t = atan2_ref(p.y, p.x);
                if (t < 0.f) t += kTwoPi;
                if (t > g.gp[1]) {
                    float to_end = t - g.gp[1];
                    float to_start = kTwoPi - t;
                    t = to_end <= to_start ? g.gp[1] : 0.f;
                }
            }
            const float st = sin_ref(t), ct = cos_ref(t);
            V3 qq = mk(FM(g.gp[0], ct), FM(g.gp[0], st), 0.f);
            s.region = REGION_CURVE;
            s.tangent = mk(-st, ct, 0.f);
            V3 d = p - qq;
            float dist = norm(d);
            s.distance = dist;
            s.normal = dist < 1e-9f ? mk(-ct, -st, 0.f) : vdiv(d, dist);
            break;
        }
        default: {  // GEOM_POLYLINE, geometry.hpp:329-365
            const V3* vt = reinterpret_cast<const V3*>(verts) + g.vtx_begin;
            const int nv = g.n_vtx;
            float best = FLT_MAX;
            V3 best_pt = mk(0.f, 0.f, 0.f), best_tan = mk(1.f, 0.f, 0.f);
            for (int i = 0; i + 1 < nv; ++i) {
                float t;
                V3 qq = closest_on_segment(vt[i], vt[i + 1], p, t);
                float d = norm(p - qq);
                if (d < best) {
                    best = d;
                    best_pt = qq;
                    V3 dir = normalized(vt[i + 1] - vt[i]);
                    if (t <= 1e-6f && i > 0) {
                        V3 prev = normalized(vt[i] - vt[i - 1]);
                        dir = normalized(dir + prev);
                    } else if (t >= 1.f - 1e-6f && i + 2 < nv) {
                        V3 next = normalized(vt[i + 2] - vt[i + 1]);
                        dir = normalized(dir + next);
                    }
                    best_tan = dir;
                }
            }
            s.region = REGION_CURVE;
            s.tangent = best_tan;
            s.distance = best;
            if (best < 1e-9f) {
                V3 ref = fabsf(best_tan.x) < 0.9f ? mk(1.f, 0.f, 0.f) : mk(0.f, 1.f, 0.f);
                s.normal = normalized(cross(best_tan, ref));
            } else {
                s.normal = vdiv(p - best_pt, best);
            }
            break;
        }
    }
    s.normal = qrotate(q, s.normal);
    s.tangent = qrotate(q, s.tangent);
    return s;
}

// geometry.hpp:29-32
__device__ __forceinline__ V3 rigid_point_velocity(const DevPose& pose, V3 p) {
    V3 w = mk(pose.ang[0], pose.ang[1], pose.ang[2]);
    return mk(pose.lin[0], pose.lin[1], pose.lin[2]) +
           cross(w, p - mk(pose.pos[0], pose.pos[1], pose.pos[2]));
}

// contact.hpp:82-92
__device__ __forceinline__ bool node_in_contact(const Sdf& s, float hw) {
    switch (s.region) {
        case REGION_SURFACE: return s.distance < 0.f;
        case REGION_EDGE: return fabsf(s.distance) < hw;
        case REGION_SPINE: return s.distance < 0.f;
        case REGION_CURVE: return s.distance < hw;
        default: return false;
    }
}

// contact.hpp:33-38
__device__ __forceinline__ float friction_drag(float vn, float vtg, float mu_k, float c_d) {
    if (vtg < 1e-12f) return 0.f;
    float f = FS(1.f, FD(FM(mu_k, vn), vtg));
    return FM(c_d, fmaxf(f, 0.f));
}

// One shape's grid correction (contact.hpp:106-133): returns the corrected velocity
// and sets delta (zero when the node is untouched).
__device__ __forceinline__ V3 contact_correct(const DevShape& g, const Sdf& s, V3 vnode, V3 vrig,
                                              V3& delta) {
    if (s.region == REGION_SPINE) {  // contact.hpp:77-80 sticky
        delta = vrig - vnode;
        return vrig;
    }
    V3 vrel = vnode - vrig;
    float vn = dot(vrel, s.normal);
    if (vn >= 0.f) {
        delta = mk(0.f, 0.f, 0.f);
        return vnode;
    }
    V3 vt;
    if (s.region == REGION_CURVE)  // contact.hpp:60-74
        vt = s.tangent * dot(vrel, s.tangent);
    else  // contact.hpp:43-56
        vt = vrel - s.normal * vn;
    float tg = norm(vt);
    V3 vc = vrig + vt * friction_drag(-vn, tg, g.mu_k, g.c_d);
    delta = vc - vnode;
    return vc;
}

}  // namespace mpmb
