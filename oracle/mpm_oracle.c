/*
 * mpm_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference
 * MPM hot path (CRESSim-MPM CPU reference, /root/reference/proj/include/mpm).
 *
 * Each function cites the reference file:line it restates ("ref: file:lines").
 * Operation order, float/double types and constants follow the reference exactly;
 * build with -O2 -ffp-contract=off (no -march, no -ffast-math) so that the result
 * is bit-identical to the reference compiled by g++ on x86-64 (no FMA).
 * Parity pinned by tests/test_oracle_pin.py (vs oracle/_ref) and tests/golden/.
 *
 * This file is the checker.  It is never linked into the product library.
 */
#include "mpm_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ math.hpp */
typedef struct { float x, y, z; } V3;
typedef struct { float m[3][3]; } M3;
typedef struct { float x, y, z, w; } Q4;

static V3 v3(float x, float y, float z) { V3 r = {x, y, z}; return r; }
static V3 v3p(const float* p) { return v3(p[0], p[1], p[2]); }
static void v3put(float* o, V3 v) { o[0] = v.x; o[1] = v.y; o[2] = v.z; }
/* ref: math.hpp:20-33 */
static V3 vadd(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
static V3 vsub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
static V3 vneg(V3 a) { return v3(-a.x, -a.y, -a.z); }
static V3 vmul(V3 a, float s) { return v3(a.x * s, a.y * s, a.z * s); }
static V3 vdiv(V3 a, float s) { return v3(a.x / s, a.y / s, a.z / s); }
static float vdot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static V3 vcross(V3 a, V3 b) {
    return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static float vnorm2(V3 a) { return vdot(a, a); }
static float vnorm(V3 a) { return sqrtf(vnorm2(a)); }
/* ref: math.hpp:35-38 */
static V3 vnormalized(V3 a) {
    float n = vnorm(a);
    return n > 0.0f ? vdiv(a, n) : v3(1, 0, 0);
}
static int visfinite(V3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }

/* ref: math.hpp:50-130 */
static M3 mzero(void) { M3 r; memset(&r, 0, sizeof r); return r; }
static M3 mident(void) { M3 r = mzero(); r.m[0][0] = r.m[1][1] = r.m[2][2] = 1; return r; }
static M3 mdiag(float a, float b, float c) {
    M3 r = mzero(); r.m[0][0] = a; r.m[1][1] = b; r.m[2][2] = c; return r;
}
static M3 mouter(V3 a, V3 b) {
    M3 r;
    r.m[0][0] = a.x * b.x; r.m[0][1] = a.x * b.y; r.m[0][2] = a.x * b.z;
    r.m[1][0] = a.y * b.x; r.m[1][1] = a.y * b.y; r.m[1][2] = a.y * b.z;
    r.m[2][0] = a.z * b.x; r.m[2][1] = a.z * b.y; r.m[2][2] = a.z * b.z;
    return r;
}
static M3 madd(M3 a, M3 b) {
    M3 r;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] + b.m[i][j];
    return r;
}
static M3 msub(M3 a, M3 b) {
    M3 r;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] - b.m[i][j];
    return r;
}
static M3 mscale(M3 a, float s) {
    M3 r;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[i][j] * s;
    return r;
}
static void maddto(M3* a, M3 b) {
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) a->m[i][j] += b.m[i][j];
}
static V3 mmulv(M3 a, V3 v) {
    return v3(a.m[0][0] * v.x + a.m[0][1] * v.y + a.m[0][2] * v.z,
              a.m[1][0] * v.x + a.m[1][1] * v.y + a.m[1][2] * v.z,
              a.m[2][0] * v.x + a.m[2][1] * v.y + a.m[2][2] * v.z);
}
static M3 mmul(M3 a, M3 b) {
    M3 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            float s = 0;
            for (int k = 0; k < 3; ++k) s += a.m[i][k] * b.m[k][j];
            r.m[i][j] = s;
        }
    return r;
}
static M3 mtrans(M3 a) {
    M3 r;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.m[i][j] = a.m[j][i];
    return r;
}
static int misfinite(M3 a) {
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) if (!isfinite(a.m[i][j])) return 0;
    return 1;
}
static M3 m9(const float* p) {
    M3 r;
    for (int i = 0; i < 9; ++i) r.m[i / 3][i % 3] = p[i];
    return r;
}
static void m9put(float* o, M3 m) { for (int i = 0; i < 9; ++i) o[i] = m.m[i / 3][i % 3]; }

/* ref: math.hpp:134-173 */
static Q4 q4(float x, float y, float z, float w) { Q4 q = {x, y, z, w}; return q; }
static Q4 q4p(const float* p) { return q4(p[0], p[1], p[2], p[3]); }
static float qnorm(Q4 q) { return sqrtf(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w); }
static Q4 qnormalized(Q4 q) {
    float n = qnorm(q);
    if (n <= 0.0f) return q4(0, 0, 0, 1);
    return q4(q.x / n, q.y / n, q.z / n, q.w / n);
}
static Q4 qconj(Q4 q) { return q4(-q.x, -q.y, -q.z, q.w); }
static Q4 qmul(Q4 a, Q4 o) {
    return q4(a.w * o.x + a.x * o.w + a.y * o.z - a.z * o.y,
              a.w * o.y - a.x * o.z + a.y * o.w + a.z * o.x,
              a.w * o.z + a.x * o.y - a.y * o.x + a.z * o.w,
              a.w * o.w - a.x * o.x - a.y * o.y - a.z * o.z);
}
static V3 qrotate(Q4 q, V3 v) {
    V3 u = v3(q.x, q.y, q.z);
    V3 t = vmul(vcross(u, v), 2.0f);
    return vadd(vadd(v, vmul(t, q.w)), vcross(u, t));
}
static V3 qrotate_inv(Q4 q, V3 v) { return qrotate(qconj(q), v); }
static M3 qtomat(Q4 q) {
    M3 r;
    float xx = q.x * q.x, yy = q.y * q.y, zz = q.z * q.z;
    float xy = q.x * q.y, xz = q.x * q.z, yz = q.y * q.z;
    float wx = q.w * q.x, wy = q.w * q.y, wz = q.w * q.z;
    r.m[0][0] = 1 - 2 * (yy + zz); r.m[0][1] = 2 * (xy - wz); r.m[0][2] = 2 * (xz + wy);
    r.m[1][0] = 2 * (xy + wz); r.m[1][1] = 1 - 2 * (xx + zz); r.m[1][2] = 2 * (yz - wx);
    r.m[2][0] = 2 * (xz - wy); r.m[2][1] = 2 * (yz + wx); r.m[2][2] = 1 - 2 * (xx + yy);
    return r;
}
/* ref: math.hpp:175-192 */
static Q4 qslerp(Q4 a, Q4 b, float t) {
    float cos_th = a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
    if (cos_th < 0) {
        b = q4(-b.x, -b.y, -b.z, -b.w);
        cos_th = -cos_th;
    }
    if (cos_th > 0.9995f) {
        Q4 r = q4(a.x + t * (b.x - a.x), a.y + t * (b.y - a.y), a.z + t * (b.z - a.z),
                  a.w + t * (b.w - a.w));
        return qnormalized(r);
    }
    float th = acosf(cos_th);
    float sa = sinf((1 - t) * th) / sinf(th);
    float sb = sinf(t * th) / sinf(th);
    return q4(sa * a.x + sb * b.x, sa * a.y + sb * b.y, sa * a.z + sb * b.z, sa * a.w + sb * b.w);
}

/* ref: math.hpp:195-199 */
typedef struct { int base[3]; float w[3][3]; float dw[3][3]; } SW;

/* ref: math.hpp:203-213 (divides by dx) */
static int spline_in_domain(V3 pos, V3 o, float dx, const int dims[3]) {
    const float p[3] = {(pos.x - o.x) / dx, (pos.y - o.y) / dx, (pos.z - o.z) / dx};
    for (int a = 0; a < 3; ++a) {
        int base = (int)floorf(p[a] - 0.5f);
        if (base < 0 || base + 2 > dims[a] - 1) return 0;
    }
    return 1;
}

/* ref: math.hpp:215-234 (multiplies by 1/dx) */
static SW spline_weights(V3 pos, V3 o, float dx) {
    SW sw;
    const float inv_dx = 1.0f / dx;
    const float p[3] = {(pos.x - o.x) * inv_dx, (pos.y - o.y) * inv_dx, (pos.z - o.z) * inv_dx};
    for (int a = 0; a < 3; ++a) {
        int base = (int)floorf(p[a] - 0.5f);
        float fx = p[a] - (float)base;
        sw.base[a] = base;
        sw.w[a][0] = 0.5f * (1.5f - fx) * (1.5f - fx);
        sw.w[a][1] = 0.75f - (fx - 1.0f) * (fx - 1.0f);
        sw.w[a][2] = 0.5f * (fx - 0.5f) * (fx - 0.5f);
        sw.dw[a][0] = (fx - 1.5f) * inv_dx;
        sw.dw[a][1] = -2.0f * (fx - 1.0f) * inv_dx;
        sw.dw[a][2] = (fx - 0.5f) * inv_dx;
    }
    return sw;
}

/* ref: math.hpp:252-271 */
typedef struct { float det; M3 inv; int invertible; } DI;
static DI det_inv(M3 a) {
    DI r;
    r.det = 0;
    r.inv = mzero();
    r.invertible = 0;
    const float c00 = a.m[1][1] * a.m[2][2] - a.m[1][2] * a.m[2][1];
    const float c01 = a.m[1][2] * a.m[2][0] - a.m[1][0] * a.m[2][2];
    const float c02 = a.m[1][0] * a.m[2][1] - a.m[1][1] * a.m[2][0];
    r.det = a.m[0][0] * c00 + a.m[0][1] * c01 + a.m[0][2] * c02;
    if (fabsf(r.det) <= 1e-12f) return r;
    const float id = 1.0f / r.det;
    r.inv.m[0][0] = c00 * id;
    r.inv.m[1][0] = c01 * id;
    r.inv.m[2][0] = c02 * id;
    r.inv.m[0][1] = (a.m[0][2] * a.m[2][1] - a.m[0][1] * a.m[2][2]) * id;
    r.inv.m[1][1] = (a.m[0][0] * a.m[2][2] - a.m[0][2] * a.m[2][0]) * id;
    r.inv.m[2][1] = (a.m[0][1] * a.m[2][0] - a.m[0][0] * a.m[2][1]) * id;
    r.inv.m[0][2] = (a.m[0][1] * a.m[1][2] - a.m[0][2] * a.m[1][1]) * id;
    r.inv.m[1][2] = (a.m[0][2] * a.m[1][0] - a.m[0][0] * a.m[1][2]) * id;
    r.inv.m[2][2] = (a.m[0][0] * a.m[1][1] - a.m[0][1] * a.m[1][0]) * id;
    r.invertible = 1;
    return r;
}

/* ref: math.hpp:273-277 */
static float mdet(M3 a) {
    return a.m[0][0] * (a.m[1][1] * a.m[2][2] - a.m[1][2] * a.m[2][1]) +
           a.m[0][1] * (a.m[1][2] * a.m[2][0] - a.m[1][0] * a.m[2][2]) +
           a.m[0][2] * (a.m[1][0] * a.m[2][1] - a.m[1][1] * a.m[2][0]);
}

static double det3d(double a[3][3]) {
    return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) +
           a[0][1] * (a[1][2] * a[2][0] - a[1][0] * a[2][2]) +
           a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
}

/* ref: math.hpp:286-340 — scaled Newton polar decomposition in double */
static int polar_decompose(M3 m, M3* R, M3* U) {
    if (!misfinite(m) || mdet(m) <= 0) return 0;
    double x[3][3];
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) x[i][j] = m.m[i][j];
    for (int iter = 0; iter < 50; ++iter) {
        double d = det3d(x);
        if (!(d > 0) || !isfinite(d)) return 0;
        double it[3][3];
        double id = 1.0 / d;
        it[0][0] = (x[1][1] * x[2][2] - x[1][2] * x[2][1]) * id;
        it[0][1] = (x[1][2] * x[2][0] - x[1][0] * x[2][2]) * id;
        it[0][2] = (x[1][0] * x[2][1] - x[1][1] * x[2][0]) * id;
        it[1][0] = (x[0][2] * x[2][1] - x[0][1] * x[2][2]) * id;
        it[1][1] = (x[0][0] * x[2][2] - x[0][2] * x[2][0]) * id;
        it[1][2] = (x[0][1] * x[2][0] - x[0][0] * x[2][1]) * id;
        it[2][0] = (x[0][1] * x[1][2] - x[0][2] * x[1][1]) * id;
        it[2][1] = (x[0][2] * x[1][0] - x[0][0] * x[1][2]) * id;
        it[2][2] = (x[0][0] * x[1][1] - x[0][1] * x[1][0]) * id;
        double nx = 0, ni = 0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                nx += x[i][j] * x[i][j];
                ni += it[i][j] * it[i][j];
            }
        double gamma = sqrt(sqrt(ni / nx));
        double delta = 0;
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) {
                double next = 0.5 * (gamma * x[i][j] + it[i][j] / gamma);
                double diff = next - x[i][j];
                delta += diff * diff;
                x[i][j] = next;
            }
        if (sqrt(delta) < 1e-8) break;
    }
    M3 r;
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r.m[i][j] = (float)x[i][j];
    M3 u = mmul(mtrans(r), m);
    *R = r;
    *U = mscale(madd(u, mtrans(u)), 0.5f);
    return 1;
}

/* ------------------------------------------------------------- materials.hpp */
/* ref: materials.hpp:20-27 */
void mpmor_lame(float E, float nu, float* mu, float* lambda) {
    *mu = E / (2 * (1 + nu));
    *lambda = E * nu / ((1 + nu) * (1 - 2 * nu));
}

/* ref: materials.hpp:35-54 — Cauchy stress accumulated in double */
static M3 neo_hookean(M3 F, float mu, float lambda) {
    double f[3][3];
    for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) f[i][j] = (double)F.m[i][j];
    double J = f[0][0] * (f[1][1] * f[2][2] - f[1][2] * f[2][1]) -
               f[0][1] * (f[1][0] * f[2][2] - f[1][2] * f[2][0]) +
               f[0][2] * (f[1][0] * f[2][1] - f[1][1] * f[2][0]);
    double Jc = J < 1e-6 ? 1e-6 : J;
    double d = (double)lambda * log(Jc);
    M3 s;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double b = f[i][0] * f[j][0] + f[i][1] * f[j][1] + f[i][2] * f[j][2];
            double v = (double)mu * (b - (i == j ? 1.0 : 0.0));
            if (i == j) v += d;
            s.m[i][j] = (float)(v / Jc);
        }
    return s;
}

/* ref: materials.hpp:59-72 */
static int corotational_project(M3 Fprev, M3 Cc, float dt, float beta, M3* out) {
    if (dt <= 0) return 0;
    M3 Ft = mmul(madd(mident(), mscale(Cc, dt)), Fprev);
    M3 R, U;
    if (!polar_decompose(Ft, &R, &U)) return 0;
    float dtrial = mdet(Ft);
    if (!(dtrial > 0)) return 0;
    M3 Fp = madd(mscale(R, beta), mscale(Ft, (1 - beta) / dtrial));
    DI ip = det_inv(Fprev);
    if (!ip.invertible) return 0;
    *out = mscale(msub(mmul(Fp, ip.inv), mident()), 1.0f / dt);
    return 1;
}

/* -------------------------------------------------------------- geometry.hpp */
typedef struct {
    int geom;
    float gp[4];
    V3* verts;
    int nv;
    int* idx;
    int ni;
    int* spine;
    int ns;
    /* pose, ref: geometry.hpp:14-18 */
    V3 pos;
    Q4 rot;
    V3 lin;
    V3 ang;
    float mu_k, c_d, hw;
    int motion;
    mpmb_keyframe* kf;
    int nkf;
    float body_mass;
    V3 inertia;
    int id;
} Shape;

typedef struct { float distance; V3 normal; V3 tangent; int region; } Sdf;

static Sdf sdf_default(void) {
    Sdf s;
    s.distance = 0;
    s.normal = v3(1, 0, 0);
    s.tangent = v3(0, 1, 0);
    s.region = MPMB_REGION_BULK;
    return s;
}

static float clampf_(float v, float lo, float hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* ref: geometry.hpp:29-32 */
static V3 rigid_point_velocity(const Shape* s, V3 p) {
    return vadd(s->lin, vcross(s->ang, vsub(p, s->pos)));
}

/* ref: geometry.hpp:136-142 */
static Sdf sdf_plane(V3 p) {
    Sdf s = sdf_default();
    s.distance = p.y;
    s.normal = v3(0, 1, 0);
    s.region = MPMB_REGION_SURFACE;
    return s;
}
/* ref: geometry.hpp:144-151 */
static Sdf sdf_sphere(float radius, V3 p) {
    Sdf s = sdf_default();
    float r = vnorm(p);
    s.distance = r - radius;
    s.normal = r > 1e-9f ? vdiv(p, r) : v3(1, 0, 0);
    s.region = MPMB_REGION_SURFACE;
    return s;
}
/* ref: geometry.hpp:153-176 */
static Sdf sdf_box(V3 h, V3 p) {
    Sdf s = sdf_default();
    s.region = MPMB_REGION_SURFACE;
    V3 q = v3(fabsf(p.x) - h.x, fabsf(p.y) - h.y, fabsf(p.z) - h.z);
    float qmax = q.x;
    if (qmax < q.y) qmax = q.y;
    if (qmax < q.z) qmax = q.z;
    if (qmax <= 0) {
        s.distance = qmax;
        if (q.x >= q.y && q.x >= q.z)
            s.normal = v3(p.x >= 0 ? 1.0f : -1.0f, 0, 0);
        else if (q.y >= q.z)
            s.normal = v3(0, p.y >= 0 ? 1.0f : -1.0f, 0);
        else
            s.normal = v3(0, 0, p.z >= 0 ? 1.0f : -1.0f);
        return s;
    }
    V3 closest = v3(clampf_(p.x, -h.x, h.x), clampf_(p.y, -h.y, h.y), clampf_(p.z, -h.z, h.z));
    V3 d = vsub(p, closest);
    s.distance = vnorm(d);
    s.normal = s.distance > 1e-9f ? vdiv(d, s.distance) : v3(1, 0, 0);
    return s;
}
/* ref: geometry.hpp:178-202 */
static Sdf sdf_quad_slicer(float hl, float hh, float sr, V3 p) {
    Sdf s = sdf_default();
    if (p.y >= hh) {
        float cx = clampf_(p.x, -hl, hl);
        V3 axis = v3(cx, hh, 0);
        V3 d = vsub(p, axis);
        float r = vnorm(d);
        s.distance = r - sr;
        s.normal = r > 1e-9f ? vdiv(d, r) : v3(0, 1, 0);
        s.region = MPMB_REGION_SPINE;
        return s;
    }
    if (fabsf(p.x) <= hl && p.y >= -hh) {
        s.distance = p.z;
        s.normal = v3(0, 0, p.z >= 0 ? 1.0f : -1.0f);
        s.region = MPMB_REGION_EDGE;
        return s;
    }
    s.region = MPMB_REGION_BULK;
    s.distance = FLT_MAX;
    return s;
}
/* ref: geometry.hpp:204-213 */
static V3 closest_on_segment(V3 a, V3 b, V3 p, float* t_out) {
    V3 ab = vsub(b, a);
    float len2 = vnorm2(ab);
    float t = len2 > 1e-18f ? clampf_(vdot(vsub(p, a), ab) / len2, 0.0f, 1.0f) : 0.0f;
    *t_out = t;
    return vadd(a, vmul(ab, t));
}
/* ref: geometry.hpp:217-242 */
static V3 closest_on_triangle(V3 a, V3 b, V3 c, V3 p, int* interior) {
    V3 ab = vsub(b, a), ac = vsub(c, a), ap = vsub(p, a);
    float d1 = vdot(ab, ap), d2 = vdot(ac, ap);
    *interior = 0;
    if (d1 <= 0 && d2 <= 0) return a;
    V3 bp = vsub(p, b);
    float d3 = vdot(ab, bp), d4 = vdot(ac, bp);
    if (d3 >= 0 && d4 <= d3) return b;
    float vc = d1 * d4 - d3 * d2;
    if (vc <= 0 && d1 >= 0 && d3 <= 0) return vadd(a, vmul(ab, d1 / (d1 - d3)));
    V3 cp = vsub(p, c);
    float d5 = vdot(ab, cp), d6 = vdot(ac, cp);
    if (d6 >= 0 && d5 <= d6) return c;
    float vb = d5 * d2 - d1 * d6;
    if (vb <= 0 && d2 >= 0 && d6 <= 0) return vadd(a, vmul(ac, d2 / (d2 - d6)));
    float va = d3 * d6 - d5 * d4;
    if (va <= 0 && (d4 - d3) >= 0 && (d5 - d6) >= 0) {
        float w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        return vadd(b, vmul(vsub(c, b), w));
    }
    float denom = 1.0f / (va + vb + vc);
    *interior = 1;
    return vadd(vadd(a, vmul(ab, vb * denom)), vmul(ac, vc * denom));
}
/* ref: geometry.hpp:244-293 */
static Sdf sdf_mesh_slicer(const Shape* g, V3 p) {
    float best_spine = FLT_MAX;
    V3 spine_pt = v3(0, 0, 0);
    for (int e = 0; e + 1 < g->ns; e += 2) {
        float t;
        V3 q = closest_on_segment(g->verts[g->spine[e]], g->verts[g->spine[e + 1]], p, &t);
        float d = vnorm(vsub(p, q));
        if (d < best_spine) {
            best_spine = d;
            spine_pt = q;
        }
    }
    float best_surf = FLT_MAX;
    V3 surf_pt = v3(0, 0, 0), surf_n = v3(0, 0, 0);
    for (int t = 0; t + 2 < g->ni; t += 3) {
        V3 a = g->verts[g->idx[t]], b = g->verts[g->idx[t + 1]], c = g->verts[g->idx[t + 2]];
        int interior;
        V3 q = closest_on_triangle(a, b, c, p, &interior);
        float d = vnorm(vsub(p, q));
        if (d < best_surf) {
            best_surf = d;
            surf_pt = q;
            surf_n = vnormalized(vcross(vsub(b, a), vsub(c, a)));
        }
    }
    Sdf s = sdf_default();
    if (best_spine <= best_surf + 1e-9f && best_spine < FLT_MAX) {
        V3 d = vsub(p, spine_pt);
        float r = vnorm(d);
        s.distance = r - g->gp[0];
        s.normal = r > 1e-9f ? vdiv(d, r) : v3(0, 1, 0);
        s.region = MPMB_REGION_SPINE;
        return s;
    }
    float side = vdot(vsub(p, surf_pt), surf_n) >= 0 ? 1.0f : -1.0f;
    s.distance = side * best_surf;
    s.normal = vmul(surf_n, side);
    s.region = MPMB_REGION_EDGE;
    return s;
}
/* ref: geometry.hpp:295-327 */
static Sdf sdf_arc(float radius, float angle, V3 p) {
    const float kTwoPi = (float)(2 * 3.14159265358979323846);
    V3 planar = v3(p.x, p.y, 0);
    float t;
    if (vnorm(planar) < 1e-9f) {
        t = 0;
    } else {
        t = atan2f(planar.y, planar.x);
        if (t < 0) t += kTwoPi;
        if (t > angle) {
            float to_end = t - angle;
            float to_start = kTwoPi - t;
            t = to_end <= to_start ? angle : 0.0f;
        }
    }
    V3 q = v3(radius * cosf(t), radius * sinf(t), 0);
    V3 tangent = v3(-sinf(t), cosf(t), 0);
    Sdf s = sdf_default();
    s.region = MPMB_REGION_CURVE;
    s.tangent = tangent;
    V3 d = vsub(p, q);
    float dist = vnorm(d);
    s.distance = dist;
    if (dist < 1e-9f)
        s.normal = v3(-cosf(t), -sinf(t), 0);
    else
        s.normal = vdiv(d, dist);
    return s;
}
/* ref: geometry.hpp:329-365 */
static Sdf sdf_polyline(const Shape* g, V3 p) {
    float best = FLT_MAX;
    V3 best_pt = v3(0, 0, 0), best_tangent = v3(1, 0, 0);
    for (int i = 0; i + 1 < g->nv; ++i) {
        float t;
        V3 q = closest_on_segment(g->verts[i], g->verts[i + 1], p, &t);
        float d = vnorm(vsub(p, q));
        if (d < best) {
            best = d;
            best_pt = q;
            V3 dir = vnormalized(vsub(g->verts[i + 1], g->verts[i]));
            if (t <= 1e-6f && i > 0) {
                V3 prev = vnormalized(vsub(g->verts[i], g->verts[i - 1]));
                dir = vnormalized(vadd(dir, prev));
            } else if (t >= 1.0f - 1e-6f && i + 2 < g->nv) {
                V3 next = vnormalized(vsub(g->verts[i + 2], g->verts[i + 1]));
                dir = vnormalized(vadd(dir, next));
            }
            best_tangent = dir;
        }
    }
    Sdf s = sdf_default();
    s.region = MPMB_REGION_CURVE;
    s.tangent = best_tangent;
    s.distance = best;
    if (best < 1e-9f) {
        V3 ref = fabsf(best_tangent.x) < 0.9f ? v3(1, 0, 0) : v3(0, 1, 0);
        s.normal = vnormalized(vcross(best_tangent, ref));
    } else {
        s.normal = vdiv(vsub(p, best_pt), best);
    }
    return s;
}
/* ref: geometry.hpp:370-395 */
static Sdf sdf_query(const Shape* g, V3 point) {
    V3 local = qrotate_inv(g->rot, vsub(point, g->pos));
    Sdf s;
    switch (g->geom) {
        case MPMB_GEOM_PLANE: s = sdf_plane(local); break;
        case MPMB_GEOM_SPHERE: s = sdf_sphere(g->gp[0], local); break;
        case MPMB_GEOM_BOX: s = sdf_box(v3(g->gp[0], g->gp[1], g->gp[2]), local); break;
        case MPMB_GEOM_QUAD_SLICER: s = sdf_quad_slicer(g->gp[0], g->gp[1], g->gp[2], local); break;
        case MPMB_GEOM_TRI_MESH_SLICER: s = sdf_mesh_slicer(g, local); break;
        case MPMB_GEOM_ARC: s = sdf_arc(g->gp[0], g->gp[1], local); break;
        default: s = sdf_polyline(g, local); break;
    }
    s.normal = qrotate(g->rot, s.normal);
    s.tangent = qrotate(g->rot, s.tangent);
    return s;
}

static void shape_free(Shape* s) {
    free(s->verts);
    free(s->idx);
    free(s->spine);
    free(s->kf);
    memset(s, 0, sizeof *s);
}

static void shape_from(Shape* s, const mpmb_shape_desc* d) {
    memset(s, 0, sizeof *s);
    s->geom = d->geometry;
    memcpy(s->gp, d->gparam, sizeof s->gp);
    if (d->n_vertices > 0) {
        s->nv = d->n_vertices;
        s->verts = (V3*)malloc(sizeof(V3) * s->nv);
        for (int i = 0; i < s->nv; ++i) s->verts[i] = v3p(d->vertices + 3 * i);
    }
    if (d->n_indices > 0) {
        s->ni = d->n_indices;
        s->idx = (int*)malloc(sizeof(int) * s->ni);
        memcpy(s->idx, d->indices, sizeof(int) * s->ni);
    }
    if (d->n_spine_edges > 0) {
        s->ns = d->n_spine_edges;
        s->spine = (int*)malloc(sizeof(int) * s->ns);
        memcpy(s->spine, d->spine_edges, sizeof(int) * s->ns);
    }
    s->pos = v3p(d->pose.position);
    s->rot = q4p(d->pose.orientation);
    s->lin = v3p(d->pose.linear_velocity);
    s->ang = v3p(d->pose.angular_velocity);
    s->mu_k = d->mu_k;
    s->c_d = d->c_d;
    s->hw = d->collision_halfwidth;
    s->motion = d->motion;
    if (d->n_keyframes > 0) {
        s->nkf = d->n_keyframes;
        s->kf = (mpmb_keyframe*)malloc(sizeof(mpmb_keyframe) * s->nkf);
        memcpy(s->kf, d->keyframes, sizeof(mpmb_keyframe) * s->nkf);
    }
    s->body_mass = d->body_mass;
    s->inertia = v3p(d->inertia);
}

/* ref: geometry.hpp:98-132 */
static int validate_geometry(const Shape* s) {
    switch (s->geom) {
        case MPMB_GEOM_PLANE: return 1;
        case MPMB_GEOM_SPHERE: return s->gp[0] > 0;
        case MPMB_GEOM_BOX: return s->gp[0] > 0 && s->gp[1] > 0 && s->gp[2] > 0;
        case MPMB_GEOM_QUAD_SLICER: return s->gp[0] > 0 && s->gp[1] > 0 && s->gp[2] > 0;
        case MPMB_GEOM_TRI_MESH_SLICER:
            if (s->nv < 3 || s->ni < 3 || s->ni % 3 != 0) return 0;
            if (!(s->gp[0] > 0) || s->ns % 2 != 0) return 0;
            for (int i = 0; i < s->ni; ++i) if (s->idx[i] < 0 || s->idx[i] >= s->nv) return 0;
            for (int i = 0; i < s->ns; ++i) if (s->spine[i] < 0 || s->spine[i] >= s->nv) return 0;
            return 1;
        case MPMB_GEOM_ARC:
            return s->gp[0] > 0 && s->gp[1] > 0 &&
                   !(s->gp[1] > (float)(2 * 3.14159265358979323846 + 1e-6));
        case MPMB_GEOM_POLYLINE: return s->nv >= 2;
    }
    return 0;
}

/* ---------------------------------------------------------- rigid_dynamics.hpp */
/* ref: rigid_dynamics.hpp:31-51 */
static void interp_pose(const mpmb_keyframe* kf, int n, float t, V3* pos, Q4* rot) {
    if (t <= kf[0].time) {
        *pos = v3p(kf[0].position);
        *rot = q4p(kf[0].orientation);
        return;
    }
    if (t >= kf[n - 1].time) {
        *pos = v3p(kf[n - 1].position);
        *rot = q4p(kf[n - 1].orientation);
        return;
    }
    int hi = 1;
    while (kf[hi].time < t) ++hi;
    const mpmb_keyframe* a = &kf[hi - 1];
    const mpmb_keyframe* b = &kf[hi];
    float u = (t - a->time) / (b->time - a->time);
    *pos = vadd(v3p(a->position), vmul(vsub(v3p(b->position), v3p(a->position)), u));
    *rot = qslerp(q4p(a->orientation), q4p(b->orientation), u);
}

/* ref: rigid_dynamics.hpp:57-73 */
static void evaluate_trajectory(const mpmb_keyframe* kf, int n, float t, V3* pos, Q4* rot,
                                V3* lin, V3* ang) {
    interp_pose(kf, n, t, pos, rot);
    const float h = 1e-4f;
    V3 p0, p1;
    Q4 q0, q1;
    interp_pose(kf, n, t - h, &p0, &q0);
    interp_pose(kf, n, t + h, &p1, &q1);
    *lin = vdiv(vsub(p1, p0), 2 * h);
    Q4 dq = q4((q1.x - q0.x) / (2 * h), (q1.y - q0.y) / (2 * h), (q1.z - q0.z) / (2 * h),
               (q1.w - q0.w) / (2 * h));
    Q4 w = qmul(dq, qconj(*rot));
    *ang = vmul(v3(w.x, w.y, w.z), 2.0f);
}

/* ref: rigid_dynamics.hpp:82-103 */
static void integrate_free_body(Shape* s, V3 impulse, V3 torque, V3 g, float dt) {
    s->lin = vadd(s->lin, vadd(vmul(impulse, 1.0f / s->body_mass), vmul(g, dt)));
    M3 R = qtomat(s->rot);
    M3 Ib = mdiag(1.0f / s->inertia.x, 1.0f / s->inertia.y, 1.0f / s->inertia.z);
    M3 Iw = mmul(mmul(R, Ib), mtrans(R));
    s->ang = vadd(s->ang, mmulv(Iw, torque));
    s->pos = vadd(s->pos, vmul(s->lin, dt));
    V3 w = s->ang;
    Q4 dq = qmul(q4(w.x, w.y, w.z, 0), s->rot);
    s->rot = qnormalized(q4(s->rot.x + 0.5f * dt * dq.x, s->rot.y + 0.5f * dt * dq.y,
                            s->rot.z + 0.5f * dt * dq.z, s->rot.w + 0.5f * dt * dq.w));
}

/* ------------------------------------------------------------------ state.hpp */
typedef struct { float mass; V3 mom; V3 vel; } Node; /* ref: state.hpp:15-20 (contact_impulse is dead scratch, contact.hpp:127) */
typedef struct { int dims[3]; float dx; V3 origin; Node* nodes; size_t n; } Grid;

typedef struct {
    size_t n;
    V3* x;
    V3* v;
    float* mass;
    float* vol0;
    M3* F;
    M3* C;
    M3* stress;
    int* mat;
    uint8_t* active;
} Particles;

typedef struct { V3 imp; V3 tq; int count; double impd[3]; double tqd[3]; } Acc;

struct mpmor_state_s {
    Grid grid;
    Particles p;
    mpmb_material* mats;
    int nmats;
    Shape* shapes;
    int nshapes;
    Acc* acc;
};

static const float kMassEps = 1e-9f; /* ref: state.hpp:13 */

/* ref: state.hpp:39-43 */
static size_t gindex(const Grid* g, int i, int j, int k) {
    return (size_t)i + (size_t)g->dims[0] * ((size_t)j + (size_t)g->dims[1] * (size_t)k);
}
/* ref: state.hpp:49-51 */
static V3 node_position(const Grid* g, int i, int j, int k) {
    return vadd(g->origin, vmul(v3((float)i, (float)j, (float)k), g->dx));
}
/* ref: state.hpp:60-62 */
static void grid_clear(Grid* g) { memset(g->nodes, 0, sizeof(Node) * g->n); }

static void particles_free(Particles* p) {
    free(p->x); free(p->v); free(p->mass); free(p->vol0); free(p->F); free(p->C);
    free(p->stress); free(p->mat); free(p->active);
    memset(p, 0, sizeof *p);
}
static void particles_alloc(Particles* p, size_t n) {
    particles_free(p);
    p->n = n;
    p->x = (V3*)calloc(n ? n : 1, sizeof(V3));
    p->v = (V3*)calloc(n ? n : 1, sizeof(V3));
    p->mass = (float*)calloc(n ? n : 1, sizeof(float));
    p->vol0 = (float*)calloc(n ? n : 1, sizeof(float));
    p->F = (M3*)calloc(n ? n : 1, sizeof(M3));
    p->C = (M3*)calloc(n ? n : 1, sizeof(M3));
    p->stress = (M3*)calloc(n ? n : 1, sizeof(M3));
    p->mat = (int*)calloc(n ? n : 1, sizeof(int));
    p->active = (uint8_t*)calloc(n ? n : 1, 1);
}
static void particles_append(Particles* p, size_t extra) {
    size_t n = p->n + extra;
    p->x = (V3*)realloc(p->x, sizeof(V3) * n);
    p->v = (V3*)realloc(p->v, sizeof(V3) * n);
    p->mass = (float*)realloc(p->mass, sizeof(float) * n);
    p->vol0 = (float*)realloc(p->vol0, sizeof(float) * n);
    p->F = (M3*)realloc(p->F, sizeof(M3) * n);
    p->C = (M3*)realloc(p->C, sizeof(M3) * n);
    p->stress = (M3*)realloc(p->stress, sizeof(M3) * n);
    p->mat = (int*)realloc(p->mat, sizeof(int) * n);
    p->active = (uint8_t*)realloc(p->active, n);
}

/* ref: math.hpp:343-356 */
static uint64_t splitmix_next(uint64_t* s) {
    uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static double splitmix_signed_unit(uint64_t* s) {
    return (splitmix_next(s) >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
}

/* ref: state.hpp:101-149 ; returns count, -1 invalid */
static long spawn_box(Particles* p, const Grid* g, V3 mn, V3 mx, int ppc, float density,
                      int mat, uint64_t seed) {
    V3 ext = vsub(mx, mn);
    if (ext.x <= 0 || ext.y <= 0 || ext.z <= 0) return -1;
    if (ppc < 1 || density <= 0) return -1;
    if (!spline_in_domain(mn, g->origin, g->dx, g->dims) ||
        !spline_in_domain(mx, g->origin, g->dx, g->dims))
        return -1;
    const float spacing = g->dx / cbrtf((float)ppc);
    const float pm = density * spacing * spacing * spacing;
    const float pv = spacing * spacing * spacing;
    long nx = lroundf(ext.x / spacing), ny = lroundf(ext.y / spacing), nz = lroundf(ext.z / spacing);
    int inx = (int)nx < 1 ? 1 : (int)nx, iny = (int)ny < 1 ? 1 : (int)ny,
        inz = (int)nz < 1 ? 1 : (int)nz;
    uint64_t rng = seed;
    const float jitter = 0.25f * spacing;
    size_t start = p->n;
    size_t count = (size_t)inx * iny * inz;
    particles_append(p, count);
    size_t q = start;
    for (int k = 0; k < inz; ++k)
        for (int j = 0; j < iny; ++j)
            for (int i = 0; i < inx; ++i) {
                V3 pos = vadd(mn, v3(((float)i + 0.5f) * spacing, ((float)j + 0.5f) * spacing,
                                     ((float)k + 0.5f) * spacing));
                pos.x += jitter * (float)splitmix_signed_unit(&rng);
                pos.y += jitter * (float)splitmix_signed_unit(&rng);
                pos.z += jitter * (float)splitmix_signed_unit(&rng);
                p->x[q] = pos;
                p->v[q] = v3(0, 0, 0);
                p->mass[q] = pm;
                p->vol0[q] = pv;
                p->F[q] = mident();
                p->C[q] = mzero();
                p->stress[q] = mzero();
                p->mat[q] = mat;
                p->active[q] = 1;
                ++q;
            }
    p->n = start + count;
    return (long)count;
}

/* ref: state.hpp:153-164 */
static int deactivate(Particles* p, const Grid* g) {
    int count = 0;
    for (size_t i = 0; i < p->n; ++i) {
        if (!p->active[i]) continue;
        if (!spline_in_domain(p->x[i], g->origin, g->dx, g->dims)) {
            p->active[i] = 0;
            ++count;
        }
    }
    return count;
}

/* ---------------------------------------------------------------- contact.hpp */
/* ref: contact.hpp:33-38 */
static float friction_drag(float vn, float vtg, float mu_k, float c_d) {
    if (vtg < 1e-12f) return 0;
    float f = 1.0f - mu_k * vn / vtg;
    return c_d * (f < 0.0f ? 0.0f : f);
}
/* ref: contact.hpp:43-56 */
static V3 correct_surface(V3 vnode, V3 vrig, V3 n, const Shape* s, V3* delta) {
    V3 vrel = vsub(vnode, vrig);
    float vn = vdot(vrel, n);
    if (vn >= 0) { *delta = v3(0, 0, 0); return vnode; }
    V3 vtg = vsub(vrel, vmul(n, vn));
    float tg = vnorm(vtg);
    V3 vnew = vmul(vtg, friction_drag(-vn, tg, s->mu_k, s->c_d));
    V3 vc = vadd(vrig, vnew);
    *delta = vsub(vc, vnode);
    return vc;
}
/* ref: contact.hpp:60-74 */
static V3 correct_curve(V3 vnode, V3 vrig, V3 n, V3 tangent, const Shape* s, V3* delta) {
    V3 vrel = vsub(vnode, vrig);
    float vn = vdot(vrel, n);
    if (vn >= 0) { *delta = v3(0, 0, 0); return vnode; }
    V3 vtg1 = vmul(tangent, vdot(vrel, tangent));
    float tg = vnorm(vtg1);
    V3 vnew = vmul(vtg1, friction_drag(-vn, tg, s->mu_k, s->c_d));
    V3 vc = vadd(vrig, vnew);
    *delta = vsub(vc, vnode);
    return vc;
}
/* ref: contact.hpp:82-92 */
static int node_in_contact(const Sdf* s, float hw) {
    switch (s->region) {
        case MPMB_REGION_SURFACE: return s->distance < 0;
        case MPMB_REGION_EDGE: return fabsf(s->distance) < hw;
        case MPMB_REGION_SPINE: return s->distance < 0;
        case MPMB_REGION_CURVE: return s->distance < hw;
    }
    return 0;
}
/* ref: contact.hpp:97-136 */
static void contact_pass(Grid* g, Shape* shapes, int ns, Acc* acc) {
    if (ns == 0) return;
    for (size_t idx = 0; idx < g->n; ++idx) {
        Node* node = &g->nodes[idx];
        if (node->mass <= kMassEps) continue;
        int i = (int)(idx % g->dims[0]);
        int j = (int)((idx / g->dims[0]) % g->dims[1]);
        int k = (int)(idx / ((size_t)g->dims[0] * g->dims[1]));
        V3 xn = node_position(g, i, j, k);
        for (int si = 0; si < ns; ++si) {
            const Shape* sh = &shapes[si];
            Sdf s = sdf_query(sh, xn);
            if (!node_in_contact(&s, sh->hw)) continue;
            V3 vr = rigid_point_velocity(sh, xn);
            V3 delta, vc;
            if (s.region == MPMB_REGION_SPINE) {
                vc = vr;
                delta = vsub(vr, node->vel);
            } else if (s.region == MPMB_REGION_CURVE) {
                vc = correct_curve(node->vel, vr, s.normal, s.tangent, sh, &delta);
            } else {
                vc = correct_surface(node->vel, vr, s.normal, sh, &delta);
            }
            if (vnorm2(delta) > 0) {
                node->vel = vc;
                node->mom = vmul(node->vel, node->mass);
                V3 imp = vmul(delta, -node->mass);
                V3 arm = vsub(xn, sh->pos);
                V3 tq = vcross(arm, imp);
                acc[si].imp = vadd(acc[si].imp, imp);
                acc[si].tq = vadd(acc[si].tq, tq);
                acc[si].count += 1;
                /* double-precision shadow of the same terms (tolerance reference) */
                double md = -(double)node->mass;
                double id[3] = {delta.x * md, delta.y * md, delta.z * md};
                double ad[3] = {arm.x, arm.y, arm.z};
                acc[si].impd[0] += id[0];
                acc[si].impd[1] += id[1];
                acc[si].impd[2] += id[2];
                acc[si].tqd[0] += ad[1] * id[2] - ad[2] * id[1];
                acc[si].tqd[1] += ad[2] * id[0] - ad[0] * id[2];
                acc[si].tqd[2] += ad[0] * id[1] - ad[1] * id[0];
            }
        }
    }
}
/* ref: contact.hpp:140-179 */
static int pushout(Particles* p, const Shape* shapes, int ns, float dx) {
    if (ns == 0) return 0;
    const float clearance = 1e-4f * dx;
    int count = 0;
    for (size_t pi = 0; pi < p->n; ++pi) {
        if (!p->active[pi]) continue;
        for (int si = 0; si < ns; ++si) {
            const Shape* sh = &shapes[si];
            Sdf s = sdf_query(sh, p->x[pi]);
            float move = 0;
            switch (s.region) {
                case MPMB_REGION_SURFACE:
                case MPMB_REGION_SPINE:
                    if (s.distance < 0) move = -s.distance + clearance;
                    break;
                case MPMB_REGION_EDGE: {
                    float target = 0.5f * sh->hw;
                    float d = fabsf(s.distance);
                    if (d < target) move = target - d + clearance;
                    break;
                }
                case MPMB_REGION_CURVE: {
                    float target = 0.5f * sh->hw;
                    if (s.distance < target) move = target - s.distance + clearance;
                    break;
                }
                default: break;
            }
            if (move > 0) {
                p->x[pi] = vadd(p->x[pi], vmul(s.normal, move));
                V3 vr = rigid_point_velocity(sh, p->x[pi]);
                float vn = vdot(vsub(p->v[pi], vr), s.normal);
                if (vn < 0) p->v[pi] = vsub(p->v[pi], vmul(s.normal, vn));
                ++count;
            }
        }
    }
    return count;
}

/* ---------------------------------------------------------------- solvers.hpp */
/* ref: solvers.hpp:30-50 */
static void apply_bc(Grid* g, int kind) {
    const int margin = 2;
    for (size_t idx = 0; idx < g->n; ++idx) {
        Node* node = &g->nodes[idx];
        if (node->mass <= kMassEps) continue;
        int i = (int)(idx % g->dims[0]);
        int j = (int)((idx / g->dims[0]) % g->dims[1]);
        int k = (int)(idx / ((size_t)g->dims[0] * g->dims[1]));
        int bx = i < margin || i >= g->dims[0] - margin;
        int by = j < margin || j >= g->dims[1] - margin;
        int bz = k < margin || k >= g->dims[2] - margin;
        if (!(bx || by || bz)) continue;
        if (kind == MPMB_BC_STICKY) {
            node->vel = v3(0, 0, 0);
        } else {
            if (bx) node->vel.x = 0;
            if (by) node->vel.y = 0;
            if (bz) node->vel.z = 0;
        }
        node->mom = vmul(node->vel, node->mass);
    }
}

/* ref: solvers.hpp:54-65 (hook = contact pass when enabled) */
static void grid_velocity_update(struct mpmor_state_s* st, V3 g, float dt, int contact, int bc,
                                 int apply_gravity) {
    Grid* grid = &st->grid;
    for (size_t i = 0; i < grid->n; ++i) {
        Node* n = &grid->nodes[i];
        if (n->mass <= kMassEps) continue;
        n->vel = vdiv(n->mom, n->mass);
        if (apply_gravity) n->vel = vadd(n->vel, vmul(g, dt));
        n->mom = vmul(n->vel, n->mass);
    }
    if (contact) contact_pass(grid, st->shapes, st->nshapes, st->acc);
    apply_bc(grid, bc);
}

/* ref: solvers.hpp:69-74 */
static void update_stress(struct mpmor_state_s* st, size_t i, int* inverted) {
    const mpmb_material* mat = &st->mats[st->p.mat[i]];
    if (mdet(st->p.F[i]) <= 0) ++*inverted;
    st->p.stress[i] = neo_hookean(st->p.F[i], mat->mu, mat->lambda);
}

/* Order perturbation (checker calibration only): 1 = P2G visits particles in reverse
 * index order.  The reference sums in index order (solvers.hpp:151); the difference
 * between the two orders is the reference's own float-reordering sensitivity, the
 * yardstick for device results that sum with atomics (SURVEY.md §7 hard part 1). */
static int g_order_mode = 0;
void mpmor_set_order_perturbation(int32_t mode) { g_order_mode = mode; }

/* ref: solvers.hpp:151-169 (P2G); stress_scale = -dt*V*m_inv for MLS, absent for PB */
static void p2g(struct mpmor_state_s* st, float dt, float m_inv, int with_stress) {
    Particles* p = &st->p;
    Grid* grid = &st->grid;
    for (size_t ii = 0; ii < p->n; ++ii) {
        const size_t i = g_order_mode == 1 ? p->n - 1 - ii : ii;
        if (!p->active[i]) continue;
        SW sw = spline_weights(p->x[i], grid->origin, grid->dx);
        M3 affine;
        if (with_stress) {
            float volume = mdet(p->F[i]) * p->vol0[i];
            affine = madd(mscale(p->C[i], p->mass[i]), mscale(p->stress[i], -dt * volume * m_inv));
        } else {
            affine = mscale(p->C[i], p->mass[i]); /* ref: solvers.hpp:222 */
        }
        for (int dk = 0; dk < 3; ++dk)
            for (int dj = 0; dj < 3; ++dj)
                for (int di = 0; di < 3; ++di) {
                    float w = sw.w[0][di] * sw.w[1][dj] * sw.w[2][dk];
                    int gi = sw.base[0] + di, gj = sw.base[1] + dj, gk = sw.base[2] + dk;
                    V3 rel = vsub(node_position(grid, gi, gj, gk), p->x[i]);
                    Node* node = &grid->nodes[gindex(grid, gi, gj, gk)];
                    node->mass += w * p->mass[i];
                    node->mom = vadd(node->mom,
                                     vmul(vadd(vmul(p->v[i], p->mass[i]), mmulv(affine, rel)), w));
                }
    }
}

/* ref: solvers.hpp:176-190 (G2P gather) */
static void g2p_gather(const Grid* grid, V3 x, V3* vnew, M3* B) {
    SW sw = spline_weights(x, grid->origin, grid->dx);
    *vnew = v3(0, 0, 0);
    *B = mzero();
    for (int dk = 0; dk < 3; ++dk)
        for (int dj = 0; dj < 3; ++dj)
            for (int di = 0; di < 3; ++di) {
                float w = sw.w[0][di] * sw.w[1][dj] * sw.w[2][dk];
                int gi = sw.base[0] + di, gj = sw.base[1] + dj, gk = sw.base[2] + dk;
                const Node* node = &grid->nodes[gindex(grid, gi, gj, gk)];
                if (node->mass <= kMassEps) continue;
                V3 rel = vsub(node_position(grid, gi, gj, gk), x);
                *vnew = vadd(*vnew, vmul(node->vel, w));
                maddto(B, mouter(vmul(node->vel, w), rel));
            }
}

/* ref: solvers.hpp:80-138 (standard MPM: PIC transfers, nodal force -dt V sigma grad w) */
mpmb_status mpmor_step_standard(mpmor_state st, float dt, const float gr[3], int32_t contact, int32_t bc,
                                mpmb_step_stats* stats) {
    int inverted = 0;
    Particles* p = &st->p;
    Grid* grid = &st->grid;
    grid_clear(grid);
    for (size_t ii = 0; ii < p->n; ++ii) {
        const size_t i = g_order_mode == 1 ? p->n - 1 - ii : ii;
        if (!p->active[i]) continue;
        SW sw = spline_weights(p->x[i], grid->origin, grid->dx);
        float volume = mdet(p->F[i]) * p->vol0[i];
        M3 impulse_m = mscale(p->stress[i], -dt * volume);
        for (int dk = 0; dk < 3; ++dk)
            for (int dj = 0; dj < 3; ++dj)
                for (int di = 0; di < 3; ++di) {
                    float w = sw.w[0][di] * sw.w[1][dj] * sw.w[2][dk];
                    V3 grad = v3(sw.dw[0][di] * sw.w[1][dj] * sw.w[2][dk], sw.w[0][di] * sw.dw[1][dj] * sw.w[2][dk],
                                 sw.w[0][di] * sw.w[1][dj] * sw.dw[2][dk]);
                    Node* node = &grid->nodes[gindex(grid, sw.base[0] + di, sw.base[1] + dj, sw.base[2] + dk)];
                    node->mass += w * p->mass[i];
                    node->mom = vadd(node->mom, vadd(vmul(p->v[i], w * p->mass[i]), mmulv(impulse_m, grad)));
                }
    }
    grid_velocity_update(st, v3p(gr), dt, contact, bc, 1);
    for (size_t i = 0; i < p->n; ++i) {
        if (!p->active[i]) continue;
        SW sw = spline_weights(p->x[i], grid->origin, grid->dx);
        V3 vnew = v3(0, 0, 0);
        M3 L = mzero();
        for (int dk = 0; dk < 3; ++dk)
            for (int dj = 0; dj < 3; ++dj)
                for (int di = 0; di < 3; ++di) {
                    float w = sw.w[0][di] * sw.w[1][dj] * sw.w[2][dk];
                    V3 grad = v3(sw.dw[0][di] * sw.w[1][dj] * sw.w[2][dk], sw.w[0][di] * sw.dw[1][dj] * sw.w[2][dk],
                                 sw.w[0][di] * sw.w[1][dj] * sw.dw[2][dk]);
                    const Node* node =
                        &grid->nodes[gindex(grid, sw.base[0] + di, sw.base[1] + dj, sw.base[2] + dk)];
                    if (node->mass <= kMassEps) continue;
                    vnew = vadd(vnew, vmul(node->vel, w));
                    maddto(&L, mouter(node->vel, grad));
                }
        p->v[i] = vnew;
        p->x[i] = vadd(p->x[i], vmul(vnew, dt));
        p->F[i] = mmul(madd(mident(), mscale(L, dt)), p->F[i]);
        update_stress(st, i, &inverted);
    }
    if (stats) {
        stats->inverted_f = inverted;
        stats->projection_failures = 0;
    }
    return MPMB_OK;
}

/* ref: solvers.hpp:141-198 */
mpmb_status mpmor_step_mls(mpmor_state st, float dt, const float gr[3], int32_t contact,
                           int32_t bc, mpmb_step_stats* stats) {
    int inverted = 0;
    Particles* p = &st->p;
    Grid* grid = &st->grid;
    grid_clear(grid);
    const float m_inv = 4.0f / (grid->dx * grid->dx);
    p2g(st, dt, m_inv, 1);
    grid_velocity_update(st, v3p(gr), dt, contact, bc, 1);
    for (size_t i = 0; i < p->n; ++i) {
        if (!p->active[i]) continue;
        V3 vnew;
        M3 B;
        g2p_gather(grid, p->x[i], &vnew, &B);
        p->v[i] = vnew;
        p->C[i] = mscale(B, m_inv);
        p->x[i] = vadd(p->x[i], vmul(vnew, dt));
        p->F[i] = mmul(madd(mident(), mscale(p->C[i], dt)), p->F[i]);
        update_stress(st, i, &inverted);
    }
    if (stats) {
        stats->inverted_f = inverted;
        stats->projection_failures = 0;
    }
    return MPMB_OK;
}

/* ref: solvers.hpp:207-279 */
mpmb_status mpmor_step_pbmpm(mpmor_state st, float dt, const float gr[3], int32_t iterations,
                             int32_t contact, int32_t bc, mpmb_step_stats* stats) {
    int failures = 0, inverted = 0;
    Particles* p = &st->p;
    Grid* grid = &st->grid;
    const float m_inv = 4.0f / (grid->dx * grid->dx);
    for (int iter = 0; iter < iterations; ++iter) {
        grid_clear(grid);
        p2g(st, dt, m_inv, 0);
        grid_velocity_update(st, v3p(gr), dt, contact, bc, iter == 0);
        for (size_t i = 0; i < p->n; ++i) {
            if (!p->active[i]) continue;
            V3 vnew;
            M3 B;
            g2p_gather(grid, p->x[i], &vnew, &B);
            p->v[i] = vnew;
            M3 Cc = mscale(B, m_inv);
            const mpmb_material* mat = &st->mats[p->mat[i]];
            M3 out;
            if (corotational_project(p->F[i], Cc, dt, mat->beta, &out))
                p->C[i] = out;
            else
                ++failures;
        }
    }
    for (size_t i = 0; i < p->n; ++i) {
        if (!p->active[i]) continue;
        p->x[i] = vadd(p->x[i], vmul(p->v[i], dt));
        p->F[i] = mmul(madd(mident(), mscale(p->C[i], dt)), p->F[i]);
        if (mdet(p->F[i]) <= 0) ++inverted;
    }
    if (stats) {
        stats->inverted_f = inverted;
        stats->projection_failures = failures;
    }
    return MPMB_OK;
}

/* ------------------------------------------------------------ state C-API */
mpmb_status mpmor_state_create(const int32_t dims[3], float dx, const float origin[3],
                               mpmor_state* out) {
    if (dims[0] < 4 || dims[1] < 4 || dims[2] < 4 || !(dx > 0)) return MPMB_INVALID_ARGUMENT;
    struct mpmor_state_s* s = (struct mpmor_state_s*)calloc(1, sizeof *s);
    for (int a = 0; a < 3; ++a) s->grid.dims[a] = dims[a];
    s->grid.dx = dx;
    s->grid.origin = v3p(origin);
    s->grid.n = (size_t)dims[0] * dims[1] * dims[2];
    s->grid.nodes = (Node*)calloc(s->grid.n, sizeof(Node));
    *out = s;
    return MPMB_OK;
}

static void free_shapes(struct mpmor_state_s* s) {
    for (int i = 0; i < s->nshapes; ++i) shape_free(&s->shapes[i]);
    free(s->shapes);
    free(s->acc);
    s->shapes = NULL;
    s->acc = NULL;
    s->nshapes = 0;
}

mpmb_status mpmor_state_destroy(mpmor_state s) {
    if (!s) return MPMB_OK;
    free(s->grid.nodes);
    particles_free(&s->p);
    free(s->mats);
    free_shapes(s);
    free(s);
    return MPMB_OK;
}

mpmb_status mpmor_state_set_materials(mpmor_state s, const mpmb_material* m, int32_t n) {
    free(s->mats);
    s->mats = (mpmb_material*)malloc(sizeof(mpmb_material) * (n ? n : 1));
    memcpy(s->mats, m, sizeof(mpmb_material) * n);
    s->nmats = n;
    return MPMB_OK;
}

mpmb_status mpmor_state_set_particles(mpmor_state s, int32_t n, const float* x, const float* v,
                                      const float* mass, const float* vol0, const float* F,
                                      const float* C, const float* stress, const int32_t* mat,
                                      const uint8_t* active) {
    particles_alloc(&s->p, (size_t)n);
    for (int i = 0; i < n; ++i) {
        s->p.x[i] = v3p(x + 3 * i);
        s->p.v[i] = v3p(v + 3 * i);
        s->p.mass[i] = mass[i];
        s->p.vol0[i] = vol0[i];
        s->p.F[i] = m9(F + 9 * i);
        s->p.C[i] = m9(C + 9 * i);
        s->p.stress[i] = stress ? m9(stress + 9 * i) : mzero();
        s->p.mat[i] = mat[i];
        s->p.active[i] = active[i];
    }
    return MPMB_OK;
}

mpmb_status mpmor_state_get_particles(mpmor_state s, int32_t n, float* x, float* v, float* mass,
                                      float* vol0, float* F, float* C, float* stress,
                                      int32_t* mat, uint8_t* active) {
    if ((size_t)n < s->p.n) return MPMB_BUFFER_TOO_SMALL;
    for (size_t i = 0; i < s->p.n; ++i) {
        if (x) v3put(x + 3 * i, s->p.x[i]);
        if (v) v3put(v + 3 * i, s->p.v[i]);
        if (mass) mass[i] = s->p.mass[i];
        if (vol0) vol0[i] = s->p.vol0[i];
        if (F) m9put(F + 9 * i, s->p.F[i]);
        if (C) m9put(C + 9 * i, s->p.C[i]);
        if (stress) m9put(stress + 9 * i, s->p.stress[i]);
        if (mat) mat[i] = s->p.mat[i];
        if (active) active[i] = s->p.active[i];
    }
    return MPMB_OK;
}

mpmb_status mpmor_state_set_shapes(mpmor_state s, const mpmb_shape_desc* d, int32_t n) {
    free_shapes(s);
    s->shapes = (Shape*)calloc(n ? n : 1, sizeof(Shape));
    s->acc = (Acc*)calloc(n ? n : 1, sizeof(Acc));
    s->nshapes = n;
    for (int i = 0; i < n; ++i) {
        shape_from(&s->shapes[i], &d[i]);
        if (!validate_geometry(&s->shapes[i])) return MPMB_INVALID_ARGUMENT;
    }
    return MPMB_OK;
}

static void pose_put(mpmb_pose* o, const Shape* s) {
    v3put(o->position, s->pos);
    o->orientation[0] = s->rot.x;
    o->orientation[1] = s->rot.y;
    o->orientation[2] = s->rot.z;
    o->orientation[3] = s->rot.w;
    v3put(o->linear_velocity, s->lin);
    v3put(o->angular_velocity, s->ang);
}

mpmb_status mpmor_state_get_shape_poses(mpmor_state s, mpmb_pose* out, int32_t n) {
    for (int i = 0; i < n && i < s->nshapes; ++i) pose_put(&out[i], &s->shapes[i]);
    return MPMB_OK;
}

mpmb_status mpmor_state_get_contact(mpmor_state s, float* imp, float* tq, int32_t* cnt,
                                    int32_t n) {
    for (int i = 0; i < n && i < s->nshapes; ++i) {
        if (imp) v3put(imp + 3 * i, s->acc[i].imp);
        if (tq) v3put(tq + 3 * i, s->acc[i].tq);
        if (cnt) cnt[i] = s->acc[i].count;
    }
    return MPMB_OK;
}

mpmb_status mpmor_state_get_contact_f64(mpmor_state s, double* imp, double* tq, int32_t n) {
    for (int i = 0; i < n && i < s->nshapes; ++i)
        for (int a = 0; a < 3; ++a) {
            if (imp) imp[3 * i + a] = s->acc[i].impd[a];
            if (tq) tq[3 * i + a] = s->acc[i].tqd[a];
        }
    return MPMB_OK;
}

mpmb_status mpmor_state_reset_contact(mpmor_state s) {
    if (s->nshapes && s->acc) memset(s->acc, 0, sizeof(Acc) * s->nshapes);
    return MPMB_OK;
}

mpmb_status mpmor_particle_pushout(mpmor_state s, int32_t* count) {
    int c = pushout(&s->p, s->shapes, s->nshapes, s->grid.dx);
    if (count) *count = c;
    return MPMB_OK;
}

mpmb_status mpmor_deactivate_out_of_domain(mpmor_state s, int32_t* count) {
    int c = deactivate(&s->p, &s->grid);
    if (count) *count = c;
    return MPMB_OK;
}

/* ref: scene.hpp:220-226 (free shapes integrate with their accumulated impulse) */
mpmb_status mpmor_integrate_free_bodies(mpmor_state s, const float g[3], float dt) {
    for (int i = 0; i < s->nshapes; ++i)
        if (s->shapes[i].motion == MPMB_MOTION_FREE_BODY)
            integrate_free_body(&s->shapes[i], s->acc[i].imp, s->acc[i].tq, v3p(g), dt);
    return MPMB_OK;
}

mpmb_status mpmor_state_get_grid(mpmor_state s, float* mass, float* mom, float* vel) {
    for (size_t i = 0; i < s->grid.n; ++i) {
        if (mass) mass[i] = s->grid.nodes[i].mass;
        if (mom) v3put(mom + 3 * i, s->grid.nodes[i].mom);
        if (vel) v3put(vel + 3 * i, s->grid.nodes[i].vel);
    }
    return MPMB_OK;
}

/*
 * Binning oracle (NEW stage; no reference function).  The stencil base cell is the
 * reference's P2G arithmetic (math.hpp:219-223: inv_dx = 1/dx; p = (x - o) * inv_dx;
 * base = (int)floor(p - 0.5)), then bricked: brick b = base >> 2 with nb = ceil(dims/4)
 * bricks per axis, key = (((bz*nby + by)*nbx + bx) << 6) | (lz<<4 | ly<<2 | lx), l = base & 3.
 * perm = original indices stably sorted by key (ties keep original order), inactive last.
 */
mpmb_status mpmor_bin_particles(mpmor_state s, uint32_t* keys, uint32_t* perm) {
    const Grid* g = &s->grid;
    const int nbx = (g->dims[0] + 3) / 4, nby = (g->dims[1] + 3) / 4;
    size_t n = s->p.n;
    uint32_t* k = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    for (size_t i = 0; i < n; ++i) {
        if (!s->p.active[i]) { k[i] = 0xFFFFFFFFu; continue; }
        SW sw = spline_weights(s->p.x[i], g->origin, g->dx);
        int b[3];
        for (int a = 0; a < 3; ++a) b[a] = sw.base[a] < 0 ? 0 : sw.base[a];
        uint32_t brick = (uint32_t)(((b[2] >> 2) * nby + (b[1] >> 2)) * nbx + (b[0] >> 2));
        uint32_t local = (uint32_t)(((b[2] & 3) << 4) | ((b[1] & 3) << 2) | (b[0] & 3));
        k[i] = (brick << 6) | local;
    }
    if (keys) memcpy(keys, k, sizeof(uint32_t) * n);
    if (perm) {
        /* stable insertion into buckets via a merge sort on (key, index) */
        uint32_t* idx = perm;
        for (size_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
        uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
        for (size_t width = 1; width < n; width *= 2) {
            for (size_t lo = 0; lo < n; lo += 2 * width) {
                size_t mid = lo + width < n ? lo + width : n;
                size_t hi = lo + 2 * width < n ? lo + 2 * width : n;
                size_t a = lo, b2 = mid, o = lo;
                while (a < mid && b2 < hi) {
                    if (k[idx[b2]] < k[idx[a]]) tmp[o++] = idx[b2++];
                    else tmp[o++] = idx[a++];
                }
                while (a < mid) tmp[o++] = idx[a++];
                while (b2 < hi) tmp[o++] = idx[b2++];
            }
            memcpy(idx, tmp, sizeof(uint32_t) * n);
        }
        free(tmp);
    }
    free(k);
    return MPMB_OK;
}

/* ------------------------------------------------------------------ scene.hpp */
struct mpmor_scene_s {
    mpmb_scene_config cfg;
    struct mpmor_state_s st;
    Acc* frame_acc;
    int* has_target;
    mpmb_keyframe* target;
    V3* start_pos;
    Q4* start_rot;
    float time;
    int status; /* 0 idle, 1 advancing, 2 ready */
    int inverted, failures, pushed, deactivated;
    int next_shape_id, next_object_id;
};

/* ref: scene.hpp:47-52 */
mpmor_scene mpmor_scene_create(const mpmb_scene_config* c) {
    if (c->substeps < 1 || c->iterations < 1) return NULL;
    struct mpmor_scene_s* s = (struct mpmor_scene_s*)calloc(1, sizeof *s);
    s->cfg = *c;
    mpmor_state tmp;
    if (mpmor_state_create(c->grid_dims, c->dx, c->origin, &tmp) != MPMB_OK) {
        free(s);
        return NULL;
    }
    s->st = *tmp;
    free(tmp);
    return s;
}

void mpmor_scene_destroy(mpmor_scene s) {
    if (!s) return;
    free(s->st.grid.nodes);
    particles_free(&s->st.p);
    free(s->st.mats);
    free_shapes(&s->st);
    free(s->frame_acc);
    free(s->has_target);
    free(s->target);
    free(s->start_pos);
    free(s->start_rot);
    free(s);
}

/* ref: scene.hpp:57-60 */
int32_t mpmor_scene_add_material(mpmor_scene s, const mpmb_material* m) {
    s->st.mats = (mpmb_material*)realloc(s->st.mats, sizeof(mpmb_material) * (s->st.nmats + 1));
    s->st.mats[s->st.nmats] = *m;
    return s->st.nmats++;
}

/* ref: scene.hpp:62-73 */
int32_t mpmor_scene_create_particle_object(mpmor_scene s, const float mn[3], const float mx[3],
                                           int32_t ppc, float density, int32_t mat,
                                           uint64_t seed) {
    if (mat < 0 || mat >= s->st.nmats) return -1;
    if (spawn_box(&s->st.p, &s->st.grid, v3p(mn), v3p(mx), ppc, density, mat, seed) < 0)
        return -1;
    return s->next_object_id++;
}

/* ref: scene.hpp:75-88 */
int32_t mpmor_scene_create_shape(mpmor_scene s, const mpmb_shape_desc* d) {
    int n = s->st.nshapes;
    s->st.shapes = (Shape*)realloc(s->st.shapes, sizeof(Shape) * (n + 1));
    s->st.acc = (Acc*)realloc(s->st.acc, sizeof(Acc) * (n + 1));
    s->frame_acc = (Acc*)realloc(s->frame_acc, sizeof(Acc) * (n + 1));
    s->has_target = (int*)realloc(s->has_target, sizeof(int) * (n + 1));
    s->target = (mpmb_keyframe*)realloc(s->target, sizeof(mpmb_keyframe) * (n + 1));
    s->start_pos = (V3*)realloc(s->start_pos, sizeof(V3) * (n + 1));
    s->start_rot = (Q4*)realloc(s->start_rot, sizeof(Q4) * (n + 1));
    Shape* sh = &s->st.shapes[n];
    shape_from(sh, d);
    if (!validate_geometry(sh) || (sh->motion == MPMB_MOTION_KINEMATIC && sh->nkf < 1)) {
        shape_free(sh);
        return -1;
    }
    for (int i = 1; sh->motion == MPMB_MOTION_KINEMATIC && i < sh->nkf; ++i)
        if (!(sh->kf[i].time > sh->kf[i - 1].time)) {
            shape_free(sh);
            return -1;
        }
    if (sh->hw <= 0) sh->hw = 0.75f * s->st.grid.dx;
    sh->id = s->next_shape_id++;
    if (sh->motion == MPMB_MOTION_KINEMATIC)
        evaluate_trajectory(sh->kf, sh->nkf, s->time, &sh->pos, &sh->rot, &sh->lin, &sh->ang);
    memset(&s->st.acc[n], 0, sizeof(Acc));
    memset(&s->frame_acc[n], 0, sizeof(Acc));
    s->has_target[n] = 0;
    s->st.nshapes = n + 1;
    return sh->id;
}

/* ref: scene.hpp:111-115 */
mpmb_status mpmor_scene_set_pose_target(mpmor_scene s, int32_t id, const float p[3],
                                        const float q[4]) {
    for (int i = 0; i < s->st.nshapes; ++i)
        if (s->st.shapes[i].id == id) {
            Q4 qn = qnormalized(q4p(q));
            s->target[i].time = 0;
            v3put(s->target[i].position, v3p(p));
            s->target[i].orientation[0] = qn.x;
            s->target[i].orientation[1] = qn.y;
            s->target[i].orientation[2] = qn.z;
            s->target[i].orientation[3] = qn.w;
            s->has_target[i] = 1;
            return MPMB_OK;
        }
    return MPMB_INVALID_ARGUMENT;
}

/* ref: scene.hpp:151-174 */
static void update_kinematic(mpmor_scene s, float t, float t0, float fdt) {
    for (int i = 0; i < s->st.nshapes; ++i) {
        Shape* sh = &s->st.shapes[i];
        if (s->has_target[i]) {
            const mpmb_keyframe* tg = &s->target[i];
            float u = clampf_((t - t0) / fdt, 0.0f, 1.0f);
            V3 sp = s->start_pos[i];
            Q4 sr = s->start_rot[i];
            V3 tp = v3p(tg->position);
            Q4 tr = q4p(tg->orientation);
            sh->pos = vadd(sp, vmul(vsub(tp, sp), u));
            sh->rot = qslerp(sr, tr, u);
            sh->lin = vdiv(vsub(tp, sp), fdt);
            Q4 dq = qmul(tr, qconj(sr));
            float angle = 2 * acosf(clampf_(dq.w, -1.0f, 1.0f));
            V3 axis = v3(dq.x, dq.y, dq.z);
            sh->ang = angle > 1e-7f ? vmul(vnormalized(axis), angle / fdt) : v3(0, 0, 0);
        } else if (sh->motion == MPMB_MOTION_KINEMATIC) {
            evaluate_trajectory(sh->kf, sh->nkf, t, &sh->pos, &sh->rot, &sh->lin, &sh->ang);
        }
    }
}

/* ref: scene.hpp:117-123, 176-249 */
mpmb_status mpmor_scene_advance(mpmor_scene s, float dt) {
    if (s->status == 1) return MPMB_LIFECYCLE_ERROR;
    if (dt <= 0) return MPMB_INVALID_ARGUMENT;
    s->status = 1;
    int ns = s->st.nshapes;
    for (int i = 0; i < ns; ++i) memset(&s->frame_acc[i], 0, sizeof(Acc));
    s->inverted = s->failures = s->pushed = s->deactivated = 0;
    for (int i = 0; i < ns; ++i) {
        s->start_pos[i] = s->st.shapes[i].pos;
        s->start_rot[i] = s->st.shapes[i].rot;
    }
    const int pb = s->cfg.solver == MPMB_SOLVER_PBMPM;
    const int n_sub = pb ? 1 : s->cfg.substeps;
    const float dt_sub = dt / (float)n_sub;
    for (int sub = 0; sub < n_sub; ++sub) {
        update_kinematic(s, s->time + (float)sub * dt_sub, s->time, dt);
        mpmor_state_reset_contact(&s->st);
        mpmb_step_stats stt;
        if (pb)
            mpmor_step_pbmpm(&s->st, dt_sub, s->cfg.gravity, s->cfg.iterations, 1,
                             s->cfg.boundary, &stt);
        else if (s->cfg.solver == MPMB_SOLVER_STANDARD)  /* scene.hpp:200-203 */
            mpmor_step_standard(&s->st, dt_sub, s->cfg.gravity, 1, s->cfg.boundary, &stt);
        else
            mpmor_step_mls(&s->st, dt_sub, s->cfg.gravity, 1, s->cfg.boundary, &stt);
        s->inverted += stt.inverted_f;
        s->failures += stt.projection_failures;
        s->pushed += pushout(&s->st.p, s->st.shapes, ns, s->st.grid.dx);
        for (int i = 0; i < ns; ++i) {
            if (s->st.shapes[i].motion == MPMB_MOTION_FREE_BODY)
                integrate_free_body(&s->st.shapes[i], s->st.acc[i].imp, s->st.acc[i].tq,
                                    v3p(s->cfg.gravity), dt_sub);
            s->frame_acc[i].imp = vadd(s->frame_acc[i].imp, s->st.acc[i].imp);
            s->frame_acc[i].tq = vadd(s->frame_acc[i].tq, s->st.acc[i].tq);
            s->frame_acc[i].count += s->st.acc[i].count;
        }
        s->deactivated += deactivate(&s->st.p, &s->st.grid);
    }
    for (int i = 0; i < ns; ++i)
        if (s->has_target[i]) {
            Shape* sh = &s->st.shapes[i];
            sh->pos = v3p(s->target[i].position);
            sh->rot = q4p(s->target[i].orientation);
            sh->lin = v3(0, 0, 0);
            sh->ang = v3(0, 0, 0);
            s->has_target[i] = 0;
        }
    s->time += dt;
    return MPMB_OK;
}

/* ref: scene.hpp:125-130, 251-278 */
mpmb_status mpmor_scene_fetch(mpmor_scene s, mpmb_frame_summary* r) {
    if (s->status != 1) return MPMB_LIFECYCLE_ERROR;
    s->status = 2;
    memset(r, 0, sizeof *r);
    r->time = s->time;
    r->n_particles = (int32_t)s->st.p.n;
    r->n_shapes = s->st.nshapes;
    for (size_t i = 0; i < s->st.p.n; ++i) {
        if (!s->st.p.active[i]) continue;
        double m = s->st.p.mass[i];
        r->total_mass += m;
        r->momentum[0] += m * s->st.p.v[i].x;
        r->momentum[1] += m * s->st.p.v[i].y;
        r->momentum[2] += m * s->st.p.v[i].z;
        r->kinetic_energy += 0.5 * m * (double)vnorm2(s->st.p.v[i]);
    }
    r->pushed_out = s->pushed;
    r->inverted_f = s->inverted;
    r->projection_failures = s->failures;
    r->deactivated = s->deactivated;
    return MPMB_OK;
}

int32_t mpmor_scene_particle_count(mpmor_scene s) { return (int32_t)s->st.p.n; }

mpmb_status mpmor_scene_get_particles(mpmor_scene s, float* x, float* v, float* F, float* C,
                                      uint8_t* active) {
    return mpmor_state_get_particles(&s->st, (int32_t)s->st.p.n, x, v, NULL, NULL, F, C, NULL,
                                     NULL, active);
}

mpmb_status mpmor_scene_shape_results(mpmor_scene s, int32_t* ids, float* imp, float* tq) {
    for (int i = 0; i < s->st.nshapes; ++i) {
        if (ids) ids[i] = s->st.shapes[i].id;
        if (imp) v3put(imp + 3 * i, s->frame_acc[i].imp);
        if (tq) v3put(tq + 3 * i, s->frame_acc[i].tq);
    }
    return MPMB_OK;
}

/* ------------------------------------------------------------ unit-level */
void mpmor_spline_weights(const float pos[3], const float origin[3], float dx, int32_t base[3],
                          float w[9], float dw[9]) {
    SW sw = spline_weights(v3p(pos), v3p(origin), dx);
    for (int a = 0; a < 3; ++a) {
        base[a] = sw.base[a];
        for (int o = 0; o < 3; ++o) { w[3 * a + o] = sw.w[a][o]; dw[3 * a + o] = sw.dw[a][o]; }
    }
}

int32_t mpmor_spline_in_domain(const float pos[3], const float origin[3], float dx,
                               const int32_t dims[3]) {
    return spline_in_domain(v3p(pos), v3p(origin), dx, dims);
}

void mpmor_neo_hookean(const float F[9], float mu, float lambda, float out[9]) {
    m9put(out, neo_hookean(m9(F), mu, lambda));
}

int32_t mpmor_polar(const float M[9], float R[9], float U[9]) {
    M3 r, u;
    if (!polar_decompose(m9(M), &r, &u)) return 0;
    m9put(R, r);
    m9put(U, u);
    return 1;
}

int32_t mpmor_corotational_project(const float Fp[9], const float Cc[9], float dt, float beta,
                                   float out[9]) {
    M3 o;
    if (!corotational_project(m9(Fp), m9(Cc), dt, beta, &o)) return 0;
    m9put(out, o);
    return 1;
}

void mpmor_sdf_query(const mpmb_shape_desc* d, const float point[3], float* distance,
                     float normal[3], float tangent[3], int32_t* region) {
    Shape s;
    shape_from(&s, d);
    Sdf r = sdf_query(&s, v3p(point));
    *distance = r.distance;
    v3put(normal, r.normal);
    v3put(tangent, r.tangent);
    *region = r.region;
    shape_free(&s);
}

void mpmor_evaluate_trajectory(const mpmb_keyframe* kf, int32_t n, float t, mpmb_pose* out) {
    Shape s;
    memset(&s, 0, sizeof s);
    evaluate_trajectory(kf, n, t, &s.pos, &s.rot, &s.lin, &s.ang);
    pose_put(out, &s);
}

int32_t mpmor_spawn_box(const int32_t dims[3], float dx, const float origin[3], const float mn[3],
                        const float mx[3], int32_t ppc, float density, uint64_t seed,
                        int32_t capacity, float* x, float* mass, float* vol0) {
    Grid g;
    memset(&g, 0, sizeof g);
    for (int a = 0; a < 3; ++a) g.dims[a] = dims[a];
    g.dx = dx;
    g.origin = v3p(origin);
    Particles p;
    memset(&p, 0, sizeof p);
    long n = spawn_box(&p, &g, v3p(mn), v3p(mx), ppc, density, 0, seed);
    if (n < 0) { particles_free(&p); return -1; }
    if (n > capacity) { particles_free(&p); return -2; }
    for (long i = 0; i < n; ++i) {
        if (x) v3put(x + 3 * i, p.x[i]);
        if (mass) mass[i] = p.mass[i];
        if (vol0) vol0[i] = p.vol0[i];
    }
    particles_free(&p);
    return (int32_t)n;
}
