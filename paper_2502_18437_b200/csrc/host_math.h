// host_math.h — host-side float math that must stay bit-identical to the reference:
// kinematic shape poses (rigid_dynamics.hpp:31-73, scene.hpp:151-174) and particle
// spawning (state.hpp:101-149).  Compiled with -ffp-contract=off like the reference
// (x86-64, no FMA), so the device receives exactly the reference's inputs.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/mpm_b200.h"

namespace mpmb::host {

struct V3 { float x = 0, y = 0, z = 0; };
struct Q4 { float x = 0, y = 0, z = 0, w = 1; };

inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 mul(V3 a, float s) { return {a.x * s, a.y * s, a.z * s}; }
inline V3 div(V3 a, float s) { return {a.x / s, a.y / s, a.z / s}; }
inline float norm(V3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }
inline V3 normalized(V3 a) {  // math.hpp:35-38
    float n = norm(a);
    return n > 0.f ? div(a, n) : V3{1, 0, 0};
}
inline Q4 qnormalized(Q4 q) {  // math.hpp:145-149
    float n = std::sqrt(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w);
    if (n <= 0.f) return Q4{};
    return {q.x / n, q.y / n, q.z / n, q.w / n};
}
inline Q4 qconj(Q4 q) { return {-q.x, -q.y, -q.z, q.w}; }
inline Q4 qmul(Q4 a, Q4 o) {  // math.hpp:151-156
    return {a.w * o.x + a.x * o.w + a.y * o.z - a.z * o.y,
            a.w * o.y - a.x * o.z + a.y * o.w + a.z * o.x,
            a.w * o.z + a.x * o.y - a.y * o.x + a.z * o.w,
            a.w * o.w - a.x * o.x - a.y * o.y - a.z * o.z};
}
inline Q4 slerp(Q4 a, Q4 b, float t) {  // math.hpp:175-192
    float c = a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
    if (c < 0) {
        b = {-b.x, -b.y, -b.z, -b.w};
        c = -c;
    }
    if (c > 0.9995f)
        return qnormalized({a.x + t * (b.x - a.x), a.y + t * (b.y - a.y), a.z + t * (b.z - a.z),
                            a.w + t * (b.w - a.w)});
    float th = std::acos(c);
    float sa = std::sin((1 - t) * th) / std::sin(th);
    float sb = std::sin(t * th) / std::sin(th);
    return {sa * a.x + sb * b.x, sa * a.y + sb * b.y, sa * a.z + sb * b.z, sa * a.w + sb * b.w};
}

struct Pose { V3 pos; Q4 rot; V3 lin; V3 ang; };

inline V3 v3(const float* p) { return {p[0], p[1], p[2]}; }
inline Q4 q4(const float* p) { return {p[0], p[1], p[2], p[3]}; }

// rigid_dynamics.hpp:31-51
inline void interp_pose(const std::vector<mpmb_keyframe>& kf, float t, V3& pos, Q4& rot) {
    if (t <= kf.front().time) {
        pos = v3(kf.front().position);
        rot = q4(kf.front().orientation);
        return;
    }
    if (t >= kf.back().time) {
        pos = v3(kf.back().position);
        rot = q4(kf.back().orientation);
        return;
    }
    size_t hi = 1;
    while (kf[hi].time < t) ++hi;
    const mpmb_keyframe& a = kf[hi - 1];
    const mpmb_keyframe& b = kf[hi];
    float u = (t - a.time) / (b.time - a.time);
    pos = add(v3(a.position), mul(sub(v3(b.position), v3(a.position)), u));
    rot = slerp(q4(a.orientation), q4(b.orientation), u);
}

// rigid_dynamics.hpp:57-73
inline Pose evaluate_trajectory(const std::vector<mpmb_keyframe>& kf, float t) {
    Pose p;
    interp_pose(kf, t, p.pos, p.rot);
    const float h = 1e-4f;
    V3 p0, p1;
    Q4 q0, q1;
    interp_pose(kf, t - h, p0, q0);
    interp_pose(kf, t + h, p1, q1);
    p.lin = div(sub(p1, p0), 2 * h);
    Q4 dq{(q1.x - q0.x) / (2 * h), (q1.y - q0.y) / (2 * h), (q1.z - q0.z) / (2 * h),
          (q1.w - q0.w) / (2 * h)};
    Q4 w = qmul(dq, qconj(p.rot));
    p.ang = mul(V3{w.x, w.y, w.z}, 2.0f);
    return p;
}

// scene.hpp:154-169: linear drive toward a one-shot pose target over the frame
inline Pose target_drive(V3 start_pos, Q4 start_rot, V3 tpos, Q4 trot, float t, float t0,
                         float fdt) {
    Pose p;
    float u = std::clamp((t - t0) / fdt, 0.0f, 1.0f);
    p.pos = add(start_pos, mul(sub(tpos, start_pos), u));
    p.rot = slerp(start_rot, trot, u);
    p.lin = div(sub(tpos, start_pos), fdt);
    Q4 dq = qmul(trot, qconj(start_rot));
    float angle = 2 * std::acos(std::clamp(dq.w, -1.0f, 1.0f));
    V3 axis{dq.x, dq.y, dq.z};
    p.ang = angle > 1e-7f ? mul(normalized(axis), angle / fdt) : V3{};
    return p;
}

// math.hpp:343-356
struct SplitMix64 {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double next_signed_unit() { return (next() >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0; }
};

// math.hpp:203-213
inline bool spline_in_domain(V3 p, V3 o, float dx, const int dims[3]) {
    const float q[3] = {(p.x - o.x) / dx, (p.y - o.y) / dx, (p.z - o.z) / dx};
    for (int a = 0; a < 3; ++a) {
        int base = static_cast<int>(std::floor(q[a] - 0.5f));
        if (base < 0 || base + 2 > dims[a] - 1) return false;
    }
    return true;
}

// state.hpp:101-149; appends positions / mass / volume; returns false when invalid
inline bool spawn_box(const int dims[3], float dx, V3 origin, V3 mn, V3 mx, int ppc, float density,
                      uint64_t seed, std::vector<float>& x, std::vector<float>& mass,
                      std::vector<float>& vol0) {
    V3 ext = sub(mx, mn);
    if (ext.x <= 0 || ext.y <= 0 || ext.z <= 0 || ppc < 1 || density <= 0) return false;
    if (!spline_in_domain(mn, origin, dx, dims) || !spline_in_domain(mx, origin, dx, dims)) return false;
    const float spacing = dx / std::cbrt(static_cast<float>(ppc));
    const float pm = density * spacing * spacing * spacing;
    const float pv = spacing * spacing * spacing;
    const int nx = std::max(1, static_cast<int>(std::lround(ext.x / spacing)));
    const int ny = std::max(1, static_cast<int>(std::lround(ext.y / spacing)));
    const int nz = std::max(1, static_cast<int>(std::lround(ext.z / spacing)));
    SplitMix64 rng{seed};
    const float jitter = 0.25f * spacing;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                V3 p = add(mn, V3{(static_cast<float>(i) + 0.5f) * spacing,
                                  (static_cast<float>(j) + 0.5f) * spacing,
                                  (static_cast<float>(k) + 0.5f) * spacing});
                p.x += jitter * static_cast<float>(rng.next_signed_unit());
                p.y += jitter * static_cast<float>(rng.next_signed_unit());
                p.z += jitter * static_cast<float>(rng.next_signed_unit());
                x.push_back(p.x);
                x.push_back(p.y);
                x.push_back(p.z);
                mass.push_back(pm);
                vol0.push_back(pv);
            }
    return true;
}

}  // namespace mpmb::host
