// mpm_b200_facade.hpp — drop-in for mpm::facade (proj/include/mpm/facade.hpp:67-219).
//
// Same function names, argument types and Status codes as the reference facade, implemented
// over the C-ABI of include/mpm_b200.h (the B200 engine).  The reference's own headers supply
// the value types (mpm::SceneConfig, mpm::Material, mpm::Shape, mpm::FrameResult, Vec3, Quat):
// build with -I<reference>/proj/include -I<this repo>/include and link libmpm_b200.so.
// Switching a caller is one line:   namespace facade = mpm_b200::facade;
#pragma once
#include <cstdint>
#include <type_traits>
#include <variant>
#include <vector>

#include "mpm/facade.hpp"  // reference value types + Status (header-only, unchanged)
#include "mpm_b200.h"

namespace mpm_b200::facade {

using Handle = mpmb_handle;  // facade.hpp:15
inline constexpr Handle kInvalidHandle = MPMB_INVALID_HANDLE;
using Status = mpm::facade::Status;  // facade.hpp:18-24 (plus device errors -> invalid_argument)

namespace detail {
inline Status status(mpmb_status s) {
    switch (s) {
        case MPMB_OK: return Status::ok;
        case MPMB_BAD_HANDLE: return Status::bad_handle;
        case MPMB_LIFECYCLE_ERROR: return Status::lifecycle_error;
        case MPMB_BUFFER_TOO_SMALL: return Status::buffer_too_small;
        default: return Status::invalid_argument;
    }
}
inline void put3(float* o, const mpm::Vec3& v) { o[0] = v.x; o[1] = v.y; o[2] = v.z; }
inline void put4(float* o, const mpm::Quat& q) { o[0] = q.x; o[1] = q.y; o[2] = q.z; o[3] = q.w; }
}  // namespace detail

inline Handle create_scene(const mpm::SceneConfig& c) {
    mpmb_scene_config k{};
    k.solver = static_cast<int32_t>(c.solver);
    k.substeps = c.substeps;
    k.iterations = c.iterations;
    detail::put3(k.gravity, c.gravity);
    for (int a = 0; a < 3; ++a) k.grid_dims[a] = c.grid_dims[a];
    k.dx = c.dx;
    detail::put3(k.origin, c.origin);
    k.boundary = c.boundary == mpm::BoundaryKind::sticky ? MPMB_BC_STICKY : MPMB_BC_SLIP;
    return mpmb_create_scene(&k);
}

inline Status destroy(Handle h) { return detail::status(mpmb_destroy(h)); }

inline Handle create_material(Handle scene, const mpm::Material& m) {
    mpmb_material k{m.kind == mpm::MaterialKind::corotational_pb ? MPMB_MAT_COROTATIONAL_PB
                                                                 : MPMB_MAT_NEO_HOOKEAN,
                    m.mu, m.lambda, m.beta};
    return mpmb_create_material(scene, &k);
}

inline Handle create_particle_object(Handle scene, Handle material, const mpm::Vec3& mn,
                                     const mpm::Vec3& mx, int particles_per_cell, mpm::Real density,
                                     uint64_t seed) {
    float a[3], b[3];
    detail::put3(a, mn);
    detail::put3(b, mx);
    return mpmb_create_particle_object(scene, material, a, b, particles_per_cell, density, seed);
}

inline Handle create_shape(Handle scene, const mpm::Shape& s) {
    mpmb_shape_desc d{};
    std::vector<float> verts;
    std::visit(
        [&](const auto& g) {
            using T = std::decay_t<decltype(g)>;
            if constexpr (std::is_same_v<T, mpm::PlaneGeom>) {
                d.geometry = MPMB_GEOM_PLANE;
            } else if constexpr (std::is_same_v<T, mpm::SphereGeom>) {
                d.geometry = MPMB_GEOM_SPHERE;
                d.gparam[0] = g.radius;
            } else if constexpr (std::is_same_v<T, mpm::BoxGeom>) {
                d.geometry = MPMB_GEOM_BOX;
                detail::put3(d.gparam, g.half_extents);
            } else if constexpr (std::is_same_v<T, mpm::QuadSlicerGeom>) {
                d.geometry = MPMB_GEOM_QUAD_SLICER;
                d.gparam[0] = g.half_length;
                d.gparam[1] = g.half_height;
                d.gparam[2] = g.spine_radius;
            } else if constexpr (std::is_same_v<T, mpm::TriangleMeshSlicerGeom>) {
                d.geometry = MPMB_GEOM_TRI_MESH_SLICER;
                d.gparam[0] = g.spine_radius;
                for (const auto& v : g.vertices) verts.insert(verts.end(), {v.x, v.y, v.z});
                d.indices = g.indices.data();
                d.n_indices = static_cast<int32_t>(g.indices.size());
                d.spine_edges = g.spine_edges.data();
                d.n_spine_edges = static_cast<int32_t>(g.spine_edges.size());
            } else if constexpr (std::is_same_v<T, mpm::ArcGeom>) {
                d.geometry = MPMB_GEOM_ARC;
                d.gparam[0] = g.radius;
                d.gparam[1] = g.angle;
            } else {
                d.geometry = MPMB_GEOM_POLYLINE;
                for (const auto& v : g.vertices) verts.insert(verts.end(), {v.x, v.y, v.z});
            }
        },
        s.geometry);
    d.vertices = verts.empty() ? nullptr : verts.data();
    d.n_vertices = static_cast<int32_t>(verts.size() / 3);
    detail::put3(d.pose.position, s.pose.position);
    detail::put4(d.pose.orientation, s.pose.orientation);
    detail::put3(d.pose.linear_velocity, s.pose.linear_velocity);
    detail::put3(d.pose.angular_velocity, s.pose.angular_velocity);
    d.mu_k = s.mu_k;
    d.c_d = s.c_d;
    d.collision_halfwidth = s.collision_halfwidth;
    d.motion = s.motion == mpm::MotionKind::kinematic   ? MPMB_MOTION_KINEMATIC
               : s.motion == mpm::MotionKind::free_body ? MPMB_MOTION_FREE_BODY
                                                        : MPMB_MOTION_FIXED;
    std::vector<mpmb_keyframe> kf;
    for (const auto& k : s.trajectory.keyframes) {
        mpmb_keyframe e{};
        e.time = k.time;
        detail::put3(e.position, k.position);
        detail::put4(e.orientation, k.orientation);
        kf.push_back(e);
    }
    d.keyframes = kf.empty() ? nullptr : kf.data();
    d.n_keyframes = static_cast<int32_t>(kf.size());
    d.body_mass = s.body.mass;
    detail::put3(d.inertia, s.body.inertia_diag);
    return mpmb_create_shape(scene, &d);
}

inline Status set_shape_pose_target(Handle scene, Handle shape, const mpm::Vec3& p, const mpm::Quat& q) {
    float a[3], b[4];
    detail::put3(a, p);
    detail::put4(b, q);
    return detail::status(mpmb_set_shape_pose_target(scene, shape, a, b));
}

inline Status advance(Handle scene, mpm::Real dt) { return detail::status(mpmb_advance(scene, dt)); }

inline Status fetch_results(Handle scene, mpm::FrameResult& out) {
    mpmb_frame_summary s{};
    mpmb_status st = mpmb_fetch_results(scene, &s);
    if (st != MPMB_OK) return detail::status(st);
    std::vector<float> x(3 * s.n_particles), v(3 * s.n_particles), imp(3 * s.n_shapes), tq(3 * s.n_shapes);
    out.active.assign(s.n_particles, 0);
    out.shape_ids.assign(s.n_shapes, 0);
    st = mpmb_result_copy(scene, x.data(), v.data(), out.active.data(), out.shape_ids.data(), imp.data(),
                          tq.data());
    if (st != MPMB_OK) return detail::status(st);
    out.time = s.time;
    out.positions.resize(s.n_particles);
    out.velocities.resize(s.n_particles);
    for (int i = 0; i < s.n_particles; ++i) {
        out.positions[i] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
        out.velocities[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
    }
    out.shape_impulses.resize(s.n_shapes);
    out.shape_torque_impulses.resize(s.n_shapes);
    for (int i = 0; i < s.n_shapes; ++i) {
        out.shape_impulses[i] = {imp[3 * i], imp[3 * i + 1], imp[3 * i + 2]};
        out.shape_torque_impulses[i] = {tq[3 * i], tq[3 * i + 1], tq[3 * i + 2]};
    }
    out.total_mass = s.total_mass;
    for (int a = 0; a < 3; ++a) out.momentum[a] = s.momentum[a];
    out.kinetic_energy = s.kinetic_energy;
    out.pushed_out = s.pushed_out;
    out.inverted_f = s.inverted_f;
    out.projection_failures = s.projection_failures;
    out.deactivated = s.deactivated;
    return Status::ok;
}

inline int particle_count(Handle scene) { return mpmb_particle_count(scene); }

inline Status copy_positions(Handle scene, float* out, size_t capacity_floats, size_t& written) {
    return detail::status(mpmb_copy_positions(scene, out, capacity_floats, &written));
}

inline Status shape_impulse(Handle scene, Handle shape, mpm::Vec3& out) {
    float o[3];
    mpmb_status st = mpmb_shape_impulse(scene, shape, o);
    if (st == MPMB_OK) out = {o[0], o[1], o[2]};
    return detail::status(st);
}

}  // namespace mpm_b200::facade
