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
#include "mpm_b200_types.hpp"

namespace mpm_b200::facade {

using Handle = mpmb_handle;  // facade.hpp:15
inline constexpr Handle kInvalidHandle = MPMB_INVALID_HANDLE;
using Status = mpm::facade::Status;  // facade.hpp:18-24 (plus device errors -> invalid_argument)

namespace detail {
using ::mpm_b200::detail::material;
using ::mpm_b200::detail::put3;
using ::mpm_b200::detail::put4;
using ::mpm_b200::detail::shape;
using ::mpm_b200::detail::ShapeStore;
inline Status status(mpmb_status s) {
    switch (s) {
        case MPMB_OK: return Status::ok;
        case MPMB_BAD_HANDLE: return Status::bad_handle;
        case MPMB_LIFECYCLE_ERROR: return Status::lifecycle_error;
        case MPMB_BUFFER_TOO_SMALL: return Status::buffer_too_small;
        default: return Status::invalid_argument;
    }
}
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
    const mpmb_material k = detail::material(m);
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
    detail::ShapeStore store;
    const mpmb_shape_desc d = detail::shape(s, store);
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
