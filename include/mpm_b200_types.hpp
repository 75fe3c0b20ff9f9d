// mpm_b200_types.hpp — conversions between the reference's value types (proj/include/mpm:
// Vec3, Quat, Shape, Material, ShapePose) and the flat C structs of include/mpm_b200.h.
// Shared by the two C++ drop-ins (mpm_b200_facade.hpp, mpm_b200_solver.hpp).
#pragma once
#include <type_traits>
#include <variant>
#include <vector>

#include "mpm/rigid_dynamics.hpp"  // reference value types (header-only, unchanged)
#include "mpm/materials.hpp"
#include "mpm_b200.h"

namespace mpm_b200::detail {

inline void put3(float* o, const mpm::Vec3& v) { o[0] = v.x; o[1] = v.y; o[2] = v.z; }
inline void put4(float* o, const mpm::Quat& q) { o[0] = q.x; o[1] = q.y; o[2] = q.z; o[3] = q.w; }
inline mpm::Vec3 get3(const float* i) { return {i[0], i[1], i[2]}; }
inline mpm::Quat get4(const float* i) {
    mpm::Quat q;
    q.x = i[0];
    q.y = i[1];
    q.z = i[2];
    q.w = i[3];
    return q;
}

inline mpmb_pose pose(const mpm::ShapePose& p) {
    mpmb_pose o{};
    put3(o.position, p.position);
    put4(o.orientation, p.orientation);
    put3(o.linear_velocity, p.linear_velocity);
    put3(o.angular_velocity, p.angular_velocity);
    return o;
}

inline mpm::ShapePose pose(const mpmb_pose& p) {
    mpm::ShapePose o;
    o.position = get3(p.position);
    o.orientation = get4(p.orientation);
    o.linear_velocity = get3(p.linear_velocity);
    o.angular_velocity = get3(p.angular_velocity);
    return o;
}

inline mpmb_material material(const mpm::Material& m) {
    return mpmb_material{m.kind == mpm::MaterialKind::corotational_pb ? MPMB_MAT_COROTATIONAL_PB : MPMB_MAT_NEO_HOOKEAN,
                         m.mu, m.lambda, m.beta};
}

// mpm::Shape -> mpmb_shape_desc; the desc points into `store`, which must outlive its use
struct ShapeStore {
    std::vector<float> verts;
    std::vector<mpmb_keyframe> kf;
};

inline mpmb_shape_desc shape(const mpm::Shape& s, ShapeStore& store) {
    mpmb_shape_desc d{};
    store.verts.clear();
    store.kf.clear();
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
                put3(d.gparam, g.half_extents);
            } else if constexpr (std::is_same_v<T, mpm::QuadSlicerGeom>) {
                d.geometry = MPMB_GEOM_QUAD_SLICER;
                d.gparam[0] = g.half_length;
                d.gparam[1] = g.half_height;
                d.gparam[2] = g.spine_radius;
            } else if constexpr (std::is_same_v<T, mpm::TriangleMeshSlicerGeom>) {
                d.geometry = MPMB_GEOM_TRI_MESH_SLICER;
                d.gparam[0] = g.spine_radius;
                for (const auto& v : g.vertices) store.verts.insert(store.verts.end(), {v.x, v.y, v.z});
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
                for (const auto& v : g.vertices) store.verts.insert(store.verts.end(), {v.x, v.y, v.z});
            }
        },
        s.geometry);
    d.vertices = store.verts.empty() ? nullptr : store.verts.data();
    d.n_vertices = static_cast<int32_t>(store.verts.size() / 3);
    d.pose = pose(s.pose);
    d.mu_k = s.mu_k;
    d.c_d = s.c_d;
    d.collision_halfwidth = s.collision_halfwidth;
    d.motion = s.motion == mpm::MotionKind::kinematic   ? MPMB_MOTION_KINEMATIC
               : s.motion == mpm::MotionKind::free_body ? MPMB_MOTION_FREE_BODY
                                                        : MPMB_MOTION_FIXED;
    for (const auto& k : s.trajectory.keyframes) {
        mpmb_keyframe e{};
        e.time = k.time;
        put3(e.position, k.position);
        put4(e.orientation, k.orientation);
        store.kf.push_back(e);
    }
    d.keyframes = store.kf.empty() ? nullptr : store.kf.data();
    d.n_keyframes = static_cast<int32_t>(store.kf.size());
    d.body_mass = s.body.mass;
    put3(d.inertia, s.body.inertia_diag);
    return d;
}

}  // namespace mpm_b200::detail
