// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Compiles the UNMODIFIED reference headers from /root/reference/proj/include
// (header-only C++20 CPU implementation of CRESSim-MPM) into
// oracle/_ref/libmpmref.so and exposes them through the same C-ABI shapes as
// include/mpm_b200.h, with the prefix mpmref_.  Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference legs may load the result.
//
// Build: oracle/Makefile (g++ -std=c++20 -O3 -DNDEBUG, no -march, no fast-math:
// the x86-64 baseline has no FMA, so the reference arithmetic is contraction-free).
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "mpm/facade.hpp"
#include "mpm/scenario.hpp"
#include "mpm/scene_spec.hpp"
#include "mpm_b200.h"

using namespace mpm;

namespace {

thread_local std::string g_err;

Vec3 v3(const float* p) { return Vec3{p[0], p[1], p[2]}; }
void put3(float* o, const Vec3& v) { o[0] = v.x; o[1] = v.y; o[2] = v.z; }
Quat q4(const float* p) { Quat q; q.x = p[0]; q.y = p[1]; q.z = p[2]; q.w = p[3]; return q; }
Mat3 m9(const float* p) {
    Mat3 m;
    for (int i = 0; i < 9; ++i) m.m[i / 3][i % 3] = p[i];
    return m;
}
void put9(float* o, const Mat3& m) {
    for (int i = 0; i < 9; ++i) o[i] = m.m[i / 3][i % 3];
}

ShapePose pose_from(const mpmb_pose& p) {
    ShapePose s;
    s.position = v3(p.position);
    s.orientation = q4(p.orientation);
    s.linear_velocity = v3(p.linear_velocity);
    s.angular_velocity = v3(p.angular_velocity);
    return s;
}
void pose_to(mpmb_pose& o, const ShapePose& s) {
    put3(o.position, s.position);
    o.orientation[0] = s.orientation.x; o.orientation[1] = s.orientation.y;
    o.orientation[2] = s.orientation.z; o.orientation[3] = s.orientation.w;
    put3(o.linear_velocity, s.linear_velocity);
    put3(o.angular_velocity, s.angular_velocity);
}

Geometry geom_from(const mpmb_shape_desc& d) {
    switch (d.geometry) {
        case MPMB_GEOM_PLANE: return PlaneGeom{};
        case MPMB_GEOM_SPHERE: return SphereGeom{d.gparam[0]};
        case MPMB_GEOM_BOX: return BoxGeom{Vec3{d.gparam[0], d.gparam[1], d.gparam[2]}};
        case MPMB_GEOM_QUAD_SLICER:
            return QuadSlicerGeom{d.gparam[0], d.gparam[1], d.gparam[2]};
        case MPMB_GEOM_TRI_MESH_SLICER: {
            TriangleMeshSlicerGeom g;
            for (int i = 0; i < d.n_vertices; ++i) g.vertices.push_back(v3(d.vertices + 3 * i));
            g.indices.assign(d.indices, d.indices + d.n_indices);
            g.spine_edges.assign(d.spine_edges, d.spine_edges + d.n_spine_edges);
            g.spine_radius = d.gparam[0];
            return g;
        }
        case MPMB_GEOM_ARC: return ArcGeom{d.gparam[0], d.gparam[1]};
        case MPMB_GEOM_POLYLINE: {
            ConnectedLineSegmentsGeom g;
            for (int i = 0; i < d.n_vertices; ++i) g.vertices.push_back(v3(d.vertices + 3 * i));
            return g;
        }
    }
    throw std::invalid_argument("unknown geometry kind");
}

Shape shape_from(const mpmb_shape_desc& d) {
    Shape s;
    s.geometry = geom_from(d);
    s.pose = pose_from(d.pose);
    s.mu_k = d.mu_k;
    s.c_d = d.c_d;
    s.collision_halfwidth = d.collision_halfwidth;
    s.motion = d.motion == MPMB_MOTION_KINEMATIC ? MotionKind::kinematic
               : d.motion == MPMB_MOTION_FREE_BODY ? MotionKind::free_body
                                                   : MotionKind::fixed;
    for (int i = 0; i < d.n_keyframes; ++i) {
        Keyframe k;
        k.time = d.keyframes[i].time;
        k.position = v3(d.keyframes[i].position);
        k.orientation = q4(d.keyframes[i].orientation);
        s.trajectory.keyframes.push_back(k);
    }
    s.body.mass = d.body_mass;
    s.body.inertia_diag = v3(d.inertia);
    return s;
}

struct RefState {
    SimState sim;
    std::vector<Shape> shapes;
    std::vector<ContactAccumulator> acc;
};

SceneConfig config_from(const mpmb_scene_config& c) {
    SceneConfig s;
    s.solver = c.solver == MPMB_SOLVER_STANDARD ? SolverKind::standard
               : c.solver == MPMB_SOLVER_PBMPM  ? SolverKind::pbmpm
                                                : SolverKind::mls;
    s.substeps = c.substeps;
    s.iterations = c.iterations;
    s.gravity = v3(c.gravity);
    for (int a = 0; a < 3; ++a) s.grid_dims[a] = c.grid_dims[a];
    s.dx = c.dx;
    s.origin = v3(c.origin);
    s.boundary = c.boundary == MPMB_BC_STICKY ? BoundaryKind::sticky : BoundaryKind::slip;
    return s;
}

// Last fetched FrameResult per scene handle (facade returns it by value).
std::unordered_map<uint64_t, FrameResult>& results() {
    static std::unordered_map<uint64_t, FrameResult> r;
    return r;
}

mpmb_status map_status(facade::Status s) {
    switch (s) {
        case facade::Status::ok: return MPMB_OK;
        case facade::Status::bad_handle: return MPMB_BAD_HANDLE;
        case facade::Status::lifecycle_error: return MPMB_LIFECYCLE_ERROR;
        case facade::Status::invalid_argument: return MPMB_INVALID_ARGUMENT;
        case facade::Status::buffer_too_small: return MPMB_BUFFER_TOO_SMALL;
    }
    return MPMB_INVALID_ARGUMENT;
}

Scene* scene_ptr(uint64_t h) { return facade::detail::registry().scene_of(h); }

}  // namespace

extern "C" {

const char* mpmref_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------ solver layer
mpmb_status mpmref_state_create(const int32_t dims[3], float dx, const float origin[3],
                                void** out) {
    try {
        auto* s = new RefState;
        s->sim.grid = Grid(dims[0], dims[1], dims[2], dx, v3(origin));
        *out = s;
        return MPMB_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return MPMB_INVALID_ARGUMENT;
    }
}

mpmb_status mpmref_state_destroy(void* st) {
    delete static_cast<RefState*>(st);
    return MPMB_OK;
}

mpmb_status mpmref_state_set_materials(void* st, const mpmb_material* m, int32_t n) {
    auto* s = static_cast<RefState*>(st);
    s->sim.materials.clear();
    for (int i = 0; i < n; ++i) {
        Material mat;
        mat.kind = m[i].kind == MPMB_MAT_COROTATIONAL_PB ? MaterialKind::corotational_pb
                                                         : MaterialKind::neo_hookean;
        mat.mu = m[i].mu;
        mat.lambda = m[i].lambda;
        mat.beta = m[i].beta;
        s->sim.materials.push_back(mat);
    }
    return MPMB_OK;
}

mpmb_status mpmref_state_set_particles(void* st, int32_t n, const float* x, const float* v,
                                       const float* mass, const float* vol0, const float* F,
                                       const float* C, const float* stress, const int32_t* mat,
                                       const uint8_t* active) {
    auto& p = static_cast<RefState*>(st)->sim.particles;
    p = ParticleStore{};
    for (int i = 0; i < n; ++i) {
        p.push_back(v3(x + 3 * i), v3(v + 3 * i), mass[i], vol0[i], mat[i]);
        p.F[i] = m9(F + 9 * i);
        p.C[i] = m9(C + 9 * i);
        if (stress) p.stress[i] = m9(stress + 9 * i);
        p.active[i] = active[i];
    }
    return MPMB_OK;
}

mpmb_status mpmref_state_get_particles(void* st, int32_t n, float* x, float* v, float* mass,
                                       float* vol0, float* F, float* C, float* stress,
                                       int32_t* mat, uint8_t* active) {
    auto& p = static_cast<RefState*>(st)->sim.particles;
    if (n < static_cast<int32_t>(p.size())) return MPMB_BUFFER_TOO_SMALL;
    for (size_t i = 0; i < p.size(); ++i) {
        if (x) put3(x + 3 * i, p.x[i]);
        if (v) put3(v + 3 * i, p.v[i]);
        if (mass) mass[i] = p.mass[i];
        if (vol0) vol0[i] = p.volume0[i];
        if (F) put9(F + 9 * i, p.F[i]);
        if (C) put9(C + 9 * i, p.C[i]);
        if (stress) put9(stress + 9 * i, p.stress[i]);
        if (mat) mat[i] = p.material_id[i];
        if (active) active[i] = p.active[i];
    }
    return MPMB_OK;
}

mpmb_status mpmref_state_set_shapes(void* st, const mpmb_shape_desc* d, int32_t n) {
    auto* s = static_cast<RefState*>(st);
    try {
        s->shapes.clear();
        for (int i = 0; i < n; ++i) {
            Shape sh = shape_from(d[i]);
            validate_geometry(sh.geometry);
            s->shapes.push_back(std::move(sh));
        }
        s->acc.assign(n, ContactAccumulator{});
    } catch (const std::exception& e) {
        g_err = e.what();
        return MPMB_INVALID_ARGUMENT;
    }
    return MPMB_OK;
}

mpmb_status mpmref_state_get_shape_poses(void* st, mpmb_pose* out, int32_t n) {
    auto* s = static_cast<RefState*>(st);
    for (int i = 0; i < n && i < static_cast<int>(s->shapes.size()); ++i)
        pose_to(out[i], s->shapes[i].pose);
    return MPMB_OK;
}

mpmb_status mpmref_state_get_contact(void* st, float* imp, float* tq, int32_t* cnt, int32_t n) {
    auto* s = static_cast<RefState*>(st);
    for (int i = 0; i < n && i < static_cast<int>(s->acc.size()); ++i) {
        if (imp) put3(imp + 3 * i, s->acc[i].impulse);
        if (tq) put3(tq + 3 * i, s->acc[i].torque_impulse);
        if (cnt) cnt[i] = s->acc[i].contact_node_count;
    }
    return MPMB_OK;
}

mpmb_status mpmref_state_reset_contact(void* st) {
    auto* s = static_cast<RefState*>(st);
    for (auto& a : s->acc) a.reset();
    return MPMB_OK;
}

mpmb_status mpmref_step_mls(void* st, float dt, const float g[3], int32_t contact, int32_t bc,
                            mpmb_step_stats* stats) {
    auto* s = static_cast<RefState*>(st);
    GridHook hook = nullptr;
    if (contact) hook = [s](Grid& grid) { apply_contact_pass(grid, s->shapes, s->acc); };
    StepStats r = step_mls(s->sim, dt, v3(g), hook,
                           bc == MPMB_BC_STICKY ? BoundaryKind::sticky : BoundaryKind::slip);
    if (stats) { stats->inverted_f = r.inverted_f; stats->projection_failures = r.projection_failures; }
    return MPMB_OK;
}

mpmb_status mpmref_step_standard(void* st, float dt, const float g[3], int32_t contact, int32_t bc,
                                 mpmb_step_stats* stats) {
    auto* s = static_cast<RefState*>(st);
    GridHook hook = nullptr;
    if (contact) hook = [s](Grid& grid) { apply_contact_pass(grid, s->shapes, s->acc); };
    StepStats r = step_standard(s->sim, dt, v3(g), hook,
                                bc == MPMB_BC_STICKY ? BoundaryKind::sticky : BoundaryKind::slip);
    if (stats) { stats->inverted_f = r.inverted_f; stats->projection_failures = r.projection_failures; }
    return MPMB_OK;
}

mpmb_status mpmref_step_pbmpm(void* st, float dt, const float g[3], int32_t iters,
                              int32_t contact, int32_t bc, mpmb_step_stats* stats) {
    auto* s = static_cast<RefState*>(st);
    GridHook hook = nullptr;
    if (contact) hook = [s](Grid& grid) { apply_contact_pass(grid, s->shapes, s->acc); };
    StepStats r = step_pbmpm(s->sim, dt, v3(g), PbmpmConfig{iters}, hook,
                             bc == MPMB_BC_STICKY ? BoundaryKind::sticky : BoundaryKind::slip);
    if (stats) { stats->inverted_f = r.inverted_f; stats->projection_failures = r.projection_failures; }
    return MPMB_OK;
}

mpmb_status mpmref_particle_pushout(void* st, int32_t* count) {
    auto* s = static_cast<RefState*>(st);
    int c = particle_pushout(s->sim.particles, s->shapes, s->sim.grid.dx);
    if (count) *count = c;
    return MPMB_OK;
}

mpmb_status mpmref_deactivate_out_of_domain(void* st, int32_t* count) {
    auto* s = static_cast<RefState*>(st);
    int c = deactivate_out_of_domain(s->sim.particles, s->sim.grid);
    if (count) *count = c;
    return MPMB_OK;
}

mpmb_status mpmref_integrate_free_bodies(void* st, const float g[3], float dt) {
    auto* s = static_cast<RefState*>(st);
    for (size_t i = 0; i < s->shapes.size(); ++i)
        if (s->shapes[i].motion == MotionKind::free_body)
            integrate_free_body(s->shapes[i].pose, s->shapes[i].body, s->acc[i].impulse,
                                s->acc[i].torque_impulse, v3(g), dt);
    return MPMB_OK;
}

mpmb_status mpmref_state_get_grid(void* st, float* mass, float* mom, float* vel) {
    auto* s = static_cast<RefState*>(st);
    const auto& nodes = s->sim.grid.nodes;
    for (size_t i = 0; i < nodes.size(); ++i) {
        if (mass) mass[i] = nodes[i].mass;
        if (mom) put3(mom + 3 * i, nodes[i].momentum);
        if (vel) put3(vel + 3 * i, nodes[i].velocity);
    }
    return MPMB_OK;
}

// Spline weights exactly as the reference computes them (for KAT / key tests).
void mpmref_spline_weights(const float pos[3], const float origin[3], float dx, int32_t base[3],
                           float w[9], float dw[9]) {
    SplineWeights sw = quadratic_bspline_weights(v3(pos), v3(origin), dx);
    for (int a = 0; a < 3; ++a) {
        base[a] = sw.base_node[a];
        for (int o = 0; o < 3; ++o) { w[3 * a + o] = sw.w[a][o]; dw[3 * a + o] = sw.dw[a][o]; }
    }
}

int32_t mpmref_spline_in_domain(const float pos[3], const float origin[3], float dx,
                                const int32_t dims[3]) {
    return spline_in_domain(v3(pos), v3(origin), dx, dims[0], dims[1], dims[2]) ? 1 : 0;
}

void mpmref_neo_hookean(const float F[9], float mu, float lambda, float out[9]) {
    put9(out, neo_hookean_cauchy_stress(m9(F), mu, lambda));
}

int32_t mpmref_polar(const float M[9], float R[9], float U[9]) {
    auto r = polar_decompose(m9(M));
    if (!r) return 0;
    put9(R, r->r);
    put9(U, r->u);
    return 1;
}

int32_t mpmref_corotational_project(const float Fp[9], const float Cc[9], float dt, float beta,
                                    float out[9]) {
    auto r = corotational_project(m9(Fp), m9(Cc), dt, beta);
    if (!r) return 0;
    put9(out, *r);
    return 1;
}

// One SDF query (geometry.hpp:370-395): distance, normal, tangent, region.
void mpmref_sdf_query(const mpmb_shape_desc* d, const float point[3], float* distance,
                      float normal[3], float tangent[3], int32_t* region) {
    Shape sh = shape_from(*d);
    SdfSample s = sdf_query(sh.geometry, sh.pose, v3(point));
    *distance = s.distance;
    put3(normal, s.normal);
    put3(tangent, s.tangent);
    *region = static_cast<int32_t>(s.region);
}

void mpmref_evaluate_trajectory(const mpmb_keyframe* kf, int32_t n, float t, mpmb_pose* out) {
    KinematicTrajectory traj;
    for (int i = 0; i < n; ++i) {
        Keyframe k;
        k.time = kf[i].time;
        k.position = v3(kf[i].position);
        k.orientation = q4(kf[i].orientation);
        traj.keyframes.push_back(k);
    }
    pose_to(*out, evaluate_trajectory(traj, t));
}

void mpmref_lame(float E, float nu, float* mu, float* lambda) {
    auto [m, l] = lame_from_young_poisson(E, nu);
    *mu = m;
    *lambda = l;
}

// ------------------------------------------------------------ facade layer
uint64_t mpmref_create_scene(const mpmb_scene_config* c) {
    return facade::create_scene(config_from(*c));
}

mpmb_status mpmref_destroy(uint64_t h) { return map_status(facade::destroy(h)); }

uint64_t mpmref_create_material(uint64_t scene, const mpmb_material* m) {
    Material mat;
    mat.kind = m->kind == MPMB_MAT_COROTATIONAL_PB ? MaterialKind::corotational_pb
                                                   : MaterialKind::neo_hookean;
    mat.mu = m->mu;
    mat.lambda = m->lambda;
    mat.beta = m->beta;
    return facade::create_material(scene, mat);
}

uint64_t mpmref_create_particle_object(uint64_t scene, uint64_t mat, const float mn[3],
                                       const float mx[3], int32_t ppc, float density,
                                       uint64_t seed) {
    return facade::create_particle_object(scene, mat, v3(mn), v3(mx), ppc, density, seed);
}

uint64_t mpmref_create_shape(uint64_t scene, const mpmb_shape_desc* d) {
    try {
        return facade::create_shape(scene, shape_from(*d));
    } catch (const std::exception& e) {
        g_err = e.what();
        return facade::kInvalidHandle;
    }
}

mpmb_status mpmref_set_shape_pose_target(uint64_t scene, uint64_t shape, const float p[3],
                                         const float q[4]) {
    return map_status(facade::set_shape_pose_target(scene, shape, v3(p), q4(q)));
}

mpmb_status mpmref_advance(uint64_t scene, float dt) {
    return map_status(facade::advance(scene, dt));
}

mpmb_status mpmref_fetch_results(uint64_t scene, mpmb_frame_summary* out) {
    FrameResult r;
    facade::Status s = facade::fetch_results(scene, r);
    if (s != facade::Status::ok) return map_status(s);
    out->time = r.time;
    out->n_particles = static_cast<int32_t>(r.positions.size());
    out->n_shapes = static_cast<int32_t>(r.shape_ids.size());
    out->total_mass = r.total_mass;
    for (int a = 0; a < 3; ++a) out->momentum[a] = r.momentum[a];
    out->kinetic_energy = r.kinetic_energy;
    out->pushed_out = r.pushed_out;
    out->inverted_f = r.inverted_f;
    out->projection_failures = r.projection_failures;
    out->deactivated = r.deactivated;
    results()[scene] = std::move(r);
    return MPMB_OK;
}

mpmb_status mpmref_result_copy(uint64_t scene, float* pos, float* vel, uint8_t* active,
                               int32_t* ids, float* imp, float* tq) {
    auto it = results().find(scene);
    if (it == results().end()) return MPMB_LIFECYCLE_ERROR;
    const FrameResult& r = it->second;
    for (size_t i = 0; i < r.positions.size(); ++i) {
        if (pos) put3(pos + 3 * i, r.positions[i]);
        if (vel) put3(vel + 3 * i, r.velocities[i]);
        if (active) active[i] = r.active[i];
    }
    for (size_t i = 0; i < r.shape_ids.size(); ++i) {
        if (ids) ids[i] = r.shape_ids[i];
        if (imp) put3(imp + 3 * i, r.shape_impulses[i]);
        if (tq) put3(tq + 3 * i, r.shape_torque_impulses[i]);
    }
    return MPMB_OK;
}

int32_t mpmref_particle_count(uint64_t scene) { return facade::particle_count(scene); }

mpmb_status mpmref_copy_positions(uint64_t scene, float* out, size_t cap, size_t* written) {
    size_t w = 0;
    facade::Status s = facade::copy_positions(scene, out, cap, w);
    if (written) *written = w;
    return map_status(s);
}

mpmb_status mpmref_shape_impulse(uint64_t scene, uint64_t shape, float out[3]) {
    Vec3 v;
    facade::Status s = facade::shape_impulse(scene, shape, v);
    if (s == facade::Status::ok) put3(out, v);
    return map_status(s);
}

mpmb_status mpmref_scene_get_particles(uint64_t scene, float* x, float* v, float* F, float* C,
                                       uint8_t* active) {
    Scene* sc = scene_ptr(scene);
    if (!sc) return MPMB_BAD_HANDLE;
    const auto& p = sc->state().particles;
    for (size_t i = 0; i < p.size(); ++i) {
        if (x) put3(x + 3 * i, p.x[i]);
        if (v) put3(v + 3 * i, p.v[i]);
        if (F) put9(F + 9 * i, p.F[i]);
        if (C) put9(C + 9 * i, p.C[i]);
        if (active) active[i] = p.active[i];
    }
    return MPMB_OK;
}

// Reference's own JSON loader (scene_spec.hpp:451-518) -> facade-registered scene.
uint64_t mpmref_load_scene(const char* path, float* dt_frame) {
    try {
        SceneSpec spec = load_scene(path);
        if (dt_frame) *dt_frame = spec.dt_frame;
        facade::detail::Entry e;
        e.kind = facade::detail::HandleKind::scene;
        e.owned = scene_from_spec(spec);
        return facade::detail::registry().insert(std::move(e));
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return facade::kInvalidHandle;
    }
}

// CPU baseline for bench.py: advance every scene `frames` times, scenes spread over
// `threads` host threads (independent Scene objects; no registry writes while running).
// Returns wall seconds.
double mpmref_advance_many(const uint64_t* scenes, int32_t n, float dt, int32_t frames,
                           int32_t threads) {
    std::vector<Scene*> ptrs(n);
    for (int i = 0; i < n; ++i) ptrs[i] = scene_ptr(scenes[i]);
    auto t0 = std::chrono::steady_clock::now();
    auto worker = [&](int tid) {
        for (int i = tid; i < n; i += threads) {
            if (!ptrs[i]) continue;
            for (int f = 0; f < frames; ++f) {
                ptrs[i]->advance(dt);
                ptrs[i]->fetch_results();
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker, t);
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
}

// ---- scenario harness (scenario.hpp), for the device metrics / writer parity tests ----
static std::vector<Vec3> vec3s(const float* p, int64_t n) {
    std::vector<Vec3> v(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) v[i] = Vec3{p[3 * i], p[3 * i + 1], p[3 * i + 2]};
    return v;
}

int32_t mpmref_compute_components(const float* pos, const uint8_t* active, int64_t n, float radius) {
    std::vector<uint8_t> a(active, active + n);
    return compute_components(vec3s(pos, n), a, radius);
}

float mpmref_nn_spacing(const float* pos, const uint8_t* active, int64_t n, float hint) {
    std::vector<uint8_t> a(active, active + n);
    return mean_nearest_neighbor_spacing(vec3s(pos, n), a, hint);
}

void mpmref_write_frame_bin(const char* path, const float* pos, int64_t n) {
    scenario_detail::write_frame_bin(path, vec3s(pos, n));
}

void mpmref_write_frame_csv(const char* path, const float* pos, int64_t n) {
    scenario_detail::write_frame_csv(path, vec3s(pos, n));
}

// run_scenario on a scene JSON file (load_scene_spec): writes metrics.csv and frame dumps
// under out_dir; returns frames done (-1 on error, message in mpmref_last_error)
int32_t mpmref_run_scenario(const char* json_path, int32_t frames, const char* out_dir, int32_t* components) {
    try {
        SceneSpec spec = load_scene(json_path);
        ScenarioSummary sum = run_scenario(spec, frames, out_dir);
        if (components) *components = sum.final_component_count;
        return sum.frames_done;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
