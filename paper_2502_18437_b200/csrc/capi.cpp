// capi.cpp — C-ABI of include/mpm_b200.h.
//
// Solver layer: mpmb_state_s = one SimState (solvers.hpp:11-15) resident in HBM.
// Facade layer: a process-global handle registry mirroring mpm::facade
// (facade.hpp:26-219) over host-side Scene records whose simulation state lives in a
// device Engine shared by all scenes of a batch.  Scene semantics follow
// mpm::Scene::run_frame (scene.hpp:176-249).  No function throws across the boundary.
#include <cfloat>
#include <cmath>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/mpm_b200.h"
#include "dd_driver.h"
#include "engine.h"
#include "host_math.h"

using namespace mpmb;

namespace {

thread_local std::string g_error;

struct StatusError : std::runtime_error {
    mpmb_status status;
    StatusError(mpmb_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] void fail(mpmb_status s, const std::string& m) { throw StatusError(s, m); }

template <class F>
mpmb_status guarded(F&& f) {
    try {
        g_error.clear();
        return f();
    } catch (const StatusError& e) {
        g_error = e.what();
        return e.status;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return MPMB_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_error = e.what();
        return MPMB_CUDA_ERROR;
    }
}

void require_device() {
    if (!device_available()) fail(MPMB_NO_DEVICE, "no CUDA device available (no CPU fallback)");
}

DevPose to_dev(const mpmb_pose& p) {
    DevPose d{};
    std::memcpy(d.pos, p.position, 12);
    std::memcpy(d.rot, p.orientation, 16);
    std::memcpy(d.lin, p.linear_velocity, 12);
    std::memcpy(d.ang, p.angular_velocity, 12);
    return d;
}
mpmb_pose from_dev(const DevPose& d) {
    mpmb_pose p{};
    std::memcpy(p.position, d.pos, 12);
    std::memcpy(p.orientation, d.rot, 16);
    std::memcpy(p.linear_velocity, d.lin, 12);
    std::memcpy(p.angular_velocity, d.ang, 12);
    return p;
}
DevPose to_dev(const host::Pose& p) {
    DevPose d{};
    d.pos[0] = p.pos.x; d.pos[1] = p.pos.y; d.pos[2] = p.pos.z;
    d.rot[0] = p.rot.x; d.rot[1] = p.rot.y; d.rot[2] = p.rot.z; d.rot[3] = p.rot.w;
    d.lin[0] = p.lin.x; d.lin[1] = p.lin.y; d.lin[2] = p.lin.z;
    d.ang[0] = p.ang.x; d.ang[1] = p.ang.y; d.ang[2] = p.ang.z;
    return d;
}
host::Pose from_devp(const DevPose& d) {
    host::Pose p;
    p.pos = {d.pos[0], d.pos[1], d.pos[2]};
    p.rot = {d.rot[0], d.rot[1], d.rot[2], d.rot[3]};
    p.lin = {d.lin[0], d.lin[1], d.lin[2]};
    p.ang = {d.ang[0], d.ang[1], d.ang[2]};
    return p;
}

// validate_geometry (geometry.hpp:98-132) + validate_trajectory (rigid_dynamics.hpp:21-27)
void validate_shape(const mpmb_shape_desc& d, bool need_trajectory) {
    const float* g = d.gparam;
    switch (d.geometry) {
        case MPMB_GEOM_PLANE: break;
        case MPMB_GEOM_SPHERE:
            if (g[0] <= 0) fail(MPMB_INVALID_ARGUMENT, "sphere: radius <= 0");
            break;
        case MPMB_GEOM_BOX:
            if (g[0] <= 0 || g[1] <= 0 || g[2] <= 0) fail(MPMB_INVALID_ARGUMENT, "box: half extents must be positive");
            break;
        case MPMB_GEOM_QUAD_SLICER:
            if (g[0] <= 0 || g[1] <= 0) fail(MPMB_INVALID_ARGUMENT, "quad slicer: zero-area blade");
            if (g[2] <= 0) fail(MPMB_INVALID_ARGUMENT, "quad slicer: spine radius <= 0");
            break;
        case MPMB_GEOM_TRI_MESH_SLICER:
            if (d.n_vertices < 3 || d.n_indices < 3 || d.n_indices % 3 != 0)
                fail(MPMB_INVALID_ARGUMENT, "mesh slicer: invalid triangle list");
            if (g[0] <= 0) fail(MPMB_INVALID_ARGUMENT, "mesh slicer: spine radius <= 0");
            if (d.n_spine_edges % 2 != 0) fail(MPMB_INVALID_ARGUMENT, "mesh slicer: spine edge list must be pairs");
            for (int i = 0; i < d.n_indices; ++i)
                if (d.indices[i] < 0 || d.indices[i] >= d.n_vertices) fail(MPMB_INVALID_ARGUMENT, "mesh slicer: index out of range");
            for (int i = 0; i < d.n_spine_edges; ++i)
                if (d.spine_edges[i] < 0 || d.spine_edges[i] >= d.n_vertices) fail(MPMB_INVALID_ARGUMENT, "mesh slicer: spine index out of range");
            break;
        case MPMB_GEOM_ARC:
            if (g[0] <= 0) fail(MPMB_INVALID_ARGUMENT, "arc: radius <= 0");
            if (g[1] <= 0 || g[1] > static_cast<float>(2 * 3.14159265358979323846 + 1e-6))
                fail(MPMB_INVALID_ARGUMENT, "arc: angle must be in (0, 2*pi]");
            break;
        case MPMB_GEOM_POLYLINE:
            if (d.n_vertices < 2) fail(MPMB_INVALID_ARGUMENT, "polyline: needs >= 2 vertices");
            break;
        default: fail(MPMB_INVALID_ARGUMENT, "unknown geometry kind");
    }
    if (need_trajectory && d.motion == MPMB_MOTION_KINEMATIC) {
        if (d.n_keyframes < 1) fail(MPMB_INVALID_ARGUMENT, "trajectory: needs >= 1 keyframe");
        for (int i = 1; i < d.n_keyframes; ++i)
            if (!(d.keyframes[i].time > d.keyframes[i - 1].time))
                fail(MPMB_INVALID_ARGUMENT, "trajectory: times must be strictly increasing");
    }
}

struct HostShape {
    int id = -1;
    EngineShape e;
    std::vector<mpmb_keyframe> keyframes;
};

EngineShape engine_shape(const mpmb_shape_desc& d) {
    EngineShape e{};
    std::memset(&e.d, 0, sizeof e.d);
    e.d.geom = d.geometry;
    e.d.motion = d.motion == MPMB_MOTION_FREE_BODY ? MOTION_FREE
                 : d.motion == MPMB_MOTION_KINEMATIC ? MOTION_KINEMATIC
                                                     : MOTION_FIXED;
    std::memcpy(e.d.gp, d.gparam, sizeof e.d.gp);
    e.d.mu_k = d.mu_k;
    e.d.c_d = d.c_d;
    e.d.hw = d.collision_halfwidth;
    e.d.body_mass = d.body_mass;
    std::memcpy(e.d.inertia, d.inertia, 12);
    e.pose = to_dev(d.pose);
    if (d.n_vertices > 0) e.verts.assign(d.vertices, d.vertices + 3 * d.n_vertices);
    if (d.n_indices > 0) e.indices.assign(d.indices, d.indices + d.n_indices);
    if (d.n_spine_edges > 0) e.spine.assign(d.spine_edges, d.spine_edges + d.n_spine_edges);
    return e;
}

}  // namespace

// =================================================================== library
extern "C" int32_t mpmb_abi_version(void) { return MPMB_ABI_VERSION; }
extern "C" int32_t mpmb_device_available(void) { return device_available() ? 1 : 0; }
extern "C" const char* mpmb_last_error(void) { return g_error.c_str(); }
extern "C" int64_t mpmb_kernel_launch_count(void) { return global_launch_count(); }

extern "C" mpmb_status mpmb_eval_stress_f32(const float* F, int64_t n, float mu, float lambda, float* sigma,
                                            float* J) {
    return guarded([&] {
        if (!F || !sigma || n < 0) fail(MPMB_INVALID_ARGUMENT, "eval_stress_f32: null argument");
        require_device();
        Engine::eval_stress_f32(F, n, mu, lambda, sigma, J);
        return MPMB_OK;
    });
}

// ============================================================== solver layer
struct mpmb_state_s {
    std::unique_ptr<Engine> eng;
    SceneGrid grid{};
    int64_t n = 0;
    std::vector<HostShape> shapes;
};

namespace {
mpmb_state_s* S(mpmb_state st) {
    if (!st) fail(MPMB_BAD_HANDLE, "null state");
    return st;
}
}  // namespace

extern "C" mpmb_status mpmb_state_create(const int32_t dims[3], float dx, const float origin[3],
                                         mpmb_state* out) {
    return guarded([&] {
        if (!dims || !origin || !out) fail(MPMB_INVALID_ARGUMENT, "null argument");
        if (dims[0] < 4 || dims[1] < 4 || dims[2] < 4)
            fail(MPMB_INVALID_ARGUMENT, "grid: dims must be >= 4 per axis");  // state.hpp:30-31
        if (!(dx > 0)) fail(MPMB_INVALID_ARGUMENT, "grid: dx must be positive");
        require_device();
        auto st = std::make_unique<mpmb_state_s>();
        for (int a = 0; a < 3; ++a) {
            st->grid.dims[a] = dims[a];
            st->grid.origin[a] = origin[a];
        }
        st->grid.dx = dx;
        st->eng = std::make_unique<Engine>(std::vector<SceneGrid>{st->grid});
        st->eng->enable_grid_readback();  // the solver-layer API exposes the grid
        *out = st.release();
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_destroy(mpmb_state st) {
    return guarded([&] {
        delete st;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_set_materials(mpmb_state st, const mpmb_material* m, int32_t n) {
    return guarded([&] {
        S(st)->eng->set_materials(std::vector<mpmb_material>(m, m + n));
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_set_particles(mpmb_state st, int32_t n, const float* x,
                                                const float* v, const float* mass,
                                                const float* vol0, const float* F, const float* C,
                                                const float* stress, const int32_t* mat,
                                                const uint8_t* active) {
    return guarded([&] {
        if (n < 0) fail(MPMB_INVALID_ARGUMENT, "negative particle count");
        if (n > 0 && (!x || !v || !mass || !vol0 || !F || !C || !mat || !active))
            fail(MPMB_INVALID_ARGUMENT, "null particle array");
        std::vector<int32_t> scene(static_cast<size_t>(n), 0);
        S(st)->eng->upload_particles(n, x, v, mass, vol0, F, C, stress, mat, active, scene.data());
        st->n = n;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_spawn_box(const int32_t dims[3], float dx, const float origin[3], const float mn[3],
                                      const float mx[3], int32_t ppc, float density, uint64_t seed, int64_t capacity,
                                      float* x, float* mass, float* vol0, int64_t* n) {
    return guarded([&] {
        if (!dims || !origin || !mn || !mx || !n) fail(MPMB_INVALID_ARGUMENT, "null argument");
        std::vector<float> px, pm, pv;
        if (!host::spawn_box(dims, dx, host::v3(origin), host::v3(mn), host::v3(mx), ppc, density, seed, px, pm, pv))
            fail(MPMB_INVALID_ARGUMENT, "spawn_box: invalid box");
        const int64_t k = static_cast<int64_t>(pm.size());
        *n = k;
        if (k > capacity) fail(MPMB_BUFFER_TOO_SMALL, "spawn_box: capacity too small");
        if (x) std::copy(px.begin(), px.end(), x);
        if (mass) std::copy(pm.begin(), pm.end(), mass);
        if (vol0) std::copy(pv.begin(), pv.end(), vol0);
        return MPMB_OK;
    });
}

// ------------------------------------------------ slab domain decomposition
extern "C" mpmb_status mpmb_state_create_slab(const int32_t dims[3], float dx, const float origin[3],
                                              int32_t slab_lo, int32_t slab_hi, int32_t margin, int64_t capacity,
                                              mpmb_state* out) {
    return guarded([&] {
        if (!dims || !origin || !out) fail(MPMB_INVALID_ARGUMENT, "null argument");
        if (dims[0] < 4 || dims[1] < 4 || dims[2] < 4) fail(MPMB_INVALID_ARGUMENT, "grid: dims must be >= 4 per axis");
        if (!(dx > 0)) fail(MPMB_INVALID_ARGUMENT, "grid: dx must be positive");
        if (slab_lo < 0 || slab_hi > dims[0] || slab_hi - slab_lo < 2 + margin || margin < 1)
            fail(MPMB_INVALID_ARGUMENT, "slab: need 0 <= lo, hi <= nx, hi - lo >= 2 + margin, margin >= 1");
        if (capacity < 0) fail(MPMB_INVALID_ARGUMENT, "slab: negative capacity");
        require_device();
        auto st = std::make_unique<mpmb_state_s>();
        for (int a = 0; a < 3; ++a) {
            st->grid.dims[a] = dims[a];
            st->grid.origin[a] = origin[a];
        }
        st->grid.dx = dx;
        st->grid.slab_lo = slab_lo;
        st->grid.slab_hi = slab_hi;
        st->grid.margin = margin;
        st->eng = std::make_unique<Engine>(std::vector<SceneGrid>{st->grid});
        st->eng->set_capacity(capacity);
        *out = st.release();
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_set_particles_ids(mpmb_state st, int32_t n, const float* x, const float* v,
                                                    const float* mass, const float* vol0, const float* F,
                                                    const float* C, const int32_t* mat, const uint8_t* active,
                                                    const uint32_t* ids) {
    return guarded([&] {
        if (n < 0) fail(MPMB_INVALID_ARGUMENT, "negative particle count");
        if (n > 0 && (!x || !v || !mass || !vol0 || !F || !C || !mat || !active || !ids))
            fail(MPMB_INVALID_ARGUMENT, "null particle array");
        std::vector<int32_t> scene(static_cast<size_t>(n), 0);
        S(st)->eng->upload_particles(n, x, v, mass, vol0, F, C, nullptr, mat, active, scene.data(), ids);
        st->n = n;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_set_exact(mpmb_state st, int32_t on) {
    return guarded([&] {
        S(st)->eng->set_exact(on != 0);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_set_stream(mpmb_state st, void* stream) {
    return guarded([&] {
        S(st)->eng->set_stream(stream);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_synchronize(mpmb_state st) {
    return guarded([&] {
        S(st)->eng->synchronize();
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_dd_halo_buffers(mpmb_state st, void** send_lo, void** send_hi, void** recv_lo,
                                            void** recv_hi, int64_t* bytes, int64_t* plane_bytes,
                                            int32_t* margin) {
    return guarded([&] {
        Engine& e = *S(st)->eng;
        e.dd_halo_buffers(send_lo, send_hi, recv_lo, recv_hi, bytes);
        if (margin) *margin = st->grid.margin;
        int y0, ny, z0, nz;
        e.dd_plane_window(&y0, &ny, &z0, &nz);
        if (plane_bytes) *plane_bytes = static_cast<int64_t>(ny) * nz * 16;  // one windowed x-plane
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_dd_set_window(mpmb_state st, int32_t y0, int32_t y1, int32_t z0, int32_t z1) {
    return guarded([&] {
        S(st)->eng->dd_set_window(y0, y1, z0, z1);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_dd_particle_window(mpmb_state st, int32_t* out) {
    return guarded([&] {
        if (!out) fail(MPMB_INVALID_ARGUMENT, "null argument");
        int w[4];
        S(st)->eng->particle_window(w);
        for (int q = 0; q < 4; ++q) out[q] = w[q];
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_dd_p2g(mpmb_state st, float dt) {
    return guarded([&] {
        S(st)->eng->p2g(true, dt, false);
        return MPMB_OK;
    });
}
extern "C" mpmb_status mpmb_dd_pack_acc(mpmb_state st) {
    return guarded([&] { S(st)->eng->dd_pack_acc(); return MPMB_OK; });
}
extern "C" mpmb_status mpmb_dd_unpack_acc(mpmb_state st) {
    return guarded([&] { S(st)->eng->dd_unpack_acc(); return MPMB_OK; });
}
extern "C" mpmb_status mpmb_dd_grid(mpmb_state st, float dt, const float g[3], int32_t contact, int32_t bc) {
    return guarded([&] {
        Engine& e = *S(st)->eng;
        e.collect_bricks();
        e.grid_update(0, dt, g, true, contact != 0, bc);
        return MPMB_OK;
    });
}
extern "C" mpmb_status mpmb_dd_pack_vel(mpmb_state st) {
    return guarded([&] { S(st)->eng->dd_pack_vel(); return MPMB_OK; });
}
extern "C" mpmb_status mpmb_dd_unpack_vel(mpmb_state st) {
    return guarded([&] { S(st)->eng->dd_unpack_vel(); return MPMB_OK; });
}
extern "C" mpmb_status mpmb_dd_g2p(mpmb_state st, float dt, int32_t pushout, int32_t deactivate) {
    return guarded([&] {
        S(st)->eng->g2p_mls(0, dt, pushout != 0, deactivate != 0);
        return MPMB_OK;
    });
}
extern "C" mpmb_status mpmb_dd_contact_sums(mpmb_state st, void** sums, void** counts, int32_t* n_shapes) {
    return guarded([&] {
        if (!sums || !counts || !n_shapes) fail(MPMB_INVALID_ARGUMENT, "null argument");
        int n = 0;
        S(st)->eng->contact_sub_buffers(sums, counts, &n);
        *n_shapes = n;
        return MPMB_OK;
    });
}
extern "C" mpmb_status mpmb_dd_free_bodies(mpmb_state st, float dt, const float g[3]) {
    return guarded([&] {
        if (dt <= 0 || !g) fail(MPMB_INVALID_ARGUMENT, "free bodies: dt must be positive");
        S(st)->eng->free_bodies(0, dt, g, true, true);
        return MPMB_OK;
    });
}
extern "C" mpmb_status mpmb_dd_migrate_pack(mpmb_state st, int64_t* n_lo, int64_t* n_hi) {
    return guarded([&] {
        if (!n_lo || !n_hi) fail(MPMB_INVALID_ARGUMENT, "null argument");
        S(st)->eng->dd_migrate_pack(n_lo, n_hi);
        return MPMB_OK;
    });
}
extern "C" mpmb_status mpmb_dd_migrate_buffers(mpmb_state st, void** send_lo, void** send_hi, void** recv_lo,
                                               void** recv_hi, int64_t* cap) {
    return guarded([&] {
        S(st)->eng->dd_migrate_buffers(send_lo, send_hi, recv_lo, recv_hi, cap);
        return MPMB_OK;
    });
}
extern "C" mpmb_status mpmb_dd_migrate_unpack(mpmb_state st, int64_t n_from_lo, int64_t n_from_hi) {
    return guarded([&] {
        if (n_from_lo < 0 || n_from_hi < 0) fail(MPMB_INVALID_ARGUMENT, "negative count");
        Engine& e = *S(st)->eng;
        e.dd_migrate_unpack(n_from_lo, n_from_hi);
        st->n = e.n_particles();
        return MPMB_OK;
    });
}
struct mpmb_dd_group_s {
    std::unique_ptr<DDGroup> g;
};

extern "C" mpmb_status mpmb_dd_group_create_local(const mpmb_state* slabs, int32_t n, mpmb_dd_group* out) {
    return guarded([&] {
        if (!slabs || n <= 0 || !out) fail(MPMB_INVALID_ARGUMENT, "dd group: slabs");
        std::vector<Engine*> e;
        for (int32_t i = 0; i < n; ++i) e.push_back(S(slabs[i])->eng.get());
        auto* g = new mpmb_dd_group_s{DDGroup::local(e)};
        *out = g;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_nccl_get_unique_id(uint8_t id[128]) {
    return guarded([&] {
        if (!id) fail(MPMB_INVALID_ARGUMENT, "null argument");
        DDGroup::nccl_unique_id(id);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_dd_group_create_nccl(mpmb_state slab, const uint8_t id[128], int32_t nranks,
                                                 int32_t rank, mpmb_dd_group* out) {
    return guarded([&] {
        if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) fail(MPMB_INVALID_ARGUMENT, "dd group: rank");
        auto* g = new mpmb_dd_group_s{DDGroup::nccl(S(slab)->eng.get(), id, nranks, rank)};
        *out = g;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_dd_group_create_comm(mpmb_state slab, void* comm, int32_t nranks, int32_t rank,
                                                 mpmb_dd_group* out) {
    return guarded([&] {
        if (!comm || !out || nranks < 1 || rank < 0 || rank >= nranks) fail(MPMB_INVALID_ARGUMENT, "dd group: rank");
        auto* g = new mpmb_dd_group_s{DDGroup::nccl_comm(S(slab)->eng.get(), comm, nranks, rank)};
        *out = g;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_dd_group_destroy(mpmb_dd_group g) {
    delete g;
    return MPMB_OK;
}

extern "C" mpmb_status mpmb_dd_run(mpmb_dd_group g, int32_t n_sub, float dt, const float gravity[3], int32_t contact,
                                   int32_t boundary, int32_t pushout, int32_t deactivate, int32_t free_bodies,
                                   int32_t migrate_every, int32_t fuse) {
    return guarded([&] {
        if (!g || !gravity) fail(MPMB_INVALID_ARGUMENT, "null argument");
        DDRunOptions o;
        o.n_sub = n_sub;
        o.dt = dt;
        for (int a = 0; a < 3; ++a) o.g[a] = gravity[a];
        o.contact = contact != 0;
        o.bc = boundary;
        o.pushout = pushout != 0;
        o.deactivate = deactivate != 0;
        o.free_bodies = free_bodies != 0;
        o.migrate_every = migrate_every;
        o.fuse = fuse != 0;
        g->g->run(o);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_dd_check(mpmb_dd_group g) {
    return guarded([&] {
        if (!g) fail(MPMB_INVALID_ARGUMENT, "null argument");
        g->g->check();
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_dd_get_stats(mpmb_dd_group g, mpmb_dd_stats* out) {
    return guarded([&] {
        if (!g || !out) fail(MPMB_INVALID_ARGUMENT, "null argument");
        const DDStats& s = g->g->stats();
        *out = mpmb_dd_stats{s.runs, s.substeps, s.host_syncs, s.host_waits, s.exchanges, s.fused, s.rebins};
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_dd_download(mpmb_state st, int64_t capacity, uint32_t* ids, float* x, float* v,
                                        uint8_t* active, int64_t* n) {
    return guarded([&] {
        if (!ids || !x || !v || !active || !n) fail(MPMB_INVALID_ARGUMENT, "null argument");
        Engine& e = *S(st)->eng;
        const int64_t k = e.download_compact(capacity, ids, x, v, active);
        *n = k;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_get_particles(mpmb_state st, int32_t n, float* x, float* v,
                                                float* mass, float* vol0, float* F, float* C,
                                                float* stress, int32_t* mat, uint8_t* active) {
    return guarded([&] {
        if (n < S(st)->n) fail(MPMB_BUFFER_TOO_SMALL, "buffer too small");
        st->eng->download_particles(0, st->n, x, v, mass, vol0, F, C, stress, mat, active);
        return MPMB_OK;
    });
}

extern "C" int32_t mpmb_state_particle_count(mpmb_state st) {
    if (!st) return -1;
    // a slab advanced by the device-resident DD driver learns its count from the device
    if (st->eng && st->eng->n_particles() != st->n && st->grid.slab_hi > st->grid.slab_lo) st->n = st->eng->n_particles();
    return static_cast<int32_t>(st->n);
}

extern "C" mpmb_status mpmb_state_set_shapes(mpmb_state st, const mpmb_shape_desc* d, int32_t n) {
    return guarded([&] {
        S(st);
        std::vector<HostShape> hs;
        std::vector<EngineShape> es;
        for (int i = 0; i < n; ++i) {
            validate_shape(d[i], false);
            HostShape h;
            h.id = i;
            h.e = engine_shape(d[i]);
            es.push_back(h.e);
            hs.push_back(std::move(h));
        }
        st->eng->set_shapes({es});
        st->shapes = std::move(hs);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_get_shape_poses(mpmb_state st, mpmb_pose* out, int32_t n) {
    return guarded([&] {
        S(st);
        std::vector<DevPose> fp = st->eng->read_free_poses();
        for (int i = 0; i < n && i < static_cast<int>(st->shapes.size()); ++i)
            out[i] = from_dev(st->shapes[i].e.d.motion == MOTION_FREE ? fp[i] : st->shapes[i].e.pose);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_get_contact(mpmb_state st, float* imp, float* tq, int32_t* cnt,
                                              int32_t n) {
    return guarded([&] {
        std::vector<double> di, dt;
        std::vector<int32_t> c;
        S(st)->eng->read_contact(0, di, dt, c);
        for (int i = 0; i < n && i < static_cast<int>(c.size()); ++i) {
            for (int a = 0; a < 3; ++a) {
                if (imp) imp[3 * i + a] = static_cast<float>(di[3 * i + a]);
                if (tq) tq[3 * i + a] = static_cast<float>(dt[3 * i + a]);
            }
            if (cnt) cnt[i] = c[i];
        }
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_reset_contact(mpmb_state st) {
    return guarded([&] {
        S(st)->eng->reset_contact(true, true);
        return MPMB_OK;
    });
}

namespace {
void fill_stats(Engine& e, mpmb_step_stats* stats) {
    if (!stats) return;
    SceneCounters c = e.read_counters()[0];
    stats->inverted_f = c.inverted_f;
    stats->projection_failures = c.projection_failures;
}
}  // namespace

extern "C" mpmb_status mpmb_step_mls(mpmb_state st, float dt, const float g[3], int32_t contact,
                                     int32_t bc, mpmb_step_stats* stats) {
    return guarded([&] {
        Engine& e = *S(st)->eng;
        e.reset_counters();
        e.bin();
        e.p2g(true, dt);
        e.grid_update(0, dt, g, true, contact != 0, bc);
        e.g2p_mls(0, dt, false, false);
        fill_stats(e, stats);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_step_standard(mpmb_state st, float dt, const float g[3], int32_t contact,
                                          int32_t bc, mpmb_step_stats* stats) {
    return guarded([&] {
        Engine& e = *S(st)->eng;
        e.reset_counters();
        e.bin();
        e.p2g(true, dt, true, true);
        e.grid_update(0, dt, g, true, contact != 0, bc);
        e.g2p_standard(0, dt, false, false);
        fill_stats(e, stats);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_step_pbmpm(mpmb_state st, float dt, const float g[3], int32_t iters,
                                       int32_t contact, int32_t bc, mpmb_step_stats* stats) {
    return guarded([&] {
        Engine& e = *S(st)->eng;
        e.reset_counters();
        e.materialize_stress();  // PB-MPM leaves the cached stress untouched (solvers.hpp:207-279)
        e.bin();
        for (int it = 0; it < iters; ++it) {
            e.p2g(false, dt);
            e.grid_update(0, dt, g, it == 0, contact != 0, bc);
            e.g2p_pb(0, dt, it == iters - 1, false, false);
        }
        if (iters <= 0) {  // commit only
            fail(MPMB_INVALID_ARGUMENT, "pbmpm: iterations must be >= 1");
        }
        fill_stats(e, stats);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_step_mls_hooked(mpmb_state st, float dt, const float g[3],
                                            int32_t contact, int32_t bc, mpmb_grid_hook hook,
                                            void* user, mpmb_step_stats* stats) {
    return guarded([&] {
        Engine& e = *S(st)->eng;
        e.reset_counters();
        e.bin();
        e.p2g(true, dt);
        e.grid_update(0, dt, g, true, contact != 0, -1);  // BC deferred until after the hook
        if (hook) {
            const int* d = st->grid.dims;
            const size_t nn = static_cast<size_t>(d[0]) * d[1] * d[2];
            std::vector<float> m(nn), p(3 * nn), v(3 * nn);
            e.download_grid(0, m.data(), p.data(), v.data());
            hook(user, static_cast<int32_t>(nn), m.data(), p.data(), v.data());
            e.upload_grid_velocity(0, m.data(), p.data(), v.data());
        }
        e.bc_pass(bc);
        e.g2p_mls(0, dt, false, false);
        fill_stats(e, stats);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_particle_pushout(mpmb_state st, int32_t* count) {
    return guarded([&] {
        Engine& e = *S(st)->eng;
        e.reset_counters();
        e.pushout(0);
        if (count) *count = e.read_counters()[0].pushed_out;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_deactivate_out_of_domain(mpmb_state st, int32_t* count) {
    return guarded([&] {
        Engine& e = *S(st)->eng;
        e.reset_counters();
        e.deactivate();
        if (count) *count = e.read_counters()[0].deactivated;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_integrate_free_bodies(mpmb_state st, const float g[3], float dt) {
    return guarded([&] {
        if (dt <= 0) fail(MPMB_INVALID_ARGUMENT, "free body: dt must be positive");
        S(st)->eng->free_bodies(0, dt, g, true, false);
        st->eng->synchronize();
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_state_get_grid(mpmb_state st, float* mass, float* mom, float* vel) {
    return guarded([&] {
        S(st)->eng->download_grid(0, mass, mom, vel);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_bin_particles(mpmb_state st, uint32_t* keys, uint32_t* perm) {
    return guarded([&] {
        const int64_t n = S(st)->n;
        std::vector<uint32_t> k(static_cast<size_t>(n)), p(static_cast<size_t>(n));
        st->eng->read_binning(k.data(), p.data());
        // the inactive tail is kept in bucket (atomic) order on the device; the API
        // reports it in original order
        const int64_t na = st->eng->n_active_sorted();
        std::sort(p.begin() + na, p.end());
        if (keys) std::memcpy(keys, k.data(), 4 * n);
        if (perm) std::memcpy(perm, p.data(), 4 * n);
        return MPMB_OK;
    });
}

// ============================================================== facade layer
namespace {

struct Batch;

struct ObjectRange {
    int id;
    size_t begin, end;
};

struct Scene {
    mpmb_scene_config cfg{};
    Batch* batch = nullptr;
    int index = 0;            // scene index inside the batch engine
    std::vector<mpmb_material> materials;
    // host particle store (original order), authoritative only while !device_valid
    std::vector<float> x, v, mass, vol0, F, C;
    std::vector<int32_t> mat;
    std::vector<uint8_t> active;
    std::vector<ObjectRange> objects;
    std::vector<HostShape> shapes;
    std::vector<std::optional<mpmb_keyframe>> targets;
    std::vector<host::Pose> start_poses;
    float time = 0;
    int next_shape_id = 0, next_object_id = 0;
    // last FrameResult
    mpmb_frame_summary res{};
    // positions / velocities / active of the last fetch: views into the batch's pinned
    // frame buffer (kept alive by `frame`; replaced only by the next fetch)
    std::shared_ptr<void> frame;
    const float* rx = nullptr;
    const float* rv = nullptr;
    const uint8_t* ra = nullptr;
    size_t rn = 0;
    std::vector<int32_t> rid;
    std::vector<float> rimp, rtq;
    bool alive = true;
    size_t count() const { return mass.size(); }
};

enum class Status { idle, advancing, results_ready };

struct Batch {
    std::vector<Scene*> scenes;
    std::unique_ptr<Engine> eng;
    std::shared_ptr<void> frame;  // pinned FrameResult buffer (x, v, active of all scenes)
    // caller arrays bound by mpmb_bind_results (page-locked in place): the FrameResult
    // destination instead of `frame`
    float* bound_x = nullptr;
    float* bound_v = nullptr;
    uint8_t* bound_a = nullptr;
    int64_t bound_n = 0;
    void unbind() {
        if (eng) eng->wait_results();  // no copy may still target the arrays
        Engine::host_unregister(bound_x);
        Engine::host_unregister(bound_v);
        Engine::host_unregister(bound_a);
        bound_x = bound_v = nullptr;
        bound_a = nullptr;
        bound_n = 0;
    }
    ~Batch() {  // the frame buffer goes before the engine: finish its copy first
        try {
            if (eng) eng->wait_results();
            if (bound_n) unbind();
        } catch (...) {  // at process exit the driver may already be gone
        }
    }
    size_t frame_bytes = 0;
    bool device_valid = false;   // device holds the newest particle state
    // advance_frames: the previous frame's last kernel was the fused G2P + this frame's first
    // P2G (run_frame, cross-frame fusion); valid only inside one advance_frames call
    bool carry_fused = false;
    bool particles_dirty = true; // host changed: re-upload
    bool shapes_dirty = true;
    Status status = Status::idle;
    int resort = 0;               // substeps between binnings (0: every 4 frames)
    int fusion = 1;               // Engine::set_fusion (mpmb_set_fusion)
    bool exact = false;           // exact mode (Engine::set_exact)
    int64_t since_sort = 1 << 30; // substeps since the last binning (runs across frames)
    bool profiling = false;
    void* stream = nullptr;
    std::vector<size_t> offsets;  // per scene: first original index in the engine
    std::vector<int> shape_offsets;
    std::vector<int> mat_offsets;
};

enum class Kind { scene, batch, material, particle_object, shape };

struct Entry {
    Kind kind;
    mpmb_handle scene = MPMB_INVALID_HANDLE;  // owner, for non-scene handles
    int inner_id = -1;
    std::unique_ptr<Scene> owned_scene;
    std::unique_ptr<Batch> owned_batch;
    Scene* scene_ptr = nullptr;
    Batch* batch_ptr = nullptr;
    bool alive = true;
};

struct Registry {
    std::mutex mu;
    std::unordered_map<mpmb_handle, Entry> entries;
    mpmb_handle next = 1;  // never reused (facade.hpp:40)
    mpmb_handle insert(Entry e) {
        mpmb_handle h = next++;
        entries.emplace(h, std::move(e));
        return h;
    }
    Entry* find(mpmb_handle h, Kind k) {
        auto it = entries.find(h);
        if (it == entries.end() || !it->second.alive || it->second.kind != k) return nullptr;
        return &it->second;
    }
    Scene* scene(mpmb_handle h) {
        Entry* e = find(h, Kind::scene);
        return e && e->scene_ptr && e->scene_ptr->alive ? e->scene_ptr : nullptr;
    }
};

Registry& reg() {
    static Registry r;
    return r;
}

bool valid_config(const mpmb_scene_config& c) {
    return c.substeps >= 1 && c.iterations >= 1 && c.grid_dims[0] >= 4 && c.grid_dims[1] >= 4 &&
           c.grid_dims[2] >= 4 && c.dx > 0;
}

// Pull the newest particle state back to the host arrays (before host-side edits).
void sync_host(Batch& b) {
    if (!b.device_valid || !b.eng) return;
    size_t total = 0;
    for (Scene* s : b.scenes) total += s->count();
    if (total == 0) return;
    std::vector<float> x(3 * total), v(3 * total), F(9 * total), C(9 * total);
    std::vector<uint8_t> a(total);
    b.eng->download_particles(0, static_cast<int64_t>(total), x.data(), v.data(), nullptr, nullptr,
                              F.data(), C.data(), nullptr, nullptr, a.data());
    for (size_t si = 0; si < b.scenes.size(); ++si) {
        Scene* s = b.scenes[si];
        const size_t o = b.offsets[si], n = s->count();
        std::copy(x.begin() + 3 * o, x.begin() + 3 * (o + n), s->x.begin());
        std::copy(v.begin() + 3 * o, v.begin() + 3 * (o + n), s->v.begin());
        std::copy(F.begin() + 9 * o, F.begin() + 9 * (o + n), s->F.begin());
        std::copy(C.begin() + 9 * o, C.begin() + 9 * (o + n), s->C.begin());
        std::copy(a.begin() + o, a.begin() + o + n, s->active.begin());
    }
    // free-body poses back to the host shape records
    std::vector<DevPose> fp = b.eng->read_free_poses();
    for (size_t si = 0; si < b.scenes.size(); ++si)
        for (size_t i = 0; i < b.scenes[si]->shapes.size(); ++i)
            if (b.scenes[si]->shapes[i].e.d.motion == MOTION_FREE)
                b.scenes[si]->shapes[i].e.pose = fp[b.shape_offsets[si] + i];
    b.device_valid = false;
    b.particles_dirty = true;
    b.shapes_dirty = true;
}

void ensure_engine(Batch& b) {
    if (b.eng) return;
    require_device();
    std::vector<SceneGrid> grids;
    for (Scene* s : b.scenes) {
        SceneGrid g{};
        for (int a = 0; a < 3; ++a) {
            g.dims[a] = s->cfg.grid_dims[a];
            g.origin[a] = s->cfg.origin[a];
        }
        g.dx = s->cfg.dx;
        grids.push_back(g);
    }
    b.eng = std::make_unique<Engine>(grids);
    if (b.stream) b.eng->set_stream(b.stream);
    b.eng->set_profiling(b.profiling);
    b.eng->set_exact(b.exact);
    b.eng->set_fusion(b.fusion);
}

void upload(Batch& b) {
    ensure_engine(b);
    if (b.particles_dirty) {
        // materials: deduplicated global table
        std::vector<mpmb_material> table;
        std::vector<std::vector<int>> remap(b.scenes.size());
        for (size_t si = 0; si < b.scenes.size(); ++si)
            for (const mpmb_material& m : b.scenes[si]->materials) {
                int found = -1;
                for (size_t t = 0; t < table.size(); ++t)
                    if (std::memcmp(&table[t], &m, sizeof m) == 0) found = static_cast<int>(t);
                if (found < 0) {
                    found = static_cast<int>(table.size());
                    table.push_back(m);
                }
                remap[si].push_back(found);
            }
        if (table.size() > 0xFFF) fail(MPMB_INVALID_ARGUMENT, "too many distinct materials");
        b.eng->set_materials(table);
        size_t total = 0;
        b.offsets.clear();
        for (Scene* s : b.scenes) {
            b.offsets.push_back(total);
            total += s->count();
        }
        std::vector<float> x, v, m, vol, F, C;
        std::vector<int32_t> mat, scene;
        std::vector<uint8_t> a;
        x.reserve(3 * total); v.reserve(3 * total); F.reserve(9 * total); C.reserve(9 * total);
        for (size_t si = 0; si < b.scenes.size(); ++si) {
            Scene* s = b.scenes[si];
            x.insert(x.end(), s->x.begin(), s->x.end());
            v.insert(v.end(), s->v.begin(), s->v.end());
            m.insert(m.end(), s->mass.begin(), s->mass.end());
            vol.insert(vol.end(), s->vol0.begin(), s->vol0.end());
            F.insert(F.end(), s->F.begin(), s->F.end());
            C.insert(C.end(), s->C.begin(), s->C.end());
            for (int32_t id : s->mat) mat.push_back(remap[si][id]);
            a.insert(a.end(), s->active.begin(), s->active.end());
            scene.insert(scene.end(), s->count(), static_cast<int32_t>(si));
        }
        b.eng->upload_particles(static_cast<int64_t>(total), x.data(), v.data(), m.data(), vol.data(),
                                F.data(), C.data(), nullptr, mat.data(), a.data(), scene.data());
        b.particles_dirty = false;
    }
    if (b.shapes_dirty) {
        std::vector<std::vector<EngineShape>> per;
        b.shape_offsets.clear();
        int off = 0;
        for (Scene* s : b.scenes) {
            b.shape_offsets.push_back(off);
            std::vector<EngineShape> v;
            for (const HostShape& h : s->shapes) v.push_back(h.e);
            off += static_cast<int>(v.size());
            per.push_back(std::move(v));
        }
        b.eng->set_shapes(per);
        b.shapes_dirty = false;
    }
    b.device_valid = true;
}

// Scene::run_frame (scene.hpp:176-249) for every scene of the batch, enqueued.
// export: the frame's last G2P writes the FrameResult (Engine::request_export) -- the last
// frame of an advance, the one fetch_results reads -- when the caller bound result arrays
// (mpmb_bind_results: a result every frame); unbound fetches gather after the frame
// cross-frame fusion (MPMB_CROSS_FRAME=0 in the environment: off, for A/B)
static bool cross_frame_fusion() {
    static const bool on = [] {
        const char* e = std::getenv("MPMB_CROSS_FRAME");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}

// into_next: another frame of the same advance_frames call follows, so when no binning falls
// between them the last G2P runs fused with that frame's first P2G (K8 across the frame
// boundary; nothing between them reads or writes particles: free bodies, pose targets and the
// next frame's pose table, counters and contact resets touch neither the planes nor the P2G
// accumulator, and the next frame's set_pose_table invalidates the shape cull)
void run_frame(Batch& b, float dt, bool last_of_advance = true, bool into_next = false) {
    // A/B of the e2e rate against the gather at fetch (MPMB_EXPORT=0 in the environment):
    // C5 +1.9 %, M1 +1.8 %, C2 +4.3 %, C1 +6 %, C3 +2 %
    static const bool pays = [] {
        const char* e = std::getenv("MPMB_EXPORT");
        return !e || std::atoi(e) != 0;
    }();
    const bool export_result = pays && last_of_advance && b.bound_n > 0;
    upload(b);
    Engine& e = *b.eng;
    const mpmb_scene_config& cfg = b.scenes[0]->cfg;
    const bool pb = cfg.solver == MPMB_SOLVER_PBMPM;
    const int n_sub = pb ? 1 : cfg.substeps;
    const float dt_sub = dt / static_cast<float>(n_sub);
    const int ns = e.n_shapes();
    bool any_free = false;
    // host: per-substep kinematic / target poses (bit-identical float math).  Only the grid
    // update and later kernels read the table, so it is built while the frame's binning
    // and first P2G already run on the device.
    auto build_pose_table = [&] {
        if (ns <= 0) return;
        std::vector<DevPose> table(static_cast<size_t>(n_sub) * ns);
        std::vector<uint8_t> ovr(table.size(), 0);
        std::vector<DevPose> fp;
        bool need_free = false;
        for (Scene* s : b.scenes)
            for (size_t i = 0; i < s->shapes.size(); ++i)
                if (s->targets[i] && s->shapes[i].e.d.motion == MOTION_FREE) need_free = true;
        if (need_free) fp = e.read_free_poses();
        for (size_t si = 0; si < b.scenes.size(); ++si) {
            Scene* s = b.scenes[si];
            s->start_poses.clear();
            for (size_t i = 0; i < s->shapes.size(); ++i) {
                const int gi = b.shape_offsets[si] + static_cast<int>(i);
                host::Pose cur = from_devp(s->shapes[i].e.d.motion == MOTION_FREE && need_free
                                               ? fp[gi] : s->shapes[i].e.pose);
                s->start_poses.push_back(cur);
                if (s->shapes[i].e.d.motion == MOTION_FREE) any_free = true;
            }
            for (int sub = 0; sub < n_sub; ++sub) {
                const float t = s->time + static_cast<float>(sub) * dt_sub;
                for (size_t i = 0; i < s->shapes.size(); ++i) {
                    const size_t slot = static_cast<size_t>(sub) * ns + b.shape_offsets[si] + i;
                    HostShape& h = s->shapes[i];
                    if (s->targets[i]) {
                        const mpmb_keyframe& tg = *s->targets[i];
                        host::Pose p = host::target_drive(s->start_poses[i].pos, s->start_poses[i].rot,
                                                          host::v3(tg.position), host::q4(tg.orientation),
                                                          t, s->time, dt);
                        table[slot] = to_dev(p);
                        ovr[slot] = 1;
                        if (h.e.d.motion != MOTION_FREE) h.e.pose = table[slot];
                    } else if (h.e.d.motion == MOTION_KINEMATIC) {
                        table[slot] = to_dev(host::evaluate_trajectory(h.keyframes, t));
                        h.e.pose = table[slot];
                    } else {
                        table[slot] = h.e.pose;
                    }
                }
            }
        }
        e.set_pose_table(n_sub, table, ovr);
    };
    e.reset_counters();
    e.reset_contact(true, true);
    // binning restores the spatial compactness of the 256-slot groups; drift inside a group
    // is absorbed by P2G's per-substep warp sort, so the full sort runs every 4 frames
    // unless the caller chose an interval (mpmb_set_resort_interval)
    const int resort = b.resort > 0 ? b.resort : 4 * n_sub;
    if (!pb) {
        // inside the frame, G2P of substep s and P2G of s+1 run as one kernel (k_g2p2g)
        // unless a binning falls between them
        const bool standard = cfg.solver == MPMB_SOLVER_STANDARD;  // scene.hpp:200-207
        const bool can_fuse = e.fuse_ok();
        bool fused_in = b.carry_fused;  // P2G of this substep already ran inside the previous kernel
        b.carry_fused = false;
        for (int sub = 0; sub < n_sub; ++sub) {
            if (b.since_sort >= resort) {
                if (fused_in) throw std::logic_error("run_frame: binning after a carried P2G");
                e.bin();
                b.since_sort = 0;
            }
            ++b.since_sort;
            if (!fused_in) e.p2g(true, dt_sub, true, standard);
            if (sub == 0) build_pose_table();
            e.grid_update(sub, dt_sub, cfg.gravity, true, true, cfg.boundary);
            const bool fuse = can_fuse && b.since_sort < resort &&
                              (sub + 1 < n_sub || (into_next && cross_frame_fusion()));
            if (fuse) {
                e.g2p2g(sub, dt_sub, standard, cfg.gravity, any_free);  // + free bodies of sub
            } else {
                if (export_result && sub + 1 == n_sub) e.request_export();
                if (standard) e.g2p_standard(sub, dt_sub, true, true);
                else e.g2p_mls(sub, dt_sub, true, true);
                if (ns > 0) e.free_bodies(sub, dt_sub, cfg.gravity, any_free, true, sub + 1 < n_sub ? sub + 1 : -1);
            }
            fused_in = fuse;
        }
        b.carry_fused = fused_in;  // the last substep fused into the next frame's first P2G
    } else {
        // PB-MPM: one step per frame; positions move only at the commit, so the per-iteration
        // group sort absorbs the drift and binning follows the same interval as MLS (every 4
        // frames by default; it cost C3 a fifth of its frame when it ran every step)
        if (b.since_sort >= resort) {
            e.bin();
            b.since_sort = 0;
        }
        ++b.since_sort;
        const bool can_fuse = e.fuse_ok();
        bool fused_in = false;  // P2G of this iteration already ran inside the previous kernel
        for (int it = 0; it < cfg.iterations; ++it) {
            const bool last = it == cfg.iterations - 1;
            if (!fused_in) e.p2g(false, dt_sub);
            if (it == 0) build_pose_table();
            e.grid_update(0, dt_sub, cfg.gravity, it == 0, true, cfg.boundary);
            fused_in = can_fuse && !last;  // the final G2P commits (solvers.hpp:269-277)
            if (fused_in) {
                e.g2p2g_pb(dt_sub);
            } else {
                if (export_result && last) e.request_export();
                e.g2p_pb(0, dt_sub, last, last, last);
            }
        }
        if (ns > 0) e.free_bodies(0, dt_sub, cfg.gravity, any_free, true);
    }
    // consume one-shot pose targets (scene.hpp:238-247)
    for (size_t si = 0; si < b.scenes.size(); ++si) {
        Scene* s = b.scenes[si];
        for (size_t i = 0; i < s->shapes.size(); ++i) {
            if (!s->targets[i]) continue;
            DevPose p{};
            std::memcpy(p.pos, s->targets[i]->position, 12);
            std::memcpy(p.rot, s->targets[i]->orientation, 16);
            s->shapes[i].e.pose = p;
            if (s->shapes[i].e.d.motion == MOTION_FREE) e.set_free_pose(b.shape_offsets[si] + static_cast<int>(i), p);
            s->targets[i].reset();
        }
        s->time += dt;
    }
}

// Scene::fetch_results / make_result (scene.hpp:125-130, 251-278) for all scenes.
void fetch(Batch& b) {
    Engine& e = *b.eng;
    size_t total = 0;
    for (Scene* s : b.scenes) total += s->count();
    const size_t bytes = 24 * total + total + 16;
    const bool bound = b.bound_n > 0 && static_cast<size_t>(b.bound_n) == total;
    if (!bound && (!b.frame || b.frame_bytes < bytes)) {
        e.wait_results();  // the previous frame's copy may still target the old buffer
        b.frame = Engine::pinned_host(bytes);
        b.frame_bytes = bytes;
    }
    float* x = bound ? b.bound_x : static_cast<float*>(b.frame.get());
    float* v = bound ? b.bound_v : x + 3 * total;
    uint8_t* a = bound ? b.bound_a : reinterpret_cast<uint8_t*>(v + 3 * total);
    // counters and contact first (a device->host copy issued after the arrays' would queue
    // behind them on the copy engine), all completed by the snapshot's one stream sync
    e.stage_small();
    std::vector<double> totals;
    // the arrays' D2H overlaps the next frame; mpmb_result_copy waits for it
    e.snapshot(x, v, a, totals, true);
    std::vector<SceneCounters> cnt;
    std::vector<double> imp, tq;
    std::vector<int32_t> cc;
    e.small_results(cnt, imp, tq, cc);
    if (b.exact) {
        e.wait_results();  // make_result (scene.hpp:256-266): FP64 sums in particle order, on the host
        for (size_t si = 0; si < b.scenes.size(); ++si) {
            const Scene* s = b.scenes[si];
            const size_t o = b.offsets[si];
            double t[5] = {0, 0, 0, 0, 0};
            for (size_t i = 0; i < s->count(); ++i) {
                if (!a[o + i]) continue;
                const double m = s->mass[i];
                const float* vi = v + 3 * (o + i);
                t[0] += m;
                t[1] += m * vi[0];
                t[2] += m * vi[1];
                t[3] += m * vi[2];
                const float n2 = vi[0] * vi[0] + vi[1] * vi[1] + vi[2] * vi[2];
                t[4] += 0.5 * m * static_cast<double>(n2);
            }
            for (int q = 0; q < 5; ++q) totals[5 * si + q] = t[q];
        }
    }
    for (size_t si = 0; si < b.scenes.size(); ++si) {
        Scene* s = b.scenes[si];
        const size_t o = b.offsets[si], n = s->count();
        s->frame = bound ? nullptr : b.frame;
        s->rx = x + 3 * o;
        s->rv = v + 3 * o;
        s->ra = a + o;
        s->rn = n;
        mpmb_frame_summary& r = s->res;
        r = mpmb_frame_summary{};
        r.time = s->time;
        r.n_particles = static_cast<int32_t>(n);
        r.n_shapes = static_cast<int32_t>(s->shapes.size());
        r.total_mass = totals[5 * si + 0];
        r.momentum[0] = totals[5 * si + 1];
        r.momentum[1] = totals[5 * si + 2];
        r.momentum[2] = totals[5 * si + 3];
        r.kinetic_energy = totals[5 * si + 4];
        r.pushed_out = cnt[si].pushed_out;
        r.inverted_f = cnt[si].inverted_f;
        r.projection_failures = cnt[si].projection_failures;
        r.deactivated = cnt[si].deactivated;
        s->rid.clear();
        s->rimp.clear();
        s->rtq.clear();
        for (size_t i = 0; i < s->shapes.size(); ++i) {
            const size_t gi = b.shape_offsets[si] + i;
            s->rid.push_back(s->shapes[i].id);
            for (int q = 0; q < 3; ++q) {
                s->rimp.push_back(static_cast<float>(imp[3 * gi + q]));
                s->rtq.push_back(static_cast<float>(tq[3 * gi + q]));
            }
        }
    }
}

Batch* batch_of_handle(Registry& r, mpmb_handle h, bool& is_batch) {
    if (Entry* e = r.find(h, Kind::batch)) {
        is_batch = true;
        return e->batch_ptr;
    }
    is_batch = false;
    Scene* s = r.scene(h);
    return s ? s->batch : nullptr;
}

}  // namespace

extern "C" mpmb_handle mpmb_create_scene(const mpmb_scene_config* c) {
    std::lock_guard<std::mutex> lk(reg().mu);
    try {
        if (!c || !valid_config(*c)) return MPMB_INVALID_HANDLE;
        Entry be{};
        be.kind = Kind::batch;
        be.owned_batch = std::make_unique<Batch>();
        Batch* b = be.owned_batch.get();
        Entry se{};
        se.kind = Kind::scene;
        se.owned_scene = std::make_unique<Scene>();
        Scene* s = se.owned_scene.get();
        s->cfg = *c;
        s->batch = b;
        b->scenes.push_back(s);
        se.scene_ptr = s;
        se.batch_ptr = b;
        // the private batch is owned by the scene handle's entry
        se.owned_batch = std::move(be.owned_batch);
        return reg().insert(std::move(se));
    } catch (...) {
        return MPMB_INVALID_HANDLE;
    }
}

extern "C" mpmb_handle mpmb_create_scene_batch(const mpmb_scene_config* c, int32_t n,
                                               mpmb_handle* out) {
    std::lock_guard<std::mutex> lk(reg().mu);
    try {
        if (!c || !valid_config(*c) || n < 1 || !out) return MPMB_INVALID_HANDLE;
        Entry be{};
        be.kind = Kind::batch;
        be.owned_batch = std::make_unique<Batch>();
        Batch* b = be.owned_batch.get();
        be.batch_ptr = b;
        const mpmb_handle bh = reg().insert(std::move(be));
        for (int i = 0; i < n; ++i) {
            Entry se{};
            se.kind = Kind::scene;
            se.owned_scene = std::make_unique<Scene>();
            Scene* s = se.owned_scene.get();
            s->cfg = *c;
            s->batch = b;
            s->index = i;
            b->scenes.push_back(s);
            se.scene_ptr = s;
            se.batch_ptr = b;
            se.scene = bh;
            out[i] = reg().insert(std::move(se));
        }
        return bh;
    } catch (...) {
        return MPMB_INVALID_HANDLE;
    }
}

extern "C" mpmb_status mpmb_destroy(mpmb_handle h) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        Registry& r = reg();
        auto it = r.entries.find(h);
        if (it == r.entries.end() || !it->second.alive) return MPMB_BAD_HANDLE;
        Entry& e = it->second;
        if (e.kind == Kind::scene || e.kind == Kind::batch) {
            // invalidate every handle owned by this scene / batch (facade.hpp:83-86)
            for (auto& kv : r.entries)
                if (kv.second.scene == h) {
                    kv.second.alive = false;
                    if (kv.second.kind == Kind::scene && kv.second.scene_ptr) {
                        kv.second.scene_ptr->alive = false;
                        for (auto& kv2 : r.entries)
                            if (kv2.second.scene == kv.first) kv2.second.alive = false;
                    }
                }
            if (e.kind == Kind::scene && e.scene_ptr) {
                Scene* s = e.scene_ptr;
                s->alive = false;
                if (s->batch && s->batch->scenes.size() > 1) {
                    // batch member: its particles leave the simulation
                    sync_host(*s->batch);
                    std::fill(s->active.begin(), s->active.end(), 0);
                }
            }
            if (e.kind == Kind::batch && e.batch_ptr) {
                // scenes are owned by their entries: release the engine now
                e.batch_ptr->eng.reset();
            }
        } else {
            Scene* s = r.scene(e.scene);
            if (s) {
                if (e.kind == Kind::shape) {  // Scene::destroy_shape (scene.hpp:90-95)
                    sync_host(*s->batch);
                    for (size_t i = 0; i < s->shapes.size(); ++i)
                        if (s->shapes[i].id == e.inner_id) {
                            s->shapes.erase(s->shapes.begin() + i);
                            s->targets.erase(s->targets.begin() + i);
                            break;
                        }
                    s->batch->shapes_dirty = true;
                } else if (e.kind == Kind::particle_object) {  // scene.hpp:97-107
                    sync_host(*s->batch);
                    for (auto ob = s->objects.begin(); ob != s->objects.end(); ++ob)
                        if (ob->id == e.inner_id) {
                            for (size_t i = ob->begin; i < ob->end; ++i) s->active[i] = 0;
                            s->objects.erase(ob);
                            break;
                        }
                    s->batch->particles_dirty = true;
                }
            }
        }
        e.alive = false;
        e.owned_scene.reset();
        if (e.kind != Kind::scene) e.owned_batch.reset();
        else e.owned_batch.reset();
        return MPMB_OK;
    });
}

extern "C" mpmb_handle mpmb_create_material(mpmb_handle sh, const mpmb_material* m) {
    std::lock_guard<std::mutex> lk(reg().mu);
    Scene* s = reg().scene(sh);
    if (!s || !m) return MPMB_INVALID_HANDLE;
    s->materials.push_back(*m);  // scene.hpp:57-60
    Entry e{};
    e.kind = Kind::material;
    e.scene = sh;
    e.inner_id = static_cast<int>(s->materials.size()) - 1;
    s->batch->particles_dirty = true;
    return reg().insert(std::move(e));
}

extern "C" mpmb_handle mpmb_create_particle_object(mpmb_handle sh, mpmb_handle mh, const float mn[3],
                                                   const float mx[3], int32_t ppc, float density,
                                                   uint64_t seed) {
    std::lock_guard<std::mutex> lk(reg().mu);
    try {
        Registry& r = reg();
        Scene* s = r.scene(sh);
        Entry* m = r.find(mh, Kind::material);
        if (!s || !m || m->scene != sh || !mn || !mx) return MPMB_INVALID_HANDLE;
        sync_host(*s->batch);
        const size_t before = s->count();
        std::vector<float> x, mass, vol0;
        if (!host::spawn_box(s->cfg.grid_dims, s->cfg.dx, host::v3(s->cfg.origin), host::v3(mn),
                             host::v3(mx), ppc, density, seed, x, mass, vol0))
            return MPMB_INVALID_HANDLE;
        const size_t n = mass.size();
        s->x.insert(s->x.end(), x.begin(), x.end());
        s->v.insert(s->v.end(), 3 * n, 0.f);
        s->mass.insert(s->mass.end(), mass.begin(), mass.end());
        s->vol0.insert(s->vol0.end(), vol0.begin(), vol0.end());
        for (size_t i = 0; i < n; ++i) {
            const float I9[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
            s->F.insert(s->F.end(), I9, I9 + 9);
            s->C.insert(s->C.end(), 9, 0.f);
        }
        s->mat.insert(s->mat.end(), n, m->inner_id);
        s->active.insert(s->active.end(), n, 1);
        const int id = s->next_object_id++;
        s->objects.push_back({id, before, before + n});
        s->batch->particles_dirty = true;
        Entry e{};
        e.kind = Kind::particle_object;
        e.scene = sh;
        e.inner_id = id;
        return r.insert(std::move(e));
    } catch (...) {
        return MPMB_INVALID_HANDLE;
    }
}

extern "C" mpmb_handle mpmb_create_shape(mpmb_handle sh, const mpmb_shape_desc* d) {
    std::lock_guard<std::mutex> lk(reg().mu);
    try {
        Scene* s = reg().scene(sh);
        if (!s || !d) return MPMB_INVALID_HANDLE;
        validate_shape(*d, true);
        sync_host(*s->batch);
        HostShape h;
        h.e = engine_shape(*d);
        if (h.e.d.hw <= 0) h.e.d.hw = 0.75f * s->cfg.dx;  // scene.hpp:79-80
        if (d->n_keyframes > 0) h.keyframes.assign(d->keyframes, d->keyframes + d->n_keyframes);
        if (h.e.d.motion == MOTION_KINEMATIC)
            h.e.pose = to_dev(host::evaluate_trajectory(h.keyframes, s->time));
        h.id = s->next_shape_id++;
        const int id = h.id;
        s->shapes.push_back(std::move(h));
        s->targets.emplace_back();
        s->batch->shapes_dirty = true;
        Entry e{};
        e.kind = Kind::shape;
        e.scene = sh;
        e.inner_id = id;
        return reg().insert(std::move(e));
    } catch (const std::exception& ex) {
        g_error = ex.what();
        return MPMB_INVALID_HANDLE;
    }
}

extern "C" mpmb_status mpmb_set_shape_pose_target(mpmb_handle sh, mpmb_handle shape,
                                                  const float p[3], const float q[4]) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        Registry& r = reg();
        Scene* s = r.scene(sh);
        Entry* e = r.find(shape, Kind::shape);
        if (!s || !e || e->scene != sh) return MPMB_BAD_HANDLE;
        for (size_t i = 0; i < s->shapes.size(); ++i)
            if (s->shapes[i].id == e->inner_id) {
                host::Q4 qn = host::qnormalized(host::q4(q));  // scene.hpp:114
                mpmb_keyframe k{};
                std::memcpy(k.position, p, 12);
                k.orientation[0] = qn.x; k.orientation[1] = qn.y;
                k.orientation[2] = qn.z; k.orientation[3] = qn.w;
                s->targets[i] = k;
                return MPMB_OK;
            }
        return MPMB_BAD_HANDLE;
    });
}

extern "C" mpmb_status mpmb_advance(mpmb_handle h, float dt) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        bool is_batch;
        Batch* b = batch_of_handle(reg(), h, is_batch);
        if (!b) return MPMB_BAD_HANDLE;
        if (!(dt > 0)) return MPMB_INVALID_ARGUMENT;  // facade.hpp:165
        if (!is_batch && b->scenes.size() > 1)
            fail(MPMB_LIFECYCLE_ERROR, "scene belongs to a batch: advance the batch handle");
        if (b->status == Status::advancing)
            fail(MPMB_LIFECYCLE_ERROR, "scene: advance while a frame is pending");
        b->status = Status::advancing;
        b->carry_fused = false;
        run_frame(*b, dt);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_advance_frames(mpmb_handle h, float dt, int32_t n_frames) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        bool is_batch;
        Batch* b = batch_of_handle(reg(), h, is_batch);
        if (!b) return MPMB_BAD_HANDLE;
        if (!(dt > 0) || n_frames < 1) return MPMB_INVALID_ARGUMENT;
        if (!is_batch && b->scenes.size() > 1)
            fail(MPMB_LIFECYCLE_ERROR, "scene belongs to a batch: advance the batch handle");
        if (b->status == Status::advancing)
            fail(MPMB_LIFECYCLE_ERROR, "scene: advance while a frame is pending");
        b->carry_fused = false;
        for (int f = 0; f < n_frames; ++f) run_frame(*b, dt, f + 1 == n_frames, f + 1 < n_frames);
        b->carry_fused = false;
        b->status = Status::advancing;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_fetch_results(mpmb_handle h, mpmb_frame_summary* out) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        bool is_batch;
        Batch* b = batch_of_handle(reg(), h, is_batch);
        if (!b) return MPMB_BAD_HANDLE;
        if (!is_batch && b->scenes.size() > 1)
            fail(MPMB_LIFECYCLE_ERROR, "scene belongs to a batch: fetch the batch handle");
        if (b->status != Status::advancing)
            fail(MPMB_LIFECYCLE_ERROR, "scene: fetch without a pending advance");
        b->status = Status::results_ready;
        fetch(*b);
        if (out)
            for (size_t i = 0; i < b->scenes.size(); ++i) out[i] = b->scenes[i]->res;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_result_copy(mpmb_handle sh, float* pos, float* vel, uint8_t* active,
                                        int32_t* ids, float* imp, float* tq) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        Scene* s = reg().scene(sh);
        if (!s) return MPMB_BAD_HANDLE;
        if ((pos || vel || active) && s->rn && s->batch && s->batch->eng) s->batch->eng->wait_results();
        // a bound destination already holds the arrays (mpmb_bind_results)
        if (pos && s->rn && pos != s->rx) std::copy(s->rx, s->rx + 3 * s->rn, pos);
        if (vel && s->rn && vel != s->rv) std::copy(s->rv, s->rv + 3 * s->rn, vel);
        if (active && s->rn && active != s->ra) std::copy(s->ra, s->ra + s->rn, active);
        if (ids) std::copy(s->rid.begin(), s->rid.end(), ids);
        if (imp) std::copy(s->rimp.begin(), s->rimp.end(), imp);
        if (tq) std::copy(s->rtq.begin(), s->rtq.end(), tq);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_bind_results(mpmb_handle h, float* pos, float* vel, uint8_t* active, int64_t n) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        bool is_batch = false;
        Batch* b = batch_of_handle(reg(), h, is_batch);
        if (!b) return MPMB_BAD_HANDLE;
        if (!is_batch && b->scenes.size() != 1)
            fail(MPMB_INVALID_ARGUMENT, "bind_results: a batch member binds through its batch handle");
        if (b->bound_n) b->unbind();
        if (!pos && !vel && !active) return MPMB_OK;
        if (!pos || !vel || !active || n <= 0) fail(MPMB_INVALID_ARGUMENT, "bind_results: three arrays and n > 0");
        int64_t total = 0;
        for (Scene* s : b->scenes) total += static_cast<int64_t>(s->count());
        if (n != total) fail(MPMB_INVALID_ARGUMENT, "bind_results: n must equal the particle count");
        Engine::host_register(pos, 12 * static_cast<size_t>(n));
        Engine::host_register(vel, 12 * static_cast<size_t>(n));
        Engine::host_register(active, static_cast<size_t>(n));
        b->bound_x = pos;
        b->bound_v = vel;
        b->bound_a = active;
        b->bound_n = n;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_result_wait(mpmb_handle h) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        bool is_batch = false;
        Batch* b = batch_of_handle(reg(), h, is_batch);
        if (!b) return MPMB_BAD_HANDLE;
        if (b->eng) b->eng->wait_results();
        return MPMB_OK;
    });
}

extern "C" int32_t mpmb_particle_count(mpmb_handle sh) {
    std::lock_guard<std::mutex> lk(reg().mu);
    Scene* s = reg().scene(sh);
    return s ? static_cast<int32_t>(s->count()) : -1;
}

namespace {
void current_particles(Scene* s, float* x, float* v, float* F, float* C, uint8_t* a) {
    Batch& b = *s->batch;
    if (b.device_valid && b.eng) {
        size_t si = 0;
        while (b.scenes[si] != s) ++si;
        b.eng->download_particles(static_cast<int64_t>(b.offsets[si]), static_cast<int64_t>(s->count()),
                                  x, v, nullptr, nullptr, F, C, nullptr, nullptr, a);
    } else {
        if (x) std::copy(s->x.begin(), s->x.end(), x);
        if (v) std::copy(s->v.begin(), s->v.end(), v);
        if (F) std::copy(s->F.begin(), s->F.end(), F);
        if (C) std::copy(s->C.begin(), s->C.end(), C);
        if (a) std::copy(s->active.begin(), s->active.end(), a);
    }
}
}  // namespace

extern "C" mpmb_status mpmb_copy_positions(mpmb_handle sh, float* out, size_t cap, size_t* written) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        Scene* s = reg().scene(sh);
        if (!s) return MPMB_BAD_HANDLE;
        const size_t w = 3 * s->count();
        if (written) *written = w;
        if (cap < w) return MPMB_BUFFER_TOO_SMALL;  // facade.hpp:197
        current_particles(s, out, nullptr, nullptr, nullptr, nullptr);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_scene_get_particles(mpmb_handle sh, float* x, float* v, float* F,
                                                float* C, uint8_t* a) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        Scene* s = reg().scene(sh);
        if (!s) return MPMB_BAD_HANDLE;
        current_particles(s, x, v, F, C, a);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_shape_impulse(mpmb_handle sh, mpmb_handle shape, float out[3]) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        Registry& r = reg();
        Scene* s = r.scene(sh);
        Entry* e = r.find(shape, Kind::shape);
        if (!s || !e || e->scene != sh) return MPMB_BAD_HANDLE;
        Batch& b = *s->batch;
        for (size_t i = 0; i < s->shapes.size(); ++i)
            if (s->shapes[i].id == e->inner_id) {
                out[0] = out[1] = out[2] = 0.f;
                if (b.eng && !b.shapes_dirty) {  // frame accumulators (scene.hpp:140-142)
                    size_t si = 0;
                    while (b.scenes[si] != s) ++si;
                    std::vector<double> imp, tq;
                    std::vector<int32_t> cc;
                    b.eng->read_contact(1, imp, tq, cc);
                    const size_t gi = b.shape_offsets[si] + i;
                    for (int q = 0; q < 3; ++q) out[q] = static_cast<float>(imp[3 * gi + q]);
                }
                return MPMB_OK;
            }
        return MPMB_BAD_HANDLE;
    });
}

namespace {
template <class F>
mpmb_status with_batch(mpmb_handle h, F&& f) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        bool is_batch;
        Batch* b = batch_of_handle(reg(), h, is_batch);
        if (!b) return MPMB_BAD_HANDLE;
        return f(*b);
    });
}
}  // namespace

extern "C" mpmb_status mpmb_set_stream(mpmb_handle h, void* stream) {
    return with_batch(h, [&](Batch& b) {
        b.stream = stream;
        if (b.eng) b.eng->set_stream(stream);
        return MPMB_OK;
    });
}

// ------------------------------------------------ scenario metrics (k_scenario.cu)
namespace {
// handle -> (batch, scenes addressed): a batch handle addresses all its scenes, a scene
// handle its own; the device state must be current (no frame pending)
Batch* metrics_target(mpmb_handle h, std::vector<size_t>& idx) {
    bool is_batch;
    Batch* b = batch_of_handle(reg(), h, is_batch);
    if (!b) return nullptr;
    if (b->status == Status::advancing) fail(MPMB_LIFECYCLE_ERROR, "metrics: fetch the pending frame first");
    if (is_batch) {
        for (size_t i = 0; i < b->scenes.size(); ++i) idx.push_back(i);
    } else {
        Scene* s = reg().scene(h);
        for (size_t i = 0; i < b->scenes.size(); ++i)
            if (b->scenes[i] == s) idx.push_back(i);
    }
    if (!b->device_valid || b->particles_dirty || b->shapes_dirty) upload(*b);
    return b;
}
}  // namespace

extern "C" mpmb_status mpmb_components(mpmb_handle h, const float* radius, int32_t* count) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        if (!radius || !count) fail(MPMB_INVALID_ARGUMENT, "null argument");
        std::vector<size_t> idx;
        Batch* b = metrics_target(h, idx);
        if (!b) return MPMB_BAD_HANDLE;
        std::vector<float> r(b->scenes.size(), radius[0]);
        for (size_t k = 0; k < idx.size(); ++k) {
            if (!(radius[k] > 0)) fail(MPMB_INVALID_ARGUMENT, "components: radius must be positive");
            r[idx[k]] = radius[k];
        }
        std::vector<int32_t> c(b->scenes.size(), 0);
        b->eng->components(r.data(), c.data());
        for (size_t k = 0; k < idx.size(); ++k) count[k] = c[idx[k]];
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_nn_spacing(mpmb_handle h, const float* cell_hint, float* spacing) {
    std::lock_guard<std::mutex> lk(reg().mu);
    return guarded([&]() -> mpmb_status {
        if (!cell_hint || !spacing) fail(MPMB_INVALID_ARGUMENT, "null argument");
        std::vector<size_t> idx;
        Batch* b = metrics_target(h, idx);
        if (!b) return MPMB_BAD_HANDLE;
        std::vector<float> cell(b->scenes.size(), cell_hint[0]);
        for (size_t k = 0; k < idx.size(); ++k) {
            if (!(cell_hint[k] > 0)) fail(MPMB_INVALID_ARGUMENT, "nn_spacing: cell hint must be positive");
            cell[idx[k]] = cell_hint[k];
        }
        size_t total = 0;
        for (Scene* s : b->scenes) total += s->count();
        std::vector<float> best2(total, FLT_MAX);
        if (total) b->eng->nn_best2(cell.data(), best2.data());
        for (size_t k = 0; k < idx.size(); ++k) {  // scenario.hpp:73-95, original order, FP64 sum
            const size_t si = idx[k], o = b->offsets[si], n = b->scenes[si]->count();
            double sum = 0;
            size_t cnt = 0;
            for (size_t i = 0; i < n; ++i)
                if (best2[o + i] < FLT_MAX) {
                    sum += std::sqrt(double(best2[o + i]));
                    ++cnt;
                }
            spacing[k] = cnt ? static_cast<float>(sum / cnt) : cell_hint[k];
        }
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_set_exact(mpmb_handle h, int32_t on) {
    return with_batch(h, [&](Batch& b) {
        b.exact = on != 0;
        if (b.eng) b.eng->set_exact(b.exact);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_set_fusion(mpmb_handle h, int32_t mode) {
    return with_batch(h, [&](Batch& b) {
        if (mode < 0 || mode > 2) return MPMB_INVALID_ARGUMENT;
        b.fusion = mode;
        if (b.eng) b.eng->set_fusion(mode);
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_set_resort_interval(mpmb_handle h, int32_t k) {
    return with_batch(h, [&](Batch& b) {
        if (k < 0) return MPMB_INVALID_ARGUMENT;
        b.resort = k;
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_set_profiling(mpmb_handle h, int32_t on) {
    return with_batch(h, [&](Batch& b) {
        b.profiling = on != 0;
        if (b.eng) {
            b.eng->set_profiling(b.profiling);
            b.eng->reset_kernel_times();
        }
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_get_profile(mpmb_handle h, mpmb_profile* out) {
    return with_batch(h, [&](Batch& b) {
        if (!out) return MPMB_INVALID_ARGUMENT;
        *out = mpmb_profile{};
        if (b.eng) {
            KernelTimes t = b.eng->kernel_times();
            out->ms_sort = t.ms_sort;
            out->ms_p2g = t.ms_p2g;
            out->ms_grid = t.ms_grid;
            out->ms_g2p = t.ms_g2p;
            out->ms_other = t.ms_other;
            out->launches = t.launches;
            out->ms_fused = t.ms_fused;
            out->n_sort = t.n_sort;
            out->n_p2g = t.n_p2g;
            out->n_grid = t.n_grid;
            out->n_g2p = t.n_g2p;
            out->n_fused = t.n_fused;
        }
        return MPMB_OK;
    });
}

extern "C" mpmb_status mpmb_synchronize(mpmb_handle h) {
    return with_batch(h, [&](Batch& b) {
        if (b.eng) b.eng->synchronize();
        return MPMB_OK;
    });
}
