// mpm_b200_solver.hpp — drop-in for the reference's SOLVER layer (proj/include/mpm), on the
// B200 engine through the C-ABI of include/mpm_b200.h:
//
//   reference (CPU, serial)                                 here (device, resident in HBM)
//   mpm::step_mls(SimState&, dt, g, hook, bc)    solvers.hpp:141-198   mpm_b200::step_mls
//   mpm::step_standard(SimState&, dt, g, hook, bc) solvers.hpp:80-138  mpm_b200::step_standard
//   mpm::step_pbmpm(SimState&, dt, g, cfg, hook, bc) solvers.hpp:207-279 mpm_b200::step_pbmpm
//   mpm::apply_contact_pass(Grid&, shapes, acc)  contact.hpp:97-136    mpm_b200::ContactHook
//   mpm::particle_pushout(ParticleStore&, shapes, dx) contact.hpp:140-179 mpm_b200::particle_pushout
//   mpm::deactivate_out_of_domain(ParticleStore&, Grid&) state.hpp:153-164 mpm_b200::deactivate_out_of_domain
//   mpm::integrate_free_body per free shape      rigid_dynamics.hpp:82-103 mpm_b200::integrate_free_bodies
//
// Two forms of every call:
//  * RESIDENT: the first argument is a mpm_b200::DeviceSim -- the SimState mirrored in HBM
//    (upload once, step many times, download when the host needs the state).  This is the
//    fast path: nothing crosses PCIe between steps.
//  * EXACT SIGNATURE: the first argument is the reference's own mpm::SimState& /
//    ParticleStore&; the call uploads, runs on the device and downloads the state (and the
//    dense grid, as the reference leaves it in SimState::grid).  Same results, but each call
//    pays the host copies -- keep a DeviceSim for repeated steps.
//
// The grid hook (solvers.hpp:19, 63: after v = p/m + g dt, before BC):
//  * mpm_b200::ContactHook{&shapes, &acc} is the hook Scene installs (scene.hpp:190-192).
//    As a std::function it is also an ordinary reference GridHook (its operator() calls
//    mpm::apply_contact_pass), so one caller line serves both libraries; the device step
//    recognises it (std::function::target) and runs the contact pass inside the grid-update
//    kernel, adding the per-shape impulse / torque / node count into `acc` as the reference
//    does (contact.hpp:127-132).
//  * any other hook runs on the host through the debug adapter (mpmb_step_mls_hooked:
//    download the dense grid, call the hook, upload it; MLS only, synchronous).
// Errors: the reference throws std::invalid_argument / std::logic_error; device failures
// (no GPU, CUDA errors) throw mpm_b200::DeviceError with mpmb_last_error().  There is no CPU
// fallback.
//
// Build: -I<reference>/proj/include -I<this repo>/include, link libmpm_b200.so.
#pragma once
#include <algorithm>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "mpm/contact.hpp"  // reference value types + apply_contact_pass (ContactHook on the reference path)
#include "mpm/solvers.hpp"
#include "mpm_b200.h"
#include "mpm_b200_types.hpp"

namespace mpm_b200 {

static_assert(sizeof(mpm::Vec3) == 12 && sizeof(mpm::Mat3) == 36, "reference Vec3 / Mat3 are packed floats");

struct DeviceError : std::runtime_error {
    mpmb_status status;
    DeviceError(mpmb_status s, const std::string& what)
        : std::runtime_error(what + ": " + mpmb_last_error()), status(s) {}
};

namespace detail {
inline void ok(mpmb_status s, const char* what) {
    if (s == MPMB_OK) return;
    if (s == MPMB_INVALID_ARGUMENT) throw std::invalid_argument(std::string(what) + ": " + mpmb_last_error());
    if (s == MPMB_LIFECYCLE_ERROR) throw std::logic_error(std::string(what) + ": " + mpmb_last_error());
    throw DeviceError(s, what);
}
inline const float* f(const std::vector<mpm::Vec3>& v) { return reinterpret_cast<const float*>(v.data()); }
inline float* f(std::vector<mpm::Vec3>& v) { return reinterpret_cast<float*>(v.data()); }
inline const float* f(const std::vector<mpm::Mat3>& v) { return reinterpret_cast<const float*>(v.data()); }
inline float* f(std::vector<mpm::Mat3>& v) { return reinterpret_cast<float*>(v.data()); }
}  // namespace detail

// The contact pass as a grid hook (see the header comment).
struct ContactHook {
    const std::vector<mpm::Shape>* shapes;
    std::vector<mpm::ContactAccumulator>* acc;
    void operator()(mpm::Grid& g) const { mpm::apply_contact_pass(g, *shapes, *acc); }
};

// A SimState mirrored in HBM (mpmb_state): grid geometry, materials, particles, and the
// shapes the contact hook / push-out / free-body integration use.
class DeviceSim {
  public:
    explicit DeviceSim(const mpm::SimState& s) {
        const int32_t dims[3] = {s.grid.dims[0], s.grid.dims[1], s.grid.dims[2]};
        float o[3];
        detail::put3(o, s.grid.origin);
        detail::ok(mpmb_state_create(dims, s.grid.dx, o, &h_), "mpmb_state_create");
        dims_[0] = dims[0], dims_[1] = dims[1], dims_[2] = dims[2];
        dx_ = s.grid.dx;
        origin_ = s.grid.origin;
        upload(s);
    }
    DeviceSim(const DeviceSim&) = delete;
    DeviceSim& operator=(const DeviceSim&) = delete;
    ~DeviceSim() { mpmb_state_destroy(h_); }

    mpmb_state handle() const { return h_; }
    int32_t size() const { return n_; }
    const int* dims() const { return dims_; }
    float dx() const { return dx_; }
    const mpm::Vec3& origin() const { return origin_; }

    // materials + ParticleStore (the cached stress included: MLS P2G reads it, solvers.hpp:156)
    void upload(const mpm::SimState& s) {
        std::vector<mpmb_material> m;
        for (const auto& x : s.materials) m.push_back(detail::material(x));
        detail::ok(mpmb_state_set_materials(h_, m.data(), static_cast<int32_t>(m.size())), "set_materials");
        const mpm::ParticleStore& p = s.particles;
        n_ = static_cast<int32_t>(p.size());
        detail::ok(mpmb_state_set_particles(h_, n_, detail::f(p.x), detail::f(p.v), p.mass.data(), p.volume0.data(),
                                            detail::f(p.F), detail::f(p.C), detail::f(p.stress),
                                            p.material_id.data(), p.active.data()),
                   "set_particles");
    }
    // ParticleStore back in original order (x, v, mass, volume0, F, C, stress, material, active)
    void download(mpm::ParticleStore& p) const {
        p.x.resize(n_), p.v.resize(n_), p.mass.resize(n_), p.volume0.resize(n_), p.F.resize(n_), p.C.resize(n_);
        p.stress.resize(n_), p.material_id.resize(n_), p.active.resize(n_);
        detail::ok(mpmb_state_get_particles(h_, n_, detail::f(p.x), detail::f(p.v), p.mass.data(), p.volume0.data(),
                                            detail::f(p.F), detail::f(p.C), detail::f(p.stress),
                                            p.material_id.data(), p.active.data()),
                   "get_particles");
    }
    // the dense grid of the last step, post-BC (node-major, as SimState::grid)
    void download(mpm::Grid& g) const {
        const size_t nn = static_cast<size_t>(dims_[0]) * dims_[1] * dims_[2];
        std::vector<float> m(nn), mom(3 * nn), vel(3 * nn);
        detail::ok(mpmb_state_get_grid(h_, m.data(), mom.data(), vel.data()), "get_grid");
        if (g.nodes.size() != nn) g = mpm::Grid(dims_[0], dims_[1], dims_[2], dx_, origin_);
        for (size_t i = 0; i < nn; ++i) {
            mpm::GridNode& n = g.nodes[i];
            n.mass = m[i];
            n.momentum = detail::get3(&mom[3 * i]);
            n.velocity = detail::get3(&vel[3 * i]);
        }
    }
    void download(mpm::SimState& s) const {
        download(s.particles);
        download(s.grid);
    }

    // Shapes as the reference passes them to apply_contact_pass / particle_pushout (poses as
    // given; free-body accumulators reset).  Re-uploaded only when they changed.
    void set_shapes(const std::vector<mpm::Shape>& shapes) {
        if (&shapes == last_shapes_ && same_poses(shapes)) return;
        std::vector<detail::ShapeStore> store(shapes.size());
        std::vector<mpmb_shape_desc> d;
        for (size_t i = 0; i < shapes.size(); ++i) d.push_back(detail::shape(shapes[i], store[i]));
        detail::ok(mpmb_state_set_shapes(h_, d.data(), static_cast<int32_t>(d.size())), "set_shapes");
        last_shapes_ = &shapes;
        poses_.clear();
        for (const auto& s : shapes) poses_.push_back(detail::pose(s.pose));
    }
    // device poses back into the shapes (free bodies move on the device)
    void get_shape_poses(std::vector<mpm::Shape>& shapes) {
        std::vector<mpmb_pose> p(shapes.size());
        detail::ok(mpmb_state_get_shape_poses(h_, p.data(), static_cast<int32_t>(p.size())), "get_shape_poses");
        for (size_t i = 0; i < shapes.size(); ++i) shapes[i].pose = detail::pose(p[i]);
        poses_ = p;
    }
    // per-shape accumulators since the last reset_contact, added into acc (contact.hpp:127-132)
    void add_contact(std::vector<mpm::ContactAccumulator>& acc) const {
        const size_t n = acc.size();
        std::vector<float> imp(3 * n), tq(3 * n);
        std::vector<int32_t> cnt(n);
        detail::ok(mpmb_state_get_contact(h_, imp.data(), tq.data(), cnt.data(), static_cast<int32_t>(n)),
                   "get_contact");
        for (size_t i = 0; i < n; ++i) {
            acc[i].impulse += detail::get3(&imp[3 * i]);
            acc[i].torque_impulse += detail::get3(&tq[3 * i]);
            acc[i].contact_node_count += cnt[i];
        }
    }
    void reset_contact() { detail::ok(mpmb_state_reset_contact(h_), "reset_contact"); }

  private:
    bool same_poses(const std::vector<mpm::Shape>& shapes) const {
        if (shapes.size() != poses_.size()) return false;
        for (size_t i = 0; i < shapes.size(); ++i) {
            const mpmb_pose p = detail::pose(shapes[i].pose);
            if (std::memcmp(&p, &poses_[i], sizeof(p)) != 0) return false;
        }
        return true;
    }
    mpmb_state h_ = nullptr;
    int32_t n_ = 0;
    int dims_[3] = {0, 0, 0};
    float dx_ = 0;
    mpm::Vec3 origin_;
    const std::vector<mpm::Shape>* last_shapes_ = nullptr;
    std::vector<mpmb_pose> poses_;
};

namespace detail {
inline int32_t bc(mpm::BoundaryKind b) { return b == mpm::BoundaryKind::sticky ? MPMB_BC_STICKY : MPMB_BC_SLIP; }

// The debug adapter's C callback: dense grid arrays <-> a reference Grid, then the hook.
struct HookCall {
    const mpm::GridHook* hook;
    int dims[3];
    float dx;
    mpm::Vec3 origin;
};
inline void hook_trampoline(void* user, int32_t n, float* mass, float* mom, float* vel) {
    HookCall& c = *static_cast<HookCall*>(user);
    mpm::Grid g(c.dims[0], c.dims[1], c.dims[2], c.dx, c.origin);
    for (int32_t i = 0; i < n; ++i) {
        g.nodes[i].mass = mass[i];
        g.nodes[i].momentum = get3(mom + 3 * i);
        g.nodes[i].velocity = get3(vel + 3 * i);
    }
    (*c.hook)(g);
    for (int32_t i = 0; i < n; ++i) {
        mass[i] = g.nodes[i].mass;
        put3(mom + 3 * i, g.nodes[i].momentum);
        put3(vel + 3 * i, g.nodes[i].velocity);
    }
}

// 0: no hook; 1: the device contact pass (ContactHook); 2: an arbitrary host hook
inline int hook_kind(DeviceSim& d, const mpm::GridHook& hook, const ContactHook*& ch) {
    ch = nullptr;
    if (!hook) return 0;
    if ((ch = hook.target<ContactHook>()) != nullptr) {
        if (ch->acc->size() < ch->shapes->size()) throw std::invalid_argument("contact: accumulator per shape");
        d.set_shapes(*ch->shapes);
        d.reset_contact();
        return 1;
    }
    return 2;
}
inline mpm::StepStats stats(const mpmb_step_stats& s) {
    mpm::StepStats o;
    o.inverted_f = s.inverted_f;
    o.projection_failures = s.projection_failures;
    return o;
}
}  // namespace detail

// ------------------------------------------------------------ resident forms (DeviceSim)
inline mpm::StepStats step_mls(DeviceSim& d, mpm::Real dt, const mpm::Vec3& gravity,
                               const mpm::GridHook& hook = nullptr,
                               mpm::BoundaryKind bc = mpm::BoundaryKind::slip) {
    float g[3];
    detail::put3(g, gravity);
    mpmb_step_stats st{};
    const ContactHook* ch;
    const int k = detail::hook_kind(d, hook, ch);
    if (k == 2) {
        detail::HookCall c{&hook, {d.dims()[0], d.dims()[1], d.dims()[2]}, d.dx(), d.origin()};
        detail::ok(mpmb_step_mls_hooked(d.handle(), dt, g, 0, detail::bc(bc), detail::hook_trampoline, &c, &st),
                   "step_mls");
        return detail::stats(st);
    }
    detail::ok(mpmb_step_mls(d.handle(), dt, g, k == 1, detail::bc(bc), &st), "step_mls");
    if (k == 1) d.add_contact(*ch->acc);
    return detail::stats(st);
}

inline mpm::StepStats step_standard(DeviceSim& d, mpm::Real dt, const mpm::Vec3& gravity,
                                    const mpm::GridHook& hook = nullptr,
                                    mpm::BoundaryKind bc = mpm::BoundaryKind::slip) {
    float g[3];
    detail::put3(g, gravity);
    mpmb_step_stats st{};
    const ContactHook* ch;
    const int k = detail::hook_kind(d, hook, ch);
    if (k == 2) throw std::invalid_argument("step_standard: host grid hooks are supported for step_mls only");
    detail::ok(mpmb_step_standard(d.handle(), dt, g, k == 1, detail::bc(bc), &st), "step_standard");
    if (k == 1) d.add_contact(*ch->acc);
    return detail::stats(st);
}

inline mpm::StepStats step_pbmpm(DeviceSim& d, mpm::Real dt, const mpm::Vec3& gravity, const mpm::PbmpmConfig& cfg,
                                 const mpm::GridHook& hook = nullptr,
                                 mpm::BoundaryKind bc = mpm::BoundaryKind::slip) {
    float g[3];
    detail::put3(g, gravity);
    mpmb_step_stats st{};
    const ContactHook* ch;
    const int k = detail::hook_kind(d, hook, ch);
    if (k == 2) throw std::invalid_argument("step_pbmpm: host grid hooks are supported for step_mls only");
    detail::ok(mpmb_step_pbmpm(d.handle(), dt, g, cfg.iterations, k == 1, detail::bc(bc), &st), "step_pbmpm");
    if (k == 1) d.add_contact(*ch->acc);  // summed over all iterations, as scene.hpp:196
    return detail::stats(st);
}

inline int particle_pushout(DeviceSim& d, const std::vector<mpm::Shape>& shapes, mpm::Real /*dx: the state's*/) {
    d.set_shapes(shapes);
    int32_t c = 0;
    detail::ok(mpmb_particle_pushout(d.handle(), &c), "particle_pushout");
    return c;
}

inline int deactivate_out_of_domain(DeviceSim& d) {
    int32_t c = 0;
    detail::ok(mpmb_deactivate_out_of_domain(d.handle(), &c), "deactivate_out_of_domain");
    return c;
}

// integrate_free_body (rigid_dynamics.hpp:82-103) for every free shape with the impulse the
// device accumulated since the last reset, as Scene::run_frame does (scene.hpp:220-226);
// the new poses are written back into `shapes`
inline void integrate_free_bodies(DeviceSim& d, std::vector<mpm::Shape>& shapes, const mpm::Vec3& gravity,
                                  mpm::Real dt) {
    d.set_shapes(shapes);
    float g[3];
    detail::put3(g, gravity);
    detail::ok(mpmb_integrate_free_bodies(d.handle(), g, dt), "integrate_free_bodies");
    d.get_shape_poses(shapes);
}

// ------------------------------------------------------------ exact-signature forms
inline mpm::StepStats step_mls(mpm::SimState& s, mpm::Real dt, const mpm::Vec3& g,
                               const mpm::GridHook& hook = nullptr,
                               mpm::BoundaryKind bc = mpm::BoundaryKind::slip) {
    DeviceSim d(s);
    const mpm::StepStats r = step_mls(d, dt, g, hook, bc);
    d.download(s);
    return r;
}

inline mpm::StepStats step_standard(mpm::SimState& s, mpm::Real dt, const mpm::Vec3& g,
                                    const mpm::GridHook& hook = nullptr,
                                    mpm::BoundaryKind bc = mpm::BoundaryKind::slip) {
    DeviceSim d(s);
    const mpm::StepStats r = step_standard(d, dt, g, hook, bc);
    d.download(s);
    return r;
}

inline mpm::StepStats step_pbmpm(mpm::SimState& s, mpm::Real dt, const mpm::Vec3& g, const mpm::PbmpmConfig& cfg,
                                 const mpm::GridHook& hook = nullptr,
                                 mpm::BoundaryKind bc = mpm::BoundaryKind::slip) {
    DeviceSim d(s);
    const mpm::StepStats r = step_pbmpm(d, dt, g, cfg, hook, bc);
    d.download(s);
    return r;
}

namespace detail {
// a state holding only the particles (push-out and deactivation never read the grid pools)
inline mpm::SimState particles_only(const mpm::ParticleStore& p, const mpm::Grid& like) {
    mpm::SimState s;
    s.grid = mpm::Grid(like.dims[0], like.dims[1], like.dims[2], like.dx, like.origin);
    s.particles = p;
    const int maxm = p.material_id.empty() ? 0 : *std::max_element(p.material_id.begin(), p.material_id.end());
    s.materials.resize(static_cast<size_t>(maxm) + 1);
    return s;
}
}  // namespace detail

inline int particle_pushout(mpm::ParticleStore& p, const std::vector<mpm::Shape>& shapes, mpm::Real dx) {
    // push-out reads only x, v, the shapes and dx (its clearance, contact.hpp:143)
    mpm::SimState s = detail::particles_only(p, mpm::Grid(4, 4, 4, dx, mpm::Vec3{}));
    DeviceSim d(s);
    const int c = particle_pushout(d, shapes, dx);
    d.download(p);
    return c;
}

inline int deactivate_out_of_domain(mpm::ParticleStore& p, const mpm::Grid& grid) {
    mpm::SimState s = detail::particles_only(p, grid);
    DeviceSim d(s);
    const int c = deactivate_out_of_domain(d);
    d.download(p);
    return c;
}

}  // namespace mpm_b200
