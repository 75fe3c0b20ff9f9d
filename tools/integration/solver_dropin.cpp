// A reference SOLVER-layer caller (the loop of Scene::run_frame, scene.hpp:199-235, written
// against solvers.hpp / contact.hpp / state.hpp directly, as the reference's own tests do)
// run twice on the same SimState: once with the reference's CPU functions (mpm::), once with
// the drop-in (mpm_b200::, include/mpm_b200_solver.hpp).  The only difference between the two
// loops is the namespace and, for the resident form, the DeviceSim in place of the SimState.
// Prints "key value" pairs that tests/test_integration.py checks.  Build: __graft_entry__.build().
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "mpm/rigid_dynamics.hpp"
#include "mpm_b200_solver.hpp"

namespace {

mpm::SimState make_state(mpm::MaterialKind kind) {
    mpm::SimState s;
    s.grid = mpm::Grid(32, 32, 32, 0.03125f, mpm::Vec3{});
    auto [mu, lambda] = mpm::lame_from_young_poisson(1e4f, 0.3f);
    mpm::Material m;
    m.kind = kind;
    m.mu = mu;
    m.lambda = lambda;
    m.beta = 0.9f;
    s.materials.push_back(m);
    mpm::spawn_box_particles(s.particles, s.grid, {0.3f, 0.12f, 0.3f}, {0.7f, 0.45f, 0.7f}, 8, 1000.f, 0, 77);
    for (auto& v : s.particles.v) v = {0.15f, -0.6f, 0.05f};
    return s;
}

std::vector<mpm::Shape> make_shapes() {
    std::vector<mpm::Shape> shapes(2);
    shapes[0].geometry = mpm::PlaneGeom{};
    shapes[0].pose.position = {0.5f, 0.1f, 0.5f};
    shapes[0].mu_k = 0.4f;
    shapes[0].c_d = 0.9f;
    shapes[0].collision_halfwidth = 0.75f * 0.03125f;
    mpm::SphereGeom ball;
    ball.radius = 0.08f;
    shapes[1].geometry = ball;
    shapes[1].pose.position = {0.5f, 0.52f, 0.5f};
    shapes[1].motion = mpm::MotionKind::free_body;
    shapes[1].body.mass = 0.5f;
    shapes[1].body.inertia_diag = {1e-3f, 1e-3f, 1e-3f};
    shapes[1].pose.linear_velocity = {0.f, -1.0f, 0.f};
    shapes[1].collision_halfwidth = 0.75f * 0.03125f;
    return shapes;
}

struct Diff {
    double x = 0, v = 0, vmax = 1e-30, C = 0, Cmax = 1e-30, F = 0, Fmax = 1e-30;
    int active_mismatch = 0;
};

Diff compare(const mpm::ParticleStore& a, const mpm::ParticleStore& b) {
    Diff d;
    for (size_t i = 0; i < a.size(); ++i) {
        d.active_mismatch += a.active[i] != b.active[i];
        const float* xa = &a.x[i].x;
        const float* xb = &b.x[i].x;
        const float* va = &a.v[i].x;
        const float* vb = &b.v[i].x;
        for (int k = 0; k < 3; ++k) {
            d.x = std::max(d.x, double(std::fabs(xa[k] - xb[k])));
            d.v = std::max(d.v, double(std::fabs(va[k] - vb[k])));
            d.vmax = std::max(d.vmax, double(std::fabs(va[k])));
        }
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                d.C = std::max(d.C, double(std::fabs(a.C[i].m[r][c] - b.C[i].m[r][c])));
                d.Cmax = std::max(d.Cmax, double(std::fabs(a.C[i].m[r][c])));
                d.F = std::max(d.F, double(std::fabs(a.F[i].m[r][c] - b.F[i].m[r][c])));
                d.Fmax = std::max(d.Fmax, double(std::fabs(a.F[i].m[r][c])));
            }
    }
    return d;
}

void report(const char* tag, const Diff& d, double dx) {
    std::printf("%s_dx %.6e\n%s_dv %.6e\n%s_dC %.6e\n%s_dF %.6e\n%s_active_mismatch %d\n", tag, d.x / dx, tag,
                d.v / d.vmax, tag, d.C / d.Cmax, tag, d.F / d.Fmax, tag, d.active_mismatch);
}

}  // namespace

int main() {
    const float dt = 0.002f;
    const mpm::Vec3 g{0.f, -9.81f, 0.f};
    const double dx = 0.03125;

    // ---- MLS, run_frame's substep loop: contact hook, push-out, free body, deactivation
    {
        mpm::SimState ref = make_state(mpm::MaterialKind::neo_hookean);
        mpm::SimState dev_host = ref;
        std::vector<mpm::Shape> shapes_ref = make_shapes(), shapes_dev = make_shapes();
        std::vector<mpm::ContactAccumulator> acc_ref(2), acc_dev(2);
        mpm_b200::DeviceSim dev(dev_host);
        int pushed_ref = 0, pushed_dev = 0, deact_ref = 0, deact_dev = 0;
        mpm::Vec3 frame_imp_ref{}, frame_imp_dev{};
        for (int s = 0; s < 60; ++s) {
            for (auto& a : acc_ref) a.reset();
            for (auto& a : acc_dev) a.reset();
            // reference: solvers.hpp / contact.hpp / state.hpp on the CPU
            mpm::step_mls(ref, dt, g, mpm_b200::ContactHook{&shapes_ref, &acc_ref}, mpm::BoundaryKind::slip);
            pushed_ref += mpm::particle_pushout(ref.particles, shapes_ref, ref.grid.dx);
            mpm::integrate_free_body(shapes_ref[1].pose, shapes_ref[1].body, acc_ref[1].impulse,
                                     acc_ref[1].torque_impulse, g, dt);
            deact_ref += mpm::deactivate_out_of_domain(ref.particles, ref.grid);
            // drop-in: the same calls, resident on the device
            mpm_b200::step_mls(dev, dt, g, mpm_b200::ContactHook{&shapes_dev, &acc_dev}, mpm::BoundaryKind::slip);
            pushed_dev += mpm_b200::particle_pushout(dev, shapes_dev, dev_host.grid.dx);
            mpm_b200::integrate_free_bodies(dev, shapes_dev, g, dt);
            deact_dev += mpm_b200::deactivate_out_of_domain(dev);
            frame_imp_ref += acc_ref[0].impulse;
            frame_imp_dev += acc_dev[0].impulse;
        }
        dev.download(dev_host);
        report("mls", compare(ref.particles, dev_host.particles), dx);
        std::printf("mls_pushed %d %d\nmls_deactivated %d %d\n", pushed_ref, pushed_dev, deact_ref, deact_dev);
        std::printf("mls_floor_impulse_y %.6e %.6e\n", frame_imp_ref.y, frame_imp_dev.y);
        std::printf("mls_ball_y %.6e %.6e\n", shapes_ref[1].pose.position.y, shapes_dev[1].pose.position.y);
        std::printf("mls_floor_nodes %d %d\n", acc_ref[0].contact_node_count, acc_dev[0].contact_node_count);
    }

    // ---- exact-signature forms on the reference's own SimState / ParticleStore
    {
        mpm::SimState ref = make_state(mpm::MaterialKind::neo_hookean);
        mpm::SimState dev = ref;
        const std::vector<mpm::Shape> shapes = make_shapes();
        std::vector<mpm::ContactAccumulator> acc_ref(2), acc_dev(2);
        for (int s = 0; s < 5; ++s) {
            mpm::step_mls(ref, dt, g, mpm_b200::ContactHook{&shapes, &acc_ref}, mpm::BoundaryKind::sticky);
            mpm_b200::step_mls(dev, dt, g, mpm_b200::ContactHook{&shapes, &acc_dev}, mpm::BoundaryKind::sticky);
            mpm::particle_pushout(ref.particles, shapes, ref.grid.dx);
            mpm_b200::particle_pushout(dev.particles, shapes, dev.grid.dx);
            mpm::deactivate_out_of_domain(ref.particles, ref.grid);
            mpm_b200::deactivate_out_of_domain(dev.particles, dev.grid);
        }
        report("exact", compare(ref.particles, dev.particles), dx);
        double gm = 0, gv = 0, gvmax = 1e-30;
        for (size_t i = 0; i < ref.grid.nodes.size(); ++i) {
            gm = std::max(gm, double(std::fabs(ref.grid.nodes[i].mass - dev.grid.nodes[i].mass)));
            if (ref.grid.nodes[i].mass <= mpm::kMassEpsilon) continue;
            const float* a = &ref.grid.nodes[i].velocity.x;
            const float* b = &dev.grid.nodes[i].velocity.x;
            for (int k = 0; k < 3; ++k) {
                gv = std::max(gv, double(std::fabs(a[k] - b[k])));
                gvmax = std::max(gvmax, double(std::fabs(a[k])));
            }
        }
        std::printf("exact_grid_dmass %.6e\nexact_grid_dv %.6e\n", gm, gv / gvmax);
    }

    // ---- PB-MPM and an arbitrary host grid hook (debug adapter)
    {
        mpm::SimState ref = make_state(mpm::MaterialKind::corotational_pb);
        mpm_b200::DeviceSim dev(ref);
        mpm::SimState out = ref;
        const std::vector<mpm::Shape> shapes = make_shapes();
        std::vector<mpm::ContactAccumulator> acc_ref(2), acc_dev(2);
        mpm::PbmpmConfig cfg;
        cfg.iterations = 5;
        const mpm::StepStats sr = mpm::step_pbmpm(ref, 0.01f, g, cfg, mpm_b200::ContactHook{&shapes, &acc_ref});
        const mpm::StepStats sd = mpm_b200::step_pbmpm(dev, 0.01f, g, cfg, mpm_b200::ContactHook{&shapes, &acc_dev});
        dev.download(out);
        report("pb", compare(ref.particles, out.particles), dx);
        std::printf("pb_failures %d %d\n", sr.projection_failures, sd.projection_failures);

        mpm::SimState ref2 = make_state(mpm::MaterialKind::neo_hookean);
        mpm::SimState dev2 = ref2;
        // a user hook: a damping zone above y = 0.35 (runs on the host through the adapter)
        const mpm::GridHook damp = [](mpm::Grid& gr) {
            for (size_t i = 0; i < gr.nodes.size(); ++i) {
                int a, b, c;
                gr.unindex(i, a, b, c);
                if (gr.nodes[i].mass > mpm::kMassEpsilon && gr.node_position(a, b, c).y > 0.35f)
                    gr.nodes[i].velocity = gr.nodes[i].velocity * 0.5f;
            }
        };
        for (int s = 0; s < 3; ++s) {
            mpm::step_mls(ref2, dt, g, damp);
            mpm_b200::step_mls(dev2, dt, g, damp);
        }
        report("hook", compare(ref2.particles, dev2.particles), dx);
    }
    std::printf("done 1\n");
    return 0;
}
