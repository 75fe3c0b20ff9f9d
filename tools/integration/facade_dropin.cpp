// Example of a reference-facade caller switched to the B200 engine by one alias
// (INTEGRATION.md).  Build: see tests/test_integration.py.
#include <cstdio>
#include "mpm_b200_facade.hpp"

namespace facade = mpm_b200::facade;  // was: namespace facade = mpm::facade;

int main() {
    mpm::SceneConfig cfg;  // 56^3, dx 0.025, MLS, 10 substeps (scene.hpp:15-24)
    facade::Handle scene = facade::create_scene(cfg);
    auto [mu, lambda] = mpm::lame_from_young_poisson(1e4f, 0.3f);
    mpm::Material m;
    m.mu = mu;
    m.lambda = lambda;
    facade::Handle mat = facade::create_material(scene, m);
    facade::create_particle_object(scene, mat, {0.4875f, 0.3f, 0.4875f}, {0.8875f, 0.7f, 0.8875f}, 8, 1000.f, 12345);
    mpm::Shape floor;
    floor.geometry = mpm::PlaneGeom{};
    floor.pose.position = {0.7f, 0.0625f, 0.7f};
    floor.mu_k = 0.4f;
    floor.c_d = 0.9f;
    facade::Handle sh = facade::create_shape(scene, floor);
    mpm::FrameResult r;
    for (int f = 0; f < 3; ++f) {
        if (facade::advance(scene, 0.02f) != facade::Status::ok) { std::printf("advance failed: %s\n", mpmb_last_error()); return 1; }
        if (facade::fetch_results(scene, r) != facade::Status::ok) return 1;
    }
    mpm::Vec3 imp;
    facade::shape_impulse(scene, sh, imp);
    std::printf("particles %zu mass %.6f min_y %.6f impulse_y %.6g\n", r.positions.size(), r.total_mass,
                r.positions[0].y, imp.y);
    facade::destroy(scene);
    return 0;
}
