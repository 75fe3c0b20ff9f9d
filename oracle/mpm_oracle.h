/*
 * mpm_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference CPU algorithm for the per-substep MPM hot
 * path (CRESSim-MPM, /root/reference/proj/include/mpm/*.hpp).  Every function in
 * mpm_oracle.c cites the reference file:line it restates and keeps the reference's
 * float operation order, so that built with -O2 -ffp-contract=off (no FMA) it is
 * bit-identical to the reference built as oracle/_ref/libmpmref.so; that claim is
 * pinned by tests/test_oracle_pin.py and the golden fixtures in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library — as the checker, never as the measured or shipped path.
 */
#ifndef MPM_ORACLE_H
#define MPM_ORACLE_H

#include "../include/mpm_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpmor_state_s* mpmor_state;
typedef struct mpmor_scene_s* mpmor_scene;

/* solver layer (same meaning as the mpmb_state_* functions) */
mpmb_status mpmor_state_create(const int32_t dims[3], float dx, const float origin[3],
                               mpmor_state* out);
mpmb_status mpmor_state_destroy(mpmor_state st);
mpmb_status mpmor_state_set_materials(mpmor_state st, const mpmb_material* m, int32_t n);
mpmb_status mpmor_state_set_particles(mpmor_state st, int32_t n, const float* x, const float* v,
                                      const float* mass, const float* vol0, const float* F,
                                      const float* C, const float* stress, const int32_t* mat,
                                      const uint8_t* active);
mpmb_status mpmor_state_get_particles(mpmor_state st, int32_t n, float* x, float* v, float* mass,
                                      float* vol0, float* F, float* C, float* stress,
                                      int32_t* mat, uint8_t* active);
mpmb_status mpmor_state_set_shapes(mpmor_state st, const mpmb_shape_desc* d, int32_t n);
mpmb_status mpmor_state_get_shape_poses(mpmor_state st, mpmb_pose* out, int32_t n);
mpmb_status mpmor_state_get_contact(mpmor_state st, float* imp, float* tq, int32_t* cnt,
                                    int32_t n);
mpmb_status mpmor_state_reset_contact(mpmor_state st);
mpmb_status mpmor_step_standard(mpmor_state st, float dt, const float g[3], int32_t contact,
                                int32_t boundary, mpmb_step_stats* stats);
mpmb_status mpmor_step_mls(mpmor_state st, float dt, const float g[3], int32_t contact,
                           int32_t bc, mpmb_step_stats* stats);
mpmb_status mpmor_step_pbmpm(mpmor_state st, float dt, const float g[3], int32_t iterations,
                             int32_t contact, int32_t bc, mpmb_step_stats* stats);
mpmb_status mpmor_particle_pushout(mpmor_state st, int32_t* count);
mpmb_status mpmor_deactivate_out_of_domain(mpmor_state st, int32_t* count);
mpmb_status mpmor_integrate_free_bodies(mpmor_state st, const float g[3], float dt);
mpmb_status mpmor_state_get_grid(mpmor_state st, float* mass, float* mom, float* vel);
/* contact pass in double precision (impulse, torque) — the tolerance reference for
 * the device's reduction order */
mpmb_status mpmor_state_get_contact_f64(mpmor_state st, double* imp, double* tq, int32_t n);
/* binning oracle: brick-major cell key + stable permutation (see mpmb_bin_particles) */
void mpmor_set_order_perturbation(int32_t mode);
mpmb_status mpmor_bin_particles(mpmor_state st, uint32_t* keys, uint32_t* perm);

/* scene layer (Scene, scene.hpp:45-294) */
mpmor_scene mpmor_scene_create(const mpmb_scene_config* c);
void mpmor_scene_destroy(mpmor_scene s);
int32_t mpmor_scene_add_material(mpmor_scene s, const mpmb_material* m);
int32_t mpmor_scene_create_particle_object(mpmor_scene s, const float mn[3], const float mx[3],
                                           int32_t ppc, float density, int32_t mat,
                                           uint64_t seed);
int32_t mpmor_scene_create_shape(mpmor_scene s, const mpmb_shape_desc* d);
mpmb_status mpmor_scene_set_pose_target(mpmor_scene s, int32_t shape_id, const float p[3],
                                        const float q[4]);
mpmb_status mpmor_scene_advance(mpmor_scene s, float dt);
mpmb_status mpmor_scene_fetch(mpmor_scene s, mpmb_frame_summary* out);
int32_t mpmor_scene_particle_count(mpmor_scene s);
mpmb_status mpmor_scene_get_particles(mpmor_scene s, float* x, float* v, float* F, float* C,
                                      uint8_t* active);
mpmb_status mpmor_scene_shape_results(mpmor_scene s, int32_t* ids, float* imp, float* tq);

/* unit-level restatements used by the KAT tests */
void mpmor_spline_weights(const float pos[3], const float origin[3], float dx, int32_t base[3],
                          float w[9], float dw[9]);
int32_t mpmor_spline_in_domain(const float pos[3], const float origin[3], float dx,
                               const int32_t dims[3]);
void mpmor_neo_hookean(const float F[9], float mu, float lambda, float out[9]);
int32_t mpmor_polar(const float M[9], float R[9], float U[9]);
int32_t mpmor_corotational_project(const float Fp[9], const float Cc[9], float dt, float beta,
                                   float out[9]);
void mpmor_sdf_query(const mpmb_shape_desc* d, const float point[3], float* distance,
                     float normal[3], float tangent[3], int32_t* region);
void mpmor_evaluate_trajectory(const mpmb_keyframe* kf, int32_t n, float t, mpmb_pose* out);
void mpmor_lame(float E, float nu, float* mu, float* lambda);
/* spawn_box_particles into caller buffers; returns count or -1 (invalid) / -2 (capacity). */
int32_t mpmor_spawn_box(const int32_t dims[3], float dx, const float origin[3], const float mn[3],
                        const float mx[3], int32_t ppc, float density, uint64_t seed,
                        int32_t capacity, float* x, float* mass, float* vol0);

#ifdef __cplusplus
}
#endif
#endif
