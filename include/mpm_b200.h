/*
 * mpm_b200.h — C-ABI of the B200-native MPM hot path (CRESSim-MPM, arxiv 2502.18437).
 *
 * Two layers, both plain C (no torch / C++ types in any signature):
 *
 *  1. Solver layer (mpmb_state_*, mpmb_step_*): one SimState resident in HBM.
 *     Replaces the free functions of the reference's header-only C++ API:
 *       mpm::step_mls                 proj/include/mpm/solvers.hpp:141-198
 *       mpm::step_pbmpm               proj/include/mpm/solvers.hpp:207-279
 *       mpm::apply_boundary_conditions proj/include/mpm/solvers.hpp:30-50
 *       mpm::apply_contact_pass       proj/include/mpm/contact.hpp:97-136  (as the step's grid hook)
 *       mpm::particle_pushout         proj/include/mpm/contact.hpp:140-179
 *       mpm::deactivate_out_of_domain proj/include/mpm/state.hpp:153-164
 *       mpm::integrate_free_body      proj/include/mpm/rigid_dynamics.hpp:82-103
 *     plus the NEW binning/sort stage (no reference function; key arithmetic of
 *     quadratic_bspline_weights math.hpp:219-225 and Grid::index state.hpp:39-43).
 *
 *  2. Scene facade (mpmb_create_scene ... mpmb_shape_impulse): the flat handle API
 *     of proj/include/mpm/facade.hpp:67-219 (itself the FFI boundary of the
 *     reference), with the same handle rules (never reused, 0 = invalid) and the
 *     same Status codes, plus batched scene replicas (mpmb_create_scene_batch)
 *     that advance together in one launch per kernel.
 *
 * Arrays are host pointers in the reference's layouts: Vec3 = 3 floats, Mat3 = 9
 * floats row-major (math.hpp:46-48), particles in ORIGINAL index order
 * (state.hpp:92-97, scene.hpp:255-257) regardless of the device-side sort.
 * No function throws; every function returns an mpmb_status (or a handle where
 * the reference facade returns one).  Without a usable CUDA device every entry
 * point that needs one returns MPMB_NO_DEVICE — there is no CPU fallback.
 */
#ifndef MPM_B200_H
#define MPM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPMB_ABI_VERSION 1

/* mpm::facade::Status (facade.hpp:18-24) + device errors. */
typedef enum {
    MPMB_OK = 0,
    MPMB_BAD_HANDLE = 1,
    MPMB_LIFECYCLE_ERROR = 2,
    MPMB_INVALID_ARGUMENT = 3,
    MPMB_BUFFER_TOO_SMALL = 4,
    MPMB_CUDA_ERROR = 5,
    MPMB_NO_DEVICE = 6
} mpmb_status;

/* mpm::SolverKind (scene.hpp:13) */
enum { MPMB_SOLVER_STANDARD = 0, MPMB_SOLVER_MLS = 1, MPMB_SOLVER_PBMPM = 2 };
/* mpm::BoundaryKind (solvers.hpp:21) */
enum { MPMB_BC_SLIP = 0, MPMB_BC_STICKY = 1 };
/* mpm::MaterialKind (materials.hpp:11) */
enum { MPMB_MAT_NEO_HOOKEAN = 0, MPMB_MAT_COROTATIONAL_PB = 1 };
/* alternatives of mpm::Geometry, in variant order (geometry.hpp:84-86) */
enum {
    MPMB_GEOM_PLANE = 0,
    MPMB_GEOM_SPHERE = 1,
    MPMB_GEOM_BOX = 2,
    MPMB_GEOM_QUAD_SLICER = 3,
    MPMB_GEOM_TRI_MESH_SLICER = 4,
    MPMB_GEOM_ARC = 5,
    MPMB_GEOM_POLYLINE = 6
};
/* mpm::MotionKind (rigid_dynamics.hpp:105) */
enum { MPMB_MOTION_FIXED = 0, MPMB_MOTION_KINEMATIC = 1, MPMB_MOTION_FREE_BODY = 2 };
/* mpm::SdfRegion (geometry.hpp:34) */
enum { MPMB_REGION_BULK = 0, MPMB_REGION_SURFACE = 1, MPMB_REGION_EDGE = 2,
       MPMB_REGION_SPINE = 3, MPMB_REGION_CURVE = 4 };

/* mpm::ShapePose (geometry.hpp:14-27); quaternion is (x, y, z, w). */
typedef struct {
    float position[3];
    float orientation[4];
    float linear_velocity[3];
    float angular_velocity[3];
} mpmb_pose;

/* mpm::Keyframe (rigid_dynamics.hpp:11-15) */
typedef struct {
    float time;
    float position[3];
    float orientation[4];
} mpmb_keyframe;

/* mpm::Material (materials.hpp:13-18) */
typedef struct {
    int32_t kind;
    float mu;
    float lambda;
    float beta;
} mpmb_material;

/*
 * mpm::Shape (rigid_dynamics.hpp:107-117) with the Geometry variant flattened.
 * gparam by geometry:
 *   sphere: [radius]; box: [hx, hy, hz]; quad slicer: [half_length, half_height,
 *   spine_radius]; tri mesh slicer: [spine_radius]; arc: [radius, angle];
 *   plane / polyline: unused.
 * vertices (local frame, 3 floats each) are used by the mesh slicer and polyline;
 * indices (triangle list) and spine_edges (vertex pairs) by the mesh slicer.
 * keyframes are read for motion == KINEMATIC (scene layer only), body_mass and
 * inertia for motion == FREE_BODY.  All pointers are copied at the call.
 */
typedef struct {
    int32_t geometry;
    float gparam[4];
    const float* vertices;
    int32_t n_vertices;
    const int32_t* indices;
    int32_t n_indices;
    const int32_t* spine_edges;
    int32_t n_spine_edges;
    mpmb_pose pose;
    float mu_k;
    float c_d;
    float collision_halfwidth;
    int32_t motion;
    const mpmb_keyframe* keyframes;
    int32_t n_keyframes;
    float body_mass;
    float inertia[3];
} mpmb_shape_desc;

/* mpm::StepStats (solvers.hpp:23-26) */
typedef struct {
    int32_t inverted_f;
    int32_t projection_failures;
} mpmb_step_stats;

/* mpm::SceneConfig (scene.hpp:15-24) */
typedef struct {
    int32_t solver;
    int32_t substeps;
    int32_t iterations;
    float gravity[3];
    int32_t grid_dims[3];
    float dx;
    float origin[3];
    int32_t boundary;
} mpmb_scene_config;

/* Scalar part of mpm::FrameResult (scene.hpp:28-43); arrays via mpmb_result_copy. */
typedef struct {
    float time;
    int32_t n_particles;
    int32_t n_shapes;
    double total_mass;
    double momentum[3];
    double kinetic_energy;
    int32_t pushed_out;
    int32_t inverted_f;
    int32_t projection_failures;
    int32_t deactivated;
} mpmb_frame_summary;

/* Device-side timing of the last advance()s, accumulated while profiling is on. */
typedef struct {
    double ms_sort;
    double ms_p2g;
    double ms_grid;
    double ms_g2p;
    double ms_other;
    int64_t launches;            /* kernels launched by the library while profiling */
    int64_t particle_substeps;   /* active particles x substeps (PB: x iterations) */
    double ms_fused;             /* k_g2p2g: G2P of substep s fused with P2G of s+1 (+ collect) */
    /* timed operations per class (one binning, P2G, grid update, G2P or fused launch each) */
    int64_t n_sort, n_p2g, n_grid, n_g2p, n_fused;
} mpmb_profile;

/* ------------------------------------------------------------------ library */
int32_t mpmb_abi_version(void);
/* 1 when a CUDA device is usable by this process, else 0. */
int32_t mpmb_device_available(void);
/* Last error text of the calling thread ("" if none). */
const char* mpmb_last_error(void);
/* Total kernels this process launched through the library. */
int64_t mpmb_kernel_launch_count(void);
/* The device's P2G stress function on n row-major F matrices (known-answer tests): the
 * cancellation-free FP32 form of neo_hookean_cauchy_stress (materials.hpp:35-54) that P2G
 * evaluates; sigma 9n floats, J (may be NULL) n floats. */
mpmb_status mpmb_eval_stress_f32(const float* F, int64_t n, float mu, float lambda, float* sigma, float* J);

/* ------------------------------------------------------------ solver layer */
typedef struct mpmb_state_s* mpmb_state;

/* mpm::Grid(nx, ny, nz, dx, origin) (state.hpp:29-37): dims >= 4, dx > 0. */
mpmb_status mpmb_state_create(const int32_t dims[3], float dx, const float origin[3],
                              mpmb_state* out);
mpmb_status mpmb_state_destroy(mpmb_state st);
mpmb_status mpmb_state_set_materials(mpmb_state st, const mpmb_material* mats, int32_t n);
/* Upload a ParticleStore (state.hpp:65-90). stress may be NULL (= cached sigma of F). */
mpmb_status mpmb_state_set_particles(mpmb_state st, int32_t n, const float* x, const float* v,
                                     const float* mass, const float* volume0, const float* F,
                                     const float* C, const float* stress,
                                     const int32_t* material_id, const uint8_t* active);
/* Download in original order; any pointer may be NULL. */
mpmb_status mpmb_state_get_particles(mpmb_state st, int32_t n, float* x, float* v, float* mass,
                                     float* volume0, float* F, float* C, float* stress,
                                     int32_t* material_id, uint8_t* active);
int32_t mpmb_state_particle_count(mpmb_state st);
/* Shapes used by the contact pass, push-out and free-body integration. */
mpmb_status mpmb_state_set_shapes(mpmb_state st, const mpmb_shape_desc* shapes, int32_t n);
mpmb_status mpmb_state_get_shape_poses(mpmb_state st, mpmb_pose* out, int32_t n);
/* ContactAccumulator per shape (contact.hpp:10-16), summed since the last reset. */
mpmb_status mpmb_state_get_contact(mpmb_state st, float* impulse, float* torque_impulse,
                                   int32_t* contact_node_count, int32_t n);
mpmb_status mpmb_state_reset_contact(mpmb_state st);

/* step_mls; contact != 0 installs apply_contact_pass over the state's shapes as the hook. */
mpmb_status mpmb_step_mls(mpmb_state st, float dt, const float gravity[3], int32_t contact,
                          int32_t boundary, mpmb_step_stats* stats);
/* step_standard (solvers.hpp:80-138): PIC transfers, nodal force -dt V sigma grad w. */
mpmb_status mpmb_step_standard(mpmb_state st, float dt, const float gravity[3], int32_t contact,
                               int32_t boundary, mpmb_step_stats* stats);
/* step_pbmpm with PbmpmConfig{iterations}. */
mpmb_status mpmb_step_pbmpm(mpmb_state st, float dt, const float gravity[3], int32_t iterations,
                            int32_t contact, int32_t boundary, mpmb_step_stats* stats);

/* Host GridHook adapter (solvers.hpp:19, 63): called after v = p/m + g dt (and after the
 * contact pass when contact != 0), before BC, with the dense grid in node-major order
 * (state.hpp:26); edits are uploaded back.  Debug path: synchronous download/upload. */
typedef void (*mpmb_grid_hook)(void* user, int32_t n_nodes, float* mass, float* momentum,
                               float* velocity);
mpmb_status mpmb_step_mls_hooked(mpmb_state st, float dt, const float gravity[3],
                                 int32_t contact, int32_t boundary, mpmb_grid_hook hook,
                                 void* user, mpmb_step_stats* stats);

mpmb_status mpmb_particle_pushout(mpmb_state st, int32_t* count);
mpmb_status mpmb_deactivate_out_of_domain(mpmb_state st, int32_t* count);
/* integrate_free_body for every FREE_BODY shape with its accumulated impulse. */
mpmb_status mpmb_integrate_free_bodies(mpmb_state st, const float gravity[3], float dt);

/* Dense grid after the last step (post-BC); any pointer may be NULL.
 * Node-major i + nx*(j + ny*k); momentum/velocity are 3 floats per node. */
mpmb_status mpmb_state_get_grid(mpmb_state st, float* mass, float* momentum, float* velocity);

/* Binning (NEW stage, K1): for every particle in original order, keys[i] = linear stencil-base
 * cell b_x + nx*(b_y + ny*b_z) (0xFFFFFFFF for inactive); perm = original indices sorted stably
 * by (key, original index), inactive last.  Any pointer may be NULL. */
mpmb_status mpmb_bin_particles(mpmb_state st, uint32_t* keys, uint32_t* perm);

/* ------------------------------------------- slab domain decomposition (DD)
 * One large scene split along x into slabs, one per rank.
 * A slab state owns global x nodes [slab_lo, slab_hi) and stores [slab_lo - margin,
 * slab_hi + 2 + margin).  All arithmetic uses the GLOBAL grid (keys, node positions, BC,
 * deactivation), so a DD run equals the single-domain run up to float summation order.
 * The production loop is the library's device-resident driver (mpmb_dd_run, below).  The
 * per-phase entries here let a caller drive the same loop itself (paper_2502_18437_b200/dd.py
 * does, as the readable restatement and for the gloo CPU tests):
 *   mpmb_dd_p2g -> pack_acc -> [exchange] -> unpack_acc -> mpmb_dd_grid -> pack_vel ->
 *   [exchange] -> unpack_vel -> mpmb_dd_g2p [-> free bodies: all-reduce the sums of
 *   mpmb_dd_contact_sums, then mpmb_dd_free_bodies on every slab]
 * and every `margin` substeps (CFL: <= 1 cell per substep) mpmb_dd_migrate_pack ->
 * [exchange] -> mpmb_dd_migrate_unpack.  Exchange rule (both phases): send_lo goes to the
 * lower neighbour's recv_hi, send_hi to the upper neighbour's recv_lo; a missing
 * neighbour's recv buffer stays zero. */
mpmb_status mpmb_state_create_slab(const int32_t dims[3], float dx, const float origin[3], int32_t slab_lo,
                                   int32_t slab_hi, int32_t margin, int64_t capacity, mpmb_state* out);
/* The reference's particle lattice of create_particle_object (state.hpp:101-149, host,
 * bit-exact): jittered ppc-per-cell points in [box_min, box_max), mass and volume0. */
mpmb_status mpmb_spawn_box(const int32_t dims[3], float dx, const float origin[3], const float box_min[3],
                           const float box_max[3], int32_t ppc, float density, uint64_t seed, int64_t capacity,
                           float* x, float* mass, float* volume0, int64_t* n);
/* Particles with explicit original indices (global ids that travel with migration). */
mpmb_status mpmb_state_set_particles_ids(mpmb_state st, int32_t n, const float* x, const float* v,
                                         const float* mass, const float* volume0, const float* F,
                                         const float* C, const int32_t* material_id, const uint8_t* active,
                                         const uint32_t* ids);
/* Exact mode for the solver layer (see mpmb_set_exact). */
mpmb_status mpmb_state_set_exact(mpmb_state st, int32_t on);
/* Stream the state's kernels run on (NULL = the library's own). */
mpmb_status mpmb_state_set_stream(mpmb_state st, void* cuda_stream);
mpmb_status mpmb_state_synchronize(mpmb_state st);
/* Halo buffers (device, `bytes` each) and their layout: plane_bytes per x-plane; in the
 * grid-sum phase send_lo carries `margin` planes and send_hi `2 + margin`, in the
 * velocity phase the reverse. */
mpmb_status mpmb_dd_halo_buffers(mpmb_state st, void** send_lo, void** send_hi, void** recv_lo, void** recv_hi,
                                 int64_t* bytes, int64_t* plane_bytes, int32_t* margin);
/* Halo window: the exchanged x-planes carry only nodes y in [y0, y1), z in [z0, z1) (clamped
 * to the slab's storage).  Every slab must use the same window; it must cover every node a
 * particle stencil can reach until the next update (mpmb_dd_particle_window + the drift
 * margin).  plane_bytes of mpmb_dd_halo_buffers follows the window.  Default: whole planes. */
mpmb_status mpmb_dd_set_window(mpmb_state st, int32_t y0, int32_t y1, int32_t z0, int32_t z1);
/* Stencil reach of this slab's active particles: {min y node, max y node, min z node,
 * max z node} (INT_MAX / INT_MIN when there are none).  Synchronises the stream. */
mpmb_status mpmb_dd_particle_window(mpmb_state st, int32_t* out);
mpmb_status mpmb_dd_p2g(mpmb_state st, float dt);  /* bins if needed; MLS P2G */
mpmb_status mpmb_dd_pack_acc(mpmb_state st);
mpmb_status mpmb_dd_unpack_acc(mpmb_state st);
mpmb_status mpmb_dd_grid(mpmb_state st, float dt, const float gravity[3], int32_t contact, int32_t boundary);
mpmb_status mpmb_dd_pack_vel(mpmb_state st);
mpmb_status mpmb_dd_unpack_vel(mpmb_state st);
mpmb_status mpmb_dd_g2p(mpmb_state st, float dt, int32_t pushout, int32_t deactivate);
/* Migration: synchronous counts; buffers hold `capacity` particles of 112 bytes. */
/* Free bodies under DD (scene.hpp:220-232 split over slabs).  Each slab sums contact over the
 * nodes it owns; the per-substep sums live in device memory (impulse + torque impulse:
 * double[6 * n_shapes], node counts: int32[n_shapes]).  The caller all-reduces them (sum)
 * across slabs after mpmb_dd_grid, then calls mpmb_dd_free_bodies after mpmb_dd_g2p:
 * integrate_free_body (rigid_dynamics.hpp:82-103) on every slab with the same sums (so every
 * slab holds the same pose), then the sums merge into the frame sums and clear. */
mpmb_status mpmb_dd_contact_sums(mpmb_state st, void** sums, void** counts, int32_t* n_shapes);
mpmb_status mpmb_dd_free_bodies(mpmb_state st, float dt, const float gravity[3]);
mpmb_status mpmb_dd_migrate_pack(mpmb_state st, int64_t* n_to_lo, int64_t* n_to_hi);
mpmb_status mpmb_dd_migrate_buffers(mpmb_state st, void** send_lo, void** send_hi, void** recv_lo, void** recv_hi,
                                    int64_t* capacity);
mpmb_status mpmb_dd_migrate_unpack(mpmb_state st, int64_t n_from_lo, int64_t n_from_hi);
/* The slab's particles (any order): ids, x, v, active; n = how many (<= capacity). */
mpmb_status mpmb_dd_download(mpmb_state st, int64_t capacity, uint32_t* ids, float* x, float* v, uint8_t* active,
                             int64_t* n);

/* --------------------------------------------------------- facade layer */
typedef uint64_t mpmb_handle;
#define MPMB_INVALID_HANDLE ((mpmb_handle)0)

mpmb_handle mpmb_create_scene(const mpmb_scene_config* config);
/* Batched replicas: n scenes with one config advancing together.  Returns the batch handle
 * and writes n scene handles; per-scene calls (materials, objects, shapes, pose targets,
 * copy_positions, shape_impulse) take the scene handles, advance/fetch take the batch. */
mpmb_handle mpmb_create_scene_batch(const mpmb_scene_config* config, int32_t n,
                                    mpmb_handle* scenes_out);
mpmb_status mpmb_destroy(mpmb_handle h);
mpmb_handle mpmb_create_material(mpmb_handle scene, const mpmb_material* mat);
mpmb_handle mpmb_create_particle_object(mpmb_handle scene, mpmb_handle material,
                                        const float min_corner[3], const float max_corner[3],
                                        int32_t particles_per_cell, float density,
                                        uint64_t seed);
mpmb_handle mpmb_create_shape(mpmb_handle scene, const mpmb_shape_desc* shape);
mpmb_status mpmb_set_shape_pose_target(mpmb_handle scene, mpmb_handle shape,
                                       const float position[3], const float orientation[4]);
/* Enqueues one frame (asynchronous; the paper's advance/fetch split). Scene or batch handle. */
mpmb_status mpmb_advance(mpmb_handle h, float dt);
/* Pipelined form of n x (advance; fetch_results) with no snapshot between frames: all
 * frames are enqueued back to back; the last one is left pending for mpmb_fetch_results.
 * (Extension; the reference's advance is synchronous, scene.hpp:117-123.) */
mpmb_status mpmb_advance_frames(mpmb_handle h, float dt, int32_t n_frames);
/* Waits for the pending frame and snapshots FrameResult. For a batch, out has n entries.
 * Returns once the scalar part (FP64 totals, counters, contact sums) is on the host; the
 * original-order arrays are gathered and copied asynchronously (they stay valid while the
 * next frame is enqueued). */
mpmb_status mpmb_fetch_results(mpmb_handle h, mpmb_frame_summary* out);
/* Arrays of the last fetched FrameResult of one scene (any pointer may be NULL):
 * positions/velocities 3n floats, active n bytes, shape ids/impulses/torques per shape.
 * Waits for the asynchronous array copy of mpmb_fetch_results. */
mpmb_status mpmb_result_copy(mpmb_handle scene, float* positions, float* velocities,
                             uint8_t* active, int32_t* shape_ids, float* shape_impulses,
                             float* shape_torque_impulses);
/* Zero-copy FrameResult arrays (extension): the caller's own arrays become the destination of
 * every later fetch_results' device->host copy (page-locked in place with cudaHostRegister, so
 * the DMA lands in them directly; no staging buffer, no host memcpy).  h = scene or batch
 * handle; for a batch the arrays cover every scene in batch order (positions/velocities 3n
 * floats, active n bytes, n = total particle count).  A fetch overwrites them; they hold the
 * newest fetched frame once mpmb_result_wait (or mpmb_result_copy) returns.  All-NULL unbinds
 * (also done by mpmb_destroy).  The reference's FrameResult owns its vectors
 * (scene.hpp:251-258); a caller that keeps one FrameResult object per scene binds its vectors. */
mpmb_status mpmb_bind_results(mpmb_handle h, float* positions, float* velocities, uint8_t* active,
                              int64_t n);
/* Waits for the array copy of the last mpmb_fetch_results (bound or internal buffer). */
mpmb_status mpmb_result_wait(mpmb_handle h);
int32_t mpmb_particle_count(mpmb_handle scene);
mpmb_status mpmb_copy_positions(mpmb_handle scene, float* out, size_t capacity_floats,
                                size_t* written_floats);
mpmb_status mpmb_shape_impulse(mpmb_handle scene, mpmb_handle shape, float out[3]);
/* Synchronous ParticleStore read-back of a scene in original order (any pointer NULL). */
mpmb_status mpmb_scene_get_particles(mpmb_handle scene, float* x, float* v, float* F, float* C,
                                     uint8_t* active);

/* Execution control: run on the caller's cudaStream_t (NULL = library stream), re-bin every
 * k substeps (0 = every 4 frames; binning only re-compacts the transfer groups, P2G re-sorts
 * each group every substep), profile kernel classes with CUDA events. */
mpmb_status mpmb_set_stream(mpmb_handle h, void* cuda_stream);
mpmb_status mpmb_set_resort_interval(mpmb_handle h, int32_t substeps);
mpmb_status mpmb_set_profiling(mpmb_handle h, int32_t on);
/* Exact mode (MLS): every substep in the reference's float arithmetic and summation order --
 * bit-identical to the reference and run to run (SPEC.md:252 deterministic mode), several
 * times slower than the default fast mode (float atomics). */
mpmb_status mpmb_set_exact(mpmb_handle h, int32_t on);
/* Substep fusion inside run_frame (Scene::run_frame, scene.hpp:199-235, MLS / standard):
 * G2P of substep s and P2G of s+1 run as one kernel.  0 off; 1 (default) and 2 on (2 was
 * "always" when 1 excluded small problems).  Results are the same up to float atomic order
 * either way. */
mpmb_status mpmb_set_fusion(mpmb_handle h, int32_t mode);
mpmb_status mpmb_get_profile(mpmb_handle h, mpmb_profile* out);
/* Blocks until every frame enqueued on h has finished. */
mpmb_status mpmb_synchronize(mpmb_handle h);

/* --------------------------------------------------- slab DD driver (device-resident)
 * The whole substep loop of a slab domain decomposition in the library (dd_driver.h):
 * P2G (fused with the previous G2P where no migration intervenes), ghost-sum exchange,
 * grid update + contact, [contact-sum all-reduce for free bodies, scene.hpp:220-232],
 * velocity exchange, G2P, free bodies, migration every `migrate_every` substeps (0: the
 * margin) -- with no host synchronisation inside a run: migration counts travel device to
 * device beside fixed-capacity payloads, the halo y/z window is set once per run from the
 * particles' reach + one cell per substep and checked on the device.  Each run reads the
 * window and error flags snapshot the run before last left in pinned memory (no stream
 * drain after the first two runs; mpmb_dd_get_stats counts), and fails with the reason if a
 * check tripped.
 *   local: the slabs of this process, ordered along x, on one device (device copies);
 *   NCCL:  one slab per process; the communicator from mpmb_nccl_get_unique_id (on one
 *          rank, shared by the caller) or the caller's own ncclComm_t.  NCCL is loaded at
 *          run time (libnccl.so.2). */
typedef struct mpmb_dd_group_s* mpmb_dd_group;
/* host_syncs: snapshot reads that drained the stream (the first two runs of a group);
 * host_waits: later reads that found the device more than one run behind the host. */
typedef struct {
    int64_t runs, substeps, host_syncs, host_waits, exchanges, fused, rebins;
} mpmb_dd_stats;
mpmb_status mpmb_dd_group_create_local(const mpmb_state* slabs, int32_t n, mpmb_dd_group* out);
mpmb_status mpmb_nccl_get_unique_id(uint8_t id[128]);
mpmb_status mpmb_dd_group_create_nccl(mpmb_state slab, const uint8_t id[128], int32_t nranks, int32_t rank,
                                      mpmb_dd_group* out);
mpmb_status mpmb_dd_group_create_comm(mpmb_state slab, void* nccl_comm, int32_t nranks, int32_t rank,
                                      mpmb_dd_group* out);
mpmb_status mpmb_dd_group_destroy(mpmb_dd_group g);
mpmb_status mpmb_dd_run(mpmb_dd_group g, int32_t n_sub, float dt, const float gravity[3], int32_t contact,
                        int32_t boundary, int32_t pushout, int32_t deactivate, int32_t free_bodies,
                        int32_t migrate_every, int32_t fuse);
mpmb_status mpmb_dd_get_stats(mpmb_dd_group g, mpmb_dd_stats* out);
/* Waits for the group's queued work; MPMB_CUDA_ERROR with the reason if a device check
 * (migration overflow, capacity, stencil reach, particle leaving the grid) tripped. */
mpmb_status mpmb_dd_check(mpmb_dd_group g);

/* --------------------------------------------------- scenario metrics (device)
 * The harness metrics of run_scenario (scenario.hpp:68-139) on the resident particles: a
 * batch handle addresses every scene (arrays of one entry per scene), a scene handle its
 * own.  No frame may be pending.  Both reproduce the reference's spatial hash, probes and
 * float arithmetic, so counts and spacings equal the reference's on identical positions.
 *   components: compute_components with link radius radius[k] (components holding >= 5%
 *               of the active particles);
 *   nn_spacing: mean_nearest_neighbor_spacing with cell hint cell_hint[k]. */
mpmb_status mpmb_components(mpmb_handle h, const float* radius, int32_t* count);
mpmb_status mpmb_nn_spacing(mpmb_handle h, const float* cell_hint, float* spacing);

#ifdef __cplusplus
}
#endif
#endif /* MPM_B200_H */
