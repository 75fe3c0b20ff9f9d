// engine.h — device engine of the B200 MPM hot path (host-side interface).
//
// One Engine holds a BATCH of independent scenes (1 for a plain Scene / SimState)
// resident in HBM and advances all of them with one launch per kernel:
//   particles  : 7 float4 planes per particle slot (112 B), sorted by (brick, cell) at
//                binning; P2G re-sorts each 256-slot group every substep
//   grid       : per-scene dense virtual grid in 4x4x4-node bricks (float4 nodes),
//                only bricks touched by P2G are updated/cleared
//   shapes     : flattened shape table + per-substep pose table + free-body poses
// Every public method enqueues on the engine's stream; only the explicit download /
// read_* methods synchronise.
#pragma once
#include <memory>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/mpm_b200.h"
#include "dev_types.h"

namespace mpmb {

struct SceneGrid {
    int dims[3];
    float dx;
    float origin[3];
    // slab domain: this engine owns global x nodes [slab_lo, slab_hi) and
    // stores [slab_lo - margin, slab_hi + 2 + margin); slab_hi <= slab_lo: the whole grid
    int slab_lo = 0, slab_hi = 0, margin = 0;
};

struct EngineShape {            // host copy of one shape (per scene, in order)
    DevShape d;
    DevPose pose;               // current pose (kinematic / fixed / initial free)
    std::vector<float> verts;   // local-frame vertices (3 floats each)
    std::vector<int> indices;
    std::vector<int> spine;
};

struct SceneCounters {          // per scene, summed since reset_counters()
    int32_t inverted_f;
    int32_t projection_failures;
    int32_t pushed_out;
    int32_t deactivated;
};

struct KernelTimes {
    double ms_sort = 0, ms_p2g = 0, ms_grid = 0, ms_g2p = 0, ms_other = 0;
    double ms_fused = 0;  // k_g2p2g (G2P of substep s + P2G of s+1) + its brick collect
    int64_t launches = 0;
    int64_t n_sort = 0, n_p2g = 0, n_grid = 0, n_g2p = 0, n_fused = 0;  // timed operations
};

class Engine {
  public:
    explicit Engine(const std::vector<SceneGrid>& scenes);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    int n_scenes() const { return static_cast<int>(scenes_.size()); }
    int64_t n_particles() const { return n_total_; }
    const SceneGrid& grid(int s) const { return scenes_[s]; }

    void set_stream(void* stream);
    void* stream() const { return stream_; }
    void set_profiling(bool on);
    KernelTimes kernel_times() const;
    void reset_kernel_times();

    // Global material table (deduplicated across scenes by the caller).
    void set_materials(const std::vector<mpmb_material>& mats);
    // Particles in ORIGINAL order (scene ranges concatenated); stress may be null.
    void upload_particles(int64_t n, const float* x, const float* v, const float* mass,
                          const float* vol0, const float* F, const float* C, const float* stress,
                          const int32_t* material, const uint8_t* active, const int32_t* scene,
                          const uint32_t* ids = nullptr);
    // Synchronous download in original order (null pointers skipped).
    void download_particles(int64_t begin, int64_t count, float* x, float* v, float* mass,
                            float* vol0, float* F, float* C, float* stress, int32_t* material,
                            uint8_t* active);
    // Shapes of all scenes: shapes[s] in order.  Resets free-body poses and accumulators.
    void set_shapes(const std::vector<std::vector<EngineShape>>& shapes);
    int n_shapes() const { return n_shapes_; }
    // Pose table for the next frame: poses[sub * n_shapes + i], override mask
    // (1 = use the table pose even for a free body).  Copied asynchronously.
    void set_pose_table(int n_sub, const std::vector<DevPose>& poses,
                        const std::vector<uint8_t>& override_mask);
    // Overwrite the device pose of free-body shape i (pose-target consumption).
    void set_free_pose(int shape, const DevPose& pose);
    std::vector<DevPose> read_free_poses();

    // ---- hot path (enqueue only) ----
    void bin();                                   // K1: keys, stable sort, gather
    // K2 / K5 (+ active-brick list); standard: the standard-MPM force transfer (mls = true)
    void p2g(bool mls, float dt, bool collect = true, bool standard = false);
    void collect_bricks();
    void grid_update(int sub, float dt, const float g[3], bool gravity, bool contact, int bc);
    void g2p_mls(int sub, float dt, bool pushout, bool deactivate);   // K4
    void g2p_standard(int sub, float dt, bool pushout, bool deactivate);  // K4, PIC (solvers.hpp:107-135)
    // K4 of substep `sub` fused with K2 of sub+1 (MLS or standard; push-out and deactivation
    // on), followed by the brick collect of sub+1: replaces g2p_* then p2g inside a frame
    // With shapes, the free bodies of `sub` (free_bodies(sub, dt, g, integrate, true, sub+1))
    // run in the collect launch; the caller then skips free_bodies.
    void g2p2g(int sub, float dt, bool standard, const float g[3], bool integrate, bool collect = true,
               bool pushout = true, bool deactivate = true);
    // fusion policy: 0 off, 1 (default) or 2 on
    // PB-MPM: G2P of a non-final iteration (no commit) + P2G of the next iteration, then the
    // brick collect (replaces g2p_pb(.., false, false, false) then p2g(false, ..))
    void g2p2g_pb(float dt);
    void set_fusion(int mode);
    // per-substep contact sums (device): double[6 * n_shapes], int32[n_shapes]
    void contact_sub_buffers(void** sums, void** counts, int* n_shapes);
    bool fuse_ok() const;
    // exact mode (k_exact.cu): MLS substeps in the reference's float order and arithmetic,
    // bit-identical to the reference and run to run; much slower than the default fast mode
    void set_exact(bool on);
    bool exact() const;
    void g2p_pb(int sub, float dt, bool commit, bool pushout, bool deactivate);  // K6
    // cull_next >= 0: also build that substep's shape cull table (saves its k_shape_cull)
    void free_bodies(int sub, float dt, const float g[3], bool integrate, bool merge, int cull_next = -1);  // K7
    void bc_pass(int bc);                         // BC alone (hook adapter)
    void materialize_stress();                    // sigma(F) -> cached stress array
    void pushout(int sub);
    void deactivate();

    // ---- results ----
    void reset_counters();
    void reset_contact(bool frame, bool sub);
    std::vector<SceneCounters> read_counters();
    // fetch's small results in one round trip: stage_small() enqueues the counters and the
    // frame's contact sums into pinned memory; after the next stream sync (snapshot) read them
    // with small_results()
    void stage_small();
    void small_results(std::vector<SceneCounters>& counters, std::vector<double>& impulse,
                       std::vector<double>& torque, std::vector<int32_t>& count);
    // contact accumulators (per shape, double): which = 0 substep, 1 frame
    void read_contact(int which, std::vector<double>& impulse, std::vector<double>& torque,
                      std::vector<int32_t>& count);
    // FrameResult snapshot for all scenes: positions/velocities/active in original order
    // (device -> pinned host), totals per scene (double).  Enqueue + wait.
    // Frame snapshot: totals are ready on return.  async: the x / v / active D2H runs on a
    // copy stream and overlaps whatever the caller enqueues next (the next frame); the host
    // arrays are valid after wait_results().  The next snapshot reuses the device staging
    // only after that copy (stream wait, no host sync).
    void snapshot(float* x, float* v, uint8_t* active, std::vector<double>& totals /*5 per scene*/,
                  bool async = false);
    void wait_results();
    // The next standalone G2P (the frame's last) exports the frame result as it writes the
    // state: x / v / active in original order into the snapshot staging and the per-scene
    // totals; the next async snapshot then only copies them (no gather, no totals pass).
    void request_export();
    // page-locked host memory (cudaMallocHost) freed with the last reference: D2H of a
    // FrameResult straight into it runs at link speed, with no staging copies
    static std::shared_ptr<void> pinned_host(size_t bytes);
    // page-lock caller memory in place (cudaHostRegister) / release it
    static void host_register(void* p, size_t bytes);
    static void host_unregister(void* p);
    // the P2G stress function (neo_hookean_f32) on n host matrices, synchronously (KATs)
    static void eval_stress_f32(const float* F, int64_t n, float mu, float lambda, float* sigma, float* J);
    // dense grid of one scene (node-major i + nx*(j + ny*k)); for tests and the hook adapter
    void download_grid(int scene, float* mass, float* momentum, float* velocity);
    // keep the momentum of nodes below kMassEps for download_grid (one more float4 per node;
    // the batched hot path leaves it off)
    void enable_grid_readback();
    void upload_grid_velocity(int scene, const float* mass, const float* momentum,
                              const float* velocity);
    // keys/perm of the binning stage (original indices), see mpmb_bin_particles
    void read_binning(uint32_t* keys, uint32_t* perm);

    // ---- scenario metrics (k_scenario.cu; scenario.hpp:68-139), synchronous ----
    // components per scene with link radius radius[scene] (>= 5% of the active particles)
    void components(const float* radius, int32_t* counts);
    // squared nearest-neighbour distance per particle in original order (FLT_MAX = none),
    // probing with cell size cell[scene]
    void nn_best2(const float* cell, float* best2);

    // ---- slab domain decomposition (k_dd.cu) ----
    // Slots for particles that may arrive by migration; call before upload_particles.
    void set_capacity(int64_t particles);
    // Device halo buffers (each `bytes`): send/recv towards the lower / upper neighbour.
    void dd_halo_buffers(void** send_lo, void** send_hi, void** recv_lo, void** recv_hi, int64_t* bytes);
    void dd_pack_acc();     // after P2G: ghost sums -> send_lo (M planes), send_hi (2+M planes)
    void dd_unpack_acc();   // add recv_hi (M planes) / recv_lo (2+M planes) into owned planes
    void dd_pack_vel();     // after the grid update: owned boundary velocities -> send_lo / send_hi
    void dd_unpack_vel();   // recv_lo -> low ghosts (M planes), recv_hi -> high ghosts (2+M)
    int dd_halo_planes(int side_send_hi, bool acc) const;
    void ensure_halo();
    // halo planes restricted to nodes y in [y0, y1), z in [z0, z1) (clamped to the storage)
    void dd_set_window(int y0, int y1, int z0, int z1);
    void dd_plane_window(int* y0, int* ny, int* z0, int* nz);
    // {min, max} stencil node reach of the active particles in y and z (synchronises)
    void particle_window(int out[4]);
    // Migration (synchronous): particles whose base left the slab are packed for the
    // neighbours; returns their counts.  Buffers hold `cap` particles of 7 float4 each.
    void dd_migrate_pack(int64_t* n_lo, int64_t* n_hi);
    void dd_migrate_buffers(void** send_lo, void** send_hi, void** recv_lo, void** recv_hi, int64_t* cap);
    void dd_migrate_unpack(int64_t n_from_lo, int64_t n_from_hi);  // appends, then bins
    // The particles (any order): original index, x, v, active; returns how many (<= capacity).
    int64_t slot_count() const;

    // ---- device-resident slab DD (dd_driver.cpp): nothing per substep waits for the host.
    // Migration counts travel device to device (fixed-capacity payloads, in-band counts),
    // arrivals are appended as extra groups by a device kernel, and errors (overflow, a
    // stencil that outran the stored planes / halo window, a particle leaving the grid) are
    // flags the driver reads once per run with the window (dd_control).
    struct DDControl {
        int window[4];  // {min base y, max base y + 2, min base z, max base z + 2}
        uint32_t group_err;  // error flags of every rank (the all-reduced window buffer's [4])
        uint32_t free_slot, arrivals, err, n_real;
    };
    void dd_window_async();                // recompute the device window (after a run)
    int* dd_window_device();               // its 8 ints {window, err, -}: the all-reduce operand
    uint32_t* dd_control_device();         // the 4 DD control words
    DDControl dd_control();                // window + control words: one D2H and a sync
    // pipelined form: the window and control words copied D2H into pinned slot `slot` behind
    // an event; read later (normally complete by then: no wait).  blocked = the read waited.
    void dd_snapshot_async(int slot);
    DDControl dd_snapshot_read(int slot, bool* blocked);
    void dd_clear_errors();
    // the migration payload capacity (particles per side; the same on every slab)
    void dd_set_migration_capacity(int64_t cap);
    // send/recv payloads (cap x 7 float4 each) and counts {sent down, up, recv below, above}
    void dd_migration_buffers(void** send_lo, void** send_hi, void** recv_lo, void** recv_hi,
                              uint32_t** counts, int64_t* cap);
    void dd_migrate_pack_async(bool has_lo, bool has_hi);
    void dd_migrate_unpack_async();
    void dd_note_count(int64_t n_real);    // the host's particle count, from dd_control
    // brick collect of substep next_sub deferred past the ghost-sum exchange (after
    // g2p2g(..., collect = false)), with the free bodies of next_sub - 1 when integrate
    void collect_deferred(int next_sub, float dt, const float g[3], bool integrate);
    int64_t download_compact(int64_t capacity, uint32_t* ids, float* x, float* v, uint8_t* active);
    int64_t n_active_sorted();

    void synchronize();  // the engine stream and any snapshot copy in flight
    int64_t launches() const { return launches_total_; }

  private:
    struct Impl;
    Impl* impl_;
    bool prepare_export(struct Params& P);  // request_export: staging + totals into P
    std::vector<SceneGrid> scenes_;
    int64_t n_total_ = 0;
    int n_shapes_ = 0;
    void* stream_ = nullptr;
    int64_t launches_total_ = 0;
};

// Process-wide launch counter (all engines).
int64_t global_launch_count();
bool device_available();

}  // namespace mpmb
