// launch.h — host launchers of the kernels (one translation unit per kernel family).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace mpmb {

// ---- K1 binning (k_sort.cu) ----
struct BinBuffers {
    uint32_t n_buckets;        // bricks of all scenes + 1 (inactive bucket last)
    uint32_t* bucket_count;    // [n_buckets]
    uint32_t* bucket_off;      // [n_buckets + 1]
    uint32_t* key;             // per slot: bucket
    uint32_t* rank;            // per slot: rank inside bucket (atomic order)
    uint8_t* cell;             // per slot: cell inside brick (6 bits)
    uint32_t* orig;            // per slot: original index
    uint32_t* e_orig;          // bucketed entries
    uint8_t* e_cell;
    uint32_t* e_src;
    uint32_t* tmp;             // scratch (per slot)
    uint32_t* g_orig;          // grouped by cell
    uint32_t* g_src;
    uint8_t* g_cell;
    uint32_t* sorted_src;      // final sorted position -> old slot
    uint32_t* sorted_orig;     // final sorted position -> original index
    uint32_t* counts;          // [0] n_active, [1] transfer groups, [2] n_active
    uint32_t* scan_tmp;        // block sums for the scans
    uint32_t* key_by_orig;     // optional (binning readback), may be null
};

void launch_bin(const Params& P, const BinBuffers& B, float4* const new_planes[kPlanes],
                int64_t n_total, cudaStream_t st, int64_t* launches);
void launch_exclusive_scan(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* tmp,
                           cudaStream_t st, int64_t* launches);

// ---- K2..K7 (k_transfer.cu, k_step.cu); max_groups = ceil(n / kGroup) ----
void launch_p2g(const Params& P, bool mls, int64_t max_groups, cudaStream_t st, bool standard = false);
// wide: one thread per slot (k_g2p_wide) for problems too small to fill the GPU with one warp
// per group
void launch_grid_update(const Params& P, int64_t max_bricks, cudaStream_t st);
void launch_shape_cull(const Params& P, cudaStream_t st);
void launch_g2p(const Params& P, bool pb, int64_t max_groups, cudaStream_t st, bool standard = false,
                bool wide = false);
// fused G2P (substep s) + P2G (substep s+1), MLS or standard MPM (k_g2p2g)
// pb: PB-MPM iteration it (G2P, no commit) + iteration it+1 (P2G)
void launch_g2p2g(const Params& P, int64_t max_groups, cudaStream_t st, bool standard = false, bool pb = false);
void launch_collect_bricks(const Params& P, uint32_t n_bricks, cudaStream_t st);
void launch_pushout(const Params& P, cudaStream_t st);
void launch_deactivate(const Params& P, cudaStream_t st);
// k_collect_free: the brick collect of the next substep + the free bodies, one launch
void launch_collect_free(const Params& P, uint32_t n_bricks, bool integrate, bool merge, int next_sub,
                         cudaStream_t st);
void launch_free_bodies(const Params& P, bool integrate, bool merge, cudaStream_t st, int next_sub = -1);
void launch_grid_bc(const Params& P, int64_t max_bricks, cudaStream_t st);

// ---- slab domain decomposition (k_dd.cu) ----
int64_t dd_plane_nodes(const Params& P);
void launch_halo(const Params& P, int mode, float4* pool, float4* buf, int x0, int w, int y0, int ny, int z0, int nz,
                 cudaStream_t st);
void launch_particle_window(const Params& P, int* out /*{ylo, yhi, zlo, zhi}*/, cudaStream_t st);
void launch_migrate_pack(const Params& P, int lo, int hi, float4* out_lo, float4* out_hi, uint32_t cap,
                         uint32_t* counts, cudaStream_t st);
void launch_migrate_unpack(const Params& P, const float4* in, uint32_t n, uint32_t first, cudaStream_t st);
void launch_download_slots(const Params& P, uint32_t* ids, float* x, float* v, uint8_t* active, uint32_t* count,
                           cudaStream_t st);
// device-resident migration (dd_driver.cpp).  DD control words = b_counts[4..7]:
// [4] free slot past the groups and the inactive tail, [5] arrivals since binning,
// [6] error flags, [7] particles on the slab (set at binning, kept by the migrations).
constexpr uint32_t kDdErrMigrationOverflow = 1u;  // more departures than the buffer capacity
constexpr uint32_t kDdErrCapacity = 2u;           // arrivals beyond the slab's slots
constexpr uint32_t kDdErrReach = 4u;              // a stencil left the stored planes / halo window
constexpr uint32_t kDdErrLeftDomain = 8u;         // a particle left the decomposed grid
void launch_window_init(int* w, cudaStream_t st);
void launch_migrate_pack_dev(const Params& P, int lo, int hi, int margin, int4 win, bool has_lo, bool has_hi,
                             float4* out_lo, float4* out_hi, uint32_t cap, uint32_t* counts, uint32_t* ctl,
                             cudaStream_t st);
void launch_migrate_unpack_dev(const Params& P, const float4* in_lo, const float4* in_hi, uint32_t cap,
                               const uint32_t* counts, uint32_t* bcounts, uint64_t n_cap, cudaStream_t st);

// ---- exact mode (k_exact.cu) ----
size_t exact_scratch_bytes(int64_t n, int64_t n_bricks);
void launch_exact_p2g(const Params& P, bool mls, void* scratch, uint2* brick_idx, uint32_t epoch, int64_t n_bricks,
                      cudaStream_t st);
void launch_exact_g2p(const Params& P, cudaStream_t st);
size_t exact_contact_scratch_bytes(uint32_t n);
void launch_exact_contact(const Params& P, uint32_t n, void* scratch, cudaStream_t st);

// ---- scenario metrics (k_scenario.cu) ----
size_t scenario_scratch_bytes(int64_t n, int n_scenes);
void launch_scenario(const Params& P, int mode, const float* cell, void* scratch, size_t scratch_bytes,
                     int32_t* count, float* best2, uint32_t* orig, int n_scenes, cudaStream_t st);

// ---- I/O (k_io.cu) ----
struct IoArrays {  // original-order device staging arrays (any may be null)
    float* x; float* v; float* mass; float* vol0; float* F; float* C; int32_t* mat;
    uint8_t* active; int32_t* scene;
    uint32_t* ids;  // upload: original index per particle (null: the upload order)
    int keep_stress;  // upload: a stress array accompanies the particles (kKeepStressBit)
};
void launch_upload(const Params& P, const IoArrays& in, int64_t n, cudaStream_t st);
void launch_download(const Params& P, const IoArrays& out, cudaStream_t st);
void launch_totals(const Params& P, double* totals /*5 per scene*/, cudaStream_t st);
// x / v / active (original order) + the totals through the inverse permutation (inv: n words)
void launch_export_pack(const float4* pad, int64_t n, float* x, float* v, uint8_t* a, cudaStream_t st);
void launch_frame_result_orig(const Params& P, uint32_t* inv, int64_t n, const IoArrays& out, double* totals,
                              cudaStream_t st);
void launch_stress(const Params& P, float* stress_orig, cudaStream_t st);
// synchronous: the P2G stress function (neo_hookean_f32) on n host matrices, for KATs
void eval_stress_f32(const float* F, int64_t n, float mu, float lambda, float* sigma, float* J);
void launch_grid_download(const Params& P, int scene, const DevScene& S, float* mass, float* mom,
                          float* vel, cudaStream_t st);
void launch_grid_upload(const Params& P, int scene, const DevScene& S, const float* mass,
                        const float* mom, const float* vel, cudaStream_t st);

}  // namespace mpmb
