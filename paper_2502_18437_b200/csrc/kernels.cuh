// kernels.cuh — sm_100a kernels of the MPM hot path.  See DESIGN.md §3 for the data
// layout and the roofline of each kernel.
//
//   K1 k_bin_*         binning / stable sort by (brick, cell, original index) (NEW stage;
//                      keys from math.hpp:219-223); P2G re-sorts each group every substep
//   K2 k_p2g<true>     MLS P2G with the stress impulse (solvers.hpp:151-169)
//   K5 k_p2g<false>    PB-MPM P2G (solvers.hpp:218-235)
//   K3 k_grid_update   v = p/m (+g dt), contact pass over the scene's shapes in order,
//                      per-shape impulse/torque reduction, BC (solvers.hpp:54-65, 30-50;
//                      contact.hpp:97-136)
//   K4 k_g2p_mls       G2P + F update (+ push-out, deactivation) (solvers.hpp:173-196,
//                      contact.hpp:140-179, state.hpp:153-164)
//   K6 k_g2p_pb        PB-MPM G2P + co-rotational projection (+ commit) (solvers.hpp:240-277)
//   K7 k_free_bodies   free-body integration + accumulator merge (rigid_dynamics.hpp:82-103,
//                      scene.hpp:220-232)
#pragma once
#include <atomic>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

#include "dev_math.cuh"

namespace mpmb {

// slots per transfer group: one warp re-sorts and processes one group per substep
constexpr int kGroup = 256;
constexpr int64_t kWideMaxSlots = 600000;  // engine: thread-per-slot G2P at or below this (A/B)
// Inside a group the particle of sorted position p lives at slot phys(p): lane L's k-th
// particle of P2G (p = 8L + k) sits at 32k + L, so a stable order makes every P2G staging
// load one contiguous 512-byte span, and G2P (p = L + 32k) touches 8 runs of 64 bytes.
__host__ __device__ __forceinline__ uint32_t group_phys(uint32_t p) { return (p & 7u) * 32u + (p >> 3); }
__host__ __device__ __forceinline__ uint32_t group_pos(uint32_t r) { return (r & 31u) * 8u + (r >> 5); }
// original index of an empty slot (group padding / allocation tail): never active, never
// downloaded
constexpr uint32_t kHoleOrig = 0xFFFFFFFFu;

// Particle slot = 7 float4 planes (112 B):
//   P0 {x.x, x.y, x.z, v.x}   P1 {v.y, v.z, C0, C1}   P2 {C2, C3, C4, C5}
//   P3 {C6, C7, C8, F0}       P4 {F1, F2, F3, F4}     P5 {F5, F6, F7, F8}
//   PR {mass, volume0, flags(u32), original index(u32)}
constexpr int kPlanes = 7;
constexpr int PR = 6;

struct Params {
    float4* pl[kPlanes];      // current particle planes (n_total slots)
    float4* pl_out[kPlanes];  // the other buffer: G2P writes the group-sorted state there
    Geo geo;                             // uniform geometry of all scenes
    float4 mats_c[kMaxConstMats];        // {kind, mu, lambda, beta}, first kMaxConstMats materials
    const DevScene* scenes;              // per scene: shape range (and host bookkeeping)
    const DevShape* shapes;
    const float* verts;
    const int* ints;
    const DevPose* pose_table;
    const uint8_t* pose_override;
    DevPose* free_pose;
    float4* cull;   // per shape, this substep: world AABB {min, bounded}, {max, 0} (k_shape_cull)
    DevPose* pose_eff;  // per shape, this substep: pose_of_sub() copied by the cull pass (one load)
    int n_shapes;
    int shapes_per_scene;  // > 0: scene s owns shapes [s k, s k + k) (batches of replicas); else 0
    const float4* mats;  // {kind, mu, lambda, beta}
    float4* grid_acc;
    float4* grid_vel;   // {v, m}; v = 0 at nodes of mass <= kMassEps
    float4* dead_mom;   // optional: {momentum, m} of nodes of mass <= kMassEps (grid readback)
    uint32_t* brick_flag;       // P2G marks of this substep (mark_bricks)
    uint32_t* brick_flag_next;  // the other array: zeroed by k_collect_bricks for the next P2G
    uint32_t* brick_stamp;
    uint32_t* active_bricks;
    uint2* active_info;  // per active brick: {bx | by << 10 | bz << 20, scene} (collect)
    uint32_t* n_active_bricks;
    const uint32_t* brick_scene;
    uint8_t* order;        // per group: kGroup bytes, slot-in-group by current stencil base
    uint32_t* group_nact;  // per group: active particles (written by P2G, replayed by G2P)
    int4* group_box;       // per group: stencil-base box {x0 | x1 << 16, y.., z.., scene or -1} (P2G sort)
    const uint32_t* n_groups;
    const uint32_t* n_active;
    int64_t n_total;          // slots (particles + holes), a fixed bound
    uint64_t total_nodes;     // grid pool length (bounds checks, MPMB_DEVICE_CHECKS)
    uint32_t debug;           // timing experiments of variant builds only (k_transfer.cu)
    // frame-end export (Engine::request_export): the frame's last G2P writes {x, v.x}, {v.y, v.z,
    // active, 0} at 2 o, 2 o + 1 (original index o < exp_n) and adds the per-scene FP64
    // totals; nullptr: off
    float4* exp_pad;
    double* exp_tot;
    int64_t exp_n;
    const float* stress_in;  // original-order uploaded sigma (first MLS P2G only)
    int use_stress_in;
    double* acc_sub;   // per shape: impulse[3], torque[3]
    int* cnt_sub;      // per shape: contact node count
    double* acc_frame;
    int* cnt_frame;
    int* counters;     // per scene: inverted, proj failures, pushed, deactivated
    // exact mode: contact terms as records {key = shape << 40 | reference node index,
    // impulse[3], torque[3]} for the ordered float sums of contact.hpp:127-129 (k_exact.cu);
    // null in the default mode (FP64 atomics)
    uint64_t* ex_ckey;
    float* ex_crec;
    uint32_t* ex_cn;
    uint32_t ex_ccap;
    int exact;  // exact mode: frame accumulators merge in float (scene.hpp:228-231)
    uint32_t epoch;
    float dt;
    float zero;  // always 0: a multiplier the compiler cannot fold (P2G accumulator reset)
    float g[3];
    int sub;
    int gravity;
    int contact;
    int bc;
    int pushout;
    int deactivate;
    int commit;
};

// Debug build (-DMPMB_DEVICE_CHECKS=1, tools/device_checks.sh): bounds of every computed slot,
// node and shared-memory index on the hot path; a violation prints its site and traps, so the
// launch fails loudly.  compute-sanitizer is not available on the GPU pool; this is the
// substitute.  Compiled out otherwise.
#ifndef MPMB_DEVICE_CHECKS
#define MPMB_DEVICE_CHECKS 0
#endif
#if MPMB_DEVICE_CHECKS
#define MPMB_DCHECK(cond)                                                                          \
    do {                                                                                           \
        if (!(cond)) {                                                                             \
            printf("MPMB_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,       \
                   __LINE__, blockIdx.x, threadIdx.x);                                             \
            __trap();                                                                              \
        }                                                                                          \
    } while (0)
#else
#define MPMB_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

// Per-scene view of the uniform geometry: scene-dependent offsets are scene x stride.
struct SceneView {
    float origin[3];
    float dx, inv_dx, m_inv;
    int dims[3];   // global dims (BC, deactivation)
    int nb[3];     // storage bricks
    uint64_t node_base;
    uint32_t brick_base;
    int scene;
};

__device__ __forceinline__ SceneView scene_view(const Params& P, int scene) {
    SceneView s;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        s.origin[a] = P.geo.origin[a];
        s.dims[a] = P.geo.dims[a];
        s.nb[a] = P.geo.nb[a];
    }
    s.dx = P.geo.dx;
    s.inv_dx = P.geo.inv_dx;
    s.m_inv = P.geo.m_inv;
    s.node_base = static_cast<uint64_t>(scene) * P.geo.nodes_per_scene;
    s.brick_base = static_cast<uint32_t>(scene) * P.geo.bricks_per_scene;
    s.scene = scene;
    return s;
}

// Stencil base in LOCAL storage coordinates: the reference's global base (math.hpp:219-224,
// bit-exact, global origin) shifted by the slab offset in x and clamped to the storage
// (memory guard only); fx is the reference's fractional coordinate.
__device__ __forceinline__ void local_base(const Geo& G, const float x[3], int b[3], float fx[3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) b[a] = stencil_base(x[a], G.origin[a], G.inv_dx, fx[a]);
    b[0] = min(max(b[0] - G.goff, 0), G.lx - 3);
    b[1] = min(max(b[1], 0), G.dims[1] - 3);
    b[2] = min(max(b[2], 0), G.dims[2] - 3);
}
// world coordinate of LOCAL node index i along axis a (state.hpp:49-51 on the global index)
__device__ __forceinline__ float node_coord(const Geo& G, int a, int i) {
    return G.origin[a] + static_cast<float>(i + (a == 0 ? G.goff : 0)) * G.dx;
}

__device__ __forceinline__ float4 material(const Params& P, uint32_t id) {
    return id < kMaxConstMats ? P.mats_c[id] : P.mats[id];
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Active-brick list from the P2G marks (warp-aggregated append; order is irrelevant).
// Brick X is active when some X - d, d in {0,1}^3 (same scene), is marked with every bit of
// d set (mark_bricks).  The marks are read across neighbours, so they cannot be cleared
// here: the flag arrays alternate per substep and this pass zeroes the OTHER one, which
// the next P2G marks.  Blocks [0, nblk) of 256 threads stride over the bricks.
__device__ __forceinline__ void collect_bricks_body(const Params& P, uint32_t n_bricks, uint32_t blk,
                                                    uint32_t nblk) {
    const unsigned full = 0xffffffffu;
    const uint32_t stride = nblk * blockDim.x;
    const uint32_t nb0 = P.geo.nb[0], nb1 = P.geo.nb[1], bps = P.geo.bricks_per_scene;
    for (uint32_t base = blk * blockDim.x; base < n_bricks; base += stride) {
        const uint32_t b = base + threadIdx.x;
        bool on = false;
        if (b < n_bricks) {
            P.brick_flag_next[b] = 0u;
            // fast path: most bricks have no mark around them (raw neighbour loads, indices
            // clamped; a nonzero word only means "decode exactly")
            uint32_t fr[8];
#pragma unroll
            for (int d = 0; d < 8; ++d) {
                const uint32_t off = (d & 1) + ((d >> 1) & 1) * nb0 + (d >> 2) * nb0 * nb1;
                fr[d] = P.brick_flag[b >= off ? b - off : 0u];
            }
            uint32_t any = 0;
#pragma unroll
            for (int d = 0; d < 8; ++d) any |= fr[d];
            if (any) {
                const uint32_t local = b % bps;
                const uint32_t bx = local % nb0, by = (local / nb0) % nb1, bz = local / (nb0 * nb1);
#pragma unroll
                for (int d = 0; d < 8; ++d) {
                    const uint32_t dx = d & 1, dy = (d >> 1) & 1, dz = d >> 2;
                    if (bx < dx || by < dy || bz < dz) continue;
                    const uint32_t f = fr[d];
                    on = on || ((f & 8u) && (f & static_cast<uint32_t>(d)) == static_cast<uint32_t>(d));
                }
            }
        }
        const unsigned m = __ballot_sync(full, on);
        if (m == 0u) continue;
        uint32_t start = 0;
        if ((threadIdx.x & 31) == 0) start = atomicAdd(P.n_active_bricks, __popc(m));
        start = __shfl_sync(full, start, 0);
        if (on) {
            const uint32_t w = start + __popc(m & lanemask_lt());
            P.active_bricks[w] = b;
            const uint32_t local = b % bps;  // (only for the ~3% active bricks)
            P.active_info[w] = make_uint2((local % nb0) | (((local / nb0) % nb1) << 10) | ((local / (nb0 * nb1)) << 20),
                                          b / bps);
        }
    }
}

struct Part {
    float x[3], v[3], C[9], F[9];
};

__device__ __forceinline__ void load_part(const Params& P, uint32_t s, Part& p) {
    float4 a = P.pl[0][s], b = P.pl[1][s], c = P.pl[2][s], d = P.pl[3][s], e = P.pl[4][s],
           f = P.pl[5][s];
    p.x[0] = a.x; p.x[1] = a.y; p.x[2] = a.z; p.v[0] = a.w;
    p.v[1] = b.x; p.v[2] = b.y; p.C[0] = b.z; p.C[1] = b.w;
    p.C[2] = c.x; p.C[3] = c.y; p.C[4] = c.z; p.C[5] = c.w;
    p.C[6] = d.x; p.C[7] = d.y; p.C[8] = d.z; p.F[0] = d.w;
    p.F[1] = e.x; p.F[2] = e.y; p.F[3] = e.z; p.F[4] = e.w;
    p.F[5] = f.x; p.F[6] = f.y; p.F[7] = f.z; p.F[8] = f.w;
}

__device__ __forceinline__ void store_part(const Params& P, uint32_t s, const Part& p) {
    P.pl[0][s] = make_float4(p.x[0], p.x[1], p.x[2], p.v[0]);
    P.pl[1][s] = make_float4(p.v[1], p.v[2], p.C[0], p.C[1]);
    P.pl[2][s] = make_float4(p.C[2], p.C[3], p.C[4], p.C[5]);
    P.pl[3][s] = make_float4(p.C[6], p.C[7], p.C[8], p.F[0]);
    P.pl[4][s] = make_float4(p.F[1], p.F[2], p.F[3], p.F[4]);
    P.pl[5][s] = make_float4(p.F[5], p.F[6], p.F[7], p.F[8]);
}

__device__ __forceinline__ const DevPose& pose_of_sub(const Params& P, int i, int sub) {
    const int t = sub * P.n_shapes + i;
    return (P.shapes[i].motion == MOTION_FREE && !P.pose_override[t]) ? P.free_pose[i]
                                                                         : P.pose_table[t];
}
__device__ __forceinline__ const DevPose& pose_of(const Params& P, int i) {
    const int t = P.sub * P.n_shapes + i;
    return (P.shapes[i].motion == MOTION_FREE && !P.pose_override[t]) ? P.free_pose[i]
                                                                         : P.pose_table[t];
}

// Node pool of a scene: LINEAR over the brick-padded dims (PX = 4 nb_x, PY = 4 nb_y):
// node (i, j, k) = (k PY + j) PX + i.  Activity is tracked per 4x4x4 brick, but a
// stencil's 27 nodes are 9 rows of 3 consecutive nodes (row bases + immediate offsets).
__device__ __forceinline__ uint32_t node_linear(const Geo& G, int i, int j, int k) {
    const uint32_t px = static_cast<uint32_t>(G.nb[0]) * 4u, py = static_cast<uint32_t>(G.nb[1]) * 4u;
    return (static_cast<uint32_t>(k) * py + static_cast<uint32_t>(j)) * px + static_cast<uint32_t>(i);
}
// row (dk, dj) of the stencil at base b starts at node_linear(b) + dk PXY + dj PX
__device__ __forceinline__ void stencil_rows(const Geo& G, const int b[3], uint32_t& base, uint32_t& px,
                                             uint32_t& pxy) {
    px = static_cast<uint32_t>(G.nb[0]) * 4u;
    pxy = px * static_cast<uint32_t>(G.nb[1]) * 4u;
    base = node_linear(G, b[0], b[1], b[2]);
}

// Cheap reject before an SDF query: false when x is provably outside every band of shape
// si at this substep (the world AABB of DevShape::lbox; unbounded shapes never cull).
__device__ __forceinline__ bool aabb_may_touch(float4 lo, float4 hi, float x, float y, float z) {
    return lo.w < 0.f || (x >= lo.x && x <= hi.x && y >= lo.y && y <= hi.y && z >= lo.z && z <= hi.z);
}
__device__ __forceinline__ bool cull_may_touch(const Params& P, int si, float x, float y, float z) {
    return aabb_may_touch(P.cull[2 * si], P.cull[2 * si + 1], x, y, z);
}

// Warp-aggregated per-scene counter add; must be called by all 32 lanes.  Lanes of a
// warp almost always share one scene: one atomic per warp, per-lane atomics otherwise.
__device__ __forceinline__ void add_scene_counter(int* counters, int scene, int slot, int value) {
    const unsigned full = 0xffffffffu;
    const unsigned has = __ballot_sync(full, value != 0);
    if (has == 0) return;
    const int lead = __ffs(has) - 1;
    const int s0 = __shfl_sync(full, scene, lead);
    const bool uniform = __all_sync(full, value == 0 || scene == s0);
    if (uniform) {
        const int total = __reduce_add_sync(full, value);
        if ((threadIdx.x & 31) == lead) atomicAdd(&counters[4 * s0 + slot], total);
    } else if (value != 0) {
        atomicAdd(&counters[4 * scene + slot], value);
    }
}

// ---- launch errors ----------------------------------------------------------------------
// A launch-configuration error (grid / block / shared-memory size, a missing opt-in) does not
// stick: the next stream synchronise still succeeds and the kernel silently never ran.  Every
// launch is therefore checked at once (no sync), and the error travels to the C-ABI status.
inline void launch_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();  // consume it: the error is reported by the exception
        throw std::runtime_error(std::string("kernel launch failed (") + what + "): " + cudaGetErrorString(e));
    }
}
#define MPMB_LAUNCHED(what) ::mpmb::launch_check(cudaGetLastError(), what)

// >48 KB dynamic shared memory is an opt-in per kernel AND per device; it is cheap, so the
// launchers keep one bit per device (64 devices) instead of a process-wide flag.
// The bit is set only after every opt-in succeeded; a racing thread repeats them (harmless).
template <class F>
inline void smem_opt_in_once(std::atomic<uint64_t>& done, F&& opt_in) {
    int dev = 0;
    launch_check(cudaGetDevice(&dev), "cudaGetDevice");
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    opt_in();
    done.fetch_or(bit, std::memory_order_release);
}
template <class K>
inline void opt_in_smem(K kernel, int bytes) {
    if (bytes > 48 * 1024)
        launch_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                     "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
}

// ---- programmatic dependent launch (PDL) for the per-substep kernel chain -------------
// A chain kernel is launched with programmatic stream serialisation: its grid may start while
// the previous kernel's last blocks drain, and waits at entry (griddepcontrol.wait) until that
// kernel has completed and its writes are visible.  Waiting first thing keeps every RAW / WAR
// order of the plain stream; what overlaps is the launch latency and block rasterisation.
// Launched without the attribute (MPMB_PDL=0) both instructions are no-ops.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("MPMB_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}
template <typename... Exp, typename... Act>
inline void launch_chain(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                         Act&&... args) {
    cudaLaunchConfig_t c{};
    c.gridDim = grid;
    c.blockDim = block;
    c.dynamicSmemBytes = smem;
    c.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    c.attrs = at;
    c.numAttrs = pdl_enabled() ? 1 : 0;
    launch_check(cudaLaunchKernelEx(&c, kernel, std::forward<Act>(args)...), "cudaLaunchKernelEx");
}

}  // namespace mpmb
