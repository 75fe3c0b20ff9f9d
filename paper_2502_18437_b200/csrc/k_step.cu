// k_step.cu — grid-side kernels of a substep: grid update + contact + BC (K3), BC alone
// (hook adapter) and free bodies + accumulator merge (K7).  Node layout {x, y, z, mass}.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "launch.h"

namespace mpmb {

// node l (0..63) of global brick gb in the linear node pool
__device__ __forceinline__ uint64_t brick_node(const Params& P, uint32_t gb, int l) {
    const uint32_t scene = gb / P.geo.bricks_per_scene;
    const uint32_t local = gb - scene * P.geo.bricks_per_scene;
    const uint32_t nb0 = static_cast<uint32_t>(P.geo.nb[0]), nb1 = static_cast<uint32_t>(P.geo.nb[1]);
    const int i = static_cast<int>((local % nb0) * 4u) + (l & 3);
    const int j = static_cast<int>(((local / nb0) % nb1) * 4u) + ((l >> 2) & 3);
    const int k = static_cast<int>((local / (nb0 * nb1)) * 4u) + (l >> 4);
    return static_cast<uint64_t>(scene) * P.geo.nodes_per_scene + node_linear(P.geo, i, j, k);
}

// Per-substep shape cull table (one block): the world AABB of each shape's local box
// (DevShape::lbox) under this substep's pose (kinematic table or integrated free pose):
// cull[2i] = {min, bounded ? 1 : -1}, cull[2i+1] = {max, 0}.
__device__ __forceinline__ void cull_shape(const Params& P, int i, int sub) {
    P.pose_eff[i] = pose_of_sub(P, i, sub);  // the contact pass and push-out of `sub` read it
    {
        const DevShape& sh = P.shapes[i];
        if (sh.lbox_h[0] < 0.f) {
            P.cull[2 * i] = make_float4(0.f, 0.f, 0.f, -1.f);
            P.cull[2 * i + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
            return;
        }
        const DevPose& pose = pose_of_sub(P, i, sub);
        const float x = pose.rot[0], y = pose.rot[1], z = pose.rot[2], w = pose.rot[3];
        const float R[3][3] = {{1.f - 2.f * (y * y + z * z), 2.f * (x * y - z * w), 2.f * (x * z + y * w)},
                               {2.f * (x * y + z * w), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - x * w)},
                               {2.f * (x * z - y * w), 2.f * (y * z + x * w), 1.f - 2.f * (x * x + y * y)}};
        float c[3], h[3];
        for (int a = 0; a < 3; ++a) {
            c[a] = pose.pos[a] + R[a][0] * sh.lbox_c[0] + R[a][1] * sh.lbox_c[1] + R[a][2] * sh.lbox_c[2];
            // |R| h, widened for a not-quite-unit quaternion and float rounding
            h[a] = (fabsf(R[a][0]) * sh.lbox_h[0] + fabsf(R[a][1]) * sh.lbox_h[1] + fabsf(R[a][2]) * sh.lbox_h[2]) *
                       1.001f + 1e-5f;
        }
        P.cull[2 * i] = make_float4(c[0] - h[0], c[1] - h[1], c[2] - h[2], 1.f);
        P.cull[2 * i + 1] = make_float4(c[0] + h[0], c[1] + h[1], c[2] + h[2], 0.f);
    }
}

__global__ void k_shape_cull(const Params P) {
    pdl_enter();
    for (int i = threadIdx.x; i < P.n_shapes; i += blockDim.x) cull_shape(P, i, P.sub);
}

void launch_shape_cull(const Params& P, cudaStream_t st) { launch_chain(k_shape_cull, 1, 128, 0, st, P); }

// ==============================================================  grid update
// 64 threads per active brick (one node each).  Reads the P2G accumulator and zeroes it
// (it is the last reader), writes {mass, velocity} for G2P.  Contact shapes are applied
// in order per node (last shape wins, contact.hpp:106-134); each warp reduces its
// per-shape impulse/torque/count with shuffles and adds them in FP64.
//
// Latency: the per-brick chain (brick -> accumulator -> shapes) is software-pipelined over
// the grid-stride loop (a stride spreads the costly contact bricks over all workers): the
// decoded brick (active_info, written by the collect) is loaded two iterations ahead, its
// accumulator and -- when every scene has the same shape count -- the first shape's cull box
// one ahead.
__global__ void __launch_bounds__(256) k_grid_update(const Params P) {
    pdl_enter();
    const uint32_t n_bricks = *P.n_active_bricks;
    const int l = threadIdx.x & 63;
    const int li = l & 3, lj = (l >> 2) & 3, lk = l >> 4;
    const uint32_t per_block = blockDim.x >> 6;
    const int lane = threadIdx.x & 31;
    const uint32_t bstride = gridDim.x * per_block;
    const uint64_t nps = P.geo.nodes_per_scene;
    const uint32_t nb0 = static_cast<uint32_t>(P.geo.nb[0]), nb1 = static_cast<uint32_t>(P.geo.nb[1]);
    const int sps = P.contact ? P.shapes_per_scene : 0;  // > 0: uniform shape ranges
    uint32_t bi = blockIdx.x * per_block + (threadIdx.x >> 6);
    uint2 in_next = bi < n_bricks ? P.active_info[bi] : make_uint2(0u, 0u);
    uint2 in_after = bi + bstride < n_bricks ? P.active_info[bi + bstride] : make_uint2(0u, 0u);
    // node of this thread in decoded brick `in`
    auto node_of = [&](uint2 in, int& i, int& j, int& k) {
        i = static_cast<int>(in.x & 1023u) * 4 + li;
        j = static_cast<int>((in.x >> 10) & 1023u) * 4 + lj;
        k = static_cast<int>(in.x >> 20) * 4 + lk;
        return static_cast<uint64_t>(in.y) * nps + node_linear(P.geo, i, j, k);
    };
    int ni, nj, nk;
    uint64_t idx_next = node_of(in_next, ni, nj, nk);
    float4 a_next = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 lo_next = make_float4(0.f, 0.f, 0.f, -1.f), hi_next = lo_next;
    if (bi < n_bricks) {
        a_next = P.grid_acc[idx_next];
        if (sps > 0) {
            lo_next = P.cull[2 * in_next.y * sps];
            hi_next = P.cull[2 * in_next.y * sps + 1];
        }
    }
    for (; bi < n_bricks; bi += bstride) {
        const uint2 in = in_next;
        const float4 a = a_next;
        const uint64_t idx = idx_next;
        const float4 lo0 = lo_next, hi0 = hi_next;
        int i, j, k;
        node_of(in, i, j, k);
        in_next = in_after;
        if (bi + bstride < n_bricks) {
            idx_next = node_of(in_next, ni, nj, nk);
            a_next = P.grid_acc[idx_next];
            if (sps > 0) {
                lo_next = P.cull[2 * in_next.y * sps];
                hi_next = P.cull[2 * in_next.y * sps + 1];
            }
        }
        if (bi + 2 * bstride < n_bricks) in_after = P.active_info[bi + 2 * bstride];
        const int scene = static_cast<int>(in.y);
        const SceneView S = scene_view(P, scene);
        int cs_begin = 0, cs_count = 0;
        float4 cs_lo = lo0, cs_hi = hi0;
        if (sps > 0) {
            cs_begin = scene * sps;
            cs_count = sps;
        } else if (P.contact) {
            cs_begin = P.scenes[scene].shape_begin;
            cs_count = P.scenes[scene].shape_count;
            if (cs_count > 0) {
                cs_lo = P.cull[2 * cs_begin];
                cs_hi = P.cull[2 * cs_begin + 1];
            }
        }
        MPMB_DCHECK(idx < P.total_nodes);
        const bool own = i >= P.geo.own_lo && i < P.geo.own_hi;
        const int ig = i + P.geo.goff;  // global x index (BC, node position)
        P.grid_acc[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (l == 0)  // the brick id, rebuilt from the decoded coordinates
            P.brick_stamp[S.brick_base + ((in.x >> 20) * nb1 + ((in.x >> 10) & 1023u)) * nb0 + (in.x & 1023u)] =
                P.epoch;
        const float m = a.w;
        const bool live = m > kMassEps;
        V3 v = mk(0.f, 0.f, 0.f);
        if (live) {  // solvers.hpp:58-61
            v = vdiv(mk(a.x, a.y, a.z), m);
            if (P.gravity) v = v + mk(P.g[0], P.g[1], P.g[2]) * P.dt;
        }
        if (P.contact && cs_count > 0) {  // contact.hpp:97-136, shapes in order
            const V3 xn = mk(FA(S.origin[0], FM(static_cast<float>(i + P.geo.goff), S.dx)),  // state.hpp:49-51
                             FA(S.origin[1], FM(static_cast<float>(j), S.dx)),
                             FA(S.origin[2], FM(static_cast<float>(k), S.dx)));
            for (int si = cs_begin; si < cs_begin + cs_count; ++si) {
                const DevShape& sh = P.shapes[si];
                V3 imp = mk(0.f, 0.f, 0.f), tq = mk(0.f, 0.f, 0.f);
                int hit = 0;
                // a slab domain sums contact only over the nodes it owns (ghosts are the
                // neighbour's; their velocities are overwritten by the halo exchange)
                const bool near = si == cs_begin ? aabb_may_touch(cs_lo, cs_hi, xn.x, xn.y, xn.z)
                                                 : cull_may_touch(P, si, xn.x, xn.y, xn.z);
                if (live && own && near) {
                    const DevPose& pose = P.pose_eff[si];  // this substep's (cull pass)
                    const Sdf s = sdf_query(sh, pose, P.verts, P.ints, xn);
                    if (node_in_contact(s, sh.hw)) {
                        V3 delta;
                        const V3 vc = contact_correct(sh, s, v, rigid_point_velocity(pose, xn), delta);
                        if (norm2(delta) > 0.f) {
                            v = vc;
                            imp = delta * (-m);
                            tq = cross(xn - mk(pose.pos[0], pose.pos[1], pose.pos[2]), imp);
                            hit = 1;
                            if (P.ex_ckey) {
                                const uint32_t r = atomicAdd(P.ex_cn, 1u);
                                if (r < P.ex_ccap) {
                                    P.ex_ckey[r] = (static_cast<uint64_t>(si) << 40) |
                                                   ((static_cast<uint64_t>(k) * S.dims[1] + j) * S.dims[0] + ig);
                                    float* o = P.ex_crec + 6ull * r;
                                    o[0] = imp.x; o[1] = imp.y; o[2] = imp.z;
                                    o[3] = tq.x; o[4] = tq.y; o[5] = tq.z;
                                }
                            }
                        }
                    }
                }
                if (!P.ex_ckey && __any_sync(0xffffffffu, hit)) {
                    float r[7] = {imp.x, imp.y, imp.z, tq.x, tq.y, tq.z, static_cast<float>(hit)};
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                        for (int q = 0; q < 7; ++q) r[q] += __shfl_xor_sync(0xffffffffu, r[q], o);
                    if (lane == 0) {
#pragma unroll
                        for (int q = 0; q < 6; ++q) atomicAdd(&P.acc_sub[6 * si + q], static_cast<double>(r[q]));
                        atomicAdd(&P.cnt_sub[si], static_cast<int>(r[6]));
                    }
                }
            }
        }
        if (live) {  // solvers.hpp:30-50 (bc < 0: deferred to k_grid_bc, hook adapter)
            const bool bxm = ig < 2 || ig >= S.dims[0] - 2;
            const bool bym = j < 2 || j >= S.dims[1] - 2;
            const bool bzm = k < 2 || k >= S.dims[2] - 2;
            if (P.bc >= 0 && (bxm || bym || bzm)) {
                if (P.bc == BC_STICKY) {
                    v = mk(0.f, 0.f, 0.f);
                } else {
                    if (bxm) v.x = 0.f;
                    if (bym) v.y = 0.f;
                    if (bzm) v.z = 0.f;
                }
            }
            P.grid_vel[idx] = make_float4(v.x, v.y, v.z, m);
        } else {
            // below kMassEps: G2P skips the node (solvers.hpp:186) -- a zero velocity makes
            // its contribution vanish without a per-node test; the momentum stays readable
            P.grid_vel[idx] = make_float4(0.f, 0.f, 0.f, m);
            if (P.dead_mom) P.dead_mom[idx] = a;
        }
    }
}

// Boundary conditions alone over the active bricks (after a host GridHook edited the grid).
__global__ void __launch_bounds__(256) k_grid_bc(const Params P) {
    const uint32_t n_bricks = *P.n_active_bricks;
    const int l = threadIdx.x & 63;
    const uint32_t per_block = blockDim.x >> 6;
    for (uint32_t bi = blockIdx.x * per_block + (threadIdx.x >> 6); bi < n_bricks;
         bi += gridDim.x * per_block) {
        const uint32_t gb = P.active_bricks[bi];
        const SceneView S = scene_view(P, static_cast<int>(P.brick_scene[gb]));
        const uint32_t local = gb - S.brick_base;
        const int bx = static_cast<int>(local % S.nb[0]);
        const int by = static_cast<int>((local / S.nb[0]) % S.nb[1]);
        const int bz = static_cast<int>(local / (static_cast<uint32_t>(S.nb[0]) * S.nb[1]));
        const int i = bx * 4 + (l & 3), j = by * 4 + ((l >> 2) & 3), k = bz * 4 + (l >> 4);
        const uint64_t idx = S.node_base + node_linear(P.geo, i, j, k);
        float4 a = P.grid_vel[idx];
        if (!(a.w > kMassEps)) continue;
        const bool bxm = i + P.geo.goff < 2 || i + P.geo.goff >= S.dims[0] - 2;
        const bool bym = j < 2 || j >= S.dims[1] - 2;
        const bool bzm = k < 2 || k >= S.dims[2] - 2;
        if (!(bxm || bym || bzm)) continue;
        if (P.bc == BC_STICKY) {
            a.x = a.y = a.z = 0.f;
        } else {
            if (bxm) a.x = 0.f;
            if (bym) a.y = 0.f;
            if (bzm) a.z = 0.f;
        }
        P.grid_vel[idx] = a;
    }
}

// ==========================================================  free bodies (K7)
// integrate_free_body (rigid_dynamics.hpp:82-103) with this substep's impulse, then merge
// the substep accumulators into the frame accumulators (scene.hpp:220-232).
// next_sub >= 0: also build the cull table of that substep (its poses are final once the free
// bodies have moved), saving the next substep's k_shape_cull launch.
__device__ __forceinline__ void free_bodies_body(const Params& P, int integrate, int merge, int next_sub) {
    for (int i = threadIdx.x; i < P.n_shapes; i += blockDim.x) {
        const DevShape& sh = P.shapes[i];
        if (integrate && sh.motion == MOTION_FREE) {
            const int t = P.sub * P.n_shapes + i;
            DevPose pose = P.pose_override[t] ? P.pose_table[t] : P.free_pose[i];
            const float J[3] = {static_cast<float>(P.acc_sub[6 * i + 0]),
                                static_cast<float>(P.acc_sub[6 * i + 1]),
                                static_cast<float>(P.acc_sub[6 * i + 2])};
            const float T[3] = {static_cast<float>(P.acc_sub[6 * i + 3]),
                                static_cast<float>(P.acc_sub[6 * i + 4]),
                                static_cast<float>(P.acc_sub[6 * i + 5])};
            const float dt = P.dt;
            const float im = FD(1.f, sh.body_mass);
#pragma unroll
            for (int a = 0; a < 3; ++a) pose.lin[a] = FA(pose.lin[a], FA(FM(J[a], im), FM(P.g[a], dt)));
            // I_world^-1 = (R * I_body^-1) * R^T (math.hpp:101-110, 163-172), reference order
            const float x = pose.rot[0], y = pose.rot[1], z = pose.rot[2], w = pose.rot[3];
            const float xx = FM(x, x), yy = FM(y, y), zz = FM(z, z);
            const float xy = FM(x, y), xz = FM(x, z), yz = FM(y, z);
            const float wx = FM(w, x), wy = FM(w, y), wz = FM(w, z);
            const float R[9] = {FS(1.f, FM(2.f, FA(yy, zz))), FM(2.f, FS(xy, wz)), FM(2.f, FA(xz, wy)),
                                FM(2.f, FA(xy, wz)), FS(1.f, FM(2.f, FA(xx, zz))), FM(2.f, FS(yz, wx)),
                                FM(2.f, FS(xz, wy)), FM(2.f, FA(yz, wx)), FS(1.f, FM(2.f, FA(xx, yy)))};
            const float D[9] = {FD(1.f, sh.inertia[0]), 0.f, 0.f, 0.f, FD(1.f, sh.inertia[1]), 0.f,
                                0.f, 0.f, FD(1.f, sh.inertia[2])};
            float RD[9], M[9];
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    float s = 0.f;
#pragma unroll
                    for (int k = 0; k < 3; ++k) s = FA(s, FM(R[3 * r + k], D[3 * k + c]));
                    RD[3 * r + c] = s;
                }
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    float s = 0.f;
#pragma unroll
                    for (int k = 0; k < 3; ++k) s = FA(s, FM(RD[3 * r + k], R[3 * c + k]));
                    M[3 * r + c] = s;
                }
#pragma unroll
            for (int a = 0; a < 3; ++a)
                pose.ang[a] = FA(pose.ang[a], FA(FA(FM(M[3 * a], T[0]), FM(M[3 * a + 1], T[1])),
                                                 FM(M[3 * a + 2], T[2])));
#pragma unroll
            for (int a = 0; a < 3; ++a) pose.pos[a] = FA(pose.pos[a], FM(pose.lin[a], dt));
            const Q4 dq = qmul(Q4{pose.ang[0], pose.ang[1], pose.ang[2], 0.f}, Q4{x, y, z, w});
            const float h = FM(0.5f, dt);
            const Q4 qn = qnormalized(Q4{FA(x, FM(h, dq.x)), FA(y, FM(h, dq.y)), FA(z, FM(h, dq.z)),
                                         FA(w, FM(h, dq.w))});
            pose.rot[0] = qn.x; pose.rot[1] = qn.y; pose.rot[2] = qn.z; pose.rot[3] = qn.w;
            P.free_pose[i] = pose;
        }
        if (merge) {
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                if (P.exact)  // the reference's float frame sums (scene.hpp:228-231)
                    P.acc_frame[6 * i + q] = static_cast<double>(
                        __fadd_rn(static_cast<float>(P.acc_frame[6 * i + q]), static_cast<float>(P.acc_sub[6 * i + q])));
                else
                    P.acc_frame[6 * i + q] += P.acc_sub[6 * i + q];
                P.acc_sub[6 * i + q] = 0.0;
            }
            P.cnt_frame[i] += P.cnt_sub[i];
            P.cnt_sub[i] = 0;
        }
        if (next_sub >= 0) cull_shape(P, i, next_sub);
    }
}

__global__ void k_free_bodies(const Params P, int integrate, int merge, int next_sub) {
    pdl_enter();
    free_bodies_body(P, integrate, merge, next_sub);
}

// The two small passes between K8 and the next grid update in one launch: the last block
// runs the free bodies (K7), the others collect the active bricks of the next substep.
// Both only read what K8 and the grid update before it wrote.
__global__ void __launch_bounds__(256) k_collect_free(const Params P, uint32_t n_bricks, int integrate, int merge,
                                                      int next_sub) {
    pdl_enter();
    if (blockIdx.x == gridDim.x - 1) free_bodies_body(P, integrate, merge, next_sub);
    else collect_bricks_body(P, n_bricks, blockIdx.x, gridDim.x - 1);
}

// ===================================================================  launchers
static int grid_for(int64_t work, int threads, int max_blocks) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return static_cast<int>(b);
}


// grid-stride blocks per SM of the grid update (MPMB_GRID_BPS in the environment: A/B).  Two
// (= the resident blocks at 106 registers: one wave, the brick pipelining spans each block's
// whole loop) measured C5 +0.2-0.6 %, M1 +0.8 %, C3 +3 %, but C2 -19 % and C1 -3 %; kept at 8.
static int grid_bps() {
    static const int v = [] {
        const char* e = std::getenv("MPMB_GRID_BPS");
        return e ? std::max(1, std::atoi(e)) : 8;
    }();
    return v;
}
void launch_grid_update(const Params& P, int64_t max_bricks, cudaStream_t st) {
    const int threads = 256;
    const int blocks = grid_for(max_bricks * 64, threads, 148 * grid_bps());
    launch_chain(k_grid_update, blocks, threads, 0, st, P);
}




void launch_collect_free(const Params& P, uint32_t n_bricks, bool integrate, bool merge, int next_sub,
                         cudaStream_t st) {
    int64_t blocks = (static_cast<int64_t>(n_bricks) + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    launch_chain(k_collect_free, static_cast<int>(blocks) + 1, 256, 0, st, P, n_bricks, integrate ? 1 : 0,
                 merge ? 1 : 0, next_sub);
}

void launch_free_bodies(const Params& P, bool integrate, bool merge, cudaStream_t st, int next_sub) {
    launch_chain(k_free_bodies, 1, 128, 0, st, P, integrate ? 1 : 0, merge ? 1 : 0, next_sub);
}

void launch_grid_bc(const Params& P, int64_t max_bricks, cudaStream_t st) {
    const int threads = 256;
    k_grid_bc<<<grid_for(max_bricks * 64, threads, 148 * 8), threads, 0, st>>>(P);
    MPMB_LAUNCHED("k_grid_bc");
}

}  // namespace mpmb
