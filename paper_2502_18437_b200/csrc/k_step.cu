// k_step.cu — per-substep kernels: P2G (K2/K5), grid update + contact + BC (K3),
// G2P (K4/K6), free bodies (K7), standalone push-out / deactivation.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "launch.h"

namespace mpmb {

// =====================================================================  P2G
// One lane per chunk (<= KMAX particles of one cell, contiguous in the chunk-interleaved
// layout: the k-th particles of the 32 chunks of a warp are adjacent -> coalesced loads).
// The lane accumulates the 27 stencil nodes x {mass, momentum} in registers while the
// stencil base stays the same, then flushes with 27 red.global.add.v4.f32.
__device__ __forceinline__ void p2g_flush(const Params& P, const DevScene& S, const int cb[3],
                                          float4 (&acc)[27]) {
    uint32_t tx[3], ty[3], tz[3];
    node_offsets(S, cb, tx, ty, tz);
    float4* g = P.grid_acc + S.node_base;
#pragma unroll
    for (int dk = 0; dk < 3; ++dk)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj)
#pragma unroll
            for (int di = 0; di < 3; ++di) {
                const int n = (dk * 3 + dj) * 3 + di;
                atomicAdd(g + (tz[dk] + ty[dj] + tx[di]), acc[n]);
                acc[n] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
    // mark the <= 8 bricks this stencil touches; first marker appends to the active list
    const int bx0 = cb[0] >> 2, bx1 = (cb[0] + 2) >> 2;
    const int by0 = cb[1] >> 2, by1 = (cb[1] + 2) >> 2;
    const int bz0 = cb[2] >> 2, bz1 = (cb[2] + 2) >> 2;
    for (int bz = bz0; bz <= bz1; ++bz)
        for (int by = by0; by <= by1; ++by)
            for (int bx = bx0; bx <= bx1; ++bx) {
                const uint32_t gb = S.brick_base + (bz * S.nb[1] + by) * S.nb[0] + bx;
                if (P.brick_flag[gb] == 0u && atomicExch(&P.brick_flag[gb], 1u) == 0u)
                    P.active_bricks[atomicAdd(P.n_active_bricks, 1u)] = gb;
            }
}

template <bool MLS>
__global__ void __launch_bounds__(128) k_p2g(const Params P) {
    const int lane = threadIdx.x & 31;
    const uint32_t n_groups = *P.n_groups;
    const uint32_t n_chunks = *P.n_chunks;
    const uint32_t wpb = blockDim.x >> 5;
    const unsigned lt = lanemask_lt();
    for (uint32_t g = blockIdx.x * wpb + (threadIdx.x >> 5); g < n_groups; g += gridDim.x * wpb) {
        const uint32_t c = g * 32u + lane;
        const int len = c < n_chunks ? P.chunk_len[c] : 0;
        const uint32_t slot0 = P.group_base[g];
        float4 acc[27];
#pragma unroll
        for (int n = 0; n < 27; ++n) acc[n] = make_float4(0.f, 0.f, 0.f, 0.f);
        int cb[3] = {INT_MIN, INT_MIN, INT_MIN};
        int cscene = -1;
        uint32_t off = 0;
        for (int k = 0; k < KMAX; ++k) {
            const unsigned mask = __ballot_sync(0xffffffffu, len > k);
            if (mask == 0u) break;
            if (len > k) {
                const uint32_t s = slot0 + off + __popc(mask & lt);
                const float4 r = P.pl[PR][s];
                const uint32_t flags = __float_as_uint(r.z);
                if (flags & kActiveBit) {
                    Part p;
                    load_part(P, s, p);
                    const int scene = static_cast<int>((flags >> kSceneShift) & kSceneMask);
                    const DevScene& S = P.scenes[scene];
                    int b[3];
                    float fx[3];
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        b[a] = stencil_base(p.x[a], S.origin[a], S.inv_dx, fx[a]);
                        b[a] = min(max(b[a], 0), S.dims[a] - 3);  // memory guard only
                    }
                    if (b[0] != cb[0] || b[1] != cb[1] || b[2] != cb[2] || scene != cscene) {
                        if (cscene >= 0) p2g_flush(P, P.scenes[cscene], cb, acc);
                        cb[0] = b[0]; cb[1] = b[1]; cb[2] = b[2];
                        cscene = scene;
                    }
                    const float m = r.x;
                    // affine = m C - dt V (4/dx^2) sigma  (solvers.hpp:154-156; PB: m C, :222)
                    float A[9];
                    if (MLS) {
                        float sig[9];
                        if (P.use_stress_in) {
                            const float* src = P.stress_in + 9ull * __float_as_uint(r.w);
#pragma unroll
                            for (int i = 0; i < 9; ++i) sig[i] = src[i];
                        } else {
                            const float4 mat = P.mats[flags & kMatMask];
                            neo_hookean(p.F, mat.y, mat.z, sig);
                        }
                        const float volume = det3(p.F) * r.y;
                        const float sc = -P.dt * volume * S.m_inv;
#pragma unroll
                        for (int i = 0; i < 9; ++i) A[i] = p.C[i] * m + sig[i] * sc;
                    } else {
#pragma unroll
                        for (int i = 0; i < 9; ++i) A[i] = p.C[i] * m;
                    }
                    float w[3][3], rel[3][3];
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        bspline_w(fx[a], w[a]);
#pragma unroll
                        for (int o = 0; o < 3; ++o)  // node_position - x (state.hpp:49-51)
                            rel[a][o] = (S.origin[a] + static_cast<float>(b[a] + o) * S.dx) - p.x[a];
                    }
                    const float mv0 = p.v[0] * m, mv1 = p.v[1] * m, mv2 = p.v[2] * m;
#pragma unroll
                    for (int dk = 0; dk < 3; ++dk) {
                        const float wz = w[2][dk];
                        const float uz0 = mv0 + A[2] * rel[2][dk];
                        const float uz1 = mv1 + A[5] * rel[2][dk];
                        const float uz2 = mv2 + A[8] * rel[2][dk];
#pragma unroll
                        for (int dj = 0; dj < 3; ++dj) {
                            const float wyz = w[1][dj] * wz;
                            const float u0 = uz0 + A[1] * rel[1][dj];
                            const float u1 = uz1 + A[4] * rel[1][dj];
                            const float u2 = uz2 + A[7] * rel[1][dj];
                            const float wm = wyz * m;
#pragma unroll
                            for (int di = 0; di < 3; ++di) {
                                const int n = (dk * 3 + dj) * 3 + di;
                                const float ww = w[0][di] * wyz;
                                const float t0 = u0 + A[0] * rel[0][di];
                                const float t1 = u1 + A[3] * rel[0][di];
                                const float t2 = u2 + A[6] * rel[0][di];
                                acc[n].x = fmaf(w[0][di], wm, acc[n].x);
                                acc[n].y = fmaf(ww, t0, acc[n].y);
                                acc[n].z = fmaf(ww, t1, acc[n].z);
                                acc[n].w = fmaf(ww, t2, acc[n].w);
                            }
                        }
                    }
                }
            }
            off += __popc(mask);
        }
        if (cscene >= 0) p2g_flush(P, P.scenes[cscene], cb, acc);
    }
}

// ==============================================================  grid update
// 64 threads per active brick (one node each).  Reads the P2G accumulator and zeroes it
// (it is the last reader), writes {mass, velocity} for G2P.  Contact shapes are applied
// in order per node (last shape wins, contact.hpp:106-134); each warp reduces its
// per-shape impulse/torque/count with shuffles and adds them in FP64.
__global__ void __launch_bounds__(256) k_grid_update(const Params P) {
    const uint32_t n_bricks = *P.n_active_bricks;
    const int l = threadIdx.x & 63;
    const uint32_t per_block = blockDim.x >> 6;
    const int lane = threadIdx.x & 31;
    for (uint32_t bi = blockIdx.x * per_block + (threadIdx.x >> 6); bi < n_bricks;
         bi += gridDim.x * per_block) {
        const uint32_t gb = P.active_bricks[bi];
        const int scene = static_cast<int>(P.brick_scene[gb]);
        const DevScene& S = P.scenes[scene];
        const uint32_t local = gb - S.brick_base;
        const int bx = static_cast<int>(local % S.nb[0]);
        const int by = static_cast<int>((local / S.nb[0]) % S.nb[1]);
        const int bz = static_cast<int>(local / (static_cast<uint32_t>(S.nb[0]) * S.nb[1]));
        const int i = bx * 4 + (l & 3), j = by * 4 + ((l >> 2) & 3), k = bz * 4 + (l >> 4);
        const uint64_t idx = S.node_base + static_cast<uint64_t>(local) * kBrickNodes + l;
        const float4 a = P.grid_acc[idx];
        P.grid_acc[idx] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (l == 0) {
            P.brick_flag[gb] = 0u;
            P.brick_stamp[gb] = P.epoch;
        }
        const float m = a.x;
        const bool live = m > kMassEps;
        V3 v = mk(0.f, 0.f, 0.f);
        if (live) {  // solvers.hpp:58-61
            v = vdiv(mk(a.y, a.z, a.w), m);
            if (P.gravity) v = v + mk(P.g[0], P.g[1], P.g[2]) * P.dt;
        }
        if (P.contact && S.shape_count > 0) {  // contact.hpp:97-136, shapes in order
            const V3 xn = mk(FA(S.origin[0], FM(static_cast<float>(i), S.dx)),  // state.hpp:49-51
                             FA(S.origin[1], FM(static_cast<float>(j), S.dx)),
                             FA(S.origin[2], FM(static_cast<float>(k), S.dx)));
            for (int si = S.shape_begin; si < S.shape_begin + S.shape_count; ++si) {
                const DevShape& sh = P.shapes[si];
                V3 imp = mk(0.f, 0.f, 0.f), tq = mk(0.f, 0.f, 0.f);
                int hit = 0;
                if (live) {
                    const DevPose& pose = pose_of(P, si);
                    const Sdf s = sdf_query(sh, pose, P.verts, P.ints, xn);
                    if (node_in_contact(s, sh.hw)) {
                        V3 delta;
                        const V3 vc = contact_correct(sh, s, v, rigid_point_velocity(pose, xn), delta);
                        if (norm2(delta) > 0.f) {
                            v = vc;
                            imp = delta * (-m);
                            tq = cross(xn - mk(pose.pos[0], pose.pos[1], pose.pos[2]), imp);
                            hit = 1;
                        }
                    }
                }
                if (__any_sync(0xffffffffu, hit)) {
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
            const bool bxm = i < 2 || i >= S.dims[0] - 2;
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
            P.grid_vel[idx] = make_float4(m, v.x, v.y, v.z);
        } else {
            P.grid_vel[idx] = a;  // below kMassEps: velocity undefined, keep momentum
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
        const DevScene& S = P.scenes[P.brick_scene[gb]];
        const uint32_t local = gb - S.brick_base;
        const int bx = static_cast<int>(local % S.nb[0]);
        const int by = static_cast<int>((local / S.nb[0]) % S.nb[1]);
        const int bz = static_cast<int>(local / (static_cast<uint32_t>(S.nb[0]) * S.nb[1]));
        const int i = bx * 4 + (l & 3), j = by * 4 + ((l >> 2) & 3), k = bz * 4 + (l >> 4);
        const uint64_t idx = S.node_base + static_cast<uint64_t>(local) * kBrickNodes + l;
        float4 a = P.grid_vel[idx];
        if (!(a.x > kMassEps)) continue;
        const bool bxm = i < 2 || i >= S.dims[0] - 2;
        const bool bym = j < 2 || j >= S.dims[1] - 2;
        const bool bzm = k < 2 || k >= S.dims[2] - 2;
        if (!(bxm || bym || bzm)) continue;
        if (P.bc == BC_STICKY) {
            a.y = a.z = a.w = 0.f;
        } else {
            if (bxm) a.y = 0.f;
            if (bym) a.z = 0.f;
            if (bzm) a.w = 0.f;
        }
        P.grid_vel[idx] = a;
    }
}

// ================================================================  G2P
// Gathers the 27 stencil velocities once per (lane, stencil base) into registers and
// reuses them across the chunk's particles.  Separable form of
//   v = sum w v_I,  B = sum (w v_I) (x_I - x_p)^T          (solvers.hpp:178-190)
// summed row by row over di, then scaled by w_y w_z.
__device__ __forceinline__ void g2p_load_nodes(const Params& P, const DevScene& S, const int b[3],
                                               V3 (&nv)[27]) {
    uint32_t tx[3], ty[3], tz[3];
    node_offsets(S, b, tx, ty, tz);
    const float4* g = P.grid_vel + S.node_base;
#pragma unroll
    for (int dk = 0; dk < 3; ++dk)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj)
#pragma unroll
            for (int di = 0; di < 3; ++di) {
                const float4 q = __ldg(g + (tz[dk] + ty[dj] + tx[di]));
                const bool live = q.x > kMassEps;  // solvers.hpp:186
                nv[(dk * 3 + dj) * 3 + di] = live ? mk(q.y, q.z, q.w) : mk(0.f, 0.f, 0.f);
            }
}

__device__ __forceinline__ void g2p_gather(const V3 (&nv)[27], const float w[3][3],
                                           const float rel[3][3], V3& vn, float B[9]) {
    vn = mk(0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 9; ++i) B[i] = 0.f;
#pragma unroll
    for (int dk = 0; dk < 3; ++dk)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            V3 a = mk(0.f, 0.f, 0.f), bb = mk(0.f, 0.f, 0.f);
#pragma unroll
            for (int di = 0; di < 3; ++di) {
                const V3 q = nv[(dk * 3 + dj) * 3 + di];
                const float wx = w[0][di], wr = w[0][di] * rel[0][di];
                a = mk(fmaf(wx, q.x, a.x), fmaf(wx, q.y, a.y), fmaf(wx, q.z, a.z));
                bb = mk(fmaf(wr, q.x, bb.x), fmaf(wr, q.y, bb.y), fmaf(wr, q.z, bb.z));
            }
            const float wyz = w[1][dj] * w[2][dk];
            const float wy = wyz * rel[1][dj], wz = wyz * rel[2][dk];
            vn = mk(fmaf(wyz, a.x, vn.x), fmaf(wyz, a.y, vn.y), fmaf(wyz, a.z, vn.z));
            // B row r = component r of velocity; column c = rel component c
            B[0] = fmaf(wyz, bb.x, B[0]); B[3] = fmaf(wyz, bb.y, B[3]); B[6] = fmaf(wyz, bb.z, B[6]);
            B[1] = fmaf(wy, a.x, B[1]);   B[4] = fmaf(wy, a.y, B[4]);   B[7] = fmaf(wy, a.z, B[7]);
            B[2] = fmaf(wz, a.x, B[2]);   B[5] = fmaf(wz, a.y, B[5]);   B[8] = fmaf(wz, a.z, B[8]);
        }
}

// Push-out of one particle against the scene's shapes, in order (contact.hpp:140-179).
__device__ __forceinline__ int pushout_particle(const Params& P, const DevScene& S, float x[3],
                                                float v[3]) {
    int pushed = 0;
    const float clearance = FM(1e-4f, S.dx);
    for (int si = S.shape_begin; si < S.shape_begin + S.shape_count; ++si) {
        const DevShape& sh = P.shapes[si];
        const DevPose& pose = pose_of(P, si);
        const Sdf s = sdf_query(sh, pose, P.verts, P.ints, mk(x[0], x[1], x[2]));
        float move = 0.f;
        if (s.region == REGION_SURFACE || s.region == REGION_SPINE) {
            if (s.distance < 0.f) move = FA(-s.distance, clearance);
        } else if (s.region == REGION_EDGE) {
            const float target = FM(0.5f, sh.hw);
            const float d = fabsf(s.distance);
            if (d < target) move = FA(FS(target, d), clearance);
        } else if (s.region == REGION_CURVE) {
            const float target = FM(0.5f, sh.hw);
            if (s.distance < target) move = FA(FS(target, s.distance), clearance);
        }
        if (move > 0.f) {
            x[0] = FA(x[0], FM(s.normal.x, move));
            x[1] = FA(x[1], FM(s.normal.y, move));
            x[2] = FA(x[2], FM(s.normal.z, move));
            const V3 vr = rigid_point_velocity(pose, mk(x[0], x[1], x[2]));
            const float vn = dot(mk(v[0], v[1], v[2]) - vr, s.normal);
            if (vn < 0.f) {
                v[0] = FS(v[0], FM(s.normal.x, vn));
                v[1] = FS(v[1], FM(s.normal.y, vn));
                v[2] = FS(v[2], FM(s.normal.z, vn));
            }
            ++pushed;
        }
    }
    return pushed;
}

// F <- (I + C dt) F  (solvers.hpp:194, 275) in the reference's Mat3 product order
// (math.hpp:101-110: s = 0; s += a_ik b_kj)
__device__ __forceinline__ void update_F(const float C[9], float dt, float F[9]) {
    float A[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) A[i] = FA((i % 4) == 0 ? 1.f : 0.f, FM(C[i], dt));
    float Fn[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            Fn[3 * i + j] = FA(FA(FM(A[3 * i], F[j]), FM(A[3 * i + 1], F[3 + j])), FM(A[3 * i + 2], F[6 + j]));
#pragma unroll
    for (int i = 0; i < 9; ++i) F[i] = Fn[i];
}

template <bool PB>
__global__ void __launch_bounds__(128) k_g2p(const Params P) {
    const int lane = threadIdx.x & 31;
    const uint32_t n_groups = *P.n_groups;
    const uint32_t n_chunks = *P.n_chunks;
    const uint32_t wpb = blockDim.x >> 5;
    const unsigned lt = lanemask_lt();
    for (uint32_t g = blockIdx.x * wpb + (threadIdx.x >> 5); g < n_groups; g += gridDim.x * wpb) {
        const uint32_t c = g * 32u + lane;
        const int len = c < n_chunks ? P.chunk_len[c] : 0;
        const uint32_t slot0 = P.group_base[g];
        V3 nv[27];
        int cb[3] = {INT_MIN, INT_MIN, INT_MIN};
        int cscene = -1, my_scene = 0;
        int n_inv = 0, n_fail = 0, n_push = 0, n_deact = 0;
        uint32_t off = 0;
        for (int k = 0; k < KMAX; ++k) {
            const unsigned mask = __ballot_sync(0xffffffffu, len > k);
            if (mask == 0u) break;
            if (len > k) {
                const uint32_t s = slot0 + off + __popc(mask & lt);
                float4 r = P.pl[PR][s];
                uint32_t flags = __float_as_uint(r.z);
                if (flags & kActiveBit) {
                    Part p;
                    load_part(P, s, p);
                    const int scene = static_cast<int>((flags >> kSceneShift) & kSceneMask);
                    my_scene = scene;
                    const DevScene& S = P.scenes[scene];
                    int b[3];
                    float fx[3];
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        b[a] = stencil_base(p.x[a], S.origin[a], S.inv_dx, fx[a]);
                        b[a] = min(max(b[a], 0), S.dims[a] - 3);
                    }
                    if (b[0] != cb[0] || b[1] != cb[1] || b[2] != cb[2] || scene != cscene) {
                        g2p_load_nodes(P, S, b, nv);
                        cb[0] = b[0]; cb[1] = b[1]; cb[2] = b[2];
                        cscene = scene;
                    }
                    float w[3][3], rel[3][3];
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        bspline_w(fx[a], w[a]);
#pragma unroll
                        for (int o = 0; o < 3; ++o)
                            rel[a][o] = (S.origin[a] + static_cast<float>(b[a] + o) * S.dx) - p.x[a];
                    }
                    V3 vn;
                    float B[9];
                    g2p_gather(nv, w, rel, vn, B);
                    p.v[0] = vn.x; p.v[1] = vn.y; p.v[2] = vn.z;
                    bool do_commit;
                    if (!PB) {  // solvers.hpp:191-195
#pragma unroll
                        for (int i = 0; i < 9; ++i) p.C[i] = B[i] * S.m_inv;
                        do_commit = true;
                    } else {  // solvers.hpp:259-267
                        float Cc[9], Cn[9];
#pragma unroll
                        for (int i = 0; i < 9; ++i) Cc[i] = B[i] * S.m_inv;
                        const float4 mat = P.mats[flags & kMatMask];
                        if (corotational_project(p.F, Cc, P.dt, mat.w, Cn)) {
#pragma unroll
                            for (int i = 0; i < 9; ++i) p.C[i] = Cn[i];
                        } else {
                            ++n_fail;
                        }
                        do_commit = P.commit != 0;
                    }
                    if (do_commit) {  // solvers.hpp:193-195 / 274-276
                        p.x[0] = FA(p.x[0], FM(p.v[0], P.dt));
                        p.x[1] = FA(p.x[1], FM(p.v[1], P.dt));
                        p.x[2] = FA(p.x[2], FM(p.v[2], P.dt));
                        update_F(p.C, P.dt, p.F);
                        if (det3(p.F) <= 0.f) ++n_inv;
                        if (P.pushout && S.shape_count > 0) n_push += pushout_particle(P, S, p.x, p.v);
                        if (P.deactivate && !spline_in_domain(mk(p.x[0], p.x[1], p.x[2]), S)) {
                            flags &= ~kActiveBit;
                            r.z = __uint_as_float(flags);
                            P.pl[PR][s] = r;
                            ++n_deact;
                        }
                    }
                    store_part(P, s, p);
                }
            }
            off += __popc(mask);
        }
        add_scene_counter(P.counters, my_scene, 0, n_inv);
        add_scene_counter(P.counters, my_scene, 1, n_fail);
        add_scene_counter(P.counters, my_scene, 2, n_push);
        add_scene_counter(P.counters, my_scene, 3, n_deact);
    }
}

// ================================================  standalone push-out / deactivation
__global__ void k_pushout(const Params P) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < P.n_total; base += stride) {
        const int64_t s = base + threadIdx.x;
        int pushed = 0, scene = 0;
        if (s < P.n_total) {
            const float4 r = P.pl[PR][s];
            const uint32_t flags = __float_as_uint(r.z);
            if (flags & kActiveBit) {
                scene = static_cast<int>((flags >> kSceneShift) & kSceneMask);
                const DevScene& S = P.scenes[scene];
                if (S.shape_count > 0) {
                    float4 a = P.pl[0][s], b = P.pl[1][s];
                    float x[3] = {a.x, a.y, a.z}, v[3] = {a.w, b.x, b.y};
                    pushed = pushout_particle(P, S, x, v);
                    if (pushed) {
                        P.pl[0][s] = make_float4(x[0], x[1], x[2], v[0]);
                        P.pl[1][s] = make_float4(v[1], v[2], b.z, b.w);
                    }
                }
            }
        }
        add_scene_counter(P.counters, scene, 2, pushed);
    }
}

__global__ void k_deactivate(const Params P) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < P.n_total; base += stride) {
        const int64_t s = base + threadIdx.x;
        int d = 0, scene = 0;
        if (s < P.n_total) {
            float4 r = P.pl[PR][s];
            uint32_t flags = __float_as_uint(r.z);
            if (flags & kActiveBit) {
                scene = static_cast<int>((flags >> kSceneShift) & kSceneMask);
                const float4 a = P.pl[0][s];
                if (!spline_in_domain(mk(a.x, a.y, a.z), P.scenes[scene])) {
                    r.z = __uint_as_float(flags & ~kActiveBit);
                    P.pl[PR][s] = r;
                    d = 1;
                }
            }
        }
        add_scene_counter(P.counters, scene, 3, d);
    }
}

// ==========================================================  free bodies (K7)
// integrate_free_body (rigid_dynamics.hpp:82-103) with this substep's impulse, then merge
// the substep accumulators into the frame accumulators (scene.hpp:220-232).
__global__ void k_free_bodies(const Params P, int integrate, int merge) {
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
                P.acc_frame[6 * i + q] += P.acc_sub[6 * i + q];
                P.acc_sub[6 * i + q] = 0.0;
            }
            P.cnt_frame[i] += P.cnt_sub[i];
            P.cnt_sub[i] = 0;
        }
    }
}

// ===================================================================  launchers
static int grid_for(int64_t work, int threads, int max_blocks) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return static_cast<int>(b);
}

void launch_p2g(const Params& P, bool mls, int64_t max_groups, cudaStream_t st) {
    const int threads = 128;
    const int blocks = grid_for(max_groups * 32, threads, 148 * 16);
    if (mls) k_p2g<true><<<blocks, threads, 0, st>>>(P);
    else k_p2g<false><<<blocks, threads, 0, st>>>(P);
}

void launch_grid_update(const Params& P, int64_t max_bricks, cudaStream_t st) {
    const int threads = 256;
    const int blocks = grid_for(max_bricks * 64, threads, 148 * 8);
    k_grid_update<<<blocks, threads, 0, st>>>(P);
}

void launch_g2p(const Params& P, bool pb, int64_t max_groups, cudaStream_t st) {
    const int threads = 128;
    const int blocks = grid_for(max_groups * 32, threads, 148 * 16);
    if (pb) k_g2p<true><<<blocks, threads, 0, st>>>(P);
    else k_g2p<false><<<blocks, threads, 0, st>>>(P);
}

void launch_pushout(const Params& P, cudaStream_t st) {
    k_pushout<<<grid_for(P.n_total, 256, 148 * 8), 256, 0, st>>>(P);
}

void launch_deactivate(const Params& P, cudaStream_t st) {
    k_deactivate<<<grid_for(P.n_total, 256, 148 * 8), 256, 0, st>>>(P);
}

void launch_free_bodies(const Params& P, bool integrate, bool merge, cudaStream_t st) {
    k_free_bodies<<<1, 128, 0, st>>>(P, integrate ? 1 : 0, merge ? 1 : 0);
}

void launch_grid_bc(const Params& P, int64_t max_bricks, cudaStream_t st) {
    const int threads = 256;
    k_grid_bc<<<grid_for(max_bricks * 64, threads, 148 * 8), threads, 0, st>>>(P);
}

}  // namespace mpmb
