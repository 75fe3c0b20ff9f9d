// k_transfer.cu — particle <-> grid transfers: P2G (K2 MLS / K5 PB-MPM) and G2P (K4 MLS /
// K6 PB-MPM, with the F update, push-out and deactivation fused), plus standalone push-out
// and deactivation for the solver-layer API.
//
// Work decomposition: one warp per GROUP of kGroup (256) consecutive slots.  The slots were
// ordered by (brick, cell) at the last binning (k_sort.cu), so a group covers a compact
// region; particles drift during a frame, so the group is RE-SORTED every substep inside
// P2G by its current stencil base: a warp counting sort over kBins shared-memory bins keyed
// by (brick low bits, cell).  Lane L then takes sorted positions [8L, 8L+8): runs of equal
// base are consecutive, whatever the drift since binning.  P2G stores the order (one byte
// per position) and G2P of the same substep replays it (x is unchanged in between).
//
// Latency hiding: each lane stages its particles' planes into shared memory with
// cp.async (LDGSTS) kStages-1 iterations ahead of use (per-lane ring, no cross-lane
// hazard), so HBM latency overlaps the arithmetic of the previous particles.
//
// P2G accumulates the 27 stencil nodes x {momentum, mass} in registers while the base
// stays the same (packed FP32x2 FMAs, FFMA2), then flushes with 27 red.global.add.v4.f32.
// G2P loads the 27 stencil velocities into registers once per base and reuses them.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "launch.h"

namespace mpmb {

// resident blocks per SM the register allocation targets (A/B-tuned)
#ifndef MPMB_P2G_MINB
#define MPMB_P2G_MINB 3
#endif
#ifndef MPMB_G2P_MINB
#define MPMB_G2P_MINB 3
#endif
#ifndef MPMB_P2G_STAGES
#define MPMB_P2G_STAGES 3
#endif
#ifndef MPMB_G2P_STAGES
#define MPMB_G2P_STAGES 3
#endif
constexpr int kStages = MPMB_P2G_STAGES;     // P2G staging ring depth (from HBM)
#ifndef MPMB_P2G_STAGES_L2
#define MPMB_P2G_STAGES_L2 2
#endif
// K8's P2G phase stages from L2 (the lines its G2P phase just wrote): a shallower ring hides
// that latency and leaves more of the SM's shared memory to L1 (A/B at C5: K8 -0.7%)
constexpr int kStagesL2 = MPMB_P2G_STAGES_L2;
// K8's MLS G2P phase evaluates the P2G's affine term (mls_affine below); its P2G phase then
// stages 5 planes instead of 7
#ifndef MPMB_K8_PREA
#define MPMB_K8_PREA 1
#endif
// K8's per-warp ring (float4 x 32 units): the G2P phase's and the P2G phase's, aliased
template <bool PB, bool STD>
__host__ __device__ constexpr int fused_ring() {
    return kStagesL2 * ((PB || STD || !MPMB_K8_PREA) ? 7 : 5) > MPMB_G2P_STAGES * ((PB || STD) ? 7 : 5)
               ? kStagesL2 * ((PB || STD || !MPMB_K8_PREA) ? 7 : 5)
               : MPMB_G2P_STAGES * ((PB || STD) ? 7 : 5);
}
constexpr int kG2PStages = MPMB_G2P_STAGES;  // G2P: one more, so particle k+1 has landed while k computes
#ifndef MPMB_WPB
#define MPMB_WPB 4  // A/B: 3 warps x 4 blocks per SM: C5 +0.5%, C1 +3%, but C2 -7%, C3 -3%
#endif
constexpr int kWarpsPerBlock = MPMB_WPB;
constexpr int kPer = kGroup / 32;  // sorted positions per lane
// G2P gathers from a per-warp shared-memory copy of the group's node box (the stencil-base
// box the P2G sort recorded, + 2 nodes per axis) when it has at most kBoxCap nodes
#ifndef MPMB_G2P_BOX
#define MPMB_G2P_BOX 1
#endif
#ifndef MPMB_BOX_CAP
#define MPMB_BOX_CAP 256
#endif
constexpr int kBoxCap = MPMB_G2P_BOX ? MPMB_BOX_CAP : 0;
// The box pays off while a launch has few groups per warp slot (latency-bound tail: the
// 874k-particle scene +4%); at C5 sizes its shared memory costs more than it saves (-1.3%,
// DESIGN.md §7), so launches with more groups than this use the plain gather.
#ifndef MPMB_BOX_MAX_GROUPS
#define MPMB_BOX_MAX_GROUPS (4 * 148 * MPMB_P2G_MINB * kWarpsPerBlock)
#endif
constexpr int64_t kBoxMaxGroupsBuild = MPMB_BOX_MAX_GROUPS;
// the launch-time bound (MPMB_BOX_MAX_GROUPS in the environment overrides it, for A/B; it
// never exceeds the build's, which sized nothing but is the tuned default)
static int64_t box_max_groups() {
    static const int64_t v = [] {
        const char* e = std::getenv("MPMB_BOX_MAX_GROUPS");
        return e ? std::min<int64_t>(std::atoll(e), kBoxMaxGroupsBuild) : kBoxMaxGroupsBuild;
    }();
    return v;
}
#define kBoxMaxGroups box_max_groups()
#ifndef MPMB_FUSED_NBIN
#define MPMB_FUSED_NBIN 1  // the fused kernel's sort reads bins its G2P phase left in shared memory
#endif
constexpr int kBins = 512;         // sort bins: ((global brick & 7) << 6) | cell
constexpr int kBinWords = kBins + kBins / 32;  // one pad word per 32 bins (conflict-free scan)
static_assert(kPer == 8, "order bytes are read as one u64 per lane");
// G2P position of lane L at iteration k.  LDGSTS costs one L1 wavefront per (8-lane phase,
// source line): lanes 8j..8j+7 take positions 64 b + 8 c + a (c = L & 7) that group_phys
// maps to ONE 128-byte line (8 (4a + b) + c), and the warp's 32 positions lie in a
// 64-position window of the sorted order (gather locality).  Increasing in k.
// (KP = 1, 32-position units: position = lane.)
template <int KP = 8>
__device__ __forceinline__ uint32_t g2p_pos(int lane, int k) {
    if (KP == 1) return static_cast<uint32_t>(lane);
    return 64u * (k >> 1) + 8u * (lane & 7) + 4u * (k & 1) + (lane >> 3);
}

// CG: bypass L1 (the staged particle stream would evict the grid lines G2P gathers)
template <bool CG>
__device__ __forceinline__ void cp_async16(float4* smem, const float4* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    if (CG) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
#ifndef MPMB_P2G_CG
#define MPMB_P2G_CG 0
#endif
#ifndef MPMB_G2P_CG
#define MPMB_G2P_CG 1  // A/B on C5: G2P -5%; P2G +1% with CG (its L1 holds nothing else)
#endif
// Warm L1 with the 9 stencil rows (3 nodes, 48 B: first and last node) of base b.
__device__ __forceinline__ void prefetch_stencil_l1(const float4* g, uint32_t px, uint32_t pxy) {
#pragma unroll
    for (int dk = 0; dk < 3; ++dk)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            const float4* row = g + (dk * pxy + dj * px);
            asm volatile("prefetch.global.L1 [%0];" ::"l"(row));
            asm volatile("prefetch.global.L1 [%0];" ::"l"(row + 2));
        }
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// Stage plane set: P2G and PB G2P read all 7 planes; MLS G2P reads x, F and flags only.
template <int NP>
struct PlaneSet;
template <>
struct PlaneSet<7> {
    __device__ static constexpr int plane(int q) { return q; }
};
template <>
struct PlaneSet<5> {  // P0 {x, vx}, P3 {C6..8, F0}, P4, P5 {F}, PR
    __device__ static constexpr int plane(int q) { return q == 0 ? 0 : (q == 4 ? PR : q + 2); }
};
template <>
struct PlaneSet<4> {  // (5 planes) P0 {x, vx}, P1 {vy, vz, A0, A1}, P2 {A2..5}, P3 {A6..8, F0}, PR
    __device__ static constexpr int plane(int q) { return q == 4 ? PR : q; }
};

// Per-lane producer of the staging ring: issues the planes of the lane's k-th sorted
// particle (lanes past their count commit an empty group, keeping the wait counts uniform).
template <int NP, int NS = kStages, bool CG = false, bool OUT = false, int PSET = NP>
struct Stager {
    float4* buf;        // this warp's ring: [NS][NP][32]
    uint32_t slot0;     // first slot of the group
    uint64_t order;     // the lane's 8 sorted particles, one slot-in-group byte each
    int cnt;            // how many of them exist
    int lane;
    __device__ __forceinline__ uint32_t slot(int k) const {
        return slot0 + static_cast<uint32_t>((order >> (8 * k)) & 0xFFu);
    }
    __device__ __forceinline__ void issue(const Params& P, int k) {
        if (k < cnt) {
            const uint32_t s = slot(k);
            MPMB_DCHECK(s < static_cast<uint64_t>(P.n_total));
            float4* dst = buf + (k % NS) * NP * 32 + lane;
#pragma unroll
            for (int q = 0; q < NP; ++q)
                cp_async16<CG>(dst + q * 32, (OUT ? P.pl_out : P.pl)[PlaneSet<PSET>::plane(q)] + s);
        }
        cp_commit();
    }
};

// =====================================================================  P2G
__device__ __forceinline__ void mark_bricks(const Params& P, const SceneView& S, const int cb[3]) {
    // ONE fire-and-forget red.or on the brick of the stencil base: bit 3 = touched, bit a =
    // the stencil crosses into the +a neighbour brick (base & 3 >= 2); k_collect_bricks
    // expands the marks to exactly the <= 8 bricks the stencils touch
    const uint32_t m = 8u | ((cb[0] & 3) >= 2 ? 1u : 0u) | ((cb[1] & 3) >= 2 ? 2u : 0u) | ((cb[2] & 3) >= 2 ? 4u : 0u);
    uint32_t* f = P.brick_flag + S.brick_base +
                  ((cb[2] >> 2) * S.nb[1] + (cb[1] >> 2)) * S.nb[0] + (cb[0] >> 2);
    asm volatile("red.global.or.b32 [%0], %1;" ::"l"(f), "r"(m) : "memory");
}

// red.global.add.v4.f32: the explicit state space keeps the 64-bit base + 32-bit offset
// addressing (a generic pointer would turn into a returning generic ATOM)
#ifndef MPMB_DEBUG_NO_RED
#define MPMB_DEBUG_NO_RED 0  // timing experiment only (wrong results): the flush REDs dropped
#endif
__device__ __forceinline__ void red_add_v4(float4* p, float2 a, float2 b, uint32_t debug = 0) {
    if (MPMB_DEBUG_NO_RED && debug) {
        if (a.x + a.y + b.x + b.y == 1.2345e30f) p->x = 0.f;
        return;
    }
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a.x), "f"(a.y), "f"(b.x),
                 "f"(b.y));
}

__device__ __forceinline__ void p2g_flush(const Params& P, const SceneView& S, const int cb[3],
                                          float2 (&pa)[27], float2 (&pb)[27]) {
    uint32_t base, px, pxy;
    stencil_rows(P.geo, cb, base, px, pxy);
    // one 64-bit stencil pointer; the 9 row offsets are warp-uniform byte counts (uniform
    // datapath), so each row costs one 64-bit add instead of an index-to-address chain
    MPMB_DCHECK(S.node_base + base + 2ull * (pxy + px) + 2 < P.total_nodes);
    MPMB_DCHECK(cb[0] >= 0 && cb[1] >= 0 && cb[2] >= 0);
    char* g = reinterpret_cast<char*>(P.grid_acc + S.node_base + base);
    const uint32_t pxb = px * 16u, pxyb = pxy * 16u;
    const float2 zero2 = f2(P.zero, P.zero);
#pragma unroll
    for (int dk = 0; dk < 3; ++dk)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            float4* row = reinterpret_cast<float4*>(g + (dk * pxyb + dj * pxb));
#pragma unroll
            for (int di = 0; di < 3; ++di) {
                const int n = (dk * 3 + dj) * 3 + di;
                red_add_v4(row + di, pa[n], pb[n], P.debug);
                pa[n] = __fmul2_rn(pa[n], zero2);  // one FFMA-pipe op per pair (a plain
                pb[n] = __fmul2_rn(pb[n], zero2);  // zero costs ptxas one MOV per register)
            }
        }
    mark_bricks(P, S, cb);
}

// The 27 node contributions of one particle (solvers.hpp:157-168):
//   momentum += w (m v + A (x_I - x_p)),  mass += w m,  w = w_x w_y w_z.
// With u_jk = m v + A_col1 r_y + A_col2 r_z:  w (m v + A r) = w_x (w_yz u_jk) + (w_x r_x)(w_yz A_col0),
// so each node costs two packed FFMA2 per pair with per-particle scalar broadcasts.
// Pairs: (mom_x, mom_y) and (mom_z, mass) -- the .y lane of the second carries m through
// u and 0 through A.
__device__ __forceinline__ void p2g_nodes(const float w[3][3], const float rel[3][3], const float A[9],
                                          float m, const float v[3], float2 (&pa)[27], float2 (&pb)[27]) {
    const float2 A01_0 = f2(A[0], A[3]), A2m_0 = f2(A[6], 0.f);
    const float2 A01_1 = f2(A[1], A[4]), A2m_1 = f2(A[7], 0.f);
    const float2 A01_2 = f2(A[2], A[5]), A2m_2 = f2(A[8], 0.f);
    const float2 mv01 = f2(v[0] * m, v[1] * m), mv2m = f2(v[2] * m, m);
    float wr0[3];
#pragma unroll
    for (int di = 0; di < 3; ++di) wr0[di] = w[0][di] * rel[0][di];
#pragma unroll
    for (int dk = 0; dk < 3; ++dk) {
        const float rz = rel[2][dk];
        const float2 uz01 = __ffma2_rn(A01_2, f2(rz, rz), mv01);
        const float2 uz2m = __ffma2_rn(A2m_2, f2(rz, rz), mv2m);
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            const float ry = rel[1][dj];
            const float wyz = w[1][dj] * w[2][dk];
            const float2 U01 = __fmul2_rn(__ffma2_rn(A01_1, f2(ry, ry), uz01), f2(wyz, wyz));
            const float2 U2m = __fmul2_rn(__ffma2_rn(A2m_1, f2(ry, ry), uz2m), f2(wyz, wyz));
            const float2 G01 = __fmul2_rn(A01_0, f2(wyz, wyz));
            const float2 G2m = __fmul2_rn(A2m_0, f2(wyz, wyz));
#pragma unroll
            for (int di = 0; di < 3; ++di) {
                const int n = (dk * 3 + dj) * 3 + di;
                const float wx = w[0][di], wr = wr0[di];
                pa[n] = __ffma2_rn(f2(wx, wx), U01, pa[n]);
                pa[n] = __ffma2_rn(f2(wr, wr), G01, pa[n]);
                pb[n] = __ffma2_rn(f2(wx, wx), U2m, pb[n]);  // .y: mass += w m
                pb[n] = __ffma2_rn(f2(wr, wr), G2m, pb[n]);
            }
        }
    }
}

// Standard MPM (solvers.hpp:96-103): momentum += v (w m) + M grad w, mass += w m, with the
// impulse matrix M = -dt V sigma and grad w = (dw_x w_y w_z, w_x dw_y w_z, w_x w_y dw_z).
// Per row (dj, dk): a = w_y w_z, b = dw_y w_z, c = w_y dw_z, U = m v a + M_col1 b + M_col2 c,
// G = M_col0 a; per node: w_x U + dw_x G -- the FFMA2 shape of p2g_nodes.
__device__ __forceinline__ void p2g_nodes_std(const float w[3][3], const float dw[3][3], const float M[9], float m,
                                              const float v[3], float2 (&pa)[27], float2 (&pb)[27]) {
    const float2 M0_01 = f2(M[0], M[3]), M0_2m = f2(M[6], 0.f);
    const float2 M1_01 = f2(M[1], M[4]), M1_2m = f2(M[7], 0.f);
    const float2 M2_01 = f2(M[2], M[5]), M2_2m = f2(M[8], 0.f);
    const float2 mv01 = f2(v[0] * m, v[1] * m), mv2m = f2(v[2] * m, m);
#pragma unroll
    for (int dk = 0; dk < 3; ++dk)
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            const float a = w[1][dj] * w[2][dk], b = dw[1][dj] * w[2][dk], c = w[1][dj] * dw[2][dk];
            const float2 U01 = __ffma2_rn(M2_01, f2(c, c), __ffma2_rn(M1_01, f2(b, b), __fmul2_rn(mv01, f2(a, a))));
            const float2 U2m = __ffma2_rn(M2_2m, f2(c, c), __ffma2_rn(M1_2m, f2(b, b), __fmul2_rn(mv2m, f2(a, a))));
            const float2 G01 = __fmul2_rn(M0_01, f2(a, a));
            const float2 G2m = __fmul2_rn(M0_2m, f2(a, a));
#pragma unroll
            for (int di = 0; di < 3; ++di) {
                const int n = (dk * 3 + dj) * 3 + di;
                const float wx = w[0][di], dx = dw[0][di];
                pa[n] = __ffma2_rn(f2(wx, wx), U01, pa[n]);
                pa[n] = __ffma2_rn(f2(dx, dx), G01, pa[n]);
                pb[n] = __ffma2_rn(f2(wx, wx), U2m, pb[n]);  // .y: mass += w m
                pb[n] = __ffma2_rn(f2(dx, dx), G2m, pb[n]);
            }
        }
}

// node_position(base + o) - x (state.hpp:49-51) along one axis with one int-to-float
// conversion per axis: the first node as the reference computes it, the next two by adding
// dx.  NOT used (MPMB_NODE_REL 0, measured): every node must sit where the reference puts
// it, origin + i dx rounded once per node.  origin + b dx + dx rounds differently (by
// ~ulp(x)) and the difference is the same for every particle of a cell, so it biases the
// affine transfer: the blade-engaged C5 replicas moved 3-8x farther from the oracle
// (x 8.6e-5 vs 2.5e-5 dx, blade impulse 1.6e-5 vs 1.9e-6 in 100 substeps).  Deriving all
// three from the fractional coordinate, (o - fx) dx, was worse still (C1: 1e-3 dx in 300
// substeps).  Both were ~1.3 % faster at C5.
#ifndef MPMB_NODE_REL
#define MPMB_NODE_REL 0
#endif
__device__ __forceinline__ void node_rel(const Geo& G, int a, int b, float x, float dx, float rel[3]) {
    rel[0] = node_coord(G, a, b) - x;
    rel[1] = rel[0] + dx;
    rel[2] = rel[1] + dx;
}

// quadratic B-spline weight derivatives (math.hpp:229-231)
__device__ __forceinline__ void bspline_dw(float fx, float inv_dx, float dw[3]) {
    dw[0] = (fx - 1.5f) * inv_dx;
    dw[1] = -2.f * (fx - 1.f) * inv_dx;
    dw[2] = (fx - 0.5f) * inv_dx;
}

// Active-brick list from the P2G marks (collect_bricks_body, kernels.cuh).
__global__ void __launch_bounds__(256) k_collect_bricks(const Params P, uint32_t n_bricks) {
    pdl_enter();
    collect_bricks_body(P, n_bricks, blockIdx.x, gridDim.x);
}

void launch_collect_bricks(const Params& P, uint32_t n_bricks, cudaStream_t st) {
    int64_t blocks = (static_cast<int64_t>(n_bricks) + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    launch_chain(k_collect_bricks, static_cast<int>(blocks), 256, 0, st, P, n_bricks);
}

__device__ __forceinline__ uint32_t bin_word(uint32_t b) { return b + (b >> 5); }

// Warp counting sort of group g by current stencil base, STABLE in the previous order:
// element (i, lane) is the particle of previous sorted position p = 32 i + lane (slot
// g*kGroup + group_phys(p)), and equal bins are ranked in (i, lane) order (warp-aggregated
// smem atomics).  Active particles come first in bin order, then inactive ones and holes
// in previous order.  Writes all kGroup order bytes (slot-in-group of each position) to
// order_s and returns the lane's 8 P2G positions [8L, 8L+8); `bins` is kBinWords words.
// nbin (fused kernel, !BOX): the bin of every previous position, computed by this warp's G2P
// phase from the new positions (0xFFFF: inactive or hole), so the sort reads shared memory
// instead of re-loading x and the flags from L2.
// the sort bin of a stencil base b of `scene`: ((global brick & 7) << 6) | cell in brick
__device__ __forceinline__ uint32_t sort_bin(const Params& P, int scene, const int b[3]) {
    const uint32_t brick = static_cast<uint32_t>(scene) * P.geo.bricks_per_scene +
                           (static_cast<uint32_t>(b[2] >> 2) * P.geo.nb[1] + static_cast<uint32_t>(b[1] >> 2)) *
                               P.geo.nb[0] +
                           static_cast<uint32_t>(b[0] >> 2);
    return ((brick & 7u) << 6) | static_cast<uint32_t>(((b[2] & 3) << 4) | ((b[1] & 3) << 2) | (b[0] & 3));
}

// KP = sorted positions per lane: 8 (the whole 256-slot group per warp) or 2 (one of its 4
// 64-position units per warp, `unit` = s of 0..3; small problems: 4x the warps).  A unit's
// positions [P0, P0 + 32 KP) map to a fixed quarter of the group's slots, so units never
// exchange particles and their sorts are independent.
// dead (optional): bit l set when 128-byte line l of the group's slots (slots 8l..8l+7) holds
// a slot that is inactive or a hole (k8_discard).
template <bool OUT, bool BOX, int KP = kPer>
__device__ __forceinline__ uint64_t group_sort(const Params& P, uint32_t g, uint32_t unit, uint32_t* bins,
                                               uint8_t* order_s, uint32_t& n_act, const uint16_t* nbin = nullptr,
                                               uint32_t* dead = nullptr, int4* box_out = nullptr) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt = lanemask_lt();
    const uint32_t slot0 = g * kGroup;
    const uint32_t p0 = unit * 32u * KP;  // first position of the unit
    uint32_t bin[KP];
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    int sc_lo = INT_MAX, sc_hi = INT_MIN;
    if (!BOX && nbin) {
#pragma unroll
        for (int i = 0; i < KP; ++i) {
            const uint32_t b = nbin[32 * i + lane];
            bin[i] = b == 0xFFFFu ? 0xFFFFFFFFu : b;
        }
    } else {
    // all 16 loads first: one memory latency per group
    float4 xa4[KP];
    uint32_t fl[KP];
#pragma unroll
    for (int i = 0; i < KP; ++i) {
        const uint32_t s = slot0 + group_phys(p0 + 32u * i + lane);
        MPMB_DCHECK(s < static_cast<uint64_t>(P.n_total));
        if (OUT) {  // written earlier in this kernel by the same warp: coherent L2 loads
            fl[i] = __float_as_uint(__ldcg(&P.pl_out[PR][s].z));
            xa4[i] = __ldcg(&P.pl_out[0][s]);
        } else {
            fl[i] = __float_as_uint(__ldg(&P.pl[PR][s].z));
            xa4[i] = __ldg(&P.pl[0][s]);
        }
    }
#pragma unroll
    for (int i = 0; i < KP; ++i) {
        bin[i] = 0xFFFFFFFFu;
        const uint32_t flags = fl[i];
        if (flags & kActiveBit) {
            const float4 a = xa4[i];
            const int scene = static_cast<int>((flags >> kSceneShift) & kSceneMask);
            const float xa[3] = {a.x, a.y, a.z};
            int b[3];
            float fx[3];
            local_base(P.geo, xa, b, fx);
            bin[i] = sort_bin(P, scene, b);
            if (BOX) {
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    lo[a] = min(lo[a], b[a]);
                    hi[a] = max(hi[a], b[a]);
                }
                sc_lo = min(sc_lo, scene);
                sc_hi = max(sc_hi, scene);
            }
        }
    }
    }
    if (BOX) {  // the group's stencil-base box for the G2P of this substep (same x, same bases)
        int4 bx;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int l = __reduce_min_sync(full, lo[a]), h = __reduce_max_sync(full, hi[a]);
            (a == 0 ? bx.x : a == 1 ? bx.y : bx.z) = l | (h << 16);
        }
        const int s0 = __reduce_min_sync(full, sc_lo), s1 = __reduce_max_sync(full, sc_hi);
        bx.w = (s0 == s1) ? s0 : -1;  // empty or several scenes: no box
        if (lane == 0) P.group_box[g * (kPer / KP) + unit] = bx;
        if (box_out) *box_out = bx;
    }
    if (dead) {  // slot group_phys(p) lies in line (p & 7) * 4 + (p >> 6)
        uint32_t m = 0;
#pragma unroll
        for (int i = 0; i < KP; ++i)
            if (bin[i] == 0xFFFFFFFFu) m |= 1u << (((lane & 7) << 2) | ((p0 + 32u * i + lane) >> 6));
        *dead = __reduce_or_sync(full, m);
    }
    for (int w = lane; w < kBinWords; w += 32) bins[w] = 0u;
    __syncwarp();
    uint32_t rank[KP];
    uint32_t n_inact = 0;
#pragma unroll
    for (int i = 0; i < KP; ++i) {
        const unsigned peers = __match_any_sync(full, bin[i]);
        const int lead = __ffs(peers) - 1;
        const unsigned inact = __ballot_sync(full, bin[i] == 0xFFFFFFFFu);
        uint32_t base = 0;
        if (bin[i] != 0xFFFFFFFFu && lane == lead) base = atomicAdd(&bins[bin_word(bin[i])], __popc(peers));
        base = __shfl_sync(full, base, lead);
        rank[i] = bin[i] != 0xFFFFFFFFu ? base + __popc(peers & lt) : n_inact + __popc(inact & lt);
        n_inact += __popc(inact);
    }
    __syncwarp();
    // exclusive scan over bins in index order: lane L owns bins [16L, 16L+16)
    constexpr int kOwn = kBins / 32;
    uint32_t c[kOwn];
    uint32_t tot = 0;
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
        c[j] = bins[bin_word(kOwn * lane + j)];
        tot += c[j];
    }
    uint32_t inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(full, inc, o);
        if (lane >= o) inc += t;
    }
    n_act = __shfl_sync(full, inc, 31);
    uint32_t run = inc - tot;
#pragma unroll
    for (int j = 0; j < kOwn; ++j) {
        bins[bin_word(kOwn * lane + j)] = run;
        run += c[j];
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < KP; ++i) {
        const uint32_t pos = bin[i] != 0xFFFFFFFFu ? bins[bin_word(bin[i])] + rank[i] : n_act + rank[i];
        MPMB_DCHECK(pos < 32u * KP && (bin[i] == 0xFFFFFFFFu || bin[i] < static_cast<uint32_t>(kBins)));
        order_s[pos] = static_cast<uint8_t>(group_phys(p0 + 32u * i + lane));
    }
    __syncwarp();
    uint64_t mine;
    if (KP == 8) mine = reinterpret_cast<const uint64_t*>(order_s)[lane];
    else if (KP == 4) mine = reinterpret_cast<const uint32_t*>(order_s)[lane];
    else if (KP == 2) mine = reinterpret_cast<const uint16_t*>(order_s)[lane];
    else mine = order_s[lane];
    __syncwarp();  // the caller reuses this shared memory for staging
    return mine;
}

// MLS affine momentum term A = m C - dt V (4/dx^2) sigma(F), V = det(F) V0 (solvers.hpp:154-156)
__device__ __forceinline__ void mls_affine(const Params& P, const float Cm[9], const float F[9], float m, float vol0,
                                           uint32_t flags, float m_inv, float A[9]) {
    float sig[9];
    const float4 mat = material(P, flags & kMatMask);
    const float J = neo_hookean_f32(F, mat.y, mat.z, sig);
    const float sc = -P.dt * (J * vol0) * m_inv;
#pragma unroll
    for (int i = 0; i < 9; ++i) A[i] = fmaf(Cm[i], m, sig[i] * sc);
}

// Inside a frame the fused kernel's G2P phase evaluates A for the P2G phase that follows
// (MPMB_K8_PREA): it has the new C and F in registers, writes A in C's planes (P1..P3) and the
// P2G phase stages 5 planes instead of 7 and skips the stress.  The next G2P recomputes C
// from the grid and never reads the old one; particles that leave the active set keep C, and
// the frame's last G2P (unfused) stores C.  A/B on the engaged C5 window: K8 -2.8 %, C5
// +2.2 %, M1 +1.5 %, C2 +1 %; the GPU parity suite unchanged.  (MPMB_K8_PREA: top of file.)

// One particle's P2G inputs (solvers.hpp:151-169 / 88-104 / 218-235) from its 7 planes:
// scene, stencil base b, weights w, rel = node - x (STD: the weight derivatives), the
// affine / impulse matrix A, mass m and velocity v.
template <bool MLS, bool STD, bool PREA = false>
__device__ __forceinline__ void p2g_prepare(const Params& P, const float4 q0, const float4 q1, const float4 q2,
                                            const float4 q3, const float4 q4, const float4 q5, const float4 r,
                                            int& scene, int b[3], float w[3][3], float rel[3][3], float A[9],
                                            float& m, float v[3]) {
    const uint32_t flags = __float_as_uint(r.z);
    const float x[3] = {q0.x, q0.y, q0.z};
    v[0] = q0.w; v[1] = q1.x; v[2] = q1.y;
    const float Cm[9] = {q1.z, q1.w, q2.x, q2.y, q2.z, q2.w, q3.x, q3.y, q3.z};
    scene = static_cast<int>((flags >> kSceneShift) & kSceneMask);
    const SceneView S = scene_view(P, scene);
    float fx[3];
    local_base(P.geo, x, b, fx);
    m = r.x;
    // affine = m C - dt V (4/dx^2) sigma  (solvers.hpp:154-156; PB: m C, :222)
    if (PREA) {  // evaluated by the fused kernel's G2P phase (mls_affine)
#pragma unroll
        for (int i = 0; i < 9; ++i) A[i] = Cm[i];
    } else if (MLS) {
        const float F[9] = {q3.w, q4.x, q4.y, q4.z, q4.w, q5.x, q5.y, q5.z, q5.w};
        float sig[9];
        float J;  // det F (solvers.hpp:154)
        if (P.use_stress_in) {  // explicitly uploaded stress cache (solvers.hpp:156)
            const float* s9 = P.stress_in + 9ull * __float_as_uint(r.w);
#pragma unroll
            for (int i = 0; i < 9; ++i) sig[i] = s9[i];
            J = det3(F);
        } else {  // cached stress == sigma(F) of the last G2P (solvers.hpp:69-74)
            const float4 mat = material(P, flags & kMatMask);
            J = neo_hookean_f32(F, mat.y, mat.z, sig);
        }
        if (STD) {  // impulse_m = sigma (-dt V), V = det(F) V0 (solvers.hpp:91-92)
            const float sc = -P.dt * (J * r.y);
#pragma unroll
            for (int i = 0; i < 9; ++i) A[i] = sig[i] * sc;
        } else {
            const float sc = -P.dt * (J * r.y) * S.m_inv;
#pragma unroll
            for (int i = 0; i < 9; ++i) A[i] = fmaf(Cm[i], m, sig[i] * sc);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 9; ++i) A[i] = Cm[i] * m;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        bspline_w(fx[a], w[a]);
        if (STD) {
            bspline_dw(fx[a], S.inv_dx, rel[a]);
        } else {
            if (MPMB_NODE_REL) {
                node_rel(P.geo, a, b[a], x[a], S.dx, rel[a]);
            } else {
#pragma unroll
                for (int o = 0; o < 3; ++o) rel[a][o] = node_coord(P.geo, a, b[a] + o) - x[a];
            }
        }
    }
}

// P2G of group g (MLS: stress impulse from F, solvers.hpp:151-169; with STD: standard MPM's
// force transfer, solvers.hpp:88-104; !MLS: PB-MPM, A = m C, solvers.hpp:218-235).  `ring` is
// this warp's staging ring (kStages x kPlanes x 32 float4), also the sort scratch.  OUT: the
// group's particles are in the other buffer (pl_out), written by this warp's G2P of the
// previous substep inside the fused kernel (k_g2p2g).
// Inside a frame the fused kernel's P2G phase is the last reader of planes P1 {v.y, v.z, C0, C1}
// and P2 {C2..C5} of the buffer its G2P phase wrote: the next G2P (MLS) reads x, F and the
// flags only and recomputes v and C from the grid.  So once the group is consumed its P1 / P2
// lines are dropped from L2 without a write-back (discard.global.L2), except lines holding an
// inactive slot or a hole (copied with all planes by the next G2P).  Units of 64 and 128
// positions own whole lines; 32-position units share them and keep theirs.  Measured (A/B,
// engaged C5 window): K8 -0.9 % (the CCTL per line costs more than the saved write-backs:
// K8 is not HBM-bound), M1 / C2 neutral; off.
#ifndef MPMB_K8_DISCARD
#define MPMB_K8_DISCARD 0
#endif
template <int KP>
__device__ __forceinline__ void k8_discard(const Params& P, uint32_t g, uint32_t unit, uint32_t dead, int lane) {
    const uint32_t p0 = unit * 32u * KP;
    const uint32_t lo = p0 >> 6, hi = (p0 + 32u * KP - 1u) >> 6;
    const uint32_t mine = (((1u << (hi - lo + 1u)) - 1u) << lo) * 0x11111111u;  // lines (c, lo..hi)
    if ((mine & ~dead) >> lane & 1u) {
        const uint64_t s = static_cast<uint64_t>(g) * kGroup + 8u * static_cast<uint32_t>(lane);
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(P.pl_out[1] + s) : "memory");
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(P.pl_out[2] + s) : "memory");
    }
}

// ---- P2G into a per-warp shared-memory node tile (MPMB_P2G_TILE, fused MLS kernel).
// The tile covers the group's stencil-base box + 2 nodes per axis (at most kTileCap nodes;
// larger boxes and groups spanning scenes keep the global REDs).  A lane's run of equal base
// is still summed in registers; its flush adds the 27 nodes into the tile instead of 27
// global REDs, and the tile goes to the grid once per group, one 16-byte RED per non-zero
// node.  Lanes flushing at the same time may share nodes (neighbouring bases): the warp adds
// node by node in program order (volatile shared accesses, the warp converged), so one lane's
// store precedes another's load of the same node; lanes flushing the SAME base add in turns.
#ifndef MPMB_P2G_TILE
#define MPMB_P2G_TILE 0
#endif
#ifndef MPMB_TILE_CAP
#define MPMB_TILE_CAP 256
#endif
constexpr int kTileCap = MPMB_P2G_TILE ? MPMB_TILE_CAP : 0;
static_assert(kBoxCap == 0 || kTileCap <= kBoxCap, "the BOX kernels keep the tile in the G2P box");
struct NodeTile {
    uint32_t s;        // shared address of this warp's tile (0: global REDs)
    int nx, nxy;       // x pitch, xy pitch
    int korg;          // tile index of base (0, 0, 0): o_z nxy + o_y nx + o_x
};
struct TileBox {       // the box decoded: origin, extent, scene (-1: no tile)
    int o[3], n[3], scene;
};
__device__ __forceinline__ TileBox tile_box(int4 bx) {
    TileBox t;
    t.o[0] = bx.x & 0xFFFF; t.o[1] = bx.y & 0xFFFF; t.o[2] = bx.z & 0xFFFF;
    t.n[0] = (bx.x >> 16) - t.o[0] + 3; t.n[1] = (bx.y >> 16) - t.o[1] + 3; t.n[2] = (bx.z >> 16) - t.o[2] + 3;
    t.scene = (bx.w >= 0 && t.n[0] * t.n[1] * t.n[2] <= kTileCap) ? bx.w : -1;
    return t;
}
// zeroes the tile of box bx (warp-uniform); .s = 0 when the box does not fit
__device__ __forceinline__ NodeTile tile_open(float4* s, int4 bx, int lane) {
    NodeTile t{0u, 0, 0, 0};
    if (s == nullptr) return t;
    const TileBox B = tile_box(bx);
    if (B.scene < 0) return t;
    t.s = static_cast<uint32_t>(__cvta_generic_to_shared(s));
    t.nx = B.n[0]; t.nxy = B.n[0] * B.n[1];
    t.korg = B.o[2] * t.nxy + B.o[1] * t.nx + B.o[0];
    const int n = t.nxy * B.n[2];
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int i = lane; i < n; i += 32) s[i] = z;
    __syncwarp();
    return t;
}
// called by the whole warp; lanes with fl set add their run (tile index key of its base)
__device__ __forceinline__ void tile_flush(const Params& P, const NodeTile& T, bool fl, int key,
                                           float2 (&pa)[27], float2 (&pb)[27], int lane) {
    const unsigned full = 0xffffffffu;
    const int k = fl ? key : -1 - lane;
    const unsigned peers = __match_any_sync(full, k);
    const int rank = __popc(peers & lanemask_lt());
    const int nr = __reduce_max_sync(full, fl ? rank : 0);
    for (int r = 0; r <= nr; ++r) {
        const bool act = fl && rank == r;
        const uint32_t a0 = T.s + 16u * static_cast<uint32_t>(act ? key : 0);
#pragma unroll
        for (int dk = 0; dk < 3; ++dk)
#pragma unroll
            for (int dj = 0; dj < 3; ++dj) {
                const uint32_t ar = a0 + 16u * static_cast<uint32_t>(dk * T.nxy + dj * T.nx);
#pragma unroll
                for (int di = 0; di < 3; ++di) {
                    const int n = (dk * 3 + dj) * 3 + di;
                    if (act) {
                        float4 v;
                        asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                                     : "r"(ar + 16u * di)
                                     : "memory");
                        v.x += pa[n].x; v.y += pa[n].y; v.z += pb[n].x; v.w += pb[n].y;
                        asm volatile("st.volatile.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ar + 16u * di), "f"(v.x),
                                     "f"(v.y), "f"(v.z), "f"(v.w)
                                     : "memory");
                    }
                }
            }
    }
    if (fl) {
        const float2 zero2 = f2(P.zero, P.zero);
#pragma unroll
        for (int n = 0; n < 27; ++n) {
            pa[n] = __fmul2_rn(pa[n], zero2);
            pb[n] = __fmul2_rn(pb[n], zero2);
        }
    }
}
// the tile to the grid (after the warp's last tile_flush): one 16-byte RED per non-zero node,
// and the brick of every such node marked touched (k_collect_bricks: bit 3 alone marks the
// brick itself)
__device__ __forceinline__ void tile_close(const Params& P, int4 bx, const float4* s, int lane) {
    __syncwarp();
    const TileBox B = tile_box(bx);
    const SceneView S = scene_view(P, B.scene);
    float4* g = P.grid_acc + S.node_base;
    const int nxy = B.n[0] * B.n[1], n = nxy * B.n[2];
    for (int i = lane; i < n; i += 32) {
        const float4 v = s[i];
        if (v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f) {
            const int z = B.o[2] + i / nxy, rem = i % nxy, y = B.o[1] + rem / B.n[0], x = B.o[0] + rem % B.n[0];
            const uint32_t nd = node_linear(P.geo, x, y, z);
            MPMB_DCHECK(S.node_base + nd < P.total_nodes);
            red_add_v4(g + nd, f2(v.x, v.y), f2(v.z, v.w));
            uint32_t* f = P.brick_flag + S.brick_base + ((z >> 2) * S.nb[1] + (y >> 2)) * S.nb[0] + (x >> 2);
            asm volatile("red.global.or.b32 [%0], %1;" ::"l"(f), "r"(8u) : "memory");
        }
    }
    __syncwarp();
}

template <bool MLS, bool STD, bool OUT, bool BOX, int KP = kPer>
__device__ __forceinline__ void p2g_group(const Params& P, uint32_t g, uint32_t unit, float4* ring, int lane,
                                          const uint16_t* nbin = nullptr, float4* tile_s = nullptr,
                                          int4 tbox = make_int4(0, 0, 0, -1)) {
    constexpr bool DISCARD = MPMB_K8_DISCARD && OUT && MLS && !STD && KP >= 2;
    constexpr bool TILE = MPMB_P2G_TILE && OUT && MLS && !STD;
    // the fused kernel's G2P phase left A in C's planes (mls_affine): 5 planes staged
    constexpr bool PREA = MPMB_K8_PREA && OUT && MLS && !STD;
    constexpr int NP = PREA ? 5 : kPlanes;
    constexpr int RI = PREA ? 4 : PR;  // ring index of the PR plane
    constexpr int NS = OUT ? kStagesL2 : kStages;
    Stager<NP, NS, OUT || MPMB_P2G_CG != 0, OUT, PREA ? 4 : NP> st;
    st.buf = ring;
    st.lane = lane;
    uint32_t* bins = reinterpret_cast<uint32_t*>(ring);  // sort scratch aliases the ring
    uint8_t* order_s = reinterpret_cast<uint8_t*>(bins + kBinWords);
    uint32_t n_act, dead = 0;
    st.order = group_sort<OUT, BOX, KP>(P, g, unit, bins, order_s, n_act, nbin, DISCARD ? &dead : nullptr,
                                        (TILE && BOX) ? &tbox : nullptr);
    if (TILE && !BOX && nbin) {  // group_sort is done with the bins: keep the box there
        if (lane == 0) *reinterpret_cast<int4*>(const_cast<uint16_t*>(nbin)) = tbox;
        __syncwarp();
    }
    st.slot0 = g * kGroup;
    st.cnt = min(max(static_cast<int>(n_act) - KP * lane, 0), KP);
    if (KP == 8)
        reinterpret_cast<uint64_t*>(P.order)[static_cast<uint64_t>(g) * 32 + lane] = st.order;
    else if (KP == 4)  // the unit's 128 order bytes at [P0, P0 + 128) of the group's 256
        reinterpret_cast<uint32_t*>(P.order)[static_cast<uint64_t>(g) * 64 + unit * 32 + lane] =
            static_cast<uint32_t>(st.order);
    else if (KP == 2)  // the unit's 64 order bytes at [P0, P0 + 64)
        reinterpret_cast<uint16_t*>(P.order)[static_cast<uint64_t>(g) * 128 + unit * 32 + lane] =
            static_cast<uint16_t>(st.order);
    else  // KP = 1: the unit's 32 order bytes at [P0, P0 + 32)
        P.order[static_cast<uint64_t>(g) * kGroup + unit * 32 + lane] = static_cast<uint8_t>(st.order);
    if (lane == 0) P.group_nact[g * (kPer / KP) + unit] = n_act;
    const int kmax = min(static_cast<int>(n_act), KP);  // lane 0 has the most
    for (int k = 0; k < NS - 1; ++k) st.issue(P, k);
    float2 pa[27], pb[27];  // (mom_x, mom_y), (mom_z, mass) per stencil node
#pragma unroll
    for (int n = 0; n < 27; ++n) {
        pa[n] = f2(0.f, 0.f);
        pb[n] = f2(0.f, 0.f);
    }
    int cb[3] = {INT_MIN, INT_MIN, INT_MIN};
    int cscene = -1;
    if (TILE) {
        const NodeTile T = tile_open(tile_s, tbox, lane);
        if (T.s) {
            int ckey = -1;  // tile index of the current run's base (one scene per tile)
            for (int k = 0; k < kmax; ++k) {
                st.issue(P, k + NS - 1);
                cp_wait<NS - 1>();
                const bool live = k < st.cnt;
                const float4* src = st.buf + (k % NS) * NP * 32 + lane;
                // the base first: the flush runs with only the accumulators live
                int key = -1;
                if (live) {
                    const float4 q0 = src[0];
                    const float xa[3] = {q0.x, q0.y, q0.z};
                    int b[3];
                    float fx[3];
                    local_base(P.geo, xa, b, fx);
                    key = b[2] * T.nxy + b[1] * T.nx + b[0] - T.korg;
                    MPMB_DCHECK(key >= 0 && key + 2 * (T.nxy + T.nx) + 2 < kTileCap);
                }
                const bool change = live && key != ckey;
                const bool fl = change && ckey >= 0;
                if (__any_sync(0xffffffffu, fl)) tile_flush(P, T, fl, ckey, pa, pb, lane);
                if (change) ckey = key;
                if (live) {
                    const float4 r = src[RI * 32];
                    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
                    const float4 q0 = src[0], q1 = src[32], q2 = src[64], q3 = src[96],
                                 q4 = PREA ? z4 : src[128], q5 = PREA ? z4 : src[160];
                    int scene, b[3];
                    float w[3][3], rel[3][3], A[9], m, v[3];
                    p2g_prepare<MLS, STD, PREA>(P, q0, q1, q2, q3, q4, q5, r, scene, b, w, rel, A, m, v);
                    p2g_nodes(w, rel, A, m, v, pa, pb);
                }
            }
            const bool fl = ckey >= 0;
            if (__any_sync(0xffffffffu, fl)) tile_flush(P, T, fl, ckey, pa, pb, lane);
            cp_wait<0>();
            __syncwarp();
            // the box again (not kept live across the loop): the sort recorded it (BOX), or the
            // G2P phase's box is in the bins' shared memory, free since the sort
            const int4 bx = BOX ? __ldcg(&P.group_box[g * (kPer / KP) + unit])
                                : *reinterpret_cast<const int4*>(nbin);
            tile_close(P, bx, tile_s, lane);
            return;
        }
    }
    for (int k = 0; k < kmax; ++k) {
        st.issue(P, k + NS - 1);
        cp_wait<NS - 1>();
        if (k >= st.cnt) continue;
        const float4* src = st.buf + (k % NS) * NP * 32 + lane;
        const float4 r = src[RI * 32];
        const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 q0 = src[0], q1 = src[32], q2 = src[64], q3 = src[96], q4 = PREA ? z4 : src[128],
                     q5 = PREA ? z4 : src[160];
        int scene, b[3];
        float w[3][3], rel[3][3], A[9], m, v[3];  // STD: rel holds the weight derivatives
        p2g_prepare<MLS, STD, PREA>(P, q0, q1, q2, q3, q4, q5, r, scene, b, w, rel, A, m, v);
        if (b[0] != cb[0] || b[1] != cb[1] || b[2] != cb[2] || scene != cscene) {
            if (cscene >= 0) p2g_flush(P, scene_view(P, cscene), cb, pa, pb);
            cb[0] = b[0]; cb[1] = b[1]; cb[2] = b[2];
            cscene = scene;
        }
        if (STD) p2g_nodes_std(w, rel, A, m, v, pa, pb);
        else p2g_nodes(w, rel, A, m, v, pa, pb);
    }
    if (cscene >= 0) p2g_flush(P, scene_view(P, cscene), cb, pa, pb);
    cp_wait<0>();
    __syncwarp();  // the ring is the next group's sort scratch; every lane's staging has landed
    if (DISCARD) k8_discard<KP>(P, g, unit, dead, lane);
}

// BOX: record each group's stencil-base box for the (box-gathering) G2P that follows
// KP: positions per lane (group_sort): one warp per group (8) or per 64-position unit (2)
template <bool MLS, bool STD = false, bool BOX = false, int KP = kPer>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, MPMB_P2G_MINB) k_p2g(const __grid_constant__ Params P) {
    pdl_enter();
    extern __shared__ float4 smem[];
    const int lane = threadIdx.x & 31;
    constexpr uint32_t U = kPer / KP;  // units per group
    const uint32_t n_units = *P.n_groups * U;
    const uint32_t wpb = blockDim.x >> 5;
    float4* ring = smem + (threadIdx.x >> 5) * (kStages * kPlanes * 32);
    for (uint32_t u = blockIdx.x * wpb + (threadIdx.x >> 5); u < n_units; u += gridDim.x * wpb)
        p2g_group<MLS, STD, false, BOX, KP>(P, u / U, u % U, ring, lane);
}

// ================================================================  G2P
// grid_vel node = {v.x, v.y, v.z, mass}; nodes at or below kMassEps carry v = 0 (grid
// update), so they contribute nothing without a per-node test (solvers.hpp:186).
//
// v = sum w v_I,  B = sum (w v_I)(x_I - x_p)^T  (solvers.hpp:178-190), summed per row
// (dk, dj) over di with the x-weights, then scaled by w_y w_z.  The 27 nodes are read
// straight from L1: the warp's 32 lanes hold 32 consecutive sorted particles (a few
// stencil bases), so each load instruction touches only a handful of lines.
// GENERIC: plain (generic-address) loads, the node box may be in shared memory; else
// read-only global loads
#ifndef MPMB_G2P_PACK
#define MPMB_G2P_PACK 0
#endif
template <bool GENERIC>
__device__ __forceinline__ void g2p_gather(const float4* g, uint32_t px, uint32_t pxy, const float w[3][3],
                                           const float rel[3][3], float vn[3], float B[9]) {
    if (MPMB_G2P_PACK) {  // z components in FFMA2 pairs as well: (a2, b2), (v2, c0_2), (c1_2, c2_2)
        float2 wxr[3];
#pragma unroll
        for (int o = 0; o < 3; ++o) wxr[o] = f2(w[0][o], w[0][o] * rel[0][o]);
        float2 v01 = f2(0.f, 0.f), vz_c0 = f2(0.f, 0.f), c12_2 = f2(0.f, 0.f);
        float2 c0_01 = f2(0.f, 0.f), c1_01 = f2(0.f, 0.f), c2_01 = f2(0.f, 0.f);
#pragma unroll
        for (int dk = 0; dk < 3; ++dk) {
            float4 q[9];
#pragma unroll
            for (int n = 0; n < 9; ++n) {
                const float4* a = reinterpret_cast<const float4*>(reinterpret_cast<const char*>(g) +
                                                                  (dk * pxy + (n / 3) * px) * 16u) + (n % 3);
                q[n] = GENERIC ? *a : __ldg(a);
            }
#pragma unroll
            for (int dj = 0; dj < 3; ++dj) {
                float2 a01 = f2(0.f, 0.f), b01 = f2(0.f, 0.f), ab2 = f2(0.f, 0.f);  // ab2 = (a2, b2)
#pragma unroll
                for (int di = 0; di < 3; ++di) {
                    const float4 nq = q[dj * 3 + di];
                    a01 = __ffma2_rn(f2(wxr[di].x, wxr[di].x), f2(nq.x, nq.y), a01);
                    b01 = __ffma2_rn(f2(wxr[di].y, wxr[di].y), f2(nq.x, nq.y), b01);
                    ab2 = __ffma2_rn(wxr[di], f2(nq.z, nq.z), ab2);
                }
                const float wyz = w[1][dj] * w[2][dk];
                const float2 wyz_r = __fmul2_rn(f2(wyz, wyz), f2(rel[1][dj], rel[2][dk]));  // (wy, wz)
                v01 = __ffma2_rn(f2(wyz, wyz), a01, v01);
                vz_c0 = __ffma2_rn(f2(wyz, wyz), ab2, vz_c0);
                c0_01 = __ffma2_rn(f2(wyz, wyz), b01, c0_01);
                c1_01 = __ffma2_rn(f2(wyz_r.x, wyz_r.x), a01, c1_01);
                c2_01 = __ffma2_rn(f2(wyz_r.y, wyz_r.y), a01, c2_01);
                c12_2 = __ffma2_rn(wyz_r, f2(ab2.x, ab2.x), c12_2);
            }
        }
        vn[0] = v01.x; vn[1] = v01.y; vn[2] = vz_c0.x;
        B[0] = c0_01.x; B[1] = c1_01.x; B[2] = c2_01.x;
        B[3] = c0_01.y; B[4] = c1_01.y; B[5] = c2_01.y;
        B[6] = vz_c0.y; B[7] = c12_2.x; B[8] = c12_2.y;
        return;
    }
    float wr0[3];
#pragma unroll
    for (int o = 0; o < 3; ++o) wr0[o] = w[0][o] * rel[0][o];
    float2 v01 = f2(0.f, 0.f);
    float v2 = 0.f;
    float2 c0_01 = f2(0.f, 0.f), c1_01 = f2(0.f, 0.f), c2_01 = f2(0.f, 0.f);
    float c0_2 = 0.f, c1_2 = 0.f, c2_2 = 0.f;
#pragma unroll
    for (int dk = 0; dk < 3; ++dk) {
        float4 q[9];
#pragma unroll
        for (int n = 0; n < 9; ++n) {
            const float4* a = reinterpret_cast<const float4*>(reinterpret_cast<const char*>(g) +
                                                              (dk * pxy + (n / 3) * px) * 16u) + (n % 3);
            q[n] = GENERIC ? *a : __ldg(a);
        }
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            float2 a01 = f2(0.f, 0.f), b01 = f2(0.f, 0.f);
            float a2 = 0.f, b2 = 0.f;  // sum wx v_z, sum wx rx v_z
#pragma unroll
            for (int di = 0; di < 3; ++di) {
                const float4 nq = q[dj * 3 + di];
                const float wx = w[0][di], wr = wr0[di];
                a01 = __ffma2_rn(f2(wx, wx), f2(nq.x, nq.y), a01);
                b01 = __ffma2_rn(f2(wr, wr), f2(nq.x, nq.y), b01);
                a2 = fmaf(wx, nq.z, a2);
                b2 = fmaf(wr, nq.z, b2);
            }
            const float wyz = w[1][dj] * w[2][dk];
            const float wy = wyz * rel[1][dj], wz = wyz * rel[2][dk];
            v01 = __ffma2_rn(f2(wyz, wyz), a01, v01);
            v2 = fmaf(wyz, a2, v2);
            c0_01 = __ffma2_rn(f2(wyz, wyz), b01, c0_01);  // column 0: rel_x
            c0_2 = fmaf(wyz, b2, c0_2);
            c1_01 = __ffma2_rn(f2(wy, wy), a01, c1_01);    // column 1: rel_y
            c1_2 = fmaf(wy, a2, c1_2);
            c2_01 = __ffma2_rn(f2(wz, wz), a01, c2_01);    // column 2: rel_z
            c2_2 = fmaf(wz, a2, c2_2);
        }
    }
    vn[0] = v01.x; vn[1] = v01.y; vn[2] = v2;
    // B row r = velocity component r, column c = rel component c
    B[0] = c0_01.x; B[1] = c1_01.x; B[2] = c2_01.x;
    B[3] = c0_01.y; B[4] = c1_01.y; B[5] = c2_01.y;
    B[6] = c0_2;    B[7] = c1_2;    B[8] = c2_2;
}

// Standard MPM gather (solvers.hpp:112-128): v = sum w v_I, L = sum v_I (x) grad w, the
// same separable row sums as g2p_gather with dw_x in place of w_x r_x and the row factors
// (w_y w_z, dw_y w_z, w_y dw_z) for the three gradient columns.
template <bool GENERIC>
__device__ __forceinline__ void g2p_gather_std(const float4* g, uint32_t px, uint32_t pxy, const float w[3][3],
                                               const float dw[3][3], float vn[3], float L[9]) {
    float2 v01 = f2(0.f, 0.f);
    float v2 = 0.f;
    float2 c0_01 = f2(0.f, 0.f), c1_01 = f2(0.f, 0.f), c2_01 = f2(0.f, 0.f);
    float c0_2 = 0.f, c1_2 = 0.f, c2_2 = 0.f;
#pragma unroll
    for (int dk = 0; dk < 3; ++dk) {
        float4 q[9];
#pragma unroll
        for (int n = 0; n < 9; ++n) {
            const float4* a = reinterpret_cast<const float4*>(reinterpret_cast<const char*>(g) +
                                                              (dk * pxy + (n / 3) * px) * 16u) + (n % 3);
            q[n] = GENERIC ? *a : __ldg(a);
        }
#pragma unroll
        for (int dj = 0; dj < 3; ++dj) {
            float2 a01 = f2(0.f, 0.f), d01 = f2(0.f, 0.f);
            float a2 = 0.f, d2 = 0.f;
#pragma unroll
            for (int di = 0; di < 3; ++di) {
                const float4 nq = q[dj * 3 + di];
                const float wx = w[0][di], dx = dw[0][di];
                a01 = __ffma2_rn(f2(wx, wx), f2(nq.x, nq.y), a01);
                d01 = __ffma2_rn(f2(dx, dx), f2(nq.x, nq.y), d01);
                a2 = fmaf(wx, nq.z, a2);
                d2 = fmaf(dx, nq.z, d2);
            }
            const float wyz = w[1][dj] * w[2][dk];
            const float gy = dw[1][dj] * w[2][dk], gz = w[1][dj] * dw[2][dk];
            v01 = __ffma2_rn(f2(wyz, wyz), a01, v01);
            v2 = fmaf(wyz, a2, v2);
            c0_01 = __ffma2_rn(f2(wyz, wyz), d01, c0_01);  // column 0: dw_x w_y w_z
            c0_2 = fmaf(wyz, d2, c0_2);
            c1_01 = __ffma2_rn(f2(gy, gy), a01, c1_01);    // column 1: w_x dw_y w_z
            c1_2 = fmaf(gy, a2, c1_2);
            c2_01 = __ffma2_rn(f2(gz, gz), a01, c2_01);    // column 2: w_x w_y dw_z
            c2_2 = fmaf(gz, a2, c2_2);
        }
    }
    vn[0] = v01.x; vn[1] = v01.y; vn[2] = v2;
    L[0] = c0_01.x; L[1] = c1_01.x; L[2] = c2_01.x;
    L[3] = c0_01.y; L[4] = c1_01.y; L[5] = c2_01.y;
    L[6] = c0_2;    L[7] = c1_2;    L[8] = c2_2;
}

// Push-out of one particle against the scene's shapes, in order (contact.hpp:140-179).
// Shapes [begin, begin + count) of the particle's scene, in order.  kCull: this substep's
// cull table is valid (inside the substep pipeline, after the grid update; lo0 / hi0 = the
// first shape's world box, cached per lane); the standalone push-out tests the shape
// directly.
template <bool kCull>
__device__ __forceinline__ int pushout_particle(const Params& P, const SceneView& S, float x[3], float v[3],
                                                int begin, int count, float4 lo0, float4 hi0) {
    int pushed = 0;
    const float clearance = FM(1e-4f, S.dx);
    for (int si = begin; si < begin + count; ++si) {
        if (kCull) {
            const bool near = si == begin ? aabb_may_touch(lo0, hi0, x[0], x[1], x[2])
                                          : cull_may_touch(P, si, x[0], x[1], x[2]);
            if (!near) continue;
        }
        const DevShape& sh = P.shapes[si];
        const DevPose& pose = kCull ? P.pose_eff[si] : pose_of(P, si);  // kCull: the cull pass's copy
        if (!kCull && !shape_may_touch(sh, pose, mk(x[0], x[1], x[2]))) continue;
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

// ---- frame-end export (Params::exp_pad; scene.hpp:251-266).  The frame's last G2P has every
// particle's final x, v and flags in registers: it writes them to the result staging at the
// particle's original index and sums the per-scene totals, so the fetch needs no inverse
// permutation, gather or totals pass over the state.  Totals: each lane sums its particles of
// one scene in FP64 in shared memory (6 rows x 32 lanes per warp: 5 sums + the scene), the
// warp adds them with one FP64 atomic per value per group (per lane when lanes hold different
// scenes) -- the sums of k_totals, in another order.
constexpr int kExportBytesPerWarp = 6 * 32 * 8;
// two 16-byte stores into one 32-byte sector per particle (k_export_pack unpads them on the copy
// stream): 7 scattered scalar stores cost the short G2P of a mid-size scene more
__device__ __forceinline__ void export_write(const Params& P, const float x[3], const float v[3], float4 r) {
    const uint32_t o = __float_as_uint(r.w);
    if (o == kHoleOrig || static_cast<int64_t>(o) >= P.exp_n) return;
    float4* d = P.exp_pad + 2ull * o;
    d[0] = make_float4(x[0], x[1], x[2], v[0]);
    d[1] = make_float4(v[1], v[2], (__float_as_uint(r.z) & kActiveBit) ? 1.f : 0.f, 0.f);
}
__device__ __forceinline__ void tot_flush_lane(const Params& P, double* T, int lane) {
    int* tag = reinterpret_cast<int*>(T + 5 * 32);
    const int sc = tag[lane];
    if (sc < 0) return;
#pragma unroll
    for (int q = 0; q < 5; ++q) {
        atomicAdd(&P.exp_tot[5 * sc + q], T[q * 32 + lane]);
        T[q * 32 + lane] = 0.0;
    }
    tag[lane] = -1;
}
__device__ __forceinline__ void tot_init(double* T, int lane) {
#pragma unroll
    for (int q = 0; q < 5; ++q) T[q * 32 + lane] = 0.0;
    reinterpret_cast<int*>(T + 5 * 32)[lane] = -1;
}
// an active particle's contribution (k_totals' expressions)
__device__ __forceinline__ void tot_add(const Params& P, double* T, int lane, int scene, float mass, const float v[3]) {
    int* tag = reinterpret_cast<int*>(T + 5 * 32);
    if (tag[lane] != scene) {
        tot_flush_lane(P, T, lane);
        tag[lane] = scene;
    }
    const double m = mass;
    const float vx = v[0], vy = v[1], vz = v[2];
    T[lane] += m;
    T[32 + lane] += m * vx;
    T[64 + lane] += m * vy;
    T[96 + lane] += m * vz;
    T[128 + lane] += 0.5 * m * static_cast<double>(vx * vx + vy * vy + vz * vz);
}
// the whole warp: when every lane holding sums holds the same scene, the sums move to lane 0
// (which adds them to the next group's, or flushes them when the scene changes); otherwise
// each lane flushes its own
__device__ __forceinline__ void tot_fold_warp(const Params& P, double* T, int lane) {
    const unsigned full = 0xffffffffu;
    int* tag = reinterpret_cast<int*>(T + 5 * 32);
    const int sc = tag[lane];
    const int top = __reduce_max_sync(full, sc);
    if (top >= 0 && __all_sync(full, sc < 0 || sc == top)) {
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            double t = T[q * 32 + lane];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(full, t, o);
            T[q * 32 + lane] = lane == 0 ? t : 0.0;
        }
        tag[lane] = lane == 0 ? top : -1;
    } else if (top >= 0) {
        tot_flush_lane(P, T, lane);
    }
    __syncwarp();
}
// kernel end (the whole block): every warp folds, then one thread adds the warps' sums, one
// FP64 atomic per value per scene per block (same-address atomics serialise in L2: one per
// warp cost C2's export 39 us)
__device__ __forceinline__ void tot_flush_block(const Params& P, double* T0, double* T, int lane) {
    tot_fold_warp(P, T, lane);
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nw = static_cast<int>(blockDim.x >> 5);
        int cur = -1;
        double acc[5] = {0, 0, 0, 0, 0};
        for (int w = 0; w < nw; ++w) {
            const double* Tw = T0 + w * (kExportBytesPerWarp / 8);
            const int sc = reinterpret_cast<const int*>(Tw + 5 * 32)[0];
            if (sc < 0) continue;
            if (sc != cur) {
                if (cur >= 0)
                    for (int q = 0; q < 5; ++q) atomicAdd(&P.exp_tot[5 * cur + q], acc[q]);
                cur = sc;
                for (int q = 0; q < 5; ++q) acc[q] = 0.0;
            }
            for (int q = 0; q < 5; ++q) acc[q] += Tw[q * 32];
        }
        if (cur >= 0)
            for (int q = 0; q < 5; ++q) atomicAdd(&P.exp_tot[5 * cur + q], acc[q]);
    }
}

__device__ __forceinline__ void store_part_out(const Params& P, uint32_t s, const Part& p, float4 r) {
    P.pl_out[0][s] = make_float4(p.x[0], p.x[1], p.x[2], p.v[0]);
    P.pl_out[1][s] = make_float4(p.v[1], p.v[2], p.C[0], p.C[1]);
    P.pl_out[2][s] = make_float4(p.C[2], p.C[3], p.C[4], p.C[5]);
    P.pl_out[3][s] = make_float4(p.C[6], p.C[7], p.C[8], p.F[0]);
    P.pl_out[4][s] = make_float4(p.F[1], p.F[2], p.F[3], p.F[4]);
    P.pl_out[5][s] = make_float4(p.F[5], p.F[6], p.F[7], p.F[8]);
    P.pl_out[PR][s] = r;
}

// F <- (I + C dt) F  (solvers.hpp:194, 275).  F only feeds the stress (never a contact
// or push-out decision), so it keeps FMA contraction: F + dt (C F).
__device__ __forceinline__ void update_F(const float C[9], float dt, float F[9]) {
    float Fn[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            Fn[3 * i + j] = fmaf(dt, fmaf(C[3 * i], F[j], fmaf(C[3 * i + 1], F[3 + j], C[3 * i + 2] * F[6 + j])),
                                 F[3 * i + j]);
#pragma unroll
    for (int i = 0; i < 9; ++i) F[i] = Fn[i];
}

// Per-lane G2P state: the shape-range cache of the last scene and the counters.
struct G2PLane {
    int my_scene = 0;
    int cs_scene = -1, cs_begin = 0, cs_count = 0;
    float4 cs_lo = make_float4(0.f, 0.f, 0.f, -1.f), cs_hi = make_float4(0.f, 0.f, 0.f, -1.f);
    int n_inv = 0, n_fail = 0, n_push = 0, n_deact = 0;
};

// One particle's G2P (MLS solvers.hpp:173-196; PB :240-277; STD :107-135) with the F update,
// push-out and deactivation; p holds x, F (PB/STD: C) on entry, the new state on exit.
// The group's node box in shared memory (g2p_group): nodes [o, o + n) per axis, row-major x,
// packed o | n << 16 per axis (few registers: they stay live across the particle loop).
struct NodeBox {
    const float4* s;  // nullptr: gather from global memory
    int a[3];
    __device__ __forceinline__ int o(int d) const { return a[d] & 0xFFFF; }
    __device__ __forceinline__ int n(int d) const { return a[d] >> 16; }
};

template <bool PB, bool STD, bool BOX = false>
__device__ __forceinline__ void g2p_particle(const Params& P, Part& p, float4& r, G2PLane& L,
                                             const NodeBox& box = NodeBox{nullptr, {0, 0, 0}}) {
    uint32_t flags = __float_as_uint(r.z);
    const int scene = static_cast<int>((flags >> kSceneShift) & kSceneMask);
    L.my_scene = scene;
    const SceneView S = scene_view(P, scene);
    int b[3];
    float fx[3];
    local_base(P.geo, p.x, b, fx);
    float w[3][3], rel[3][3];  // STD: rel holds the weight derivatives
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        bspline_w(fx[a], w[a]);
        if (STD) {
            bspline_dw(fx[a], S.inv_dx, rel[a]);
        } else if (MPMB_NODE_REL) {
            node_rel(P.geo, a, b[a], p.x[a], S.dx, rel[a]);
        } else {
#pragma unroll
            for (int o = 0; o < 3; ++o) rel[a][o] = node_coord(P.geo, a, b[a] + o) - p.x[a];
        }
    }
    float B[9];  // STD: the velocity gradient L
    {
        // one gather: from the shared-memory node box when the stencil lies in it (generic
        // loads), else from the global pool
        uint32_t base, px, pxy;
        stencil_rows(P.geo, b, base, px, pxy);
        MPMB_DCHECK(S.node_base + base + 2ull * (pxy + px) + 2 < P.total_nodes);
        const float4* gp = P.grid_vel + S.node_base + base;
        const int r0 = b[0] - box.o(0), r1 = b[1] - box.o(1), r2 = b[2] - box.o(2);
        if (BOX && box.s && r0 >= 0 && r0 + 3 <= box.n(0) && r1 >= 0 && r1 + 3 <= box.n(1) && r2 >= 0 &&
            r2 + 3 <= box.n(2)) {
            px = static_cast<uint32_t>(box.n(0));
            pxy = px * static_cast<uint32_t>(box.n(1));
            gp = box.s + (r2 * box.n(1) + r1) * box.n(0) + r0;
        }
        if (STD) g2p_gather_std<BOX>(gp, px, pxy, w, rel, p.v, B);
        else g2p_gather<BOX>(gp, px, pxy, w, rel, p.v, B);
    }
    bool do_commit;
    if (STD) {  // solvers.hpp:130-134: x += v dt, F = (I + L dt) F; C unchanged
        do_commit = true;
    } else if (!PB) {  // solvers.hpp:191-195
#pragma unroll
        for (int i = 0; i < 9; ++i) p.C[i] = B[i] * S.m_inv;
        do_commit = true;
    } else {  // solvers.hpp:259-267
        float Cc[9], Cn[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) Cc[i] = B[i] * S.m_inv;
        const float4 mat = material(P, flags & kMatMask);
        if (corotational_project(p.F, Cc, P.dt, mat.w, Cn)) {
#pragma unroll
            for (int i = 0; i < 9; ++i) p.C[i] = Cn[i];
        } else {
            ++L.n_fail;
        }
        do_commit = P.commit != 0;
    }
    if (do_commit) {  // solvers.hpp:193-195 / 274-276
        p.x[0] = FA(p.x[0], FM(p.v[0], P.dt));
        p.x[1] = FA(p.x[1], FM(p.v[1], P.dt));
        p.x[2] = FA(p.x[2], FM(p.v[2], P.dt));
        update_F(STD ? B : p.C, P.dt, p.F);
        if (det3(p.F) <= 0.f) ++L.n_inv;
        if (P.pushout) {
            if (scene != L.cs_scene) {  // per-lane cache of the scene's shape range
                L.cs_scene = scene;
                L.cs_begin = P.scenes[scene].shape_begin;
                L.cs_count = P.scenes[scene].shape_count;
                if (L.cs_count > 0) {
                    L.cs_lo = P.cull[2 * L.cs_begin];
                    L.cs_hi = P.cull[2 * L.cs_begin + 1];
                }
            }
            if (L.cs_count > 0)
                L.n_push += pushout_particle<true>(P, S, p.x, p.v, L.cs_begin, L.cs_count, L.cs_lo, L.cs_hi);
        }
        if (P.deactivate && !spline_in_domain(mk(p.x[0], p.x[1], p.x[2]), S)) {
            flags &= ~kActiveBit;
            r.z = __uint_as_float(flags);
            ++L.n_deact;
        }
    }
}

// G2P of group g (PB: PB-MPM, solvers.hpp:240-277; STD: standard MPM, PIC velocity + L,
// solvers.hpp:107-135, C travels unchanged; neither: MLS-MPM, solvers.hpp:173-196).  Replays
// the order P2G sorted this group into (positions are unchanged since); lane L takes
// positions g2p_pos(L, k): the warp's 32 lanes gather around a few neighbouring stencils at
// every iteration.  Every position is written to the other buffer at slot
// group_phys(pos): the state leaves G2P in the new order.  `ring`: this warp's staging ring.
template <bool PB, bool STD, bool BOX, int KP = kPer, bool PREA = false>
__device__ __forceinline__ void g2p_group(const Params& P, uint32_t g, uint32_t unit, float4* ring, int lane,
                                          float4* box_s = nullptr, uint16_t* nbin = nullptr, int4* nbox = nullptr,
                                          double* tot = nullptr) {
    // nbox (with nbin): the stencil-base box of the new positions, group_sort's encoding
    int blo[3] = {INT_MAX, INT_MAX, INT_MAX}, bhi[3] = {INT_MIN, INT_MIN, INT_MIN};
    int sc_lo = INT_MAX, sc_hi = INT_MIN;
    constexpr int NP = (PB || STD) ? 7 : 5;
    constexpr int NS = kG2PStages;
    Stager<NP, NS, MPMB_G2P_CG != 0> st;
    st.buf = ring;
    st.lane = lane;
    const uint32_t p0 = unit * 32u * KP;  // the unit's first position (group_sort)
    const uint32_t n_act = P.group_nact[g * (kPer / KP) + unit];
    st.cnt = 0;
    {
        const uint8_t* ob = P.order + static_cast<uint64_t>(g) * kGroup + p0;
        uint64_t o = 0;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
            o |= static_cast<uint64_t>(ob[g2p_pos<KP>(lane, k)]) << (8 * k);
            st.cnt += g2p_pos<KP>(lane, k) < n_act ? 1 : 0;
        }
        st.order = o;
    }
    st.slot0 = g * kGroup;
    const int kmax = __reduce_max_sync(0xffffffffu, st.cnt);
    for (int k = 0; k < NS - 1; ++k) st.issue(P, k);
    NodeBox box{nullptr, {0, 0, 0}};
    if (BOX && box_s) {
        const int4 gb = P.group_box[g * (kPer / KP) + unit];
        if (gb.w >= 0) {
            const int ox = gb.x & 0xFFFF, oy = gb.y & 0xFFFF, oz = gb.z & 0xFFFF;
            const int nx = (gb.x >> 16) - ox + 3, ny = (gb.y >> 16) - oy + 3, nz = (gb.z >> 16) - oz + 3;
            const int rows = ny * nz;
            if (nx <= 32 && rows * nx <= kBoxCap) {
                // lanes cover rpi rows of nx nodes per step: coalesced row segments
                const int rpi = 32 / nx;
                const int lx = lane % nx, lr = lane / nx;
                if (lr < rpi) {
                    const float4* gv = P.grid_vel + static_cast<uint64_t>(gb.w) * P.geo.nodes_per_scene;
                    int j = lr % ny, k = lr / ny;
                    for (int r = lr; r < rows; r += rpi) {
                        box_s[r * nx + lx] = __ldg(gv + node_linear(P.geo, ox + lx, oy + j, oz + k));
                        j += rpi;
                        while (j >= ny) {
                            j -= ny;
                            ++k;
                        }
                    }
                }
                box.s = box_s;
                box.a[0] = ox | (nx << 16);
                box.a[1] = oy | (ny << 16);
                box.a[2] = oz | (nz << 16);
            }
        }
        __syncwarp();
    }
    G2PLane L;
    for (int k = 0; k < kmax; ++k) {
        st.issue(P, k + NS - 1);
        cp_wait<(NS > 3 ? NS - 2 : NS - 1)>();  // particles k (and k+1) have landed
        if (k >= st.cnt) continue;
        if (NS > 3 && k + 1 < st.cnt) {  // warm L1 with the next particle's stencil rows
            const float4 xn = st.buf[((k + 1) % NS) * NP * 32 + lane];
            int bn[3];
            float fn[3];
            const float xq[3] = {xn.x, xn.y, xn.z};
            local_base(P.geo, xq, bn, fn);
            const uint32_t sn = (__float_as_uint(st.buf[((k + 1) % NS) * NP * 32 + (NP - 1) * 32 + lane].z) >>
                                 kSceneShift) & kSceneMask;
            uint32_t base, px, pxy;
            stencil_rows(P.geo, bn, base, px, pxy);
            prefetch_stencil_l1(P.grid_vel + sn * P.geo.nodes_per_scene + base, px, pxy);
        }
        const uint32_t so = st.slot0 + group_phys(p0 + g2p_pos<KP>(lane, k));
        MPMB_DCHECK(so < static_cast<uint64_t>(P.n_total) && g2p_pos<KP>(lane, k) < 32u * KP);
        const float4* src = st.buf + (k % NS) * NP * 32 + lane;
        float4 r = src[(NP - 1) * 32];
        Part p;
        {
            const float4 q0 = src[0];
            p.x[0] = q0.x; p.x[1] = q0.y; p.x[2] = q0.z;
            if (PB || STD) {
                const float4 q1 = src[32], q2 = src[64], q3 = src[96], q4 = src[128], q5 = src[160];
                p.C[0] = q1.z; p.C[1] = q1.w; p.C[2] = q2.x; p.C[3] = q2.y; p.C[4] = q2.z;
                p.C[5] = q2.w; p.C[6] = q3.x; p.C[7] = q3.y; p.C[8] = q3.z;
                p.F[0] = q3.w; p.F[1] = q4.x; p.F[2] = q4.y; p.F[3] = q4.z; p.F[4] = q4.w;
                p.F[5] = q5.x; p.F[6] = q5.y; p.F[7] = q5.z; p.F[8] = q5.w;
            } else {
                const float4 q3 = src[32], q4 = src[64], q5 = src[96];
                p.F[0] = q3.w; p.F[1] = q4.x; p.F[2] = q4.y; p.F[3] = q4.z; p.F[4] = q4.w;
                p.F[5] = q5.x; p.F[6] = q5.y; p.F[7] = q5.z; p.F[8] = q5.w;
            }
        }
        g2p_particle<PB, STD, BOX>(P, p, r, L, box);
        if (PREA && (__float_as_uint(r.z) & kActiveBit)) {  // A for the fused P2G phase, in C's place
            float A[9];
            mls_affine(P, p.C, p.F, r.x, r.y, __float_as_uint(r.z), scene_view(P, L.my_scene).m_inv, A);
#pragma unroll
            for (int i = 0; i < 9; ++i) p.C[i] = A[i];
        }
        store_part_out(P, so, p, r);
        if (tot) {  // frame-end export (the standalone G2P only)
            export_write(P, p.x, p.v, r);
            if (__float_as_uint(r.z) & kActiveBit) tot_add(P, tot, lane, L.my_scene, r.x, p.v);
        }
        if (nbin) {  // the fused P2G phase sorts by these (group_sort)
            uint32_t b16 = 0xFFFFu;
            if (__float_as_uint(r.z) & kActiveBit) {
                int b[3];
                float fx[3];
                local_base(P.geo, p.x, b, fx);
                b16 = sort_bin(P, L.my_scene, b);
                if (nbox) {
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        blo[a] = min(blo[a], b[a]);
                        bhi[a] = max(bhi[a], b[a]);
                    }
                    sc_lo = min(sc_lo, L.my_scene);
                    sc_hi = max(sc_hi, L.my_scene);
                }
            }
            nbin[g2p_pos<KP>(lane, k)] = static_cast<uint16_t>(b16);
        }
    }
    // inactive particles and holes of the group move to their new slots unchanged
    for (int k = st.cnt; k < KP; ++k) {
        if (nbin) nbin[g2p_pos<KP>(lane, k)] = 0xFFFFu;
        const uint32_t si = st.slot(k), so = st.slot0 + group_phys(p0 + g2p_pos<KP>(lane, k));
        MPMB_DCHECK(si < static_cast<uint64_t>(P.n_total) && so < static_cast<uint64_t>(P.n_total));
        float4 q[kPlanes];
#pragma unroll
        for (int j = 0; j < kPlanes; ++j) q[j] = P.pl[j][si];
#pragma unroll
        for (int j = 0; j < kPlanes; ++j) P.pl_out[j][so] = q[j];
        if (tot) {
            const float x[3] = {q[0].x, q[0].y, q[0].z}, v[3] = {q[0].w, q[1].x, q[1].y};
            export_write(P, x, v, q[PR]);
        }
    }
    if (tot) tot_fold_warp(P, tot, lane);
    if (nbox) {
        const unsigned full = 0xffffffffu;
        int4 bx;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int l = __reduce_min_sync(full, blo[a]), h = __reduce_max_sync(full, bhi[a]);
            (a == 0 ? bx.x : a == 1 ? bx.y : bx.z) = l | (h << 16);
        }
        const int s0 = __reduce_min_sync(full, sc_lo), s1 = __reduce_max_sync(full, sc_hi);
        bx.w = (s0 == s1) ? s0 : -1;
        *nbox = bx;
    }
    add_scene_counter(P.counters, L.my_scene, 0, L.n_inv);
    add_scene_counter(P.counters, L.my_scene, 1, L.n_fail);
    add_scene_counter(P.counters, L.my_scene, 2, L.n_push);
    add_scene_counter(P.counters, L.my_scene, 3, L.n_deact);
    cp_wait<0>();
    __syncwarp();  // the ring is reused by the next group (or the fused P2G)
}

template <bool PB, bool STD = false, bool BOX = false, int KP = kPer>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, MPMB_G2P_MINB) k_g2p(const __grid_constant__ Params P) {
    pdl_enter();
    extern __shared__ float4 smem[];
    constexpr int NP = (PB || STD) ? 7 : 5;
    const int lane = threadIdx.x & 31;
    constexpr uint32_t U = kPer / KP;
    const uint32_t n_units = *P.n_groups * U;
    const uint32_t wpb = blockDim.x >> 5;
    float4* ring = smem + (threadIdx.x >> 5) * (kG2PStages * NP * 32);
    float4* box = BOX ? smem + wpb * (kG2PStages * NP * 32) + (threadIdx.x >> 5) * kBoxCap : nullptr;
    // frame-end export: per-warp totals rows after the rings and boxes (launch_g2p sizes them)
    double* tot = nullptr;
    if (P.exp_pad) {
        tot = reinterpret_cast<double*>(smem + wpb * (kG2PStages * NP * 32 + (BOX ? kBoxCap : 0))) +
              (threadIdx.x >> 5) * (kExportBytesPerWarp / 8);
        tot_init(tot, lane);
        __syncwarp();
    }
    for (uint32_t u = blockIdx.x * wpb + (threadIdx.x >> 5); u < n_units; u += gridDim.x * wpb)
        g2p_group<PB, STD, BOX, KP>(P, u / U, u % U, ring, lane, box, nullptr, nullptr, tot);
    if (tot) tot_flush_block(P, tot - (threadIdx.x >> 5) * (kExportBytesPerWarp / 8), tot, lane);
}

// Fused G2P of substep s + P2G of substep s+1 (MLS / standard MPM inside a frame), one warp
// per group: the reference runs push-out, free-body integration and deactivation between
// them (scene.hpp:209-235), and only deactivation and push-out touch particles; both are
// fused into the G2P phase, free bodies only need the contact sums of substep s.  The G2P
// phase writes the group in its new order to the other buffer; the P2G phase of the same
// warp re-sorts and stages it from there while the lines are still in L2, so the state
// crosses HBM once per substep (read x, F, flags; write everything) and the P2G load
// latency is an L2 latency.  Grid pools: G2P reads grid_vel (substep s), P2G accumulates
// into grid_acc (zeroed by the grid update of substep s), so the phases never alias.
// PB: PB-MPM iterations of one step (solvers.hpp:240-277 then 218-235): G2P of iteration it
// (no commit) fused with P2G of iteration it+1 (A = m C).
template <bool STD, bool PB = false, bool BOX = false, int KP = kPer>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, MPMB_P2G_MINB) k_g2p2g(const __grid_constant__ Params P) {
    pdl_enter();
    // the active-brick count of substep s+1 (read by the grid update of s, appended to by
    // the collect after this kernel): zeroed here instead of by a memset node, which would
    // break the programmatic-launch chain
    if (blockIdx.x == 0 && threadIdx.x == 0) *P.n_active_bricks = 0u;
    extern __shared__ float4 smem[];
    const int lane = threadIdx.x & 31;
    constexpr uint32_t U = kPer / KP;
    const uint32_t n_units = *P.n_groups * U;
    const uint32_t wpb = blockDim.x >> 5;
    constexpr int kRing = fused_ring<PB, STD>();
    float4* ring = smem + (threadIdx.x >> 5) * (kRing * 32);
    float4* box = BOX ? smem + wpb * (kRing * 32) + (threadIdx.x >> 5) * kBoxCap : nullptr;
    // per-warp bins of the new positions (kGroup u16): written by the G2P phase, read by the sort
    uint16_t* nbin = (BOX || !MPMB_FUSED_NBIN)
                         ? nullptr
                         : reinterpret_cast<uint16_t*>(smem + wpb * (kRing * 32)) + (threadIdx.x >> 5) * kGroup;
    // P2G tile (MLS): the G2P box's shared memory when there is one (free in the P2G phase),
    // else its own region after the bins
    constexpr bool TILE = MPMB_P2G_TILE && !PB && !STD;
    float4* tile = !TILE ? nullptr
                         : BOX ? box
                               : smem + wpb * (kRing * 32 + kGroup / 8) + (threadIdx.x >> 5) * kTileCap;
    for (uint32_t u = blockIdx.x * wpb + (threadIdx.x >> 5); u < n_units; u += gridDim.x * wpb) {
        int4 nb = make_int4(0, 0, 0, -1);
        g2p_group<PB, STD, BOX, KP, MPMB_K8_PREA && !PB && !STD>(P, u / U, u % U, ring, lane, box, nbin,
                                                                 (TILE && nbin) ? &nb : nullptr);
        __syncwarp();  // orders this warp's stores of the group (and nbin) before the P2G phase
        p2g_group<!PB, STD, true, BOX, KP>(P, u / U, u % U, ring, lane, nbin, tile, nb);
    }
}

// Wide G2P for small problems, where one warp per group would leave most SMs idle: one
// thread per slot, written to the same slot of the other buffer (inactive particles and
// holes copied unchanged).  The slot layout stays as binned; P2G's group sort is stable on
// any input order, so it pairs with the grouped P2G (a thread-per-slot P2G loses its
// register accumulation to L2 atomic contention: measured 1.8x slower at C2).
template <bool PB, bool STD = false>
__global__ void __launch_bounds__(128) k_g2p_wide(const __grid_constant__ Params P) {
    pdl_enter();
    extern __shared__ float4 smem[];
    const int lane = threadIdx.x & 31;
    double* tot = nullptr;  // frame-end export (launch_g2p gives it the rows)
    if (P.exp_pad) {
        tot = reinterpret_cast<double*>(smem) + (threadIdx.x >> 5) * (kExportBytesPerWarp / 8);
        tot_init(tot, lane);
        __syncwarp();
    }
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < P.n_total; base += stride) {
        const int64_t s = base + threadIdx.x;  // the warp stays converged for the counters
        G2PLane L;
        if (s < P.n_total) {
            float4 r = P.pl[PR][s];
            if (__float_as_uint(r.w) == kHoleOrig || !(__float_as_uint(r.z) & kActiveBit)) {
                float4 q[kPlanes];
#pragma unroll
                for (int j = 0; j < kPlanes; ++j) q[j] = P.pl[j][s];
#pragma unroll
                for (int j = 0; j < kPlanes; ++j) P.pl_out[j][s] = q[j];
                if (tot) {
                    const float x[3] = {q[0].x, q[0].y, q[0].z}, v[3] = {q[0].w, q[1].x, q[1].y};
                    export_write(P, x, v, q[PR]);
                }
            } else {
                Part p;
                const float4 q0 = P.pl[0][s], q3 = P.pl[3][s], q4 = P.pl[4][s], q5 = P.pl[5][s];
                p.x[0] = q0.x; p.x[1] = q0.y; p.x[2] = q0.z;
                p.F[0] = q3.w; p.F[1] = q4.x; p.F[2] = q4.y; p.F[3] = q4.z; p.F[4] = q4.w;
                p.F[5] = q5.x; p.F[6] = q5.y; p.F[7] = q5.z; p.F[8] = q5.w;
                if (PB || STD) {
                    const float4 q1 = P.pl[1][s], q2 = P.pl[2][s];
                    p.C[0] = q1.z; p.C[1] = q1.w; p.C[2] = q2.x; p.C[3] = q2.y; p.C[4] = q2.z;
                    p.C[5] = q2.w; p.C[6] = q3.x; p.C[7] = q3.y; p.C[8] = q3.z;
                }
                g2p_particle<PB, STD>(P, p, r, L);
                store_part_out(P, static_cast<uint32_t>(s), p, r);
                if (tot) {
                    export_write(P, p.x, p.v, r);
                    if (__float_as_uint(r.z) & kActiveBit) tot_add(P, tot, lane, L.my_scene, r.x, p.v);
                }
            }
        }
        add_scene_counter(P.counters, L.my_scene, 0, L.n_inv);
        add_scene_counter(P.counters, L.my_scene, 1, L.n_fail);
        add_scene_counter(P.counters, L.my_scene, 2, L.n_push);
        add_scene_counter(P.counters, L.my_scene, 3, L.n_deact);
    }
    if (tot) tot_flush_block(P, tot - (threadIdx.x >> 5) * (kExportBytesPerWarp / 8), tot, lane);
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
                const SceneView S = scene_view(P, scene);
                if (P.scenes[S.scene].shape_count > 0) {
                    float4 a = P.pl[0][s], b = P.pl[1][s];
                    float x[3] = {a.x, a.y, a.z}, v[3] = {a.w, b.x, b.y};
                    const float4 none = make_float4(0.f, 0.f, 0.f, -1.f);
                    pushed = pushout_particle<false>(P, S, x, v, P.scenes[S.scene].shape_begin,
                                                     P.scenes[S.scene].shape_count, none, none);
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
                if (!spline_in_domain(mk(a.x, a.y, a.z), scene_view(P, scene))) {
                    r.z = __uint_as_float(flags & ~kActiveBit);
                    P.pl[PR][s] = r;
                    d = 1;
                }
            }
        }
        add_scene_counter(P.counters, scene, 3, d);
    }
}

// ===================================================================  launchers
// grid-stride block cap of the transfer kernels, per SM (MPMB_XFER_BPS in the environment: A/B):
// 6 = two waves of the 3 resident blocks; against 16: C5 +0.3 %, M1 +1.3 %, C3 +0.5 %, C1 / C2
// unchanged (3, one wave: M1 -13 %, the tail of the grid-stride loop is one warp's groups)
static int xfer_cap() {
    static const int v = [] {
        const char* e = std::getenv("MPMB_XFER_BPS");
        return 148 * (e ? std::max(1, std::atoi(e)) : 6);
    }();
    return v;
}
static int grid_for(int64_t work, int threads, int max_blocks) {
    int64_t b = (work + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return static_cast<int>(b);
}

// dynamic shared memory per block: warps x stages x planes x 32 lanes x 16 B; kernels above
// 48 KB opt in once per device (opt_in_smem, kernels.cuh)

// Small problems (at most this many 256-slot groups) give every 64-position unit its own warp
// (KP = 2: 4x the warps, shorter serial chains; the node box is always on there).  The
// decision is a function of the engine's group bound, so P2G, G2P and the fused kernel of
// one engine always agree.  MPMB_SPLIT_MAX_GROUPS (environment) overrides, for A/B.
#ifndef MPMB_SPLIT_MAX_GROUPS
#define MPMB_SPLIT_MAX_GROUPS 512  // A/B: C1 (129 groups) +45 %; C2 and C3 (1,024) -17 % / +5 %, M1 (4,101) -23 %
#endif
// The smallest problems (at most this many groups) go one step further: 32-position units
// (KP = 1, one particle per lane, 8x the warps).  MPMB_TINY_MAX_GROUPS (environment)
// overrides, for A/B.
#ifndef MPMB_TINY_MAX_GROUPS
#define MPMB_TINY_MAX_GROUPS 0  // A/B at C1 (129 groups): 256 -> -12 % (K8 26.5 vs 23.3 us)
#endif
static bool tiny_units(int64_t max_groups) {
    static const int64_t lim = [] {
        const char* e = std::getenv("MPMB_TINY_MAX_GROUPS");
        return e ? std::atoll(e) : static_cast<int64_t>(MPMB_TINY_MAX_GROUPS);
    }();
    return kBoxCap > 0 && max_groups <= std::min<int64_t>(lim, kBoxMaxGroups);
}
static bool split_units(int64_t max_groups) {
    static const int64_t lim = [] {
        const char* e = std::getenv("MPMB_SPLIT_MAX_GROUPS");
        return e ? std::atoll(e) : static_cast<int64_t>(MPMB_SPLIT_MAX_GROUPS);
    }();
    return kBoxCap > 0 && max_groups <= std::min<int64_t>(lim, kBoxMaxGroups);
}
#ifndef MPMB_SPLIT_KP
#define MPMB_SPLIT_KP 2
#endif
constexpr int kSplitKP = MPMB_SPLIT_KP;  // positions per lane when split (2 or 4)
// PB-MPM (no stress in P2G, FP64 polar in G2P): 128-position units pay off up to the node-box
// bound (A/B, C3 at 1,024 groups: +8 %; MLS there: C2 -13 %, M1 -9 %)
constexpr int kPbSplitKP = 4;
static bool split_pb(int64_t max_groups) { return kBoxCap > 0 && max_groups <= kBoxMaxGroups; }

void launch_p2g(const Params& P, bool mls, int64_t max_groups, cudaStream_t st, bool standard) {
    const int threads = kWarpsPerBlock * 32;
    const int smem = kWarpsPerBlock * kStages * kPlanes * 32 * static_cast<int>(sizeof(float4));
    const bool split = split_units(max_groups);
    const int blocks = grid_for(max_groups * (split ? kPer / kSplitKP : 1) * 32, threads, xfer_cap());
    static std::atomic<uint64_t> attr{0};
    smem_opt_in_once(attr, [&] {
        opt_in_smem(k_p2g<true>, smem);
        opt_in_smem(k_p2g<false>, smem);
        opt_in_smem(k_p2g<true, true>, smem);
        opt_in_smem(k_p2g<true, false, true>, smem);
        opt_in_smem(k_p2g<false, false, true>, smem);
        opt_in_smem(k_p2g<true, true, true>, smem);
        opt_in_smem(k_p2g<true, false, true, kSplitKP>, smem);
        opt_in_smem(k_p2g<false, false, true, kSplitKP>, smem);
        opt_in_smem(k_p2g<true, true, true, kSplitKP>, smem);
        opt_in_smem(k_p2g<false, false, true, kPbSplitKP>, smem);
        opt_in_smem(k_p2g<true, false, true, 1>, smem);
        opt_in_smem(k_p2g<true, true, true, 1>, smem);
    });
    if (!mls && !standard && split_pb(max_groups)) {
        const int b4 = grid_for(max_groups * (kPer / kPbSplitKP) * 32, threads, xfer_cap());
        launch_chain(k_p2g<false, false, true, kPbSplitKP>, b4, threads, smem, st, P);
        return;
    }
    if ((mls || standard) && tiny_units(max_groups)) {
        const int b1 = grid_for(max_groups * kPer * 32, threads, xfer_cap());
        if (standard) launch_chain(k_p2g<true, true, true, 1>, b1, threads, smem, st, P);
        else launch_chain(k_p2g<true, false, true, 1>, b1, threads, smem, st, P);
        return;
    }
    if (split) {
        if (standard) launch_chain(k_p2g<true, true, true, kSplitKP>, blocks, threads, smem, st, P);
        else if (mls) launch_chain(k_p2g<true, false, true, kSplitKP>, blocks, threads, smem, st, P);
        else launch_chain(k_p2g<false, false, true, kSplitKP>, blocks, threads, smem, st, P);
        return;
    }
    if (kBoxCap > 0 && max_groups <= kBoxMaxGroups) {  // the G2P after it gathers from boxes
        if (standard) launch_chain(k_p2g<true, true, true>, blocks, threads, smem, st, P);
        else if (mls) launch_chain(k_p2g<true, false, true>, blocks, threads, smem, st, P);
        else launch_chain(k_p2g<false, false, true>, blocks, threads, smem, st, P);
        return;
    }
    if (standard) launch_chain(k_p2g<true, true>, blocks, threads, smem, st, P);
    else if (mls) launch_chain(k_p2g<true>, blocks, threads, smem, st, P);
    else launch_chain(k_p2g<false>, blocks, threads, smem, st, P);
}

void launch_g2p(const Params& P, bool pb, int64_t max_groups, cudaStream_t st, bool standard, bool wide) {
    // frame-end export (P.exp_pad): the totals rows after the rings and boxes
    const int ex = P.exp_pad ? kWarpsPerBlock * kExportBytesPerWarp : 0;
    if (wide) {
        const int b = grid_for(P.n_total, 128, 148 * 16);
        const int exw = P.exp_pad ? 4 * kExportBytesPerWarp : 0;
        if (standard) launch_chain(k_g2p_wide<false, true>, b, 128, exw, st, P);
        else if (pb) launch_chain(k_g2p_wide<true>, b, 128, exw, st, P);
        else launch_chain(k_g2p_wide<false>, b, 128, exw, st, P);
        return;
    }
    const int threads = kWarpsPerBlock * 32;
    const bool split = split_units(max_groups);
    const int blocks = grid_for(max_groups * (split ? kPer / kSplitKP : 1) * 32, threads, xfer_cap());
    const bool box = kBoxCap > 0 && max_groups <= kBoxMaxGroups;
    const int boxb = kWarpsPerBlock * kBoxCap * static_cast<int>(sizeof(float4));
    const int smem7 = kWarpsPerBlock * kG2PStages * 7 * 32 * static_cast<int>(sizeof(float4)) + ex;
    const int smem5 = kWarpsPerBlock * kG2PStages * 5 * 32 * static_cast<int>(sizeof(float4)) + ex;
    static std::atomic<uint64_t> attr{0};
    smem_opt_in_once(attr, [&] {  // sized with the export rows: the larger of the two launches
        const int x7 = kWarpsPerBlock * kG2PStages * 7 * 32 * static_cast<int>(sizeof(float4)) +
                       kWarpsPerBlock * kExportBytesPerWarp;
        const int x5 = kWarpsPerBlock * kG2PStages * 5 * 32 * static_cast<int>(sizeof(float4)) +
                       kWarpsPerBlock * kExportBytesPerWarp;
        opt_in_smem(k_g2p<true>, x7);
        opt_in_smem(k_g2p<false, true>, x7);
        opt_in_smem(k_g2p<false>, x5);
        opt_in_smem(k_g2p<true, false, true>, x7 + boxb);
        opt_in_smem(k_g2p<false, true, true>, x7 + boxb);
        opt_in_smem(k_g2p<false, false, true>, x5 + boxb);
        opt_in_smem(k_g2p<true, false, true, kSplitKP>, x7 + boxb);
        opt_in_smem(k_g2p<false, true, true, kSplitKP>, x7 + boxb);
        opt_in_smem(k_g2p<false, false, true, kSplitKP>, x5 + boxb);
        opt_in_smem(k_g2p<true, false, true, kPbSplitKP>, x7 + boxb);
        opt_in_smem(k_g2p<false, true, true, 1>, x7 + boxb);
        opt_in_smem(k_g2p<false, false, true, 1>, x5 + boxb);
    });
    if (pb && !standard && split_pb(max_groups)) {
        const int b4 = grid_for(max_groups * (kPer / kPbSplitKP) * 32, threads, xfer_cap());
        launch_chain(k_g2p<true, false, true, kPbSplitKP>, b4, threads, smem7 + boxb, st, P);
        return;
    }
    if (!pb && tiny_units(max_groups)) {
        const int b1 = grid_for(max_groups * kPer * 32, threads, xfer_cap());
        if (standard) launch_chain(k_g2p<false, true, true, 1>, b1, threads, smem7 + boxb, st, P);
        else launch_chain(k_g2p<false, false, true, 1>, b1, threads, smem5 + boxb, st, P);
        return;
    }
    if (split) {
        if (standard) launch_chain(k_g2p<false, true, true, kSplitKP>, blocks, threads, smem7 + boxb, st, P);
        else if (pb) launch_chain(k_g2p<true, false, true, kSplitKP>, blocks, threads, smem7 + boxb, st, P);
        else launch_chain(k_g2p<false, false, true, kSplitKP>, blocks, threads, smem5 + boxb, st, P);
        return;
    }
    if (box) {
        if (standard) launch_chain(k_g2p<false, true, true>, blocks, threads, smem7 + boxb, st, P);
        else if (pb) launch_chain(k_g2p<true, false, true>, blocks, threads, smem7 + boxb, st, P);
        else launch_chain(k_g2p<false, false, true>, blocks, threads, smem5 + boxb, st, P);
        return;
    }
    if (standard) launch_chain(k_g2p<false, true>, blocks, threads, smem7, st, P);
    else if (pb) launch_chain(k_g2p<true>, blocks, threads, smem7, st, P);
    else launch_chain(k_g2p<false>, blocks, threads, smem5, st, P);
}

void launch_g2p2g(const Params& P0, int64_t max_groups, cudaStream_t st, bool standard, bool pb) {
    Params P = P0;
    if (MPMB_DEBUG_NO_RED) P.debug = std::getenv("MPMB_DEBUG_NO_RED") ? 1u : 0u;
    const int threads = kWarpsPerBlock * 32;
    const bool split = split_units(max_groups);
    const int blocks = grid_for(max_groups * (split ? kPer / kSplitKP : 1) * 32, threads, xfer_cap());
    const bool box = kBoxCap > 0 && max_groups <= kBoxMaxGroups;
    const int ring = (pb || standard) ? fused_ring<true, false>() : fused_ring<false, false>();
    const int smem = kWarpsPerBlock * (ring * 32 * static_cast<int>(sizeof(float4)) + kGroup * 2 +  // + nbin
                                       ((pb || standard) ? 0 : kTileCap * static_cast<int>(sizeof(float4))));
    const int smem_box = kWarpsPerBlock * (ring * 32 + kBoxCap) * static_cast<int>(sizeof(float4));
    const int smem_max = kWarpsPerBlock * (fused_ring<true, false>() * 32 + std::max(kBoxCap, kGroup / 8 + kTileCap)) *
                         static_cast<int>(sizeof(float4));
    static std::atomic<uint64_t> attr{0};
    smem_opt_in_once(attr, [&] {
        opt_in_smem(k_g2p2g<false>, smem_max);
        opt_in_smem(k_g2p2g<true>, smem_max);
        opt_in_smem(k_g2p2g<false, true>, smem_max);
        opt_in_smem(k_g2p2g<false, false, true>, smem_max);
        opt_in_smem(k_g2p2g<true, false, true>, smem_max);
        opt_in_smem(k_g2p2g<false, true, true>, smem_max);
        opt_in_smem(k_g2p2g<false, false, true, kSplitKP>, smem_max);
        opt_in_smem(k_g2p2g<true, false, true, kSplitKP>, smem_max);
        opt_in_smem(k_g2p2g<false, true, true, kSplitKP>, smem_max);
        opt_in_smem(k_g2p2g<false, true, true, kPbSplitKP>, smem_max);
        opt_in_smem(k_g2p2g<false, false, true, 1>, smem_max);
        opt_in_smem(k_g2p2g<true, false, true, 1>, smem_max);
    });
    if (pb && split_pb(max_groups)) {
        const int b4 = grid_for(max_groups * (kPer / kPbSplitKP) * 32, threads, xfer_cap());
        launch_chain(k_g2p2g<false, true, true, kPbSplitKP>, b4, threads, smem_box, st, P);
        return;
    }
    if (!pb && tiny_units(max_groups)) {
        const int b1 = grid_for(max_groups * kPer * 32, threads, xfer_cap());
        if (standard) launch_chain(k_g2p2g<true, false, true, 1>, b1, threads, smem_box, st, P);
        else launch_chain(k_g2p2g<false, false, true, 1>, b1, threads, smem_box, st, P);
        return;
    }
    if (split) {
        if (pb) launch_chain(k_g2p2g<false, true, true, kSplitKP>, blocks, threads, smem_box, st, P);
        else if (standard) launch_chain(k_g2p2g<true, false, true, kSplitKP>, blocks, threads, smem_box, st, P);
        else launch_chain(k_g2p2g<false, false, true, kSplitKP>, blocks, threads, smem_box, st, P);
        return;
    }
    if (box) {
        if (pb) launch_chain(k_g2p2g<false, true, true>, blocks, threads, smem_box, st, P);
        else if (standard) launch_chain(k_g2p2g<true, false, true>, blocks, threads, smem_box, st, P);
        else launch_chain(k_g2p2g<false, false, true>, blocks, threads, smem_box, st, P);
        return;
    }
    if (pb) launch_chain(k_g2p2g<false, true>, blocks, threads, smem, st, P);
    else if (standard) launch_chain(k_g2p2g<true>, blocks, threads, smem, st, P);
    else launch_chain(k_g2p2g<false>, blocks, threads, smem, st, P);
}

void launch_pushout(const Params& P, cudaStream_t st) {
    k_pushout<<<grid_for(P.n_total, 256, 148 * 8), 256, 0, st>>>(P);
    MPMB_LAUNCHED("k_pushout");
}

void launch_deactivate(const Params& P, cudaStream_t st) {
    k_deactivate<<<grid_for(P.n_total, 256, 148 * 8), 256, 0, st>>>(P);
    MPMB_LAUNCHED("k_deactivate");
}

}  // namespace mpmb
