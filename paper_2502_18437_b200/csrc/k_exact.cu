// k_exact.cu — the EXACT mode of the MLS substep: the reference's float arithmetic, in the
// reference's order, on the device ("deterministic mode"; SURVEY.md §7 hard part
// 5).  Every operation is an explicit IEEE round-to-nearest intrinsic (no contraction),
// expressions keep the reference's operand order, and every sum runs in the reference's
// sequence, so a substep reproduces solvers.hpp:141-198 bit for bit and run to run.
//
//   P2G   node-major gather.  The reference scatters particles in original index order, so
//         a node's mass / momentum is the float sum of its contributions in increasing
//         original index.  Particles are sorted by (base cell, original index) (CUB radix
//         sort, 64-bit keys); each node merges the 27 cell lists that reach it by original
//         index and accumulates w * m and (v m + A rel) * w exactly as solvers.hpp:157-168.
//   G2P   per particle, nodes in (dk, dj, di) order, skipping mass <= eps (solvers.hpp:
//         176-196); sigma in FP64 with the reference's divide (materials.hpp:35-54).
//
// The fast mode (k_transfer.cu) stays the default; exact mode trades speed for identity.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include "launch.h"

namespace mpmb {

namespace {

#define DM __dmul_rn
#define DA __dadd_rn
#define DS __dsub_rn

// math.hpp:215-234 with explicit rounding (no contraction)
__device__ __forceinline__ void spline_exact(const float x[3], const Geo& G, int base[3], float w[3][3]) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float p = FM(FS(x[a], G.origin[a]), G.inv_dx);
        const int b = static_cast<int>(floorf(FS(p, 0.5f)));
        const float fx = FS(p, static_cast<float>(b));
        base[a] = b;
        const float u = FS(1.5f, fx), c = FS(fx, 1.f), e = FS(fx, 0.5f);
        w[a][0] = FM(FM(0.5f, u), u);
        w[a][1] = FS(0.75f, FM(c, c));
        w[a][2] = FM(FM(0.5f, e), e);
    }
}

// A (row-major) * r, row i: (a_i0 r0 + a_i1 r1) + a_i2 r2 (math.hpp Mat3 * Vec3)
__device__ __forceinline__ void mulv(const float A[9], const float r[3], float o[3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i) o[i] = FA(FA(FM(A[3 * i], r[0]), FM(A[3 * i + 1], r[1])), FM(A[3 * i + 2], r[2]));
}

__device__ __forceinline__ bool live_slot(const Params& P, int64_t s, uint32_t& flags, uint32_t& orig) {
    const float4 r = P.pl[PR][s];
    flags = __float_as_uint(r.z);
    orig = __float_as_uint(r.w);
    return orig != kHoleOrig && (flags & kActiveBit);
}

int blocks_of(int64_t n, int t) {
    int64_t b = (n + t - 1) / t;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return static_cast<int>(b);
}

// Per particle: sort key (global base-cell id << 32 | original index), the P2G inputs
// {x, v, m, affine (solvers.hpp:154-156), weights} and the brick marks.
constexpr int kPrepF4 = 7;  // x3 v3 m | A9 | w9 -> 25 floats in 7 float4
__global__ void k_ex_prep(const Params P, int mls, uint64_t* key, uint32_t* val, float4* prep) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        uint32_t flags, orig;
        val[s] = static_cast<uint32_t>(s);
        if (!live_slot(P, s, flags, orig)) {
            key[s] = ~0ull;
            continue;
        }
        Part p;
        load_part(P, static_cast<uint32_t>(s), p);
        const float4 r = P.pl[PR][s];
        const float m = r.x;
        int base[3];
        float w[3][3];
        spline_exact(p.x, P.geo, base, w);
        const int scene = static_cast<int>((flags >> kSceneShift) & kSceneMask);
        const SceneView S = scene_view(P, scene);
        float A[9];
        if (mls) {  // MLS: C m + sigma (-dt V m_inv), V = det(F) V0 (solvers.hpp:154-156)
            float sig[9];
            if (P.use_stress_in) {
                const float* s9 = P.stress_in + 9ull * orig;
#pragma unroll
                for (int i = 0; i < 9; ++i) sig[i] = s9[i];
            } else {
                const float4 mat = material(P, flags & kMatMask);
                neo_hookean(p.F, mat.y, mat.z, sig);
            }
            const float volume = FM(det3(p.F), r.y);
            const float sc = FM(FM(-P.dt, volume), S.m_inv);
#pragma unroll
            for (int i = 0; i < 9; ++i) A[i] = FA(FM(p.C[i], m), FM(sig[i], sc));
        } else {  // PB-MPM: C m (solvers.hpp:222)
#pragma unroll
            for (int i = 0; i < 9; ++i) A[i] = FM(p.C[i], m);
        }
        float4* o = prep + static_cast<uint64_t>(s) * kPrepF4;
        o[0] = make_float4(p.x[0], p.x[1], p.x[2], p.v[0]);
        o[1] = make_float4(p.v[1], p.v[2], m, A[0]);
        o[2] = make_float4(A[1], A[2], A[3], A[4]);
        o[3] = make_float4(A[5], A[6], A[7], A[8]);
        o[4] = make_float4(w[0][0], w[0][1], w[0][2], w[1][0]);
        o[5] = make_float4(w[1][1], w[1][2], w[2][0], w[2][1]);
        o[6] = make_float4(w[2][2], 0.f, 0.f, 0.f);
        int lb[3];
        float fx[3];
        local_base(P.geo, p.x, lb, fx);
        const uint32_t brick = S.brick_base + (static_cast<uint32_t>(lb[2] >> 2) * P.geo.nb[1] +
                                               static_cast<uint32_t>(lb[1] >> 2)) * P.geo.nb[0] +
                               static_cast<uint32_t>(lb[0] >> 2);
        const uint32_t cell = static_cast<uint32_t>(((lb[2] & 3) << 4) | ((lb[1] & 3) << 2) | (lb[0] & 3));
        key[s] = (static_cast<uint64_t>((brick << 6) | cell) << 32) | orig;
        const uint32_t mk = 8u | ((lb[0] & 3) >= 2 ? 1u : 0u) | ((lb[1] & 3) >= 2 ? 2u : 0u) | ((lb[2] & 3) >= 2 ? 4u : 0u);
        atomicOr(&P.brick_flag[brick], mk);
    }
}

// active brick -> index (stamped with the epoch so nothing needs clearing)
__global__ void k_ex_index(const Params P, uint2* brick_idx, uint32_t epoch) {
    const uint32_t n = *P.n_active_bricks;
    for (uint32_t a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x)
        brick_idx[P.active_bricks[a]] = make_uint2(epoch, a);
}

// cell ranges of the sorted keys: range[active index * 64 + cell] = [start, end)
__global__ void k_ex_ranges(const Params P, const uint64_t* skey, const uint2* brick_idx, uint32_t epoch,
                            uint2* range) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < P.n_total; t += stride) {
        const uint64_t k = skey[t];
        if (k == ~0ull) continue;
        const uint32_t c = static_cast<uint32_t>(k >> 32);
        const bool first = t == 0 || static_cast<uint32_t>(skey[t - 1] >> 32) != c;
        const bool last = t + 1 == P.n_total || skey[t + 1] == ~0ull || static_cast<uint32_t>(skey[t + 1] >> 32) != c;
        if (!first && !last) continue;
        const uint2 bi = brick_idx[c >> 6];
        if (bi.x != epoch) continue;  // cannot happen: a particle's base brick is active
        uint2* r = range + static_cast<uint64_t>(bi.y) * 64 + (c & 63u);
        if (first) r->x = static_cast<uint32_t>(t);
        if (last) r->y = static_cast<uint32_t>(t + 1);
    }
}

// One thread per node of an active brick: merge the (<= 27) cell lists that reach the node by
// original index and accumulate exactly as solvers.hpp:157-168.
__global__ void __launch_bounds__(64) k_ex_gather(const Params P, const uint64_t* skey, const uint32_t* sval,
                                                  const float4* prep, const uint2* brick_idx, uint32_t epoch,
                                                  const uint2* range) {
    const uint32_t n_act = *P.n_active_bricks;
    const int l = threadIdx.x;
    for (uint32_t a = blockIdx.x; a < n_act; a += gridDim.x) {
        const uint32_t gb = P.active_bricks[a];
        const int scene = static_cast<int>(gb / P.geo.bricks_per_scene);
        const SceneView S = scene_view(P, scene);
        const uint32_t local = gb - S.brick_base;
        const int nb0 = P.geo.nb[0], nb1 = P.geo.nb[1];
        const int i = static_cast<int>(local % nb0) * 4 + (l & 3);
        const int j = static_cast<int>((local / nb0) % nb1) * 4 + ((l >> 2) & 3);
        const int k = static_cast<int>(local / (nb0 * nb1)) * 4 + (l >> 4);
        uint32_t cur[27], end[27], head[27];
#pragma unroll
        for (int d = 0; d < 27; ++d) {
            cur[d] = end[d] = 0;
            head[d] = 0xFFFFFFFFu;
            const int bi = i - d % 3, bj = j - (d / 3) % 3, bk = k - d / 9;  // base cell of the source
            if (bi < 0 || bj < 0 || bk < 0) continue;
            const uint32_t cb = S.brick_base + (static_cast<uint32_t>(bk >> 2) * nb1 + static_cast<uint32_t>(bj >> 2)) * nb0 +
                                static_cast<uint32_t>(bi >> 2);
            const uint2 idx = brick_idx[cb];
            if (idx.x != epoch) continue;
            const uint2 rg = range[static_cast<uint64_t>(idx.y) * 64 + (((bk & 3) << 4) | ((bj & 3) << 2) | (bi & 3))];
            cur[d] = rg.x;
            end[d] = rg.y;
            if (rg.x < rg.y) head[d] = static_cast<uint32_t>(skey[rg.x]);
        }
        // node position (state.hpp:49-51), global index
        const float npos[3] = {FA(S.origin[0], FM(static_cast<float>(i + P.geo.goff), S.dx)),
                               FA(S.origin[1], FM(static_cast<float>(j), S.dx)),
                               FA(S.origin[2], FM(static_cast<float>(k), S.dx))};
        float mass = 0.f, mom[3] = {0.f, 0.f, 0.f};
        while (true) {
            uint32_t best = 0xFFFFFFFFu;
            int bd = -1;
#pragma unroll
            for (int d = 0; d < 27; ++d)
                if (head[d] < best) {
                    best = head[d];
                    bd = d;
                }
            if (bd < 0) break;
            uint32_t t = 0;
            int di = 0, dj = 0, dk = 0;
#pragma unroll
            for (int d = 0; d < 27; ++d)
                if (d == bd) {
                    t = cur[d];
                    cur[d] = t + 1;
                    head[d] = t + 1 < end[d] ? static_cast<uint32_t>(skey[t + 1]) : 0xFFFFFFFFu;
                    di = d % 3;
                    dj = (d / 3) % 3;
                    dk = d / 9;
                }
            const float4* q = prep + static_cast<uint64_t>(sval[t]) * kPrepF4;
            const float4 q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3], q4 = q[4], q5 = q[5], q6 = q[6];
            const float x[3] = {q0.x, q0.y, q0.z}, v[3] = {q0.w, q1.x, q1.y};
            const float m = q1.z;
            const float A[9] = {q1.w, q2.x, q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w};
            const float wx[3] = {q4.x, q4.y, q4.z}, wy[3] = {q4.w, q5.x, q5.y}, wz[3] = {q5.z, q5.w, q6.x};
            const float w = FM(FM(wx[di], wy[dj]), wz[dk]);
            const float rel[3] = {FS(npos[0], x[0]), FS(npos[1], x[1]), FS(npos[2], x[2])};
            float ar[3];
            mulv(A, rel, ar);
            mass = FA(mass, FM(w, m));
#pragma unroll
            for (int c = 0; c < 3; ++c) mom[c] = FA(mom[c], FM(FA(FM(v[c], m), ar[c]), w));
        }
        P.grid_acc[S.node_base + node_linear(P.geo, i, j, k)] = make_float4(mom[0], mom[1], mom[2], mass);
    }
}

// G2P, solvers.hpp:173-196 in the reference's order and arithmetic, per particle in place.
__global__ void k_ex_g2p(const Params P) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        uint32_t flags, orig;
        if (!live_slot(P, s, flags, orig)) continue;
        Part p;
        load_part(P, static_cast<uint32_t>(s), p);
        const int scene = static_cast<int>((flags >> kSceneShift) & kSceneMask);
        const SceneView S = scene_view(P, scene);
        (void)orig;
        int base[3];
        float w[3][3];
        spline_exact(p.x, P.geo, base, w);
        float vn[3] = {0.f, 0.f, 0.f}, B[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int dk = 0; dk < 3; ++dk)
            for (int dj = 0; dj < 3; ++dj)
                for (int di = 0; di < 3; ++di) {
                    const float ww = FM(FM(w[0][di], w[1][dj]), w[2][dk]);
                    const int gi = base[0] + di, gj = base[1] + dj, gk = base[2] + dk;
                    const float4 node = P.grid_vel[S.node_base + node_linear(P.geo, gi - P.geo.goff, gj, gk)];
                    if (node.w <= kMassEps) continue;
                    const float rel[3] = {FS(FA(S.origin[0], FM(static_cast<float>(gi), S.dx)), p.x[0]),
                                          FS(FA(S.origin[1], FM(static_cast<float>(gj), S.dx)), p.x[1]),
                                          FS(FA(S.origin[2], FM(static_cast<float>(gk), S.dx)), p.x[2])};
                    const float vw[3] = {FM(node.x, ww), FM(node.y, ww), FM(node.z, ww)};
#pragma unroll
                    for (int r = 0; r < 3; ++r) {
                        vn[r] = FA(vn[r], vw[r]);
#pragma unroll
                        for (int c = 0; c < 3; ++c) B[3 * r + c] = FA(B[3 * r + c], FM(vw[r], rel[c]));
                    }
                }
        p.v[0] = vn[0]; p.v[1] = vn[1]; p.v[2] = vn[2];
#pragma unroll
        for (int i = 0; i < 9; ++i) p.C[i] = FM(B[i], S.m_inv);
        p.x[0] = FA(p.x[0], FM(p.v[0], P.dt));
        p.x[1] = FA(p.x[1], FM(p.v[1], P.dt));
        p.x[2] = FA(p.x[2], FM(p.v[2], P.dt));
        // F = (I + C dt) F: Mat3 + Mat3, then Mat3 * Mat3 row-column (a b0 + a b1) + a b2
        float M[9], Fn[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) M[i] = FA(i % 4 == 0 ? 1.f : 0.f, FM(p.C[i], P.dt));
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c)
                Fn[3 * r + c] = FA(FA(FM(M[3 * r], p.F[c]), FM(M[3 * r + 1], p.F[3 + c])), FM(M[3 * r + 2], p.F[6 + c]));
#pragma unroll
        for (int i = 0; i < 9; ++i) p.F[i] = Fn[i];
        // push-out and deactivation follow as the standalone kernels (contact.hpp:140-179,
        // state.hpp:153-164): they depend on the particle and the substep's poses only
        store_part(P, static_cast<uint32_t>(s), p);
        if (det3(p.F) <= 0.f) atomicAdd(&P.counters[4 * scene + 0], 1);
    }
}

__global__ void k_ex_iota(uint32_t* v, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}

__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t* a, uint32_t n, uint64_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// contact.hpp:127-129: acc[si].impulse += imp; acc[si].torque += tq, node by node in grid
// index order, in float, on top of what the accumulator already holds.  The records of one
// shape are contiguous after the sort; one thread per shape walks them serially.
__global__ void k_ex_contact_sum(const Params P, const uint64_t* skey, const uint32_t* sval, uint32_t n) {
    for (int si = threadIdx.x; si < P.n_shapes; si += blockDim.x) {
        const uint32_t b = lower_bound_u64(skey, n, static_cast<uint64_t>(si) << 40);
        const uint32_t e = lower_bound_u64(skey, n, static_cast<uint64_t>(si + 1) << 40);
        float acc[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[q] = static_cast<float>(P.acc_sub[6 * si + q]);
        for (uint32_t r = b; r < e; ++r) {
            const float* t = P.ex_crec + 6ull * sval[r];
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = FA(acc[q], t[q]);
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) P.acc_sub[6 * si + q] = static_cast<double>(acc[q]);
        P.cnt_sub[si] += static_cast<int>(e - b);
    }
}

}  // namespace

size_t exact_contact_scratch_bytes(uint32_t n) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), static_cast<int>(n));
    return 3 * 256 + 8 * static_cast<size_t>(n) + 8 * static_cast<size_t>(n) + temp;
}

// Ordered contact sums of one substep's n records (P.ex_ckey / P.ex_crec).
void launch_exact_contact(const Params& P, uint32_t n, void* scratch, cudaStream_t st) {
    if (n == 0 || P.n_shapes == 0) return;
    char* m = static_cast<char*>(scratch);
    auto take = [&m](size_t b) {
        char* p = m;
        m += (b + 255) & ~static_cast<size_t>(255);
        return p;
    };
    auto* skey = reinterpret_cast<uint64_t*>(take(8ull * n));
    auto* val = reinterpret_cast<uint32_t*>(take(4ull * n));
    auto* sval = reinterpret_cast<uint32_t*>(take(4ull * n));
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, P.ex_ckey, skey, val, sval, static_cast<int>(n));
    void* tmp = take(temp);
    k_ex_iota<<<blocks_of(n, 256), 256, 0, st>>>(val, n);
    MPMB_LAUNCHED("k_ex_iota");
    cub::DeviceRadixSort::SortPairs(tmp, temp, P.ex_ckey, skey, val, sval, static_cast<int>(n), 0, 64, st);
    k_ex_contact_sum<<<1, 128, 0, st>>>(P, skey, sval, n);
    MPMB_LAUNCHED("k_ex_contact_sum");
}

size_t exact_scratch_bytes(int64_t n, int64_t n_bricks) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), static_cast<int>(n));
    const size_t a = 2 * 8 * n + 2 * 4 * n + 16 * kPrepF4 * n + 8 * 64 * n_bricks + temp;
    return a + 16 * 256;
}

// Exact P2G: keys/prep (+ marks), sort, collect, brick index, cell ranges, gather.
void launch_exact_p2g(const Params& P, bool mls, void* scratch, uint2* brick_idx, uint32_t epoch, int64_t n_bricks,
                      cudaStream_t st) {
    const int64_t n = P.n_total;
    char* m = static_cast<char*>(scratch);
    auto take = [&m](size_t b) {
        char* p = m;
        m += (b + 255) & ~static_cast<size_t>(255);
        return p;
    };
    auto* key = reinterpret_cast<uint64_t*>(take(8 * n));
    auto* skey = reinterpret_cast<uint64_t*>(take(8 * n));
    auto* val = reinterpret_cast<uint32_t*>(take(4 * n));
    auto* sval = reinterpret_cast<uint32_t*>(take(4 * n));
    auto* prep = reinterpret_cast<float4*>(take(16 * kPrepF4 * n));
    uint2* bidx = brick_idx;  // persistent, epoch-stamped
    auto* range = reinterpret_cast<uint2*>(take(8 * 64 * n_bricks));
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, key, skey, val, sval, static_cast<int>(n));
    void* tmp = take(temp);
    k_ex_prep<<<blocks_of(n, 256), 256, 0, st>>>(P, mls ? 1 : 0, key, val, prep);
    MPMB_LAUNCHED("k_ex_prep");
    cub::DeviceRadixSort::SortPairs(tmp, temp, key, skey, val, sval, static_cast<int>(n), 0, 64, st);
    launch_collect_bricks(P, static_cast<uint32_t>(n_bricks), st);
    k_ex_index<<<blocks_of(n_bricks, 256), 256, 0, st>>>(P, bidx, epoch);
    MPMB_LAUNCHED("k_ex_index");
    cudaMemsetAsync(range, 0, 8 * 64 * n_bricks, st);
    k_ex_ranges<<<blocks_of(n, 256), 256, 0, st>>>(P, skey, bidx, epoch, range);
    MPMB_LAUNCHED("k_ex_ranges");
    k_ex_gather<<<blocks_of(n_bricks * 64, 64), 64, 0, st>>>(P, skey, sval, prep, bidx, epoch, range);
    MPMB_LAUNCHED("k_ex_gather");
}

void launch_exact_g2p(const Params& P, cudaStream_t st) {
    k_ex_g2p<<<blocks_of(P.n_total, 128), 128, 0, st>>>(P);
    MPMB_LAUNCHED("k_ex_g2p");
}

}  // namespace mpmb
