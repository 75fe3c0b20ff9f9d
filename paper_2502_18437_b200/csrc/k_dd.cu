// k_dd.cu — slab domain decomposition: halo planes of the
// node pools and particle migration.  A slab owns global x nodes [lo, hi) and stores
// [lo - M, hi + 2 + M) (local [0, lx)); owned = local [own_lo, own_hi) = [M, M + hi - lo).
//
//   after P2G    ghost sums out:  local [0, M) -> lower neighbour, local [own_hi, lx) -> upper;
//                the owner adds them into local [own_hi - M, own_hi) / [own_lo, own_lo + 2 + M)
//   after grid   owned velocities back: [own_lo, own_lo + 2 + M) -> lower neighbour's high
//                ghosts, [own_hi - M, own_hi) -> upper neighbour's low ghosts
//   at binning   particles whose global base x left [lo, hi) move to the neighbour
//
// Halo buffers hold x-planes restricted to a y/z window (default: the whole storage
// extent; dd_set_window narrows it to the particles' reach).
#include <cuda_runtime.h>

#include <climits>

#include "dd_ops.h"
#include "launch.h"

namespace mpmb {

static int dd_blocks(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return static_cast<int>(b);
}

// mode 0: copy pool -> buf; 1: add buf into pool (and mark the brick of every node with
// mass); 2: copy buf -> pool.  Only the y/z window [y0, y0 + ny) x [z0, z0 + nz) of each
// x-plane travels (Engine::dd_set_window): buf element ((xr * nz) + z - z0) * ny + y - y0.
template <int MODE>
__global__ void k_halo(const Params P, float4* pool, float4* buf, int x0, int w, int y0, int ny, int z0, int nz) {
    const int64_t n = static_cast<int64_t>(w) * ny * nz;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride) {
        const int y = y0 + static_cast<int>(e % ny);
        const int z = z0 + static_cast<int>((e / ny) % nz);
        const int xr = static_cast<int>(e / (static_cast<int64_t>(ny) * nz));
        const int x = x0 + xr;
        const uint64_t idx = node_linear(P.geo, x, y, z);
        if (MODE == 0) {
            buf[e] = pool[idx];
        } else if (MODE == 1) {
            const float4 q = buf[e];
            if (q.w != 0.f || q.x != 0.f || q.y != 0.f || q.z != 0.f) {
                float4 a = pool[idx];
                a.x += q.x; a.y += q.y; a.z += q.z; a.w += q.w;
                pool[idx] = a;
                atomicOr(&P.brick_flag[(static_cast<uint32_t>(z >> 2) * P.geo.nb[1] + static_cast<uint32_t>(y >> 2)) *
                                           P.geo.nb[0] + static_cast<uint32_t>(x >> 2)],
                         8u);  // the node's own brick (mark_bricks encoding)
            }
        } else {
            pool[idx] = buf[e];
        }
    }
}

int64_t dd_plane_nodes(const Params& P) {
    return static_cast<int64_t>(P.geo.nb[1]) * 4 * P.geo.nb[2] * 4;
}

void launch_halo(const Params& P, int mode, float4* pool, float4* buf, int x0, int w, int y0, int ny, int z0, int nz,
                 cudaStream_t st) {
    const int64_t n = static_cast<int64_t>(ny) * nz * w;
    if (n <= 0) return;
    const int blocks = dd_blocks(n, 256);
    if (mode == 0) k_halo<0><<<blocks, 256, 0, st>>>(P, pool, buf, x0, w, y0, ny, z0, nz);
    else if (mode == 1) k_halo<1><<<blocks, 256, 0, st>>>(P, pool, buf, x0, w, y0, ny, z0, nz);
    else k_halo<2><<<blocks, 256, 0, st>>>(P, pool, buf, x0, w, y0, ny, z0, nz);
    MPMB_LAUNCHED("k_halo");
}

// Node window of the active particles' stencils in y and z: out = {min base y, max base
// y + 2, min base z, max base z + 2} (atomicMin / atomicMax; initialised by the host).
__global__ void k_particle_window(const Params P, int* out) {
    int ylo = INT_MAX, yhi = INT_MIN, zlo = INT_MAX, zhi = INT_MIN;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        const float4 r = P.pl[PR][s];
        if (__float_as_uint(r.w) == kHoleOrig || !(__float_as_uint(r.z) & kActiveBit)) continue;
        const float4 a = P.pl[0][s];
        float f;
        const int by = stencil_base(a.y, P.geo.origin[1], P.geo.inv_dx, f);
        const int bz = stencil_base(a.z, P.geo.origin[2], P.geo.inv_dx, f);
        ylo = min(ylo, by); yhi = max(yhi, by + 2);
        zlo = min(zlo, bz); zhi = max(zhi, bz + 2);
    }
    for (int o = 16; o > 0; o >>= 1) {
        ylo = min(ylo, __shfl_xor_sync(0xffffffffu, ylo, o));
        yhi = max(yhi, __shfl_xor_sync(0xffffffffu, yhi, o));
        zlo = min(zlo, __shfl_xor_sync(0xffffffffu, zlo, o));
        zhi = max(zhi, __shfl_xor_sync(0xffffffffu, zhi, o));
    }
    if ((threadIdx.x & 31) == 0 && ylo <= yhi) {
        atomicMin(&out[0], ylo);
        atomicMax(&out[1], yhi);
        atomicMin(&out[2], zlo);
        atomicMax(&out[3], zhi);
    }
}

void launch_particle_window(const Params& P, int* out, cudaStream_t st) {
    k_particle_window<<<dd_blocks(P.n_total, 256), 256, 0, st>>>(P, out);
    MPMB_LAUNCHED("k_particle_window");
}

// Particles whose global stencil base x left [lo, hi): packed (7 float4 each) into the
// lower / upper send buffer, their slots turned into holes.  counts[0/1] = lower / upper.
__global__ void k_migrate_pack(const Params P, int lo, int hi, float4* out_lo, float4* out_hi, uint32_t cap,
                               uint32_t* counts) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        const float4 r = P.pl[PR][s];
        // active particles only: inactive ones are frozen wherever they are
        if (__float_as_uint(r.w) == kHoleOrig || !(__float_as_uint(r.z) & kActiveBit)) continue;
        const float x = P.pl[0][s].x;
        float fx;
        const int b = stencil_base(x, P.geo.origin[0], P.geo.inv_dx, fx);  // math.hpp:219-224
        if (b >= lo && b < hi) continue;
        const int side = b < lo ? 0 : 1;
        const uint32_t k = atomicAdd(&counts[side], 1u);
        if (k >= cap) continue;  // overflow: reported by the count, the host fails loudly
        float4* out = (side == 0 ? out_lo : out_hi) + static_cast<uint64_t>(k) * kPlanes;
#pragma unroll
        for (int q = 0; q < kPlanes; ++q) out[q] = P.pl[q][s];
#pragma unroll
        for (int q = 0; q < PR; ++q) P.pl[q][s] = make_float4(0.f, 0.f, 0.f, 0.f);
        P.pl[PR][s] = make_float4(0.f, 0.f, 0.f, __uint_as_float(kHoleOrig));
    }
}

void launch_migrate_pack(const Params& P, int lo, int hi, float4* out_lo, float4* out_hi, uint32_t cap,
                         uint32_t* counts, cudaStream_t st) {
    k_migrate_pack<<<dd_blocks(P.n_total, 256), 256, 0, st>>>(P, lo, hi, out_lo, out_hi, cap, counts);
    MPMB_LAUNCHED("k_migrate_pack");
}

// Received particles into the holes past the last occupied slot (slots [first, first + n)).
__global__ void k_migrate_unpack(const Params P, const float4* in, uint32_t n, uint32_t first) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t s = first + i;
#pragma unroll
        for (int q = 0; q < kPlanes; ++q) P.pl[q][s] = in[static_cast<uint64_t>(i) * kPlanes + q];
    }
}

void launch_migrate_unpack(const Params& P, const float4* in, uint32_t n, uint32_t first, cudaStream_t st) {
    if (n == 0) return;
    k_migrate_unpack<<<dd_blocks(n, 256), 256, 0, st>>>(P, in, n, first);
    MPMB_LAUNCHED("k_migrate_unpack");
}

// ---------------------------------------------------------------------------------
// Device-resident migration (the C++ driver, dd_driver.cpp): counts never visit the host.
// ctl = the slab's DD control words (b_counts + 4, launch.h): [0] free slot, [1] arrivals
// since binning, [2] error flags (kDdErr*), [3] particles on the slab.
// counts = {sent down, sent up, received from below, received from above}.

__global__ void k_window_init(int* w) {
    w[0] = INT_MAX; w[1] = INT_MIN; w[2] = INT_MAX; w[3] = INT_MIN;
    w[4] = w[5] = w[6] = w[7] = 0;
}

__global__ void k_add_f64(double* dst, const double* src, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[i] += src[i];
}
__global__ void k_add_i32(int32_t* dst, const int32_t* src, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        dst[i] += src[i];
}
// the empty window (INT_MAX, INT_MIN) negates to INT_MIN + 1 .. fine for MIN; INT_MIN itself
// has no negation, so the hi ends are clamped first
__global__ void k_window_min_form(int32_t* w, const uint32_t* ctl) {
    w[1] = -max(w[1], INT_MIN + 1);
    w[3] = -max(w[3], INT_MIN + 1);
    w[4] = -static_cast<int32_t>(ctl[2] & 0x7FFFFFFFu);
}
__global__ void k_window_from_min_form(int32_t* w) {
    w[1] = -w[1];
    w[3] = -w[3];
    w[4] = -w[4];
}

void dd_add_f64(double* dst, const double* src, int64_t n, void* stream) {
    if (n <= 0) return;
    k_add_f64<<<dd_blocks(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, src, n);
    MPMB_LAUNCHED("k_add_f64");
}
void dd_add_i32(int32_t* dst, const int32_t* src, int64_t n, void* stream) {
    if (n <= 0) return;
    k_add_i32<<<dd_blocks(n, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, src, n);
    MPMB_LAUNCHED("k_add_i32");
}
void dd_window_to_min_form(int32_t* w, const uint32_t* ctl, void* stream) {
    k_window_min_form<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(w, ctl);
    MPMB_LAUNCHED("k_window_min_form");
}
void dd_window_from_min_form(int32_t* w, void* stream) {
    k_window_from_min_form<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(w);
    MPMB_LAUNCHED("k_window_from_min_form");
}

void launch_window_init(int* w, cudaStream_t st) {
    k_window_init<<<1, 1, 0, st>>>(w);
    MPMB_LAUNCHED("k_window_init");
}

// Pack the particles whose stencil base left [lo, hi) (as k_migrate_pack) and check the
// reach every particle's stencil had since the window was set: base x inside the stored
// planes [lo - M, hi + M) and base y / z inside the halo window [y0, y1 - 2) x [z0, z1 - 2)
// (otherwise P2G clamped it or its ghost sums did not travel: kDdErrReach).
__global__ void k_migrate_pack_dev(const Params P, int lo, int hi, int margin, int4 win, int has_lo, int has_hi,
                                   float4* out_lo, float4* out_hi, uint32_t cap, uint32_t* counts, uint32_t* ctl) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    uint32_t err = 0;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        const float4 r = P.pl[PR][s];
        if (__float_as_uint(r.w) == kHoleOrig || !(__float_as_uint(r.z) & kActiveBit)) continue;
        const float4 a = P.pl[0][s];
        float f;
        const int b = stencil_base(a.x, P.geo.origin[0], P.geo.inv_dx, f);  // math.hpp:219-224
        const int by = stencil_base(a.y, P.geo.origin[1], P.geo.inv_dx, f);
        const int bz = stencil_base(a.z, P.geo.origin[2], P.geo.inv_dx, f);
        if (b < lo - margin || b >= hi + margin || by < win.x || by + 3 > win.y || bz < win.z || bz + 3 > win.w)
            err |= kDdErrReach;
        if (b >= lo && b < hi) continue;
        const int side = b < lo ? 0 : 1;
        if (!(side == 0 ? has_lo : has_hi)) {
            err |= kDdErrLeftDomain;
            continue;
        }
        const uint32_t k = atomicAdd(&counts[side], 1u);
        if (k >= cap) {
            err |= kDdErrMigrationOverflow;
            continue;
        }
        float4* out = (side == 0 ? out_lo : out_hi) + static_cast<uint64_t>(k) * kPlanes;
#pragma unroll
        for (int q = 0; q < kPlanes; ++q) out[q] = P.pl[q][s];
#pragma unroll
        for (int q = 0; q < PR; ++q) P.pl[q][s] = make_float4(0.f, 0.f, 0.f, 0.f);
        P.pl[PR][s] = make_float4(0.f, 0.f, 0.f, __uint_as_float(kHoleOrig));
    }
    if (err) atomicOr(&ctl[2], err);
}

void launch_migrate_pack_dev(const Params& P, int lo, int hi, int margin, int4 win, bool has_lo, bool has_hi,
                             float4* out_lo, float4* out_hi, uint32_t cap, uint32_t* counts, uint32_t* ctl,
                             cudaStream_t st) {
    k_migrate_pack_dev<<<dd_blocks(P.n_total, 256), 256, 0, st>>>(P, lo, hi, margin, win, has_lo ? 1 : 0,
                                                                    has_hi ? 1 : 0, out_lo, out_hi, cap, counts, ctl);
    MPMB_LAUNCHED("k_migrate_pack_dev");
}

// Arrivals start a fresh transfer group: inside a group the transfers place the particle of
// sorted position p at slot group_phys(p), so a partly filled group does not keep its
// particles in its first slots and nothing may be appended behind them.
__device__ __forceinline__ uint64_t round_up_group(uint64_t s) {
    return (s + kGroup - 1) / kGroup * kGroup;
}

// Arrivals (counts[2] from below, counts[3] from above) appended at the first group boundary
// at or past the free slot, into BOTH plane buffers (the transfers rewrite grouped slots
// only, which must start identical).
__global__ void k_migrate_unpack_dev(const Params P, const float4* in_lo, const float4* in_hi, uint32_t cap,
                                     const uint32_t* counts, const uint32_t* ctl, uint32_t* ctl_err) {
    const uint32_t n0 = min(counts[2], cap), n1 = min(counts[3], cap);
    const uint64_t first = round_up_group(ctl[0]);
    const int64_t n = static_cast<int64_t>(n0) + n1;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t slot = first + static_cast<uint64_t>(i);
        if (slot >= static_cast<uint64_t>(P.n_total)) {
            atomicOr(ctl_err, kDdErrCapacity);
            continue;
        }
        const float4* src = i < n0 ? in_lo + static_cast<uint64_t>(i) * kPlanes
                                   : in_hi + static_cast<uint64_t>(i - n0) * kPlanes;
#pragma unroll
        for (int q = 0; q < kPlanes; ++q) {
            const float4 v = src[q];
            P.pl[q][slot] = v;
            P.pl_out[q][slot] = v;
        }
    }
}

// One thread: free slot, arrival and particle counts, and the transfer groups, which grow to
// cover the appended slots (their group sort puts holes and inactive particles last).
__global__ void k_migrate_finalize(uint32_t* bcounts, uint32_t cap, const uint32_t* counts, uint64_t n_cap) {
    uint32_t* ctl = bcounts + 4;
    const uint32_t sent = min(counts[0], cap) + min(counts[1], cap);
    const uint32_t arr = min(counts[2], cap) + min(counts[3], cap);
    if (arr == 0) {
        ctl[3] -= sent;
        return;
    }
    uint64_t fs = round_up_group(round_up_group(ctl[0]) + arr);  // the arrivals' groups are closed
    if (fs > n_cap) {
        ctl[2] |= kDdErrCapacity;
        fs = n_cap;
    }
    ctl[0] = static_cast<uint32_t>(fs);
    ctl[1] += arr;
    ctl[3] = ctl[3] + arr - sent;
    const uint32_t groups = static_cast<uint32_t>(fs / kGroup);
    if (groups > bcounts[1]) {
        bcounts[1] = groups;
        bcounts[3] = groups * static_cast<uint32_t>(kGroup);
    }
}

void launch_migrate_unpack_dev(const Params& P, const float4* in_lo, const float4* in_hi, uint32_t cap,
                               const uint32_t* counts, uint32_t* bcounts, uint64_t n_cap, cudaStream_t st) {
    k_migrate_unpack_dev<<<dd_blocks(2 * static_cast<int64_t>(cap), 256), 256, 0, st>>>(P, in_lo, in_hi, cap, counts,
                                                                                          bcounts + 4, bcounts + 6);
    MPMB_LAUNCHED("k_migrate_unpack_dev");
    k_migrate_finalize<<<1, 1, 0, st>>>(bcounts, cap, counts, n_cap);
    MPMB_LAUNCHED("k_migrate_finalize");
}

// The slab's particles compacted (warp-aggregated append, any order): original index, x,
// v, active; *count = how many.
__global__ void k_download_slots(const Params P, uint32_t* ids, float* x, float* v, uint8_t* active,
                                 uint32_t* count) {
    const unsigned full = 0xffffffffu;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < P.n_total; base += stride) {
        const int64_t s = base + threadIdx.x;
        float4 r = make_float4(0.f, 0.f, 0.f, __uint_as_float(kHoleOrig));
        if (s < P.n_total) r = P.pl[PR][s];
        const bool real = __float_as_uint(r.w) != kHoleOrig;
        const unsigned m = __ballot_sync(full, real);
        if (!m) continue;
        uint32_t start = 0;
        if ((threadIdx.x & 31) == 0) start = atomicAdd(count, __popc(m));
        start = __shfl_sync(full, start, 0);
        if (!real) continue;
        const uint64_t k = start + __popc(m & lanemask_lt());
        const float4 a = P.pl[0][s], b = P.pl[1][s];
        ids[k] = __float_as_uint(r.w);
        x[3 * k] = a.x; x[3 * k + 1] = a.y; x[3 * k + 2] = a.z;
        v[3 * k] = a.w; v[3 * k + 1] = b.x; v[3 * k + 2] = b.y;
        active[k] = (__float_as_uint(r.z) & kActiveBit) ? 1 : 0;
    }
}

void launch_download_slots(const Params& P, uint32_t* ids, float* x, float* v, uint8_t* active, uint32_t* count,
                           cudaStream_t st) {
    k_download_slots<<<dd_blocks(P.n_total, 256), 256, 0, st>>>(P, ids, x, v, active, count);
    MPMB_LAUNCHED("k_download_slots");
}

}  // namespace mpmb
