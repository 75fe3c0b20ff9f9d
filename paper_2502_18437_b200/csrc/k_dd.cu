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
