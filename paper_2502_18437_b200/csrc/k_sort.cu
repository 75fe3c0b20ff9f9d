// k_sort.cu — K1: particle binning / stable sort by (brick, cell, original index), run once
// per frame (or per resort interval); P2G refines each 256-slot group every substep.  No reference function exists for
// this stage (the reference transfers in particle-index order, solvers.hpp:151); the
// key arithmetic is the reference's stencil base (math.hpp:219-223, bit-exact).
//
// Pipeline (all on device, no host round trip):
//   keys      bucket = brick of the stencil base, warp-aggregated rank in the bucket
//   scan      bucket offsets (exclusive scan; the inactive bucket is last)
//   scatter   entries to their bucket
//   local     per bucket: counting sort by cell (64 bins) + rank by original index in
//             the cell -> (brick, cell, original index) order
//   gather    physical permutation of the 7 planes into that order
#include <cuda_runtime.h>

#include "launch.h"

namespace mpmb {

// ------------------------------------------------------------------- scan
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t& total) {
    constexpr int NW = kScanThreads / 32;
    __shared__ uint32_t warp_tot[NW + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const uint32_t w = lane < NW ? warp_tot[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < NW) warp_tot[lane] = wi - w;
        if (lane == NW - 1) warp_tot[NW] = wi;
    }
    __syncthreads();
    const uint32_t excl = warp_tot[wid] + inc - v;
    total = warp_tot[NW];
    __syncthreads();
    return excl;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t* in, int64_t n,
                                                              uint32_t* sums) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i)
        if (base + i < n) s += in[base + i];
    uint32_t total;
    block_exclusive_scan(s, total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// single block: exclusive scan of the tile sums in place
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(uint32_t* sums, int n) {
    uint32_t carry = 0;
    for (int base = 0; base < n; base += kScanThreads) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < n ? sums[i] : 0u;
        uint32_t total;
        const uint32_t e = block_exclusive_scan(v, total);
        if (i < n) sums[i] = carry + e;
        carry += total;
    }
    if (threadIdx.x == 0) sums[n] = carry;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint32_t* in, int64_t n,
                                                            const uint32_t* sums, uint32_t* out,
                                                            int n_tiles) {
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
    uint32_t vals[kScanItems];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        vals[i] = base + i < n ? in[base + i] : 0u;
        s += vals[i];
    }
    uint32_t total;
    uint32_t e = block_exclusive_scan(s, total) + sums[blockIdx.x];
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = e;
        e += vals[i];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = sums[n_tiles];
}

void launch_exclusive_scan(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* tmp,
                           cudaStream_t st, int64_t* launches) {
    const int tiles = static_cast<int>((n + kScanTile - 1) / kScanTile);
    const int t = tiles > 0 ? tiles : 1;
    k_scan_reduce<<<t, kScanThreads, 0, st>>>(in, n, tmp);
    MPMB_LAUNCHED("k_scan_reduce");
    k_scan_sums<<<1, kScanThreads, 0, st>>>(tmp, t);
    MPMB_LAUNCHED("k_scan_sums");
    k_scan_down<<<t, kScanThreads, 0, st>>>(in, n, tmp, out, t);
    MPMB_LAUNCHED("k_scan_down");
    *launches += 3;
}

// ------------------------------------------------------------------- keys
__global__ void __launch_bounds__(256) k_bin_keys(const Params P, BinBuffers B) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < P.n_total; base += stride) {
        const int64_t s = base + threadIdx.x;
        const bool valid = s < P.n_total;
        uint32_t bucket = 0xFFFFFFFFu, cell = 0, orig = 0;
        if (valid) {
            const float4 r = P.pl[PR][s];
            const uint32_t flags = __float_as_uint(r.z);
            orig = __float_as_uint(r.w);
            if (orig == kHoleOrig) {
                bucket = B.n_buckets - 1;  // empty slot: sorted last, never gathered
            } else if (flags & kActiveBit) {
                const int scene = static_cast<int>((flags >> kSceneShift) & kSceneMask);
                const SceneView S = scene_view(P, scene);
                const float4 a = P.pl[0][s];
                const float x[3] = {a.x, a.y, a.z};
                int b[3];
                float fx[3];
                local_base(P.geo, x, b, fx);
                const uint32_t local = (static_cast<uint32_t>(b[2] >> 2) * S.nb[1] +
                                        static_cast<uint32_t>(b[1] >> 2)) * S.nb[0] +
                                       static_cast<uint32_t>(b[0] >> 2);
                bucket = S.brick_base + local;
                cell = static_cast<uint32_t>(((b[2] & 3) << 4) | ((b[1] & 3) << 2) | (b[0] & 3));
                if (B.key_by_orig) B.key_by_orig[orig] = (local << 6) | cell;
            } else {
                bucket = B.n_buckets - 2;
                if (B.key_by_orig) B.key_by_orig[orig] = 0xFFFFFFFFu;
            }
        }
        // warp-aggregated rank inside the bucket (sorted input: usually one bucket per warp)
        const unsigned peers = __match_any_sync(full, bucket);
        const int leader = __ffs(peers) - 1;
        uint32_t start = 0;
        if (valid && lane == leader) start = atomicAdd(&B.bucket_count[bucket], __popc(peers));
        start = __shfl_sync(full, start, leader);
        if (valid) {
            B.key[s] = bucket;
            B.rank[s] = start + __popc(peers & lanemask_lt());
            B.cell[s] = static_cast<uint8_t>(cell);
            B.orig[s] = orig;
        }
    }
}

__global__ void __launch_bounds__(256) k_bin_scatter(BinBuffers B, int64_t n) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < n; s += stride) {
        const uint32_t pos = B.bucket_off[B.key[s]] + B.rank[s];
        B.e_orig[pos] = B.orig[s];
        B.e_cell[pos] = B.cell[s];
        B.e_src[pos] = static_cast<uint32_t>(s);
    }
}

// One block per bucket (grid-stride): counting sort by cell, then rank by original index.
// Inactive particles keep their bucket order (grid-wide copy: the bucket can be large);
// holes need no sorted entry (the gather fills everything past the real particles).
__global__ void __launch_bounds__(256) k_bin_rest(BinBuffers B) {
    const uint32_t beg = B.bucket_off[B.n_buckets - 2], end = B.bucket_off[B.n_buckets - 1];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t q = beg + blockIdx.x * blockDim.x + threadIdx.x; q < end; q += stride) {
        B.sorted_src[q] = B.e_src[q];
        B.sorted_orig[q] = B.e_orig[q];
    }
}

// Buckets of at most kLocalCap entries sort in shared memory: counting sort by cell (atomic
// ranks), then each entry's rank inside its cell by original index (cells hold ~8 entries).
// Larger buckets take the same steps through global scratch.
constexpr int kLocalCap = 2048;
constexpr int kLocalPer = kLocalCap / 256;
__global__ void __launch_bounds__(256) k_bin_local(BinBuffers B) {
    __shared__ uint32_t hist[64];
    __shared__ uint32_t cstart[64];
    __shared__ uint32_t s_orig[kLocalCap];
    __shared__ uint32_t s_src[kLocalCap];
    __shared__ uint8_t s_cell[kLocalCap];
    __shared__ uint32_t s_list[256];
    __shared__ uint32_t s_n;
    const uint32_t inactive = B.n_buckets - 2;  // the inactive and hole buckets: k_bin_rest
    // most bricks are empty: each block scans 256 buckets at a time (coalesced offsets), lists
    // the non-empty ones, then sorts them one by one
    for (uint32_t base = blockIdx.x * 256u; base < inactive; base += gridDim.x * 256u) {
        if (threadIdx.x == 0) s_n = 0u;
        __syncthreads();
        {
            const uint32_t b = base + threadIdx.x;
            const bool ne = b < inactive && B.bucket_off[b + 1] > B.bucket_off[b];
            const unsigned m = __ballot_sync(0xffffffffu, ne);
            uint32_t w0 = 0;
            if ((threadIdx.x & 31) == 0 && m) w0 = atomicAdd(&s_n, static_cast<uint32_t>(__popc(m)));
            w0 = __shfl_sync(0xffffffffu, w0, 0);
            if (ne) s_list[w0 + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = b;
        }
        __syncthreads();
        const uint32_t n_list = s_n;
        for (uint32_t li = 0; li < n_list; ++li) {
            const uint32_t b = s_list[li];
            const uint32_t beg = B.bucket_off[b], end = B.bucket_off[b + 1];
            const bool local = end - beg <= static_cast<uint32_t>(kLocalCap);
            if (threadIdx.x < 64) hist[threadIdx.x] = 0u;
            __syncthreads();
            uint32_t cr[kLocalPer];  // shared-memory path: cell << 16 | rank of this thread's entries
            if (local) {
#pragma unroll
                for (int i = 0; i < kLocalPer; ++i) {
                    const uint32_t q = beg + threadIdx.x + 256u * i;
                    cr[i] = 0xFFFFFFFFu;
                    if (q < end) {
                        const uint32_t cl = B.e_cell[q];
                        cr[i] = (cl << 16) | atomicAdd(&hist[cl], 1u);
                    }
                }
            } else {
                for (uint32_t q = beg + threadIdx.x; q < end; q += blockDim.x)
                    B.tmp[q] = atomicAdd(&hist[B.e_cell[q]], 1u);
            }
            __syncthreads();
            if (threadIdx.x < 32) {  // exclusive scan of 64 bins by one warp
                const uint32_t a = hist[2 * threadIdx.x], cc = hist[2 * threadIdx.x + 1];
                uint32_t inc = a + cc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
                    if (threadIdx.x >= o) inc += t;
                }
                const uint32_t ex = inc - a - cc;
                cstart[2 * threadIdx.x] = ex;
                cstart[2 * threadIdx.x + 1] = ex + a;
            }
            __syncthreads();
            if (local) {
#pragma unroll
                for (int i = 0; i < kLocalPer; ++i) {
                    if (cr[i] == 0xFFFFFFFFu) continue;
                    const uint32_t q = beg + threadIdx.x + 256u * i;
                    const uint32_t cl = cr[i] >> 16;
                    const uint32_t d = cstart[cl] + (cr[i] & 0xFFFFu);
                    s_orig[d] = B.e_orig[q];
                    s_src[d] = B.e_src[q];
                    s_cell[d] = static_cast<uint8_t>(cl);
                }
                __syncthreads();
                for (uint32_t d = threadIdx.x; d < end - beg; d += blockDim.x) {
                    const uint32_t cl = s_cell[d];
                    const uint32_t o = s_orig[d];
                    const uint32_t lo = cstart[cl], hi = lo + hist[cl];
                    uint32_t rk = 0;
                    for (uint32_t f = lo; f < hi; ++f) rk += s_orig[f] < o ? 1u : 0u;
                    B.sorted_src[beg + lo + rk] = s_src[d];
                    B.sorted_orig[beg + lo + rk] = o;
                }
            } else {
                for (uint32_t q = beg + threadIdx.x; q < end; q += blockDim.x) {
                    const uint32_t cl = B.e_cell[q];
                    const uint32_t d = beg + cstart[cl] + B.tmp[q];
                    B.g_orig[d] = B.e_orig[q];
                    B.g_src[d] = B.e_src[q];
                    B.g_cell[d] = static_cast<uint8_t>(cl);
                }
                __syncthreads();
                for (uint32_t q = beg + threadIdx.x; q < end; q += blockDim.x) {
                    const uint32_t cl = B.g_cell[q];
                    const uint32_t o = B.g_orig[q];
                    const uint32_t lo = beg + cstart[cl], hi = lo + hist[cl];
                    uint32_t rk = 0;
                    for (uint32_t f = lo; f < hi; ++f) rk += B.g_orig[f] < o ? 1u : 0u;
                    B.sorted_src[lo + rk] = B.g_src[q];
                    B.sorted_orig[lo + rk] = o;
                }
            }
            __syncthreads();
        }
        __syncthreads();  // s_list / s_n are rewritten for the next range
    }
}

// Physical permutation of the 7 planes into the group layout (launch.h), and the counts
// the transfers read: [0] n_active, [1] transfer groups G, [2] n_active, [3] tail start
// G*kGroup.  Slots [0, G*kGroup): group g holds sorted entries g*kGroup + p at slot
// g*kGroup + group_phys(p), holes past n_active; then the inactive particles; then holes.
__global__ void __launch_bounds__(256) k_bin_gather(const Params P, BinBuffers B, int64_t n_cap,
                                                    float4* n0, float4* n1, float4* n2, float4* n3,
                                                    float4* n4, float4* n5, float4* n6) {
    float4* np[kPlanes] = {n0, n1, n2, n3, n4, n5, n6};
    const uint32_t n_active = B.bucket_off[B.n_buckets - 2];
    const uint32_t n_real = B.bucket_off[B.n_buckets - 1];
    const uint32_t groups = (n_active + kGroup - 1) / kGroup;
    const uint32_t tail = groups * kGroup;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        B.counts[0] = n_active;
        B.counts[1] = groups;
        B.counts[2] = n_active;
        B.counts[3] = tail;
        B.counts[4] = tail + (n_real - n_active);  // DD: first free slot (launch.h)
        B.counts[5] = 0;                           // DD: arrivals since binning
        B.counts[7] = n_real;                      // DD: particles on the slab
    }
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t d = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; d < n_cap; d += stride) {
        uint32_t src = kHoleOrig;
        if (d < tail) {
            const uint32_t q = static_cast<uint32_t>(d / kGroup) * kGroup +
                               group_pos(static_cast<uint32_t>(d % kGroup));
            if (q < n_active) src = B.sorted_src[q];
        } else if (d < static_cast<int64_t>(tail) + (n_real - n_active)) {
            src = B.sorted_src[n_active + static_cast<uint32_t>(d - tail)];
        }
        if (src != kHoleOrig) {
            MPMB_DCHECK(src < static_cast<uint64_t>(P.n_total));
#pragma unroll
            for (int p = 0; p < kPlanes; ++p) np[p][d] = P.pl[p][src];
        } else {
#pragma unroll
            for (int p = 0; p < PR; ++p) np[p][d] = make_float4(0.f, 0.f, 0.f, 0.f);
            np[PR][d] = make_float4(0.f, 0.f, 0.f, __uint_as_float(kHoleOrig));
        }
    }
}

// The transfers rewrite only the grouped slots each substep (G2P into the other buffer);
// the tail (inactive particles + holes) must be identical in both buffers.
// Q.pl = the freshly gathered buffer, Q.pl_out = the other one.
__global__ void __launch_bounds__(256) k_bin_tail(const Params Q, BinBuffers B, int64_t n_cap) {
    const int64_t tail = B.counts[3];
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t d = tail + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; d < n_cap; d += stride) {
#pragma unroll
        for (int p = 0; p < kPlanes; ++p) Q.pl_out[p][d] = Q.pl[p][d];
    }
}

static int blocks_for(int64_t n, int threads, int cap) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return static_cast<int>(b);
}

void launch_bin(const Params& P, const BinBuffers& B, float4* const new_planes[kPlanes],
                int64_t n_total, cudaStream_t st, int64_t* launches) {
    // n_total: slot capacity of both buffers (particles + holes)
    cudaMemsetAsync(B.bucket_count, 0, sizeof(uint32_t) * B.n_buckets, st);
    const int cap = 148 * 16;
    k_bin_keys<<<blocks_for(n_total, 256, cap), 256, 0, st>>>(P, B);
    MPMB_LAUNCHED("k_bin_keys");
    launch_exclusive_scan(B.bucket_count, B.bucket_off, B.n_buckets, B.scan_tmp, st, launches);
    k_bin_scatter<<<blocks_for(n_total, 256, cap), 256, 0, st>>>(B, n_total);
    MPMB_LAUNCHED("k_bin_scatter");
    k_bin_local<<<blocks_for(static_cast<int64_t>(B.n_buckets), 256, 148 * 8), 256, 0, st>>>(B);
    MPMB_LAUNCHED("k_bin_local");
    k_bin_rest<<<blocks_for(n_total, 256, cap), 256, 0, st>>>(B);
    MPMB_LAUNCHED("k_bin_rest");
    k_bin_gather<<<blocks_for(n_total, 256, cap), 256, 0, st>>>(
        P, B, n_total, new_planes[0], new_planes[1], new_planes[2], new_planes[3],
        new_planes[4], new_planes[5], new_planes[6]);
    MPMB_LAUNCHED("k_bin_gather");
    Params Q = P;
    for (int q = 0; q < kPlanes; ++q) {
        Q.pl_out[q] = P.pl[q];
        Q.pl[q] = new_planes[q];
    }
    k_bin_tail<<<blocks_for(n_total / 8, 256, cap), 256, 0, st>>>(Q, B, n_total);
    MPMB_LAUNCHED("k_bin_tail");
    *launches += 6;
}

}  // namespace mpmb
