// k_scenario.cu — the scenario-harness metrics on the device:
// compute_components (scenario.hpp:100-139) and mean_nearest_neighbor_spacing
// (scenario.hpp:68-96) over the engine's resident particles, every scene of a batch at once.
//
// Both use the reference's spatial hash exactly: cell = floor(x / cell_size) per axis (float
// division), masked to 21 bits and packed (scenario.hpp:30-35); the candidates of particle
// i are the particles of the cells holding the probes p_i + d * cell, d in {-1,0,1}^3
// (float mul, then add; scenario.hpp:82-84, 112-114), tested with the float squared
// distance (x*x + y*y) + z*z.  Identical candidate sets and tests make the component count
// exact (union-find connectivity does not depend on the order of unions) and every
// nearest-neighbour distance bit-identical; the FP64 mean of the distances is summed on
// the host in original particle order, as the reference does.
//
// Pipeline: keys (scene-salted 64-bit hash of the cell) -> CUB radix sort of (key, slot)
// -> per particle 27 probes, binary search, full-key check -> lock-free union-find
// (CAS-hooking the larger root under the smaller) -> flatten -> component sizes -> per
// scene count of components holding >= ceil(5% of the scene's active particles).
#include <cuda_runtime.h>

#include <cfloat>
#include <cub/device/device_radix_sort.cuh>

#include "launch.h"

namespace mpmb {

namespace {

__device__ __forceinline__ uint64_t cell_key(float x, float y, float z, float cell) {
    auto q = [cell](float v) -> uint64_t {
        return static_cast<uint64_t>(static_cast<int64_t>(floorf(__fdiv_rn(v, cell))) & 0x1fffff);
    };
    return q(x) | (q(y) << 21) | (q(z) << 42);
}

__device__ __forceinline__ uint64_t salt(uint64_t k, uint32_t scene) {
    uint64_t h = k ^ (static_cast<uint64_t>(scene) * 0x9E3779B97F4A7C15ull);
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    return h == ~0ull ? h - 1 : h;  // ~0 marks "no particle"
}

__device__ __forceinline__ float dist2(float4 a, float4 b) {
    const float dx = __fsub_rn(a.x, b.x), dy = __fsub_rn(a.y, b.y), dz = __fsub_rn(a.z, b.z);
    return __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
}

__device__ __forceinline__ bool live(const Params& P, int64_t s, uint32_t& scene) {
    const float4 r = P.pl[PR][s];
    const uint32_t f = __float_as_uint(r.z);
    scene = (f >> kSceneShift) & kSceneMask;
    return __float_as_uint(r.w) != kHoleOrig && (f & kActiveBit);
}

// per slot: hashed key (sorted last when not an active particle), full cell key, slot id
__global__ void k_cc_keys(const Params P, const float* cell, uint64_t* hkey, uint64_t* ckey, uint32_t* val,
                          int* parent, uint32_t* n_act) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        uint32_t sc;
        val[s] = static_cast<uint32_t>(s);
        parent[s] = static_cast<int>(s);
        if (!live(P, s, sc)) {
            hkey[s] = ~0ull;
            continue;
        }
        const float4 a = P.pl[0][s];
        const uint64_t k = cell_key(a.x, a.y, a.z, cell[sc]);
        ckey[s] = k;
        hkey[s] = salt(k, sc);
        atomicAdd(&n_act[sc], 1u);
    }
}

__device__ __forceinline__ int64_t lower_bound(const uint64_t* a, int64_t n, uint64_t k) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ int find_root(int* parent, int x) {
    volatile int* p = parent;
    while (true) {
        const int q = p[x];
        if (q == x) return x;
        const int g = p[q];
        if (g != q) atomicCAS(&parent[x], q, g);  // path halving
        x = q;
    }
}

__device__ void unite(int* parent, int a, int b) {
    while (true) {
        a = find_root(parent, a);
        b = find_root(parent, b);
        if (a == b) return;
        if (a > b) {
            const int t = a;
            a = b;
            b = t;
        }
        if (atomicCAS(&parent[b], b, a) == b) return;
    }
}

// MODE 0: unite every pair within `cell` (compute_components); MODE 1: nearest neighbour
// distance^2 per particle (mean_nearest_neighbor_spacing), j != i
template <int MODE>
__global__ void k_cc_probe(const Params P, const float* cell, const uint64_t* skey, const uint32_t* sval,
                           const uint64_t* ckey, int* parent, float* best2_out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        uint32_t sc;
        if (!live(P, s, sc)) continue;
        const float c = cell[sc];
        const float r2 = __fmul_rn(c, c);
        const float4 pi = P.pl[0][s];
        float best2 = FLT_MAX;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const float px = __fadd_rn(pi.x, __fmul_rn(static_cast<float>(dx), c));
                    const float py = __fadd_rn(pi.y, __fmul_rn(static_cast<float>(dy), c));
                    const float pz = __fadd_rn(pi.z, __fmul_rn(static_cast<float>(dz), c));
                    const uint64_t k = cell_key(px, py, pz, c);
                    const uint64_t h = salt(k, sc);
                    for (int64_t t = lower_bound(skey, P.n_total, h); t < P.n_total && skey[t] == h; ++t) {
                        const uint32_t j = sval[t];
                        uint32_t scj;
                        live(P, j, scj);
                        if (ckey[j] != k || scj != sc) continue;  // hash collision
                        const float d2 = dist2(pi, P.pl[0][j]);
                        if (MODE == 0) {
                            if (d2 <= r2) unite(parent, static_cast<int>(s), static_cast<int>(j));
                        } else if (j != static_cast<uint32_t>(s) && d2 < best2) {
                            best2 = d2;
                        }
                    }
                }
        if (MODE == 1) best2_out[s] = best2;
    }
}

__global__ void k_cc_sizes(const Params P, int* parent, uint32_t* size) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        uint32_t sc;
        if (!live(P, s, sc)) continue;
        const int r = find_root(parent, static_cast<int>(s));
        atomicAdd(&size[r], 1u);
    }
}

__global__ void k_cc_count(const Params P, const int* parent, const uint32_t* size, const uint32_t* n_act,
                           int32_t* count) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        uint32_t sc;
        if (!live(P, s, sc) || parent[s] != static_cast<int>(s)) continue;
        // threshold = ceil(0.05 * n_active) in double, as scenario.hpp:133-134
        const uint64_t thr = static_cast<uint64_t>(ceil(0.05 * static_cast<double>(n_act[sc])));
        if (size[s] >= thr) atomicAdd(&count[sc], 1);
    }
}

__global__ void k_cc_orig(const Params P, uint32_t* orig) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride)
    {
        uint32_t sc;
        orig[s] = live(P, s, sc) ? __float_as_uint(P.pl[PR][s].w) : kHoleOrig;  // active particles only
    }
}

int blocks(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return static_cast<int>(b);
}

}  // namespace

// Scratch for one call (device): sized for n slots and s scenes.
struct CcScratch {
    uint64_t *hkey, *skey, *ckey;
    uint32_t *val, *sval, *size, *n_act;
    int* parent;
    void* temp;
    size_t temp_bytes;
};

size_t cc_temp_bytes(int64_t n) {
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                                    static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                    static_cast<int>(n));
    return b;
}

// mode 0: components per scene into count[]; mode 1: nearest-neighbour d^2 per slot into
// best2[] and the slot's original index into orig[]
void launch_scenario(const Params& P, int mode, const float* cell, void* scratch_mem, size_t scratch_bytes,
                     int32_t* count, float* best2, uint32_t* orig, int n_scenes, cudaStream_t st) {
    const int64_t n = P.n_total;
    char* m = static_cast<char*>(scratch_mem);
    auto take = [&m](size_t b) {
        char* p = m;
        m += (b + 255) & ~static_cast<size_t>(255);
        return p;
    };
    CcScratch S{};
    S.hkey = reinterpret_cast<uint64_t*>(take(8 * n));
    S.skey = reinterpret_cast<uint64_t*>(take(8 * n));
    S.ckey = reinterpret_cast<uint64_t*>(take(8 * n));
    S.val = reinterpret_cast<uint32_t*>(take(4 * n));
    S.sval = reinterpret_cast<uint32_t*>(take(4 * n));
    S.size = reinterpret_cast<uint32_t*>(take(4 * n));
    S.parent = reinterpret_cast<int*>(take(4 * n));
    S.n_act = reinterpret_cast<uint32_t*>(take(4 * static_cast<size_t>(n_scenes)));
    S.temp_bytes = cc_temp_bytes(n);
    S.temp = take(S.temp_bytes);
    (void)scratch_bytes;
    cudaMemsetAsync(S.n_act, 0, 4 * static_cast<size_t>(n_scenes), st);
    cudaMemsetAsync(S.size, 0, 4 * n, st);
    k_cc_keys<<<blocks(n), 256, 0, st>>>(P, cell, S.hkey, S.ckey, S.val, S.parent, S.n_act);
    MPMB_LAUNCHED("k_cc_keys");
    cub::DeviceRadixSort::SortPairs(S.temp, S.temp_bytes, S.hkey, S.skey, S.val, S.sval, static_cast<int>(n), 0, 64,
                                    st);
    if (mode == 0) {
        k_cc_probe<0><<<blocks(n), 256, 0, st>>>(P, cell, S.skey, S.sval, S.ckey, S.parent, nullptr);
        MPMB_LAUNCHED("k_cc_probe");
        k_cc_sizes<<<blocks(n), 256, 0, st>>>(P, S.parent, S.size);
        MPMB_LAUNCHED("k_cc_sizes");
        cudaMemsetAsync(count, 0, 4 * static_cast<size_t>(n_scenes), st);
        k_cc_count<<<blocks(n), 256, 0, st>>>(P, S.parent, S.size, S.n_act, count);
        MPMB_LAUNCHED("k_cc_count");
    } else {
        k_cc_probe<1><<<blocks(n), 256, 0, st>>>(P, cell, S.skey, S.sval, S.ckey, S.parent, best2);
        MPMB_LAUNCHED("k_cc_probe");
        k_cc_orig<<<blocks(n), 256, 0, st>>>(P, orig);
        MPMB_LAUNCHED("k_cc_orig");
    }
}

size_t scenario_scratch_bytes(int64_t n, int n_scenes) {
    const size_t a = 3 * 8 * n + 4 * 4 * n + 4 * static_cast<size_t>(n_scenes) + cc_temp_bytes(n);
    return a + 16 * 256;
}

}  // namespace mpmb
