// k_io.cu — boundary kernels: original-order upload/download of the ParticleStore
// (state.hpp:65-90), FrameResult totals (scene.hpp:251-266), dense grid export/import
// for the GridHook adapter (solvers.hpp:19, 63).
#include <cuda_runtime.h>

#include "launch.h"

namespace mpmb {

static int blocks_for(int64_t n, int threads, int cap) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return static_cast<int>(b);
}

// Slot = original index (the layout before the first binning); slots [n, n_total) are holes.
__global__ void k_upload(const Params P, IoArrays in, int64_t n) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < P.n_total; i += stride) {
        if (i >= n) {
#pragma unroll
            for (int q = 0; q < PR; ++q) P.pl[q][i] = make_float4(0.f, 0.f, 0.f, 0.f);
            P.pl[PR][i] = make_float4(0.f, 0.f, 0.f, __uint_as_float(kHoleOrig));
            continue;
        }
        Part p;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            p.x[a] = in.x[3 * i + a];
            p.v[a] = in.v[3 * i + a];
        }
#pragma unroll
        for (int a = 0; a < 9; ++a) {
            p.F[a] = in.F[9 * i + a];
            p.C[a] = in.C[9 * i + a];
        }
        store_part(P, static_cast<uint32_t>(i), p);
        uint32_t flags = (static_cast<uint32_t>(in.mat[i]) & kMatMask) |
                         ((static_cast<uint32_t>(in.scene[i]) & kSceneMask) << kSceneShift);
        if (in.active[i]) flags |= kActiveBit;
        else if (in.keep_stress) flags |= kKeepStressBit;
        P.pl[PR][i] = make_float4(in.mass[i], in.vol0[i], __uint_as_float(flags),
                                  __uint_as_float(in.ids ? in.ids[i] : static_cast<uint32_t>(i)));
    }
}

__global__ void k_download(const Params P, IoArrays out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        const float4 r = P.pl[PR][s];
        const uint32_t flags = __float_as_uint(r.z);
        const uint32_t o32 = __float_as_uint(r.w);
        if (o32 == kHoleOrig) continue;
        const uint64_t o = o32;
        if (out.x || out.v) {  // P0 {x, v.x}, P1 {v.y, v.z, ...}: the FrameResult planes only
            const float4 a = P.pl[0][s], b = P.pl[1][s];
            if (out.x) { out.x[3 * o] = a.x; out.x[3 * o + 1] = a.y; out.x[3 * o + 2] = a.z; }
            if (out.v) { out.v[3 * o] = a.w; out.v[3 * o + 1] = b.x; out.v[3 * o + 2] = b.y; }
        }
        if (out.F || out.C) {
            Part p;
            load_part(P, static_cast<uint32_t>(s), p);
            if (out.F) for (int a = 0; a < 9; ++a) out.F[9 * o + a] = p.F[a];
            if (out.C) for (int a = 0; a < 9; ++a) out.C[9 * o + a] = p.C[a];
        }
        if (out.mass) out.mass[o] = r.x;
        if (out.vol0) out.vol0[o] = r.y;
        if (out.mat) out.mat[o] = static_cast<int32_t>(flags & kMatMask);
        if (out.active) out.active[o] = (flags & kActiveBit) ? 1 : 0;
        if (out.scene) out.scene[o] = static_cast<int32_t>((flags >> kSceneShift) & kSceneMask);
    }
}

// Per-scene double totals: mass, momentum[3], kinetic energy (scene.hpp:258-266).
// Slots are grouped by scene, so a block's slots belong to very few scenes: threads
// accumulate per "current scene" and the block reduces runs of equal scene through shared
// memory before one FP64 atomic per (block, scene, value) -- same-address atomics from
// every warp serialise in L2 and dominated the old per-warp version.
constexpr int kTotThreads = 256;
constexpr int kTotPerThread = 16;
__global__ void __launch_bounds__(kTotThreads) k_totals(const Params P, double* totals) {
    __shared__ double red[5][kTotThreads];
    __shared__ int scn[kTotThreads];
    const int64_t span = static_cast<int64_t>(kTotThreads) * kTotPerThread;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * span; base < P.n_total;
         base += static_cast<int64_t>(gridDim.x) * span) {
        double t[5] = {0, 0, 0, 0, 0};
        int scene = -1;
        for (int i = 0; i < kTotPerThread; ++i) {  // coalesced: stride blockDim per step
            const int64_t s = base + static_cast<int64_t>(i) * kTotThreads + threadIdx.x;
            if (s >= P.n_total) break;
            const float4 r = P.pl[PR][s];
            const uint32_t flags = __float_as_uint(r.z);
            if (!(flags & kActiveBit)) continue;
            const int sc = static_cast<int>((flags >> kSceneShift) & kSceneMask);
            if (sc != scene) {
                if (scene >= 0)
                    for (int q = 0; q < 5; ++q) atomicAdd(&totals[5 * scene + q], t[q]);
                scene = sc;
                for (int q = 0; q < 5; ++q) t[q] = 0.0;
            }
            const float4 a = P.pl[0][s], b = P.pl[1][s];
            const double m = r.x;
            const float vx = a.w, vy = b.x, vz = b.y;
            t[0] += m;
            t[1] += m * vx;
            t[2] += m * vy;
            t[3] += m * vz;
            t[4] += 0.5 * m * static_cast<double>(vx * vx + vy * vy + vz * vz);
        }
        // runs of equal scene across the block's threads are summed by thread 0
        scn[threadIdx.x] = scene;
        for (int q = 0; q < 5; ++q) red[q][threadIdx.x] = t[q];
        __syncthreads();
        if (threadIdx.x == 0) {
            int cur = -1;
            double acc[5] = {0, 0, 0, 0, 0};
            for (int k = 0; k < kTotThreads; ++k) {
                const int sc = scn[k];
                if (sc < 0) continue;
                if (sc != cur) {
                    if (cur >= 0)
                        for (int q = 0; q < 5; ++q) atomicAdd(&totals[5 * cur + q], acc[q]);
                    cur = sc;
                    for (int q = 0; q < 5; ++q) acc[q] = 0.0;
                }
                for (int q = 0; q < 5; ++q) acc[q] += red[q][k];
            }
            if (cur >= 0)
                for (int q = 0; q < 5; ++q) atomicAdd(&totals[5 * cur + q], acc[q]);
        }
        __syncthreads();
    }
}

// FrameResult (scene.hpp:251-266) in two passes: the slot of every original index (one
// scattered word per particle), then an original-order pass that gathers x, v, flags from
// those slots and writes the x / v / active staging coalesced, with the per-scene FP64 totals
// of k_totals.  (One slot-order pass with scattered 4-byte stores was 35% slower.)
__global__ void k_inv_perm(const Params P, uint32_t* inv, int64_t n) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        const uint32_t o = __float_as_uint(P.pl[PR][s].w);
        if (o != kHoleOrig && static_cast<int64_t>(o) < n) inv[o] = static_cast<uint32_t>(s);
    }
}

__global__ void __launch_bounds__(kTotThreads) k_frame_result_orig(const Params P, const uint32_t* inv, int64_t n,
                                                                   IoArrays out, double* totals) {
    __shared__ double red[5][kTotThreads];
    __shared__ int scn[kTotThreads];
    const int64_t span = static_cast<int64_t>(kTotThreads) * kTotPerThread;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * span; base < n; base += static_cast<int64_t>(gridDim.x) * span) {
        double t[5] = {0, 0, 0, 0, 0};
        int scene = -1;
        for (int i = 0; i < kTotPerThread; ++i) {
            const int64_t o = base + static_cast<int64_t>(i) * kTotThreads + threadIdx.x;
            if (o >= n) break;
            const uint32_t s = inv[o];
            const float4 r = P.pl[PR][s];
            const float4 a = P.pl[0][s], b = P.pl[1][s];
            const uint32_t flags = __float_as_uint(r.z);
            const bool act = (flags & kActiveBit) != 0;
            if (out.x) { out.x[3 * o] = a.x; out.x[3 * o + 1] = a.y; out.x[3 * o + 2] = a.z; }
            if (out.v) { out.v[3 * o] = a.w; out.v[3 * o + 1] = b.x; out.v[3 * o + 2] = b.y; }
            if (out.active) out.active[o] = act ? 1 : 0;
            if (!act || !totals) continue;
            const int sc = static_cast<int>((flags >> kSceneShift) & kSceneMask);
            if (sc != scene) {
                if (scene >= 0)
                    for (int q = 0; q < 5; ++q) atomicAdd(&totals[5 * scene + q], t[q]);
                scene = sc;
                for (int q = 0; q < 5; ++q) t[q] = 0.0;
            }
            const double m = r.x;
            const float vx = a.w, vy = b.x, vz = b.y;
            t[0] += m;
            t[1] += m * vx;
            t[2] += m * vy;
            t[3] += m * vz;
            t[4] += 0.5 * m * static_cast<double>(vx * vx + vy * vy + vz * vz);
        }
        if (!totals) continue;  // arrays only (block-uniform)
        scn[threadIdx.x] = scene;
        for (int q = 0; q < 5; ++q) red[q][threadIdx.x] = t[q];
        __syncthreads();
        if (threadIdx.x == 0) {
            int cur = -1;
            double acc[5] = {0, 0, 0, 0, 0};
            for (int k = 0; k < kTotThreads; ++k) {
                const int sc = scn[k];
                if (sc < 0) continue;
                if (sc != cur) {
                    if (cur >= 0)
                        for (int q = 0; q < 5; ++q) atomicAdd(&totals[5 * cur + q], acc[q]);
                    cur = sc;
                    for (int q = 0; q < 5; ++q) acc[q] = 0.0;
                }
                for (int q = 0; q < 5; ++q) acc[q] += red[q][k];
            }
            if (cur >= 0)
                for (int q = 0; q < 5; ++q) atomicAdd(&totals[5 * cur + q], acc[q]);
        }
        __syncthreads();
    }
}

// sigma(F) into an original-order array (materialises the cached stress, solvers.hpp:69-74).
__global__ void k_stress(const Params P, float* out) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s < P.n_total; s += stride) {
        const float4 r = P.pl[PR][s];
        const uint32_t flags = __float_as_uint(r.z);
        if (__float_as_uint(r.w) == kHoleOrig) continue;
        const uint64_t o = __float_as_uint(r.w);
        if (P.use_stress_in || (flags & kKeepStressBit)) {
            if (out != P.stress_in)
                for (int a = 0; a < 9; ++a) out[9 * o + a] = P.stress_in[9 * o + a];
            continue;
        }
        Part p;
        load_part(P, static_cast<uint32_t>(s), p);
        const float4 mat = material(P, flags & kMatMask);
        float sig[9];
        neo_hookean(p.F, mat.y, mat.z, sig);
        for (int a = 0; a < 9; ++a) out[9 * o + a] = sig[a];
    }
}

// Dense node-major export of one scene's grid after the last update: nodes of bricks
// updated in the current epoch carry {mass, velocity}; below eps the momentum is in
// dead_mom (allocated by Engine::enable_grid_readback).
__global__ void k_grid_download(const Params P, DevScene S, int64_t n_nodes, float* mass,
                                float* mom, float* vel) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n_nodes; q += stride) {
        const int i = static_cast<int>(q % S.dims[0]);
        const int j = static_cast<int>((q / S.dims[0]) % S.dims[1]);
        const int k = static_cast<int>(q / (static_cast<int64_t>(S.dims[0]) * S.dims[1]));
        const uint32_t local = ((k >> 2) * S.nb[1] + (j >> 2)) * S.nb[0] + (i >> 2);
        const uint32_t gb = S.brick_base + local;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        const uint64_t idx = S.node_base + node_linear(P.geo, i, j, k);
        if (P.brick_stamp[gb] == P.epoch) a = P.grid_vel[idx];
        const bool live = a.w > kMassEps;  // node = {x, y, z, mass}
        if (!live && P.brick_stamp[gb] == P.epoch && P.dead_mom) a = P.dead_mom[idx];
        if (mass) mass[q] = a.w;
        if (vel) {
            vel[3 * q + 0] = live ? a.x : 0.f;
            vel[3 * q + 1] = live ? a.y : 0.f;
            vel[3 * q + 2] = live ? a.z : 0.f;
        }
        if (mom) {  // solvers.hpp:48, 61: momentum = velocity * mass after the update
            mom[3 * q + 0] = live ? __fmul_rn(a.x, a.w) : a.x;
            mom[3 * q + 1] = live ? __fmul_rn(a.y, a.w) : a.y;
            mom[3 * q + 2] = live ? __fmul_rn(a.z, a.w) : a.z;
        }
    }
}

__global__ void k_grid_upload(const Params P, DevScene S, int64_t n_nodes, const float* mass,
                              const float* mom, const float* vel) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n_nodes; q += stride) {
        const int i = static_cast<int>(q % S.dims[0]);
        const int j = static_cast<int>((q / S.dims[0]) % S.dims[1]);
        const int k = static_cast<int>(q / (static_cast<int64_t>(S.dims[0]) * S.dims[1]));
        const uint32_t local = ((k >> 2) * S.nb[1] + (j >> 2)) * S.nb[0] + (i >> 2);
        const uint32_t gb = S.brick_base + local;
        if (P.brick_stamp[gb] != P.epoch) continue;
        const float m = mass[q];
        const bool live = m > kMassEps;
        const uint64_t idx = S.node_base + node_linear(P.geo, i, j, k);
        P.grid_vel[idx] = live ? make_float4(vel[3 * q], vel[3 * q + 1], vel[3 * q + 2], m)
                               : make_float4(0.f, 0.f, 0.f, m);
        if (!live && P.dead_mom) P.dead_mom[idx] = make_float4(mom[3 * q], mom[3 * q + 1], mom[3 * q + 2], m);
    }
}

// frame-end export staging (2 float4 per original index) -> the packed x / v / active arrays
__global__ void k_export_pack(const float4* pad, int64_t n, float* x, float* v, uint8_t* a) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < n; o += stride) {
        const float4 p = pad[2 * o], q = pad[2 * o + 1];
        if (x) { x[3 * o] = p.x; x[3 * o + 1] = p.y; x[3 * o + 2] = p.z; }
        if (v) { v[3 * o] = p.w; v[3 * o + 1] = q.x; v[3 * o + 2] = q.y; }
        if (a) a[o] = q.z != 0.f ? 1 : 0;
    }
}
void launch_export_pack(const float4* pad, int64_t n, float* x, float* v, uint8_t* a, cudaStream_t st) {
    k_export_pack<<<blocks_for(n, 256, 148 * 16), 256, 0, st>>>(pad, n, x, v, a);
    MPMB_LAUNCHED("k_export_pack");
}

void launch_upload(const Params& P, const IoArrays& in, int64_t n, cudaStream_t st) {
    k_upload<<<blocks_for(n, 256, 148 * 16), 256, 0, st>>>(P, in, n);
    MPMB_LAUNCHED("k_upload");
}
void launch_download(const Params& P, const IoArrays& out, cudaStream_t st) {
    k_download<<<blocks_for(P.n_total, 256, 148 * 16), 256, 0, st>>>(P, out);
    MPMB_LAUNCHED("k_download");
}
void launch_frame_result_orig(const Params& P, uint32_t* inv, int64_t n, const IoArrays& out, double* totals,
                              cudaStream_t st) {
    k_inv_perm<<<blocks_for(P.n_total, 256, 148 * 16), 256, 0, st>>>(P, inv, n);
    MPMB_LAUNCHED("k_inv_perm");
    k_frame_result_orig<<<blocks_for(n, kTotThreads * kTotPerThread, 148 * 8), kTotThreads, 0, st>>>(P, inv, n, out,
                                                                                                   totals);
    MPMB_LAUNCHED("k_frame_result_orig");
}
void launch_totals(const Params& P, double* totals, cudaStream_t st) {
    k_totals<<<blocks_for(P.n_total, kTotThreads * kTotPerThread, 148 * 8), kTotThreads, 0, st>>>(P, totals);
    MPMB_LAUNCHED("k_totals");
}
void launch_stress(const Params& P, float* stress_orig, cudaStream_t st) {
    k_stress<<<blocks_for(P.n_total, 256, 148 * 16), 256, 0, st>>>(P, stress_orig);
    MPMB_LAUNCHED("k_stress");
}
void launch_grid_download(const Params& P, int, const DevScene& S, float* mass, float* mom,
                          float* vel, cudaStream_t st) {
    const int64_t n = static_cast<int64_t>(S.dims[0]) * S.dims[1] * S.dims[2];
    k_grid_download<<<blocks_for(n, 256, 148 * 16), 256, 0, st>>>(P, S, n, mass, mom, vel);
    MPMB_LAUNCHED("k_grid_download");
}
void launch_grid_upload(const Params& P, int, const DevScene& S, const float* mass,
                        const float* mom, const float* vel, cudaStream_t st) {
    const int64_t n = static_cast<int64_t>(S.dims[0]) * S.dims[1] * S.dims[2];
    k_grid_upload<<<blocks_for(n, 256, 148 * 16), 256, 0, st>>>(P, S, n, mass, mom, vel);
    MPMB_LAUNCHED("k_grid_upload");
}

// ---- device evaluation of the P2G stress (known-answer tests of neo_hookean_f32) ----
__global__ void k_eval_stress_f32(const float* F, int64_t n, float mu, float lambda, float* s, float* J) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float f[9], o[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) f[k] = F[9 * i + k];
    const float j = neo_hookean_f32(f, mu, lambda, o);
#pragma unroll
    for (int k = 0; k < 9; ++k) s[9 * i + k] = o[k];
    if (J) J[i] = j;
}

void eval_stress_f32(const float* F, int64_t n, float mu, float lambda, float* s, float* J) {
    if (n <= 0) return;
    float *dF = nullptr, *ds = nullptr, *dJ = nullptr;
    auto ck = [](cudaError_t e, const char* w) { launch_check(e, w); };
    ck(cudaMalloc(&dF, 36 * n), "cudaMalloc");
    ck(cudaMalloc(&ds, 36 * n), "cudaMalloc");
    ck(cudaMalloc(&dJ, 4 * n), "cudaMalloc");
    ck(cudaMemcpy(dF, F, 36 * n, cudaMemcpyHostToDevice), "h2d");
    k_eval_stress_f32<<<static_cast<unsigned>((n + 255) / 256), 256>>>(dF, n, mu, lambda, ds, dJ);
    MPMB_LAUNCHED("k_eval_stress_f32");
    ck(cudaMemcpy(s, ds, 36 * n, cudaMemcpyDeviceToHost), "d2h");
    if (J) ck(cudaMemcpy(J, dJ, 4 * n, cudaMemcpyDeviceToHost), "d2h");
    cudaFree(dF);
    cudaFree(ds);
    cudaFree(dJ);
}

}  // namespace mpmb
