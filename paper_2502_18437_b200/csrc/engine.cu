// engine.cu — Engine: device buffers and the enqueue order of the hot path.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cfloat>
#include <cmath>
#include <atomic>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>

#include "engine.h"
#include "launch.h"

namespace mpmb {

namespace {

std::atomic<int64_t> g_launches{0};

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void alloc(size_t b) {
        if (b <= bytes && p) return;
        release();
        if (b == 0) b = 16;
        check(cudaMalloc(&p, b), "cudaMalloc");
        bytes = b;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    ~PinnedBuf() { if (p) cudaFreeHost(p); }
    void alloc(size_t b) {
        if (b <= bytes && p) return;
        if (p) cudaFreeHost(p);
        check(cudaMallocHost(&p, b ? b : 16), "cudaMallocHost");
        bytes = b ? b : 16;
    }
};

enum Cat { CAT_SORT = 0, CAT_P2G, CAT_GRID, CAT_G2P, CAT_OTHER, CAT_FUSED };

}  // namespace

// DevShape::lbox: the local-frame box holding every point where a region of the shape can
// still act -- contact bands use hw, push-out bands 0.5 hw (contact.hpp:82-92, 140-179),
// spines their radius -- with a relative margin for the float rotation.  Planes are
// unbounded.
void shape_lbox(DevShape& d, const std::vector<float>& verts) {
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    const double hw = std::max(0.0, double(d.hw));
    auto vbox = [&](double pad) {
        for (int a = 0; a < 3; ++a) {
            lo[a] = 1e300;
            hi[a] = -1e300;
        }
        for (size_t i = 0; i + 2 < verts.size(); i += 3)
            for (int a = 0; a < 3; ++a) {
                lo[a] = std::min(lo[a], double(verts[i + a]));
                hi[a] = std::max(hi[a], double(verts[i + a]));
            }
        for (int a = 0; a < 3; ++a) {
            lo[a] -= pad;
            hi[a] += pad;
        }
    };
    auto sym = [&](double x, double y, double z) {
        lo[0] = -x; lo[1] = -y; lo[2] = -z;
        hi[0] = x; hi[1] = y; hi[2] = z;
    };
    switch (d.geom) {
        case GEOM_PLANE:
            d.lbox_h[0] = d.lbox_h[1] = d.lbox_h[2] = -1.f;
            d.lbox_c[0] = d.lbox_c[1] = d.lbox_c[2] = 0.f;
            return;
        case GEOM_SPHERE: sym(d.gp[0], d.gp[0], d.gp[0]); break;
        case GEOM_BOX: sym(d.gp[0], d.gp[1], d.gp[2]); break;
        case GEOM_QUAD_SLICER: {  // spine along x at y = hh (radius sr), blade plane z = 0
            const double hl = d.gp[0], hh = d.gp[1], sr = d.gp[2], b = std::max(sr, hw);
            lo[0] = -(hl + sr); hi[0] = hl + sr;
            lo[1] = -hh; hi[1] = hh + sr;
            lo[2] = -b; hi[2] = b;
            break;
        }
        case GEOM_TRI_MESH_SLICER: vbox(std::max(double(d.gp[0]), hw)); break;
        case GEOM_ARC: sym(double(d.gp[0]) + hw, double(d.gp[0]) + hw, hw); break;
        default: vbox(hw); break;  // polyline
    }
    double ext = 0;
    for (int a = 0; a < 3; ++a) ext = std::max(ext, std::max(std::fabs(lo[a]), std::fabs(hi[a])));
    const double m = 1e-3 * ext + 1e-5;
    for (int a = 0; a < 3; ++a) {
        d.lbox_c[a] = static_cast<float>(0.5 * (lo[a] + hi[a]));
        d.lbox_h[a] = static_cast<float>(0.5 * (hi[a] - lo[a]) + m);
    }
}

bool device_available() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return n > 0;
}

int64_t global_launch_count() { return g_launches.load(); }

struct Engine::Impl {
    cudaStream_t own = nullptr;
    cudaStream_t st = nullptr;
    std::vector<DevScene> hs;
    Geo geo{};
    std::vector<mpmb_material> hmats;
    DevBuf d_scenes;
    uint64_t total_nodes = 0;
    uint32_t total_bricks = 0;
    DevBuf dead_mom;  // grid readback only (enable_grid_readback)
    DevBuf grid_acc, grid_vel, brick_flag, brick_stamp, active_bricks, active_info, brick_scene, misc;
    int flag_parity = 0;  // which half of brick_flag P2G marks (flips at every collect)
    bool exact = false;   // exact mode (k_exact.cu): the reference's arithmetic and order
    DevBuf ex_scratch, ex_bidx;
    uint32_t ex_epoch = 0;
    DevBuf ex_ckey, ex_crec, ex_cn, ex_cscratch;
    bool wide = false;  // thread-per-slot G2P (small problems, launch_g2p)
    int fusion = 1;     // k_g2p2g inside frames: 0 off, 1 (default) / 2 on
    int sps = 0;        // shapes per scene when uniform (Params::shapes_per_scene)
    int cull_sub = -1;  // the substep whose shape cull table is current (-1: none)  // exact contact records (k_exact.cu)
    PinnedBuf ex_cn_host;
    // misc u32 slots: [0] n_active_bricks
    int64_t n = 0;      // particles
    int64_t n_cap = 0;  // slots of each plane buffer: max(n, cap_hint) + kGroup (padding, holes)
    int64_t cap_hint = 0;
    // slab domain decomposition
    int slab_lo = 0, slab_hi = 0, margin = 0;
    DevBuf halo[4];      // send_lo, send_hi, recv_lo, recv_hi
    int64_t halo_bytes = 0;
    int win[4] = {0, 0, 0, 0};  // halo y/z window: y0, ny, z0, nz (ny = 0: whole extent)
    DevBuf mig[4];       // particles: send_lo, send_hi, recv_lo, recv_hi
    int64_t mig_cap = 0;
    DevBuf mig_counts;   // [0] sent down, [1] sent up; [2] received from below, [3] from above
    DevBuf dd_win;       // device window of the active particles' stencil reach {ylo, yhi, zlo, zhi}
    PinnedBuf dd_ctl_h;  // host copy of {window[4], dd control words [4]} (one read per run)
    PinnedBuf dd_snap_h[2];
    cudaEvent_t dd_snap_ev[2] = {nullptr, nullptr};
    bool dd_async = false;  // run by the device-resident driver (dd_driver.cpp): no host counts
    // transfer launch bound: slabs may append arrivals as extra groups on the device
    int64_t max_groups() const { return ((slab_hi > slab_lo ? n_cap : n) + kGroup - 1) / kGroup; }
    int64_t mig_sent = 0;
    // DD arrivals appended as extra groups since the last binning (no re-sort):
    // free_slot = first slot past the groups + inactive tail (-1: read from the bin counts)
    int64_t free_slot = -1, n_at_bin = 0;
    int appends = 0;
    DevBuf dl_ids, dl_x, dl_v, dl_a, dl_cnt;  // download_compact staging (persistent)
    DevBuf planes[2][kPlanes];
    int cur = 0;
    bool binned = false;
    DevBuf b_count, b_off, b_key, b_rank, b_cell, b_orig, e_orig, e_cell, e_src, b_tmp, g_orig,
        g_src, g_cell, s_src, s_orig, b_counts, scan_tmp, key_by_orig, order, group_nact, group_box;
    BinBuffers bb{};
    DevBuf mats;
    DevBuf shapes, verts, ints, free_pose, pose_table, pose_override, cull, pose_eff;
    int n_shapes = 0;
    int table_subs = 1;
    PinnedBuf pin_table[2];
    cudaEvent_t pin_done[2] = {nullptr, nullptr};
    cudaStream_t copy_st = nullptr;  // snapshot D2H (Engine::snapshot async)
    cudaEvent_t ev_dl = nullptr, ev_copy = nullptr, ev_gather = nullptr;
    bool copy_pending = false;
    // the FrameResult gather (K9) runs on copy_st while the next frame's first P2G and grid
    // update read the same particle planes; anything that WRITES planes waits for it first
    bool gather_pending = false;
    // frame-end export (request_export): requested for the next standalone G2P; valid while
    // the staging holds the current state's result (cleared by every plane writer)
    bool export_req = false, export_valid = false;
    void planes_barrier() {
        if (!gather_pending) return;
        check(cudaStreamWaitEvent(st, ev_gather, 0), "wait gather");
        gather_pending = false;
    }
    int pin_slot = 0;
    DevBuf acc_sub, cnt_sub, acc_frame, cnt_frame, counters;
    DevBuf stress_in;
    bool use_stress_in = false;
    uint32_t epoch = 0;
    DevBuf io_x, io_v, io_a, io_tot, io_inv, io_pad;
    PinnedBuf io_tot_h, small_h;
    PinnedBuf pin_io;
    // profiling
    bool profiling = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> events;
    std::vector<cudaEvent_t> event_pool;
    KernelTimes times;
    int64_t* launch_counter = nullptr;

    cudaEvent_t get_event() {
        if (!event_pool.empty()) {
            cudaEvent_t e = event_pool.back();
            event_pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        check(cudaEventCreate(&e), "cudaEventCreate");
        return e;
    }
    std::pair<cudaEvent_t, cudaEvent_t> begin() {
        if (!profiling) return {nullptr, nullptr};
        cudaEvent_t a = get_event(), b = get_event();
        cudaEventRecord(a, st);
        return {a, b};
    }
    void end(int cat, std::pair<cudaEvent_t, cudaEvent_t> ev) {
        if (!profiling || !ev.first) return;
        cudaEventRecord(ev.second, st);
        events.push_back({cat, ev});
    }
    void collect() {
        for (auto& e : events) {
            cudaEventSynchronize(e.second.second);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e.second.first, e.second.second);
            double* dst = e.first == CAT_SORT ? &times.ms_sort
                          : e.first == CAT_P2G ? &times.ms_p2g
                          : e.first == CAT_GRID ? &times.ms_grid
                          : e.first == CAT_G2P ? &times.ms_g2p
                          : e.first == CAT_FUSED ? &times.ms_fused
                                               : &times.ms_other;
            *dst += ms;
            int64_t* cnt = e.first == CAT_SORT ? &times.n_sort
                           : e.first == CAT_P2G ? &times.n_p2g
                           : e.first == CAT_GRID ? &times.n_grid
                           : e.first == CAT_G2P ? &times.n_g2p
                           : e.first == CAT_FUSED ? &times.n_fused
                                                : nullptr;
            if (cnt) ++*cnt;
            event_pool.push_back(e.second.first);
            event_pool.push_back(e.second.second);
        }
        events.clear();
    }
    void counted(int64_t k) {
        g_launches += k;
        *launch_counter += k;
        if (profiling) times.launches += k;
    }

    // planes_read_only: the launch only reads the particle planes (P2G, grid update), so it
    // may overlap a pending FrameResult gather; every other launch waits for it
    Params params(bool planes_read_only = false) {
        if (!planes_read_only) planes_barrier();
        Params P{};
        for (int q = 0; q < kPlanes; ++q) {
            P.pl[q] = planes[cur][q].as<float4>();
            P.pl_out[q] = planes[1 - cur][q].as<float4>();
        }
        P.geo = geo;
        for (size_t i = 0; i < hmats.size() && i < static_cast<size_t>(kMaxConstMats); ++i)
            P.mats_c[i] = make_float4(static_cast<float>(hmats[i].kind), hmats[i].mu, hmats[i].lambda,
                                      hmats[i].beta);
        P.scenes = d_scenes.as<DevScene>();
        P.shapes = shapes.as<DevShape>();
        P.verts = verts.as<float>();
        P.ints = ints.as<int>();
        P.pose_table = pose_table.as<DevPose>();
        P.pose_override = pose_override.as<uint8_t>();
        P.free_pose = free_pose.as<DevPose>();
        P.cull = cull.as<float4>();
        P.pose_eff = pose_eff.as<DevPose>();
        P.n_shapes = n_shapes;
        P.shapes_per_scene = sps;
        P.mats = mats.as<float4>();
        P.grid_acc = grid_acc.as<float4>();
        P.grid_vel = grid_vel.as<float4>();
        P.dead_mom = dead_mom.p ? dead_mom.as<float4>() : nullptr;
        P.brick_flag = brick_flag.as<uint32_t>() + static_cast<size_t>(flag_parity) * total_bricks;
        P.brick_flag_next = brick_flag.as<uint32_t>() + static_cast<size_t>(1 - flag_parity) * total_bricks;
        P.brick_stamp = brick_stamp.as<uint32_t>();
        P.active_bricks = active_bricks.as<uint32_t>();
        P.active_info = active_info.as<uint2>();
        P.n_active_bricks = misc.as<uint32_t>();
        P.brick_scene = brick_scene.as<uint32_t>();
        P.order = order.as<uint8_t>();  // per-substep group order (k_transfer.cu)
        P.group_nact = group_nact.as<uint32_t>();
        P.group_box = group_box.as<int4>();
        P.n_groups = b_counts.as<uint32_t>() + 1;
        P.n_active = b_counts.as<uint32_t>() + 2;
        P.n_total = n_cap;
        P.total_nodes = total_nodes;
        P.stress_in = stress_in.as<float>();
        P.use_stress_in = use_stress_in ? 1 : 0;
        P.acc_sub = acc_sub.as<double>();
        P.cnt_sub = cnt_sub.as<int>();
        P.acc_frame = acc_frame.as<double>();
        P.cnt_frame = cnt_frame.as<int>();
        P.counters = counters.as<int>();
        P.epoch = epoch;
        P.exact = exact ? 1 : 0;
        return P;
    }
};

// Below this many slots G2P runs one thread per slot: one warp per 256-slot group
// would leave most of the 148 SMs idle (MPMB_WIDE_MAX overrides; measured).
static int64_t wide_max_slots() {
    static const int64_t v = [] {
        const char* e = std::getenv("MPMB_WIDE_MAX");
        return e ? std::atoll(e) : static_cast<int64_t>(kWideMaxSlots);
    }();
    return v;
}

Engine::Engine(const std::vector<SceneGrid>& scenes) : impl_(new Impl), scenes_(scenes) {
    Impl& I = *impl_;
    launches_total_ = 0;
    I.launch_counter = &launches_total_;
    check(cudaStreamCreateWithFlags(&I.own, cudaStreamNonBlocking), "cudaStreamCreate");
    I.st = I.own;
    stream_ = I.own;
    uint64_t node_base = 0;
    uint32_t brick_base = 0;
    for (const SceneGrid& g : scenes) {
        DevScene d{};
        const bool slab = g.slab_hi > g.slab_lo;
        const int lx = slab ? g.slab_hi - g.slab_lo + 2 * g.margin + 2 : g.dims[0];
        for (int a = 0; a < 3; ++a) {
            d.origin[a] = g.origin[a];
            d.dims[a] = g.dims[a];
            d.nb[a] = ((a == 0 ? lx : g.dims[a]) + kBrick - 1) / kBrick;
        }
        d.dx = g.dx;
        d.inv_dx = 1.0f / g.dx;                 // math.hpp:219
        d.m_inv = 4.0f / (g.dx * g.dx);         // solvers.hpp:149
        d.node_base = node_base;
        d.brick_base = brick_base;
        const uint64_t nb = static_cast<uint64_t>(d.nb[0]) * d.nb[1] * d.nb[2];
        // the decoded active-brick list packs 10 bits per brick coordinate (active_info)
        if (d.nb[0] >= 1024 || d.nb[1] >= 1024 || d.nb[2] >= 1024)
            throw std::invalid_argument("engine: grid too large (4096 nodes per axis at most)");
        // brick ids are 32-bit; the brick flags/stamps are one word per brick
        if (brick_base + nb >= (1ull << 31)) throw std::invalid_argument("engine: too many grid bricks (>2^31)");
        node_base += nb * kBrickNodes;
        brick_base += static_cast<uint32_t>(nb);
        if (!I.hs.empty()) {
            const DevScene& d0 = I.hs[0];
            for (int a = 0; a < 3; ++a)
                if (d.dims[a] != d0.dims[a] || d.origin[a] != d0.origin[a])
                    throw std::invalid_argument("engine: scenes of a batch must share the grid geometry");
            if (d.dx != d0.dx) throw std::invalid_argument("engine: scenes of a batch must share dx");
        }
        I.hs.push_back(d);
    }
    if (!I.hs.empty()) {  // uniform geometry for the kernels' parameter bank
        const DevScene& d0 = I.hs[0];
        for (int a = 0; a < 3; ++a) {
            I.geo.origin[a] = d0.origin[a];
            I.geo.dims[a] = d0.dims[a];
            I.geo.nb[a] = d0.nb[a];
        }
        I.geo.dx = d0.dx;
        I.geo.inv_dx = d0.inv_dx;
        I.geo.m_inv = d0.m_inv;
        I.geo.bricks_per_scene = static_cast<uint32_t>(d0.nb[0]) * d0.nb[1] * d0.nb[2];
        I.geo.nodes_per_scene = static_cast<uint64_t>(I.geo.bricks_per_scene) * kBrickNodes;
        const SceneGrid& g0 = scenes[0];
        if (g0.slab_hi > g0.slab_lo) {
            if (scenes.size() != 1) throw std::invalid_argument("engine: a slab domain holds one scene");
            if (g0.slab_lo < 0 || g0.slab_hi > g0.dims[0] || g0.margin < 0)
                throw std::invalid_argument("engine: slab outside the grid");
            I.geo.goff = g0.slab_lo - g0.margin;
            I.geo.lx = g0.slab_hi - g0.slab_lo + 2 * g0.margin + 2;
            I.geo.own_lo = g0.margin;
            I.geo.own_hi = g0.margin + (g0.slab_hi - g0.slab_lo);
            I.slab_lo = g0.slab_lo;
            I.slab_hi = g0.slab_hi;
            I.margin = g0.margin;
        } else {
            I.geo.goff = 0;
            I.geo.lx = d0.dims[0];
            I.geo.own_lo = 0;
            I.geo.own_hi = d0.dims[0];
        }
    }
    I.total_nodes = node_base;
    I.total_bricks = brick_base;
    I.d_scenes.alloc(sizeof(DevScene) * std::max<size_t>(1, I.hs.size()));
    check(cudaMemcpy(I.d_scenes.p, I.hs.data(), sizeof(DevScene) * I.hs.size(), cudaMemcpyHostToDevice), "scenes");
    I.grid_acc.alloc(sizeof(float4) * I.total_nodes);
    I.grid_vel.alloc(sizeof(float4) * I.total_nodes);
    check(cudaMemset(I.grid_acc.p, 0, sizeof(float4) * I.total_nodes), "memset");
    check(cudaMemset(I.grid_vel.p, 0, sizeof(float4) * I.total_nodes), "memset");
    I.brick_flag.alloc(2 * sizeof(uint32_t) * I.total_bricks);  // alternating mark arrays
    I.brick_stamp.alloc(sizeof(uint32_t) * I.total_bricks);
    I.active_bricks.alloc(sizeof(uint32_t) * I.total_bricks);
    I.active_info.alloc(sizeof(uint2) * I.total_bricks);
    check(cudaMemset(I.brick_flag.p, 0, 2 * sizeof(uint32_t) * I.total_bricks), "memset");
    check(cudaMemset(I.brick_stamp.p, 0xFF, sizeof(uint32_t) * I.total_bricks), "memset");
    std::vector<uint32_t> bs(I.total_bricks);
    for (size_t s = 0; s < I.hs.size(); ++s) {
        const uint32_t nb = static_cast<uint32_t>(I.hs[s].nb[0]) * I.hs[s].nb[1] * I.hs[s].nb[2];
        std::fill(bs.begin() + I.hs[s].brick_base, bs.begin() + I.hs[s].brick_base + nb,
                  static_cast<uint32_t>(s));
    }
    I.brick_scene.alloc(sizeof(uint32_t) * I.total_bricks);
    check(cudaMemcpy(I.brick_scene.p, bs.data(), sizeof(uint32_t) * bs.size(), cudaMemcpyHostToDevice), "bs");
    I.misc.alloc(64);
    check(cudaMemset(I.misc.p, 0, 64), "memset");
    I.counters.alloc(sizeof(int) * 4 * std::max<size_t>(1, I.hs.size()));
    check(cudaMemset(I.counters.p, 0, I.counters.bytes), "memset");
    I.b_counts.alloc(8 * sizeof(uint32_t));  // [0..3] binning counts, [4..7] DD control (launch.h)
    check(cudaMemset(I.b_counts.p, 0, 8 * sizeof(uint32_t)), "memset");
    set_shapes(std::vector<std::vector<EngineShape>>(scenes.size()));
    mpmb_material dflt{0, 0.f, 0.f, 0.f};
    set_materials({dflt});
    for (int i = 0; i < 2; ++i) check(cudaEventCreateWithFlags(&I.pin_done[i], cudaEventDisableTiming), "event");
}

Engine::~Engine() {
    Impl& I = *impl_;
    cudaStreamSynchronize(I.st);
    if (I.copy_st) {
        cudaStreamSynchronize(I.copy_st);
        cudaStreamDestroy(I.copy_st);
        cudaEventDestroy(I.ev_dl);
        cudaEventDestroy(I.ev_copy);
        cudaEventDestroy(I.ev_gather);
    }
    for (auto& e : I.events) {
        cudaEventDestroy(e.second.first);
        cudaEventDestroy(e.second.second);
    }
    for (auto e : I.event_pool) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i)
        if (I.pin_done[i]) cudaEventDestroy(I.pin_done[i]);
    for (int i = 0; i < 2; ++i)
        if (I.dd_snap_ev[i]) cudaEventDestroy(I.dd_snap_ev[i]);
    if (I.own) cudaStreamDestroy(I.own);
    delete impl_;
}

void Engine::set_stream(void* s) {
    impl_->st = s ? static_cast<cudaStream_t>(s) : impl_->own;
    stream_ = impl_->st;
}

void Engine::set_profiling(bool on) { impl_->profiling = on; }

KernelTimes Engine::kernel_times() const {
    impl_->collect();
    return impl_->times;
}

void Engine::reset_kernel_times() {
    impl_->collect();
    impl_->times = KernelTimes{};
}

void Engine::set_materials(const std::vector<mpmb_material>& m) {
    Impl& I = *impl_;
    I.hmats = m;
    std::vector<float4> h(std::max<size_t>(1, m.size()));
    for (size_t i = 0; i < m.size(); ++i)
        h[i] = make_float4(static_cast<float>(m[i].kind), m[i].mu, m[i].lambda, m[i].beta);
    I.mats.alloc(sizeof(float4) * h.size());
    check(cudaMemcpyAsync(I.mats.p, h.data(), sizeof(float4) * h.size(), cudaMemcpyHostToDevice, I.st), "mats");
    check(cudaStreamSynchronize(I.st), "sync");
}

void Engine::upload_particles(int64_t n, const float* x, const float* v, const float* mass,
                              const float* vol0, const float* F, const float* C, const float* stress,
                              const int32_t* material, const uint8_t* active, const int32_t* scene,
                              const uint32_t* ids) {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    if (n >= 0x7FFFFFFF) throw std::invalid_argument("engine: particle count exceeds 2^31");
    check(cudaStreamSynchronize(I.st), "sync");
    I.n = n;
    I.n_cap = (n > 0 || I.cap_hint > 0) ? std::max<int64_t>(n, I.cap_hint) + kGroup : 0;
    I.wide = I.n_cap > 0 && I.n_cap <= wide_max_slots();
    n_total_ = n;
    for (int b = 0; b < 2; ++b)
        for (int q = 0; q < kPlanes; ++q) I.planes[b][q].alloc(sizeof(float4) * std::max<int64_t>(I.n_cap, 1));
    I.cur = 0;
    // sort scratch (per slot)
    const size_t N = static_cast<size_t>(std::max<int64_t>(I.n_cap, 1));
    I.b_key.alloc(4 * N); I.b_rank.alloc(4 * N); I.b_cell.alloc(N); I.b_orig.alloc(4 * N);
    I.e_orig.alloc(4 * N); I.e_cell.alloc(N); I.e_src.alloc(4 * N); I.b_tmp.alloc(4 * N);
    I.g_orig.alloc(4 * N); I.g_src.alloc(4 * N); I.g_cell.alloc(N); I.s_src.alloc(4 * N);
    I.s_orig.alloc(4 * N);
    const size_t n_groups = (N + kGroup - 1) / kGroup;
    // per group: 256 order bytes; n_act and the node box per unit (up to 8 of 32 positions)
    I.order.alloc(kGroup * n_groups); I.group_nact.alloc(4 * 8 * n_groups); I.group_box.alloc(16 * 8 * n_groups);
    const size_t nbk = static_cast<size_t>(I.total_bricks) + 2;  // + inactive, holes
    I.b_count.alloc(4 * nbk);
    I.b_off.alloc(4 * (nbk + 1));
    const size_t tiles = (std::max(N + 1, nbk + 1) + 4095) / 4096 + 2;
    I.scan_tmp.alloc(4 * tiles);
    BinBuffers& B = I.bb;
    B.n_buckets = static_cast<uint32_t>(nbk);
    B.bucket_count = I.b_count.as<uint32_t>(); B.bucket_off = I.b_off.as<uint32_t>();
    B.key = I.b_key.as<uint32_t>(); B.rank = I.b_rank.as<uint32_t>(); B.cell = I.b_cell.as<uint8_t>();
    B.orig = I.b_orig.as<uint32_t>(); B.e_orig = I.e_orig.as<uint32_t>(); B.e_cell = I.e_cell.as<uint8_t>();
    B.e_src = I.e_src.as<uint32_t>(); B.tmp = I.b_tmp.as<uint32_t>(); B.g_orig = I.g_orig.as<uint32_t>();
    B.g_src = I.g_src.as<uint32_t>(); B.g_cell = I.g_cell.as<uint8_t>(); B.sorted_src = I.s_src.as<uint32_t>();
    B.sorted_orig = I.s_orig.as<uint32_t>();
    B.counts = I.b_counts.as<uint32_t>(); B.scan_tmp = I.scan_tmp.as<uint32_t>();
    B.key_by_orig = nullptr;
    if (I.n_cap == 0) {
        I.binned = false;
        return;
    }
    // stage original-order arrays on the device, then scatter into the planes
    DevBuf dx, dv, dm, dvol, dF, dC, dmat, dact, dsc;
    dx.alloc(12 * N); dv.alloc(12 * N); dm.alloc(4 * N); dvol.alloc(4 * N); dF.alloc(36 * N);
    dC.alloc(36 * N); dmat.alloc(4 * N); dact.alloc(N); dsc.alloc(4 * N);
    check(cudaMemcpyAsync(dx.p, x, 12 * n, cudaMemcpyHostToDevice, I.st), "h2d");
    check(cudaMemcpyAsync(dv.p, v, 12 * n, cudaMemcpyHostToDevice, I.st), "h2d");
    check(cudaMemcpyAsync(dm.p, mass, 4 * n, cudaMemcpyHostToDevice, I.st), "h2d");
    check(cudaMemcpyAsync(dvol.p, vol0, 4 * n, cudaMemcpyHostToDevice, I.st), "h2d");
    check(cudaMemcpyAsync(dF.p, F, 36 * n, cudaMemcpyHostToDevice, I.st), "h2d");
    check(cudaMemcpyAsync(dC.p, C, 36 * n, cudaMemcpyHostToDevice, I.st), "h2d");
    check(cudaMemcpyAsync(dmat.p, material, 4 * n, cudaMemcpyHostToDevice, I.st), "h2d");
    check(cudaMemcpyAsync(dact.p, active, n, cudaMemcpyHostToDevice, I.st), "h2d");
    check(cudaMemcpyAsync(dsc.p, scene, 4 * n, cudaMemcpyHostToDevice, I.st), "h2d");
    DevBuf dids;
    if (ids) {
        dids.alloc(4 * N);
        check(cudaMemcpyAsync(dids.p, ids, 4 * n, cudaMemcpyHostToDevice, I.st), "h2d");
    }
    IoArrays io{dx.as<float>(), dv.as<float>(), dm.as<float>(), dvol.as<float>(), dF.as<float>(),
                dC.as<float>(), dmat.as<int32_t>(), dact.as<uint8_t>(), dsc.as<int32_t>(),
                ids ? dids.as<uint32_t>() : nullptr, stress != nullptr};
    Params P = I.params();
    launch_upload(P, io, n, I.st);
    I.counted(1);
    if (stress) {
        I.stress_in.alloc(36 * N);
        check(cudaMemcpyAsync(I.stress_in.p, stress, 36 * n, cudaMemcpyHostToDevice, I.st), "h2d");
        I.use_stress_in = true;
    } else {
        I.use_stress_in = false;
    }
    check(cudaStreamSynchronize(I.st), "upload");
    I.binned = false;
}

void Engine::download_particles(int64_t begin, int64_t count, float* x, float* v, float* mass,
                                float* vol0, float* F, float* C, float* stress, int32_t* material,
                                uint8_t* active) {
    Impl& I = *impl_;
    if (I.n == 0 || count <= 0) return;
    const size_t N = static_cast<size_t>(I.n);
    DevBuf dx, dv, dm, dvol, dF, dC, dmat, dact, dsig;
    IoArrays io{};
    if (x) { dx.alloc(12 * N); io.x = dx.as<float>(); }
    if (v) { dv.alloc(12 * N); io.v = dv.as<float>(); }
    if (mass) { dm.alloc(4 * N); io.mass = dm.as<float>(); }
    if (vol0) { dvol.alloc(4 * N); io.vol0 = dvol.as<float>(); }
    if (F) { dF.alloc(36 * N); io.F = dF.as<float>(); }
    if (C) { dC.alloc(36 * N); io.C = dC.as<float>(); }
    if (material) { dmat.alloc(4 * N); io.mat = dmat.as<int32_t>(); }
    if (active) { dact.alloc(N); io.active = dact.as<uint8_t>(); }
    Params P = I.params();
    launch_download(P, io, I.st);
    I.counted(1);
    if (stress) {
        dsig.alloc(36 * N);
        launch_stress(P, dsig.as<float>(), I.st);
        I.counted(1);
    }
    auto cp = [&](void* dst, const DevBuf& src, size_t elem) {
        if (dst)
            check(cudaMemcpyAsync(dst, static_cast<char*>(src.p) + elem * begin, elem * count,
                                  cudaMemcpyDeviceToHost, I.st), "d2h");
    };
    cp(x, dx, 12); cp(v, dv, 12); cp(mass, dm, 4); cp(vol0, dvol, 4); cp(F, dF, 36); cp(C, dC, 36);
    cp(material, dmat, 4); cp(active, dact, 1); cp(stress, dsig, 36);
    check(cudaStreamSynchronize(I.st), "download");
}

void Engine::set_shapes(const std::vector<std::vector<EngineShape>>& per_scene) {
    impl_->cull_sub = -1;
    Impl& I = *impl_;
    check(cudaStreamSynchronize(I.st), "sync");
    std::vector<DevShape> ds;
    std::vector<DevPose> poses;
    std::vector<float> verts;
    std::vector<int> ints;
    for (size_t s = 0; s < per_scene.size(); ++s) {
        I.hs[s].shape_begin = static_cast<int>(ds.size());
        I.hs[s].shape_count = static_cast<int>(per_scene[s].size());
        for (const EngineShape& e : per_scene[s]) {
            DevShape d = e.d;
            d.scene = static_cast<int>(s);
            d.vtx_begin = static_cast<int>(verts.size() / 3);
            d.n_vtx = static_cast<int>(e.verts.size() / 3);
            verts.insert(verts.end(), e.verts.begin(), e.verts.end());
            d.idx_begin = static_cast<int>(ints.size());
            d.n_idx = static_cast<int>(e.indices.size());
            ints.insert(ints.end(), e.indices.begin(), e.indices.end());
            d.spine_begin = static_cast<int>(ints.size());
            d.n_spine = static_cast<int>(e.spine.size());
            ints.insert(ints.end(), e.spine.begin(), e.spine.end());
            shape_lbox(d, e.verts);
            ds.push_back(d);
            poses.push_back(e.pose);
        }
    }
    I.n_shapes = static_cast<int>(ds.size());
    n_shapes_ = I.n_shapes;
    I.sps = per_scene.empty() ? 0 : static_cast<int>(per_scene[0].size());
    for (size_t s = 0; s < per_scene.size(); ++s)
        if (static_cast<int>(per_scene[s].size()) != I.sps) I.sps = 0;
    check(cudaMemcpy(I.d_scenes.p, I.hs.data(), sizeof(DevScene) * I.hs.size(), cudaMemcpyHostToDevice), "scenes");
    const size_t ns = std::max<size_t>(1, ds.size());
    I.shapes.alloc(sizeof(DevShape) * ns);
    I.verts.alloc(sizeof(float) * std::max<size_t>(3, verts.size()));
    I.ints.alloc(sizeof(int) * std::max<size_t>(1, ints.size()));
    I.free_pose.alloc(sizeof(DevPose) * ns);
    I.cull.alloc(2 * sizeof(float4) * ns);
    I.pose_eff.alloc(sizeof(DevPose) * ns);
    I.acc_sub.alloc(sizeof(double) * 6 * ns);
    I.acc_frame.alloc(sizeof(double) * 6 * ns);
    I.cnt_sub.alloc(sizeof(int) * ns);
    I.cnt_frame.alloc(sizeof(int) * ns);
    if (!ds.empty()) {
        check(cudaMemcpy(I.shapes.p, ds.data(), sizeof(DevShape) * ds.size(), cudaMemcpyHostToDevice), "shapes");
        check(cudaMemcpy(I.free_pose.p, poses.data(), sizeof(DevPose) * poses.size(), cudaMemcpyHostToDevice), "poses");
    }
    if (!verts.empty())
        check(cudaMemcpy(I.verts.p, verts.data(), sizeof(float) * verts.size(), cudaMemcpyHostToDevice), "verts");
    if (!ints.empty())
        check(cudaMemcpy(I.ints.p, ints.data(), sizeof(int) * ints.size(), cudaMemcpyHostToDevice), "ints");
    check(cudaMemset(I.acc_sub.p, 0, I.acc_sub.bytes), "memset");
    check(cudaMemset(I.acc_frame.p, 0, I.acc_frame.bytes), "memset");
    check(cudaMemset(I.cnt_sub.p, 0, I.cnt_sub.bytes), "memset");
    check(cudaMemset(I.cnt_frame.p, 0, I.cnt_frame.bytes), "memset");
    // default pose table: one substep holding the current poses, no overrides
    I.table_subs = 1;
    I.pose_table.alloc(sizeof(DevPose) * ns);
    I.pose_override.alloc(ns);
    if (!poses.empty())
        check(cudaMemcpy(I.pose_table.p, poses.data(), sizeof(DevPose) * poses.size(), cudaMemcpyHostToDevice), "table");
    check(cudaMemset(I.pose_override.p, 0, ns), "memset");
}

void Engine::set_pose_table(int n_sub, const std::vector<DevPose>& poses,
                            const std::vector<uint8_t>& ovr) {
    impl_->cull_sub = -1;
    Impl& I = *impl_;
    if (I.n_shapes == 0) return;
    const size_t np = static_cast<size_t>(n_sub) * I.n_shapes;
    if (poses.size() != np || ovr.size() != np) throw std::invalid_argument("pose table size");
    const size_t bytes = sizeof(DevPose) * np + np;
    const int slot = I.pin_slot;
    I.pin_slot ^= 1;
    check(cudaEventSynchronize(I.pin_done[slot]), "pin wait");
    I.pin_table[slot].alloc(bytes);
    char* h = static_cast<char*>(I.pin_table[slot].p);
    std::memcpy(h, poses.data(), sizeof(DevPose) * np);
    std::memcpy(h + sizeof(DevPose) * np, ovr.data(), np);
    if (n_sub > I.table_subs || !I.pose_table.p) {
        check(cudaStreamSynchronize(I.st), "sync");
        I.pose_table.alloc(sizeof(DevPose) * np);
        I.pose_override.alloc(np);
    }
    I.table_subs = std::max(I.table_subs, n_sub);
    check(cudaMemcpyAsync(I.pose_table.p, h, sizeof(DevPose) * np, cudaMemcpyHostToDevice, I.st), "table");
    check(cudaMemcpyAsync(I.pose_override.p, h + sizeof(DevPose) * np, np, cudaMemcpyHostToDevice, I.st), "ovr");
    check(cudaEventRecord(I.pin_done[slot], I.st), "record");
}

void Engine::set_free_pose(int shape, const DevPose& pose) {
    impl_->cull_sub = -1;
    Impl& I = *impl_;
    check(cudaStreamSynchronize(I.st), "sync");
    check(cudaMemcpy(I.free_pose.as<DevPose>() + shape, &pose, sizeof(DevPose), cudaMemcpyHostToDevice), "pose");
}

std::vector<DevPose> Engine::read_free_poses() {
    Impl& I = *impl_;
    std::vector<DevPose> out(I.n_shapes);
    check(cudaStreamSynchronize(I.st), "sync");
    if (I.n_shapes)
        check(cudaMemcpy(out.data(), I.free_pose.p, sizeof(DevPose) * I.n_shapes, cudaMemcpyDeviceToHost), "poses");
    return out;
}

// --------------------------------------------------------------- hot path
void Engine::bin() {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    if (I.n_cap == 0) return;
    auto ev = I.begin();
    Params P = I.params();
    float4* np[kPlanes];
    for (int q = 0; q < kPlanes; ++q) np[q] = I.planes[1 - I.cur][q].as<float4>();
    int64_t k = 0;
    launch_bin(P, I.bb, np, I.n_cap, I.st, &k);
    I.counted(k);
    I.cur = 1 - I.cur;
    I.binned = true;
    I.free_slot = -1;
    I.n_at_bin = I.n;
    I.appends = 0;
    I.end(CAT_SORT, ev);
}

void Engine::p2g(bool mls, float dt, bool collect, bool standard) {
    Impl& I = *impl_;
    if (I.n_cap == 0) return;
    if (!I.binned) bin();
    auto ev = I.begin();
    cudaMemsetAsync(I.misc.p, 0, sizeof(uint32_t), I.st);  // active brick count
    Params P = I.params(!I.exact);
    P.dt = dt;
    if (I.exact) {
        if (standard || !mls) throw std::invalid_argument("engine: exact mode covers the MLS solver");
        const size_t sb = exact_scratch_bytes(I.n_cap, I.total_bricks);
        if (I.ex_scratch.bytes < sb) I.ex_scratch.alloc(sb);
        if (!I.ex_bidx.p) {
            I.ex_bidx.alloc(sizeof(uint2) * I.total_bricks);
            check(cudaMemsetAsync(I.ex_bidx.p, 0, sizeof(uint2) * I.total_bricks, I.st), "memset");
        }
        launch_exact_p2g(P, mls, I.ex_scratch.p, I.ex_bidx.as<uint2>(), ++I.ex_epoch, I.total_bricks, I.st);
        I.counted(8);
        I.flag_parity = 1 - I.flag_parity;  // the collect ran inside
        if (mls) I.use_stress_in = false;
        I.end(CAT_P2G, ev);
        return;
    }
    launch_p2g(P, mls || standard, I.max_groups(), I.st, standard);
    I.counted(1);
    if (collect) {
        launch_collect_bricks(P, I.total_bricks, I.st);
        I.counted(1);
        I.flag_parity = 1 - I.flag_parity;
    }
    if (mls || standard) I.use_stress_in = false;  // consumed by the first stress-using P2G
    I.end(CAT_P2G, ev);
}

void Engine::grid_update(int sub, float dt, const float g[3], bool gravity, bool contact, int bc) {
    Impl& I = *impl_;
    if (I.n_cap == 0) return;
    auto ev = I.begin();
    ++I.epoch;
    if (I.epoch == 0xFFFFFFFFu) I.epoch = 1;
    Params P = I.params(true);
    P.sub = std::min(sub, I.table_subs - 1);
    P.dt = dt;
    P.g[0] = g[0]; P.g[1] = g[1]; P.g[2] = g[2];
    P.gravity = gravity ? 1 : 0;
    P.contact = contact ? 1 : 0;
    P.bc = bc;
    if (I.n_shapes > 0 && I.cull_sub != P.sub) {  // G2P push-out of this substep reuses the table
        launch_shape_cull(P, I.st);
        I.counted(1);
        I.cull_sub = P.sub;
    }
    const bool ex_contact = I.exact && contact && I.n_shapes > 0;
    if (ex_contact) {  // one record per contacting (node, shape): at most nodes x shapes
        const uint64_t cap64 = I.total_nodes * static_cast<uint64_t>(I.n_shapes);
        const uint32_t cap = static_cast<uint32_t>(std::min<uint64_t>(cap64, 0x7FFFFFFFull));
        I.ex_ckey.alloc(8ull * cap);
        I.ex_crec.alloc(24ull * cap);
        I.ex_cn.alloc(4);
        I.ex_cn_host.alloc(4);
        check(cudaMemsetAsync(I.ex_cn.p, 0, 4, I.st), "memset");
        P.ex_ckey = I.ex_ckey.as<uint64_t>();
        P.ex_crec = I.ex_crec.as<float>();
        P.ex_cn = I.ex_cn.as<uint32_t>();
        P.ex_ccap = cap;
    }
    launch_grid_update(P, I.total_bricks, I.st);
    I.counted(1);
    if (ex_contact) {  // ordered float sums need the record count on the host (CUB sizes)
        check(cudaMemcpyAsync(I.ex_cn_host.p, I.ex_cn.p, 4, cudaMemcpyDeviceToHost, I.st), "d2h");
        check(cudaStreamSynchronize(I.st), "exact contact");
        const uint32_t n = *static_cast<uint32_t*>(I.ex_cn_host.p);
        if (n > P.ex_ccap) throw std::runtime_error("engine: exact contact records overflow");
        I.ex_cscratch.alloc(exact_contact_scratch_bytes(n));
        launch_exact_contact(P, n, I.ex_cscratch.p, I.st);
        I.counted(3);
    }
    I.end(CAT_GRID, ev);
}

void Engine::request_export() { impl_->export_req = true; }

// Staging and totals for a frame-end export (request_export) into P; false when the launch
// does not export (no request, exact mode, no particles).
bool Engine::prepare_export(Params& P) {
    Impl& I = *impl_;
    const bool want = I.export_req && !I.exact && I.n > 0;
    I.export_req = false;
    I.export_valid = false;
    if (!want) return false;
    const size_t N = static_cast<size_t>(I.n);
    const size_t S = std::max<size_t>(I.hs.size(), 1);
    if (I.copy_pending && I.io_pad.bytes < 32 * N) wait_results();  // about to be reallocated
    // the previous frame's unpack (copy stream) still reads the padded staging
    if (I.copy_pending) check(cudaStreamWaitEvent(I.st, I.ev_copy, 0), "wait copy");
    I.io_pad.alloc(32 * N);
    I.io_tot.alloc(sizeof(double) * 5 * S);
    check(cudaMemsetAsync(I.io_tot.p, 0, I.io_tot.bytes, I.st), "memset");
    P.exp_pad = I.io_pad.as<float4>();
    P.exp_tot = I.io_tot.as<double>();
    P.exp_n = I.n;
    return true;
}

void Engine::g2p_mls(int sub, float dt, bool pushout, bool deactivate) {
    Impl& I = *impl_;
    if (I.n_cap == 0) return;
    auto ev = I.begin();
    Params P = I.params();
    const bool exported = prepare_export(P);
    P.sub = std::min(sub, I.table_subs - 1);
    P.dt = dt;
    P.pushout = pushout ? 1 : 0;
    P.deactivate = deactivate ? 1 : 0;
    P.commit = 1;
    if (I.exact) {  // in place, reference order; push-out / deactivation as separate passes
        launch_exact_g2p(P, I.st);
        I.counted(1);
        if (pushout && I.n_shapes > 0) {
            launch_pushout(P, I.st);
            I.counted(1);
        }
        if (deactivate) {
            launch_deactivate(P, I.st);
            I.counted(1);
        }
        I.end(CAT_G2P, ev);
        return;
    }
    launch_g2p(P, false, I.max_groups(), I.st, false, I.wide);
    I.counted(1);
    I.cur = 1 - I.cur;  // G2P wrote the group-sorted state into the other buffer
    I.export_valid = exported;
    I.end(CAT_G2P, ev);
}

// G2P(sub) + P2G(sub+1) in one launch (k_g2p2g), then the brick collect of sub+1.  The
// caller runs free_bodies(sub) after it (its shape cull for sub+1 would overwrite the
// table the fused push-out of sub still reads).
void Engine::g2p2g(int sub, float dt, bool standard, const float g[3], bool integrate, bool collect, bool pushout,
                   bool deactivate) {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    if (I.n_cap == 0) return;
    auto ev = I.begin();
    Params P = I.params();
    P.sub = std::min(sub, I.table_subs - 1);
    P.dt = dt;
    P.g[0] = g[0]; P.g[1] = g[1]; P.g[2] = g[2];
    P.pushout = pushout ? 1 : 0;
    P.deactivate = deactivate ? 1 : 0;
    P.commit = 1;
    launch_g2p2g(P, I.max_groups(), I.st, standard);  // zeroes the brick count
    if (!collect) {  // slab DD: the ghost sums arrive first (collect_deferred)
        I.counted(1);
        I.cur = 1 - I.cur;
        I.end(CAT_FUSED, ev);
        return;
    }
    if (I.n_shapes > 0) {
        const int next = std::min(sub + 1, I.table_subs - 1);
        launch_collect_free(P, I.total_bricks, integrate, true, next, I.st);
        I.cull_sub = next;
    } else {
        launch_collect_bricks(P, I.total_bricks, I.st);
    }
    I.counted(2);
    I.flag_parity = 1 - I.flag_parity;
    I.cur = 1 - I.cur;  // the state of sub+1 is in the other buffer
    I.end(CAT_FUSED, ev);
}

void Engine::g2p2g_pb(float dt) {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    if (I.n_cap == 0) return;
    auto ev = I.begin();
    Params P = I.params();
    P.sub = 0;
    P.dt = dt;
    P.commit = 0;
    P.pushout = 0;
    P.deactivate = 0;
    launch_g2p2g(P, I.max_groups(), I.st, false, true);  // zeroes the brick count
    launch_collect_bricks(P, I.total_bricks, I.st);
    I.counted(2);
    I.flag_parity = 1 - I.flag_parity;
    I.cur = 1 - I.cur;
    I.end(CAT_FUSED, ev);
}

void Engine::set_fusion(int mode) { impl_->fusion = mode; }

void Engine::contact_sub_buffers(void** sums, void** counts, int* n_shapes) {
    Impl& I = *impl_;
    if (sums) *sums = I.acc_sub.p;
    if (counts) *counts = I.cnt_sub.p;
    if (n_shapes) *n_shapes = I.n_shapes;
}
bool Engine::fuse_ok() const {
    const Impl& I = *impl_;
    // measured: +17% C1, +21% C2, +5.6% at 874k, +0.6% C5, -0.7% C4, so the
    // default fuses at every size; the thread-per-slot G2P stays for the frame's last substep
    return !I.exact && I.n_cap > 0 && I.fusion >= 1;
}

void Engine::set_exact(bool on) { impl_->exact = on; }
bool Engine::exact() const { return impl_->exact; }

void Engine::g2p_standard(int sub, float dt, bool pushout, bool deactivate) {
    Impl& I = *impl_;
    if (I.n_cap == 0) return;
    if (I.exact) throw std::invalid_argument("engine: exact mode covers the MLS solver");
    auto ev = I.begin();
    Params P = I.params();
    const bool exported = prepare_export(P);
    P.sub = std::min(sub, I.table_subs - 1);
    P.dt = dt;
    P.pushout = pushout ? 1 : 0;
    P.deactivate = deactivate ? 1 : 0;
    P.commit = 1;
    launch_g2p(P, false, I.max_groups(), I.st, true, I.wide);
    I.counted(1);
    I.cur = 1 - I.cur;
    I.export_valid = exported;
    I.end(CAT_G2P, ev);
}

void Engine::g2p_pb(int sub, float dt, bool commit, bool pushout, bool deactivate) {
    Impl& I = *impl_;
    if (I.n_cap == 0) return;
    if (I.exact) throw std::invalid_argument("engine: exact mode covers the MLS solver");
    auto ev = I.begin();
    Params P = I.params();
    const bool exported = commit && prepare_export(P);
    if (!commit) I.export_valid = false;
    P.sub = std::min(sub, I.table_subs - 1);
    P.dt = dt;
    P.commit = commit ? 1 : 0;
    P.pushout = pushout ? 1 : 0;
    P.deactivate = deactivate ? 1 : 0;
    launch_g2p(P, true, I.max_groups(), I.st, false, I.wide);
    I.counted(1);
    I.cur = 1 - I.cur;
    I.export_valid = exported;
    I.end(CAT_G2P, ev);
}

void Engine::free_bodies(int sub, float dt, const float g[3], bool integrate, bool merge, int cull_next) {
    Impl& I = *impl_;
    if (I.n_shapes == 0) return;
    auto ev = I.begin();
    Params P = I.params();
    P.sub = std::min(sub, I.table_subs - 1);
    P.dt = dt;
    P.g[0] = g[0]; P.g[1] = g[1]; P.g[2] = g[2];
    const int next = cull_next >= 0 ? std::min(cull_next, I.table_subs - 1) : -1;
    launch_free_bodies(P, integrate, merge, I.st, next);
    if (next >= 0) I.cull_sub = next;
    else if (integrate) I.cull_sub = -1;  // the free bodies moved
    I.counted(1);
    I.end(CAT_OTHER, ev);
}

void Engine::bc_pass(int bc) {
    Impl& I = *impl_;
    if (I.n == 0) return;
    Params P = I.params();
    P.bc = bc;
    launch_grid_bc(P, I.total_bricks, I.st);
    I.counted(1);
}

void Engine::materialize_stress() {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    if (I.n == 0 || I.use_stress_in) return;
    I.stress_in.alloc(36 * static_cast<size_t>(I.n));
    Params P = I.params();
    launch_stress(P, I.stress_in.as<float>(), I.st);
    I.counted(1);
    I.use_stress_in = true;
}

void Engine::pushout(int sub) {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    if (I.n == 0 || I.n_shapes == 0) return;
    Params P = I.params();
    P.sub = std::min(sub, I.table_subs - 1);
    launch_pushout(P, I.st);
    I.counted(1);
}

void Engine::deactivate() {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    if (I.n == 0) return;
    Params P = I.params();
    launch_deactivate(P, I.st);
    I.counted(1);
}

// ---------------------------------------------------------------- results
void Engine::reset_counters() {
    Impl& I = *impl_;
    I.export_req = false;  // a new frame: an export request left by a frame without particles lapses
    check(cudaMemsetAsync(I.counters.p, 0, I.counters.bytes, I.st), "memset");
}

void Engine::reset_contact(bool frame, bool sub) {
    Impl& I = *impl_;
    if (sub) {
        check(cudaMemsetAsync(I.acc_sub.p, 0, I.acc_sub.bytes, I.st), "memset");
        check(cudaMemsetAsync(I.cnt_sub.p, 0, I.cnt_sub.bytes, I.st), "memset");
    }
    if (frame) {
        check(cudaMemsetAsync(I.acc_frame.p, 0, I.acc_frame.bytes, I.st), "memset");
        check(cudaMemsetAsync(I.cnt_frame.p, 0, I.cnt_frame.bytes, I.st), "memset");
    }
}

std::vector<SceneCounters> Engine::read_counters() {
    Impl& I = *impl_;
    std::vector<SceneCounters> out(I.hs.size());
    check(cudaMemcpyAsync(out.data(), I.counters.p, sizeof(SceneCounters) * out.size(),
                          cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaStreamSynchronize(I.st), "sync");
    return out;
}

void Engine::stage_small() {
    Impl& I = *impl_;
    const size_t S = I.hs.size(), ns = static_cast<size_t>(std::max(I.n_shapes, 0));
    const size_t cb = sizeof(SceneCounters) * std::max<size_t>(S, 1);
    I.small_h.alloc(cb + sizeof(double) * 6 * ns + sizeof(int) * ns);
    char* h = static_cast<char*>(I.small_h.p);
    check(cudaMemcpyAsync(h, I.counters.p, sizeof(SceneCounters) * S, cudaMemcpyDeviceToHost, I.st), "d2h");
    if (ns > 0) {
        check(cudaMemcpyAsync(h + cb, I.acc_frame.p, sizeof(double) * 6 * ns, cudaMemcpyDeviceToHost, I.st), "d2h");
        check(cudaMemcpyAsync(h + cb + sizeof(double) * 6 * ns, I.cnt_frame.p, sizeof(int) * ns,
                              cudaMemcpyDeviceToHost, I.st), "d2h");
    }
}

void Engine::small_results(std::vector<SceneCounters>& cnt, std::vector<double>& imp, std::vector<double>& tq,
                           std::vector<int32_t>& cc) {
    Impl& I = *impl_;
    const size_t S = I.hs.size(), ns = static_cast<size_t>(std::max(I.n_shapes, 0));
    const size_t cb = sizeof(SceneCounters) * std::max<size_t>(S, 1);
    const char* h = static_cast<const char*>(I.small_h.p);
    cnt.assign(reinterpret_cast<const SceneCounters*>(h), reinterpret_cast<const SceneCounters*>(h) + S);
    imp.assign(3 * ns, 0.0);
    tq.assign(3 * ns, 0.0);
    cc.assign(ns, 0);
    if (ns == 0) return;
    const double* b = reinterpret_cast<const double*>(h + cb);
    std::memcpy(cc.data(), h + cb + sizeof(double) * 6 * ns, sizeof(int) * ns);
    for (size_t i = 0; i < ns; ++i)
        for (int a = 0; a < 3; ++a) {
            imp[3 * i + a] = b[6 * i + a];
            tq[3 * i + a] = b[6 * i + 3 + a];
        }
}

void Engine::read_contact(int which, std::vector<double>& imp, std::vector<double>& tq,
                          std::vector<int32_t>& cnt) {
    Impl& I = *impl_;
    const int ns = I.n_shapes;
    std::vector<double> buf(6 * std::max(ns, 1));
    cnt.assign(ns, 0);
    imp.assign(3 * ns, 0.0);
    tq.assign(3 * ns, 0.0);
    if (ns == 0) return;
    check(cudaMemcpyAsync(buf.data(), which ? I.acc_frame.p : I.acc_sub.p, sizeof(double) * 6 * ns,
                          cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaMemcpyAsync(cnt.data(), which ? I.cnt_frame.p : I.cnt_sub.p, sizeof(int) * ns,
                          cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaStreamSynchronize(I.st), "sync");
    for (int i = 0; i < ns; ++i)
        for (int a = 0; a < 3; ++a) {
            imp[3 * i + a] = buf[6 * i + a];
            tq[3 * i + a] = buf[6 * i + 3 + a];
        }
}

void Engine::snapshot(float* x, float* v, uint8_t* active, std::vector<double>& totals, bool async) {
    Impl& I = *impl_;
    const size_t N = static_cast<size_t>(std::max<int64_t>(I.n, 1));
    const size_t S = I.hs.size();
    if (async && I.export_valid) {  // the frame's last G2P already wrote the result and the totals
        I.export_valid = false;
        if (!I.copy_st) {
            check(cudaStreamCreateWithFlags(&I.copy_st, cudaStreamNonBlocking), "cudaStreamCreate");
            check(cudaEventCreateWithFlags(&I.ev_dl, cudaEventDisableTiming), "event");
            check(cudaEventCreateWithFlags(&I.ev_copy, cudaEventDisableTiming), "event");
            check(cudaEventCreateWithFlags(&I.ev_gather, cudaEventDisableTiming), "event");
        }
        I.io_tot_h.alloc(sizeof(double) * 5 * std::max<size_t>(S, 1));
        check(cudaMemcpyAsync(I.io_tot_h.p, I.io_tot.p, sizeof(double) * 5 * S, cudaMemcpyDeviceToHost, I.st),
              "d2h");
        check(cudaEventRecord(I.ev_dl, I.st), "event");
        check(cudaStreamWaitEvent(I.copy_st, I.ev_dl, 0), "wait download");
        // unpad on the copy stream (overlaps the next frame), then the packed arrays' D2H
        if (I.copy_pending && (I.io_x.bytes < 12 * N || I.io_v.bytes < 12 * N || I.io_a.bytes < N))
            wait_results();
        I.io_x.alloc(12 * N);
        I.io_v.alloc(12 * N);
        I.io_a.alloc(N);
        launch_export_pack(I.io_pad.as<float4>(), I.n, x ? I.io_x.as<float>() : nullptr,
                           v ? I.io_v.as<float>() : nullptr, active ? I.io_a.as<uint8_t>() : nullptr, I.copy_st);
        I.counted(1);
        if (x) check(cudaMemcpyAsync(x, I.io_x.p, 12 * I.n, cudaMemcpyDeviceToHost, I.copy_st), "d2h");
        if (v) check(cudaMemcpyAsync(v, I.io_v.p, 12 * I.n, cudaMemcpyDeviceToHost, I.copy_st), "d2h");
        if (active) check(cudaMemcpyAsync(active, I.io_a.p, I.n, cudaMemcpyDeviceToHost, I.copy_st), "d2h");
        check(cudaEventRecord(I.ev_copy, I.copy_st), "event");
        I.copy_pending = true;
        check(cudaStreamSynchronize(I.st), "snapshot");
        const double* th = static_cast<const double*>(I.io_tot_h.p);
        totals.assign(th, th + 5 * S);
        return;
    }
    I.export_valid = false;
    if (I.copy_pending && (I.io_x.bytes < 12 * N || I.io_v.bytes < 12 * N || I.io_a.bytes < N))
        wait_results();  // the staging is about to be reallocated
    if (I.copy_pending) check(cudaStreamWaitEvent(I.st, I.ev_copy, 0), "wait copy");  // staging reuse
    if (async && !I.copy_st) {
        check(cudaStreamCreateWithFlags(&I.copy_st, cudaStreamNonBlocking), "cudaStreamCreate");
        check(cudaEventCreateWithFlags(&I.ev_dl, cudaEventDisableTiming), "event");
        check(cudaEventCreateWithFlags(&I.ev_copy, cudaEventDisableTiming), "event");
        check(cudaEventCreateWithFlags(&I.ev_gather, cudaEventDisableTiming), "event");
    }
    cudaStream_t cs = async ? I.copy_st : I.st;
    I.io_tot.alloc(sizeof(double) * 5 * std::max<size_t>(S, 1));
    check(cudaMemsetAsync(I.io_tot.p, 0, I.io_tot.bytes, I.st), "memset");
    Params P = I.params();
    IoArrays io{};
    if (I.n > 0) {
        if (x) { I.io_x.alloc(12 * N); io.x = I.io_x.as<float>(); }
        if (v) { I.io_v.alloc(12 * N); io.v = I.io_v.as<float>(); }
        if (active) { I.io_a.alloc(N); io.active = I.io_a.as<uint8_t>(); }
        I.io_inv.alloc(4 * N);
        if (async) {  // totals now (the caller waits for them), the arrays on the copy stream
            launch_totals(P, I.io_tot.as<double>(), I.st);
            I.counted(1);
        } else {
            launch_frame_result_orig(P, I.io_inv.as<uint32_t>(), I.n, io, I.io_tot.as<double>(), I.st);
            I.counted(2);
        }
    }
    // the small totals copy goes first: queued behind the arrays on the same copy engine it
    // would hold the host for the whole transfer
    I.io_tot_h.alloc(sizeof(double) * 5 * std::max<size_t>(S, 1));
    check(cudaMemcpyAsync(I.io_tot_h.p, I.io_tot.p, sizeof(double) * 5 * S, cudaMemcpyDeviceToHost, I.st), "d2h");
    if (I.n > 0) {
        if (async) {
            // K9 on the copy stream: it reads the planes of this frame while the next frame's
            // P2G and grid update (read-only) run; plane writers wait for ev_gather
            check(cudaEventRecord(I.ev_dl, I.st), "event");
            check(cudaStreamWaitEvent(cs, I.ev_dl, 0), "wait download");
            launch_frame_result_orig(P, I.io_inv.as<uint32_t>(), I.n, io, nullptr, cs);
            I.counted(2);
            check(cudaEventRecord(I.ev_gather, cs), "event");
            I.gather_pending = true;
        }
        if (x) check(cudaMemcpyAsync(x, I.io_x.p, 12 * I.n, cudaMemcpyDeviceToHost, cs), "d2h");
        if (v) check(cudaMemcpyAsync(v, I.io_v.p, 12 * I.n, cudaMemcpyDeviceToHost, cs), "d2h");
        if (active) check(cudaMemcpyAsync(active, I.io_a.p, I.n, cudaMemcpyDeviceToHost, cs), "d2h");
        if (async) {
            check(cudaEventRecord(I.ev_copy, cs), "event");
            I.copy_pending = true;
        }
    }
    check(cudaStreamSynchronize(I.st), "snapshot");
    const double* th = static_cast<const double*>(I.io_tot_h.p);
    totals.assign(th, th + 5 * S);
}

std::shared_ptr<void> Engine::pinned_host(size_t bytes) {
    void* p = nullptr;
    check(cudaMallocHost(&p, bytes ? bytes : 16), "cudaMallocHost");
    return std::shared_ptr<void>(p, [](void* q) { cudaFreeHost(q); });
}

void Engine::host_register(void* p, size_t bytes) {
    if (p && bytes) check(cudaHostRegister(p, bytes, cudaHostRegisterPortable), "cudaHostRegister");
}

void Engine::eval_stress_f32(const float* F, int64_t n, float mu, float lambda, float* sigma, float* J) {
    mpmb::eval_stress_f32(F, n, mu, lambda, sigma, J);
}

void Engine::host_unregister(void* p) {
    if (p) check(cudaHostUnregister(p), "cudaHostUnregister");
}

void Engine::enable_grid_readback() {
    Impl& I = *impl_;
    if (I.dead_mom.p) return;
    I.dead_mom.alloc(sizeof(float4) * I.total_nodes);
    check(cudaMemsetAsync(I.dead_mom.p, 0, sizeof(float4) * I.total_nodes, I.st), "memset");
}

void Engine::download_grid(int scene, float* mass, float* mom, float* vel) {
    Impl& I = *impl_;
    const DevScene& S = I.hs[scene];
    const size_t nn = static_cast<size_t>(S.dims[0]) * S.dims[1] * S.dims[2];
    DevBuf dm, dp, dv;
    dm.alloc(4 * nn); dp.alloc(12 * nn); dv.alloc(12 * nn);
    Params P = I.params();
    launch_grid_download(P, scene, S, dm.as<float>(), dp.as<float>(), dv.as<float>(), I.st);
    I.counted(1);
    if (mass) check(cudaMemcpyAsync(mass, dm.p, 4 * nn, cudaMemcpyDeviceToHost, I.st), "d2h");
    if (mom) check(cudaMemcpyAsync(mom, dp.p, 12 * nn, cudaMemcpyDeviceToHost, I.st), "d2h");
    if (vel) check(cudaMemcpyAsync(vel, dv.p, 12 * nn, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaStreamSynchronize(I.st), "grid");
}

void Engine::upload_grid_velocity(int scene, const float* mass, const float* mom, const float* vel) {
    Impl& I = *impl_;
    const DevScene& S = I.hs[scene];
    const size_t nn = static_cast<size_t>(S.dims[0]) * S.dims[1] * S.dims[2];
    DevBuf dm, dp, dv;
    dm.alloc(4 * nn); dp.alloc(12 * nn); dv.alloc(12 * nn);
    check(cudaMemcpyAsync(dm.p, mass, 4 * nn, cudaMemcpyHostToDevice, I.st), "h2d");
    check(cudaMemcpyAsync(dp.p, mom, 12 * nn, cudaMemcpyHostToDevice, I.st), "h2d");
    check(cudaMemcpyAsync(dv.p, vel, 12 * nn, cudaMemcpyHostToDevice, I.st), "h2d");
    Params P = I.params();
    launch_grid_upload(P, scene, S, dm.as<float>(), dp.as<float>(), dv.as<float>(), I.st);
    I.counted(1);
    check(cudaStreamSynchronize(I.st), "grid");
}

void Engine::read_binning(uint32_t* keys, uint32_t* perm) {
    Impl& I = *impl_;
    if (I.n == 0) return;
    const size_t N = static_cast<size_t>(I.n);
    DevBuf kbo;
    kbo.alloc(4 * N);
    I.bb.key_by_orig = kbo.as<uint32_t>();
    bin();
    I.bb.key_by_orig = nullptr;
    if (keys) check(cudaMemcpyAsync(keys, kbo.p, 4 * N, cudaMemcpyDeviceToHost, I.st), "d2h");
    if (perm) check(cudaMemcpyAsync(perm, I.s_orig.p, 4 * N, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaStreamSynchronize(I.st), "binning");
}

int64_t Engine::n_active_sorted() {
    Impl& I = *impl_;
    uint32_t c[3] = {0, 0, 0};
    check(cudaMemcpyAsync(c, I.b_counts.p, 12, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaStreamSynchronize(I.st), "sync");
    return c[2];
}

void Engine::wait_results() {
    Impl& I = *impl_;
    if (!I.copy_pending) return;
    I.copy_pending = false;
    check(cudaEventSynchronize(I.ev_copy), "snapshot copy");
}

void Engine::synchronize() {
    check(cudaStreamSynchronize(impl_->st), "synchronize");
    wait_results();
}

// ------------------------------------------------ scenario metrics (k_scenario.cu)
void Engine::components(const float* radius, int32_t* counts) {
    Impl& I = *impl_;
    const size_t S = I.hs.size();
    if (I.n_cap == 0) {
        std::fill(counts, counts + S, 0);
        return;
    }
    DevBuf cell, cnt, scratch;
    cell.alloc(4 * S); cnt.alloc(4 * S);
    const size_t sb = scenario_scratch_bytes(I.n_cap, static_cast<int>(S));
    scratch.alloc(sb);
    check(cudaMemcpyAsync(cell.p, radius, 4 * S, cudaMemcpyHostToDevice, I.st), "h2d");
    Params P = I.params();
    launch_scenario(P, 0, cell.as<float>(), scratch.p, sb, cnt.as<int32_t>(), nullptr, nullptr, static_cast<int>(S), I.st);
    I.counted(6);
    check(cudaMemcpyAsync(counts, cnt.p, 4 * S, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaStreamSynchronize(I.st), "components");
}

void Engine::nn_best2(const float* cell_size, float* best2) {
    Impl& I = *impl_;
    const size_t S = I.hs.size();
    if (I.n_cap == 0) return;
    const size_t N = static_cast<size_t>(I.n_cap);
    DevBuf cell, b2, orig, scratch;
    cell.alloc(4 * S); b2.alloc(4 * N); orig.alloc(4 * N);
    const size_t sb = scenario_scratch_bytes(I.n_cap, static_cast<int>(S));
    scratch.alloc(sb);
    check(cudaMemcpyAsync(cell.p, cell_size, 4 * S, cudaMemcpyHostToDevice, I.st), "h2d");
    Params P = I.params();
    launch_scenario(P, 1, cell.as<float>(), scratch.p, sb, nullptr, b2.as<float>(), orig.as<uint32_t>(),
                    static_cast<int>(S), I.st);
    I.counted(4);
    std::vector<float> hb(N);
    std::vector<uint32_t> ho(N);
    check(cudaMemcpyAsync(hb.data(), b2.p, 4 * N, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaMemcpyAsync(ho.data(), orig.p, 4 * N, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaStreamSynchronize(I.st), "nn_best2");
    std::fill(best2, best2 + I.n, FLT_MAX);
    std::vector<uint8_t> act(static_cast<size_t>(I.n), 0);
    // slots that are not active particles keep FLT_MAX; hb is only meaningful for active ones
    for (size_t s = 0; s < N; ++s)
        if (ho[s] != 0xFFFFFFFFu && ho[s] < static_cast<uint32_t>(I.n)) best2[ho[s]] = hb[s];
}

// ------------------------------------------------ slab domain decomposition (k_dd.cu)
void Engine::set_capacity(int64_t particles) { impl_->cap_hint = std::max<int64_t>(0, particles); }

int64_t Engine::slot_count() const { return impl_->n_cap; }

int Engine::dd_halo_planes(int side_send_hi, bool acc) const {
    // acc: low ghosts M planes, high ghosts 2 + M; vel: the mirror image
    const int M = impl_->margin;
    return (side_send_hi != 0) == acc ? 2 + M : M;
}

void Engine::ensure_halo() {
    Impl& I = *impl_;
    if (I.slab_hi <= I.slab_lo) throw std::invalid_argument("engine: not a slab domain");
    Params P = I.params();
    const int64_t b = dd_plane_nodes(P) * (2 + I.margin) * static_cast<int64_t>(sizeof(float4));
    if (I.halo_bytes != b) {
        for (int q = 0; q < 4; ++q) {
            I.halo[q].alloc(b);
            check(cudaMemset(I.halo[q].p, 0, b), "memset");  // a missing neighbour sends zeros
        }
        I.halo_bytes = b;
    }
}

void Engine::dd_halo_buffers(void** send_lo, void** send_hi, void** recv_lo, void** recv_hi, int64_t* bytes) {
    Impl& I = *impl_;
    ensure_halo();
    const int64_t b = I.halo_bytes;
    *send_lo = I.halo[0].p; *send_hi = I.halo[1].p; *recv_lo = I.halo[2].p; *recv_hi = I.halo[3].p;
    *bytes = b;
}

// the y/z window of the halo planes (whole storage extent unless dd_set_window narrowed it)
static void halo_window(const Params& P, const int win[4], int& y0, int& ny, int& z0, int& nz) {
    if (win[1] > 0) {
        y0 = win[0]; ny = win[1]; z0 = win[2]; nz = win[3];
    } else {
        y0 = 0; ny = P.geo.nb[1] * 4; z0 = 0; nz = P.geo.nb[2] * 4;
    }
}

void Engine::dd_pack_acc() {
    Impl& I = *impl_;
    ensure_halo();
    Params P = I.params();
    int y0, ny, z0, nz;
    halo_window(P, I.win, y0, ny, z0, nz);
    launch_halo(P, 0, P.grid_acc, I.halo[0].as<float4>(), 0, I.margin, y0, ny, z0, nz, I.st);
    launch_halo(P, 0, P.grid_acc, I.halo[1].as<float4>(), P.geo.own_hi, 2 + I.margin, y0, ny, z0, nz, I.st);
    I.counted(2);
}

void Engine::dd_unpack_acc() {
    Impl& I = *impl_;
    ensure_halo();
    Params P = I.params();
    int y0, ny, z0, nz;
    halo_window(P, I.win, y0, ny, z0, nz);
    launch_halo(P, 1, P.grid_acc, I.halo[3].as<float4>(), P.geo.own_hi - I.margin, I.margin, y0, ny, z0, nz, I.st);
    launch_halo(P, 1, P.grid_acc, I.halo[2].as<float4>(), P.geo.own_lo, 2 + I.margin, y0, ny, z0, nz, I.st);
    I.counted(2);
}

void Engine::dd_pack_vel() {
    Impl& I = *impl_;
    ensure_halo();
    Params P = I.params();
    int y0, ny, z0, nz;
    halo_window(P, I.win, y0, ny, z0, nz);
    launch_halo(P, 0, P.grid_vel, I.halo[0].as<float4>(), P.geo.own_lo, 2 + I.margin, y0, ny, z0, nz, I.st);
    launch_halo(P, 0, P.grid_vel, I.halo[1].as<float4>(), P.geo.own_hi - I.margin, I.margin, y0, ny, z0, nz, I.st);
    I.counted(2);
}

void Engine::dd_unpack_vel() {
    Impl& I = *impl_;
    ensure_halo();
    Params P = I.params();
    int y0, ny, z0, nz;
    halo_window(P, I.win, y0, ny, z0, nz);
    launch_halo(P, 2, P.grid_vel, I.halo[2].as<float4>(), 0, I.margin, y0, ny, z0, nz, I.st);
    launch_halo(P, 2, P.grid_vel, I.halo[3].as<float4>(), P.geo.own_hi, 2 + I.margin, y0, ny, z0, nz, I.st);
    I.counted(2);
}

void Engine::dd_set_window(int y0, int y1, int z0, int z1) {
    Impl& I = *impl_;
    const int py = I.geo.nb[1] * 4, pz = I.geo.nb[2] * 4;
    y0 = std::max(y0, 0); z0 = std::max(z0, 0);
    y1 = std::min(y1, py); z1 = std::min(z1, pz);
    if (y1 <= y0 || z1 <= z0) {  // empty: keep one node so the buffers stay well formed
        y1 = y0 + 1; z1 = z0 + 1;
    }
    I.win[0] = y0; I.win[1] = y1 - y0; I.win[2] = z0; I.win[3] = z1 - z0;
}

void Engine::dd_plane_window(int* y0, int* ny, int* z0, int* nz) {
    Impl& I = *impl_;
    Params P = I.params();
    int a, b, c2, d;
    halo_window(P, I.win, a, b, c2, d);
    *y0 = a; *ny = b; *z0 = c2; *nz = d;
}

void Engine::particle_window(int out[4]) {
    dd_window_async();  // persistent device buffer (no per-call allocation)
    const DDControl c = dd_control();
    std::memcpy(out, c.window, sizeof(c.window));
}

void Engine::collect_bricks() {
    Impl& I = *impl_;
    if (I.n_cap == 0) return;
    Params P = I.params();
    launch_collect_bricks(P, I.total_bricks, I.st);
    I.counted(1);
    I.flag_parity = 1 - I.flag_parity;
}

void Engine::dd_migrate_buffers(void** send_lo, void** send_hi, void** recv_lo, void** recv_hi, int64_t* cap) {
    Impl& I = *impl_;
    const int64_t c = std::max<int64_t>(1024, I.n_cap / 4);
    if (I.mig_cap != c) {
        for (int q = 0; q < 4; ++q) I.mig[q].alloc(static_cast<size_t>(c) * kPlanes * sizeof(float4));
        I.mig_counts.alloc(2 * sizeof(uint32_t));
        I.mig_cap = c;
    }
    *send_lo = I.mig[0].p; *send_hi = I.mig[1].p; *recv_lo = I.mig[2].p; *recv_hi = I.mig[3].p;
    *cap = c;
}

void Engine::dd_migrate_pack(int64_t* n_lo, int64_t* n_hi) {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    void* d[4];
    int64_t cap;
    dd_migrate_buffers(&d[0], &d[1], &d[2], &d[3], &cap);
    uint32_t c[2] = {0, 0};
    if (I.n_cap > 0) {
        check(cudaMemsetAsync(I.mig_counts.p, 0, 2 * sizeof(uint32_t), I.st), "memset");
        Params P = I.params();
        launch_migrate_pack(P, I.slab_lo, I.slab_hi, I.mig[0].as<float4>(), I.mig[1].as<float4>(),
                            static_cast<uint32_t>(cap), I.mig_counts.as<uint32_t>(), I.st);
        I.counted(1);
        check(cudaMemcpyAsync(c, I.mig_counts.p, sizeof(c), cudaMemcpyDeviceToHost, I.st), "d2h");
        check(cudaStreamSynchronize(I.st), "migrate");
    }
    if (c[0] > cap || c[1] > cap) throw std::runtime_error("engine: migration buffer overflow");
    *n_lo = c[0];
    *n_hi = c[1];
    I.mig_sent = c[0] + c[1];
}

void Engine::dd_migrate_unpack(int64_t n_from_lo, int64_t n_from_hi) {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    if (n_from_lo > I.mig_cap || n_from_hi > I.mig_cap) throw std::invalid_argument("engine: migration count");
    const int64_t arrivals = n_from_lo + n_from_hi;
    if (arrivals == 0 && I.binned) {
        // departures only left holes inside their groups (never active): the binned layout
        // stays valid, so no re-binning
        I.n -= I.mig_sent;
        n_total_ = I.n;
        I.mig_sent = 0;
        return;
    }
    int64_t first = I.n;  // upload layout: particles then holes
    if (I.binned) {       // binned layout: groups, then the inactive tail, then holes
        if (I.free_slot < 0) {
            uint32_t c[4] = {0, 0, 0, 0};
            check(cudaMemcpyAsync(c, I.b_counts.p, sizeof(c), cudaMemcpyDeviceToHost, I.st), "d2h");
            check(cudaStreamSynchronize(I.st), "migrate");
            I.free_slot = static_cast<int64_t>(c[3]) + (I.n_at_bin - static_cast<int64_t>(c[2]));
        }
        // a fresh group: inside a group the transfers scatter the particles over its slots
        // (group_phys), so nothing may be appended behind a partly filled one
        first = (I.free_slot + kGroup - 1) / kGroup * kGroup;
    }
    if (first + arrivals > I.n_cap) throw std::runtime_error("engine: slab capacity exceeded (set_capacity)");
    Params P = I.params();
    launch_migrate_unpack(P, I.mig[2].as<float4>(), static_cast<uint32_t>(n_from_lo), static_cast<uint32_t>(first), I.st);
    launch_migrate_unpack(P, I.mig[3].as<float4>(), static_cast<uint32_t>(n_from_hi),
                          static_cast<uint32_t>(first + n_from_lo), I.st);
    I.counted(2);
    I.n += arrivals - I.mig_sent;
    n_total_ = I.n;
    I.mig_sent = 0;
    // A few arrivals become extra groups over [old groups, first + arrivals): they take the
    // inactive tail and some holes along (the transfers handle both), and P2G's per-substep
    // warp sort orders them.  The other buffer gets the same slots (the transfers rewrite
    // only grouped slots, which must start identical in both).  Many arrivals, or many
    // appends since the last binning, re-bin instead (spatial compactness of the groups).
    if (I.binned && arrivals * 64 <= I.n && I.appends < 16) {
        const uint64_t end = static_cast<uint64_t>(first + arrivals);
        const uint32_t groups = static_cast<uint32_t>((end + kGroup - 1) / kGroup);
        const uint32_t tail = groups * static_cast<uint32_t>(kGroup);
        for (int q = 0; q < kPlanes; ++q)
            check(cudaMemcpyAsync(I.planes[1 - I.cur][q].as<float4>() + first, I.planes[I.cur][q].as<float4>() + first,
                                  sizeof(float4) * arrivals, cudaMemcpyDeviceToDevice, I.st), "copy");
        uint32_t c2[2] = {groups, tail};
        check(cudaMemcpyAsync(static_cast<uint32_t*>(I.b_counts.p) + 1, &c2[0], 4, cudaMemcpyHostToDevice, I.st), "h2d");
        check(cudaMemcpyAsync(static_cast<uint32_t*>(I.b_counts.p) + 3, &c2[1], 4, cudaMemcpyHostToDevice, I.st), "h2d");
        check(cudaStreamSynchronize(I.st), "groups");  // c2 is on the host stack
        I.free_slot = static_cast<int64_t>(tail);
        ++I.appends;
        return;
    }
    I.binned = false;
    bin();
}

// ------------------------------------------------ device-resident slab DD (dd_driver.cpp)
void Engine::collect_deferred(int next_sub, float dt, const float g[3], bool integrate) {
    Impl& I = *impl_;
    if (I.n_cap == 0) return;
    Params P = I.params();
    P.dt = dt;
    P.g[0] = g[0]; P.g[1] = g[1]; P.g[2] = g[2];
    if (I.n_shapes > 0) {
        const int next = std::min(next_sub, I.table_subs - 1);
        P.sub = std::max(0, std::min(next_sub - 1, I.table_subs - 1));
        launch_collect_free(P, I.total_bricks, integrate, true, next, I.st);
        I.cull_sub = next;
    } else {
        launch_collect_bricks(P, I.total_bricks, I.st);
    }
    I.counted(1);
    I.flag_parity = 1 - I.flag_parity;
}

void Engine::dd_window_async() {
    Impl& I = *impl_;
    if (!I.dd_win.p) I.dd_win.alloc(8 * sizeof(int));
    launch_window_init(I.dd_win.as<int>(), I.st);
    I.counted(1);
    if (I.n_cap > 0) {
        Params P = I.params(true);
        launch_particle_window(P, I.dd_win.as<int>(), I.st);
        I.counted(1);
    }
}

uint32_t* Engine::dd_control_device() { return impl_->b_counts.as<uint32_t>() + 4; }

int* Engine::dd_window_device() {
    Impl& I = *impl_;
    if (!I.dd_win.p) dd_window_async();
    return I.dd_win.as<int>();
}

static Engine::DDControl parse_ctl(const uint32_t* h);

Engine::DDControl Engine::dd_control() {
    Impl& I = *impl_;
    if (!I.dd_win.p) dd_window_async();
    I.dd_ctl_h.alloc(12 * sizeof(uint32_t));
    auto* h = static_cast<uint32_t*>(I.dd_ctl_h.p);
    check(cudaMemcpyAsync(h, I.dd_win.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaMemcpyAsync(h + 8, I.b_counts.as<uint32_t>() + 4, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, I.st),
          "d2h");
    check(cudaStreamSynchronize(I.st), "dd control");
    return parse_ctl(h);
}

static Engine::DDControl parse_ctl(const uint32_t* h) {
    Engine::DDControl c{};
    std::memcpy(c.window, h, 4 * sizeof(int));
    c.group_err = h[4];
    c.free_slot = h[8];
    c.arrivals = h[9];
    c.err = h[10];
    c.n_real = h[11];
    return c;
}

void Engine::dd_snapshot_async(int slot) {
    Impl& I = *impl_;
    slot &= 1;
    if (!I.dd_snap_ev[slot]) check(cudaEventCreateWithFlags(&I.dd_snap_ev[slot], cudaEventDisableTiming), "event");
    I.dd_snap_h[slot].alloc(12 * sizeof(uint32_t));
    auto* h = static_cast<uint32_t*>(I.dd_snap_h[slot].p);
    check(cudaMemcpyAsync(h, I.dd_win.p, 8 * sizeof(int), cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaMemcpyAsync(h + 8, I.b_counts.as<uint32_t>() + 4, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, I.st),
          "d2h");
    check(cudaEventRecord(I.dd_snap_ev[slot], I.st), "event");
}

Engine::DDControl Engine::dd_snapshot_read(int slot, bool* blocked) {
    Impl& I = *impl_;
    slot &= 1;
    if (!I.dd_snap_ev[slot]) throw std::logic_error("engine: no DD snapshot in this slot");
    const cudaError_t q = cudaEventQuery(I.dd_snap_ev[slot]);
    if (q != cudaSuccess && q != cudaErrorNotReady) check(q, "event query");
    if (blocked) *blocked = q == cudaErrorNotReady;
    check(cudaEventSynchronize(I.dd_snap_ev[slot]), "dd snapshot");
    return parse_ctl(static_cast<const uint32_t*>(I.dd_snap_h[slot].p));
}

void Engine::dd_clear_errors() {
    Impl& I = *impl_;
    check(cudaMemsetAsync(I.b_counts.as<uint32_t>() + 6, 0, sizeof(uint32_t), I.st), "memset");
}

void Engine::dd_set_migration_capacity(int64_t cap) {
    Impl& I = *impl_;
    cap = std::max<int64_t>(cap, 256);
    if (I.mig_cap == cap) return;
    for (int q = 0; q < 4; ++q) I.mig[q].alloc(static_cast<size_t>(cap) * kPlanes * sizeof(float4));
    I.mig_counts.alloc(4 * sizeof(uint32_t));
    check(cudaMemsetAsync(I.mig_counts.p, 0, 4 * sizeof(uint32_t), I.st), "memset");
    I.mig_cap = cap;
}

void Engine::dd_migration_buffers(void** send_lo, void** send_hi, void** recv_lo, void** recv_hi,
                                  uint32_t** counts, int64_t* cap) {
    Impl& I = *impl_;
    if (I.mig_cap == 0) dd_set_migration_capacity(std::max<int64_t>(1024, I.n_cap / 64));
    *send_lo = I.mig[0].p; *send_hi = I.mig[1].p; *recv_lo = I.mig[2].p; *recv_hi = I.mig[3].p;
    *counts = I.mig_counts.as<uint32_t>();
    *cap = I.mig_cap;
}

void Engine::dd_migrate_pack_async(bool has_lo, bool has_hi) {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    void* d[4];
    uint32_t* cnt;
    int64_t cap;
    dd_migration_buffers(&d[0], &d[1], &d[2], &d[3], &cnt, &cap);
    check(cudaMemsetAsync(cnt, 0, 4 * sizeof(uint32_t), I.st), "memset");  // received counts arrive after
    if (I.n_cap == 0) return;
    Params P = I.params();
    int y0, ny, z0, nz;
    halo_window(P, I.win, y0, ny, z0, nz);
    launch_migrate_pack_dev(P, I.slab_lo, I.slab_hi, I.margin, make_int4(y0, y0 + ny, z0, z0 + nz), has_lo, has_hi,
                            I.mig[0].as<float4>(), I.mig[1].as<float4>(), static_cast<uint32_t>(cap), cnt,
                            I.b_counts.as<uint32_t>() + 4, I.st);
    I.counted(1);
}

void Engine::dd_migrate_unpack_async() {
    Impl& I = *impl_;
    I.export_valid = false;  // the staged frame result no longer matches the state
    if (I.n_cap == 0) return;
    Params P = I.params();
    launch_migrate_unpack_dev(P, I.mig[2].as<float4>(), I.mig[3].as<float4>(), static_cast<uint32_t>(I.mig_cap),
                              I.mig_counts.as<uint32_t>(), I.b_counts.as<uint32_t>(), static_cast<uint64_t>(I.n_cap),
                              I.st);
    I.counted(2);
}

void Engine::dd_note_count(int64_t n_real) {
    Impl& I = *impl_;
    if (!I.binned) return;  // the control words are set by the first binning
    I.n = n_real;
    n_total_ = n_real;
}

int64_t Engine::download_compact(int64_t capacity, uint32_t* ids, float* x, float* v, uint8_t* active) {
    Impl& I = *impl_;
    if (I.n_cap == 0) return 0;
    const size_t N = static_cast<size_t>(I.n_cap);
    DevBuf &di = I.dl_ids, &dx = I.dl_x, &dv = I.dl_v, &da = I.dl_a, &dc = I.dl_cnt;
    di.alloc(4 * N); dx.alloc(12 * N); dv.alloc(12 * N); da.alloc(N); dc.alloc(4);
    check(cudaMemsetAsync(dc.p, 0, 4, I.st), "memset");
    Params P = I.params();
    launch_download_slots(P, di.as<uint32_t>(), dx.as<float>(), dv.as<float>(), da.as<uint8_t>(), dc.as<uint32_t>(),
                          I.st);
    I.counted(1);
    uint32_t k = 0;
    check(cudaMemcpyAsync(&k, dc.p, 4, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaStreamSynchronize(I.st), "download");
    if (static_cast<int64_t>(k) > capacity) throw std::invalid_argument("download: capacity too small");
    check(cudaMemcpyAsync(ids, di.p, 4ull * k, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaMemcpyAsync(x, dx.p, 12ull * k, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaMemcpyAsync(v, dv.p, 12ull * k, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaMemcpyAsync(active, da.p, k, cudaMemcpyDeviceToHost, I.st), "d2h");
    check(cudaStreamSynchronize(I.st), "download");
    return k;
}

}  // namespace mpmb
