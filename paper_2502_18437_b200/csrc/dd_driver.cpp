// dd_driver.cpp — device-resident slab DD driver (dd_driver.h).  Host C++; kernels are
// reached through Engine methods and dd_ops.h.
#include "dd_driver.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types and enums only: the functions are loaded with dlopen

#include <algorithm>
#include <climits>
#include <cstring>
#include <stdexcept>
#include <string>

#include "dd_ops.h"

namespace mpmb {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// NCCL loaded at run time: the copy torch already mapped (same soname), else the system one.
struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;

    static Nccl& get() {
        static Nccl n = [] {
            Nccl a;
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
            if (!h) throw std::runtime_error(std::string("slab DD over NCCL: cannot load libnccl.so.2: ") + dlerror());
            auto sym = [&](const char* name) {
                void* f = dlsym(h, name);
                if (!f) throw std::runtime_error(std::string("slab DD over NCCL: missing symbol ") + name);
                return f;
            };
            a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
            a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
            a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
            a.send = reinterpret_cast<decltype(a.send)>(sym("ncclSend"));
            a.recv = reinterpret_cast<decltype(a.recv)>(sym("ncclRecv"));
            a.group_start = reinterpret_cast<decltype(a.group_start)>(sym("ncclGroupStart"));
            a.group_end = reinterpret_cast<decltype(a.group_end)>(sym("ncclGroupEnd"));
            a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(sym("ncclAllReduce"));
            a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
            return a;
        }();
        return n;
    }
    void ok(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL error in ") + what + ": " + error_string(r));
    }
};

struct Halo {
    void *send_lo, *send_hi, *recv_lo, *recv_hi;
};
Halo halo_of(Engine* e) {
    Halo h{};
    int64_t bytes = 0;
    e->dd_halo_buffers(&h.send_lo, &h.send_hi, &h.recv_lo, &h.recv_hi, &bytes);
    return h;
}

struct Mig {
    void *send_lo, *send_hi, *recv_lo, *recv_hi;
    uint32_t* counts;  // {sent down, sent up, received from below, received from above}
    int64_t cap;
};
Mig mig_of(Engine* e) {
    Mig m{};
    e->dd_migration_buffers(&m.send_lo, &m.send_hi, &m.recv_lo, &m.recv_hi, &m.counts, &m.cap);
    return m;
}

}  // namespace

// ------------------------------------------------------------------ transports
class DDTransport {
  public:
    virtual ~DDTransport() = default;
    cudaStream_t st = nullptr;
    // global position of local slab i and the number of slabs
    virtual int index(size_t i) const = 0;
    virtual int count() const = 0;
    // every slab sends send_lo (bytes_down) down and send_hi (bytes_up) up; what arrives
    // from below is the lower slab's up payload, from above the upper's down payload
    virtual void halo(const std::vector<Engine*>& s, size_t bytes_down, size_t bytes_up) = 0;
    // counts (4 B each way) and the fixed-capacity payloads
    virtual void migrate(const std::vector<Engine*>& s) = 0;
    // per-shape contact sums of the substep summed over every slab, on every slab
    virtual void contact_sums(const std::vector<Engine*>& s) = 0;
    // end of a run: every slab's window of the particles' reach (NCCL: all-reduced with the
    // error flags of every rank) and control words, copied to pinned host slot `slot`
    virtual void snapshot(const std::vector<Engine*>& s, int slot) = 0;
    // start of a later run: the union window and the OR of the error flags from slot `slot`;
    // returns how many reads had to wait for the device
    virtual int64_t read(const std::vector<Engine*>& s, int slot, int win[4], uint32_t& err,
                         std::vector<uint32_t>& n_real, std::vector<uint32_t>& arrivals,
                         std::vector<uint32_t>& free_slot) = 0;
    // the migration payload capacity every slab uses (must agree)
    virtual int64_t agree_max(int64_t v) = 0;
};

namespace {

class LocalTransport final : public DDTransport {
  public:
    explicit LocalTransport(size_t n) : n_(n) {}
    int index(size_t i) const override { return static_cast<int>(i); }
    int count() const override { return static_cast<int>(n_); }
    void halo(const std::vector<Engine*>& s, size_t down, size_t up) override {
        for (size_t i = 0; i < s.size(); ++i) {
            const Halo h = halo_of(s[i]);
            if (i > 0) ck(cudaMemcpyAsync(halo_of(s[i - 1]).recv_hi, h.send_lo, down, cudaMemcpyDeviceToDevice, st), "halo");
            if (i + 1 < s.size())
                ck(cudaMemcpyAsync(halo_of(s[i + 1]).recv_lo, h.send_hi, up, cudaMemcpyDeviceToDevice, st), "halo");
        }
    }
    void migrate(const std::vector<Engine*>& s) override {
        for (size_t i = 0; i < s.size(); ++i) {
            const Mig m = mig_of(s[i]);
            const size_t pay = static_cast<size_t>(m.cap) * 7 * 16;
            if (i > 0) {
                const Mig d = mig_of(s[i - 1]);
                ck(cudaMemcpyAsync(d.counts + 3, m.counts + 0, 4, cudaMemcpyDeviceToDevice, st), "migrate");
                ck(cudaMemcpyAsync(d.recv_hi, m.send_lo, pay, cudaMemcpyDeviceToDevice, st), "migrate");
            }
            if (i + 1 < s.size()) {
                const Mig u = mig_of(s[i + 1]);
                ck(cudaMemcpyAsync(u.counts + 2, m.counts + 1, 4, cudaMemcpyDeviceToDevice, st), "migrate");
                ck(cudaMemcpyAsync(u.recv_lo, m.send_hi, pay, cudaMemcpyDeviceToDevice, st), "migrate");
            }
        }
    }
    void contact_sums(const std::vector<Engine*>& s) override {
        if (s.size() < 2) return;
        void *s0, *c0;
        int ns = 0;
        s[0]->contact_sub_buffers(&s0, &c0, &ns);
        if (ns == 0) return;
        for (size_t i = 1; i < s.size(); ++i) {
            void *si, *ci;
            s[i]->contact_sub_buffers(&si, &ci, nullptr);
            dd_add_f64(static_cast<double*>(s0), static_cast<const double*>(si), 6 * ns, st);
            dd_add_i32(static_cast<int32_t*>(c0), static_cast<const int32_t*>(ci), ns, st);
        }
        for (size_t i = 1; i < s.size(); ++i) {
            void *si, *ci;
            s[i]->contact_sub_buffers(&si, &ci, nullptr);
            ck(cudaMemcpyAsync(si, s0, 6 * sizeof(double) * ns, cudaMemcpyDeviceToDevice, st), "contact");
            ck(cudaMemcpyAsync(ci, c0, sizeof(int32_t) * ns, cudaMemcpyDeviceToDevice, st), "contact");
        }
    }
    void snapshot(const std::vector<Engine*>& s, int slot) override {
        for (Engine* e : s) {
            e->dd_window_async();
            e->dd_snapshot_async(slot);
        }
    }
    int64_t read(const std::vector<Engine*>& s, int slot, int win[4], uint32_t& err, std::vector<uint32_t>& n_real,
                 std::vector<uint32_t>& arrivals, std::vector<uint32_t>& free_slot) override {
        win[0] = INT_MAX; win[1] = INT_MIN; win[2] = INT_MAX; win[3] = INT_MIN;
        err = 0;
        int64_t waits = 0;
        for (size_t i = 0; i < s.size(); ++i) {
            bool blocked = false;
            const Engine::DDControl c = s[i]->dd_snapshot_read(slot, &blocked);
            waits += blocked ? 1 : 0;
            win[0] = std::min(win[0], c.window[0]);
            win[1] = std::max(win[1], c.window[1]);
            win[2] = std::min(win[2], c.window[2]);
            win[3] = std::max(win[3], c.window[3]);
            err |= c.err;
            n_real[i] = c.n_real;
            arrivals[i] = c.arrivals;
            free_slot[i] = c.free_slot;
        }
        return waits;
    }
    int64_t agree_max(int64_t v) override { return v; }

  private:
    size_t n_;
};

class NcclTransport final : public DDTransport {
  public:
    NcclTransport(ncclComm_t comm, int nranks, int rank, bool own)
        : nccl_(Nccl::get()), comm_(comm), n_(nranks), r_(rank), own_(own) {}
    ~NcclTransport() override {
        if (own_ && comm_) nccl_.comm_destroy(comm_);
    }
    int index(size_t) const override { return r_; }
    int count() const override { return n_; }
    void halo(const std::vector<Engine*>& s, size_t down, size_t up) override {
        const Halo h = halo_of(s[0]);
        nccl_.ok(nccl_.group_start(), "ncclGroupStart");
        if (r_ > 0) {
            nccl_.ok(nccl_.send(h.send_lo, down, ncclChar, r_ - 1, comm_, st), "ncclSend");
            nccl_.ok(nccl_.recv(h.recv_lo, up, ncclChar, r_ - 1, comm_, st), "ncclRecv");
        }
        if (r_ + 1 < n_) {
            nccl_.ok(nccl_.send(h.send_hi, up, ncclChar, r_ + 1, comm_, st), "ncclSend");
            nccl_.ok(nccl_.recv(h.recv_hi, down, ncclChar, r_ + 1, comm_, st), "ncclRecv");
        }
        nccl_.ok(nccl_.group_end(), "ncclGroupEnd");
    }
    void migrate(const std::vector<Engine*>& s) override {
        const Mig m = mig_of(s[0]);
        const size_t pay = static_cast<size_t>(m.cap) * 7 * 16;
        nccl_.ok(nccl_.group_start(), "ncclGroupStart");
        if (r_ > 0) {
            nccl_.ok(nccl_.send(m.counts + 0, 1, ncclUint32, r_ - 1, comm_, st), "ncclSend");
            nccl_.ok(nccl_.recv(m.counts + 2, 1, ncclUint32, r_ - 1, comm_, st), "ncclRecv");
            nccl_.ok(nccl_.send(m.send_lo, pay, ncclChar, r_ - 1, comm_, st), "ncclSend");
            nccl_.ok(nccl_.recv(m.recv_lo, pay, ncclChar, r_ - 1, comm_, st), "ncclRecv");
        }
        if (r_ + 1 < n_) {
            nccl_.ok(nccl_.send(m.counts + 1, 1, ncclUint32, r_ + 1, comm_, st), "ncclSend");
            nccl_.ok(nccl_.recv(m.counts + 3, 1, ncclUint32, r_ + 1, comm_, st), "ncclRecv");
            nccl_.ok(nccl_.send(m.send_hi, pay, ncclChar, r_ + 1, comm_, st), "ncclSend");
            nccl_.ok(nccl_.recv(m.recv_hi, pay, ncclChar, r_ + 1, comm_, st), "ncclRecv");
        }
        nccl_.ok(nccl_.group_end(), "ncclGroupEnd");
    }
    void contact_sums(const std::vector<Engine*>& s) override {
        void *sums, *cnt;
        int ns = 0;
        s[0]->contact_sub_buffers(&sums, &cnt, &ns);
        if (ns == 0 || n_ == 1) return;
        nccl_.ok(nccl_.group_start(), "ncclGroupStart");
        nccl_.ok(nccl_.all_reduce(sums, sums, 6 * ns, ncclFloat64, ncclSum, comm_, st), "ncclAllReduce");
        nccl_.ok(nccl_.all_reduce(cnt, cnt, ns, ncclInt32, ncclSum, comm_, st), "ncclAllReduce");
        nccl_.ok(nccl_.group_end(), "ncclGroupEnd");
    }
    void snapshot(const std::vector<Engine*>& s, int slot) override {
        Engine* e = s[0];
        e->dd_window_async();
        int* w = e->dd_window_device();
        // window and error flags of every rank in one MIN all-reduce: {ylo, -yhi, zlo, -zhi, -err}
        dd_window_to_min_form(w, e->dd_control_device(), st);
        if (n_ > 1) nccl_.ok(nccl_.all_reduce(w, w, 5, ncclInt32, ncclMin, comm_, st), "ncclAllReduce");
        dd_window_from_min_form(w, st);
        e->dd_snapshot_async(slot);
    }
    int64_t read(const std::vector<Engine*>& s, int slot, int win[4], uint32_t& err, std::vector<uint32_t>& n_real,
                 std::vector<uint32_t>& arrivals, std::vector<uint32_t>& free_slot) override {
        bool blocked = false;
        const Engine::DDControl c = s[0]->dd_snapshot_read(slot, &blocked);
        std::memcpy(win, c.window, sizeof(c.window));
        err = c.group_err | c.err;
        n_real[0] = c.n_real;
        arrivals[0] = c.arrivals;
        free_slot[0] = c.free_slot;
        return blocked ? 1 : 0;
    }
    int64_t agree_max(int64_t v) override {
        int64_t* d = nullptr;
        ck(cudaMalloc(&d, sizeof(int64_t)), "cudaMalloc");
        ck(cudaMemcpyAsync(d, &v, sizeof(v), cudaMemcpyHostToDevice, st), "h2d");
        nccl_.ok(nccl_.all_reduce(d, d, 1, ncclInt64, ncclMax, comm_, st), "ncclAllReduce");
        ck(cudaMemcpyAsync(&v, d, sizeof(v), cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "agree");
        cudaFree(d);
        return v;
    }

  private:
    Nccl& nccl_;
    ncclComm_t comm_;
    int n_, r_;
    bool own_;
};

}  // namespace

// ------------------------------------------------------------------ group
std::unique_ptr<DDGroup> DDGroup::local(const std::vector<Engine*>& slabs) {
    if (slabs.empty()) throw std::invalid_argument("dd group: no slabs");
    std::unique_ptr<DDGroup> g(new DDGroup());
    g->slabs_ = slabs;
    g->tr_ = std::make_unique<LocalTransport>(slabs.size());
    // ONE stream for every slab: the device copies order against all their kernels
    g->tr_->st = static_cast<cudaStream_t>(slabs[0]->stream());
    for (Engine* e : slabs) e->set_stream(g->tr_->st);
    int64_t cap = 0;
    for (Engine* e : slabs) cap = std::max(cap, std::max<int64_t>(1024, e->slot_count() / 64));
    for (Engine* e : slabs) e->dd_set_migration_capacity(cap);
    return g;
}

void DDGroup::nccl_unique_id(uint8_t out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    Nccl& n = Nccl::get();
    ncclUniqueId id;
    n.ok(n.get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, 128);
}

std::unique_ptr<DDGroup> DDGroup::nccl(Engine* slab, const uint8_t unique_id[128], int nranks, int rank) {
    Nccl& n = Nccl::get();
    ncclUniqueId id;
    std::memcpy(&id, unique_id, 128);
    ncclComm_t comm = nullptr;
    n.ok(n.comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank");
    std::unique_ptr<DDGroup> g(new DDGroup());
    g->slabs_ = {slab};
    g->tr_ = std::make_unique<NcclTransport>(comm, nranks, rank, true);
    g->tr_->st = static_cast<cudaStream_t>(slab->stream());
    const int64_t cap = g->tr_->agree_max(std::max<int64_t>(1024, slab->slot_count() / 64));
    slab->dd_set_migration_capacity(cap);
    return g;
}

std::unique_ptr<DDGroup> DDGroup::nccl_comm(Engine* slab, void* comm, int nranks, int rank) {
    std::unique_ptr<DDGroup> g(new DDGroup());
    g->slabs_ = {slab};
    g->tr_ = std::make_unique<NcclTransport>(static_cast<ncclComm_t>(comm), nranks, rank, false);
    g->tr_->st = static_cast<cudaStream_t>(slab->stream());
    const int64_t cap = g->tr_->agree_max(std::max<int64_t>(1024, slab->slot_count() / 64));
    slab->dd_set_migration_capacity(cap);
    return g;
}

DDGroup::~DDGroup() = default;

namespace {
void throw_if(uint32_t err) {
    if (!err) return;
    std::string m = "slab DD:";
    if (err & 1u) m += " migration buffer overflow;";
    if (err & 2u) m += " slab capacity exceeded (set_capacity);";
    if (err & 4u) m += " a particle's stencil left the stored planes or the halo window (CFL > 1 cell/substep?);";
    if (err & 8u) m += " a particle left the decomposed grid;";
    throw std::runtime_error(m);
}
}  // namespace

void DDGroup::check() {
    // a fresh snapshot in the slot the next run would read anyway: it is overwritten before use
    const int slot = static_cast<int>(stats_.runs & 1);
    tr_->snapshot(slabs_, slot);
    int w[4];
    uint32_t err = 0;
    std::vector<uint32_t> n_real(slabs_.size()), arrivals(slabs_.size()), free_slot(slabs_.size());
    tr_->read(slabs_, slot, w, err, n_real, arrivals, free_slot);
    for (size_t i = 0; i < slabs_.size(); ++i) slabs_[i]->dd_note_count(n_real[i]);
    throw_if(err);
}

void DDGroup::run(const DDRunOptions& o) {
    if (o.n_sub <= 0) return;
    if (o.dt <= 0) throw std::invalid_argument("dd run: dt must be positive");
    std::vector<Engine*>& S = slabs_;
    DDTransport& T = *tr_;
    const size_t k = S.size();
    const int margin = S[0]->dd_halo_planes(0, true);  // acc: low ghosts = M planes
    const int every = o.migrate_every > 0 ? o.migrate_every : std::max(1, margin);
    if (every > margin) throw std::invalid_argument("dd run: migrate_every exceeds the slab margin");

    // ---- window, error flags and counts, pipelined: run r reads the snapshot taken at the
    // end of run r - 2 (slot r % 2), long complete while the device works on run r - 1, so
    // the host does not wait; the window is then widened by the drift of runs r - 1 and r.
    // The first two runs snapshot the current state and wait for it.
    int w[4];
    uint32_t err = 0;
    std::vector<uint32_t> n_real(k), arrivals(k), free_slot(k);
    const int slot = static_cast<int>(stats_.runs & 1);
    int drift = o.n_sub;
    const bool fresh = stats_.runs < 2;
    if (fresh) T.snapshot(S, slot);
    else drift += last_n_sub_;
    const int64_t waited = T.read(S, slot, w, err, n_real, arrivals, free_slot);
    if (fresh) stats_.host_syncs += static_cast<int64_t>(k);  // drained the queue just issued
    else stats_.host_waits += waited;                         // the device was > 1 run behind
    throw_if(err);
    for (size_t i = 0; i < k; ++i) {
        S[i]->dd_note_count(n_real[i]);
        // re-bin after many arrivals (the appended groups are not spatially compact), or when
        // the appended groups -- each migration opens fresh ones -- used a quarter of the spare
        // slots (the snapshot is two runs old: the rest covers those runs)
        const int64_t spare = S[i]->slot_count() - static_cast<int64_t>(n_real[i]);
        const int64_t used = static_cast<int64_t>(free_slot[i]) - static_cast<int64_t>(n_real[i]);
        if (arrivals[i] > 0 && (static_cast<int64_t>(arrivals[i]) * 64 > static_cast<int64_t>(n_real[i]) ||
                                used * 4 > spare)) {
            S[i]->bin();
            ++stats_.rebins;
        }
    }
    if (w[0] > w[1]) w[0] = w[1] = w[2] = w[3] = 0;  // no active particle anywhere
    const int pad = drift + 1;  // one cell per substep (CFL), checked on the device
    for (Engine* e : S) e->dd_set_window(w[0] - pad, w[1] + 1 + pad, w[2] - pad, w[3] + 1 + pad);
    int y0, ny, z0, nz;
    S[0]->dd_plane_window(&y0, &ny, &z0, &nz);
    const size_t plane = static_cast<size_t>(ny) * nz * 16;
    const size_t acc_down = plane * margin, acc_up = plane * (2 + margin);  // ghost sums
    const size_t vel_down = acc_up, vel_up = acc_down;                      // owned velocities

    const bool fuse = o.fuse && S[0]->fuse_ok();
    bool fused_in = false;
    for (int s = 0; s < o.n_sub; ++s) {
        if (!fused_in)
            for (Engine* e : S) e->p2g(true, o.dt, false);
        for (Engine* e : S) e->dd_pack_acc();
        T.halo(S, acc_down, acc_up);
        for (Engine* e : S) {
            e->dd_unpack_acc();
            if (fused_in) e->collect_deferred(0, o.dt, o.g, o.free_bodies);  // + free bodies of s - 1
            else e->collect_bricks();
            e->grid_update(0, o.dt, o.g, true, o.contact, o.bc);
        }
        if (o.free_bodies) T.contact_sums(S);
        for (Engine* e : S) e->dd_pack_vel();
        T.halo(S, vel_down, vel_up);
        stats_.exchanges += 2;
        const bool migrate_now = (s + 1) % every == 0 && T.count() > 1;
        const bool fuse_now = fuse && s + 1 < o.n_sub && !migrate_now;
        for (Engine* e : S) {
            e->dd_unpack_vel();
            if (fuse_now) {
                e->g2p2g(0, o.dt, false, o.g, o.free_bodies, false, o.pushout, o.deactivate);
            } else {
                e->g2p_mls(0, o.dt, o.pushout, o.deactivate);
                if (o.free_bodies) e->free_bodies(0, o.dt, o.g, true, true);
            }
        }
        if (migrate_now) {
            for (size_t i = 0; i < k; ++i) {
                const int gi = T.index(i);
                S[i]->dd_migrate_pack_async(gi > 0, gi + 1 < T.count());
            }
            T.migrate(S);
            for (Engine* e : S) e->dd_migrate_unpack_async();
            ++stats_.exchanges;
        }
        if (fuse_now) ++stats_.fused;
        fused_in = fuse_now;
        ++stats_.substeps;
    }
    // the snapshot run r + 2 reads (the window from here on, with the error flags)
    T.snapshot(S, slot);
    last_n_sub_ = o.n_sub;
    ++stats_.runs;
}

}  // namespace mpmb
