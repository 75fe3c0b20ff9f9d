// dd_driver.h — device-resident slab domain decomposition.
//
// One DDGroup advances the slabs of a domain decomposition along x.  Per substep it enqueues
// (scene.hpp:176-249 order, MLS):
//   P2G (or the P2G half of the fused kernel of the previous substep) -> ghost sums out ->
//   exchange -> ghost sums in -> brick collect -> grid update + contact -> [all-reduce of
//   the per-shape contact sums when free bodies exist] -> owned velocities out -> exchange ->
//   ghost velocities in -> G2P (fused with the next P2G unless a migration falls between)
//   -> free bodies -> every `migrate_every` substeps: migration (pack, exchange of counts +
//   fixed-capacity payloads, device-side append).
// Nothing in that loop waits for the host: counts stay on the device, the halo y/z window is
// set once per run from the particles' reach (widened by one cell per substep, CFL) and
// checked on the device.  Each run reads one control snapshot per slab (window, error flags,
// particle count), taken at the end of the run before last: in steady state the host never
// drains the stream (DDStats::host_syncs counts the reads that did: the first two runs).
//
// Transports: LOCAL (every slab in this process on one device; device copies -- the 1-GPU
// emulation of the ranks, which never waits on another kernel) and NCCL (one slab per
// process; ncclSend / ncclRecv inside ncclGroupStart / End and ncclAllReduce, all on the
// slab's stream).  NCCL is loaded at run time (dlopen libnccl.so.2: the copy torch already
// loaded, else the system one), so the library has no link-time dependency on it.
#pragma once
#include <cstdint>
#include <memory>
#include <vector>

#include "engine.h"

namespace mpmb {

struct DDRunOptions {
    int n_sub = 1;
    float dt = 0.f;
    float g[3] = {0.f, 0.f, 0.f};
    bool contact = true;
    int bc = 0;
    bool pushout = true;
    bool deactivate = true;
    bool free_bodies = false;  // all-reduce contact sums each substep, integrate on every slab
    int migrate_every = 0;     // 0: the slab margin
    bool fuse = true;          // G2P(s) + P2G(s+1) in one kernel where no migration intervenes
};

struct DDStats {
    int64_t runs = 0, substeps = 0;
    int64_t host_syncs = 0;     // snapshot reads that drained the stream (the first two runs)
    int64_t host_waits = 0;     // later reads that waited: the device was > 1 run behind the host
    int64_t exchanges = 0;      // halo / migration exchange rounds
    int64_t fused = 0;          // substeps whose G2P ran fused with the next P2G
    int64_t rebins = 0;
};

class DDTransport;

class DDGroup {
  public:
    // local group: slabs ordered along x, all on this process's device
    static std::unique_ptr<DDGroup> local(const std::vector<Engine*>& slabs);
    // NCCL: this process's slab, rank `rank` of `nranks` in the communicator created from
    // `unique_id` (ncclGetUniqueId on one rank, shared by the caller) or given as `comm`
    static std::unique_ptr<DDGroup> nccl(Engine* slab, const uint8_t unique_id[128], int nranks, int rank);
    static std::unique_ptr<DDGroup> nccl_comm(Engine* slab, void* comm, int nranks, int rank);
    static void nccl_unique_id(uint8_t out[128]);
    ~DDGroup();

    void run(const DDRunOptions& o);
    // wait for everything enqueued, then fail with the reason if a device check tripped
    void check();
    const DDStats& stats() const { return stats_; }

  private:
    DDGroup() = default;
    std::vector<Engine*> slabs_;
    std::unique_ptr<DDTransport> tr_;
    int last_n_sub_ = 0;   // substeps of the previous run (the pipelined window's drift)
    DDStats stats_;
};

}  // namespace mpmb
