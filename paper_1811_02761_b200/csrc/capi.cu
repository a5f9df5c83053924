// extern "C" boundary (include/g2/capi.h): exceptions -> status codes, plus the
// NCCL all-gather exchange for sharded multi-GPU steps.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include <memory>
#include <string>

#include "../../include/g2/capi.h"
#include "engine.cuh"
#include "snapshot.hpp"

struct g2_engine {
    std::unique_ptr<g2::Engine> e;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return G2_OK;
    } catch (const g2::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const g2::SnapshotError& e) {  // the reference's data_error
        g_err = e.what();
        return G2_DATA_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return G2_INTERNAL;
    }
}

g2::GravParamsH to_h(const g2_grav_params* p) {
    g2::GravParamsH h;
    if (p) h.G = p->G, h.eps = p->eps, h.dacc = p->dacc;
    return h;
}
g2::EngineConfigH to_h(const g2_engine_config* c) {
    g2::EngineConfigH h;
    if (c) {
        h.leaf_cap = c->leaf_cap, h.group_size = c->group_size, h.list_capacity = c->list_capacity;
        h.frontier_cap = c->frontier_cap, h.count_ops = c->count_ops != 0, h.bootstrap_theta = c->bootstrap_theta;
        h.bootstrap_direct_limit = c->bootstrap_direct_limit, h.threads = c->threads;
    }
    return h;
}
g2::StepSchemeH to_h(const g2_step_scheme* s) {
    g2::StepSchemeH h;
    if (s) h.eta = s->eta, h.dt_max = s->dt_max, h.adaptive = s->adaptive != 0, h.fixed_level = s->fixed_level;
    return h;
}
g2::TunerConfigH to_h(const g2_tuner_config* t) {
    g2::TunerConfigH h;
    if (t) h.min_interval = t->min_interval, h.max_interval = t->max_interval, h.initial_interval = t->initial_interval;
    return h;
}
void put(const g2::EventsH& e, g2_events* o) {
    if (o) o->interactions = e.interactions, o->mac_evals = e.mac_evals, o->list_pushes = e.list_pushes;
}

// ---- NCCL, loaded lazily so the library has no hard dependency on it --------------
struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
    Nccl() {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        get_unique_id = reinterpret_cast<decltype(get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        comm_init_rank = reinterpret_cast<decltype(comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        all_gather = reinterpret_cast<decltype(all_gather)>(dlsym(h, "ncclAllGather"));
        all_reduce = reinterpret_cast<decltype(all_reduce)>(dlsym(h, "ncclAllReduce"));
        comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        error_string = reinterpret_cast<decltype(error_string)>(dlsym(h, "ncclGetErrorString"));
        ok = get_unique_id && comm_init_rank && all_gather && all_reduce && comm_destroy && error_string;
    }
};
Nccl& nccl() {
    static Nccl n;
    if (!n.ok) throw g2::Error(G2_INTERNAL, "NCCL (libnccl.so.2) not loadable");
    return n;
}
#define G2_NCCL(expr)                                                                                \
    do {                                                                                             \
        ncclResult_t _r = (expr);                                                                    \
        if (_r != ncclSuccess) throw g2::Error(G2_INTERNAL, std::string("NCCL: ") + nccl().error_string(_r)); \
    } while (0)

__global__ void unpack_kernel(const float4* __restrict__ gathered, float4* __restrict__ accum,
                              const uint32_t* n_active, uint32_t gs, uint32_t world, uint32_t per_rank) {
    const uint32_t na = *n_active;
    const uint32_t ng = (na + gs - 1) / gs;
    for (uint32_t r = 0; r < world; ++r) {
        uint32_t lo, hi;
        g2::equal_shard(ng, int(r), int(world), lo, hi);
        lo *= gs, hi = min(hi * gs, na);
        for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; lo + j < hi; j += gridDim.x * blockDim.x)
            accum[lo + j] = gathered[size_t(r) * per_rank + j];
    }
}

// Sharded walk exchange: rank r owns accumulator slots
// [lo_r*gs, hi_r*gs); each rank contributes a fixed-size window so the
// gather has equal counts, then every rank scatters all windows back.  The
// transport is one ncclAllGather (one process per GPU) or device copies
// between Simulations of one process (LocalExchange).
struct ShardExchange : g2::Exchange {
    int world = 1;
    g2::DBuf<float4> gathered;
    static size_t window(const g2::Simulation& sim, int world) { return g2::shard_window(sim.n(), sim.group_size(), world); }
    g2::DBuf<float4> gathered_slices;  // [world][walk_slice_slots()] every rank's slice region
    void prepare(g2::Simulation& sim) {  // before the first step: the accumulator must not move later
        sim.engine().reserve_accum(std::max(2 * sim.n() + 64 * sim.group_size(),
                                            g2::walk_slice_base(sim.n()) + g2::walk_slice_slots()));
        gathered.reserve(window(sim, world) * world);
        gathered_slices.reserve(g2::walk_slice_slots() * world);
    }
    void slice_source(g2::Simulation&, const float4*& src, size_t& stride) override {
        src = gathered_slices.p;
        stride = g2::walk_slice_slots();
    }
    virtual void transport(g2::Simulation& sim, const float4* send, size_t per_rank) = 0;
    void allgather_acc(g2::Simulation& sim) override {
        auto& eng = sim.engine();
        const size_t per_rank = window(sim, world);
        transport(sim, eng.accum() + size_t(sim.shard_lo()) * sim.group_size(), per_rank);
        G2_COUNT(1), unpack_kernel<<<256, 256, 0, eng.stream()>>>(gathered.p, eng.accum(), sim.n_active_dev(),
                                                                 uint32_t(sim.group_size()), uint32_t(world),
                                                                 uint32_t(per_rank));
        G2_CUDA(cudaGetLastError());
    }
};

struct NcclExchange final : ShardExchange {
    ncclComm_t comm = nullptr;
    ~NcclExchange() override {
        if (comm) nccl().comm_destroy(comm);
    }
    void transport(g2::Simulation& sim, const float4* send, size_t per_rank) override {
        G2_NCCL(nccl().all_gather(send, gathered.p, per_rank * 4, ncclFloat32, comm, sim.engine().stream()));
        G2_NCCL(nccl().all_gather(sim.engine().slice_region(), gathered_slices.p, g2::walk_slice_slots() * 4,
                                  ncclFloat32, comm, sim.engine().stream()));
    }
    g2::DBuf<double> tbuf;
    void agree_times(g2::Simulation& sim, double& walk, double& build, bool sum_walk) override {
        cudaStream_t s = sim.engine().stream();
        tbuf.reserve(2);
        double h[2] = {walk, build};
        G2_CUDA(cudaMemcpyAsync(tbuf.p, h, sizeof h, cudaMemcpyHostToDevice, s));
        G2_NCCL(nccl().all_reduce(tbuf.p, tbuf.p, 1, ncclFloat64, sum_walk ? ncclSum : ncclMax, comm, s));
        G2_NCCL(nccl().all_reduce(tbuf.p + 1, tbuf.p + 1, 1, ncclFloat64, ncclMax, comm, s));
        G2_CUDA(cudaMemcpyAsync(h, tbuf.p, sizeof h, cudaMemcpyDeviceToHost, s));
        G2_CUDA(cudaStreamSynchronize(s));
        walk = h[0], build = h[1];
    }
};

// In-process mesh: several Simulations (one host thread each, any devices)
// exchange through device-to-device copies between two barriers.
struct LocalMesh {
    std::vector<g2::Simulation*> sims;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t phase = 0;
    std::vector<double> tw, tb;
    void agree(int rank, double& walk, double& build, bool sum_walk) {
        {
            std::lock_guard<std::mutex> lk(m);
            if (tw.size() != sims.size()) tw.assign(sims.size(), 0.0), tb.assign(sims.size(), 0.0);
            tw[rank] = walk, tb[rank] = build;
        }
        barrier();
        double w = sum_walk ? 0.0 : tw[0], b = tb[0];
        for (size_t q = 0; q < sims.size(); ++q) {  // fixed rank order: identical on every rank
            w = sum_walk ? w + tw[q] : std::max(w, tw[q]);
            b = std::max(b, tb[q]);
        }
        barrier();  // nobody overwrites its slot before everyone has read
        walk = w, build = b;
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t ph = phase;
        if (++arrived == int(sims.size())) {
            arrived = 0;
            ++phase;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return phase != ph; });
        }
    }
};

struct LocalExchange final : ShardExchange {
    std::shared_ptr<LocalMesh> mesh;
    void transport(g2::Simulation& sim, const float4*, size_t per_rank) override {
        cudaStream_t s = sim.engine().stream();
        G2_CUDA(cudaStreamSynchronize(s));  // own walk done
        mesh->barrier();                    // every rank's walk done
        for (int q = 0; q < world; ++q) {
            g2::Simulation* o = mesh->sims[q];
            G2_CUDA(cudaMemcpyAsync(gathered.p + size_t(q) * per_rank,
                                    o->engine().accum() + size_t(o->shard_lo()) * o->group_size(),
                                    per_rank * sizeof(float4), cudaMemcpyDefault, s));
            G2_CUDA(cudaMemcpyAsync(gathered_slices.p + size_t(q) * g2::walk_slice_slots(), o->engine().slice_region(),
                                    g2::walk_slice_slots() * sizeof(float4), cudaMemcpyDefault, s));
        }
        G2_CUDA(cudaStreamSynchronize(s));
        mesh->barrier();  // nobody reuses its accumulator before everyone copied
    }
    void agree_times(g2::Simulation& sim, double& walk, double& build, bool sum_walk) override {
        mesh->agree(sim.rank(), walk, build, sum_walk);
    }
};

// ---- fused peer exchange (SURVEY §8e "fused-collective option") -----------------
// No collective at all: the walk kernel itself stores every finished group's
// accumulators into each peer rank's accumulator buffer (NVLink P2P stores through
// IPC-mapped pointers, or plain device pointers for an in-process mesh), overlapped
// with the rest of the walk.  Then one signal/wait pair on device flags (release /
// acquire at system scope) orders those stores before the peers' correct.
// Accumulators are double-buffered by step parity: a rank can only start pushing
// step k + 2 after every rank finished walking step k + 1, hence after every rank's
// correct of step k read the buffer; the zero pass touches only the own shard.
struct PeerFlags {
    uint64_t* f[g2::kMaxPeers];
};

__global__ void peer_signal_kernel(PeerFlags peers, int world, int self, uint64_t epoch) {
    const int q = threadIdx.x;
    __threadfence_system();
    if (q < world)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peers.f[q] + self), "l"(epoch) : "memory");
}
// the tuner inputs of this rank into slot [self] of every rank's times array, then the epoch flag
struct PeerTimes {
    double* t[g2::kMaxPeers];
};
__global__ void peer_times_kernel(PeerTimes times, PeerFlags peers, int world, int self, uint64_t epoch, double walk,
                                  double build) {
    const int q = threadIdx.x;
    if (q < world) times.t[q][2 * self] = walk, times.t[q][2 * self + 1] = build;
    __threadfence_system();
    __syncwarp();
    if (q < world)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(peers.f[q] + self), "l"(epoch) : "memory");
}

// bounded: a rank that never arrives (crashed, hung, or a mismatched step count) turns into a
// ResourceError at the end of the step instead of a GPU spinning forever
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__global__ void peer_wait_kernel(const uint64_t* flags, int world, uint64_t epoch, uint64_t timeout_ns,
                                 g2::DevFlags* df) {
    const int q = threadIdx.x;
    if (q < world) {
        const uint64_t t0 = global_ns();
        while (true) {
            uint64_t v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + q) : "memory");
            if (v >= epoch) break;
            if (global_ns() - t0 > timeout_ns) {
                atomicExch(&df->peer_timeout, 1);
                break;
            }
            __nanosleep(200);
        }
    }
    __syncwarp();
    __threadfence_system();
}

// the device-side exchange barrier's patience: G2_PEER_TIMEOUT_S seconds (default 120; ranks meet
// at it once per step, so only a dead or diverged peer comes near it)
uint64_t peer_timeout_ns() {
    static const uint64_t ns = [] {
        const char* e = std::getenv("G2_PEER_TIMEOUT_S");
        const double sec = e ? std::atof(e) : 120.0;
        return uint64_t((sec > 0.0 ? sec : 120.0) * 1e9);
    }();
    return ns;
}

struct PeerExchange final : g2::Exchange {
    int world = 1, self = 0;
    uint64_t epoch = 0;
    float4* buf[2] = {};                        // own accumulators (exported)
    uint64_t* flags = nullptr;                  // own arrival flags [kMaxPeers] (exported)
    uint32_t* cost[2] = {};                     // own per-group cost arrays (exported)
    double* times = nullptr;                    // own tuner-input slots [kMaxPeers][2] (exported)
    uint64_t* tflags = nullptr;                 // own arrival flags of the tuner exchange (exported)
    uint64_t tepoch = 0;
    double* ptimes[g2::kMaxPeers] = {};
    uint64_t* ptflags[g2::kMaxPeers] = {};
    double* htimes = nullptr;                   // pinned read-back
    uint32_t* ngrec = nullptr;                  // [2] group counts behind cost[0], cost[1] (local)
    float4* pbuf[g2::kMaxPeers][2] = {};        // every rank's accumulators as seen from here
    uint64_t* pflags[g2::kMaxPeers] = {};
    uint32_t* pcost[g2::kMaxPeers][2] = {};
    std::vector<void*> opened;                  // IPC mappings to close
    int device = 0;
    // In-process mesh (all ranks in one context): the ranks meet at a host barrier after their walks
    // instead of device flags -- a device-side spin would sit at the head of shared copy/launch
    // queues and starve the ranks it waits for.
    std::shared_ptr<LocalMesh> mesh;

    void alloc(g2::Simulation& sim, int w, int r) {
        world = w, self = r;
        device = sim.engine().device();
        G2_CUDA(cudaSetDevice(device));
        const size_t slots = g2::walk_slice_base(sim.n()) + g2::walk_slice_slots();  // groups, then slices
        for (auto& b : buf) {
            G2_CUDA(cudaMalloc(&b, slots * sizeof(float4)));
            G2_CUDA(cudaMemset(b, 0, slots * sizeof(float4)));
        }
        G2_CUDA(cudaMalloc(&flags, g2::kMaxPeers * sizeof(uint64_t)));
        G2_CUDA(cudaMemset(flags, 0, g2::kMaxPeers * sizeof(uint64_t)));
        const size_t groups = sim.n() / sim.group_size() + 64;
        for (auto& c : cost) G2_CUDA(cudaMalloc(&c, groups * sizeof(uint32_t)));
        G2_CUDA(cudaMalloc(&ngrec, 2 * sizeof(uint32_t)));
        G2_CUDA(cudaMemset(ngrec, 0xff, 2 * sizeof(uint32_t)));  // no history: equal shards first
        G2_CUDA(cudaMalloc(&times, 2 * g2::kMaxPeers * sizeof(double)));
        G2_CUDA(cudaMalloc(&tflags, g2::kMaxPeers * sizeof(uint64_t)));
        G2_CUDA(cudaMemset(tflags, 0, g2::kMaxPeers * sizeof(uint64_t)));
        G2_CUDA(cudaMallocHost(&htimes, 2 * g2::kMaxPeers * sizeof(double)));
        pbuf[self][0] = buf[0], pbuf[self][1] = buf[1], pflags[self] = flags;
        pcost[self][0] = cost[0], pcost[self][1] = cost[1];
        ptimes[self] = times, ptflags[self] = tflags;
    }
    ~PeerExchange() override {
        for (void* p : opened) cudaIpcCloseMemHandle(p);
        for (auto& b : buf)
            if (b) cudaFree(b);
        for (auto& c : cost)
            if (c) cudaFree(c);
        if (flags) cudaFree(flags);
        if (ngrec) cudaFree(ngrec);
        if (times) cudaFree(times);
        if (tflags) cudaFree(tflags);
        if (htimes) cudaFreeHost(htimes);
    }
    bool device_shards() const override { return true; }
    void before_walk(g2::Simulation& sim) override {
        const int par = int(epoch & 1);
        float4* peers[g2::kMaxPeers] = {};
        uint32_t* costs[g2::kMaxPeers] = {};
        for (int q = 0; q < world; ++q) peers[q] = pbuf[q][par], costs[q] = pcost[q][par];
        static const bool equal = std::getenv("G2_EQUAL_SHARDS") != nullptr;  // development A/B
        sim.engine().set_peer_push(world, self, buf[par], peers, equal ? nullptr : costs, cost[par ^ 1],
                                   ngrec + (par ^ 1), ngrec + par);
    }
    void allgather_acc(g2::Simulation& sim) override {
        ++epoch;
        cudaStream_t s = sim.engine().stream();
        if (mesh) {
            G2_CUDA(cudaStreamSynchronize(s));  // own walk (and its pushes) complete
            mesh->barrier();                    // every rank's walk complete
            return;
        }
        PeerFlags pf{};
        for (int q = 0; q < world; ++q) pf.f[q] = pflags[q];
        G2_COUNT(1), peer_signal_kernel<<<1, 32, 0, s>>>(pf, world, self, epoch);
        G2_COUNT(1), peer_wait_kernel<<<1, 32, 0, s>>>(flags, world, epoch, peer_timeout_ns(),
                                                        sim.engine().dev_flags());
        G2_CUDA(cudaGetLastError());
    }
    void agree_times(g2::Simulation& sim, double& walk, double& build, bool sum_walk) override {
        if (mesh) {
            mesh->agree(self, walk, build, sum_walk);
            return;
        }
        cudaStream_t s = sim.engine().stream();
        ++tepoch;
        PeerTimes pt{};
        PeerFlags pf{};
        for (int q = 0; q < world; ++q) pt.t[q] = ptimes[q], pf.f[q] = ptflags[q];
        G2_COUNT(1), peer_times_kernel<<<1, 32, 0, s>>>(pt, pf, world, self, tepoch, walk, build);
        G2_COUNT(1), peer_wait_kernel<<<1, 32, 0, s>>>(tflags, world, tepoch, peer_timeout_ns(),
                                                        sim.engine().dev_flags());
        G2_CUDA(cudaGetLastError());
        G2_CUDA(cudaMemcpyAsync(htimes, times, 2 * world * sizeof(double), cudaMemcpyDeviceToHost, s));
        G2_CUDA(cudaStreamSynchronize(s));
        sim.engine().check_flags();  // a peer that never arrived: ResourceError now, not next step
        double w = sum_walk ? 0.0 : htimes[0], b = htimes[1];
        for (int q = 0; q < world; ++q) {
            w = sum_walk ? w + htimes[2 * q] : std::max(w, htimes[2 * q]);
            b = std::max(b, htimes[2 * q + 1]);
        }
        walk = w, build = b;
    }
};
constexpr int kP2PHandles = 7;
constexpr size_t kP2PHandleBytes = kP2PHandles * sizeof(cudaIpcMemHandle_t);

}  // namespace

struct g2_sim {
    std::unique_ptr<g2::Simulation> s;
    std::unique_ptr<g2::Exchange> ex;
    std::unique_ptr<PeerExchange> pending;  // exported, peers not opened yet
};


extern "C" {

const char* g2_last_error(void) { return g_err.c_str(); }

void g2_default_params(g2_grav_params* p) {
    g2::GravParamsH h;
    p->G = h.G, p->eps = h.eps, p->dacc = h.dacc;
}
void g2_default_engine_config(g2_engine_config* c) {
    g2::EngineConfigH h;
    c->leaf_cap = h.leaf_cap, c->group_size = h.group_size, c->list_capacity = h.list_capacity;
    c->frontier_cap = h.frontier_cap, c->count_ops = h.count_ops, c->bootstrap_theta = h.bootstrap_theta;
    c->bootstrap_direct_limit = h.bootstrap_direct_limit, c->threads = h.threads;
}
void g2_default_step_scheme(g2_step_scheme* s) {
    g2::StepSchemeH h;
    s->eta = h.eta, s->dt_max = h.dt_max, s->adaptive = h.adaptive, s->fixed_level = h.fixed_level;
}
void g2_default_tuner_config(g2_tuner_config* t) {
    g2::TunerConfigH h;
    t->min_interval = h.min_interval, t->max_interval = h.max_interval, t->initial_interval = h.initial_interval;
}

int g2_engine_create(const g2_grav_params* p, const g2_engine_config* c, int device, g2_engine** out) {
    return guarded([&] {
        auto* h = new g2_engine;
        try {
            h->e = std::make_unique<g2::Engine>(to_h(p), to_h(c), device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}
void g2_engine_destroy(g2_engine* e) { delete e; }
int g2_engine_build(g2_engine* e, size_t n, const double* mass, const double* pos) {
    return guarded([&] { e->e->build(n, mass, pos, true); });
}
int g2_engine_build_structure(g2_engine* e, size_t n, const double* mass, const double* pos) {
    return guarded([&] { e->e->build(n, mass, pos, false); });
}
int g2_engine_refresh(g2_engine* e, size_t n, const double* mass, const double* pos) {
    return guarded([&] { e->e->refresh(n, mass, pos); });
}
int g2_engine_has_tree(const g2_engine* e) { return e->e->has_tree() ? 1 : 0; }
int g2_engine_evaluate(g2_engine* e, size_t n, const double* mass, const double* pos, const double* acc_old_mag,
                       size_t n_targets, const uint32_t* targets, double* acc_inout, double* pot_out,
                       g2_events* events) {
    return guarded([&] {
        put(e->e->evaluate(n, mass, pos, acc_old_mag, n_targets, targets, acc_inout, pot_out), events);
    });
}
int g2_engine_bootstrap(g2_engine* e, size_t n, const double* mass, const double* pos, double* acc_out,
                        double* acc_old_mag_inout, g2_events* events) {
    return guarded([&] { put(e->e->bootstrap(n, mass, pos, acc_out, acc_old_mag_inout), events); });
}
int g2_engine_tree_size(const g2_engine* e, size_t* n, size_t* ncells) {
    return guarded([&] {
        if (n) *n = e->e->n();
        if (ncells) *ncells = e->e->ncells();
    });
}
int g2_sim_tree_size(g2_sim* s, size_t* n, size_t* ncells) {
    return guarded([&] {
        if (n) *n = s->s->engine().n();
        if (ncells) *ncells = s->s->engine().ncells();
    });
}
int g2_sim_get_tree(g2_sim* s, double* bbox4, uint64_t* keys, uint32_t* perm, uint32_t* rank, uint32_t* cells4,
                    uint8_t* depth, double* nodes5) {
    return guarded([&] { s->s->engine().get_tree(bbox4, keys, perm, rank, cells4, depth, nodes5); });
}
int g2_engine_get_tree(g2_engine* e, double* bbox4, uint64_t* keys, uint32_t* perm, uint32_t* rank,
                       uint32_t* cells4, uint8_t* depth, double* nodes5) {
    return guarded([&] { e->e->get_tree(bbox4, keys, perm, rank, cells4, depth, nodes5); });
}
int g2_engine_set_params(g2_engine* e, const g2_grav_params* p) {
    return guarded([&] {
        if (!(p->dacc > 0.0)) throw g2::Error(G2_DATA_ERROR, "GravityEngine: dacc must be positive");
        if (p->eps < 0.0) throw g2::Error(G2_DATA_ERROR, "GravityEngine: eps must be non-negative");
        e->e->params() = to_h(p);
    });
}

int g2_direct_sum(size_t n, const double* mass, const double* pos, double G, double eps, int device,
                  double* acc_out) {
    return guarded([&] {
        g2::GravParamsH p;
        p.G = G, p.eps = eps;
        g2::EngineConfigH c;
        c.bootstrap_direct_limit = ~size_t(0);
        g2::Engine eng(p, c, device);
        std::unique_ptr<double[]> amag(new double[n ? n : 1]());
        eng.bootstrap(n, mass, pos, acc_out, amag.get());
    });
}

int g2_direct_sum_targets(size_t n, const double* mass, const double* pos, double G, double eps, size_t n_targets,
                          const uint32_t* targets, int device, double* acc_out) {
    return guarded([&] {
        G2_CUDA(cudaSetDevice(device));
        for (size_t j = 0; j < n_targets; ++j)
            if (targets[j] >= n) throw g2::Error(G2_DATA_ERROR, "direct_sum_targets: target out of range");
        g2::DBuf<double> p3, m, out;
        g2::DBuf<double4> xyzm;
        g2::DBuf<uint32_t> tg;
        p3.reserve(3 * n + 3), m.reserve(n + 1), xyzm.reserve(n + 1), tg.reserve(n_targets + 1);
        out.reserve(3 * n_targets + 3);
        G2_CUDA(cudaMemcpy(p3.p, pos, 3 * n * 8, cudaMemcpyHostToDevice));
        G2_CUDA(cudaMemcpy(m.p, mass, n * 8, cudaMemcpyHostToDevice));
        G2_CUDA(cudaMemcpy(tg.p, targets, n_targets * 4, cudaMemcpyHostToDevice));
        g2::launch_pack_identity(p3.p, m.p, xyzm.p, n, nullptr);
        g2::launch_direct_targets(xyzm.p, n, tg.p, n_targets, G, eps, out.p, nullptr);
        G2_CUDA(cudaMemcpy(acc_out, out.p, 3 * n_targets * 8, cudaMemcpyDeviceToHost));
    });
}

int g2_block_level(size_t n, const double* acc_mag, const g2_step_scheme* s, double eps, int device, int* levels) {
    return guarded([&] {
        G2_CUDA(cudaSetDevice(device));
        g2::DBuf<double> a;
        g2::DBuf<int> l;
        a.reserve(n ? n : 1), l.reserve(n ? n : 1);
        G2_CUDA(cudaMemcpy(a.p, acc_mag, n * 8, cudaMemcpyHostToDevice));
        const g2::StepSchemeH h = to_h(s);
        g2::launch_block_levels(a.p, n, g2::SchemeDev{h.eta, h.dt_max, eps, h.adaptive ? 1 : 0, h.fixed_level}, l.p,
                                nullptr);
        G2_CUDA(cudaMemcpy(levels, l.p, n * sizeof(int), cudaMemcpyDeviceToHost));
    });
}

int g2_compute_diagnostics(size_t n, const double* mass, const double* pos, const double* vel,
                           const double* acc_old_mag, const g2_grav_params* p, int device, g2_diagnostics* out) {
    return guarded([&] {
        *out = g2_diagnostics{};
        if (n == 0) return;
        G2_CUDA(cudaSetDevice(device));
        constexpr size_t kDirectPotentialLimit = size_t(1) << 17;  // diagnostics.hpp:26
        const bool direct = n <= kDirectPotentialLimit;
        g2::DBuf<double> p3, m, v3;
        g2::DBuf<double4> xyzm;
        g2::DBuf<g2::DevFlags> flags;
        p3.reserve(3 * n), m.reserve(n), v3.reserve(3 * n), xyzm.reserve(n), flags.reserve(1);
        G2_CUDA(cudaMemset(flags.p, 0, sizeof(g2::DevFlags)));
        G2_CUDA(cudaMemcpy(p3.p, pos, 3 * n * 8, cudaMemcpyHostToDevice));
        G2_CUDA(cudaMemcpy(m.p, mass, n * 8, cudaMemcpyHostToDevice));
        G2_CUDA(cudaMemcpy(v3.p, vel, 3 * n * 8, cudaMemcpyHostToDevice));
        g2::launch_pack_identity(p3.p, m.p, xyzm.p, n, nullptr);
        double km[4], w = 0.0;
        g2::diagnostics_device(m.p, v3.p, xyzm.p, n, p->G, p->eps, direct, km, &w, flags.p, nullptr);
        g2::DevFlags f;
        G2_CUDA(cudaMemcpy(&f, flags.p, sizeof f, cudaMemcpyDeviceToHost));
        if (f.singularity) throw g2::Error(G2_SINGULARITY, "direct_potential_energy: coincident particles");
        if (!direct) {
            // the reference's high-accuracy tree potential (diagnostics.cpp:19-31)
            g2::GravParamsH tp;
            tp.G = p->G, tp.eps = p->eps, tp.dacc = 0x1.0p-20;
            g2::EngineConfigH c;
            c.count_ops = false;
            g2::Engine eng(tp, c, device);
            eng.build(n, mass, pos, true);
            std::vector<double> am(acc_old_mag ? acc_old_mag : nullptr, acc_old_mag ? acc_old_mag + n : nullptr);
            if (!acc_old_mag) am.assign(n, 0.0);
            std::vector<double> acc(3 * n), pot(n, 0.0);
            eng.evaluate(n, mass, pos, am.data(), 0, nullptr, acc.data(), pot.data());
            for (size_t i = 0; i < n; ++i) w += 0.5 * mass[i] * pot[i];
        }
        out->kinetic = km[0];
        out->momentum[0] = km[1], out->momentum[1] = km[2], out->momentum[2] = km[3];
        out->potential = w;
        out->total = out->kinetic + out->potential;
        out->virial_ratio = out->potential != 0.0 ? -2.0 * out->kinetic / out->potential : 0.0;
    });
}

int g2_snapshot_info(const char* path, size_t* n, double* time, double* G, double* eps) {
    return guarded([&] {
        const g2::SnapshotHeader h = g2::read_snapshot_header(path);
        if (n) *n = size_t(h.n);
        if (time) *time = h.time;
        if (G) *G = h.G;
        if (eps) *eps = h.eps;
    });
}
int g2_read_snapshot(const char* path, size_t cap, double* mass, double* pos, double* vel, size_t* n, double* time,
                     double* G, double* eps) {
    return guarded([&] {
        const g2::SnapshotHeader h = g2::read_snapshot(path, mass, pos, vel, cap);
        if (n) *n = size_t(h.n);
        if (time) *time = h.time;
        if (G) *G = h.G;
        if (eps) *eps = h.eps;
    });
}
int g2_write_snapshot(const char* path, size_t n, const double* mass, const double* pos, const double* vel,
                      double time, const g2_grav_params* p) {
    return guarded([&] { g2::write_snapshot(path, n, mass, pos, vel, time, p->G, p->eps); });
}

int g2_predict(size_t n, double* pos, double* vel, const double* acc, double dt, int device) {
    return guarded([&] {
        G2_CUDA(cudaSetDevice(device));
        g2::DBuf<double> p, v, a;
        p.reserve(3 * n + 3), v.reserve(3 * n + 3), a.reserve(3 * n + 3);
        G2_CUDA(cudaMemcpy(p.p, pos, 3 * n * 8, cudaMemcpyHostToDevice));
        G2_CUDA(cudaMemcpy(v.p, vel, 3 * n * 8, cudaMemcpyHostToDevice));
        G2_CUDA(cudaMemcpy(a.p, acc, 3 * n * 8, cudaMemcpyHostToDevice));
        g2::launch_predict_aos(p.p, v.p, a.p, n, dt, nullptr);
        G2_CUDA(cudaMemcpy(pos, p.p, 3 * n * 8, cudaMemcpyDeviceToHost));
        G2_CUDA(cudaMemcpy(vel, v.p, 3 * n * 8, cudaMemcpyDeviceToHost));
    });
}

int g2_sim_create(size_t n, const double* mass, const double* pos, const double* vel, const g2_grav_params* p,
                  const g2_step_scheme* s, const g2_engine_config* c, const g2_tuner_config* t, int device,
                  g2_sim** out) {
    return guarded([&] {
        auto* h = new g2_sim;
        try {
            h->s = std::make_unique<g2::Simulation>(n, mass, pos, vel, to_h(p), to_h(s), to_h(c), to_h(t), device);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}
int g2_sim_create_from_snapshot(const char* path, double dacc, const g2_step_scheme* s, const g2_engine_config* c,
                                const g2_tuner_config* t, int device, g2_sim** out) {
    return guarded([&] {
        const g2::SnapshotHeader h = g2::read_snapshot_header(path);
        g2::check_snapshot_size(path, h);  // before sizing any buffer by the file's count
        const size_t n = size_t(h.n);
        G2_CUDA(cudaSetDevice(device));
        double* buf = nullptr;  // pinned: the reads land where the H2D copies stream from
        G2_CUDA(cudaMallocHost(&buf, 7 * n * sizeof(double)));
        std::unique_ptr<double, decltype(&cudaFreeHost)> hold(buf, &cudaFreeHost);
        g2::read_snapshot(path, buf, buf + n, buf + 4 * n, n);
        const g2_grav_params p{h.G, h.eps, dacc};
        auto* sim = new g2_sim;
        try {
            sim->s = std::make_unique<g2::Simulation>(n, buf, buf + n, buf + 4 * n, to_h(&p), to_h(s), to_h(c), to_h(t),
                                                      device);
        } catch (...) {
            delete sim;
            throw;
        }
        *out = sim;
    });
}
int g2_sim_write_snapshot(g2_sim* s, const char* path) {
    return guarded([&] {
        const size_t n = s->s->n();
        std::vector<double> m(n), p(3 * n), v(3 * n);
        double time = 0.0;
        s->s->get_state(p.data(), v.data(), nullptr, nullptr, nullptr, &time);
        s->s->get_mass(m.data());
        const auto& gp = s->s->grav_params();
        g2::write_snapshot(path, n, m.data(), p.data(), v.data(), time, gp.G, gp.eps);
    });
}
void g2_sim_destroy(g2_sim* s) { delete s; }
int g2_sim_init(g2_sim* s) {
    return guarded([&] { s->s->init(); });
}
int g2_sim_step(g2_sim* s, g2_step_result* r) {
    return guarded([&] {
        const g2::StepResultH x = s->s->step();
        if (!r) return;
        r->walk_tree = x.timings.walk_tree, r->calc_node = x.timings.calc_node, r->make_tree = x.timings.make_tree;
        r->predict = x.timings.predict, r->correct = x.timings.correct;
        put(x.events, &r->events);
        r->active = x.active, r->rebuild_interval = x.rebuild_interval, r->rebuilt = x.rebuilt ? 1 : 0;
        r->wall_seconds = x.wall_seconds;
    });
}
int g2_sim_set_fixed_rebuild_interval(g2_sim* s, size_t interval) {
    return guarded([&] { s->s->set_fixed_rebuild_interval(interval); });
}
int g2_sim_get_state(g2_sim* s, double* pos, double* vel, double* acc, double* acc_old_mag, uint8_t* level,
                     double* time) {
    return guarded([&] { s->s->get_state(pos, vel, acc, acc_old_mag, level, time); });
}
int g2_sim_set_state(g2_sim* s, const double* pos, const double* vel) {
    return guarded([&] { s->s->set_state(pos, vel); });
}
int g2_sim_set_phase_overlap(g2_sim* s, int on) {
    return guarded([&] { s->s->set_phase_overlap(on != 0); });
}
int g2_sim_set_rebuild_every_step(g2_sim* s, int on) {
    return guarded([&] { s->s->set_rebuild_every_step(on != 0); });
}
int g2_sim_set_tuner_model(g2_sim* s, double flop_rate, double build_seconds_per_particle) {
    return guarded([&] {
        if (flop_rate > 0.0 && !(build_seconds_per_particle >= 0.0))
            throw g2::Error(G2_DATA_ERROR, "set_tuner_model: build time per particle must be >= 0");
        s->s->set_tuner_model(flop_rate, build_seconds_per_particle);
    });
}
int g2_sim_tuner_interval(g2_sim* s, size_t* interval) {
    return guarded([&] { *interval = s->s->tuner().interval(); });
}

int g2_sim_sort_stats(g2_sim* s, unsigned long long* bucket_sorts, unsigned long long* radix_fallbacks) {
    return guarded([&] {
        *bucket_sorts = s->s->engine().bucket_sorts();
        *radix_fallbacks = s->s->engine().bucket_fallbacks();
    });
}

void g2_mesh_shard(unsigned n_groups, int rank, int world, unsigned* lo, unsigned* hi) {
    uint32_t a = 0, b = 0;
    if (world >= 1 && rank >= 0 && rank < world) g2::equal_shard(n_groups, rank, world, a, b);
    *lo = a, *hi = b;
}
size_t g2_mesh_window(size_t n, size_t group_size, int world) {
    return world >= 1 && group_size >= 1 ? g2::shard_window(n, group_size, world) : 0;
}
unsigned g2_slice_owner(const float* root_child_mass, unsigned n_children, unsigned slice, unsigned n_heavy,
                        int world) {
    return g2::slice_owner_of(root_child_mass, n_children, slice, n_heavy, unsigned(std::max(1, world)));
}

int g2_sim_walk_records(g2_sim* s, unsigned* used, size_t* capacity) {
    return guarded([&] {
        uint32_t q[16];
        s->s->engine().read_qstate(q);
        *used = q[6];
        *capacity = s->s->engine().task_pool_capacity();
    });
}

int g2_sim_walk_kernel_seconds(g2_sim* s, double* seconds) {
    return guarded([&] { *seconds = s->s->engine().last_walk_kernel_seconds(); });
}

int g2_sim_walk_slices(g2_sim* s, unsigned* heavy_groups, unsigned* slices) {
    return guarded([&] {
        uint32_t q[16];
        s->s->engine().read_qstate(q);
        *slices = q[7];
        *heavy_groups = q[9] ? q[7] / q[9] : 0u;
    });
}

int g2_sim_stream(g2_sim* s, void** stream) {
    return guarded([&] { *stream = reinterpret_cast<void*>(s->s->engine().stream()); });
}
unsigned long long g2_launch_count(void) { return g2::launch_counter().load(); }
size_t g2_autotune(double build_time, size_t n_hist, const double* hist, size_t min_interval, size_t max_interval,
                   size_t current_interval) {
    try {
        g2::RebuildTuner t(g2::TunerConfigH{min_interval, max_interval, current_interval});
        t.record_build(build_time);
        for (size_t k = 0; k < n_hist; ++k) t.record_walk(hist[k]);
        return t.autotune();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 0;
    }
}

int g2_nccl_unique_id(unsigned char id[128]) {
    return guarded([&] {
        ncclUniqueId u;
        G2_NCCL(nccl().get_unique_id(&u));
        static_assert(sizeof(u) == 128, "ncclUniqueId size");
        std::memcpy(id, &u, 128);
    });
}
int g2_sim_set_mesh(g2_sim* s, int rank, int world, const unsigned char id[128]) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world) throw g2::Error(G2_DATA_ERROR, "set_mesh: bad rank/world");
        // world == 1 is a real (one-rank) communicator: the step runs the same sharded path and
        // NCCL collectives as on a larger mesh
        auto ex = std::make_unique<NcclExchange>();
        ncclUniqueId u;
        std::memcpy(&u, id, 128);
        G2_NCCL(nccl().comm_init_rank(&ex->comm, world, u, rank));
        ex->world = world;
        ex->prepare(*s->s);
        s->s->set_shard(rank, world, ex.get());
        s->ex = std::move(ex);
    });
}

size_t g2_p2p_handle_bytes(void) { return kP2PHandleBytes; }

int g2_sim_p2p_export(g2_sim* s, int rank, int world, void* handle) {
    return guarded([&] {
        if (world < 2 || world > g2::kMaxPeers || rank < 0 || rank >= world)
            throw g2::Error(G2_DATA_ERROR, "p2p_export: bad rank/world (2 <= world <= 8)");
        auto ex = std::make_unique<PeerExchange>();
        ex->alloc(*s->s, world, rank);
        auto* h = static_cast<cudaIpcMemHandle_t*>(handle);
        G2_CUDA(cudaIpcGetMemHandle(&h[0], ex->buf[0]));
        G2_CUDA(cudaIpcGetMemHandle(&h[1], ex->buf[1]));
        G2_CUDA(cudaIpcGetMemHandle(&h[2], ex->flags));
        G2_CUDA(cudaIpcGetMemHandle(&h[3], ex->cost[0]));
        G2_CUDA(cudaIpcGetMemHandle(&h[4], ex->cost[1]));
        G2_CUDA(cudaIpcGetMemHandle(&h[5], ex->times));
        G2_CUDA(cudaIpcGetMemHandle(&h[6], ex->tflags));
        s->pending = std::move(ex);
    });
}

int g2_sim_set_mesh_p2p(g2_sim* s, int rank, int world, const void* handles) {
    return guarded([&] {
        PeerExchange* ex = s->pending.get();
        if (!ex || ex->world != world || ex->self != rank)
            throw g2::Error(G2_DATA_ERROR, "set_mesh_p2p: call g2_sim_p2p_export with the same rank/world first");
        const auto* h = static_cast<const cudaIpcMemHandle_t*>(handles);
        G2_CUDA(cudaSetDevice(ex->device));
        for (int q = 0; q < world; ++q) {
            if (q == rank) continue;
            void* p[kP2PHandles];
            for (int k = 0; k < kP2PHandles; ++k) {
                G2_CUDA(cudaIpcOpenMemHandle(&p[k], h[kP2PHandles * q + k], cudaIpcMemLazyEnablePeerAccess));
                ex->opened.push_back(p[k]);
            }
            ex->ptimes[q] = static_cast<double*>(p[5]), ex->ptflags[q] = static_cast<uint64_t*>(p[6]);
            ex->pbuf[q][0] = static_cast<float4*>(p[0]), ex->pbuf[q][1] = static_cast<float4*>(p[1]);
            ex->pflags[q] = static_cast<uint64_t*>(p[2]);
            ex->pcost[q][0] = static_cast<uint32_t*>(p[3]), ex->pcost[q][1] = static_cast<uint32_t*>(p[4]);
        }
        s->s->set_shard(rank, world, ex);
        s->ex = std::move(s->pending);
    });
}

int g2_sim_set_mesh_local_p2p(g2_sim** sims, int world) {
    return guarded([&] {
        if (world < 2 || world > g2::kMaxPeers) throw g2::Error(G2_DATA_ERROR, "set_mesh_local_p2p: 2 <= world <= 8");
        std::vector<PeerExchange*> ex(world);
        auto mesh = std::make_shared<LocalMesh>();
        for (int r = 0; r < world; ++r) mesh->sims.push_back(sims[r]->s.get());
        for (int r = 0; r < world; ++r) {
            auto e = std::make_unique<PeerExchange>();
            e->alloc(*sims[r]->s, world, r);
            e->mesh = mesh;
            ex[r] = e.get();
            sims[r]->ex = std::move(e);
        }
        for (int r = 0; r < world; ++r) {
            for (int q = 0; q < world; ++q) {
                ex[r]->pbuf[q][0] = ex[q]->buf[0], ex[r]->pbuf[q][1] = ex[q]->buf[1];
                ex[r]->pflags[q] = ex[q]->flags;
                ex[r]->pcost[q][0] = ex[q]->cost[0], ex[r]->pcost[q][1] = ex[q]->cost[1];
                ex[r]->ptimes[q] = ex[q]->times, ex[r]->ptflags[q] = ex[q]->tflags;
                if (ex[q]->device != ex[r]->device) {
                    int ok = 0;
                    G2_CUDA(cudaDeviceCanAccessPeer(&ok, ex[r]->device, ex[q]->device));
                    if (!ok) throw g2::Error(G2_INTERNAL, "set_mesh_local_p2p: devices without peer access");
                    cudaSetDevice(ex[r]->device);
                    const cudaError_t e = cudaDeviceEnablePeerAccess(ex[q]->device, 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) G2_CUDA(e);
                    cudaGetLastError();
                }
            }
            sims[r]->s->set_shard(r, world, ex[r]);
        }
    });
}

int g2_sim_set_mesh_local(g2_sim** sims, int world) {
    return guarded([&] {
        if (world < 1) throw g2::Error(G2_DATA_ERROR, "set_mesh_local: world must be >= 1");
        auto mesh = std::make_shared<LocalMesh>();
        for (int r = 0; r < world; ++r) mesh->sims.push_back(sims[r]->s.get());
        for (int r = 0; r < world; ++r) {
            if (world == 1) {
                sims[r]->s->set_shard(0, 1, nullptr);
                continue;
            }
            auto ex = std::make_unique<LocalExchange>();
            ex->world = world;
            ex->mesh = mesh;
            ex->prepare(*sims[r]->s);
            sims[r]->s->set_shard(r, world, ex.get());
            sims[r]->ex = std::move(ex);
        }
    });
}

}  // extern "C"
