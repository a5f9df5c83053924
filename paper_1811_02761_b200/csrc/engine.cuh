// Host-side engine and simulation driver (C++), the implementation behind the
// C-ABI in include/g2/capi.h.  Mirrors gravitree's GravityEngine
// (engine.hpp:29-66) and Simulation (integrator.hpp:54-91); all particle state
// lives on the device in Morton order of the last build.
#pragma once

#include <chrono>
#include <vector>

#include "kernels.cuh"
#include "bucket_sort.cuh"
#include "radix_sort.cuh"

namespace g2 {

struct GravParamsH {
    double G = 1.0, eps = 0.0, dacc = 0.001953125;  // particle_system.hpp:53-57
};
struct EngineConfigH {  // engine.hpp:14-23
    size_t leaf_cap = 8, group_size = 32, list_capacity = 1024, frontier_cap = 0;
    bool count_ops = true;
    double bootstrap_theta = 0.5;
    size_t bootstrap_direct_limit = 65536;
    unsigned threads = 0;
};
struct EventsH {
    uint64_t interactions = 0, mac_evals = 0, list_pushes = 0;
};

// pinned host block the step/build boundary read-backs land in (one synchronisation each)
struct HostSync {
    DevFlags flags;
    unsigned long long events[3];
    unsigned long long tnext;
    uint32_t na;
    uint32_t ls[kMaxDepth + 3];
    uint32_t recs;  // task records the last walk allocated (sizes the pool for the next)
    int bucket_gate;  // the last rebuild's bucket sort overflowed (its radix fallback ran)
};

class Engine {
public:
    Engine(GravParamsH p, EngineConfigH c, int device);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // ---- host-order API (GravityEngine) -------------------------------------
    void build(size_t n, const double* mass, const double* pos, bool with_nodes);
    void refresh(size_t n, const double* mass, const double* pos);
    // targets == nullptr: all particles.  acc_out (3n) written for targets only;
    // pot_out (n, nullable) likewise.  acc_old_mag (n) in original order.
    EventsH evaluate(size_t n, const double* mass, const double* pos, const double* acc_old_mag, size_t n_targets,
                     const uint32_t* targets, double* acc_out, double* pot_out);
    EventsH bootstrap(size_t n, const double* mass, const double* pos, double* acc_out, double* acc_old_mag_out);
    bool has_tree() const { return has_tree_; }
    size_t n() const { return n_; }
    size_t ncells() const { return ncells_; }
    void get_tree(double* bbox4, uint64_t* keys, uint32_t* perm, uint32_t* rank, uint32_t* cells4, uint8_t* depth,
                  double* nodes5);
    const GravParamsH& params() const { return p_; }
    GravParamsH& params() { return p_; }
    const EngineConfigH& config() const { return c_; }

    // ---- device-level operations (used by Simulation) -------------------------
    void reserve(size_t n);
    // Morton-sort the particles currently in xyzm_s() (position k holds original
    // id ids[k]); reorders xyzm_s and returns src (new position k <- old src[k]).
    // new Morton order of the resident state; returns src (new k <- old position).  rank_cur null:
    // storage-order sort + tie repair (rank_ left stale); else the (key, id) sort via key_by_id.
    // cube_partials: the bbox partials of the current positions are already in bbox_partials() (the
    // predict kernel wrote them), only the final reduction runs
    // defer_perm: the caller writes perm (= ids gathered by the returned order) itself
    const uint32_t* rebuild_sorted(const uint32_t* ids, const uint32_t* rank_cur, bool cube_partials = false,
                                   bool defer_perm = false);
    double* bbox_partials() { return bbox_part_.p; }
    DevFlags* dev_flags() { return flags_.p; }
    bool take_tie_overflow();  // true (and clears) if a tie run was too long for the repair (staged by split)
    bool take_bucket_overflow();  // true (and clears) if the last rebuild's bucket sort overflowed (ditto)
    // rebuild sorts so far: by the bucket sort, and by its radix fallback (an overflowed bucket)
    unsigned long long bucket_sorts() const { return bucket_sorts_; }
    size_t task_pool_capacity() const { return rec_cap_; }
    void read_qstate(uint32_t* q16) {  // the last walk's queue state (diagnostics; synchronises)
        G2_CUDA(cudaMemcpyAsync(q16, qstate_.p, 16 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s_));
        G2_CUDA(cudaStreamSynchronize(s_));
    }
    unsigned long long bucket_fallbacks() const { return bucket_fallbacks_; }
    // boundary read-backs: enqueue copies into the pinned staging block, one sync, then inspect
    HostSync* host_sync() { return hs_; }
    void enqueue_flags();
    void enqueue_events();
    void sync();
    void raise_flags();  // throws for the staged device flags
    // syncs; true (and the pool grows) if the last walk ran out of task records.  Such a walk skipped
    // donations: exact, but not bit-reproducible; synchronous callers walk again.  A Simulation step
    // only grows the pool for the next step (its pool starts at n/8 records, far above any measured
    // need: 0.1 n at M31 2^20 all-active).
    bool walk_pool_overflow();
    void events_host(EventsH& ev) const;
    void ensure_rank();        // rank_ = inverse of perm_ if a storage-order rebuild left it stale
    void split_and_nodes(bool with_nodes);
    // overlap: the internal levels run on a side stream, joined by the next walk (after its group
    // spheres) or the next calc_nodes; calc_tail_stream() is where they end
    void calc_nodes(bool overlap = false);
    void join_calc();
    double last_walk_kernel_seconds();  // device time of the last walk kernel (CUDA events on its stream)
    cudaStream_t calc_tail_stream() const { return calc_join_pending_ ? side_ : s_; }
    // walk sinks (sorted positions) with acc_old_mag (sorted); results into
    // ax_s/ay_s/az_s/pot_s at the sinks' sorted positions.
    // slice_rank/slice_world: the ranks the whole-system groups' slices are dealt to; combine: form
    // the sliced groups' results now (false: the caller calls combine_slices after the exchange)
    EventsH walk(const uint32_t* sinks, const uint32_t* n_sinks_dev, uint32_t n_sinks_cap, const double* amag_s,
                 bool with_pot, bool sync_events, uint32_t group_lo = 0, uint32_t group_hi = ~0u,
                 bool finalize = true, int slice_rank = 0, int slice_world = 1, bool combine = true);
    // the last walk's sliced groups from the slice partials (slice j at src + owner(j) * stride + 32 j)
    void combine_slices(const float4* src, size_t stride, int world);
    const float4* slice_region() { return accum() + walk_slice_base(n_); }
    // accum slots -> FP64 accelerations at the sinks' sorted positions
    int device() const { return device_; }
    float4* accum() { return accum_ext_ ? accum_ext_ : accum_.p; }
    // fused peer exchange for the next walks: accumulate into `accum` (an exported buffer) and
    // push finished groups to `peers` (world entries, [self] unused); world <= 1 turns it off
    // peer_cost: every rank's cost array of this step ([self] = own); cost_prev / ng_prev: the own copy
    // of the previous step's costs and their group count, ng_cur: where this step records its count
    void set_peer_push(int world, int self, float4* accum, float4* const* peers, uint32_t* const* peer_cost = nullptr,
                       const uint32_t* cost_prev = nullptr, const uint32_t* ng_prev = nullptr,
                       uint32_t* ng_cur = nullptr) {
        peer_world_ = world, peer_self_ = self, accum_ext_ = world > 1 ? accum : nullptr;
        for (int q = 0; q < kMaxPeers; ++q) {
            peer_accum_[q] = world > 1 && q < world ? peers[q] : nullptr;
            peer_cost_[q] = world > 1 && q < world && peer_cost ? peer_cost[q] : nullptr;
        }
        cost_prev_ = cost_prev, ng_prev_ = ng_prev, ng_cur_ = ng_cur;
    }
    size_t accum_cap() const { return accum_.cap; }
    void reserve_accum(size_t slots) { accum_.reserve(slots); }
    void direct_sum_orig(const double4* xyzm_orig, size_t n, double* ax, double* ay, double* az);
    // FP32 range of the walk: G x total mass must be a finite float (data_error otherwise);
    // the largest mass selects the guarded flush when the self-pair factor G m / eps^3 could overflow
    void note_masses(size_t n, const double* mass);
    void check_flags();  // syncs and throws on device-side errors
    void read_events(EventsH& ev);

    cudaStream_t stream() const { return s_; }
    double4* xyzm_s() { return xyzm_s_.p; }
    double4* xyzm_alt() { return xyzm_alt_.p; }
    void swap_xyzm() { std::swap(xyzm_s_.p, xyzm_alt_.p); }
    uint32_t* perm() { return perm_.p; }
    uint32_t* rank() { return rank_.p; }
    double* ax_s() { return ax_s_.p; }
    double* ay_s() { return ay_s_.p; }
    double* az_s() { return az_s_.p; }
    double* pot_s() { return pot_s_.p; }
    uint64_t* group_inter() { return group_inter_.p; }
    void set_n(size_t n) { n_ = n; }
    void mark_tree(bool v) { has_tree_ = v; }
    uint32_t* n_groups_dev() { return n_groups_.p; }

private:
    void ensure_cells(size_t cap);
    void ensure_task_pool(size_t records);
    void ensure_queue(size_t records);
    void sort_keys_identity_payload(size_t n);  // keys in keys_a_ by original id -> perm_, keys sorted
    void upload_orig(size_t n, const double* mass, const double* pos);

    GravParamsH p_;
    EngineConfigH c_;
    int device_;
    cudaStream_t s_ = nullptr;
    cudaStream_t side_ = nullptr;  // calc_node's internal levels (calc_nodes(true))
    cudaEvent_t calc_fork_ = nullptr, calc_join_ = nullptr;
    bool calc_join_pending_ = false;
    cudaEvent_t walk_ev_[2] = {nullptr, nullptr};  // around the walk kernel launch
    bool walk_ev_valid_ = false;
    size_t n_ = 0, cap_ = 0, ncells_ = 0, cell_cap_ = 0;
    HostSync* hs_ = nullptr;  // pinned
    bool has_tree_ = false;
    bool rank_valid_ = true;  // rank_ matches perm_ (false after a storage-order rebuild)
    uint32_t max_level_width_ = 0;
    double mass_max_ = 0.0;  // largest particle mass seen by note_masses

    DBuf<double> pos3_, mass_, amag_o_;   // host-order staging
    DBuf<double4> xyzm_o_, xyzm_s_, xyzm_alt_;
    DBuf<uint64_t> keys_a_, keys_b_;
    DBuf<uint32_t> vals_a_, vals_b_, perm_, rank_, src_, tgt_rank_;
    DBuf<double> amag_s_, ax_s_, ay_s_, az_s_, pot_s_, out_;
    DBuf<uint32_t> first_child_, child_count_, first_, count_;
    DBuf<uint8_t> depth_;
    DBuf<WNode> nodes_;
    DBuf<WNode32> nodes32_;
    uint32_t ls_host_[kMaxDepth + 3] = {};  // host copy of level_start of the current topology
    DBuf<float4> rel_;
    DBuf<uint32_t> leaf_of_;
    DBuf<uint32_t> heavy_;
    DBuf<uint8_t> sliced_;
    WalkBuffers last_walk_{};  // the last walk's buffers (combine_slices)
    double walk_G_ = 1.0;
    DBuf<uint4> int_list_;                  // internal cells per depth (launch_tree_topology)
    DBuf<uint32_t> int_count_, calc_sync_;
    DBuf<uint32_t> level_start_, tile_counters_;
    DBuf<uint64_t> split_status_;
    DBuf<uint32_t> split_tiles_;
    BucketScratch bucket_;  // rebuild bucket sort (bucket_sort.cu)
    bool bucket_pending_ = false;  // the last rebuild_sorted launched a bucket sort (gate read at the split sync)
    bool bucket_overflow_ = false;
    unsigned long long bucket_sorts_ = 0, bucket_fallbacks_ = 0;
    DBuf<double> bbox_part_;
    DBuf<Cube> cube_;
    DBuf<uint32_t> sinks_, sinks_alt_, n_sinks_, n_groups_;
    DBuf<GroupRec> groups_;
    DBuf<float4> accum_;
    DBuf<uint32_t> gcost_, shard_, order_, order_scratch_;
    DBuf<uint4> trec_;          // walk task records (deterministic combination of split groups)
    DBuf<float4> tacc_;         // [rec_cap * 32] their accumulators
    DBuf<uint32_t> batch_rec_;  // [queue_cap] record of each donated slot
    size_t rec_cap_ = 0;
    uint32_t queue_cap_ = 0, ring_bits_ = 20;
    bool grow_pool_ = false;    // a walk ran out of task records: double the pool before the next
    uint32_t* peer_cost_[kMaxPeers] = {};
    const uint32_t* cost_prev_ = nullptr;
    const uint32_t* ng_prev_ = nullptr;
    uint32_t* ng_cur_ = nullptr;
    float4* accum_ext_ = nullptr;
    float4* peer_accum_[kMaxPeers] = {};
    int peer_world_ = 1, peer_self_ = 0;
    DBuf<unsigned long long> events_;
    DBuf<uint64_t> queue_;
    DBuf<uint32_t> batch_;
    DBuf<uint32_t> qstate_, spill_, level_count_;
    DBuf<uint64_t> group_inter_;
    DBuf<uint4> trace_;
    DBuf<uint32_t> trace_n_;
    DBuf<DevFlags> flags_;
    SortScratch sort_;
};

// ---- rebuild auto-tuner: host restatement of rebuild_tuner.{hpp,cpp} ------------
struct TunerConfigH {
    size_t min_interval = 1, max_interval = 128, initial_interval = 8;
};
class RebuildTuner {
public:
    explicit RebuildTuner(TunerConfigH c = {});
    size_t interval() const { return interval_; }
    size_t steps_since_rebuild() const { return steps_; }
    bool should_rebuild() const { return steps_ >= std::max<size_t>(interval_, 2); }  // rebuild_tuner.hpp:26
    void record_build(double s) { build_time_ = s; }
    void record_walk(double s) {
        hist_.push_back(s);
        ++steps_;
    }
    void on_rebuild();
    void reset_cycle() {
        hist_.clear();
        steps_ = 0;
    }
    void set_interval(size_t i);
    size_t autotune() const;  // autotune_rebuild (rebuild_tuner.cpp:28-61)
    double build_time() const { return build_time_; }
    const std::vector<double>& history() const { return hist_; }

private:
    TunerConfigH c_;
    size_t interval_, steps_ = 0;
    double build_time_ = 0.0;
    std::vector<double> hist_;
};

struct StepSchemeH {  // integrator.hpp:18-23
    double eta = 0.5, dt_max = 0.0625;
    bool adaptive = true;
    int fixed_level = 0;
};
struct PhaseTimingsH {
    double walk_tree = 0, calc_node = 0, make_tree = 0, predict = 0, correct = 0;
};
struct StepResultH {
    PhaseTimingsH timings;
    EventsH events;
    size_t active = 0, rebuild_interval = 0;
    bool rebuilt = false;
    double wall_seconds = 0.0;
};

// Multi-GPU hook: after the walk, each rank holds accelerations of its own
// groups; the exchange makes all ranks hold all of them (one all-gather).
struct Exchange {
    virtual ~Exchange() = default;
    virtual void before_walk(class Simulation&) {}  // e.g. point the walk at this step's exchange buffers
    virtual bool device_shards() const { return false; }  // the walk splits the groups on the device
    virtual void allgather_acc(class Simulation& sim) = 0;
    // where every rank's slice partials are after allgather_acc (default: pushed into this rank's region)
    virtual void slice_source(class Simulation& sim, const float4*& src, size_t& stride);
    // make the rebuild tuner's inputs identical on every rank (the rebuild decision reorders all state,
    // and the exchange addresses accumulators by slot): walk := sum (modelled time: each rank's share of
    // the walk work; the sum is the single-rank value) or max (measured) over ranks; build := max
    virtual void agree_times(class Simulation& sim, double& walk, double& build, bool sum_walk) = 0;
};

class Simulation {
public:
    Simulation(size_t n, const double* mass, const double* pos, const double* vel, GravParamsH p, StepSchemeH sc,
               EngineConfigH ec, TunerConfigH tc, int device);
    void init();
    StepResultH step();
    void set_fixed_rebuild_interval(size_t k) {
        autotune_ = false;
        tuner_.set_interval(k);
    }
    // orig-order host copies
    void get_state(double* pos, double* vel, double* acc, double* acc_old_mag, uint8_t* level, double* time);
    void get_mass(double* mass);  // original order
    const GravParamsH& grav_params() const { return p_; }
    void set_state(const double* pos, const double* vel);  // overwrite pos/vel (orig order), keeps the rest
    Engine& engine() { return eng_; }
    RebuildTuner& tuner() { return tuner_; }
    double time() const { return time_; }
    bool initialized() const { return initialized_; }
    size_t n() const { return n_; }
    void set_rebuild_every_step(bool v) { rebuild_every_step_ = v; }
    void set_phase_overlap(bool v) { phase_overlap_ = v; }
    // the rebuild tuner's clock: CUDA-event phase times (flop_rate <= 0, the default), or a
    // deterministic model -- walk = walk Flop (27 I + 5 M, op_counters.hpp:50-63) / flop_rate, build =
    // build_s_per_particle x n -- which makes the rebuild schedule, hence the trajectory, reproducible
    void set_tuner_model(double flop_rate, double build_s_per_particle) {
        model_rate_ = flop_rate, model_build_ = build_s_per_particle;
    }
    int rank() const { return rank_; }
    void set_shard(int rank, int world, Exchange* ex) {
        rank_ = rank, world_ = world, exchange_ = ex;
    }
    // shard helpers for the exchange
    uint32_t active_count() const { return last_active_; }
    const uint32_t* sinks() const { return sinks_.p; }
    uint32_t shard_lo() const { return shard_lo_; }
    uint32_t shard_hi() const { return shard_hi_; }
    const uint32_t* n_active_dev() const { return n_active_.p; }
    size_t group_size() const { return eng_.config().group_size; }

private:
    StepState state();
    void reorder(const uint32_t* src, uint32_t* perm_out = nullptr);
    void rebuild_order(bool cube_partials = false);          // new Morton order + topology of the resident state
    const uint32_t* rank_cur();    // original id -> current position (computed on demand)
    double elapsed(cudaEvent_t a, cudaEvent_t b);

    Engine eng_;
    GravParamsH p_;
    StepSchemeH sc_;
    RebuildTuner tuner_;
    size_t n_;
    bool initialized_ = false, autotune_ = true, rebuild_every_step_ = false;
    bool phase_overlap_ = true;  // calc_node's internal levels beside the compaction and group spheres
    double model_rate_ = 0.0, model_build_ = 0.0;
    uint64_t now_ = 0;
    double tick_ = 0.0, time_ = 0.0;
    uint32_t last_active_ = 0;
    int rank_ = 0, world_ = 1;
    Exchange* exchange_ = nullptr;
    uint32_t shard_lo_ = 0, shard_hi_ = ~0u;

    DBuf<double> vx_, vy_, vz_, ax_, ay_, az_, amag_;
    DBuf<double> vx2_, vy2_, vz2_, ax2_, ay2_, az2_, amag2_;
    DBuf<uint8_t> level_, level2_, active_, active2_;
    DBuf<uint64_t> last_, last2_;
    DBuf<uint32_t> ids_, ids2_, rank_cur_, sinks_, n_active_, compact_ctr_;
    bool rank_cur_valid_ = true;
    DBuf<uint64_t> compact_status_;
    DBuf<unsigned long long> t_next_;
    DBuf<double> io_, io2_;  // host-transfer staging (original particle order)
    cudaEvent_t ev_[12];
};

}  // namespace g2
