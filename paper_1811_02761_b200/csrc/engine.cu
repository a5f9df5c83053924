// Host implementation of Engine / Simulation / RebuildTuner (see engine.cuh).
#include "engine.cuh"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>

namespace g2 {
namespace {

constexpr int kB = 256;
inline unsigned gridn(size_t n) { return std::max(1u, std::min<unsigned>(ceil_div(n, kB), kNumSMs * 16)); }

// AoS xyz (3n) [+ gather by src] -> SoA
__global__ void deinterleave_kernel(const double* __restrict__ v3, const uint32_t* __restrict__ src, double* x,
                                    double* y, double* z, size_t n) {
    for (size_t i = blockIdx.x * size_t(kB) + threadIdx.x; i < n; i += size_t(gridDim.x) * kB) {
        const size_t j = src ? src[i] : i;
        x[i] = v3[3 * j], y[i] = v3[3 * j + 1], z[i] = v3[3 * j + 2];
    }
}
// out3[3*j] = x[idx[j]]...  (idx nullable => identity)
__global__ void interleave_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                  const double* __restrict__ z, const uint32_t* __restrict__ idx, double* out3,
                                  size_t n) {
    for (size_t j = blockIdx.x * size_t(kB) + threadIdx.x; j < n; j += size_t(gridDim.x) * kB) {
        const size_t k = idx ? idx[j] : j;
        out3[3 * j] = x[k], out3[3 * j + 1] = y[k], out3[3 * j + 2] = z[k];
    }
}
__global__ void gather_scalar_kernel(const double* __restrict__ in, const uint32_t* __restrict__ idx, double* out,
                                     size_t n) {
    for (size_t j = blockIdx.x * size_t(kB) + threadIdx.x; j < n; j += size_t(gridDim.x) * kB)
        out[j] = in[idx ? idx[j] : j];
}
__global__ void xyzm_to_pos3_kernel(const double4* __restrict__ xyzm, const uint32_t* __restrict__ idx, double* pos3,
                                    size_t n) {
    for (size_t j = blockIdx.x * size_t(kB) + threadIdx.x; j < n; j += size_t(gridDim.x) * kB) {
        const double4 q = xyzm[idx ? idx[j] : j];
        pos3[3 * j] = q.x, pos3[3 * j + 1] = q.y, pos3[3 * j + 2] = q.z;
    }
}
// positions (orig order, 3n) written into sorted state through rank
__global__ void set_pos_kernel(double4* xyzm, const double* __restrict__ pos3, const uint32_t* __restrict__ ids,
                               size_t n) {
    for (size_t k = blockIdx.x * size_t(kB) + threadIdx.x; k < n; k += size_t(gridDim.x) * kB) {
        const size_t id = ids[k];
        double4 q = xyzm[k];
        q.x = pos3[3 * id], q.y = pos3[3 * id + 1], q.z = pos3[3 * id + 2];
        xyzm[k] = q;
    }
}
// the whole per-particle state gathered into the new Morton order in one pass
struct ReorderArgs {
    const double4* xin;
    double4* xout;
    const double* in[7];
    double* out[7];
    const uint8_t *lin, *ain;
    uint8_t *lout, *aout;
    const uint64_t* tin;
    uint64_t* tout;
    const uint32_t* iin;  // original ids by position
    uint32_t* iout;
    uint32_t* iout2;      // nullable: a second copy of the new ids (the engine's perm)
};
__global__ void __launch_bounds__(kB) reorder_kernel(ReorderArgs r, const uint32_t* __restrict__ src, size_t n) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    for (size_t i = blockIdx.x * size_t(kB) + threadIdx.x; i < n; i += size_t(gridDim.x) * kB) {
        const uint32_t j = src[i];
        r.xout[i] = r.xin[j];
#pragma unroll
        for (int k = 0; k < 7; ++k) r.out[k][i] = r.in[k][j];
        r.lout[i] = r.lin[j];
        r.aout[i] = r.ain[j];
        r.tout[i] = r.tin[j];
        const uint32_t id = r.iin[j];
        r.iout[i] = id;
        if (r.iout2) r.iout2[i] = id;
    }
}
__global__ void fill_u8_kernel(uint8_t* p, uint8_t v, size_t n) {
    for (size_t j = blockIdx.x * size_t(kB) + threadIdx.x; j < n; j += size_t(gridDim.x) * kB) p[j] = v;
}
__global__ void frontier_check_kernel(const uint32_t* __restrict__ cnt, size_t m, uint32_t cap, DevFlags* flags) {
    for (size_t j = blockIdx.x * size_t(kB) + threadIdx.x; j < m; j += size_t(gridDim.x) * kB)
        if (cnt[j] > cap) flags->resource_error = 1;
}

double seconds(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

// =============================================================================================
Engine::Engine(GravParamsH p, EngineConfigH c, int device) : p_(p), c_(c), device_(device) {
    if (c_.group_size < 1) throw Error(kDataError, "GravityEngine: group_size must be >= 1");
    if (!(p_.dacc > 0.0)) throw Error(kDataError, "GravityEngine: dacc must be positive");
    if (p_.eps < 0.0) throw Error(kDataError, "GravityEngine: eps must be non-negative");
    if (c_.group_size > 32)
        throw Error(kDataError, "GravityEngine: group_size > 32 is not supported by the warp-per-group walk");
    G2_CUDA(cudaSetDevice(device_));
    G2_CUDA(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
    flags_.reserve(1);
    G2_CUDA(cudaMemsetAsync(flags_.p, 0, sizeof(DevFlags), s_));
    level_start_.reserve(kMaxDepth + 3);
    tile_counters_.reserve(kMaxDepth + 1);
    cube_.reserve(1);
    bbox_part_.reserve(6 * std::max<size_t>(kNumSMs * 16, kNumSMs * 4));  // launch_bbox or predict_blocks records
    n_sinks_.reserve(1);
    n_groups_.reserve(1);
    events_.reserve(3);
    qstate_.reserve(16);
    ensure_queue(size_t(1) << 20);
    spill_.reserve(walk_resident_warps() * walk_spill_words());
    G2_CUDA(cudaMallocHost(&hs_, sizeof(HostSync)));
    *hs_ = HostSync{};
}

Engine::~Engine() {
    for (auto e : walk_ev_)
        if (e) cudaEventDestroy(e);
    if (side_) {
        cudaStreamSynchronize(side_);
        cudaStreamDestroy(side_);
        cudaEventDestroy(calc_fork_);
        cudaEventDestroy(calc_join_);
    }
    if (s_) {
        cudaStreamSynchronize(s_);
        cudaStreamDestroy(s_);
    }
    if (hs_) cudaFreeHost(hs_);
}

void Engine::reserve(size_t n) {
    if (n <= cap_) return;
    pos3_.reserve(3 * n), mass_.reserve(n), amag_o_.reserve(n);
    xyzm_o_.reserve(n), xyzm_s_.reserve(n), xyzm_alt_.reserve(n);
    keys_a_.reserve(n), keys_b_.reserve(n);
    vals_a_.reserve(n), vals_b_.reserve(n), perm_.reserve(n), rank_.reserve(n), src_.reserve(n),
        tgt_rank_.reserve(n);
    amag_s_.reserve(n), ax_s_.reserve(n), ay_s_.reserve(n), az_s_.reserve(n), pot_s_.reserve(n), out_.reserve(3 * n);
    sinks_.reserve(n), sinks_alt_.reserve(n);
    groups_.reserve(n), accum_.reserve(walk_slice_base(n) + walk_slice_slots()), group_inter_.reserve(n),
        rel_.reserve(n), leaf_of_.reserve(n);
    heavy_.reserve(walk_heavy_words()), sliced_.reserve(n);
    ensure_cells(std::max<size_t>(n + 64, 1024));
    cap_ = n;
    ensure_task_pool(std::max<size_t>(size_t(1) << 16, n / 4));  // no allocation inside a timed walk
    order_.reserve(n + 1), order_scratch_.reserve(walk_order_scratch_words(n));
}

void Engine::ensure_task_pool(size_t want) {
    if (want <= rec_cap_) return;
    G2_CUDA(cudaStreamSynchronize(s_));
    trec_.reserve(want), tacc_.reserve(want * 32);
    rec_cap_ = want;
    ensure_queue(want);
}

// The donated-task ring holds at least as many slots as the task pool has records: a walk's tickets
// (one per donated task, each with its own record) then never wrap, so a donor never waits for a slot.
void Engine::ensure_queue(size_t records) {
    uint32_t bits = 20;
    while (bits < 31 && (size_t(1) << bits) < records) ++bits;
    if ((size_t(1) << bits) <= queue_cap_) return;
    if (queue_cap_) G2_CUDA(cudaStreamSynchronize(s_));
    queue_cap_ = uint32_t(1u << bits), ring_bits_ = bits;
    queue_.reserve(queue_cap_);
    batch_.reserve(size_t(queue_cap_) * 32);
    batch_rec_.reserve(queue_cap_);
    G2_CUDA(cudaMemsetAsync(queue_.p, 0xff, size_t(queue_cap_) * sizeof(uint64_t), s_));
}

void Engine::ensure_cells(size_t cap) {
    if (cap <= cell_cap_) return;
    first_child_.reserve(cap), child_count_.reserve(cap), first_.reserve(cap), count_.reserve(cap);
    depth_.reserve(cap), nodes_.reserve(cap), nodes32_.reserve(cap), int_list_.reserve(cap);
    int_count_.reserve(kMaxDepth + 1), calc_sync_.reserve(calc_sync_words());
    split_status_.reserve(cap / 32 + 64);
    cell_cap_ = cap;
}

// Results read back at a step/build boundary share one pinned staging block and ONE
// stream synchronisation (each extra host round trip idles the GPU between steps).
void Engine::enqueue_flags() {
    G2_CUDA(cudaMemcpyAsync(&hs_->flags, flags_.p, sizeof(DevFlags), cudaMemcpyDeviceToHost, s_));
}
void Engine::enqueue_events() {
    G2_CUDA(cudaMemcpyAsync(hs_->events, events_.p, sizeof hs_->events, cudaMemcpyDeviceToHost, s_));
    G2_CUDA(cudaMemcpyAsync(&hs_->recs, qstate_.p + 6, sizeof(uint32_t), cudaMemcpyDeviceToHost, s_));
}
void Engine::sync() {
    join_calc();
    G2_CUDA(cudaStreamSynchronize(s_));
}

void Engine::check_flags() {
    enqueue_flags();
    sync();
    raise_flags();
}

bool Engine::walk_pool_overflow() {
    enqueue_flags();
    sync();
    if (!hs_->flags.task_pool) return false;
    grow_pool_ = true;
    hs_->flags.task_pool = 0;
    G2_CUDA(cudaMemsetAsync(&flags_.p->task_pool, 0, sizeof(int), s_));
    return true;
}

void Engine::raise_flags() {
    if (hs_->flags.task_pool) {  // not an error: results stay exact, the next walk gets a larger pool
        grow_pool_ = true;
        hs_->flags.task_pool = 0;
        G2_CUDA(cudaMemsetAsync(&flags_.p->task_pool, 0, sizeof(int), s_));
    }
    const DevFlags f = hs_->flags;
    if (f.data_error || f.resource_error || f.singularity || f.stack_overflow || f.queue_overflow || f.peer_timeout) {
        G2_CUDA(cudaMemset(flags_.p, 0, sizeof(DevFlags)));
        if (f.singularity) throw Error(kSingularity, "direct_sum: coincident particles with zero softening");
        if (f.data_error == 1) throw Error(kDataError, "bounding_cube: non-finite position");
        if (f.data_error) throw Error(kDataError, "morton_key: position outside root cube");
        if (f.resource_error) throw Error(kResourceError, "walk_tree_group: frontier queue exhausted");
        if (f.peer_timeout)
            throw Error(kResourceError, "peer exchange: a rank did not reach the exchange barrier in time "
                                        "(G2_PEER_TIMEOUT_S); this step's accelerations are incomplete");
        throw Error(kInternal, "walk: internal stack/queue overflow");
    }
}

void Engine::note_masses(size_t n, const double* mass) {
    double mx = 0.0, tot = 0.0;
    for (size_t i = 0; i < n; ++i) mx = std::max(mx, mass[i]), tot += mass[i];
    // node masses and list entries are FP32 in the walk: their sums must stay finite there (NaN
    // masses pass, as in the reference, which does not validate an engine's system)
    if (std::fabs(p_.G) * tot > double(FLT_MAX) / 2)
        throw Error(kDataError, "particle system: total mass x G exceeds the FP32 range of the walk");
    mass_max_ = mx;
}

void Engine::upload_orig(size_t n, const double* mass, const double* pos) {
    note_masses(n, mass);
    G2_CUDA(cudaMemcpyAsync(pos3_.p, pos, 3 * n * sizeof(double), cudaMemcpyHostToDevice, s_));
    G2_CUDA(cudaMemcpyAsync(mass_.p, mass, n * sizeof(double), cudaMemcpyHostToDevice, s_));
}

void Engine::sort_keys_identity_payload(size_t n) {
    // keys_a_ holds the key of original particle i at index i
    const bool alt = radix_sort_pairs<uint64_t>(keys_a_.p, vals_a_.p, keys_b_.p, vals_b_.p, n, 63, true, sort_, s_);
    uint64_t* ks = alt ? keys_b_.p : keys_a_.p;
    uint32_t* vs = alt ? vals_b_.p : vals_a_.p;
    if (ks != keys_a_.p) G2_CUDA(cudaMemcpyAsync(keys_a_.p, ks, n * 8, cudaMemcpyDeviceToDevice, s_));
    G2_CUDA(cudaMemcpyAsync(perm_.p, vs, n * 4, cudaMemcpyDeviceToDevice, s_));
    launch_invert_perm(perm_.p, rank_.p, n, s_);
    rank_valid_ = true;
}

void Engine::build(size_t n, const double* mass, const double* pos, bool with_nodes) {
    if (n < 1) throw Error(kDataError, "build_tree: empty system");
    if (c_.leaf_cap < 1) throw Error(kDataError, "build_tree: leaf_cap must be >= 1");
    if (n >= (size_t(1) << 31)) throw Error(kDataError, "build_tree: n must be < 2^31");
    reserve(n);
    n_ = n;
    upload_orig(n, mass, pos);
    launch_pack_identity(pos3_.p, mass_.p, xyzm_o_.p, n, s_);
    launch_bbox(xyzm_o_.p, n, bbox_part_.p, cube_.p, flags_.p, s_);
    launch_keys(xyzm_o_.p, nullptr, n, cube_.p, keys_a_.p, flags_.p, s_);
    sort_keys_identity_payload(n);
    launch_pack_sorted(pos3_.p, mass_.p, perm_.p, xyzm_s_.p, n, s_);
    has_tree_ = false;
    check_flags();
    split_and_nodes(with_nodes);
    has_tree_ = true;
}

// development: descents / displacement of the storage-order keys (how sorted the input is)
__global__ void disorder_kernel(const uint64_t* __restrict__ k, size_t n, unsigned long long* out) {
    unsigned long long d = 0, big = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i + 1 < n; i += size_t(gridDim.x) * blockDim.x) {
        d += k[i] > k[i + 1];
        big += (k[i] >> 33) > (k[i + 1] >> 33);  // descent in the top 10 levels
    }
    atomicAdd(&out[0], d);
    atomicAdd(&out[1], big);
}
// development: displacement |k - src[k]| of the new Morton order against the storage order
__global__ void displacement_kernel(const uint32_t* __restrict__ src, size_t n, unsigned long long* out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const long long d = llabs((long long)src[i] - (long long)i);
        const int b = d == 0 ? 0 : min(31, 64 - __clzll((unsigned long long)d));  // bucket: bit length
        atomicAdd(&out[b], 1ull);
    }
}
static void debug_displacement(const uint32_t* src, size_t n, cudaStream_t s) {
    static unsigned long long* buf = nullptr;
    if (!buf) cudaMalloc(&buf, 32 * 8);
    cudaMemsetAsync(buf, 0, 32 * 8, s);
    displacement_kernel<<<148 * 4, 256, 0, s>>>(src, n, buf);
    unsigned long long h[32];
    cudaMemcpyAsync(h, buf, sizeof h, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "[g2 build] displacement bit-length histogram:");
    for (int b = 0; b < 32; ++b)
        if (h[b]) std::fprintf(stderr, " %d:%llu", b, h[b]);
    std::fprintf(stderr, "\n");
}
static void debug_disorder(const uint64_t* k, size_t n, cudaStream_t s) {
    static unsigned long long* buf = nullptr;
    if (!buf) cudaMalloc(&buf, 16);
    cudaMemsetAsync(buf, 0, 16, s);
    disorder_kernel<<<148 * 4, 256, 0, s>>>(k, n, buf);
    unsigned long long h[2];
    cudaMemcpyAsync(h, buf, 16, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "[g2 build] storage-order descents %llu (%.3f%%), top-10-level descents %llu\n", h[0],
                 100.0 * h[0] / double(n), h[1]);
}

// development: G2_PHASE_DEBUG=1 prints device sub-phase times of each rebuild
static bool phase_debug() {
    static const bool on = std::getenv("G2_PHASE_DEBUG") != nullptr;
    return on;
}
static cudaEvent_t dbg_ev[8];
static void dbg_mark(int i, cudaStream_t s) {
    if (!phase_debug()) return;
    if (!dbg_ev[i]) cudaEventCreate(&dbg_ev[i]);
    cudaEventRecord(dbg_ev[i], s);
}

const uint32_t* Engine::rebuild_sorted(const uint32_t* ids, const uint32_t* rank_cur, bool cube_partials,
                                       bool defer_perm) {
    const size_t n = n_;
    dbg_mark(0, s_);
    if (cube_partials)
        launch_bbox_final(bbox_part_.p, predict_blocks(n), cube_.p, s_);
    else
        launch_bbox(xyzm_s_.p, n, bbox_part_.p, cube_.p, flags_.p, s_);
    if (!rank_cur) {
        // keys in storage order sorted with the storage position as payload (no scatter into id
        // order, no rank gather); equal-key runs are then put in original-id order in place.  The
        // storage order is the previous Morton order, so the bucket sort (bucket_sort.cu) normally
        // sorts; the key kernel + onesweep radix sort behind it run only if its gate opened
        static const bool no_bucket = std::getenv("G2_NO_BUCKET_SORT") != nullptr;  // development A/B
        bool alt = false;
        bucket_pending_ =
            !no_bucket && launch_bucket_sort(xyzm_s_.p, n, cube_.p, bucket_, keys_a_.p, vals_a_.p, flags_.p, s_);
        if (!bucket_pending_) {
            launch_keys(xyzm_s_.p, nullptr, n, cube_.p, keys_a_.p, flags_.p, s_);
            if (phase_debug()) debug_disorder(keys_a_.p, n, s_);
            alt = radix_sort_pairs<uint64_t>(keys_a_.p, vals_a_.p, keys_b_.p, vals_b_.p, n, 63, true, sort_, s_);
        }
        dbg_mark(1, s_);
        if (alt) {
            std::swap(keys_a_.p, keys_b_.p);
            std::swap(keys_a_.cap, keys_b_.cap);
        }
        uint32_t* src = alt ? vals_b_.p : vals_a_.p;
        launch_fix_ties(keys_a_.p, src, ids, n, flags_.p, s_);
        if (phase_debug()) debug_displacement(src, n, s_);
        DBuf<uint32_t>& v = alt ? vals_b_ : vals_a_;  // the sort's output becomes src_ (no copy)
        std::swap(src_.p, v.p);
        std::swap(src_.cap, v.cap);
        // perm[k] = original id at new position k (a deferring caller writes it in its state gather)
        if (!defer_perm) launch_gather_u32(ids, src_.p, perm_.p, n, s_);
        rank_valid_ = false;
    } else {
        launch_keys(xyzm_s_.p, ids, n, cube_.p, keys_a_.p, flags_.p, s_);  // keys by original id
        dbg_mark(1, s_);
        sort_keys_identity_payload(n);                                      // perm = original ids in Morton order
        launch_gather_u32(rank_cur, perm_.p, src_.p, n, s_);               // new k <- old position of perm[k]
    }
    dbg_mark(2, s_);
    return src_.p;  // the caller gathers the state (positions included) into the new order
}

void Engine::ensure_rank() {
    if (rank_valid_) return;
    launch_invert_perm(perm_.p, rank_.p, n_, s_);
    rank_valid_ = true;
}

bool Engine::take_bucket_overflow() {
    const bool o = bucket_overflow_;
    bucket_overflow_ = false;
    return o;
}

bool Engine::take_tie_overflow() {
    // the flags were staged with the level sizes at split_and_nodes' synchronisation
    if (!hs_->flags.tie_run) return false;
    hs_->flags.tie_run = 0;
    G2_CUDA(cudaMemsetAsync(&flags_.p->tie_run, 0, sizeof(int), s_));
    return true;
}

void Engine::split_and_nodes(bool with_nodes) {
    const size_t n = n_;
    bool topo_done = false;
    while (true) {
        G2_CUDA(cudaMemsetAsync(level_start_.p, 0, (kMaxDepth + 3) * sizeof(uint32_t), s_));
        G2_CUDA(cudaMemsetAsync(tile_counters_.p, 0, (kMaxDepth + 1) * sizeof(uint32_t), s_));
        G2_CUDA(cudaMemsetAsync(split_status_.p, 0, (cell_cap_ / 32 + 64) * sizeof(uint64_t), s_));
        split_tiles_.reserve(split_tile_words(n));
        SplitArgs a{keys_a_.p,  first_child_.p, child_count_.p, first_.p,
                    count_.p,   depth_.p,       level_start_.p, split_status_.p,
                    tile_counters_.p, uint32_t(cell_cap_), uint32_t(std::min<size_t>(c_.leaf_cap, 0xffffffffu)),
                    flags_.p, split_tiles_.p, leaf_of_.p, int_list_.p, int_count_.p,
                    bucket_pending_ ? bucket_.gate.p : nullptr};
        dbg_mark(3, s_);
        topo_done = launch_split(a, uint32_t(n), s_);
        dbg_mark(4, s_);
        uint32_t* ls = hs_->ls;
        G2_CUDA(cudaMemcpyAsync(ls, level_start_.p, sizeof hs_->ls, cudaMemcpyDeviceToHost, s_));
        if (bucket_pending_)
            G2_CUDA(cudaMemcpyAsync(&hs_->bucket_gate, bucket_.gate.p, sizeof(int), cudaMemcpyDeviceToHost, s_));
        enqueue_flags();
        sync();
        if (bucket_pending_) {
            ++(hs_->bucket_gate ? bucket_fallbacks_ : bucket_sorts_);
            bucket_overflow_ = hs_->bucket_gate != 0;
            bucket_pending_ = false;
        }
        if (phase_debug() && dbg_ev[0]) {
            float t[4] = {0, 0, 0, 0};
            cudaEventElapsedTime(&t[0], dbg_ev[0], dbg_ev[1]);
            cudaEventElapsedTime(&t[1], dbg_ev[1], dbg_ev[2]);
            cudaEventElapsedTime(&t[2], dbg_ev[2], dbg_ev[3]);
            cudaEventElapsedTime(&t[3], dbg_ev[3], dbg_ev[4]);
            std::fprintf(stderr, "[g2 build] bbox+keys %.3f ms  sort %.3f ms  gathers %.3f ms  split %.3f ms\n", t[0],
                         t[1], t[2], t[3]);
        }
        const size_t total = ls[kMaxDepth + 1];
        if (total <= cell_cap_) {
            ncells_ = total;
            std::copy(ls, ls + kMaxDepth + 3, ls_host_);
            max_level_width_ = 0;
            for (int d = 0; d <= kMaxDepth; ++d) max_level_width_ = std::max(max_level_width_, ls[d + 1] - ls[d]);
            break;
        }
        ensure_cells(total + total / 4 + 1024);
    }
    // (a bucket sort over capacity produced a placeholder order: the caller redoes the ordering)
    if (!bucket_overflow_ && !topo_done)
        launch_tree_topology(first_child_.p, child_count_.p, first_.p, count_.p, depth_.p, level_start_.p, ncells_,
                             uint32_t(cell_cap_), leaf_of_.p, int_list_.p, int_count_.p, s_);
    if (with_nodes) calc_nodes();
}

void Engine::calc_nodes(bool overlap) {
    join_calc();
    if (overlap && !side_) {
        G2_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
        G2_CUDA(cudaEventCreateWithFlags(&calc_fork_, cudaEventDisableTiming));
        G2_CUDA(cudaEventCreateWithFlags(&calc_join_, cudaEventDisableTiming));
    }
    launch_calc_node(xyzm_s_.p, n_, child_count_.p, first_.p, count_.p, level_start_.p, ls_host_, leaf_of_.p, int_list_.p,
                     int_count_.p, calc_sync_.p, nodes_.p, nodes32_.p, rel_.p, s_, overlap ? side_ : nullptr,
                     calc_fork_);
    if (overlap) {
        G2_CUDA(cudaEventRecord(calc_join_, side_));
        calc_join_pending_ = true;
    }
}

double Engine::last_walk_kernel_seconds() {
    if (!walk_ev_valid_) return 0.0;
    G2_CUDA(cudaEventSynchronize(walk_ev_[1]));
    float ms = 0.f;
    G2_CUDA(cudaEventElapsedTime(&ms, walk_ev_[0], walk_ev_[1]));
    return ms * 1e-3;
}

void Engine::join_calc() {
    if (!calc_join_pending_) return;
    G2_CUDA(cudaStreamWaitEvent(s_, calc_join_, 0));
    calc_join_pending_ = false;
}

void Engine::refresh(size_t n, const double* mass, const double* pos) {
    if (!has_tree_) throw Error(kDataError, "GravityEngine::refresh: no tree built");
    if (n != n_) throw Error(kDataError, "GravityEngine::refresh: particle count differs from the tree");
    upload_orig(n, mass, pos);
    launch_pack_sorted(pos3_.p, mass_.p, perm_.p, xyzm_s_.p, n, s_);
    calc_nodes();
    check_flags();
}

void Engine::read_events(EventsH& ev) {
    enqueue_events();
    sync();
    events_host(ev);
}
void Engine::events_host(EventsH& ev) const {
    ev.interactions = hs_->events[0], ev.mac_evals = hs_->events[1], ev.list_pushes = hs_->events[2];
}


EventsH Engine::walk(const uint32_t* sinks, const uint32_t* n_sinks_dev, uint32_t n_sinks_cap, const double* amag_s,
                     bool with_pot, bool sync_events, uint32_t group_lo, uint32_t group_hi, bool finalize,
                     int slice_rank, int slice_world, bool combine) {
    EventsH ev;
    if (c_.list_capacity < 1) throw Error(kDataError, "InteractionList: capacity must be >= 1");
    G2_CUDA(cudaMemsetAsync(events_.p, 0, 3 * sizeof(unsigned long long), s_));
    const uint32_t gs = uint32_t(c_.group_size);
    const uint32_t ng_cap = (n_sinks_cap + gs - 1) / gs;
    const size_t cap = c_.frontier_cap ? c_.frontier_cap : 8 * n_;
    const bool check = cap < max_level_width_;
    TreeView tv{xyzm_s_.p, nodes_.p, uint32_t(n_), nodes32_.p, rel_.p, leaf_of_.p};
    WalkBuffers b{};
    b.sinks = sinks;
    b.n_sinks = n_sinks_dev;
    b.groups = groups_.p;
    b.n_groups = n_groups_.p;
    b.accum = accum();
    b.world = peer_world_, b.self = peer_self_;
    {
        // task records: one per donated task (plus the donating initial task); sized from the group
        // count, doubled whenever a walk ran short (a skipped donation keeps results exact but makes
        // the task tree, hence the FP32 summation order, depend on timing)
        // the pool follows the previous walk's use (x1.5); a shortfall doubles it
        ensure_task_pool(std::max<size_t>(grow_pool_ ? 2 * rec_cap_ : 0, size_t(hs_->recs) * 3 / 2));
        grow_pool_ = false;
        b.trec = trec_.p, b.tacc = tacc_.p, b.batch_rec = batch_rec_.p;
        b.rec_cap = uint32_t(std::min<size_t>(rec_cap_, 0xffffffffu));
    }
    if (peer_world_ > 1) {
        gcost_.reserve(ng_cap + 1);
        b.gcost = gcost_.p;
        for (int q = 0; q < kMaxPeers; ++q) b.peer_accum[q] = peer_accum_[q], b.peer_cost[q] = peer_cost_[q];
        // shards computed on the device (no host round trip): cost-balanced when a cost history is
        // given, else equal group counts
        shard_.reserve(2);
        b.shard = shard_.p;
        if (peer_cost_[peer_self_] && ng_cur_) b.cost_prev = cost_prev_, b.ng_prev = ng_prev_, b.ng_cur = ng_cur_;
    }
    b.events = events_.p;
    b.queue = queue_.p;
    b.batch = batch_.p;
    b.queue_cap = queue_cap_;
    b.ring_bits = ring_bits_;
    b.qstate = qstate_.p;
    b.spill = spill_.p;
    b.group_lo = group_lo;
    b.group_hi = group_hi;
    if (check) {
        level_count_.reserve(size_t(ng_cap) * (kMaxDepth + 1));
        G2_CUDA(cudaMemsetAsync(level_count_.p, 0, size_t(ng_cap) * (kMaxDepth + 1) * 4, s_));
        b.level_count = level_count_.p;
    }
    b.group_inter = group_inter_.p;
    static const bool no_order = std::getenv("G2_NO_ORDER") != nullptr;  // development A/B
    if (!no_order) {
        order_.reserve(ng_cap + 1);  // no-op unless targets with duplicates outnumber the particles
        order_scratch_.reserve(walk_order_scratch_words(ng_cap));
        b.order = order_.p, b.order_scratch = order_scratch_.p;
    }
    static const char* trace_path = std::getenv("G2_WALK_TRACE");  // development: per-task timeline
    if (trace_path) {
        trace_.reserve(2 * (size_t(1) << 23));
        trace_n_.reserve(1);
        G2_CUDA(cudaMemsetAsync(trace_n_.p, 0, 4, s_));
        b.trace = trace_.p, b.trace_n = trace_n_.p, b.trace_cap = 1u << 23;
    }
    b.heavy = heavy_.p, b.sliced = sliced_.p;
    b.slice_base = uint32_t(walk_slice_base(n_));
    b.slice_world = std::max(1, slice_world), b.slice_rank = slice_rank;
    G2_CUDA(cudaMemsetAsync(heavy_.p, 0, sizeof(uint32_t), s_));
    G2_CUDA(cudaMemsetAsync(group_inter_.p, 0, size_t(ng_cap) * 8, s_));
    // the group spheres, shards and accumulator clearing read no node: they may overlap calc_node's
    // internal levels (calc_nodes(true)), joined before the first kernel that reads the tree
    launch_groups(tv, amag_s, b, gs, n_sinks_cap, s_);
    launch_walk_prep(b, n_sinks_cap, gs, s_);
    join_calc();
    WalkParams wp{p_.G, p_.eps, p_.dacc, c_.bootstrap_theta, uint32_t(std::min<size_t>(cap, 0xffffffffu)),
                  c_.count_ops ? 1 : 0, 0};
    wp.mass_max = mass_max_;
    // tighter dacc means more work per group, none of which needs splitting finer than before:
    // the donation trigger grows as (2^-9 / dacc)^(1/3), x1 .. x8 (a function of dacc only, so every
    // rank and every run uses the same one)
    {
        const double f = std::clamp(std::cbrt(0.001953125 / p_.dacc), 1.0, 8.0);
        wp.donate_pushes = uint32_t(wp.donate_pushes * f), wp.donate_few = uint32_t(wp.donate_few * f);
    }
    static const char* dp = std::getenv("G2_DONATE_PUSHES");  // development: donation-trigger sweeps
    static const char* df = std::getenv("G2_DONATE_FEW");
    if (dp) wp.donate_pushes = uint32_t(std::max(1, std::atoi(dp)));
    if (df) wp.donate_few = uint32_t(std::max(1, std::atoi(df)));
    static const char* dsc = std::getenv("G2_DONATE_SCALE");
    if (dsc) wp.donate_scale = uint32_t(std::max(1, std::atoi(dsc)));
    if (!walk_ev_[0])
        for (auto& e : walk_ev_) G2_CUDA(cudaEventCreate(&e));
    launch_walk(tv, wp, b, with_pot, n_sinks_cap, gs, flags_.p, s_, walk_ev_, false);
    walk_ev_valid_ = true;
    if (check)
        G2_COUNT(1), frontier_check_kernel<<<gridn(size_t(ng_cap) * (kMaxDepth + 1)), kB, 0, s_>>>(
            level_count_.p, size_t(ng_cap) * (kMaxDepth + 1), uint32_t(std::min<size_t>(cap, 0xffffffffu)),
            flags_.p);
    last_walk_ = b;
    walk_G_ = p_.G;
    if (combine) combine_slices(slice_region(), 0, 1);
    if (finalize) launch_walk_finalize(b, n_sinks_cap, ax_s_.p, ay_s_.p, az_s_.p, with_pot ? pot_s_.p : nullptr, s_);
    if (trace_path) {
        uint32_t nt = 0;
        G2_CUDA(cudaMemcpyAsync(&nt, trace_n_.p, 4, cudaMemcpyDeviceToHost, s_));
        G2_CUDA(cudaStreamSynchronize(s_));
        nt = std::min(nt, 1u << 23);
        std::vector<uint4> h(2 * size_t(nt));
        G2_CUDA(cudaMemcpy(h.data(), trace_.p, h.size() * sizeof(uint4), cudaMemcpyDeviceToHost));
        if (FILE* f = std::fopen(trace_path, "wb")) {
            std::fwrite(h.data(), sizeof(uint4), h.size(), f);
            std::fclose(f);
        }
    }
    if (sync_events) read_events(ev);
    return ev;
}

void Engine::combine_slices(const float4* src, size_t stride, int world) {
    TreeView tv{xyzm_s_.p, nodes_.p, uint32_t(n_), nodes32_.p, rel_.p, leaf_of_.p};
    WalkBuffers b = last_walk_;
    b.accum = accum();
    uint32_t* cost = peer_world_ > 1 && peer_cost_[peer_self_] ? peer_cost_[peer_self_] : nullptr;
    launch_walk_combine(b, tv, src, stride, world, walk_G_, cost, s_);
}

void Exchange::slice_source(Simulation& sim, const float4*& src, size_t& stride) {
    src = sim.engine().slice_region();
    stride = 0;
}

EventsH Engine::evaluate(size_t n, const double* mass, const double* pos, const double* acc_old_mag,
                         size_t n_targets, const uint32_t* targets, double* acc_out, double* pot_out) {
    if (!has_tree_) throw Error(kDataError, "GravityEngine::evaluate: no tree built");
    if (n != n_) throw Error(kDataError, "GravityEngine::evaluate: particle count differs from the tree");
    if (targets && n_targets == 0) return {};
    ensure_rank();
    const size_t nt = targets ? n_targets : n;
    if (targets)
        for (size_t j = 0; j < nt; ++j)
            if (targets[j] >= n) throw Error(kDataError, "GravityEngine::evaluate: target index out of range");
    upload_orig(n, mass, pos);
    launch_pack_sorted(pos3_.p, mass_.p, perm_.p, xyzm_s_.p, n, s_);
    // leaf particles at the positions given here, node attributes of the last build/refresh
    launch_leaf_rel(xyzm_s_.p, child_count_.p, first_.p, count_.p, nodes32_.p, uint32_t(ncells_), rel_.p, s_);
    G2_CUDA(cudaMemcpyAsync(amag_o_.p, acc_old_mag, n * sizeof(double), cudaMemcpyHostToDevice, s_));
    launch_gather_f64(amag_o_.p, perm_.p, amag_s_.p, n, s_);
    const uint32_t* out_idx;
    if (targets) {
        // sinks = ranks of the targets, sorted (engine.cpp:39-41); duplicates kept
        G2_CUDA(cudaMemcpyAsync(vals_b_.p, targets, nt * 4, cudaMemcpyHostToDevice, s_));
        launch_gather_u32(rank_.p, vals_b_.p, tgt_rank_.p, nt, s_);
        G2_CUDA(cudaMemcpyAsync(sinks_.p, tgt_rank_.p, nt * 4, cudaMemcpyDeviceToDevice, s_));
        int bits = 1;
        while ((size_t(1) << bits) < n) ++bits;
        const bool alt = radix_sort_pairs<uint32_t>(sinks_.p, vals_a_.p, sinks_alt_.p, vals_b_.p, nt, bits, true,
                                                    sort_, s_);
        if (alt) G2_CUDA(cudaMemcpyAsync(sinks_.p, sinks_alt_.p, nt * 4, cudaMemcpyDeviceToDevice, s_));
        out_idx = tgt_rank_.p;
    } else {
        launch_iota(sinks_.p, n, s_);
        out_idx = rank_.p;
    }
    const uint32_t nt32 = uint32_t(nt);
    G2_CUDA(cudaMemcpyAsync(n_sinks_.p, &nt32, 4, cudaMemcpyHostToDevice, s_));
    // a walk whose task-record pool ran short skipped donations (results exact, but the task tree --
    // hence the FP32 summation order -- then depends on timing): walk again with the grown pool
    EventsH ev = walk(sinks_.p, n_sinks_.p, nt32, amag_s_.p, pot_out != nullptr, false);
    while (walk_pool_overflow()) ev = walk(sinks_.p, n_sinks_.p, nt32, amag_s_.p, pot_out != nullptr, false);
    // results for the targets in target order
    G2_COUNT(1), interleave_kernel<<<gridn(nt), kB, 0, s_>>>(ax_s_.p, ay_s_.p, az_s_.p, out_idx, out_.p, nt);
    std::vector<double> acc(3 * nt), pot(pot_out ? nt : 0);
    G2_CUDA(cudaMemcpyAsync(acc.data(), out_.p, 3 * nt * sizeof(double), cudaMemcpyDeviceToHost, s_));
    if (pot_out) {
        G2_COUNT(1), gather_scalar_kernel<<<gridn(nt), kB, 0, s_>>>(pot_s_.p, out_idx, amag_o_.p, nt);
        G2_CUDA(cudaMemcpyAsync(pot.data(), amag_o_.p, nt * sizeof(double), cudaMemcpyDeviceToHost, s_));
    }
    read_events(ev);
    check_flags();
    for (size_t j = 0; j < nt; ++j) {
        const size_t id = targets ? targets[j] : j;
        acc_out[3 * id] = acc[3 * j], acc_out[3 * id + 1] = acc[3 * j + 1], acc_out[3 * id + 2] = acc[3 * j + 2];
        if (pot_out) pot_out[id] = pot[j];
    }
    return ev;
}

void Engine::direct_sum_orig(const double4* xyzm_orig, size_t n, double* ax, double* ay, double* az) {
    launch_direct_sum(xyzm_orig, n, p_.G, p_.eps, ax, ay, az, flags_.p, s_);
}

EventsH Engine::bootstrap(size_t n, const double* mass, const double* pos, double* acc_out, double* acc_old_mag_io) {
    EventsH ev;
    if (n <= c_.bootstrap_direct_limit) {  // engine.cpp:91-94
        if (n < 1) throw Error(kDataError, "direct_sum: empty system");
        reserve(n);
        upload_orig(n, mass, pos);
        launch_pack_identity(pos3_.p, mass_.p, xyzm_o_.p, n, s_);
        direct_sum_orig(xyzm_o_.p, n, ax_s_.p, ay_s_.p, az_s_.p);
        ev.interactions = uint64_t(n) * (n - 1);
        G2_COUNT(1), interleave_kernel<<<gridn(n), kB, 0, s_>>>(ax_s_.p, ay_s_.p, az_s_.p, nullptr, out_.p, n);
        launch_norm3(ax_s_.p, ay_s_.p, az_s_.p, amag_o_.p, n, s_);
        G2_CUDA(cudaMemcpyAsync(acc_out, out_.p, 3 * n * sizeof(double), cudaMemcpyDeviceToHost, s_));
        G2_CUDA(cudaMemcpyAsync(acc_old_mag_io, amag_o_.p, n * sizeof(double), cudaMemcpyDeviceToHost, s_));
        check_flags();
        return ev;
    }
    if (!has_tree_) build(n, mass, pos, true);
    ev = evaluate(n, mass, pos, acc_old_mag_io, 0, nullptr, acc_out, nullptr);
    for (size_t i = 0; i < n; ++i) {
        const double x = acc_out[3 * i], y = acc_out[3 * i + 1], z = acc_out[3 * i + 2];
        acc_old_mag_io[i] = std::sqrt(x * x + y * y + z * z);
    }
    return ev;
}

void Engine::get_tree(double* bbox4, uint64_t* keys, uint32_t* perm, uint32_t* rank, uint32_t* cells4,
                      uint8_t* depth, double* nodes5) {
    if (!has_tree_) throw Error(kDataError, "get_tree: no tree built");
    const size_t n = n_, nc = ncells_;
    ensure_rank();
    if (bbox4) G2_CUDA(cudaMemcpyAsync(bbox4, cube_.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, s_));
    if (keys) G2_CUDA(cudaMemcpyAsync(keys, keys_a_.p, n * 8, cudaMemcpyDeviceToHost, s_));
    if (perm) G2_CUDA(cudaMemcpyAsync(perm, perm_.p, n * 4, cudaMemcpyDeviceToHost, s_));
    if (rank) G2_CUDA(cudaMemcpyAsync(rank, rank_.p, n * 4, cudaMemcpyDeviceToHost, s_));
    std::vector<uint32_t> fc(nc), cc(nc), f(nc), c(nc);
    std::vector<WNode> nd(nodes5 ? nc : 0);
    G2_CUDA(cudaMemcpyAsync(fc.data(), first_child_.p, nc * 4, cudaMemcpyDeviceToHost, s_));
    G2_CUDA(cudaMemcpyAsync(cc.data(), child_count_.p, nc * 4, cudaMemcpyDeviceToHost, s_));
    G2_CUDA(cudaMemcpyAsync(f.data(), first_.p, nc * 4, cudaMemcpyDeviceToHost, s_));
    G2_CUDA(cudaMemcpyAsync(c.data(), count_.p, nc * 4, cudaMemcpyDeviceToHost, s_));
    if (depth) G2_CUDA(cudaMemcpyAsync(depth, depth_.p, nc, cudaMemcpyDeviceToHost, s_));
    if (nodes5) G2_CUDA(cudaMemcpyAsync(nd.data(), nodes_.p, nc * sizeof(WNode), cudaMemcpyDeviceToHost, s_));
    G2_CUDA(cudaStreamSynchronize(s_));
    for (size_t i = 0; i < nc; ++i) {
        if (cells4) cells4[4 * i] = fc[i], cells4[4 * i + 1] = cc[i], cells4[4 * i + 2] = f[i], cells4[4 * i + 3] = c[i];
        if (nodes5) {
            nodes5[5 * i] = nd[i].mass;
            nodes5[5 * i + 1] = nd[i].cx, nodes5[5 * i + 2] = nd[i].cy, nodes5[5 * i + 3] = nd[i].cz;
            nodes5[5 * i + 4] = nd[i].extent;
        }
    }
}

// =============================================================================================
RebuildTuner::RebuildTuner(TunerConfigH c) : c_(c), interval_(c.initial_interval) {
    if (c_.min_interval < 1 || c_.max_interval < c_.min_interval)
        throw Error(kDataError, "RebuildTuner: bad interval bounds");
    interval_ = std::clamp(interval_, c_.min_interval, c_.max_interval);
}
void RebuildTuner::set_interval(size_t i) { interval_ = std::clamp(i, c_.min_interval, c_.max_interval); }
void RebuildTuner::on_rebuild() {
    const size_t fit = autotune();
    interval_ = std::clamp((interval_ + fit + 1) / 2, c_.min_interval, c_.max_interval);
    hist_.clear();
    steps_ = 0;
}
size_t RebuildTuner::autotune() const {
    if (hist_.size() < 2) return interval_;
    std::vector<double> slopes;
    for (size_t j = 1; j < hist_.size(); ++j)
        for (size_t i = 0; i < j; ++i) slopes.push_back((hist_[j] - hist_[i]) / double(j - i));
    std::nth_element(slopes.begin(), slopes.begin() + slopes.size() / 2, slopes.end());
    double slope = std::max(0.0, slopes[slopes.size() / 2]);
    std::vector<double> res(hist_.size());
    for (size_t k = 0; k < hist_.size(); ++k) res[k] = hist_[k] - slope * double(k);
    std::nth_element(res.begin(), res.begin() + res.size() / 2, res.end());
    const double intercept = res[res.size() / 2];
    size_t best_m = c_.min_interval;
    double best = 0.0;
    for (size_t m = c_.min_interval; m <= c_.max_interval; ++m) {
        const double md = double(m);
        const double cost = build_time_ / md + intercept + slope * (md - 1.0) / 2.0;
        if (m == c_.min_interval || cost <= best) best = cost, best_m = m;
    }
    return best_m;
}

// =============================================================================================
Simulation::Simulation(size_t n, const double* mass, const double* pos, const double* vel, GravParamsH p,
                       StepSchemeH sc, EngineConfigH ec, TunerConfigH tc, int device)
    : eng_(p, ec, device), p_(p), sc_(sc), tuner_(tc), n_(n) {
    if (!(sc_.dt_max > 0.0)) throw Error(kDataError, "Simulation: dt_max must be positive");
    if (!(sc_.eta > 0.0)) throw Error(kDataError, "Simulation: eta must be positive");
    if (n < 1) throw Error(kDataError, "Simulation: empty system");
    for (size_t i = 0; i < n; ++i) {  // ParticleSystem::validate (octree.cpp:14-22)
        if (!(mass[i] > 0.0) || !std::isfinite(mass[i]))
            throw Error(kDataError, "particle system: non-positive or non-finite mass");
        for (int a = 0; a < 3; ++a)
            if (!std::isfinite(pos[3 * i + a]) || !std::isfinite(vel[3 * i + a]))
                throw Error(kDataError, "particle system: non-finite state");
    }
    tick_ = sc_.dt_max / double(uint64_t(1) << kMaxBlockLevel);
    eng_.note_masses(n, mass);
    eng_.reserve(n);
    eng_.set_n(n);
    cudaStream_t s = eng_.stream();
    for (auto* b : {&vx_, &vy_, &vz_, &ax_, &ay_, &az_, &amag_, &vx2_, &vy2_, &vz2_, &ax2_, &ay2_, &az2_, &amag2_})
        b->reserve(n);
    level_.reserve(n), level2_.reserve(n), active_.reserve(n), active2_.reserve(n);
    last_.reserve(n), last2_.reserve(n);
    ids_.reserve(n), ids2_.reserve(n), rank_cur_.reserve(n), sinks_.reserve(n), n_active_.reserve(1);
    compact_ctr_.reserve(1);
    compact_status_.reserve(n / 4096 + 8);
    t_next_.reserve(1);
    // state in original order until the first build
    DBuf<double> tmp3, tmpm;
    tmp3.reserve(3 * n), tmpm.reserve(n);
    G2_CUDA(cudaMemcpyAsync(tmp3.p, pos, 3 * n * 8, cudaMemcpyHostToDevice, s));
    G2_CUDA(cudaMemcpyAsync(tmpm.p, mass, n * 8, cudaMemcpyHostToDevice, s));
    launch_pack_identity(tmp3.p, tmpm.p, eng_.xyzm_s(), n, s);
    G2_CUDA(cudaMemcpyAsync(tmp3.p, vel, 3 * n * 8, cudaMemcpyHostToDevice, s));
    G2_COUNT(1), deinterleave_kernel<<<gridn(n), kB, 0, s>>>(tmp3.p, nullptr, vx_.p, vy_.p, vz_.p, n);
    for (auto* b : {&ax_, &ay_, &az_, &amag_}) G2_CUDA(cudaMemsetAsync(b->p, 0, n * 8, s));
    G2_CUDA(cudaMemsetAsync(level_.p, 0, n, s));
    G2_CUDA(cudaMemsetAsync(last_.p, 0, n * 8, s));
    launch_iota(ids_.p, n, s);
    launch_iota(rank_cur_.p, n, s);
    G2_CUDA(cudaStreamSynchronize(s));
    for (auto& e : ev_) G2_CUDA(cudaEventCreate(&e));
}

StepState Simulation::state() {
    return StepState{eng_.xyzm_s(), vx_.p, vy_.p, vz_.p, ax_.p, ay_.p, az_.p, amag_.p, level_.p, last_.p};
}

void Simulation::reorder(const uint32_t* src, uint32_t* perm_out) {
    cudaStream_t s = eng_.stream();
    const size_t n = n_;
    DBuf<double>* pairs[][2] = {{&vx_, &vx2_}, {&vy_, &vy2_}, {&vz_, &vz2_}, {&ax_, &ax2_},
                                {&ay_, &ay2_}, {&az_, &az2_}, {&amag_, &amag2_}};
    ReorderArgs r;
    r.xin = eng_.xyzm_s(), r.xout = eng_.xyzm_alt();
    for (int k = 0; k < 7; ++k) r.in[k] = pairs[k][0]->p, r.out[k] = pairs[k][1]->p;
    r.lin = level_.p, r.lout = level2_.p, r.ain = active_.p, r.aout = active2_.p, r.tin = last_.p, r.tout = last2_.p;
    r.iin = ids_.p, r.iout = ids2_.p, r.iout2 = perm_out;  // ids[src[k]] == the engine's perm[k]
    G2_COUNT(1), launch_pdl(reorder_kernel, dim3(gridn(n)), dim3(kB), size_t(0), s, r, src, n);  // one pass over the index for all state
    for (auto& pr : pairs) std::swap(pr[0]->p, pr[1]->p);
    eng_.swap_xyzm();
    std::swap(level_.p, level2_.p);
    std::swap(active_.p, active2_.p);
    std::swap(last_.p, last2_.p);
    std::swap(ids_.p, ids2_.p);
    rank_cur_valid_ = false;  // original id -> position: rebuilt on demand (API boundary only)
}

const uint32_t* Simulation::rank_cur() {
    if (!rank_cur_valid_) {
        launch_invert_perm(ids_.p, rank_cur_.p, n_, eng_.stream());
        rank_cur_valid_ = true;
    }
    return rank_cur_.p;
}

void Simulation::rebuild_order(bool cube_partials) {
    const uint32_t* src = eng_.rebuild_sorted(ids_.p, nullptr, cube_partials, true);
    reorder(src, eng_.perm());
    eng_.split_and_nodes(false);  // syncs once to size the levels
    // a bucket over capacity (its output was the identity order: the state is unchanged) or a long
    // run of equal keys: redo the ordering with the (key, original id) sort
    const bool bucket_overflow = eng_.take_bucket_overflow();
    if (eng_.take_tie_overflow() || bucket_overflow) {
        src = eng_.rebuild_sorted(ids_.p, rank_cur());
        reorder(src);
        eng_.split_and_nodes(false);
    }
    eng_.mark_tree(true);
}

double Simulation::elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    G2_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms * 1e-3;
}

void Simulation::init() {
    cudaStream_t s = eng_.stream();
    const size_t n = n_;
    const EngineConfigH& c = eng_.config();
    if (n <= c.bootstrap_direct_limit) {  // engine.cpp:91-94: state is still in original order
        eng_.direct_sum_orig(eng_.xyzm_s(), n, ax_.p, ay_.p, az_.p);
    } else {
        rebuild_order();
        eng_.calc_nodes();
        launch_iota(sinks_.p, n, s);
        const uint32_t n32 = uint32_t(n);
        G2_CUDA(cudaMemcpyAsync(n_active_.p, &n32, 4, cudaMemcpyHostToDevice, s));
        eng_.walk(sinks_.p, n_active_.p, uint32_t(n), amag_.p, false, false);  // amag == 0: geometric MAC
        while (eng_.walk_pool_overflow()) eng_.walk(sinks_.p, n_active_.p, uint32_t(n), amag_.p, false, false);
        G2_CUDA(cudaMemcpyAsync(ax_.p, eng_.ax_s(), n * 8, cudaMemcpyDeviceToDevice, s));
        G2_CUDA(cudaMemcpyAsync(ay_.p, eng_.ay_s(), n * 8, cudaMemcpyDeviceToDevice, s));
        G2_CUDA(cudaMemcpyAsync(az_.p, eng_.az_s(), n * 8, cudaMemcpyDeviceToDevice, s));
    }
    launch_norm3(ax_.p, ay_.p, az_.p, amag_.p, n, s);
    SchemeDev sd{sc_.eta, sc_.dt_max, p_.eps, sc_.adaptive ? 1 : 0, sc_.fixed_level};
    if (sc_.adaptive)
        launch_assign_levels(state(), n, sd, s);
    else
        G2_COUNT(1), fill_u8_kernel<<<gridn(n), kB, 0, s>>>(level_.p, uint8_t(std::clamp(sc_.fixed_level, 0, kMaxBlockLevel)), n);
    eng_.check_flags();
    initialized_ = true;
}

StepResultH Simulation::step() {
    if (!initialized_) throw Error(kDataError, "Simulation::step: init() not called");
    const auto t0 = std::chrono::steady_clock::now();
    cudaStream_t s = eng_.stream();
    const size_t n = n_;
    StepResultH r;
    StepState st = state();
    SchemeDev sd{sc_.eta, sc_.dt_max, p_.eps, sc_.adaptive ? 1 : 0, sc_.fixed_level};

    G2_CUDA(cudaEventRecord(ev_[0], s));
    launch_tnext(st, n, t_next_.p, s);
    const bool rebuild = !eng_.has_tree() || rebuild_every_step_ || tuner_.should_rebuild();
    // a rebuilding step's predict also reduces the bounding-cube partials (no separate pass)
    launch_predict(st, n, t_next_.p, now_, tick_, active_.p, s, rebuild ? eng_.bbox_partials() : nullptr,
                   eng_.dev_flags());
    G2_CUDA(cudaEventRecord(ev_[1], s));

    if (rebuild) {
        if (autotune_)
            tuner_.on_rebuild();
        else
            tuner_.reset_cycle();
        rebuild_order(true);
        G2_CUDA(cudaEventRecord(ev_[2], s));
        eng_.calc_nodes(phase_overlap_);
        G2_CUDA(cudaEventRecord(ev_[3], eng_.calc_tail_stream()));
    } else {
        G2_CUDA(cudaEventRecord(ev_[2], s));
        eng_.calc_nodes(phase_overlap_);  // internal levels beside the compaction and the group spheres
        G2_CUDA(cudaEventRecord(ev_[3], eng_.calc_tail_stream()));
    }
    st = state();
    // active set in (new) Morton order == reference's rank-sorted targets (engine.cpp:39-41)
    launch_compact(active_.p, n, sinks_.p, n_active_.p, compact_status_.p, compact_ctr_.p, s);
    uint32_t lo = 0, hi = ~0u;
    if (exchange_) {
        // contiguous equal shard of the groups (cost-balanced sharding: see DESIGN.md)
        uint32_t na = 0;
        if (!exchange_ || !exchange_->device_shards()) {  // host-side equal shards (copy / NCCL meshes)
            HostSync* hs = eng_.host_sync();
            G2_CUDA(cudaMemcpyAsync(&hs->na, n_active_.p, 4, cudaMemcpyDeviceToHost, s));
            G2_CUDA(cudaStreamSynchronize(s));
            na = hs->na;
        }
        const uint32_t gs = uint32_t(eng_.config().group_size);
        const uint32_t ng = (na + gs - 1) / gs;
        equal_shard(ng, rank_, world_, lo, hi);
    }
    shard_lo_ = lo, shard_hi_ = hi;
    const bool sharded = exchange_ != nullptr;  // a mesh (a one-rank NCCL mesh included)
    if (sharded) exchange_->before_walk(*this);
    eng_.walk(sinks_.p, n_active_.p, uint32_t(n), amag_.p, false, false, lo, hi, false, sharded ? rank_ : 0,
              sharded ? world_ : 1, !sharded);
    G2_CUDA(cudaEventRecord(ev_[4], s));
    if (sharded) {
        exchange_->allgather_acc(*this);  // every rank receives every group's accelerations
        const float4* src = nullptr;      // and every slice of the whole-system groups
        size_t stride = 0;
        exchange_->slice_source(*this, src, stride);
        eng_.combine_slices(src, stride, world_);
    }
    G2_CUDA(cudaEventRecord(ev_[5], s));
    launch_correct(st, sinks_.p, n_active_.p, uint32_t(n), eng_.accum(), t_next_.p, now_, tick_, sd, s);
    if (sharded) eng_.set_peer_push(1, 0, nullptr, nullptr);  // other walks (init, evaluate) stay local
    G2_CUDA(cudaEventRecord(ev_[6], s));

    HostSync* hs = eng_.host_sync();
    G2_CUDA(cudaMemcpyAsync(&hs->tnext, t_next_.p, 8, cudaMemcpyDeviceToHost, s));
    G2_CUDA(cudaMemcpyAsync(&hs->na, n_active_.p, 4, cudaMemcpyDeviceToHost, s));
    eng_.enqueue_events();
    eng_.enqueue_flags();
    eng_.sync();
    eng_.raise_flags();
    eng_.events_host(r.events);
    const unsigned long long tn = hs->tnext;
    const uint32_t na = hs->na;
    r.timings.predict = elapsed(ev_[0], ev_[1]);
    if (rebuild) {
        r.timings.make_tree = elapsed(ev_[1], ev_[2]);
        r.rebuilt = true;
    }
    r.timings.calc_node = elapsed(ev_[2], ev_[3]);
    r.timings.walk_tree = elapsed(ev_[3], ev_[4]);
    r.timings.correct = elapsed(ev_[5], ev_[6]);
    double tw = r.timings.walk_tree, tb = r.timings.make_tree + r.timings.calc_node;
    const bool model = model_rate_ > 0.0;
    if (model) {
        tw = (27.0 * double(r.events.interactions) + 5.0 * double(r.events.mac_evals)) / model_rate_;
        tb = model_build_ * double(n);
    }
    // every rank must take the same rebuild decisions: identical tuner inputs
    if (exchange_ && autotune_ && !rebuild_every_step_) exchange_->agree_times(*this, tw, tb, model);
    tuner_.record_walk(tw);
    if (rebuild) tuner_.record_build(tb);
    last_active_ = na;
    r.active = na;
    now_ = tn;
    time_ = double(now_) * tick_;
    r.rebuild_interval = tuner_.interval();
    r.wall_seconds = seconds(t0);
    return r;
}

void Simulation::get_state(double* pos, double* vel, double* acc, double* acc_old_mag, uint8_t* level,
                           double* time) {
    // gathers into the caller's (original) particle order on the device, then one
    // D2H per array straight into the caller's buffer (pinned buffers stream at full speed)
    cudaStream_t s = eng_.stream();
    const size_t n = n_;
    io_.reserve(3 * n);
    const uint32_t* at = rank_cur();  // original id -> current position
    if (pos) {
        G2_COUNT(1), xyzm_to_pos3_kernel<<<gridn(n), kB, 0, s>>>(eng_.xyzm_s(), at, io_.p, n);
        G2_CUDA(cudaMemcpyAsync(pos, io_.p, 3 * n * 8, cudaMemcpyDeviceToHost, s));
        G2_CUDA(cudaStreamSynchronize(s));
    }
    auto fetch3 = [&](const double* x, const double* y, const double* z, double* out) {
        G2_COUNT(1), interleave_kernel<<<gridn(n), kB, 0, s>>>(x, y, z, at, io_.p, n);
        G2_CUDA(cudaMemcpyAsync(out, io_.p, 3 * n * 8, cudaMemcpyDeviceToHost, s));
        G2_CUDA(cudaStreamSynchronize(s));
    };
    if (vel) fetch3(vx_.p, vy_.p, vz_.p, vel);
    if (acc) fetch3(ax_.p, ay_.p, az_.p, acc);
    if (acc_old_mag) {
        G2_COUNT(1), gather_scalar_kernel<<<gridn(n), kB, 0, s>>>(amag_.p, at, io_.p, n);
        G2_CUDA(cudaMemcpyAsync(acc_old_mag, io_.p, n * 8, cudaMemcpyDeviceToHost, s));
        G2_CUDA(cudaStreamSynchronize(s));
    }
    if (level) {
        launch_gather_u8(level_.p, at, reinterpret_cast<uint8_t*>(io_.p), n, s);
        G2_COUNT(1);
        G2_CUDA(cudaMemcpyAsync(level, io_.p, n, cudaMemcpyDeviceToHost, s));
        G2_CUDA(cudaStreamSynchronize(s));
    }
    if (time) *time = time_;
}

__global__ void xyzm_to_mass_kernel(const double4* __restrict__ xyzm, const uint32_t* __restrict__ idx, double* mass,
                                    size_t n) {
    for (size_t j = blockIdx.x * size_t(kB) + threadIdx.x; j < n; j += size_t(gridDim.x) * kB) mass[j] = xyzm[idx[j]].w;
}

void Simulation::get_mass(double* mass) {
    cudaStream_t s = eng_.stream();
    io_.reserve(3 * n_);
    G2_COUNT(1), xyzm_to_mass_kernel<<<gridn(n_), kB, 0, s>>>(eng_.xyzm_s(), rank_cur(), io_.p, n_);
    G2_CUDA(cudaMemcpyAsync(mass, io_.p, n_ * 8, cudaMemcpyDeviceToHost, s));
    G2_CUDA(cudaStreamSynchronize(s));
}

void Simulation::set_state(const double* pos, const double* vel) {
    cudaStream_t s = eng_.stream();
    const size_t n = n_;
    io_.reserve(3 * n);
    io2_.reserve(3 * n);
    // both uploads back to back (one copy direction: no kernel bubble between them), then the scatters
    if (pos) G2_CUDA(cudaMemcpyAsync(io_.p, pos, 3 * n * 8, cudaMemcpyHostToDevice, s));
    if (vel) G2_CUDA(cudaMemcpyAsync(io2_.p, vel, 3 * n * 8, cudaMemcpyHostToDevice, s));
    if (pos) G2_COUNT(1), set_pos_kernel<<<gridn(n), kB, 0, s>>>(eng_.xyzm_s(), io_.p, ids_.p, n);
    if (vel) G2_COUNT(1), deinterleave_kernel<<<gridn(n), kB, 0, s>>>(io2_.p, ids_.p, vx_.p, vy_.p, vz_.p, n);
    G2_CUDA(cudaStreamSynchronize(s));
}

}  // namespace g2
