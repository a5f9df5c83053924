// Kernel-launch entry points shared between the .cu translation units.
#pragma once

#include "common.cuh"

namespace g2 {

// Root cube (vec3.hpp:53-63) as computed by bounding_cube (octree.cpp:24-49).
struct Cube {
    double cx, cy, cz, half;
};

// Sink group (traversal.hpp:49-54): AABB centre, radius, a_min of its members,
// which are sinks[first, first + count) (sorted particle indices).
struct alignas(16) GroupRec {
    double cx, cy, cz, radius, a_min;
    uint32_t first, count;
};

// Device view of the octree.  Particle arrays are in Morton (rank) order of
// the last build; xyzm packs position and mass.
struct TreeView {
    const double4* xyzm;   // [n] sorted
    const WNode* nodes;    // [ncells]
    uint32_t n;
    const WNode32* nodes32;  // [ncells] compact walk records
    const float4* rel;       // [n] leaf-relative positions + mass (sorted order)
    const uint32_t* leaf_of; // [n] leaf cell of each particle
};

// ---- tree.cu -----------------------------------------------------------------
// bbox partials -> cube; then keys in ORIGINAL index order (key_by_id[id]).
void launch_bbox(const double4* xyzm, size_t n, double* partials, Cube* cube, DevFlags* flags, cudaStream_t s);
void launch_bbox_final(const double* partials, unsigned nb, Cube* cube, cudaStream_t s);
// key of the particle stored at position i goes to key_by_id[id_of_pos[i]] (nullptr: identity)
void launch_keys(const double4* xyzm, const uint32_t* id_of_pos, size_t n, const Cube* cube, uint64_t* key_by_id,
                 DevFlags* flags, cudaStream_t s);

struct SplitArgs {
    const uint64_t* keys;     // sorted
    uint32_t* first_child;
    uint32_t* child_count;
    uint32_t* first;
    uint32_t* count;
    uint8_t* depth;
    uint32_t* level_start;    // [kMaxDepth + 3]
    uint64_t* status;         // look-back words, zeroed
    uint32_t* tile_counters;  // [kMaxDepth + 1], zeroed
    uint32_t cell_cap;
    uint32_t leaf_cap;
    DevFlags* flags;
    uint32_t* tiles;          // split_tile_words(n) scratch for the non-recursive split (nullable)
    // topology outputs (see launch_tree_topology), written by the non-recursive split's last pass
    uint32_t* leaf_of;
    uint4* int_list;
    uint32_t* int_count;
    const int* topo_gate;     // nullable: a set word means a placeholder order (no topology written)
};
size_t split_tile_words(size_t n);
// returns true when the split also wrote the topology outputs (leaf_of, int_list, int_count)
bool launch_split(const SplitArgs& a, uint32_t n, cudaStream_t s);

// Per topology (after every split): leaf_of (the leaf cell of every particle) and the internal cells
// of each depth d at int_list[level_start[d] + i], i < int_count[d], as (cell, first_child,
// child_count, depth) (int_list: [cell_cap]).
void launch_tree_topology(const uint32_t* first_child, const uint32_t* child_count, const uint32_t* first,
                          const uint32_t* count, const uint8_t* depth, const uint32_t* level_start, size_t ncells,
                          uint32_t cell_cap, uint32_t* leaf_of, uint4* int_list, uint32_t* int_count, cudaStream_t s);
// calc_node over the whole tree (octree.cpp:108-162): the leaves (warps over particle chunks), then
// the internal levels deepest first from the per-depth lists (one launch per wide level, one block
// per run of narrow levels); also writes the compact walk records and the leaf-relative particle
// offsets.  level_start_host: the host copy of level_start (level widths).  s_internal (nullable):
// the internal levels go to that stream, forked from s after the leaves through `fork`.
void launch_calc_node(const double4* xyzm, size_t n, const uint32_t* child_count, const uint32_t* first,
                      const uint32_t* count, const uint32_t* level_start,
                      const uint32_t* level_start_host, const uint32_t* leaf_of, const uint4* int_list,
                      const uint32_t* int_count, uint32_t* sync, WNode* nodes, WNode32* nodes32, float4* rel,
                      cudaStream_t s, cudaStream_t s_internal = nullptr, cudaEvent_t fork = nullptr);
size_t calc_sync_words();  // device scratch words of launch_calc_node's `sync`
// leaf-relative offsets of the CURRENT positions against the existing nodes (GravityEngine::evaluate
// walks fresh positions with the node attributes of the last build/refresh, engine.cpp:31-81)
void launch_leaf_rel(const double4* xyzm, const uint32_t* child_count, const uint32_t* first, const uint32_t* count,
                     const WNode32* nodes32, uint32_t ncells, float4* rel, cudaStream_t s);

// out[k] = in[src[k]] gathers
void launch_gather_f64(const double* in, const uint32_t* src, double* out, size_t n, cudaStream_t s);
void launch_gather_u8(const uint8_t* in, const uint32_t* src, uint8_t* out, size_t n, cudaStream_t s);
void launch_gather_u32(const uint32_t* in, const uint32_t* src, uint32_t* out, size_t n, cudaStream_t s);
// equal-key runs of a storage-order sort: src (storage positions) re-ordered by ids[src] within runs
void launch_fix_ties(const uint64_t* keys, uint32_t* src, const uint32_t* ids, size_t n, DevFlags* flags,
                     cudaStream_t s);
// rank[perm[k]] = k
void launch_invert_perm(const uint32_t* perm, uint32_t* rank, size_t n, cudaStream_t s);
// xyzm[k] = (pos[3*id], ..., mass[id]) with id = perm[k] (host-order upload -> sorted)
void launch_pack_sorted(const double* pos3, const double* mass, const uint32_t* perm, double4* xyzm, size_t n,
                        cudaStream_t s);
void launch_pack_identity(const double* pos3, const double* mass, double4* xyzm, size_t n, cudaStream_t s);
void launch_iota(uint32_t* out, size_t n, cudaStream_t s);

// ---- walk.cu ----------------------------------------------------------------
struct WalkParams {
    double G, eps, dacc, theta;
    uint32_t frontier_cap;    // 0 = unchecked (cap cannot bind)
    int count_ops;
    int force_geometric;      // 1: geometric MAC for every group
    // a task donates half of its pending cells after writing D list entries since its last donation,
    // D = clamp(donate_scale x groups per producer warp, donate_few, donate_pushes): small walks
    // (block steps) split their groups finer; deterministic: D depends on the TOTAL group count only
    uint32_t donate_pushes = 4096, donate_few = 512, donate_scale = 256;  // sweeps: profiles/r2_donation_sweep.md
    double mass_max = 0.0;    // largest particle mass (host-known): guards the FP32 self-pair factor
};
constexpr int kMaxPeers = 8;
struct WalkBuffers {
    const uint32_t* sinks;    // [n_sinks] sorted particle indices
    const uint32_t* n_sinks;  // device scalar
    GroupRec* groups;         // [cap]
    uint32_t* n_groups;       // device scalar (written by group setup)
    float4* accum;            // [n_sinks] ax, ay, az, pot (zeroed by the walk launcher)
    unsigned long long* events;  // [3]
    uint64_t* queue;          // donated-task slots: (group << 32) | cell count
    uint32_t* batch;          // [queue_cap * 32] cells of each donated slot
    const uint32_t* order;    // [n_groups] initial-task order (heaviest first), written by the launcher when
                              // order_scratch is given; nullable: group index order
    uint32_t* order_scratch;  // [walk_order_scratch_words(n)] bucket counters + tile counts of the ordering
    uint32_t queue_cap;       // ring slots (1 << ring_bits, >= the task pool: tickets never wrap in a walk)
    uint32_t ring_bits;
    uint32_t* qstate;         // [16]: init claimed, donated reserved, pending, n_init, donated consumed,
                              //      shard lo, task records used, slices (all ranks), slices of this rank,
                              //      slices per heavy group, groups of the shard
    uint32_t* spill;          // per-warp stack spill
    uint32_t* level_count;    // [n_groups * 22] frontier-cap check (nullable)
    uint64_t* group_inter;    // [n_groups] per-group interactions (nullable)
    uint4* trace;             // optional per-task trace records (development), 2 x uint4 each
    uint32_t* trace_n;
    uint32_t trace_cap;
    uint32_t group_lo, group_hi;  // shard of groups to walk (hi = ~0u: all)
    // deterministic combination of split groups: every donated task has a record (parent, pending,
    // first child, next sibling) and a 32-sink accumulator slot; a task's subtree total is its own
    // partial plus its children's totals in donation order, formed by whichever finishes last
    uint4* trec;                        // [rec_cap] task records
    float4* tacc;                       // [rec_cap * 32] partial, then subtree, accumulators
    uint32_t* batch_rec;                // [queue_cap] record of the task in each donated slot
    uint32_t rec_cap;
    // fused peer exchange (world > 1): the task that completes a group stores the group's final
    // accumulators straight into every peer rank's accumulator (IPC-mapped, same slot layout)
    float4* peer_accum[kMaxPeers];      // peer accumulators, [self] unused
    int world, self;
    // cost-balanced shards (peer exchange): every group's list-entry count of this step goes to every
    // rank's cost_out; the next step splits the groups by the previous step's costs on the device
    uint32_t* gcost;                    // [n_groups] entry counts accumulated over a group's tasks
    uint32_t* peer_cost[kMaxPeers];     // this step's cost arrays of every rank ([self] = own)
    const uint32_t* cost_prev;          // own copy of the previous step's costs (nullable: equal shards)
    const uint32_t* ng_prev;            // groups behind cost_prev
    uint32_t* ng_cur;                   // groups of this step (written by the shard kernel)
    uint32_t* shard;                    // [2] device lo, hi (group indices) when cost-balanced
    // whole-system groups: a group whose sphere radius reaches kHeavyFrac of the root's
    // extent is cut into one slice per root child, the same slices for any rank count; slice j runs
    // on rank owner(j) (dealt by expected cost) and its partial goes to slot j of every rank's slice region (accum +
    // walk_slice_base(n)); walk_combine_slices then sums each group's slices in slice order
    uint32_t* heavy;                    // [kMaxHeavy + 1]: candidates' count, then the heavy groups (sorted)
    uint8_t* sliced;                    // [n_groups] 1: the group runs as slices (not an initial task)
    uint32_t slice_base;                // accumulator slot of slice 0 (walk_slice_base(n))
    int slice_world, slice_rank;        // the ranks the slices are dealt to (1, 0: all here)
};
size_t walk_slice_base(size_t n);      // first slice slot after n sinks
// the rank that walks slice j (nk root children of masses w, nh sliced groups, world ranks)
__host__ __device__ uint32_t slice_owner_of(const float* w, uint32_t nk, uint32_t j, uint32_t nh, uint32_t world);
// contiguous equal shard [lo, hi) of ng groups for rank of world (the copy / NCCL meshes)
__host__ __device__ inline void equal_shard(uint32_t ng, int rank, int world, uint32_t& lo, uint32_t& hi) {
    lo = uint32_t(uint64_t(ng) * uint32_t(rank) / uint32_t(world));
    hi = uint32_t(uint64_t(ng) * uint32_t(rank + 1) / uint32_t(world));
}
// the fixed per-rank window of accumulator slots every rank contributes to the copy / NCCL gather
inline size_t shard_window(size_t n, size_t gs, int world) {
    const size_t ng_max = (n + gs - 1) / gs;
    return ((ng_max + size_t(world) - 1) / size_t(world)) * gs;
}
size_t walk_slice_slots();             // slice-region slots (kMaxHeavy x 8 slices x 32 sinks)
size_t walk_heavy_words();
// every heavy group's accumulators = G x the sum of its slices in slice order (slice j read from
// slices + owner(j) * rank_stride + 32 j); zero cost for heavy groups in cost (nullable)
void launch_walk_combine(const WalkBuffers& b, const TreeView& t, const float4* slices, size_t rank_stride, int world,
                         double G, uint32_t* cost, cudaStream_t s);
size_t walk_spill_words();
size_t walk_order_scratch_words(size_t n_groups);
size_t walk_resident_warps();
void launch_groups(const TreeView& t, const double* acc_old_mag, const WalkBuffers& b, uint32_t group_size,
                   uint32_t n_sinks_cap, cudaStream_t s);
// kernel_ev (nullable): two events recorded around the walk kernel itself; prep = false: the caller
// ran launch_walk_prep (the part that reads no node) already
void launch_walk_prep(const WalkBuffers& b, uint32_t n_sinks_cap, uint32_t group_size, cudaStream_t s);
void launch_walk(const TreeView& t, const WalkParams& p, const WalkBuffers& b, bool with_pot, uint32_t n_sinks_cap,
                 uint32_t group_size, DevFlags* flags, cudaStream_t s, const cudaEvent_t* kernel_ev = nullptr,
                 bool prep = true);
// acc_out/pot_out in sorted order for the sinks (FP64)
void launch_walk_finalize(const WalkBuffers& b, uint32_t n_sinks_cap, double* ax, double* ay, double* az,
                          double* pot, cudaStream_t s);

// ---- integrate.cu -------------------------------------------------------------
void launch_direct_sum(const double4* xyzm, size_t n, double G, double eps, double* ax, double* ay, double* az,
                       DevFlags* flags, cudaStream_t s);
void launch_direct_targets(const double4* xyzm, size_t n, const uint32_t* targets, size_t nt, double G, double eps,
                           double* acc3, cudaStream_t s);
// compute_diagnostics (diagnostics.cpp:10-38) on the device: kinetic energy + momentum (kin_mom4), and
// when direct_potential the FP64 direct potential energy (n <= 2^17 path) into *w_direct; synchronises
void diagnostics_device(const double* mass, const double* vel3, const double4* xyzm, size_t n, double G, double eps,
                        bool direct_potential, double* kin_mom4, double* w_direct, DevFlags* flags, cudaStream_t s);
void launch_norm3(const double* ax, const double* ay, const double* az, double* out, size_t n, cudaStream_t s);
struct StepState {
    double4* xyzm;
    double *vx, *vy, *vz, *ax, *ay, *az, *amag;
    uint8_t* level;
    uint64_t* last_update;
};
void launch_tnext(const StepState& st, size_t n, unsigned long long* t_next, cudaStream_t s);
// bbox_partials (nullable): also the bounding-cube partials of the predicted positions, predict_blocks(n)
// records of 6 (launch_bbox_final turns them into the cube)
void launch_predict(const StepState& st, size_t n, const unsigned long long* t_next, uint64_t now, double tick,
                    uint8_t* active_flag, cudaStream_t s, double* bbox_partials = nullptr, DevFlags* flags = nullptr);
unsigned predict_blocks(size_t n);
// stream compaction of flags into sinks (order preserving), count into *n_out
void launch_compact(const uint8_t* flags, size_t n, uint32_t* out, uint32_t* n_out, uint64_t* status,
                    uint32_t* counter, cudaStream_t s);
struct SchemeDev {
    double eta, dt_max, eps;
    int adaptive, fixed_level;
};
// acc4: the walk's accumulator slots (sink order), FP32 -> FP64 exactly
void launch_correct(const StepState& st, const uint32_t* sinks, const uint32_t* n_sinks, uint32_t n_cap,
                    const float4* acc4, const unsigned long long* t_next, uint64_t now, double tick, SchemeDev sc,
                    cudaStream_t s);
void launch_assign_levels(const StepState& st, size_t n, SchemeDev sc, cudaStream_t s);
// free-function forms used by the C-ABI parity entry points
void launch_block_levels(const double* acc_mag, size_t n, SchemeDev sc, int* levels, cudaStream_t s);
void launch_predict_aos(double* pos3, double* vel3, const double* acc3, size_t n, double dt, cudaStream_t s);

}  // namespace g2
