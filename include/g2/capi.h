/* g2 — B200-native GOTHIC-style octree gravity: the drop-in C ABI.
 *
 * Plain pointers and sizes only.  Every entry point replaces one member of
 * the reference C++ operator API (gravitree, /root/reference/proj/core); the
 * citation next to each declaration names the interface it stands in for.
 * Array conventions follow gravitree's ParticleSystem (particle_system.hpp:
 * 14-49): positions/velocities/accelerations are `double[3*n]` xyz
 * interleaved (a std::vector<Vec3> reinterpreted), masses `double[n]`,
 * indices in the caller's (original) particle order.  Host buffers in, host
 * buffers out; all device state stays resident between calls.
 *
 * Status codes (errors.hpp:8-23, CLI exit codes main.cpp:30-33):
 *   G2_OK 0, G2_INTERNAL 1, G2_DATA_ERROR 3, G2_RESOURCE_ERROR 4,
 *   G2_SINGULARITY 5 (a data_error subclass in the reference).
 * g2_last_error() returns the thread-local message of the last failure.
 */
#ifndef G2_CAPI_H
#define G2_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { G2_OK = 0, G2_INTERNAL = 1, G2_DATA_ERROR = 3, G2_RESOURCE_ERROR = 4, G2_SINGULARITY = 5 };

/* GravParams (particle_system.hpp:53-57) */
typedef struct {
    double G, eps, dacc;
} g2_grav_params;

/* EngineConfig (engine.hpp:14-23).  group_size must be 1..32 (one warp per
 * group; larger is rejected with G2_DATA_ERROR); list_capacity only has to be
 * >= 1 (results do not depend on it, test_gravity.cpp:213-229); frontier_cap
 * (0 = 8n) is honoured as the error contract of traversal.cpp:145-146;
 * threads is ignored on the device. */
typedef struct {
    size_t leaf_cap, group_size, list_capacity, frontier_cap;
    int count_ops;
    double bootstrap_theta;
    size_t bootstrap_direct_limit;
    unsigned threads;
} g2_engine_config;

/* TraversalEvents (op_counters.hpp:33-46) */
typedef struct {
    uint64_t interactions, mac_evals, list_pushes;
} g2_events;

/* StepScheme (integrator.hpp:18-23) and TunerConfig (rebuild_tuner.hpp:9-13) */
typedef struct {
    double eta, dt_max;
    int adaptive, fixed_level;
} g2_step_scheme;
typedef struct {
    size_t min_interval, max_interval, initial_interval;
} g2_tuner_config;

/* StepResult (integrator.hpp:43-50) with PhaseTimings (phase_timings.hpp:6-23);
 * phase times are device (CUDA-event) seconds, wall_seconds is host wall time. */
typedef struct {
    double walk_tree, calc_node, make_tree, predict, correct;
    g2_events events;
    size_t active, rebuild_interval;
    int rebuilt;
    double wall_seconds;
} g2_step_result;

typedef struct g2_engine g2_engine;
typedef struct g2_sim g2_sim;

const char* g2_last_error(void);
void g2_default_params(g2_grav_params* p);          /* GravParams{} */
void g2_default_engine_config(g2_engine_config* c); /* EngineConfig{} */
void g2_default_step_scheme(g2_step_scheme* s);     /* StepScheme{} */
void g2_default_tuner_config(g2_tuner_config* t);   /* TunerConfig{} */

/* ---- GravityEngine (engine.hpp:29-66, engine.cpp:13-103) ---------------- */
/* GravityEngine(GravParams, EngineConfig)  engine.cpp:13-18 */
int g2_engine_create(const g2_grav_params* p, const g2_engine_config* c, int device, g2_engine** out);
void g2_engine_destroy(g2_engine* e);
/* build / build_structure / refresh   engine.cpp:20-29 */
int g2_engine_build(g2_engine* e, size_t n, const double* mass, const double* pos);
int g2_engine_build_structure(g2_engine* e, size_t n, const double* mass, const double* pos);
int g2_engine_refresh(g2_engine* e, size_t n, const double* mass, const double* pos);
int g2_engine_has_tree(const g2_engine* e);
/* evaluate(system, targets, pot_out)  engine.cpp:31-81.  targets == NULL:
 * all particles (engine.cpp:83-87).  acc_inout[3n] / pot_out[n] (nullable)
 * are written for the targets only, like system.acc / pot_out. */
int g2_engine_evaluate(g2_engine* e, size_t n, const double* mass, const double* pos, const double* acc_old_mag,
                       size_t n_targets, const uint32_t* targets, double* acc_inout, double* pot_out,
                       g2_events* events);
/* bootstrap(system)  engine.cpp:89-103: fills acc[3n] and acc_old_mag[n]
 * (acc_old_mag is read first: all-zero selects the geometric MAC). */
int g2_engine_bootstrap(g2_engine* e, size_t n, const double* mass, const double* pos, double* acc_out,
                        double* acc_old_mag_inout, g2_events* events);
/* tree() accessors (octree.hpp:32-42): sizes, then flat copies.
 * cells4 = {first_child, child_count, first, count} per cell, nodes5 =
 * {mass, com.x, com.y, com.z, extent}; any pointer may be NULL. */
int g2_engine_tree_size(const g2_engine* e, size_t* n, size_t* ncells);
int g2_engine_get_tree(g2_engine* e, double* bbox4, uint64_t* keys, uint32_t* perm, uint32_t* rank,
                       uint32_t* cells4, uint8_t* depth, double* nodes5);
/* params().dacc setter (engine.hpp:40 exposes a mutable params()) */
int g2_engine_set_params(g2_engine* e, const g2_grav_params* p);

/* ---- free functions -------------------------------------------------------- */
/* direct_sum (gravity.cpp:18-43), on the device, FP64, bit-identical order */
int g2_direct_sum(size_t n, const double* mass, const double* pos, double G, double eps, int device, double* acc_out);
/* direct summation onto a subset of targets (accuracy oracle at large N, §8f):
 * acc_out[3*n_targets] in target order; FP64, chunked over sources */
int g2_direct_sum_targets(size_t n, const double* mass, const double* pos, double G, double eps, size_t n_targets,
                          const uint32_t* targets, int device, double* acc_out);
/* block_level (integrator.cpp:21-33) evaluated by the device kernel */
int g2_block_level(size_t n, const double* acc_mag, const g2_step_scheme* s, double eps, int device, int* levels);
/* predict (integrator.cpp:40-45) on the device; pos/vel updated in place */
int g2_predict(size_t n, double* pos, double* vel, const double* acc, double dt, int device);

/* Diagnostics (diagnostics.hpp:9-15) and compute_diagnostics (diagnostics.cpp:10-38): kinetic
 * energy and momentum, potential energy by FP64 direct summation up to 2^17 particles
 * (kDirectPotentialLimit) and beyond by a dacc = 2^-20 tree walk with potentials that uses
 * acc_old_mag as the system's (NULL: zeros => geometric MAC, as for a fresh ParticleSystem).
 * Throws (G2_SINGULARITY) on coincident particles with eps == 0 on the direct path. */
typedef struct {
    double kinetic, potential, total;
    double momentum[3];
    double virial_ratio;
} g2_diagnostics;
int g2_compute_diagnostics(size_t n, const double* mass, const double* pos, const double* vel,
                           const double* acc_old_mag, const g2_grav_params* p, int device, g2_diagnostics* out);

/* ---- OCTF snapshots (snapshot.hpp:10-30, snapshot.cpp:65-121) ----------------
 * Little-endian "OCTF", u32 version 1, u64 n, f64 time, G, eps, f64 mass[n], pos[3n], vel[3n]:
 * the arrays ARE the C-ABI layout.  Failures are G2_DATA_ERROR with the reference's messages
 * (bad magic / unsupported version / zero particle count / truncated <field> at byte <offset>).
 * g2_read_snapshot fills caller buffers of capacity cap (g2_snapshot_info gives n first). */
int g2_snapshot_info(const char* path, size_t* n, double* time, double* G, double* eps);
int g2_read_snapshot(const char* path, size_t cap, double* mass, double* pos, double* vel, size_t* n, double* time,
                     double* G, double* eps);
/* atomic (temp file + rename), write_snapshot(path, system, params) */
int g2_write_snapshot(const char* path, size_t n, const double* mass, const double* pos, const double* vel,
                      double time, const g2_grav_params* p);

/* ---- Simulation (integrator.hpp:54-91, integrator.cpp:56-164) ------------- */
int g2_sim_create(size_t n, const double* mass, const double* pos, const double* vel, const g2_grav_params* p,
                  const g2_step_scheme* s, const g2_engine_config* c, const g2_tuner_config* t, int device,
                  g2_sim** out);
void g2_sim_destroy(g2_sim* s);
int g2_sim_init(g2_sim* s);
int g2_sim_step(g2_sim* s, g2_step_result* r);
int g2_sim_set_fixed_rebuild_interval(g2_sim* s, size_t interval);
/* state in original particle order; any pointer may be NULL */
int g2_sim_get_state(g2_sim* s, double* pos, double* vel, double* acc, double* acc_old_mag, uint8_t* level,
                     double* time);
/* overwrite positions / velocities (original order) of the device-resident state */
int g2_sim_set_state(g2_sim* s, const double* pos, const double* vel);
/* engine().tree() of the simulation (integrator.hpp:62, engine.hpp:47): the tree of the last
 * rebuild; node attributes are those of the last calc_node (refresh).  Same layout as
 * g2_engine_get_tree. */
int g2_sim_tree_size(g2_sim* s, size_t* n, size_t* ncells);
int g2_sim_get_tree(g2_sim* s, double* bbox4, uint64_t* keys, uint32_t* perm, uint32_t* rank, uint32_t* cells4,
                    uint8_t* depth, double* nodes5);
/* Simulation from a snapshot file: read straight into pinned host memory and uploaded (no AoS
 * conversion); GravParams = (snapshot G, snapshot eps, dacc), as the reference CLI builds them. */
int g2_sim_create_from_snapshot(const char* path, double dacc, const g2_step_scheme* s, const g2_engine_config* c,
                                const g2_tuner_config* t, int device, g2_sim** out);
/* the device-resident state (original order) written as a snapshot with the simulation's time, G, eps */
int g2_sim_write_snapshot(g2_sim* s, const char* path);
/* extension: rebuild the tree every step (the all-active "full step" benchmark) */
int g2_sim_set_rebuild_every_step(g2_sim* s, int on);
/* extension: overlap independent phases of a step on a side stream (default on): calc_node's internal
 * levels beside the walk's compaction and group spheres.  Off: every phase alone on the step's stream
 * (the per-phase rooflines) */
int g2_sim_set_phase_overlap(g2_sim* s, int on);
int g2_sim_tuner_interval(g2_sim* s, size_t* interval);
/* extension (diagnostics): how the Simulation's rebuilds sorted so far -- by the bucket sort of the
 * nearly sorted storage order, and by its onesweep radix fallback (a bucket over capacity) */
int g2_sim_sort_stats(g2_sim* s, unsigned long long* bucket_sorts, unsigned long long* radix_fallbacks);
/* extension (diagnostics): the last step walk's whole-system groups cut into slices (one per root
 * child) and the number of slices over all ranks; synchronises the simulation's stream */
int g2_sim_walk_slices(g2_sim* s, unsigned* heavy_groups, unsigned* slices);
/* extension (diagnostics): task records the last step's walk used (split groups' ordered combination)
 * and the pool's capacity; synchronises the simulation's stream */
int g2_sim_walk_records(g2_sim* s, unsigned* used, size_t* capacity);
/* extension (measurement): device seconds of the last walk kernel alone (CUDA events around its launch,
 * on its stream; the step's walk_tree phase also holds the group set-up kernels) */
int g2_sim_walk_kernel_seconds(g2_sim* s, double* seconds);
/* mesh arithmetic (host code, callable without a GPU): the contiguous equal shard [lo, hi)
 * of n_groups for a rank (copy / NCCL meshes), the fixed per-rank window of accumulator slots those
 * meshes gather, and the rank that walks slice `slice` of the whole-system groups (root children
 * masses root_child_mass[n_children], n_heavy sliced groups) */
void g2_mesh_shard(unsigned n_groups, int rank, int world, unsigned* lo, unsigned* hi);
size_t g2_mesh_window(size_t n, size_t group_size, int world);
unsigned g2_slice_owner(const float* root_child_mass, unsigned n_children, unsigned slice, unsigned n_heavy,
                        int world);
/* extension: the rebuild tuner's clock (RebuildTuner::record_walk/record_build, rebuild_tuner.hpp:18-31).
 * flop_rate <= 0: CUDA-event phase times (default).  flop_rate > 0: a deterministic model -- walk
 * seconds = (27 interactions + 5 MAC evaluations) / flop_rate (op_counters.hpp:50-63), build seconds =
 * build_seconds_per_particle x n -- so the rebuild schedule, hence the trajectory, is reproducible.
 * On a mesh every rank feeds its tuner the same inputs either way (sum of the ranks' modelled walk
 * times, or max of measured ones), so every rank takes the same rebuild decisions. */
int g2_sim_set_tuner_model(g2_sim* s, double flop_rate, double build_seconds_per_particle);

/* the CUDA stream (cudaStream_t) all of the simulation's work is issued on,
 * so callers can time it with their own events */
int g2_sim_stream(g2_sim* s, void** stream);
/* kernels launched by this library since load (benchmark evidence) */
unsigned long long g2_launch_count(void);
/* autotune_rebuild (rebuild_tuner.cpp:28-61) on a walk-time history: host logic */
size_t g2_autotune(double build_time, size_t n_hist, const double* hist, size_t min_interval, size_t max_interval,
                   size_t current_interval);
/* sample_model (models.cpp:442-460), bit-identical to the reference, multithreaded
 * (threads 0 = all cores); returns 0 or G2_DATA_ERROR (message: g2_ics_last_error) */
int g2_sample_model(const char* name, size_t n, uint64_t seed, unsigned threads, double* mass, double* pos,
                    double* vel);
const char* g2_ics_last_error(void);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink) --------------------- */
/* NCCL unique id (128 bytes) for rank 0 to broadcast out of band */
int g2_nccl_unique_id(unsigned char id[128]);
/* join a communicator; the simulation then walks only its shard of sink
 * groups and all-gathers the new accelerations each step */
int g2_sim_set_mesh(g2_sim* s, int rank, int world, const unsigned char id[128]);
/* in-process mesh: sims[0..world) (one host thread per step call, any devices)
 * shard the sink groups and exchange accelerations by device copies */
int g2_sim_set_mesh_local(g2_sim** sims, int world);
/* fused peer exchange, no collective: the walk kernel stores each finished sink
 * group's accelerations straight into every peer's accumulator (NVLink P2P stores
 * through CUDA IPC mappings), then device flags order them before the correct.
 * Every rank exports g2_p2p_handle_bytes() bytes, the handles of all ranks are
 * exchanged out of band (rank order), then each rank opens its peers'. 2 <= world <= 8. */
size_t g2_p2p_handle_bytes(void);
int g2_sim_p2p_export(g2_sim* s, int rank, int world, void* handle);
int g2_sim_set_mesh_p2p(g2_sim* s, int rank, int world, const void* handles);
/* the same fused exchange between Simulations of one process (any devices with peer access) */
int g2_sim_set_mesh_local_p2p(g2_sim** sims, int world);

#ifdef __cplusplus
}
#endif
#endif /* G2_CAPI_H */
