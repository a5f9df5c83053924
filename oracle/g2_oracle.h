/* ORACLE / TEST INFRASTRUCTURE ONLY — plain-C restatement of the gravitree
 * hot path (the CPU checker).  Never linked into the product library.
 * See g2_oracle.c for the per-function reference citations. */
#ifndef G2_ORACLE_H
#define G2_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { G2O_OK = 0, G2O_DATA = 3, G2O_RESOURCE = 4, G2O_SINGULAR = 5 };

typedef struct {
    double cx, cy, cz, half;
} g2o_cube;

typedef struct {
    uint32_t first_child, child_count, first, count;
    uint8_t depth;
} g2o_cell;

typedef struct {
    double mass, cx, cy, cz, extent;
} g2o_node;

typedef struct {
    size_t n, ncells, leaf_cap;
    g2o_cube bbox;
    uint64_t* keys;
    uint32_t* perm;
    uint32_t* rank;
    g2o_cell* cells;
    g2o_node* nodes;
} g2o_tree;

typedef struct {
    uint64_t interactions, mac_evals, list_pushes;
} g2o_events;

int g2o_bounding_cube(size_t n, const double* pos, g2o_cube* out);
int g2o_morton_key(const double* p, const g2o_cube* c, uint64_t* key);
int g2o_build_tree(size_t n, const double* mass, const double* pos, size_t leaf_cap, int with_nodes, g2o_tree** out);
void g2o_calc_node(g2o_tree* t, const double* mass, const double* pos);
void g2o_tree_free(g2o_tree* t);
/* flat getters for ctypes */
void g2o_tree_get(const g2o_tree* t, double* bbox4, uint64_t* keys, uint32_t* perm, uint32_t* rank,
                  uint32_t* cells4, uint8_t* depth, double* nodes5);
size_t g2o_tree_ncells(const g2o_tree* t);

/* GravityEngine::evaluate for `targets` (NULL = all), with the reference's
 * grouping, MAC, BFS and list-flush order; FP64 throughout. */
int g2o_evaluate(const g2o_tree* t, size_t n, const double* mass, const double* pos, const double* acc_old_mag,
                 size_t n_targets, const uint32_t* targets, double G, double eps, double dacc, size_t group_size,
                 size_t list_capacity, size_t frontier_cap, double theta, int count_ops, unsigned threads,
                 double* acc_out, double* pot_out, g2o_events* ev, uint64_t* group_interactions);
int g2o_groups(size_t n, const double* pos, const double* acc_old_mag, const uint32_t* rank, size_t n_targets,
               const uint32_t* targets, size_t group_size, double* out5);
int g2o_direct_sum(size_t n, const double* mass, const double* pos, double G, double eps, unsigned threads,
                   double* acc_out);
int g2o_block_level(double acc_mag, double eta, double dt_max, int adaptive, int fixed_level, double eps);
void g2o_predict(size_t n, double* pos, double* vel, const double* acc, double dt);
size_t g2o_autotune(double build_time, size_t n_hist, const double* hist, size_t min_i, size_t max_i, size_t cur);
const char* g2o_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
