/* ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the gravitree hot path (reference:
 * /root/reference/proj/core).  It is the CPU checker the GPU parity tests
 * compare against, and it is itself pinned against the reference library
 * (oracle/_ref) and the golden fixtures in tests/golden (tests/test_oracle.py).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * it; the product library never links it.
 *
 * Arithmetic mirrors the reference operation by operation in IEEE FP64 with
 * no contraction (-ffp-contract=off), so keys, perm, cells, node attributes,
 * group spheres, MAC decisions, events and accelerations are bit-identical
 * to the reference for the same inputs.
 */
#include "g2_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[256];
const char* g2o_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

static inline double dmin(double a, double b) { return b < a ? b : a; } /* std::min(a,b) */
static inline double dmax(double a, double b) { return a < b ? b : a; } /* std::max(a,b) */

/* ---- morton.hpp:14-49 ------------------------------------------------- */
static uint64_t expand_bits(uint64_t v) { /* morton.hpp:14-22 */
    v &= 0x1fffff;
    v = (v | v << 32) & 0x001f00000000ffffULL;
    v = (v | v << 16) & 0x001f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
}

static uint32_t quantize(double v, double lo, double width) { /* morton.hpp:29-34 */
    const double t = (v - lo) / width * 2097152.0;
    if (t <= 0.0) return 0;
    const uint64_t q = (uint64_t)t;
    return q > 2097151u ? 2097151u : (uint32_t)q;
}

int g2o_morton_key(const double* p, const g2o_cube* c, uint64_t* key) { /* morton.hpp:38-44 */
    const double lox = c->cx - c->half, loy = c->cy - c->half, loz = c->cz - c->half;
    const double hix = c->cx + c->half, hiy = c->cy + c->half, hiz = c->cz + c->half;
    if (!(p[0] >= lox && p[0] <= hix && p[1] >= loy && p[1] <= hiy && p[2] >= loz && p[2] <= hiz))
        return fail(G2O_DATA, "morton_key: position outside root cube");
    const double w = 2.0 * c->half;
    *key = (expand_bits(quantize(p[0], lox, w)) << 2) | (expand_bits(quantize(p[1], loy, w)) << 1) |
           expand_bits(quantize(p[2], loz, w));
    return G2O_OK;
}

static unsigned digit_at(uint64_t key, int depth) { return (unsigned)(key >> (3 * (20 - depth))) & 7u; }

/* ---- octree.cpp:24-49 ------------------------------------------------- */
int g2o_bounding_cube(size_t n, const double* pos, g2o_cube* out) {
    if (n == 0) return fail(G2O_DATA, "bounding_cube: no particles");
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (size_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a)
            if (!isfinite(pos[3 * i + a])) return fail(G2O_DATA, "bounding_cube: non-finite position");
        for (int a = 0; a < 3; ++a) {
            lo[a] = dmin(lo[a], pos[3 * i + a]);
            hi[a] = dmax(hi[a], pos[3 * i + a]);
        }
    }
    double c[3];
    for (int a = 0; a < 3; ++a) c[a] = (lo[a] + hi[a]) * 0.5; /* 0.5 * (lo + hi) */
    /* half-width from the rounded centre, in the reference's order x,x,y,y,z,z */
    const double d[6] = {lo[0] - c[0], hi[0] - c[0], lo[1] - c[1], hi[1] - c[1], lo[2] - c[2], hi[2] - c[2]};
    double h = 0.0;
    for (int k = 0; k < 6; ++k) h = dmax(h, fabs(d[k]));
    out->cx = c[0];
    out->cy = c[1];
    out->cz = c[2];
    out->half = h * (1.0 + 1e-12);
    if (out->half == 0.0) out->half = 1.0;
    return G2O_OK;
}

/* ---- octree.cpp:51-106 ------------------------------------------------ */
typedef struct {
    uint64_t key;
    uint32_t idx;
} kv;
static int kv_cmp(const void* a, const void* b) { /* std::pair lexicographic order */
    const kv *x = a, *y = b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

int g2o_build_tree(size_t n, const double* mass, const double* pos, size_t leaf_cap, int with_nodes,
                   g2o_tree** out) {
    if (n < 1) return fail(G2O_DATA, "build_tree: empty system");
    if (leaf_cap < 1) return fail(G2O_DATA, "build_tree: leaf_cap must be >= 1");
    g2o_tree* t = calloc(1, sizeof *t);
    t->n = n;
    t->leaf_cap = leaf_cap;
    int rc = g2o_bounding_cube(n, pos, &t->bbox);
    if (rc) {
        free(t);
        return rc;
    }
    kv* order = malloc(n * sizeof *order);
    for (size_t i = 0; i < n; ++i) {
        rc = g2o_morton_key(pos + 3 * i, &t->bbox, &order[i].key);
        if (rc) {
            free(order);
            free(t);
            return rc;
        }
        order[i].idx = (uint32_t)i;
    }
    qsort(order, n, sizeof *order, kv_cmp);
    t->keys = malloc(n * 8);
    t->perm = malloc(n * 4);
    t->rank = malloc(n * 4);
    for (size_t k = 0; k < n; ++k) {
        t->keys[k] = order[k].key;
        t->perm[k] = order[k].idx;
        t->rank[order[k].idx] = (uint32_t)k;
    }
    free(order);

    /* breadth-first split (octree.cpp:74-102): children appended in digit order */
    size_t cap = 2 * n / leaf_cap + 16, nc = 1;
    g2o_cell* cells = malloc(cap * sizeof *cells);
    cells[0] = (g2o_cell){0, 0, 0, (uint32_t)n, 0};
    for (size_t c = 0; c < nc; ++c) {
        const g2o_cell cell = cells[c];
        if (cell.count <= leaf_cap || cell.depth >= 21) continue;
        const uint32_t end = cell.first + cell.count;
        uint32_t lo = cell.first, first_child = (uint32_t)nc, child_count = 0;
        for (unsigned dg = 0; dg < 8 && lo != end; ++dg) {
            /* upper_bound: first key in [lo,end) whose digit exceeds dg */
            uint32_t a = lo, b = end;
            while (a < b) {
                const uint32_t mid = a + (b - a) / 2;
                if (dg < digit_at(t->keys[mid], cell.depth))
                    b = mid;
                else
                    a = mid + 1;
            }
            const uint32_t hi = a;
            if (hi != lo) {
                if (nc == cap) {
                    cap *= 2;
                    cells = realloc(cells, cap * sizeof *cells);
                }
                cells[nc++] = (g2o_cell){0, 0, lo, hi - lo, (uint8_t)(cell.depth + 1)};
                ++child_count;
            }
            lo = hi;
        }
        cells[c].first_child = first_child;
        cells[c].child_count = child_count;
    }
    t->cells = cells;
    t->ncells = nc;
    t->nodes = calloc(nc, sizeof *t->nodes);
    if (with_nodes) g2o_calc_node(t, mass, pos);
    *out = t;
    return G2O_OK;
}

/* ---- octree.cpp:108-162 (calc_one_node + deepest-run-first sweep) ---- */
static void calc_one(g2o_tree* t, const double* mass, const double* pos, size_t c) {
    const g2o_cell* cell = &t->cells[c];
    g2o_node* nd = &t->nodes[c];
    double m = 0.0, wx = 0.0, wy = 0.0, wz = 0.0;
    if (cell->child_count == 0) {
        for (uint32_t k = cell->first; k < cell->first + cell->count; ++k) {
            const uint32_t i = t->perm[k];
            m += mass[i];
            wx += mass[i] * pos[3 * i]; /* weighted += mass * pos */
            wy += mass[i] * pos[3 * i + 1];
            wz += mass[i] * pos[3 * i + 2];
        }
        const double inv = 1.0 / m;
        nd->mass = m;
        nd->cx = wx * inv;
        nd->cy = wy * inv;
        nd->cz = wz * inv;
        double e2 = 0.0;
        for (uint32_t k = cell->first; k < cell->first + cell->count; ++k) {
            const uint32_t i = t->perm[k];
            const double dx = pos[3 * i] - nd->cx, dy = pos[3 * i + 1] - nd->cy, dz = pos[3 * i + 2] - nd->cz;
            e2 = dmax(e2, dx * dx + dy * dy + dz * dz);
        }
        nd->extent = sqrt(e2);
    } else {
        for (uint32_t ch = cell->first_child; ch < cell->first_child + cell->child_count; ++ch) {
            const g2o_node* q = &t->nodes[ch];
            m += q->mass;
            wx += q->mass * q->cx;
            wy += q->mass * q->cy;
            wz += q->mass * q->cz;
        }
        const double inv = 1.0 / m;
        nd->mass = m;
        nd->cx = wx * inv;
        nd->cy = wy * inv;
        nd->cz = wz * inv;
        double ext = 0.0;
        for (uint32_t ch = cell->first_child; ch < cell->first_child + cell->child_count; ++ch) {
            const g2o_node* q = &t->nodes[ch];
            const double dx = q->cx - nd->cx, dy = q->cy - nd->cy, dz = q->cz - nd->cz;
            ext = dmax(ext, sqrt(dx * dx + dy * dy + dz * dz) + q->extent);
        }
        nd->extent = ext;
    }
}

void g2o_calc_node(g2o_tree* t, const double* mass, const double* pos) {
    /* children always follow parents in BFS order, so a reverse sweep is a valid
       deepest-first order; each cell's result depends only on its children. */
    for (size_t c = t->ncells; c-- > 0;) calc_one(t, mass, pos, c);
}

void g2o_tree_free(g2o_tree* t) {
    if (!t) return;
    free(t->keys);
    free(t->perm);
    free(t->rank);
    free(t->cells);
    free(t->nodes);
    free(t);
}

size_t g2o_tree_ncells(const g2o_tree* t) { return t->ncells; }

void g2o_tree_get(const g2o_tree* t, double* bbox4, uint64_t* keys, uint32_t* perm, uint32_t* rank,
                  uint32_t* cells4, uint8_t* depth, double* nodes5) {
    if (bbox4) {
        bbox4[0] = t->bbox.cx;
        bbox4[1] = t->bbox.cy;
        bbox4[2] = t->bbox.cz;
        bbox4[3] = t->bbox.half;
    }
    if (keys) memcpy(keys, t->keys, t->n * 8);
    if (perm) memcpy(perm, t->perm, t->n * 4);
    if (rank) memcpy(rank, t->rank, t->n * 4);
    for (size_t c = 0; c < t->ncells; ++c) {
        if (cells4) {
            cells4[4 * c] = t->cells[c].first_child;
            cells4[4 * c + 1] = t->cells[c].child_count;
            cells4[4 * c + 2] = t->cells[c].first;
            cells4[4 * c + 3] = t->cells[c].count;
        }
        if (depth) depth[c] = t->cells[c].depth;
        if (nodes5) memcpy(nodes5 + 5 * c, &t->nodes[c], 5 * sizeof(double));
    }
}

/* ---- traversal.cpp:16-38 make_group ------------------------------------ */
typedef struct {
    const uint32_t* members;
    size_t count;
    double cx, cy, cz, radius, a_min;
} group_t;

static group_t make_group(const double* pos, const double* acc_old_mag, const uint32_t* members, size_t count) {
    group_t g = {members, count, 0, 0, 0, 0, 0};
    if (count == 0) return g;
    double lo[3], hi[3];
    for (int a = 0; a < 3; ++a) lo[a] = hi[a] = pos[3 * members[0] + a];
    double a_min = acc_old_mag[members[0]];
    for (size_t k = 0; k < count; ++k) {
        const uint32_t i = members[k];
        for (int a = 0; a < 3; ++a) {
            lo[a] = dmin(lo[a], pos[3 * i + a]);
            hi[a] = dmax(hi[a], pos[3 * i + a]);
        }
        a_min = dmin(a_min, acc_old_mag[i]);
    }
    g.cx = (lo[0] + hi[0]) * 0.5;
    g.cy = (lo[1] + hi[1]) * 0.5;
    g.cz = (lo[2] + hi[2]) * 0.5;
    double r2 = 0.0;
    for (size_t k = 0; k < count; ++k) {
        const uint32_t i = members[k];
        const double dx = pos[3 * i] - g.cx, dy = pos[3 * i + 1] - g.cy, dz = pos[3 * i + 2] - g.cz;
        r2 = dmax(r2, dx * dx + dy * dy + dz * dz);
    }
    g.radius = sqrt(r2);
    g.a_min = a_min;
    return g;
}

/* ---- traversal.cpp:40-56 MACs ------------------------------------------- */
static double group_distance(const g2o_node* nd, const group_t* g) {
    const double dx = g->cx - nd->cx, dy = g->cy - nd->cy, dz = g->cz - nd->cz;
    return dmax(0.0, sqrt(dx * dx + dy * dy + dz * dz) - g->radius);
}
static int mac_accept(const g2o_node* nd, const group_t* g, double G, double dacc) {
    const double d = group_distance(nd, g);
    if (d <= 0.0) return 0;
    const double d2 = d * d;
    const double lhs = G * nd->mass * nd->extent * nd->extent / (d2 * d2);
    return lhs <= dacc * g->a_min;
}
static int mac_accept_geometric(const g2o_node* nd, const group_t* g, double theta) {
    const double d = group_distance(nd, g);
    if (d <= 0.0) return 0;
    return nd->extent <= theta * d;
}

/* ---- traversal.cpp:61-156 walk_tree_group ----------------------------------- */
typedef struct {
    const g2o_tree* t;
    const double *mass, *pos;
    double G, eps2, dacc, theta;
    size_t list_cap, frontier_cap;
    int with_pot;
} walk_ctx;

typedef struct {
    double *lx, *ly, *lz, *lm;
    size_t size;
    uint32_t *front, *next;
    double *ax, *ay, *az, *phi;
} scratch_t;

static void flush(const walk_ctx* w, scratch_t* s, const group_t* g, g2o_events* ev) {
    if (s->size == 0) return;
    ev->interactions += (uint64_t)s->size * g->count;
    for (size_t m = 0; m < g->count; ++m) {
        const uint32_t i = g->members[m];
        const double rx = w->pos[3 * i], ry = w->pos[3 * i + 1], rz = w->pos[3 * i + 2];
        double ax = s->ax[m], ay = s->ay[m], az = s->az[m], ph = w->with_pot ? s->phi[m] : 0.0;
        for (size_t e = 0; e < s->size; ++e) {
            const double dx = s->lx[e] - rx, dy = s->ly[e] - ry, dz = s->lz[e] - rz;
            const double r2 = dx * dx + dy * dy + dz * dz + w->eps2;
            if (r2 == 0.0) continue;
            const double inv = 1.0 / sqrt(r2);
            const double inv3 = inv * inv * inv; /* traversal.cpp:75-76 */
            const double f = w->G * s->lm[e] * inv3;
            ax += f * dx;
            ay += f * dy;
            az += f * dz;
            if (w->with_pot && (dx * dx + dy * dy + dz * dz) > 0.0) ph -= w->G * s->lm[e] * inv;
        }
        s->ax[m] = ax;
        s->ay[m] = ay;
        s->az[m] = az;
        if (w->with_pot) s->phi[m] = ph;
    }
    s->size = 0;
}

static void push(const walk_ctx* w, scratch_t* s, const group_t* g, g2o_events* ev, double x, double y, double z,
                 double m) {
    if (s->size == w->list_cap) flush(w, s, g, ev);
    s->lx[s->size] = x;
    s->ly[s->size] = y;
    s->lz[s->size] = z;
    s->lm[s->size] = m;
    ++s->size;
    ++ev->list_pushes;
}

static int walk_group(const walk_ctx* w, scratch_t* s, const group_t* g, int geometric, g2o_events* ev) {
    const g2o_tree* t = w->t;
    for (size_t m = 0; m < g->count; ++m) {
        s->ax[m] = s->ay[m] = s->az[m] = 0.0;
        if (w->with_pot) s->phi[m] = 0.0;
    }
    size_t nf = 1, nn;
    s->front[0] = 0;
    while (nf) {
        nn = 0;
        for (size_t f = 0; f < nf; ++f) {
            const uint32_t c = s->front[f];
            const g2o_cell* cell = &t->cells[c];
            const g2o_node* nd = &t->nodes[c];
            ++ev->mac_evals;
            const int acc = geometric ? mac_accept_geometric(nd, g, w->theta) : mac_accept(nd, g, w->G, w->dacc);
            if (acc) {
                push(w, s, g, ev, nd->cx, nd->cy, nd->cz, nd->mass);
            } else if (cell->child_count == 0) {
                for (uint32_t k = cell->first; k < cell->first + cell->count; ++k) {
                    const uint32_t j = t->perm[k];
                    push(w, s, g, ev, w->pos[3 * j], w->pos[3 * j + 1], w->pos[3 * j + 2], w->mass[j]);
                }
            } else {
                if (nn + cell->child_count > w->frontier_cap)
                    return fail(G2O_RESOURCE, "walk_tree_group: frontier queue exhausted");
                for (uint32_t ch = cell->first_child; ch < cell->first_child + cell->child_count; ++ch)
                    s->next[nn++] = ch;
            }
        }
        uint32_t* tmp = s->front;
        s->front = s->next;
        s->next = tmp;
        nf = nn;
    }
    flush(w, s, g, ev);
    return G2O_OK;
}

typedef struct {
    const walk_ctx* w;
    const uint32_t* ordered;
    size_t n_ord, group_size, g_lo, g_hi;
    const double* acc_old_mag;
    double *acc_out, *pot_out;
    uint64_t* group_inter;
    g2o_events ev;
    int rc;
} job_t;

static void* run_job(void* arg) {
    job_t* j = arg;
    const walk_ctx* w = j->w;
    scratch_t s;
    s.lx = malloc(w->list_cap * 8);
    s.ly = malloc(w->list_cap * 8);
    s.lz = malloc(w->list_cap * 8);
    s.lm = malloc(w->list_cap * 8);
    s.size = 0;
    /* a frontier level never exceeds the cell count */
    s.front = malloc((w->t->ncells + 1) * 4);
    s.next = malloc((w->t->ncells + 1) * 4);
    s.ax = malloc(j->group_size * 8);
    s.ay = malloc(j->group_size * 8);
    s.az = malloc(j->group_size * 8);
    s.phi = malloc(j->group_size * 8);
    memset(&j->ev, 0, sizeof j->ev);
    j->rc = 0;
    for (size_t gi = j->g_lo; gi < j->g_hi && !j->rc; ++gi) {
        const size_t lo = gi * j->group_size;
        const size_t cnt = (j->n_ord - lo) < j->group_size ? (j->n_ord - lo) : j->group_size;
        const group_t g = make_group(w->pos, j->acc_old_mag, j->ordered + lo, cnt);
        g2o_events gev = {0, 0, 0};
        j->rc = walk_group(w, &s, &g, g.a_min <= 0.0, &gev);
        if (j->group_inter) j->group_inter[gi] = gev.interactions;
        j->ev.interactions += gev.interactions;
        j->ev.mac_evals += gev.mac_evals;
        j->ev.list_pushes += gev.list_pushes;
        for (size_t m = 0; m < cnt; ++m) {
            const uint32_t i = g.members[m];
            j->acc_out[3 * i] = s.ax[m];
            j->acc_out[3 * i + 1] = s.ay[m];
            j->acc_out[3 * i + 2] = s.az[m];
            if (j->pot_out) j->pot_out[i] = s.phi[m];
        }
    }
    free(s.lx), free(s.ly), free(s.lz), free(s.lm), free(s.front), free(s.next);
    free(s.ax), free(s.ay), free(s.az), free(s.phi);
    return NULL;
}

static const uint32_t* g_rank_for_sort;
static int rank_cmp(const void* a, const void* b) {
    const uint32_t ra = g_rank_for_sort[*(const uint32_t*)a], rb = g_rank_for_sort[*(const uint32_t*)b];
    return ra < rb ? -1 : (ra > rb);
}

static uint32_t* order_targets(const uint32_t* rank, size_t n, size_t n_targets, const uint32_t* targets) {
    /* engine.cpp:38-41: sinks in Morton rank order (counting placement; ranks are unique) */
    uint32_t* ordered = malloc((n_targets ? n_targets : 1) * 4);
    if (targets) {
        memcpy(ordered, targets, n_targets * 4);
        g_rank_for_sort = rank;
        qsort(ordered, n_targets, 4, rank_cmp);
    } else {
        for (size_t i = 0; i < n; ++i) ordered[rank[i]] = (uint32_t)i;
    }
    return ordered;
}

int g2o_evaluate(const g2o_tree* t, size_t n, const double* mass, const double* pos, const double* acc_old_mag,
                 size_t n_targets, const uint32_t* targets, double G, double eps, double dacc, size_t group_size,
                 size_t list_capacity, size_t frontier_cap, double theta, int count_ops, unsigned threads,
                 double* acc_out, double* pot_out, g2o_events* ev, uint64_t* group_interactions) {
    if (group_size < 1) return fail(G2O_DATA, "group_size must be >= 1");
    if (list_capacity < 1) return fail(G2O_DATA, "InteractionList: capacity must be >= 1");
    memset(ev, 0, sizeof *ev);
    if (!targets) n_targets = n;
    if (n_targets == 0) return G2O_OK;
    uint32_t* ordered = order_targets(t->rank, n, n_targets, targets);
    walk_ctx w = {t, mass, pos, G, eps * eps, dacc, theta, list_capacity, frontier_cap ? frontier_cap : 8 * n,
                  pot_out != NULL};
    const size_t ng = (n_targets + group_size - 1) / group_size;
    if (threads < 1) threads = 1;
    if (threads > ng) threads = (unsigned)ng;
    job_t* jobs = calloc(threads, sizeof *jobs);
    pthread_t* th = calloc(threads, sizeof *th);
    for (unsigned k = 0; k < threads; ++k) {
        jobs[k] = (job_t){&w, ordered, n_targets, group_size, ng * k / threads, ng * (k + 1) / threads,
                          acc_old_mag, acc_out, pot_out, group_interactions, {0, 0, 0}, 0};
        if (k) pthread_create(&th[k], NULL, run_job, &jobs[k]);
    }
    run_job(&jobs[0]);
    int rc = 0;
    for (unsigned k = 0; k < threads; ++k) {
        if (k) pthread_join(th[k], NULL);
        if (jobs[k].rc && !rc) rc = jobs[k].rc;
        ev->interactions += jobs[k].ev.interactions;
        ev->mac_evals += jobs[k].ev.mac_evals;
        ev->list_pushes += jobs[k].ev.list_pushes;
    }
    if (!count_ops) memset(ev, 0, sizeof *ev); /* traversal.cpp:155 */
    free(jobs);
    free(th);
    free(ordered);
    return rc;
}

int g2o_groups(size_t n, const double* pos, const double* acc_old_mag, const uint32_t* rank, size_t n_targets,
               const uint32_t* targets, size_t group_size, double* out5) {
    uint32_t* ordered = order_targets(rank, n, n_targets, targets);
    if (!targets) n_targets = n;
    const size_t ng = (n_targets + group_size - 1) / group_size;
    for (size_t gi = 0; gi < ng; ++gi) {
        const size_t lo = gi * group_size;
        const size_t cnt = (n_targets - lo) < group_size ? (n_targets - lo) : group_size;
        const group_t g = make_group(pos, acc_old_mag, ordered + lo, cnt);
        out5[5 * gi] = g.cx;
        out5[5 * gi + 1] = g.cy;
        out5[5 * gi + 2] = g.cz;
        out5[5 * gi + 3] = g.radius;
        out5[5 * gi + 4] = g.a_min;
    }
    free(ordered);
    return G2O_OK;
}

/* ---- gravity.cpp:18-43 direct_sum --------------------------------------------- */
typedef struct {
    size_t n, lo, hi;
    const double *mass, *pos;
    double G, eps2;
    double* acc;
    int rc;
} ds_job;

static void* ds_run(void* arg) {
    ds_job* j = arg;
    for (size_t i = j->lo; i < j->hi; ++i) {
        const double rx = j->pos[3 * i], ry = j->pos[3 * i + 1], rz = j->pos[3 * i + 2];
        double ax = 0.0, ay = 0.0, az = 0.0;
        for (size_t k = 0; k < j->n; ++k) {
            if (k == i) continue;
            const double dx = j->pos[3 * k] - rx, dy = j->pos[3 * k + 1] - ry, dz = j->pos[3 * k + 2] - rz;
            const double d2 = dx * dx + dy * dy + dz * dz;
            if (j->eps2 == 0.0 && d2 == 0.0) {
                j->rc = G2O_SINGULAR;
                return NULL;
            }
            const double r2 = d2 + j->eps2; /* softened_accel, gravity.hpp:15-20 */
            if (r2 == 0.0) continue;
            const double inv = 1.0 / sqrt(r2);
            const double f = j->G * j->mass[k] * inv * inv * inv;
            ax += f * dx;
            ay += f * dy;
            az += f * dz;
        }
        j->acc[3 * i] = ax;
        j->acc[3 * i + 1] = ay;
        j->acc[3 * i + 2] = az;
    }
    return NULL;
}

int g2o_direct_sum(size_t n, const double* mass, const double* pos, double G, double eps, unsigned threads,
                   double* acc_out) {
    if (n < 1) return fail(G2O_DATA, "direct_sum: empty system");
    if (threads < 1) threads = 1;
    if (threads > n) threads = (unsigned)n;
    ds_job* jobs = calloc(threads, sizeof *jobs);
    pthread_t* th = calloc(threads, sizeof *th);
    for (unsigned k = 0; k < threads; ++k) {
        jobs[k] = (ds_job){n, n * k / threads, n * (k + 1) / threads, mass, pos, G, eps * eps, acc_out, 0};
        if (k) pthread_create(&th[k], NULL, ds_run, &jobs[k]);
    }
    ds_run(&jobs[0]);
    int rc = 0;
    for (unsigned k = 0; k < threads; ++k) {
        if (k) pthread_join(th[k], NULL);
        if (jobs[k].rc) rc = jobs[k].rc;
    }
    free(jobs);
    free(th);
    if (rc) return fail(rc, "direct_sum: coincident particles with zero softening");
    return G2O_OK;
}

/* ---- integrator.cpp:21-45 ----------------------------------------------------- */
int g2o_block_level(double acc_mag, double eta, double dt_max, int adaptive, int fixed_level, double eps) {
    if (!adaptive) return fixed_level < 0 ? 0 : (fixed_level > 24 ? 24 : fixed_level);
    if (acc_mag <= 0.0) return 0;
    const double dt = eta * sqrt(eps / acc_mag);
    if (dt <= 0.0) return 24;
    if (dt >= dt_max) return 0;
    int level = (int)ceil(log2(dt_max / dt));
    level = level < 0 ? 0 : (level > 24 ? 24 : level);
    while (level < 24 && dt_max / (double)(1ull << level) > dt) ++level;
    while (level > 0 && dt_max / (double)(1ull << (level - 1)) <= dt) --level;
    return level;
}

void g2o_predict(size_t n, double* pos, double* vel, const double* acc, double dt) {
    const double h = 0.5 * dt * dt;
    for (size_t i = 0; i < 3 * n; ++i) {
        pos[i] += vel[i] * dt + acc[i] * h;
        vel[i] += acc[i] * dt;
    }
}

/* ---- rebuild_tuner.cpp:28-61 ---------------------------------------------------- */
static int dcmp(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return x < y ? -1 : (x > y);
}
size_t g2o_autotune(double build_time, size_t n_hist, const double* hist, size_t min_i, size_t max_i, size_t cur) {
    if (n_hist < 2) return cur;
    size_t ns = n_hist * (n_hist - 1) / 2, k = 0;
    double* slopes = malloc(ns * sizeof *slopes);
    for (size_t j = 1; j < n_hist; ++j)
        for (size_t i = 0; i < j; ++i) slopes[k++] = (hist[j] - hist[i]) / (double)(j - i);
    qsort(slopes, ns, sizeof *slopes, dcmp); /* nth_element(mid) == sorted[mid] */
    double slope = slopes[ns / 2];
    if (slope < 0.0) slope = 0.0;
    double* res = malloc(n_hist * sizeof *res);
    for (size_t i = 0; i < n_hist; ++i) res[i] = hist[i] - slope * (double)i;
    qsort(res, n_hist, sizeof *res, dcmp);
    const double intercept = res[n_hist / 2];
    free(slopes);
    free(res);
    size_t best_m = min_i;
    double best = 0.0;
    for (size_t m = min_i; m <= max_i; ++m) {
        const double md = (double)m;
        const double cost = build_time / md + intercept + slope * (md - 1.0) / 2.0;
        if (m == min_i || cost <= best) {
            best = cost;
            best_m = m;
        }
    }
    return best_m;
}
