/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle ("port") of the splb hot path.
 *
 * A plain-C restatement of the reference algorithm, implementing the same
 * C-ABI as include/splbcu.h so the parity tests, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg can drive it through the same Python mirror as
 * the B200 engine.  Single-threaded, literal arithmetic (no folding), built
 * with -ffp-contract=off like the reference (proj/CMakeLists.txt:15).
 * Workers are simulated sequentially; the mailbox exchange becomes memcpy.
 *
 * Parity pinned: tests/test_oracle.py checks this port against the golden
 * vectors in tests/golden/ (made by tests/golden/make_golden.py from the
 * unmodified reference via oracle/_ref/libsplbref.so) and, when present,
 * against oracle/_ref directly.
 *
 * Each function cites the reference file:line it restates
 * (/root/reference/proj/include/splb/...).
 */
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "splbcu.h"

/* ---- errors ---------------------------------------------------------------- */
static __thread char g_err[512];
static int set_err(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}
const char* splbcu_last_error(void) { return g_err; }
const char* splbcu_version(void) { return "splb C oracle (port, single-threaded)"; }

/* ---- lattice (lattice.hpp:20-149) ----------------------------------------- */
#define Q 19
static const int CV[Q][3] = {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
                             {0, 0, 1},  {0, 0, -1},  {1, 1, 0},  {-1, -1, 0}, {1, -1, 0},
                             {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
                             {0, 1, 1},  {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};
static const int INV[Q] = {0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17};
static double W_[Q];
static double CD[Q][3];
static const double CS2 = 1.0 / 3.0;
static void lattice_init(void) {
    static int done = 0;
    if (done) return;
    for (int i = 0; i < Q; ++i) {
        W_[i] = i == 0 ? 1.0 / 3.0 : (i <= 6 ? 1.0 / 18.0 : 1.0 / 36.0);
        for (int a = 0; a < 3; ++a) CD[i][a] = (double)CV[i][a];
    }
    done = 1;
}

typedef struct { double rho, ux, uy, uz; } macro_t;

/* kernel::macro_of (lattice.hpp:106-119) */
static macro_t macro_of(const double* f) {
    double rho = f[0], mx = f[0] * CD[0][0], my = f[0] * CD[0][1], mz = f[0] * CD[0][2];
    for (int i = 1; i < Q; ++i) {
        rho += f[i];
        mx += f[i] * CD[i][0];
        my += f[i] * CD[i][1];
        mz += f[i] * CD[i][2];
    }
    macro_t m = {rho, mx / rho, my / rho, mz / rho};
    return m;
}
/* kernel::usq_term (122-124) */
static double usq_term(const macro_t* m) { return 1.5 * (m->ux * m->ux + m->uy * m->uy + m->uz * m->uz); }
/* kernel::feq (128-133) */
static double feq(int i, const macro_t* m, double usq15) {
    const double cu3 = 3.0 * (CD[i][0] * m->ux + CD[i][1] * m->uy + CD[i][2] * m->uz);
    return W_[i] * m->rho * (1.0 + cu3 + 0.5 * cu3 * cu3 - usq15);
}
/* kernel::relax (136-138) */
static double relax(double f, double fe, double omega) { return f - omega * (f - fe); }
/* kernel::ladd_term (142-147) */
static double ladd_term(int i, double rho, const double ub[3]) {
    const double cu = CD[i][0] * ub[0] + CD[i][1] * ub[1] + CD[i][2] * ub[2];
    return 2.0 * W_[i] * rho * cu * 3.0;
}
static double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

void splbcu_params_default(splbcu_params* p) {
    memset(p, 0, sizeof(*p));
    p->tau = 0.9;
    p->rho0 = 1.0;
    p->dt_s = 1.0;
    p->workers = 1;
    p->exchange_timeout_s = 30.0;
}

/* equilibrium (lattice.hpp:152-158) */
void splbcu_equilibrium(double rho, const double u[3], double out[19]) {
    lattice_init();
    macro_t m = {rho, u[0], u[1], u[2]};
    const double usq = usq_term(&m);
    for (int i = 0; i < Q; ++i) out[i] = feq(i, &m, usq);
}
/* moments (lattice.hpp:162-170) */
int splbcu_moments(const double f[19], double* rho, double u[3]) {
    lattice_init();
    double r = f[0];
    for (int i = 1; i < Q; ++i) r += f[i];
    if (!(r > 0.0)) return set_err(SPLBCU_ERR_DEGENERATE, "moments: non-positive density rho=%f", r);
    macro_t m = macro_of(f);
    *rho = m.rho;
    u[0] = m.ux, u[1] = m.uy, u[2] = m.uz;
    return 0;
}
/* bgk_collide (lattice.hpp:173-185) */
int splbcu_bgk_collide(const double f[19], double tau, double out[19]) {
    lattice_init();
    if (!(tau > 1.0 / 2.0))
        return set_err(SPLBCU_ERR_RUNTIME, "RelaxationParams: tau must exceed dt/2, got tau=%f dt=%f", tau, 1.0);
    double r = f[0];
    for (int i = 1; i < Q; ++i) r += f[i];
    if (!(r > 0.0)) return set_err(SPLBCU_ERR_DEGENERATE, "bgk_collide: non-positive density rho=%f", r);
    macro_t m = macro_of(f);
    const double usq = usq_term(&m), omega = 1.0 / tau;
    for (int i = 0; i < Q; ++i) out[i] = relax(f[i], feq(i, &m, usq), omega);
    return 0;
}

/* ---- TimeTable (boundary.hpp:18-74) ----------------------------------------- */
typedef struct { double* t; double* v; uint32_t n; double period; } table_t;

static int table_validate(const table_t* tb) {
    if (tb->n == 0) return set_err(SPLBCU_ERR_CONFIG, "time table: empty table");
    for (uint32_t k = 1; k < tb->n; ++k)
        if (!(tb->t[k] > tb->t[k - 1])) return set_err(SPLBCU_ERR_CONFIG, "time table: times must be strictly ascending");
    if (tb->period != 0.0) {
        if (!(tb->period > 0.0)) return set_err(SPLBCU_ERR_CONFIG, "time table: period must be > 0");
        if (!(tb->t[tb->n - 1] < tb->period)) return set_err(SPLBCU_ERR_CONFIG, "time table: nodes must lie inside one period");
        if (!(tb->t[0] >= 0.0)) return set_err(SPLBCU_ERR_CONFIG, "time table: periodic table starts before t=0");
    }
    return 0;
}
static double table_at(const table_t* tb, double t) {
    if (tb->n == 1 && tb->period == 0.0) return tb->v[0];
    double tbq = t;
    if (tb->period > 0.0) {
        tbq = fmod(t, tb->period);
        if (tbq < 0.0) tbq += tb->period;
    }
    for (uint32_t k = 0; k < tb->n; ++k)
        if (tbq == tb->t[k]) return tb->v[k];
    if (tb->period == 0.0) {
        if (tbq <= tb->t[0]) return tb->v[0];
        if (tbq >= tb->t[tb->n - 1]) return tb->v[tb->n - 1];
    }
    uint32_t after = 0; /* upper_bound */
    while (after < tb->n && !(tbq < tb->t[after])) ++after;
    double t0, v0, t1, v1;
    if (after == 0) {
        t0 = tb->t[tb->n - 1] - tb->period, v0 = tb->v[tb->n - 1], t1 = tb->t[0], v1 = tb->v[0];
    } else if (after == tb->n) {
        t0 = tb->t[tb->n - 1], v0 = tb->v[tb->n - 1], t1 = tb->t[0] + tb->period, v1 = tb->v[0];
    } else {
        t0 = tb->t[after - 1], v0 = tb->v[after - 1], t1 = tb->t[after], v1 = tb->v[after];
    }
    return v0 + (v1 - v0) * ((tbq - t0) / (t1 - t0));
}
int splbcu_timetable_at(const double* t, const double* v, uint32_t n, double period, double tq, double* out) {
    table_t tb = {(double*)t, (double*)v, n, period};
    int rc = table_validate(&tb);
    if (rc) return rc;
    *out = table_at(&tb, tq);
    return 0;
}

/* iolet_weight (boundary.hpp:107-113) */
static double weight_of(const splbcu_iolet* io, const int32_t* c) {
    const double d[3] = {(double)c[0] - io->center[0], (double)c[1] - io->center[1], (double)c[2] - io->center[2]};
    const double axial = dot3(d, io->normal);
    const double r[3] = {d[0] - io->normal[0] * axial, d[1] - io->normal[1] * axial, d[2] - io->normal[2] * axial};
    const double w = 1.0 - dot3(r, r) / (io->radius * io->radius);
    return w < 0.0 ? 0.0 : (w > 1.0 ? 1.0 : w);
}
double splbcu_iolet_weight(const splbcu_iolet* io, const int32_t c[3]) { return weight_of(io, c); }

/* ---- domain (geometry.hpp:64-271) ------------------------------------------- */
struct splbcu_domain {
    double voxel_size;
    uint64_t n;
    int32_t* coords;
    uint8_t* types;
    uint8_t* kind;
    uint16_t* iol;
    splbcu_iolet* iolets;
    uint32_t nio;
    uint64_t tr[12];
    /* lookup: keys sorted + site index */
    uint64_t* skeys;
    uint32_t* sidx;
};

/* coord_key (geometry.hpp:82-86) */
static uint64_t coord_key(int32_t x, int32_t y, int32_t z) {
    const int64_t b = (int64_t)1 << 20;
    return ((uint64_t)(x + b) << 42) | ((uint64_t)(y + b) << 21) | (uint64_t)(z + b);
}
typedef struct { uint64_t k; uint32_t i; } kv_t;
static int kv_cmp(const void* a, const void* b) {
    const kv_t* x = a;
    const kv_t* y = b;
    if (x->k != y->k) return x->k < y->k ? -1 : 1;
    return x->i < y->i ? -1 : (x->i > y->i);
}
/* index_coords (geometry.hpp:90-98): a sorted key table; duplicates rejected */
static int build_index(const int32_t* c, uint64_t n, uint64_t** keys, uint32_t** idx) {
    kv_t* kv = malloc(sizeof(kv_t) * (n ? n : 1));
    for (uint64_t s = 0; s < n; ++s) kv[s].k = coord_key(c[3 * s], c[3 * s + 1], c[3 * s + 2]), kv[s].i = (uint32_t)s;
    qsort(kv, n, sizeof(kv_t), kv_cmp);
    for (uint64_t s = 1; s < n; ++s)
        if (kv[s].k == kv[s - 1].k) {
            free(kv);
            return set_err(SPLBCU_ERR_GEOMETRY, "classify_sites: duplicate voxel");
        }
    *keys = malloc(8 * (n ? n : 1));
    *idx = malloc(4 * (n ? n : 1));
    for (uint64_t s = 0; s < n; ++s) (*keys)[s] = kv[s].k, (*idx)[s] = kv[s].i;
    free(kv);
    return 0;
}
static int64_t lookup(const uint64_t* keys, const uint32_t* idx, uint64_t n, int32_t x, int32_t y, int32_t z) {
    const uint64_t k = coord_key(x, y, z);
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t m = (lo + hi) / 2;
        if (keys[m] < k) lo = m + 1;
        else hi = m;
    }
    return (lo < n && keys[lo] == k) ? (int64_t)idx[lo] : -1;
}
static int64_t dom_find(const struct splbcu_domain* d, int32_t x, int32_t y, int32_t z) {
    return lookup(d->skeys, d->sidx, d->n, x, y, z);
}

static void domain_free(struct splbcu_domain* d) {
    if (!d) return;
    free(d->coords), free(d->types), free(d->kind), free(d->iol), free(d->iolets), free(d->skeys), free(d->sidx);
    free(d);
}
void splbcu_domain_free(splbcu_domain* d) { domain_free(d); }

/* crosses_iolet (geometry.hpp:102-113) */
static int crosses(const double a[3], const double b[3], const splbcu_iolet* io) {
    const double da[3] = {a[0] - io->center[0], a[1] - io->center[1], a[2] - io->center[2]};
    const double db[3] = {b[0] - io->center[0], b[1] - io->center[1], b[2] - io->center[2]};
    const double sa = dot3(da, io->normal), sb = dot3(db, io->normal);
    if (!(sa > 0.0 && sb <= 0.0)) return 0;
    const double t = sa / (sa - sb);
    const double p[3] = {a[0] + t * (b[0] - a[0]), a[1] + t * (b[1] - a[1]), a[2] + t * (b[2] - a[2])};
    const double dd[3] = {p[0] - io->center[0], p[1] - io->center[1], p[2] - io->center[2]};
    const double r2 = dot3(dd, dd);
    const double rmax = io->radius + 1.0;
    return r2 <= rmax * rmax;
}

static const struct splbcu_domain* g_sort_dom;
static int site_cmp(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    const struct splbcu_domain* d = g_sort_dom;
    if (d->types[x] != d->types[y]) return d->types[x] < d->types[y] ? -1 : 1;
    for (int ax = 2; ax >= 0; --ax)
        if (d->coords[3 * x + ax] != d->coords[3 * y + ax]) return d->coords[3 * x + ax] < d->coords[3 * y + ax] ? -1 : 1;
    return 0;
}

static int norm_ok(const splbcu_iolet* io) { return !(fabs(sqrt(dot3(io->normal, io->normal)) - 1.0) > 1e-12); }

/* classify_sites (geometry.hpp:139-208) */
int splbcu_domain_classify(const int32_t* vox, uint64_t n, const splbcu_iolet* iolets, uint32_t nio, double vs,
                           splbcu_domain** out) {
    if (n == 0) return set_err(SPLBCU_ERR_GEOMETRY, "classify_sites: empty voxel set");
    for (uint32_t k = 0; k < nio; ++k)
        if (!norm_ok(&iolets[k])) return set_err(SPLBCU_ERR_GEOMETRY, "classify_sites: iolet %u normal is not unit length", k);
    struct splbcu_domain* t = calloc(1, sizeof *t);
    t->n = n;
    t->coords = malloc(12 * n);
    memcpy(t->coords, vox, 12 * n);
    int rc = build_index(t->coords, n, &t->skeys, &t->sidx);
    if (rc) {
        domain_free(t);
        return rc;
    }
    t->types = malloc(n);
    t->kind = malloc(18 * n);
    t->iol = calloc(18 * n, 2);
    uint64_t* cnt = calloc(nio ? nio : 1, 8);
    for (uint64_t s = 0; s < n; ++s) {
        const int32_t* c = &t->coords[3 * s];
        const double a[3] = {c[0], c[1], c[2]};
        int wall = 0, inlet = 0, outlet = 0;
        for (int i = 1; i < Q; ++i) {
            const int32_t tx = c[0] + CV[i][0], ty = c[1] + CV[i][1], tz = c[2] + CV[i][2];
            uint8_t k = 0;
            uint16_t id = 0;
            if (dom_find(t, tx, ty, tz) < 0) {
                k = 1;
                const double b[3] = {tx, ty, tz};
                for (uint32_t io = 0; io < nio; ++io)
                    if (crosses(a, b, &iolets[io])) {
                        k = iolets[io].kind == 0 ? 2 : 3;
                        id = (uint16_t)io;
                        ++cnt[io];
                        break;
                    }
            }
            t->kind[18 * s + i - 1] = k;
            t->iol[18 * s + i - 1] = id;
            wall |= k == 1, inlet |= k == 2, outlet |= k == 3;
        }
        if (inlet && outlet) {
            set_err(SPLBCU_ERR_GEOMETRY, "classify_sites: site (%d,%d,%d) carries both inlet and outlet links", c[0],
                    c[1], c[2]);
            free(cnt);
            domain_free(t);
            return SPLBCU_ERR_GEOMETRY;
        }
        t->types[s] = inlet ? (wall ? 4 : 2) : outlet ? (wall ? 5 : 3) : (wall ? 1 : 0);
    }
    for (uint32_t io = 0; io < nio; ++io)
        if (cnt[io] == 0) {
            free(cnt);
            domain_free(t);
            return set_err(SPLBCU_ERR_GEOMETRY, "classify_sites: iolet %u intersects no boundary links", io);
        }
    free(cnt);
    /* stable order by (type, z, y, x) — keys are unique so qsort is exact */
    uint32_t* ord = malloc(4 * n);
    for (uint64_t s = 0; s < n; ++s) ord[s] = (uint32_t)s;
    g_sort_dom = t;
    qsort(ord, n, 4, site_cmp);
    struct splbcu_domain* d = calloc(1, sizeof *d);
    d->n = n;
    d->voxel_size = vs;
    d->coords = malloc(12 * n);
    d->types = malloc(n);
    d->kind = malloc(18 * n);
    d->iol = malloc(36 * n);
    for (uint64_t g = 0; g < n; ++g) {
        const uint32_t s = ord[g];
        memcpy(&d->coords[3 * g], &t->coords[3 * s], 12);
        d->types[g] = t->types[s];
        memcpy(&d->kind[18 * g], &t->kind[18 * s], 18);
        memcpy(&d->iol[18 * g], &t->iol[18 * s], 36);
    }
    free(ord);
    domain_free(t);
    d->nio = nio;
    d->iolets = malloc(sizeof(splbcu_iolet) * (nio ? nio : 1));
    memcpy(d->iolets, iolets, sizeof(splbcu_iolet) * nio);
    uint64_t pos = 0;
    for (int ty = 0; ty < 6; ++ty) {
        d->tr[2 * ty] = pos;
        while (pos < n && d->types[pos] == ty) ++pos;
        d->tr[2 * ty + 1] = pos;
    }
    build_index(d->coords, n, &d->skeys, &d->sidx);
    *out = d;
    return 0;
}

/* validate_domain (geometry.hpp:212-271) */
int splbcu_domain_validate(const splbcu_domain* d) {
    if (d->n == 0) return set_err(SPLBCU_ERR_GEOMETRY, "domain: empty site list");
    if (!(d->voxel_size > 0.0)) return set_err(SPLBCU_ERR_GEOMETRY, "domain: voxel size must be positive");
    for (uint32_t k = 0; k < d->nio; ++k)
        if (!norm_ok(&d->iolets[k])) return set_err(SPLBCU_ERR_GEOMETRY, "domain: iolet %u normal is not unit length", k);
    uint64_t pos = 0;
    for (int t = 0; t < 6; ++t) {
        if (d->tr[2 * t] != pos || d->tr[2 * t + 1] < pos || d->tr[2 * t + 1] > d->n)
            return set_err(SPLBCU_ERR_GEOMETRY, "domain: type_ranges do not partition the sites");
        pos = d->tr[2 * t + 1];
        for (uint64_t s = d->tr[2 * t]; s < d->tr[2 * t + 1]; ++s)
            if (d->types[s] != t) return set_err(SPLBCU_ERR_GEOMETRY, "domain: site type outside its range");
    }
    if (pos != d->n) return set_err(SPLBCU_ERR_GEOMETRY, "domain: type_ranges do not partition the sites");
    for (uint64_t s = 0; s < d->n; ++s) {
        int wall = 0, inlet = 0, outlet = 0;
        const int32_t* c = &d->coords[3 * s];
        for (int i = 1; i < Q; ++i) {
            const uint8_t k = d->kind[18 * s + i - 1];
            const int in_set = dom_find(d, c[0] + CV[i][0], c[1] + CV[i][1], c[2] + CV[i][2]) >= 0;
            if (k == 0) {
                if (!in_set) return set_err(SPLBCU_ERR_GEOMETRY, "domain: inconsistent link closure");
            } else {
                if (in_set) return set_err(SPLBCU_ERR_GEOMETRY, "domain: inconsistent link closure");
                if (k != 1 && d->iol[18 * s + i - 1] >= d->nio)
                    return set_err(SPLBCU_ERR_GEOMETRY, "domain: link references unknown iolet");
            }
            wall |= k == 1, inlet |= k == 2, outlet |= k == 3;
        }
        if (inlet && outlet) return set_err(SPLBCU_ERR_GEOMETRY, "domain: site carries both inlet and outlet links");
        const int expect = inlet ? (wall ? 4 : 2) : outlet ? (wall ? 5 : 3) : (wall ? 1 : 0);
        if (d->types[s] != expect) return set_err(SPLBCU_ERR_GEOMETRY, "domain: collision type inconsistent with links");
    }
    return 0;
}

static splbcu_iolet mk_iolet(int kind, double cx_, double cy_, double cz_, double nz_, double r) {
    splbcu_iolet io;
    io.kind = kind;
    io.center[0] = cx_, io.center[1] = cy_, io.center[2] = cz_;
    io.normal[0] = 0.0, io.normal[1] = 0.0, io.normal[2] = nz_;
    io.radius = r;
    return io;
}

/* build_pipe (geometry.hpp:285-308) */
int splbcu_domain_build_pipe(int32_t radius, int32_t length, double vs, splbcu_domain** out) {
    if (radius < 2 || length < 4) return set_err(SPLBCU_ERR_GEOMETRY, "build_pipe: need radius >= 2 and length >= 4");
    const double r2 = (double)radius * radius;
    uint64_t cap = 1024, n = 0;
    int32_t* v = malloc(12 * cap);
    for (int z = 0; z < length; ++z)
        for (int y = -radius - 2; y <= radius + 2; ++y)
            for (int x = -radius - 2; x <= radius + 2; ++x) {
                const double dx = x - 0.375, dy = y - 0.5;
                if (dx * dx + dy * dy < r2) {
                    if (n == cap) v = realloc(v, 12 * (cap *= 2));
                    v[3 * n] = x, v[3 * n + 1] = y, v[3 * n + 2] = z, ++n;
                }
            }
    splbcu_iolet io[2] = {mk_iolet(0, 0.375, 0.5, -0.5, 1.0, radius),
                          mk_iolet(1, 0.375, 0.5, (double)(length - 1) + 0.5, -1.0, radius)};
    int rc = splbcu_domain_classify(v, n, io, 2, vs, out);
    free(v);
    return rc;
}

/* build_bifurcation (geometry.hpp:313-363) */
int splbcu_domain_build_bifurcation(int32_t tr, int32_t br, int32_t tl, int32_t bl, double vs, splbcu_domain** out) {
    if (tr < 2 || br < 2 || tl < 4 || bl < 4)
        return set_err(SPLBCU_ERR_GEOMETRY, "build_bifurcation: need radii >= 2 and lengths >= 4");
    const double slope = 0.5;
    const int xmax = (int)ceil(slope * bl) + tr + br + 2;
    const int rmax = (tr > br ? tr : br) + 2;
    uint64_t cap = 1024, n = 0;
    int32_t* v = malloc(12 * cap);
    for (int z = 0; z < tl + bl; ++z)
        for (int y = -rmax; y <= rmax; ++y)
            for (int x = -xmax; x <= xmax; ++x) {
                const double dy = y - 0.5;
                int fluid;
                if (z < tl) {
                    const double dx = x - 0.375;
                    fluid = dx * dx + dy * dy < tr * tr;
                } else {
                    const double xc = slope * (z - tl + 1);
                    const double dp = (x - 0.375 - xc), dm = (x - 0.375 + xc);
                    fluid = dp * dp + dy * dy < br * br || dm * dm + dy * dy < br * br;
                }
                if (fluid) {
                    if (n == cap) v = realloc(v, 12 * (cap *= 2));
                    v[3 * n] = x, v[3 * n + 1] = y, v[3 * n + 2] = z, ++n;
                }
            }
    const double zend = (double)(tl + bl - 1) + 0.5, xend = slope * bl;
    splbcu_iolet io[3] = {mk_iolet(0, 0.375, 0.5, -0.5, 1.0, tr), mk_iolet(1, 0.375 + xend, 0.5, zend, -1.0, br),
                          mk_iolet(1, 0.375 - xend, 0.5, zend, -1.0, br)};
    int rc = splbcu_domain_classify(v, n, io, 3, vs, out);
    free(v);
    return rc;
}
int splbcu_domain_build_tree(int32_t a, int32_t b, int32_t c, double d_, double e, double f, splbcu_domain** o) {
    (void)a, (void)b, (void)c, (void)d_, (void)e, (void)f, (void)o;
    return set_err(SPLBCU_ERR_CONFIG, "oracle: the tree generator is product-only; pass its arrays");
}
int splbcu_domain_build_channel(int32_t a, int32_t b, int32_t c, double d_, splbcu_domain** o) {
    (void)a, (void)b, (void)c, (void)d_, (void)o;
    return set_err(SPLBCU_ERR_CONFIG, "oracle: the channel generator is product-only; pass its arrays");
}

int splbcu_domain_from_arrays(uint64_t n, const int32_t* coords, const uint8_t* types, const uint8_t* kind,
                              const uint16_t* iol, const splbcu_iolet* io, uint32_t nio, const uint64_t* tr,
                              double vs, splbcu_domain** out) {
    struct splbcu_domain* d = calloc(1, sizeof *d);
    d->n = n;
    d->voxel_size = vs;
    d->coords = malloc(12 * (n ? n : 1));
    memcpy(d->coords, coords, 12 * n);
    d->types = malloc(n ? n : 1);
    memcpy(d->types, types, n);
    d->kind = malloc(18 * (n ? n : 1));
    memcpy(d->kind, kind, 18 * n);
    d->iol = calloc(18 * (n ? n : 1), 2);
    for (uint64_t q = 0; q < 18 * n; ++q) d->iol[q] = kind[q] >= 2 && iol ? iol[q] : 0;
    d->nio = nio;
    d->iolets = malloc(sizeof(splbcu_iolet) * (nio ? nio : 1));
    memcpy(d->iolets, io, sizeof(splbcu_iolet) * nio);
    memcpy(d->tr, tr, sizeof d->tr);
    int rc = build_index(d->coords, n, &d->skeys, &d->sidx);
    if (!rc) rc = splbcu_domain_validate(d);
    if (rc) {
        domain_free(d);
        return rc;
    }
    *out = d;
    return 0;
}
int splbcu_domain_read(const char* p, splbcu_domain** o) {
    (void)p, (void)o;
    return set_err(SPLBCU_ERR_CONFIG, "oracle: no file I/O");
}
int splbcu_domain_write(const splbcu_domain* d, const char* p) {
    (void)d, (void)p;
    return set_err(SPLBCU_ERR_CONFIG, "oracle: no file I/O");
}
uint64_t splbcu_domain_n_sites(const splbcu_domain* d) { return d->n; }
uint32_t splbcu_domain_n_iolets(const splbcu_domain* d) { return d->nio; }
double splbcu_domain_voxel_size(const splbcu_domain* d) { return d->voxel_size; }
int splbcu_domain_export(const splbcu_domain* d, int32_t* coords, uint8_t* types, uint8_t* kind, uint16_t* iol,
                         splbcu_iolet* io, uint64_t* tr) {
    if (coords) memcpy(coords, d->coords, 12 * d->n);
    if (types) memcpy(types, d->types, d->n);
    if (kind) memcpy(kind, d->kind, 18 * d->n);
    if (iol) memcpy(iol, d->iol, 36 * d->n);
    if (io) memcpy(io, d->iolets, sizeof(splbcu_iolet) * d->nio);
    if (tr) memcpy(tr, d->tr, sizeof d->tr);
    return 0;
}

/* ---- partition (decomp.hpp:65-188) ------------------------------------------ */
typedef struct {
    uint32_t* sites;
    uint32_t n, n_edge;
    uint64_t er[12], mr[12];
    int32_t* nb;
    uint32_t n_nb;
} part_t;
struct splbcu_partition {
    int W;
    uint64_t n;
    int32_t* owner;
    uint32_t* local;
    part_t* parts;
    int borrowed;
};

static int g_axis;
static const int32_t* g_c;
static int geo_cmp(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    const int32_t *ca = &g_c[3 * x], *cb = &g_c[3 * y];
    if (ca[g_axis] != cb[g_axis]) return ca[g_axis] < cb[g_axis] ? -1 : 1;
    for (int ax = 2; ax >= 0; --ax)
        if (ca[ax] != cb[ax]) return ca[ax] < cb[ax] ? -1 : 1;
    return 0;
}

static void part_free(struct splbcu_partition* p) {
    if (!p) return;
    for (int w = 0; w < p->W; ++w) free(p->parts[w].sites), free(p->parts[w].nb);
    free(p->parts), free(p->owner), free(p->local), free(p);
}
void splbcu_partition_free(splbcu_partition* p) {
    if (p && !p->borrowed) part_free(p);
}

static int do_partition(const struct splbcu_domain* d, int W, struct splbcu_partition** out) {
    const uint64_t n = d->n;
    if (W < 1) return set_err(SPLBCU_ERR_RUNTIME, "partition: nWorkers must be >= 1");
    if ((uint64_t)W > n)
        return set_err(SPLBCU_ERR_RUNTIME, "partition: nWorkers (%d) exceeds site count (%llu)", W, (unsigned long long)n);
    struct splbcu_partition* p = calloc(1, sizeof *p);
    p->W = W;
    p->n = n;
    p->owner = calloc(n, 4);
    p->local = calloc(n, 4);
    /* longest_axis (decomp.hpp:44-56) */
    int32_t lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    for (uint64_t s = 0; s < n; ++s)
        for (int a = 0; a < 3; ++a) {
            if (d->coords[3 * s + a] < lo[a]) lo[a] = d->coords[3 * s + a];
            if (d->coords[3 * s + a] > hi[a]) hi[a] = d->coords[3 * s + a];
        }
    int axis = 2;
    for (int a = 1; a >= 0; --a)
        if (hi[a] - lo[a] > hi[axis] - lo[axis]) axis = a;
    uint32_t* order = malloc(4 * n);
    for (uint64_t s = 0; s < n; ++s) order[s] = (uint32_t)s;
    g_axis = axis, g_c = d->coords;
    qsort(order, n, 4, geo_cmp);
    /* plane counts in ascending plane order (the std::map of decomp.hpp:90) */
    uint64_t np = 0;
    int32_t* plane = malloc(4 * n);
    uint64_t* pc = malloc(8 * n);
    for (uint64_t k = 0; k < n; ++k) {
        const int32_t c = d->coords[3 * order[k] + axis];
        if (np == 0 || plane[np - 1] != c) plane[np] = c, pc[np] = 0, ++np;
        ++pc[np - 1];
    }
    if ((uint64_t)W <= np) {
        int32_t* cut = malloc(4 * (size_t)W);
        uint64_t it = 0, rem_sites = n, rem_planes = np;
        for (int w = 0; w < W - 1; ++w) {
            const uint64_t left = (uint64_t)(W - w);
            const uint64_t target = (rem_sites + left - 1) / left;
            uint64_t taken = 0, pt = 0;
            while (it != np && rem_planes - pt > (uint64_t)(W - 1 - w)) {
                if (pt > 0 && taken >= target) break;
                taken += pc[it];
                ++pt;
                ++it;
            }
            cut[w] = plane[it - 1];
            rem_sites -= taken;
            rem_planes -= pt;
        }
        for (uint64_t s = 0; s < n; ++s) {
            const int32_t c = d->coords[3 * s + axis];
            int w = 0;
            while (w < W - 1 && c > cut[w]) ++w;
            p->owner[s] = w;
        }
        free(cut);
    } else {
        const uint64_t q = n / (uint64_t)W, r = n % (uint64_t)W;
        uint64_t pos = 0;
        for (int w = 0; w < W; ++w) {
            const uint64_t take = q + ((uint64_t)w < r ? 1 : 0);
            for (uint64_t k = 0; k < take; ++k) p->owner[order[pos++]] = w;
        }
    }
    free(order), free(plane), free(pc);
    /* edges (decomp.hpp:132-153) */
    char* edge = calloc(n, 1);
    char* nbm = calloc((size_t)W * W, 1);
    for (uint64_t s = 0; s < n; ++s) {
        const int32_t* c = &d->coords[3 * s];
        for (int i = 1; i < Q; ++i) {
            if (d->kind[18 * s + i - 1] != 0) continue;
            const int64_t t = dom_find(d, c[0] + CV[i][0], c[1] + CV[i][1], c[2] + CV[i][2]);
            if (p->owner[t] != p->owner[s]) edge[s] = 1, nbm[(size_t)p->owner[s] * W + p->owner[t]] = 1;
        }
    }
    p->parts = calloc((size_t)W, sizeof(part_t));
    for (uint64_t s = 0; s < n; ++s) p->parts[p->owner[s]].n++;
    for (int w = 0; w < W; ++w) p->parts[w].sites = malloc(4 * (p->parts[w].n ? p->parts[w].n : 1)), p->parts[w].n = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (uint64_t s = 0; s < n; ++s)
            if ((pass == 0) == (edge[s] != 0)) {
                part_t* pt = &p->parts[p->owner[s]];
                p->local[s] = pt->n;
                pt->sites[pt->n++] = (uint32_t)s;
                if (pass == 0) pt->n_edge++;
            }
    for (int w = 0; w < W; ++w) {
        part_t* pt = &p->parts[w];
        pt->nb = malloc(4 * (size_t)W);
        for (int v = 0; v < W; ++v)
            if (nbm[(size_t)w * W + v]) pt->nb[pt->n_nb++] = v;
        uint64_t pos = 0;
        for (int t = 0; t < 6; ++t) {
            pt->er[2 * t] = pos;
            while (pos < pt->n_edge && d->types[pt->sites[pos]] == t) ++pos;
            pt->er[2 * t + 1] = pos;
        }
        pos = pt->n_edge;
        for (int t = 0; t < 6; ++t) {
            pt->mr[2 * t] = pos;
            while (pos < pt->n && d->types[pt->sites[pos]] == t) ++pos;
            pt->mr[2 * t + 1] = pos;
        }
    }
    free(edge), free(nbm);
    *out = p;
    return 0;
}

int splbcu_partition_create(const splbcu_domain* d, int32_t W, splbcu_partition** out) { return do_partition(d, W, out); }
int splbcu_partition_global(const splbcu_partition* p, int32_t* owner, uint32_t* li) {
    if (owner) memcpy(owner, p->owner, 4 * p->n);
    if (li) memcpy(li, p->local, 4 * p->n);
    return 0;
}
int splbcu_partition_part_shape(const splbcu_partition* p, int32_t w, uint32_t* ns, uint32_t* ne, uint32_t* nn) {
    if (w < 0 || w >= p->W) return set_err(SPLBCU_ERR_CONFIG, "partition: worker out of range");
    if (ns) *ns = p->parts[w].n;
    if (ne) *ne = p->parts[w].n_edge;
    if (nn) *nn = p->parts[w].n_nb;
    return 0;
}
int splbcu_partition_part(const splbcu_partition* p, int32_t w, uint32_t* sites, uint64_t* er, uint64_t* mr, int32_t* nb) {
    if (w < 0 || w >= p->W) return set_err(SPLBCU_ERR_CONFIG, "partition: worker out of range");
    const part_t* pt = &p->parts[w];
    if (sites) memcpy(sites, pt->sites, 4 * pt->n);
    if (er) memcpy(er, pt->er, sizeof pt->er);
    if (mr) memcpy(mr, pt->mr, sizeof pt->mr);
    if (nb) memcpy(nb, pt->nb, 4 * pt->n_nb);
    return 0;
}
double splbcu_partition_imbalance(const splbcu_partition* p) {
    uint64_t lo = UINT64_MAX, hi = 0;
    for (int w = 0; w < p->W; ++w) {
        if (p->parts[w].n < lo) lo = p->parts[w].n;
        if (p->parts[w].n > hi) hi = p->parts[w].n;
    }
    return lo == 0 ? INFINITY : (double)hi / (double)lo;
}

/* ---- streaming maps (layout.hpp:153-286) and exchange (exchange.hpp) --------- */
typedef struct { uint32_t site; uint8_t dir; uint32_t target; } xlink_t;
typedef struct { xlink_t* v; uint32_t n, cap; } xlist_t;

typedef struct {
    uint32_t n, shared;
    uint32_t* dest;   /* 18n */
    uint8_t* op;
    uint16_t* iol;
    uint32_t* recv_dest;
    uint32_t* send_site;
    uint8_t* send_dir;
    int32_t* seg_nb;
    uint32_t *seg_base, *seg_count, n_seg;
    /* store */
    double *fa, *fb;
    int a_old;
} worker_t;

struct splbcu_sim {
    struct splbcu_domain* dom; /* borrowed pointer copy semantics: we keep our own copy */
    struct splbcu_partition* part;
    splbcu_params prm;
    double omega;
    table_t* tables;
    int* bc_kind;
    uint32_t nbc;
    worker_t* wk;
    double** mail; /* per (from,to): message buffer */
    uint32_t* mail_n;
    uint64_t steps;
    double loop_s;
    /* captures */
    uint64_t ncap;
    uint64_t* cap_step;
    double** cap_f;
    /* series */
    uint64_t rows;
    double **smax, **sp, **sq; /* [iolet] arrays of rows */
    /* per (iolet) obs site list (global ascending) */
    uint32_t** obs;
    uint32_t* nobs;
    double* staged; /* per iolet */
    int* staged_vel;
};

static size_t sidx(const worker_t* w, int layout, uint32_t s, int i) {
    return layout == 0 ? (size_t)Q * s + i : (size_t)i * w->n + s;
}
static double* f_old(worker_t* w) { return w->a_old ? w->fa : w->fb; }
static double* f_new(worker_t* w) { return w->a_old ? w->fb : w->fa; }

static void xpush(xlist_t* l, xlink_t x) {
    if (l->n == l->cap) l->v = realloc(l->v, sizeof(xlink_t) * (l->cap = l->cap ? 2 * l->cap : 16));
    l->v[l->n++] = x;
}

/* build_cross_links (layout.hpp:153-176) + build_streaming_map (181-286) */
static int build_maps(struct splbcu_sim* S) {
    const struct splbcu_domain* d = S->dom;
    const struct splbcu_partition* pa = S->part;
    const int W = pa->W;
    xlist_t* cross = calloc((size_t)W * W, sizeof(xlist_t));
    for (uint64_t s = 0; s < d->n; ++s) {
        const int32_t* c = &d->coords[3 * s];
        for (int i = 1; i < Q; ++i) {
            if (d->kind[18 * s + i - 1] != 0) continue;
            const int64_t t = dom_find(d, c[0] + CV[i][0], c[1] + CV[i][1], c[2] + CV[i][2]);
            if (pa->owner[s] != pa->owner[t]) {
                xlink_t x = {(uint32_t)s, (uint8_t)i, (uint32_t)t};
                xpush(&cross[(size_t)pa->owner[s] * W + pa->owner[t]], x);
            }
        }
    }
    for (int w = 0; w < W; ++w) {
        worker_t* wk = &S->wk[w];
        const part_t* pt = &pa->parts[w];
        wk->n = pt->n;
        wk->n_seg = pt->n_nb;
        wk->seg_nb = malloc(4 * (pt->n_nb + 1));
        wk->seg_base = malloc(4 * (pt->n_nb + 1));
        wk->seg_count = malloc(4 * (pt->n_nb + 1));
        uint32_t base = 0;
        for (uint32_t k = 0; k < pt->n_nb; ++k) {
            const int nb = pt->nb[k];
            const uint32_t cnt = cross[(size_t)w * W + nb].n, rcnt = cross[(size_t)nb * W + w].n;
            if (cnt != rcnt) return set_err(SPLBCU_ERR_RUNTIME, "build_streaming_map: asymmetric cross-link counts");
            wk->seg_nb[k] = nb, wk->seg_base[k] = base, wk->seg_count[k] = cnt;
            base += cnt;
        }
        wk->shared = base;
        wk->recv_dest = calloc(base + 1, 4);
        wk->send_site = calloc(base + 1, 4);
        wk->send_dir = calloc(base + 1, 1);
        /* slot of each outgoing (site, dir): per site a small table */
        uint32_t* slot_of = malloc(4 * 18 * (size_t)(pt->n ? pt->n : 1));
        for (size_t q = 0; q < 18 * (size_t)pt->n; ++q) slot_of[q] = UINT32_MAX;
        for (uint32_t k = 0; k < pt->n_nb; ++k) {
            const int nb = pt->nb[k];
            const xlist_t* outl = &cross[(size_t)w * W + nb];
            for (uint32_t j = 0; j < outl->n; ++j) {
                const uint32_t sl = pa->local[outl->v[j].site];
                slot_of[18 * (size_t)sl + outl->v[j].dir - 1] = wk->seg_base[k] + j;
                wk->send_site[wk->seg_base[k] + j] = sl;
                wk->send_dir[wk->seg_base[k] + j] = outl->v[j].dir;
            }
            const xlist_t* inl = &cross[(size_t)nb * W + w];
            for (uint32_t j = 0; j < inl->n; ++j)
                wk->recv_dest[wk->seg_base[k] + j] = (uint32_t)sidx(wk, S->prm.layout, pa->local[inl->v[j].target], inl->v[j].dir);
        }
        wk->dest = malloc(4 * 18 * (size_t)(pt->n ? pt->n : 1));
        wk->op = malloc(18 * (size_t)(pt->n ? pt->n : 1));
        wk->iol = malloc(36 * (size_t)(pt->n ? pt->n : 1));
        for (uint32_t sl = 0; sl < pt->n; ++sl) {
            const uint32_t g = pt->sites[sl];
            const int32_t* c = &d->coords[3 * (size_t)g];
            for (int i = 1; i < Q; ++i) {
                const size_t q = 18 * (size_t)sl + i - 1;
                const uint8_t k = d->kind[18 * (size_t)g + i - 1];
                wk->iol[q] = 0;
                if (k == 0) {
                    const int64_t tg = dom_find(d, c[0] + CV[i][0], c[1] + CV[i][1], c[2] + CV[i][2]);
                    if (pa->owner[tg] == w) {
                        wk->dest[q] = (uint32_t)sidx(wk, S->prm.layout, pa->local[tg], i);
                        wk->op[q] = 0;
                    } else {
                        wk->dest[q] = (uint32_t)((size_t)Q * pt->n + slot_of[q]);
                        wk->op[q] = 1;
                    }
                } else {
                    wk->dest[q] = (uint32_t)sidx(wk, S->prm.layout, sl, INV[i]);
                    wk->op[q] = k == 1 ? 2 : 3;
                    if (k >= 2) wk->iol[q] = d->iol[18 * (size_t)g + i - 1];
                }
            }
        }
        free(slot_of);
    }
    for (int q = 0; q < W * W; ++q) free(cross[q].v);
    free(cross);
    return 0;
}

/* ---- engine (engine.hpp:121-650) ------------------------------------------------ */
static void record_state(struct splbcu_sim* S, int w, uint64_t step, const double* f);
static void record_obs(struct splbcu_sim* S, int w, uint64_t row, const double* f);

int splbcu_sim_create(const splbcu_domain* d, const splbcu_bc* bcs, uint32_t nbc, const splbcu_params* prm,
                      splbcu_sim** out) {
    lattice_init();
    int rc = splbcu_domain_validate(d);
    if (rc) return rc;
    if (prm->workers < 1) return set_err(SPLBCU_ERR_CONFIG, "engine: workers must be >= 1");
    if (nbc != d->nio)
        return set_err(SPLBCU_ERR_CONFIG, "engine: boundary conditions configured for %u iolets but the geometry declares %u",
                       nbc, d->nio);
    for (uint32_t k = 0; k < nbc; ++k) {
        table_t tb = {(double*)bcs[k].times, (double*)bcs[k].values, bcs[k].n_nodes, bcs[k].period};
        if ((rc = table_validate(&tb))) return rc;
        if (bcs[k].kind == 0)
            for (uint32_t j = 0; j < tb.n; ++j)
                if (!(tb.v[j] / CS2 > 0.0))
                    return set_err(SPLBCU_ERR_CONFIG, "pressure BC: ghost density must stay positive (table value %f)", tb.v[j]);
    }
    if (!(prm->tau > 0.5)) return set_err(SPLBCU_ERR_CONFIG, "engine: tau must exceed 0.5");
    struct splbcu_sim* S = calloc(1, sizeof *S);
    S->dom = (struct splbcu_domain*)d;
    S->prm = *prm;
    S->omega = 1.0 / prm->tau;
    if ((rc = do_partition(d, prm->workers, &S->part))) {
        free(S);
        return rc;
    }
    S->nbc = nbc;
    S->tables = calloc(nbc + 1, sizeof(table_t));
    S->bc_kind = calloc(nbc + 1, sizeof(int));
    for (uint32_t k = 0; k < nbc; ++k) {
        table_t* tb = &S->tables[k];
        tb->n = bcs[k].n_nodes;
        tb->period = bcs[k].period;
        tb->t = malloc(8 * tb->n);
        tb->v = malloc(8 * tb->n);
        memcpy(tb->t, bcs[k].times, 8 * tb->n);
        memcpy(tb->v, bcs[k].values, 8 * tb->n);
        S->bc_kind[k] = bcs[k].kind;
    }
    const int W = prm->workers;
    S->wk = calloc((size_t)W, sizeof(worker_t));
    if ((rc = build_maps(S))) return rc;
    double eq[Q];
    const double zero[3] = {0, 0, 0};
    splbcu_equilibrium(prm->rho0, zero, eq);
    for (int w = 0; w < W; ++w) {
        worker_t* wk = &S->wk[w];
        const size_t tot = (size_t)Q * wk->n + wk->shared;
        wk->fa = calloc(tot + 1, 8);
        wk->fb = calloc(tot + 1, 8);
        wk->a_old = 1;
        for (uint32_t s = 0; s < wk->n; ++s)
            for (int i = 0; i < Q; ++i) f_old(wk)[sidx(wk, prm->layout, s, i)] = eq[i];
    }
    S->mail = calloc((size_t)W * W, sizeof(double*));
    S->mail_n = calloc((size_t)W * W, 4);
    S->staged = calloc(nbc + 1, 8);
    S->staged_vel = calloc(nbc + 1, sizeof(int));
    /* init_observation (engine.hpp:262-288) */
    S->obs = calloc(d->nio + 1, sizeof(uint32_t*));
    S->nobs = calloc(d->nio + 1, 4);
    for (uint32_t k = 0; k < d->nio; ++k) {
        S->obs[k] = malloc(4 * (d->n ? d->n : 1));
        for (uint64_t g = 0; g < d->n; ++g) {
            int member = 0;
            for (int i = 0; i < 18; ++i)
                if (d->kind[18 * g + i] >= 2 && d->iol[18 * g + i] == k) member = 1;
            if (member) S->obs[k][S->nobs[k]++] = (uint32_t)g;
        }
    }
    S->smax = calloc(d->nio + 1, sizeof(double*));
    S->sp = calloc(d->nio + 1, sizeof(double*));
    S->sq = calloc(d->nio + 1, sizeof(double*));
    *out = S;
    return 0;
}

static void push_range(struct splbcu_sim* S, int w, uint32_t b, uint32_t e) {
    worker_t* wk = &S->wk[w];
    const int lay = S->prm.layout;
    const double* fo = f_old(wk);
    double* fn = f_new(wk);
    double f[Q];
    for (uint32_t s = b; s < e; ++s) {
        for (int i = 0; i < Q; ++i) f[i] = fo[sidx(wk, lay, s, i)];
        const macro_t m = macro_of(f);
        const double usq = usq_term(&m);
        fn[sidx(wk, lay, s, 0)] = relax(f[0], feq(0, &m, usq), S->omega);
        for (int i = 1; i < Q; ++i) {
            const size_t q = 18 * (size_t)s + i - 1;
            double fp = relax(f[i], feq(i, &m, usq), S->omega);
            if (wk->op[q] == 3) {
                /* iolet_link_value (engine.hpp:385-402) */
                const uint16_t io = wk->iol[q];
                const splbcu_iolet* geo = &S->dom->iolets[io];
                const uint32_t g = S->part->parts[w].sites[s];
                if (S->staged_vel[io]) {
                    const double sw = S->staged[io] * weight_of(geo, &S->dom->coords[3 * (size_t)g]);
                    const double ub[3] = {geo->normal[0] * sw, geo->normal[1] * sw, geo->normal[2] * sw};
                    fp = fp - ladd_term(i, m.rho, ub);
                } else {
                    const double un = m.ux * geo->normal[0] + m.uy * geo->normal[1] + m.uz * geo->normal[2];
                    macro_t gh = {S->staged[io], geo->normal[0] * un, geo->normal[1] * un, geo->normal[2] * un};
                    fp = feq(INV[i], &gh, usq_term(&gh));
                }
            }
            fn[wk->dest[q]] = fp;
        }
    }
}

static void advance_group(struct splbcu_sim* S, int w, int edge) {
    const part_t* pt = &S->part->parts[w];
    const uint64_t* r = edge ? pt->er : pt->mr;
    push_range(S, w, (uint32_t)r[0], (uint32_t)r[3]);   /* Inner+Wall merged */
    push_range(S, w, (uint32_t)r[4], (uint32_t)r[11]);  /* iolet types */
}

static void phase_send(struct splbcu_sim* S, int w) {
    worker_t* wk = &S->wk[w];
    const int W = S->part->W;
    const double* fn = f_new(wk) + (size_t)Q * wk->n;
    for (uint32_t k = 0; k < wk->n_seg; ++k) {
        const int nb = wk->seg_nb[k];
        double** box = &S->mail[(size_t)w * W + nb];
        *box = realloc(*box, 8 * (wk->seg_count[k] + 1));
        memcpy(*box, fn + wk->seg_base[k], 8 * wk->seg_count[k]);
        S->mail_n[(size_t)w * W + nb] = wk->seg_count[k];
    }
}

static void phase_receive(struct splbcu_sim* S, int w) {
    worker_t* wk = &S->wk[w];
    const int W = S->part->W;
    double* fo = f_old(wk) + (size_t)Q * wk->n;
    for (uint32_t k = 0; k < wk->n_seg; ++k)
        memcpy(fo + wk->seg_base[k], S->mail[(size_t)wk->seg_nb[k] * W + w], 8 * wk->seg_count[k]);
    /* phase_post_receive (engine.hpp:534-542) */
    double* fn = f_new(wk);
    for (uint32_t slot = 0; slot < wk->shared; ++slot) fn[wk->recv_dest[slot]] = fo[slot];
}

static void fields_of_worker(struct splbcu_sim* S, int w, const double* f, double* out) {
    worker_t* wk = &S->wk[w];
    double fl[Q];
    for (uint32_t s = 0; s < wk->n; ++s) {
        for (int i = 0; i < Q; ++i) fl[i] = f[sidx(wk, S->prm.layout, s, i)];
        const macro_t m = macro_of(fl);
        double* o = out + 4 * (size_t)S->part->parts[w].sites[s];
        o[0] = m.rho, o[1] = m.ux, o[2] = m.uy, o[3] = m.uz;
    }
}

/* per-run observation buffer: [iolet][row][pos][3], indexed by global order */
static double** g_obsbuf;

static void record_obs(struct splbcu_sim* S, int w, uint64_t row, const double* f) {
    if (!S->prm.observe_iolets) return;
    worker_t* wk = &S->wk[w];
    double fl[Q];
    for (uint32_t k = 0; k < S->dom->nio; ++k) {
        const splbcu_iolet* geo = &S->dom->iolets[k];
        for (uint32_t p = 0; p < S->nobs[k]; ++p) {
            const uint32_t g = S->obs[k][p];
            if (S->part->owner[g] != w) continue;
            const uint32_t s = S->part->local[g];
            for (int i = 0; i < Q; ++i) fl[i] = f[sidx(wk, S->prm.layout, s, i)];
            const macro_t m = macro_of(fl);
            double* o = &g_obsbuf[k][3 * ((size_t)row * S->nobs[k] + p)];
            o[0] = sqrt(m.ux * m.ux + m.uy * m.uy + m.uz * m.uz);
            o[1] = CS2 * m.rho;
            o[2] = m.ux * geo->normal[0] + m.uy * geo->normal[1] + m.uz * geo->normal[2];
        }
    }
}

static void record_state(struct splbcu_sim* S, int w, uint64_t step, const double* f) {
    if (S->prm.capture_period > 0 && step % S->prm.capture_period == 0)
        for (uint64_t c = 0; c < S->ncap; ++c)
            if (S->cap_step[c] == step) {
                fields_of_worker(S, w, f, S->cap_f[c]);
                break;
            }
    record_obs(S, w, step, f);
}

int splbcu_sim_run(splbcu_sim* S, uint64_t n) {
    const int W = S->part->W;
    const uint32_t nio = S->dom->nio;
    /* prepare_records (engine.hpp:290-315) */
    if (S->prm.capture_period > 0)
        for (uint64_t st = S->steps; st <= S->steps + n; ++st) {
            if (st % S->prm.capture_period) continue;
            if (S->ncap && S->cap_step[S->ncap - 1] == st) continue;
            S->cap_step = realloc(S->cap_step, 8 * (S->ncap + 1));
            S->cap_f = realloc(S->cap_f, sizeof(double*) * (S->ncap + 1));
            S->cap_step[S->ncap] = st;
            S->cap_f[S->ncap] = calloc(4 * S->dom->n, 8);
            S->ncap++;
        }
    const uint64_t rows = S->steps + n + 1;
    if (S->prm.observe_iolets) {
        g_obsbuf = calloc(nio + 1, sizeof(double*));
        for (uint32_t k = 0; k < nio; ++k) g_obsbuf[k] = calloc(3 * rows * S->nobs[k] + 1, 8);
    }
    if (S->steps == 0)
        for (int w = 0; w < W; ++w) record_state(S, w, 0, f_old(&S->wk[w]));
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    for (uint64_t k = 0; k < n; ++k) {
        const uint64_t step = S->steps + k;
        const double tt = (double)(step + 1) * S->prm.dt_s;
        for (uint32_t io = 0; io < S->nbc; ++io) {
            S->staged_vel[io] = S->bc_kind[io] == 1;
            S->staged[io] = S->staged_vel[io] ? table_at(&S->tables[io], tt) : table_at(&S->tables[io], tt) / CS2;
        }
        for (int w = 0; w < W; ++w) {
            advance_group(S, w, 1);
            if (S->prm.sequence == 0) phase_send(S, w);
        }
        for (int w = 0; w < W; ++w) {
            advance_group(S, w, 0);
            if (S->prm.sequence != 0) phase_send(S, w);
        }
        for (int w = 0; w < W; ++w) phase_receive(S, w);
        const uint64_t done = step + 1;
        for (int w = 0; w < W; ++w) {
            worker_t* wk = &S->wk[w];
            if (S->prm.capture_period > 0 && done % S->prm.capture_period == 0) record_state(S, w, done, f_new(wk));
            else record_obs(S, w, done, f_new(wk));
            wk->a_old = !wk->a_old;
        }
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    S->loop_s += (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    S->steps += n;
    /* assemble_series (engine.hpp:602-629) */
    if (S->prm.observe_iolets) {
        const uint64_t first = S->rows;
        for (uint32_t k = 0; k < nio; ++k) {
            S->smax[k] = realloc(S->smax[k], 8 * rows);
            S->sp[k] = realloc(S->sp[k], 8 * rows);
            S->sq[k] = realloc(S->sq[k], 8 * rows);
            for (uint64_t row = first; row < rows; ++row) {
                double vmax = 0.0, psum = 0.0, qsum = 0.0;
                for (uint32_t p = 0; p < S->nobs[k]; ++p) {
                    const double* v = &g_obsbuf[k][3 * (row * S->nobs[k] + p)];
                    vmax = vmax < v[0] ? v[0] : vmax;
                    psum += v[1];
                    qsum += v[2];
                }
                S->smax[k][row] = vmax;
                S->sp[k][row] = psum / (double)S->nobs[k];
                S->sq[k][row] = qsum;
            }
        }
        S->rows = rows;
        for (uint32_t k = 0; k < nio; ++k) free(g_obsbuf[k]);
        free(g_obsbuf);
        g_obsbuf = NULL;
    }
    return 0;
}

int splbcu_nccl_unique_id(uint8_t o[128]) {
    (void)o;
    return set_err(SPLBCU_ERR_CONFIG, "oracle: no NCCL path");
}
int splbcu_sim_create_dist(const splbcu_domain* a, const splbcu_bc* b, uint32_t c, const splbcu_params* d, int32_t e,
                           int32_t f, const uint8_t g[128], splbcu_sim** h) {
    (void)a, (void)b, (void)c, (void)d, (void)e, (void)f, (void)g, (void)h;
    return set_err(SPLBCU_ERR_CONFIG, "oracle: no NCCL path");
}
uint64_t splbcu_sim_steps_run(const splbcu_sim* S) { return S->steps; }
double splbcu_sim_step_loop_seconds(const splbcu_sim* S) { return S->loop_s; }
double splbcu_sim_device_loop_seconds(const splbcu_sim* S) { return S->loop_s; }
int splbcu_sim_snapshot(splbcu_sim* S, double* out) {
    for (int w = 0; w < S->part->W; ++w) fields_of_worker(S, w, f_old(&S->wk[w]), out);
    return 0;
}
int32_t splbcu_sim_n_workers(const splbcu_sim* S) { return S->part->W; }
int32_t splbcu_sim_worker_is_local(const splbcu_sim* S, int32_t w) { return w >= 0 && w < S->part->W; }
int splbcu_sim_store_shape(const splbcu_sim* S, int32_t w, uint32_t* n, uint32_t* sh) {
    if (n) *n = S->wk[w].n;
    if (sh) *sh = S->wk[w].shared;
    return 0;
}
int splbcu_sim_get_f(splbcu_sim* S, int32_t w, int32_t which, double* host) {
    worker_t* wk = &S->wk[w];
    memcpy(host, which == 0 ? f_old(wk) : f_new(wk), 8 * ((size_t)Q * wk->n + wk->shared));
    return 0;
}
int splbcu_sim_set_f(splbcu_sim* S, int32_t w, int32_t which, const double* host) {
    worker_t* wk = &S->wk[w];
    memcpy(which == 0 ? f_old(wk) : f_new(wk), host, 8 * ((size_t)Q * wk->n + wk->shared));
    return 0;
}
int splbcu_sim_map_shape(const splbcu_sim* S, int32_t w, uint32_t* n, uint32_t* sh, uint32_t* ns) {
    if (n) *n = S->wk[w].n;
    if (sh) *sh = S->wk[w].shared;
    if (ns) *ns = S->wk[w].n_seg;
    return 0;
}
int splbcu_sim_export_map(splbcu_sim* S, int32_t w, uint32_t* dest, uint8_t* op, uint16_t* iol, uint32_t* rd,
                          uint32_t* ss, uint8_t* sd, int32_t* sn, uint32_t* sb, uint32_t* sc) {
    const worker_t* wk = &S->wk[w];
    if (dest) memcpy(dest, wk->dest, 4 * 18 * (size_t)wk->n);
    if (op) memcpy(op, wk->op, 18 * (size_t)wk->n);
    if (iol) memcpy(iol, wk->iol, 36 * (size_t)wk->n);
    if (rd) memcpy(rd, wk->recv_dest, 4 * (size_t)wk->shared);
    if (ss) memcpy(ss, wk->send_site, 4 * (size_t)wk->shared);
    if (sd) memcpy(sd, wk->send_dir, wk->shared);
    if (sn) memcpy(sn, wk->seg_nb, 4 * wk->n_seg);
    if (sb) memcpy(sb, wk->seg_base, 4 * wk->n_seg);
    if (sc) memcpy(sc, wk->seg_count, 4 * wk->n_seg);
    return 0;
}
/* StreamingMap::sources (layout.hpp:104-119, 237-282): the pull-side source
 * of slot (s, inverse(i)) follows from link i of s. */
int splbcu_sim_export_sources(splbcu_sim* S, int32_t w, uint32_t* src, uint8_t* op, uint16_t* iol) {
    const worker_t* wk = &S->wk[w];
    const int lay = S->prm.layout;
    for (uint32_t s = 0; s < wk->n; ++s)
        for (int i = 1; i < Q; ++i) {
            const size_t q = 18 * (size_t)s + (size_t)(i - 1);
            const size_t g = 18 * (size_t)s + (size_t)(INV[i] - 1);
            uint32_t site = s;
            uint8_t o;
            uint16_t io = 0;
            switch (wk->op[q]) {
                case 0: /* ToLocal: dest = idx(local(tg), i) */
                    site = lay == 0 ? wk->dest[q] / Q : wk->dest[q] - (uint32_t)i * wk->n;
                    o = 0;
                    break;
                case 1: site = 0; o = 1; break; /* FromRemote */
                case 2: o = 2; break;            /* SelfBounce */
                default: o = 3; io = wk->iol[q]; break;
            }
            if (src) src[g] = site;
            if (op) op[g] = o;
            if (iol) iol[g] = io;
        }
    return 0;
}
const splbcu_partition* splbcu_sim_partition(const splbcu_sim* S) {
    S->part->borrowed = 1;
    return S->part;
}
uint64_t splbcu_sim_n_captures(const splbcu_sim* S) { return S->ncap; }
int splbcu_sim_capture(const splbcu_sim* S, uint64_t k, uint64_t* step, double* f) {
    if (k >= S->ncap) return set_err(SPLBCU_ERR_CONFIG, "capture index out of range");
    if (step) *step = S->cap_step[k];
    if (f) memcpy(f, S->cap_f[k], 8 * 4 * S->dom->n);
    return 0;
}
uint64_t splbcu_sim_series_rows(const splbcu_sim* S) { return S->rows; }
int splbcu_sim_series(const splbcu_sim* S, uint32_t k, double* a, double* b, double* c) {
    if (k >= S->dom->nio) return set_err(SPLBCU_ERR_CONFIG, "series: iolet out of range");
    if (a) memcpy(a, S->smax[k], 8 * S->rows);
    if (b) memcpy(b, S->sp[k], 8 * S->rows);
    if (c) memcpy(c, S->sq[k], 8 * S->rows);
    return 0;
}
/* write_snapshots (snapshot.hpp:15-29) */
int splbcu_sim_write_snapshots(const splbcu_sim* S, const char* path) {
    FILE* f = fopen(path, "wb");
    if (!f) return set_err(SPLBCU_ERR_RUNTIME, "snapshot write: cannot open %s", path);
    int ok = 1;
    for (uint64_t c = 0; c < S->ncap; ++c) {
        ok &= fwrite(&S->cap_step[c], 8, 1, f) == 1;
        ok &= fwrite(S->cap_f[c], 8, 4 * S->dom->n, f) == 4 * S->dom->n;
    }
    ok &= fclose(f) == 0;
    return ok ? 0 : set_err(SPLBCU_ERR_RUNTIME, "snapshot write: stream failure");
}
/* series_csv (snapshot.hpp:59-82) */
int splbcu_sim_series_csv(const splbcu_sim* S, double dt_s, char* buf, size_t cap, size_t* len) {
    size_t n = 0, sz = 1024;
    char* out = malloc(sz);
    char b[256];
#define APPEND(str)                                          \
    do {                                                     \
        size_t l_ = strlen(str);                             \
        while (n + l_ + 1 > sz) out = realloc(out, sz *= 2); \
        memcpy(out + n, str, l_);                            \
        n += l_;                                             \
    } while (0)
    APPEND("step,time_s");
    const uint32_t nio = S->rows ? S->dom->nio : 0;
    for (uint32_t k = 0; k < nio; ++k) {
        snprintf(b, sizeof b, ",iolet%u_max_speed,iolet%u_pressure,iolet%u_flow", k, k, k);
        APPEND(b);
    }
    APPEND("\n");
    for (uint64_t row = 0; row < S->rows; ++row) {
        snprintf(b, sizeof b, "%llu,%.17g", (unsigned long long)row, (double)row * dt_s);
        APPEND(b);
        for (uint32_t k = 0; k < nio; ++k) {
            snprintf(b, sizeof b, ",%.17g,%.17g,%.17g", S->smax[k][row], S->sp[k][row], S->sq[k][row]);
            APPEND(b);
        }
        APPEND("\n");
    }
#undef APPEND
    if (len) *len = n;
    if (buf && cap) {
        const size_t m = n < cap - 1 ? n : cap - 1;
        memcpy(buf, out, m);
        buf[m] = '\0';
    }
    free(out);
    return 0;
}
int splbcu_sim_set_kernel_timing(splbcu_sim* S, int32_t on) {
    (void)S, (void)on;
    return 0;
}
int splbcu_sim_kernel_stats(const splbcu_sim* S, double* a, uint64_t* b, uint64_t* c) {
    (void)S;
    if (a) *a = 0;
    if (b) *b = 0;
    if (c) *c = 0;
    return 0;
}
/* ---- geometry sources: the oracle builds whole domains only ---------------- */
struct splbcu_source {
    int kind; /* 0 pipe, 1 bifurcation */
    int32_t a, b, c, d;
    double vs;
};
static int new_source(int kind, int32_t a, int32_t b, int32_t c, int32_t d, double vs, splbcu_source** out) {
    splbcu_source* s = (splbcu_source*)calloc(1, sizeof *s);
    if (!s) return set_err(SPLBCU_ERR_RUNTIME, "out of memory");
    s->kind = kind, s->a = a, s->b = b, s->c = c, s->d = d, s->vs = vs;
    *out = s;
    return SPLBCU_OK;
}
int splbcu_source_pipe(int32_t r, int32_t l, double vs, splbcu_source** o) {
    if (r < 2 || l < 4) return set_err(SPLBCU_ERR_GEOMETRY, "build_pipe: need radius >= 2 and length >= 4");
    return new_source(0, r, l, 0, 0, vs, o);
}
int splbcu_source_bifurcation(int32_t tr, int32_t br, int32_t tl, int32_t bl, double vs, splbcu_source** o) {
    if (tr < 2 || br < 2 || tl < 4 || bl < 4)
        return set_err(SPLBCU_ERR_GEOMETRY, "build_bifurcation: need radii >= 2 and lengths >= 4");
    return new_source(1, tr, br, tl, bl, vs, o);
}
int splbcu_source_tree(int32_t a, int32_t b, int32_t c, double d_, double e, double f, splbcu_source** o) {
    (void)a, (void)b, (void)c, (void)d_, (void)e, (void)f, (void)o;
    return set_err(SPLBCU_ERR_CONFIG, "oracle: the tree generator is product-only; pass its arrays");
}
int splbcu_source_channel(int32_t a, int32_t b, int32_t c, double d_, splbcu_source** o) {
    (void)a, (void)b, (void)c, (void)d_, (void)o;
    return set_err(SPLBCU_ERR_CONFIG, "oracle: the channel generator is product-only; pass its arrays");
}
int splbcu_source_build(const splbcu_source* s, splbcu_domain** out) {
    if (!s) return set_err(SPLBCU_ERR_CONFIG, "null source");
    return s->kind == 0 ? splbcu_domain_build_pipe(s->a, s->b, s->vs, out)
                        : splbcu_domain_build_bifurcation(s->a, s->b, s->c, s->d, s->vs, out);
}
int splbcu_source_window(const splbcu_source* s, int32_t n, int32_t w, int32_t* slab, splbcu_domain** win,
                         splbcu_partition** part) {
    (void)s, (void)n, (void)w, (void)slab, (void)win, (void)part;
    return set_err(SPLBCU_ERR_CONFIG, "oracle: slab-local windows are product-only");
}
int splbcu_window_info(const splbcu_domain* d, uint64_t* a, int32_t* b, int32_t* c, uint64_t* e) {
    (void)d, (void)a, (void)b, (void)c, (void)e;
    return set_err(SPLBCU_ERR_CONFIG, "domain is not a source window");
}
void splbcu_source_free(splbcu_source* s) { free(s); }
int splbcu_sim_create_dist_source(const splbcu_source* a, const splbcu_bc* b, uint32_t c, const splbcu_params* d,
                                  int32_t e, int32_t f, const uint8_t g[128], splbcu_sim** h) {
    (void)a, (void)b, (void)c, (void)d, (void)e, (void)f, (void)g, (void)h;
    return set_err(SPLBCU_ERR_CONFIG, "oracle: no NCCL path");
}
uint64_t splbcu_sim_series_d2h_bytes(const splbcu_sim* S) {
    (void)S;
    return 0;
}
int32_t splbcu_sim_slab_local(const splbcu_sim* S) {
    (void)S;
    return 0;
}
uint64_t splbcu_sim_n_sites(const splbcu_sim* S) { return S->dom->n; }

uint64_t splbcu_sim_launch_count(const splbcu_sim* S) {
    (void)S;
    return 0;
}
int32_t splbcu_sim_bulk_kernel(const splbcu_sim* S) {
    (void)S;
    return -1;
}
void splbcu_sim_destroy(splbcu_sim* S) {
    if (!S) return;
    for (int w = 0; w < S->part->W; ++w) {
        worker_t* wk = &S->wk[w];
        free(wk->dest), free(wk->op), free(wk->iol), free(wk->recv_dest), free(wk->send_site), free(wk->send_dir);
        free(wk->seg_nb), free(wk->seg_base), free(wk->seg_count), free(wk->fa), free(wk->fb);
    }
    for (int q = 0; q < S->part->W * S->part->W; ++q) free(S->mail[q]);
    for (uint32_t k = 0; k < S->nbc; ++k) free(S->tables[k].t), free(S->tables[k].v);
    for (uint32_t k = 0; k < S->dom->nio; ++k) free(S->obs[k]), free(S->smax[k]), free(S->sp[k]), free(S->sq[k]);
    for (uint64_t c = 0; c < S->ncap; ++c) free(S->cap_f[c]);
    free(S->cap_f), free(S->cap_step), free(S->obs), free(S->nobs), free(S->smax), free(S->sp), free(S->sq);
    free(S->mail), free(S->mail_n), free(S->staged), free(S->staged_vel), free(S->tables), free(S->bc_kind), free(S->wk);
    S->part->borrowed = 0;
    part_free(S->part);
    free(S);
}
