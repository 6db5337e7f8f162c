/* oracle/nau_oracle.c — TEST INFRASTRUCTURE (see nau_oracle.h header note).
 *
 * CPU restatement of the reference hot path. Each function cites the
 * reference file:line (relative to /root/reference/proj) it follows.
 * Compiled with -ffp-contract=off; operation order is the reference's
 * (C++ left-associative evaluation, index-order reductions).
 */
#include "nau_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <limits.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>
#include <string.h>

static const double kPi = 3.14159265358979323846;

/* include/nauticle/domain.hpp:26-33, src/domain.cpp:27-47 */
void nor_domain_init(nor_domain* d, int dim, const int* min_cells, const int* max_cells,
                     const double* cell_size, const int* kinds) {
    memset(d, 0, sizeof(*d));
    d->dim = dim;
    for (int a = 0; a < 3; ++a) {
        int mn = 0, mx = 1, kind = NOR_CUTOFF;
        double cs = 1.0;
        if (a < dim) {
            mn = min_cells[a];
            mx = max_cells[a];
            cs = cell_size[a];
            kind = kinds[a];
        }
        d->cells[a] = mx - mn;
        d->cs[a] = cs;
        d->lo[a] = mn * cs;
        d->hi[a] = mx * cs;
        d->ext[a] = d->hi[a] - d->lo[a];
        d->kind[a] = kind;
    }
}

long nor_ncells(const nor_domain* d) {
    long t = 1;
    for (int a = 0; a < d->dim; ++a) t *= d->cells[a];
    return t;
}

/* src/particle_system.cpp:20-31 */
int nor_cell_index(const nor_domain* d, int axis, double x) {
    const double lo = d->lo[axis];
    const double size = d->cs[axis];
    const int n = d->cells[axis];
    int c = (int)floor((x - lo) / size);
    if (d->kind[axis] == NOR_PERIODIC) {
        c %= n;
        if (c < 0) c += n;
        return c;
    }
    return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

/* src/particle_system.cpp:33-54: active particles in ascending index, axis 0 fastest. */
long nor_build_cells(const nor_domain* d, int n, const double* pos, const uint8_t* active,
                     int* cell_of, int* cell_start, int* cell_count, int* sorted) {
    const long nc = nor_ncells(d);
    const int dim = d->dim;
    for (long c = 0; c < nc; ++c) cell_count[c] = 0;
    for (int i = 0; i < n; ++i) {
        cell_of[i] = -1;
        if (!active[i]) continue;
        int flat = 0;
        for (int a = dim - 1; a >= 0; --a) {
            double x = pos[(long)a * n + i];
            if (d->kind[a] == NOR_CUTOFF && (x < d->lo[a] || x > d->hi[a])) return 1 + (long)i;
            flat = flat * d->cells[a] + nor_cell_index(d, a, x);
        }
        cell_of[i] = flat;
        cell_count[flat]++;
    }
    int acc = 0;
    for (long c = 0; c < nc; ++c) {
        cell_start[c] = acc;
        acc += cell_count[c];
    }
    int* cursor = (int*)malloc(sizeof(int) * (size_t)(nc > 0 ? nc : 1));
    for (long c = 0; c < nc; ++c) cursor[c] = cell_start[c];
    for (int i = 0; i < n; ++i)
        if (cell_of[i] >= 0) sorted[cursor[cell_of[i]]++] = i;
    free(cursor);
    return 0;
}

/* src/particle_system.cpp:56-90 */
long nor_boundary_shift(const nor_domain* d, int n, double* pos, uint8_t* active) {
    long warnings = 0;
    for (int i = 0; i < n; ++i) {
        if (!active[i]) continue;
        for (int a = 0; a < d->dim; ++a) {
            double* x = &pos[(long)a * n + i];
            const double lo = d->lo[a], hi = d->hi[a];
            switch (d->kind[a]) {
                case NOR_PERIODIC:
                    if (*x < lo || *x >= hi) {
                        double w = fmod(*x - lo, d->ext[a]);
                        if (w < 0.0) w += d->ext[a];
                        *x = lo + w;
                        if (*x >= hi) *x = lo;
                    }
                    break;
                case NOR_SYMMETRIC:
                    if (*x < lo || *x > hi) ++warnings;
                    break;
                default:
                    if (*x < lo || *x > hi) active[i] = 0;
                    break;
            }
            if (!active[i]) break;
        }
    }
    return warnings;
}

/* ---- neighbour enumeration: include/nauticle/particle_system.hpp:59-138 ---- */

typedef struct {
    int j;
    double rel[3];
    double guide[3];
} cand_t;

typedef struct {
    cand_t* c;
    int n, cap;
} cand_buf;

static void push(cand_buf* b, int j, const double* rel, const double* guide) {
    if (b->n == b->cap) {
        b->cap = b->cap ? 2 * b->cap : 1024;
        b->c = (cand_t*)realloc(b->c, sizeof(cand_t) * (size_t)b->cap);
    }
    cand_t* t = &b->c[b->n++];
    t->j = j;
    for (int a = 0; a < 3; ++a) {
        t->rel[a] = rel[a];
        t->guide[a] = guide[a];
    }
}


/* ---- host threads: a dynamic parallel-for over particles (the role of
 * ThreadPool::parallel_blocks, thread_pool.hpp:20-46; particles are independent) ---- */
typedef void (*nor_body_fn)(void* arg, int i, cand_buf* b);
typedef struct {
    nor_body_fn fn;
    void* arg;
    int n, chunk;
    atomic_int next;
} nor_pfor;

static void* pfor_worker(void* p) {
    nor_pfor* t = (nor_pfor*)p;
    cand_buf b = {0, 0, 0};
    for (;;) {
        int s = atomic_fetch_add(&t->next, t->chunk);
        if (s >= t->n) break;
        int e = s + t->chunk < t->n ? s + t->chunk : t->n;
        for (int i = s; i < e; ++i) t->fn(t->arg, i, &b);
    }
    free(b.c);
    return NULL;
}

static int nor_threads(void) {
    const char* e = getenv("NOR_THREADS");
    long t = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
    return t < 1 ? 1 : (t > 256 ? 256 : (int)t);
}

static void parallel_for(int n, int chunk, nor_body_fn fn, void* arg) {
    nor_pfor t;
    t.fn = fn;
    t.arg = arg;
    t.n = n;
    t.chunk = chunk;
    atomic_init(&t.next, 0);
    int nt = nor_threads();
    if ((long)nt * chunk > n) nt = (n + chunk - 1) / chunk;
    if (nt <= 1) {
        pfor_worker(&t);
        return;
    }
    pthread_t th[256];
    for (int k = 1; k < nt; ++k) pthread_create(&th[k], NULL, pfor_worker, &t);
    pfor_worker(&t);
    for (int k = 1; k < nt; ++k) pthread_join(th[k], NULL);
}

static void candidates(const nor_ps* ps, int i, cand_buf* out) {
    out->n = 0;
    if (!ps->active[i]) return;
    const nor_domain* dom = &ps->dom;
    const int d = dom->dim;
    const int n = ps->n;
    int opt_cell[3][5];
    double opt_shift[3][5];
    int opt_reflect[3][5];
    int count[3] = {1, 1, 1};
    int ci_flat = ps->cell_of[i];
    int ci[3];
    ci[0] = ci_flat % dom->cells[0];
    ci[1] = (ci_flat / dom->cells[0]) % dom->cells[1];
    ci[2] = ci_flat / (dom->cells[0] * dom->cells[1]);
    for (int a = 0; a < d; ++a) {
        const int nc = dom->cells[a];
        const double ext = dom->ext[a];
        int k = 0;
        for (int o = -1; o <= 1; ++o) {
            int c = ci[a] + o;
            double shift = 0.0;
            if (c < 0) {
                if (dom->kind[a] != NOR_PERIODIC) continue;
                c += nc;
                shift = -ext;
            } else if (c >= nc) {
                if (dom->kind[a] != NOR_PERIODIC) continue;
                c -= nc;
                shift = ext;
            }
            opt_cell[a][k] = c;
            opt_shift[a][k] = shift;
            opt_reflect[a][k] = 0;
            ++k;
        }
        if (dom->kind[a] == NOR_SYMMETRIC) {
            if (ci[a] == 0) {
                opt_cell[a][k] = 0;
                opt_shift[a][k] = 0.0;
                opt_reflect[a][k] = -1;
                ++k;
            }
            if (ci[a] == nc - 1) {
                opt_cell[a][k] = nc - 1;
                opt_shift[a][k] = 0.0;
                opt_reflect[a][k] = 1;
                ++k;
            }
        }
        count[a] = k;
    }
    double xi[3] = {0, 0, 0};
    for (int a = 0; a < d; ++a) xi[a] = ps->pos[(long)a * n + i];
    int sel[3] = {0, 0, 0};
    for (;;) {
        int flat = 0;
        for (int a = d - 1; a >= 0; --a) flat = flat * dom->cells[a] + opt_cell[a][sel[a]];
        double guide[3] = {1, 1, 1};
        for (int a = 0; a < d; ++a) guide[a] = opt_reflect[a][sel[a]] != 0 ? -1.0 : 1.0;
        const int s = ps->cell_start[flat], e = s + ps->cell_count[flat];
        for (int q = s; q < e; ++q) {
            const int j = ps->sorted[q];
            double rel[3] = {0, 0, 0};
            int skip = 0;
            for (int a = 0; a < d; ++a) {
                const double xj = ps->pos[(long)a * n + j];
                double img;
                if (opt_reflect[a][sel[a]] == 0)
                    img = xj + opt_shift[a][sel[a]];
                else if (opt_reflect[a][sel[a]] < 0)
                    img = 2.0 * dom->lo[a] - xj;
                else
                    img = 2.0 * dom->hi[a] - xj;
                double r = img - xi[a];
                if (fabs(r) > dom->cs[a]) {
                    skip = 1;
                    break;
                }
                rel[a] = r;
            }
            if (skip) continue;
            push(out, j, rel, guide);
        }
        int a = 0;
        for (; a < d; ++a) {
            if (++sel[a] < count[a]) break;
            sel[a] = 0;
        }
        if (a == d) break;
    }
}

/* Eigen norm through the shim: sqrt of the index-order sum of squares. */
static double norm_d(const double* v, int d) {
    double s = v[0] * v[0];
    for (int a = 1; a < d; ++a) s = s + v[a] * v[a];
    return sqrt(s);
}

typedef struct {
    nor_ps* ps;
    double radius;
    int* counts;
} nc_arg;

static void nc_body(void* p, int i, cand_buf* b) {
    nc_arg* a = (nc_arg*)p;
    candidates(a->ps, i, b);
    int c = 0;
    for (int k = 0; k < b->n; ++k)
        if (norm_d(b->c[k].rel, a->ps->dom.dim) <= a->radius) ++c;
    a->counts[i] = c;
}

void nor_neighbor_counts(nor_ps* ps, double radius, int* counts) {
    nc_arg a = {ps, radius, counts};
    parallel_for(ps->n, 256, nc_body, &a);
}

/* ---- smoothing kernels: src/kernel.cpp:37-69 (Wendland); cubic spline is new ---- */

static double kernel_alpha(int family, int kdim, double h) {
    if (family == NOR_K_WENDLAND) {
        switch (kdim) {
            case 1: return 3.0 / (4.0 * h);
            case 2: return 7.0 / (4.0 * kPi * h * h);
            default: return 21.0 / (16.0 * kPi * h * h * h);
        }
    }
    switch (kdim) { /* Monaghan M4 cubic spline, support 2h */
        case 1: return 2.0 / (3.0 * h);
        case 2: return 10.0 / (7.0 * kPi * h * h);
        default: return 1.0 / (kPi * h * h * h);
    }
}

static double kval(int family, double alpha, double h, double dist) {
    double q = dist / h;
    if (q >= 2.0) return 0.0;
    if (family == NOR_K_WENDLAND) {
        double t = 1.0 - 0.5 * q;
        double t2 = t * t;
        return alpha * t2 * t2 * (2.0 * q + 1.0);
    }
    if (q < 1.0) return alpha * (1.0 - 1.5 * q * q + 0.75 * q * q * q);
    double t = 2.0 - q;
    return alpha * (0.25 * t * t * t);
}

static double kdq(int family, double alpha, double q) {
    if (q >= 2.0) return 0.0;
    if (family == NOR_K_WENDLAND) {
        double t = 1.0 - 0.5 * q;
        return -5.0 * alpha * q * t * t * t;
    }
    if (q < 1.0) return alpha * (-3.0 * q + 2.25 * q * q);
    double t = 2.0 - q;
    return alpha * (-0.75 * t * t);
}

/* kernel.cpp:62-69: grad = rel * (-dW/dq / (h d)); zero beyond support. */
static void kgrad(int family, double alpha, double h, const double* rel, int d, double* g) {
    double dist = norm_d(rel, d);
    double q = dist / h;
    if (q >= 2.0) {
        for (int a = 0; a < d; ++a) g[a] = 0.0;
        return;
    }
    double scale = -kdq(family, alpha, q) / (h * dist);
    for (int a = 0; a < d; ++a) g[a] = rel[a] * scale;
}

double nor_kernel_value(int family, int kdim, double h, double d) {
    return kval(family, kernel_alpha(family, kdim, h), h, d);
}
double nor_kernel_dq(int family, int kdim, double h, double q) {
    return kdq(family, kernel_alpha(family, kdim, h), q);
}

/* ---- operand access (interactions.cpp:13-15; tensor.cpp:115-126 mirror) ---- */

static double opv(const nor_operand* o, int n, int c, int j) {
    return o->field ? o->field[(long)c * n + j] : o->value[c];
}

/* mirror(): value(r,c) * srow * scol, column-major component c = col*rows + row. */
static void fetch_mirrored(const nor_operand* o, int n, int j, const double* guide, int gd,
                           double* out) {
    const int rows = o->rows, cols = o->cols;
    const int scalar = rows == 1 && cols == 1;
    for (int c = 0; c < cols; ++c)
        for (int r = 0; r < rows; ++r) {
            double v = opv(o, n, c * rows + r, j);
            if (!scalar) {
                double srow = r < gd ? guide[r] : 1.0;
                double scol = (cols == 1 || c >= gd) ? 1.0 : guide[c];
                v = v * srow * scol;
            }
            out[c * rows + r] = v;
        }
}

static int any_reflected(const double* guide, int d) {
    for (int a = 0; a < d; ++a)
        if (guide[a] < 0) return 1;
    return 0;
}

/* interactions.cpp:32-38 */
static void warn_coincident(const nor_ps* ps, int i, int j, const double* guide, long* warns) {
    if (i == j) return;
    if (any_reflected(guide, ps->dom.dim)) return;
    ++*warns;
}

/* interactions.cpp:288-316 (Hertz) and the restated linear spring-dashpot law. */
static void contact_force(int law, double Ri, double Rj, double Pi, double Pj, double nui,
                          double nuj, double mi, double mj, double friction, double zeta,
                          const double* rel, const double* vi, const double* vj, int d,
                          double* f, int* err) {
    for (int a = 0; a < d; ++a) f[a] = 0.0;
    double dist = norm_d(rel, d);
    double overlap = Ri + Rj - dist;
    if (overlap <= 0.0 || dist <= 0.0) return;
    double normal, n_ji[3], dv[3];
    for (int a = 0; a < d; ++a) n_ji[a] = rel[a] / dist;
    for (int a = 0; a < d; ++a) dv[a] = vj[a] - vi[a];
    double dd = dv[0] * n_ji[0];
    for (int a = 1; a < d; ++a) dd = dd + dv[a] * n_ji[a];
    double overlap_rate = -dd;
    if (law == NOR_DEM_LSD) {
        double kn = Pi;
        double m_eff = mi * mj / (mi + mj);
        double c_n = 2.0 * zeta * sqrt(m_eff * kn);
        normal = kn * overlap + c_n * overlap_rate;
    } else {
        double Ei = Pi, Ej = Pj;
        if (Ei <= 0.0 || Ej <= 0.0 || Ri <= 0.0 || Rj <= 0.0) {
            *err = 1;
            return;
        }
        double r_eff = Ri * Rj / (Ri + Rj);
        double m_eff = mi * mj / (mi + mj);
        double e_eff = Ei * Ej / (Ej * (1.0 - nui * nui) + Ei * (1.0 - nuj * nuj));
        double k_hz = 4.0 / 3.0 * sqrt(r_eff) * e_eff;
        double c_hz = sqrt(m_eff * k_hz) / 8.0 * 1.0;
        normal = k_hz * pow(overlap, 1.5) + c_hz * pow(overlap, 0.25) * overlap_rate;
    }
    for (int a = 0; a < d; ++a) f[a] = -(n_ji[a] * normal);
    if (friction != 0.0) {
        double v_ij[3], v_t[3];
        for (int a = 0; a < d; ++a) v_ij[a] = vi[a] - vj[a];
        double dn = v_ij[0] * n_ji[0];
        for (int a = 1; a < d; ++a) dn = dn + v_ij[a] * n_ji[a];
        for (int a = 0; a < d; ++a) v_t[a] = -v_ij[a] + n_ji[a] * dn;
        double vt_norm = norm_d(v_t, d);
        if (vt_norm > 1e-12) {
            double s = friction * fabs(normal) / vt_norm;
            for (int a = 0; a < d; ++a) f[a] = f[a] + v_t[a] * s;
        }
    }
}

/* One particle i of InteractionOp::eval (interactions.cpp:40-316). Returns 0 and the
 * result in out[c*n + i], or 1 with the offending index in *bad. Coincident-pair and
 * at-goal warnings are added to *warns. `b` is a per-thread candidate buffer. */
static int interact_one(int op, int kfamily, int kdim, const nor_ps* ps, const nor_operand* ops,
                        int nops, double* out, int out_comps, int i, cand_buf* bp, long* warns,
                        long* bad) {
    const int n = ps->n;
    const int d = ps->dom.dim;
    cand_buf b = *bp;
    int rc = 0;
    do {
        double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        if (op == NOR_GRAVITY) { /* interactions.cpp:195-214 */
            double G = opv(&ops[1], n, 0, i);
            double eps = nops > 2 ? opv(&ops[2], n, 0, i) : 0.0;
            for (int j = 0; j < n; ++j) {
                if (j == i || !ps->active[j]) continue;
                double rel[3];
                for (int a = 0; a < d; ++a) rel[a] = ps->pos[(long)a * n + j] - ps->pos[(long)a * n + i];
                double r2 = rel[0] * rel[0];
                for (int a = 1; a < d; ++a) r2 = r2 + rel[a] * rel[a];
                r2 = r2 + eps * eps;
                if (r2 == 0.0) {
                    rc = 1;
                    *bad = i;
                    break;
                }
                double m_j = opv(&ops[0], n, 0, j);
                double s = G * m_j / pow(r2, 1.5);
                for (int a = 0; a < d; ++a) acc[a] = acc[a] + rel[a] * s;
            }
            if (rc) break;
            for (int c = 0; c < out_comps; ++c) out[(long)c * n + i] = acc[c];
            continue;
        }
        candidates(ps, i, &b);
        if (op <= NOR_SPH_A) {
            /* sph_context: interactions.cpp:22-27 */
            double radius = opv(&ops[3], n, 0, i);
            if (!(radius > 0.0)) {
                rc = 1;
                *bad = i;
                break;
            }
            double h = 0.5 * radius;
            double alpha = kernel_alpha(kfamily, kdim, h);
            const nor_operand* A = &ops[0];
            const int ac = A->rows * A->cols;
            double a_i[9];
            for (int c = 0; c < ac; ++c) a_i[c] = opv(A, n, c, i);
            double rho_i = 0.0;
            if (op == NOR_SPH_G11 || op == NOR_SPH_A) {
                rho_i = opv(&ops[2], n, 0, i);
                if (rho_i == 0.0) {
                    rc = 1;
                    *bad = i;
                    break;
                }
            }
            for (int k = 0; k < b.n && rc == 0; ++k) {
                const cand_t* cd = &b.c[k];
                const int j = cd->j;
                double dist = norm_d(cd->rel, d);
                double g[3];
                switch (op) {
                    case NOR_SPH_S: { /* interactions.cpp:40-58 */
                        if (dist > radius) break;
                        double w = kval(kfamily, alpha, h, dist);
                        if (w == 0.0) break;
                        double rho_j = opv(&ops[2], n, 0, j);
                        if (rho_j == 0.0) {
                            rc = 1;
                            *bad = j;
                            break;
                        }
                        double m_j = opv(&ops[1], n, 0, j);
                        double a_j[9];
                        fetch_mirrored(A, n, j, cd->guide, d, a_j);
                        double s = m_j / rho_j * w;
                        for (int c = 0; c < ac; ++c) acc[c] = acc[c] + a_j[c] * s;
                        break;
                    }
                    case NOR_SPH_D00: { /* interactions.cpp:60-79 */
                        if (dist <= 0.0 || dist > radius) break;
                        double rho_j = opv(&ops[2], n, 0, j);
                        if (rho_j == 0.0) {
                            rc = 1;
                            *bad = j;
                            break;
                        }
                        double m_j = opv(&ops[1], n, 0, j);
                        double a_j[9];
                        fetch_mirrored(A, n, j, cd->guide, d, a_j);
                        kgrad(kfamily, alpha, h, cd->rel, d, g);
                        double dt = (a_j[0] - a_i[0]) * g[0];
                        for (int a = 1; a < d; ++a) dt = dt + (a_j[a] - a_i[a]) * g[a];
                        acc[0] = acc[0] + dt * (m_j / rho_j);
                        break;
                    }
                    case NOR_SPH_G11: { /* interactions.cpp:81-102 */
                        if (dist <= 0.0 || dist > radius) break;
                        double rho_j = opv(&ops[2], n, 0, j);
                        if (rho_j == 0.0) {
                            rc = 1;
                            *bad = j;
                            break;
                        }
                        double a_j = opv(A, n, 0, j);
                        double m_j = opv(&ops[1], n, 0, j);
                        kgrad(kfamily, alpha, h, cd->rel, d, g);
                        double s = m_j * (a_i[0] / (rho_i * rho_i) + a_j / (rho_j * rho_j));
                        for (int a = 0; a < d; ++a) acc[a] = acc[a] + g[a] * s;
                        break;
                    }
                    case NOR_SPH_L0: { /* interactions.cpp:104-126 */
                        if (dist > radius) break;
                        if (dist <= 0.0) {
                            warn_coincident(ps, i, j, cd->guide, warns);
                            break;
                        }
                        double rho_j = opv(&ops[2], n, 0, j);
                        if (rho_j == 0.0) {
                            rc = 1;
                            *bad = j;
                            break;
                        }
                        double a_j = opv(A, n, 0, j);
                        double m_j = opv(&ops[1], n, 0, j);
                        kgrad(kfamily, alpha, h, cd->rel, d, g);
                        double rg = cd->rel[0] * g[0];
                        for (int a = 1; a < d; ++a) rg = rg + cd->rel[a] * g[a];
                        acc[0] = acc[0] + 2.0 * (a_j - a_i[0]) * rg / (dist * dist) * m_j / rho_j;
                        break;
                    }
                    case NOR_SPH_A: { /* interactions.cpp:128-150 */
                        if (dist > radius) break;
                        if (dist <= 0.0) {
                            warn_coincident(ps, i, j, cd->guide, warns);
                            break;
                        }
                        double v_j[9];
                        fetch_mirrored(A, n, j, cd->guide, d, v_j);
                        double ap = (v_j[0] - a_i[0]) * cd->rel[0];
                        for (int a = 1; a < d; ++a) ap = ap + (v_j[a] - a_i[a]) * cd->rel[a];
                        if (ap >= 0.0) break;
                        double m_j = opv(&ops[1], n, 0, j);
                        double pi_ij = ap / (rho_i * dist * dist);
                        kgrad(kfamily, alpha, h, cd->rel, d, g);
                        double s = m_j * pi_ij;
                        for (int a = 0; a < d; ++a) acc[a] = acc[a] + g[a] * s;
                        break;
                    }
                }
            }
            if (rc) break;
            if (op == NOR_SPH_G11)
                for (int a = 0; a < d; ++a) acc[a] = rho_i * acc[a];
            for (int c = 0; c < out_comps; ++c) out[(long)c * n + i] = acc[c];
            continue;
        }
        if (op == NOR_SFM) { /* eval_social_force, interactions.cpp:216-257 */
            double v_i[3], e0[3], drv[3] = {0, 0, 0};
            for (int a = 0; a < d; ++a) v_i[a] = opv(&ops[0], n, a, i);
            const double v0 = opv(&ops[1], n, 0, i);
            const double radius_i = opv(&ops[3], n, 0, i);
            const double rep_a = opv(&ops[4], n, 0, i), rep_b = opv(&ops[5], n, 0, i);
            const double body_k = opv(&ops[6], n, 0, i), c_i = opv(&ops[7], n, 0, i);
            const double m_i = opv(&ops[8], n, 0, i), tau = opv(&ops[9], n, 0, i);
            if (!(tau > 0.0) || !(m_i > 0.0)) { /* 228-229 */
                rc = 1;
                *bad = i;
                break;
            }
            for (int a = 0; a < d; ++a) e0[a] = opv(&ops[2], n, a, i) - ps->pos[(long)a * n + i];
            const double e0n = norm_d(e0, d);
            if (e0n > 0.0) {
                const double s = v0 / e0n;
                for (int a = 0; a < d; ++a) drv[a] = (e0[a] * s - v_i[a]) / tau;
            } else {
                ++*warns; /* agent already at its desired position */
            }
            double cs_min = ps->dom.cs[0];
            for (int a = 1; a < d; ++a) cs_min = ps->dom.cs[a] < cs_min ? ps->dom.cs[a] : cs_min;
            for (int k = 0; k < b.n; ++k) {
                const cand_t* cd = &b.c[k];
                const int j = cd->j;
                const double d_ji = norm_d(cd->rel, d);
                if (!(d_ji > 0.0 && d_ji < cs_min)) continue;
                const double r_ij = radius_i + opv(&ops[3], n, 0, j);
                const double c_ij = 0.5 * (c_i + opv(&ops[7], n, 0, j));
                const double body = r_ij - d_ji > 0.0 ? body_k * (r_ij - d_ji) : 0.0;
                const double s = rep_a * exp((r_ij - d_ji) / rep_b) + body - c_ij;
                for (int a = 0; a < d; ++a) acc[a] = acc[a] + (cd->rel[a] / d_ji) * s;
            }
            for (int a = 0; a < d; ++a) out[(long)a * n + i] = drv[a] - acc[a] / m_i;
            continue;
        }
        /* DEM: dem_sum, interactions.cpp:152-193 (Hertz) / restated LSD law */
        {
            const int images_only = op == NOR_DEM_BOUNDARY;
            const int as_force = op == NOR_DEM_BOUNDARY;
            const int law = op == NOR_DEM_LSD ? NOR_DEM_LSD : NOR_DEM_HERTZ;
            double radius = opv(&ops[6], n, 0, i);
            double v_i[3];
            for (int a = 0; a < d; ++a) v_i[a] = opv(&ops[0], n, a, i);
            double Ri = opv(&ops[1], n, 0, i);
            double Pi = opv(&ops[2], n, 0, i);
            double nui = opv(&ops[3], n, 0, i);
            double mi = opv(&ops[4], n, 0, i);
            double fr = opv(&ops[5], n, 0, i);
            double zeta = 0.0;
            if (law == NOR_DEM_LSD) { /* restitution en -> damping ratio */
                double le = log(nui);
                zeta = -le / sqrt(kPi * kPi + le * le);
            }
            for (int k = 0; k < b.n; ++k) {
                const cand_t* cd = &b.c[k];
                const int j = cd->j;
                double dist = norm_d(cd->rel, d);
                if (dist > radius) continue;
                if (images_only && !any_reflected(cd->guide, d)) continue;
                if (dist <= 0.0) {
                    if (law == NOR_DEM_HERTZ) warn_coincident(ps, i, j, cd->guide, warns);
                    continue;
                }
                double Rj = opv(&ops[1], n, 0, j);
                double Pj = opv(&ops[2], n, 0, j);
                double nuj = opv(&ops[3], n, 0, j);
                double mj = opv(&ops[4], n, 0, j);
                if (Rj + Ri - dist <= 0.0) continue;
                double v_j[9], f[3];
                fetch_mirrored(&ops[0], n, j, cd->guide, d, v_j);
                int err = 0;
                contact_force(law, Ri, Rj, Pi, Pj, nui, nuj, mi, mj, fr, zeta, cd->rel, v_i, v_j,
                              d, f, &err);
                if (err) {
                    rc = 1;
                    *bad = i;
                    break;
                }
                for (int a = 0; a < d; ++a) acc[a] = acc[a] + f[a];
            }
            if (rc) break;
            if (!as_force)
                for (int a = 0; a < d; ++a) acc[a] = acc[a] / mi;
            for (int c = 0; c < out_comps; ++c) out[(long)c * n + i] = acc[c];
        }
    } while (0);
    *bp = b;
    return rc;
}

/* The per-equation loop of Case::solve_equation (case.cpp:31-54) over host threads
 * (ThreadPool::parallel_blocks, thread_pool.hpp:20-46, also evaluates particles
 * independently). Serial semantics are kept: the reported error is the one of the
 * lowest failing particle, and warnings count up to and including that particle. */
typedef struct {
    int op, kfamily, kdim, nops, out_comps;
    const nor_ps* ps;
    const nor_operand* ops;
    double* out;
    long* warns;
    pthread_mutex_t mu;
    long first_fail, fail_bad;
} ia_arg;

static void ia_body(void* p, int i, cand_buf* b) {
    ia_arg* a = (ia_arg*)p;
    if (!a->ps->active[i]) return;
    long w = 0, bd = -1;
    int rc = interact_one(a->op, a->kfamily, a->kdim, a->ps, a->ops, a->nops, a->out,
                          a->out_comps, i, b, &w, &bd);
    a->warns[i] = w;
    if (rc) {
        pthread_mutex_lock(&a->mu);
        if (i < a->first_fail) {
            a->first_fail = i;
            a->fail_bad = bd;
        }
        pthread_mutex_unlock(&a->mu);
    }
}

int nor_interact(int op, int kfamily, int kdim, nor_ps* ps, const nor_operand* ops, int nops,
                 double* out, int out_comps, long* bad) {
    const int n = ps->n;
    ia_arg a;
    a.op = op;
    a.kfamily = kfamily;
    a.kdim = kdim;
    a.nops = nops;
    a.out_comps = out_comps;
    a.ps = ps;
    a.ops = ops;
    a.out = out;
    a.warns = (long*)calloc((size_t)(n > 0 ? n : 1), sizeof(long));
    pthread_mutex_init(&a.mu, NULL);
    a.first_fail = LONG_MAX;
    a.fail_bad = -1;
    parallel_for(n, op == NOR_GRAVITY ? 8 : 64, ia_body, &a);
    pthread_mutex_destroy(&a.mu);
    long wsum = 0;
    for (long i = 0; i < n && i <= a.first_fail; ++i) wsum += a.warns[i];
    free(a.warns);
    ps->warnings += wsum;
    *bad = -1;
    if (a.first_fail != LONG_MAX) {
        *bad = a.fail_bad;
        return 1;
    }
    return 0;
}

/* src/sfl/ast.cpp:180-191: x + xdot * dt, active particles only (case.cpp:36-40). */
void nor_euler(int n, int comps, const uint8_t* active, const double* x, const double* xdot,
               double dt, double* out) {
    for (int c = 0; c < comps; ++c)
        for (int i = 0; i < n; ++i) {
            long k = (long)c * n + i;
            out[k] = active[i] ? x[k] + dt * xdot[k] : x[k];
        }
}

/* include/nauticle/sfl/random_state.hpp:22-41 */
static uint64_t mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

void nor_uniform_draws(uint64_t seed, int n, int ndraws, double a, double b, double* out) {
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < ndraws; ++k) {
            uint64_t x = mix(mix(seed ^ 0x6e61757469636c65ULL) ^ mix((uint64_t)i + 0x9e3779b9ULL) ^
                             (uint64_t)k);
            double u = (double)(x >> 11) * 0x1.0p-53;
            out[(long)k * n + i] = a + u * (b - a);
        }
}
