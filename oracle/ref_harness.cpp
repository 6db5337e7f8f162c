// oracle/ref_harness.cpp — TEST INFRASTRUCTURE (never on the product path).
//
// A C-ABI over the *unmodified* reference sources in /root/reference/proj,
// compiled against oracle/shim/Eigen/Dense by oracle/Makefile into
// oracle/_ref/libnauticle_ref.so. It drives the reference exactly the way the
// reference's own test fixture does (tests/helpers.hpp:26-80, CaseBuilder):
// Workspace + ParticleSystem + parse_expression + Case::solve_step over
// ThreadPool(P) (src/case.cpp:9-67, include/nauticle/thread_pool.hpp:20-46).
//
// Used by tests/ (golden fixtures, pinning oracle/nau_oracle.c) and by
// bench.py's reference arm / cpu_baseline leg only.
//
// The two laws BASELINE.json needs but the reference lacks (cubic-spline
// kernel, linear spring-dashpot DEM) are restated here as rules passed to the
// reference's public interact() (include/nauticle/interactions.hpp:29-36),
// following the pattern of tests/test_interactions.cpp:475-494.

// Standard headers first: the private->public trick below must not touch them.
#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <functional>
#include <map>
#include <memory>
#include <numbers>
#include <optional>
#include <ostream>
#include <sstream>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

// cells_ / cell_of_ have no accessor (particle_system.hpp:145-147); the cell
// tables are a parity probe, so this TU alone reads them directly.
#define private public
#include "nauticle/particle_system.hpp"
#undef private

#include "nauticle/assemble.hpp"
#include "nauticle/case.hpp"
#include "nauticle/io/case_document.hpp"
#include "nauticle/error.hpp"
#include "nauticle/interactions.hpp"
#include "nauticle/io/vtk.hpp"
#include "nauticle/kernel.hpp"
#include "nauticle/sfl/parser.hpp"

using namespace nauticle;

namespace {

thread_local std::string g_err;

struct Ref {
    std::unique_ptr<Case> cs = std::make_unique<Case>();
    std::map<std::string, sfl::NodePtr> parsed;  // keeps parsed trees alive
};

int fail(const std::exception& e) {
    g_err = e.what();
    if (auto* ne = dynamic_cast<const Error*>(&e)) return 1 + static_cast<int>(ne->kind());
    return 99;
}

Tensor tensor_from(int rows, int cols, const double* v) {
    Tensor t = Tensor::zeros(rows, cols);
    for (int c = 0; c < cols; ++c)
        for (int r = 0; r < rows; ++r) t(r, c) = v[c * rows + r];
    return t;
}

sfl::NodePtr parse(Ref* h, const std::string& expr) {
    sfl::ParseContext ctx{h->cs->workspace, &h->cs->random, h->cs->generation_ptr()};
    return sfl::parse_expression(expr, ctx);
}

// Component-major SoA write of one tensor per particle: out[k*n + i].
void put(double* out, int n, int i, const Tensor& t) {
    for (int c = 0; c < t.cols(); ++c)
        for (int r = 0; r < t.rows(); ++r) out[(c * t.rows() + r) * static_cast<long>(n) + i] = t(r, c);
}

// ---- restated laws absent from the reference (parity unpinned by its tests) ----

// Cubic spline (Monaghan M4), support 2h. Keyword "Wc3D220", D = dimension.
struct CubicKernel {
    double h, alpha;
    CubicKernel(int dim, double h_) : h(h_) {
        const double pi = std::numbers::pi;
        switch (dim) {
            case 1: alpha = 2.0 / (3.0 * h); break;
            case 2: alpha = 10.0 / (7.0 * pi * h * h); break;
            default: alpha = 1.0 / (pi * h * h * h); break;
        }
    }
    double value(double d) const {
        double q = d / h;
        if (q >= 2.0) return 0.0;
        if (q < 1.0) return alpha * (1.0 - 1.5 * q * q + 0.75 * q * q * q);
        double t = 2.0 - q;
        return alpha * (0.25 * t * t * t);
    }
    double dvalue_dq(double q) const {
        if (q >= 2.0) return 0.0;
        if (q < 1.0) return alpha * (-3.0 * q + 2.25 * q * q);
        double t = 2.0 - q;
        return alpha * (-0.75 * t * t);
    }
    Tensor gradient(const Tensor& rel) const {
        double d = rel.mat().norm();
        double q = d / h;
        if (q >= 2.0) return Tensor::zeros(rel.rows(), 1);
        double scale = -dvalue_dq(q) / (h * d);
        return Tensor(Tensor::Storage(rel.mat() * scale));
    }
};

// Same pair rules as src/interactions.cpp:40-150, with the kernel swapped.
Tensor cubic_rule(Ref* h, const std::string& op, int dim_kernel,
                  const std::vector<sfl::ExpressionNode*>& ops, int i) {
    const ParticleSystem& ps = *h->cs->workspace.particle_system();
    auto sc = [&](int slot, int j) { return ops[slot]->evaluate(j, 0).value(); };
    double radius = sc(3, i);
    CubicKernel k(dim_kernel, 0.5 * radius);
    const int d = ps.domain().dimension();
    if (op == "sph_S") {
        Tensor a_i = ops[0]->evaluate(i, 0);
        Tensor zero = Tensor::zeros(a_i.rows(), a_i.cols());
        return interact(ps, i, zero, [&](const Tensor& rel, int j, const Tensor&, const Tensor& g) {
            double dd = rel.mat().norm();
            if (dd > radius) return zero;
            double w = k.value(dd);
            if (w == 0.0) return zero;
            double rho_j = sc(2, j);
            double m_j = sc(1, j);
            Tensor a_j = mirror(ops[0]->evaluate(j, 0), g);
            return a_j * Tensor(m_j / rho_j * w);
        });
    }
    if (op == "sph_G11") {
        double a_i = sc(0, i), rho_i = sc(2, i);
        Tensor zero = Tensor::zeros(d, 1);
        Tensor sum = interact(ps, i, zero, [&](const Tensor& rel, int j, const Tensor&, const Tensor&) {
            double dd = rel.mat().norm();
            if (dd <= 0.0 || dd > radius) return zero;
            double rho_j = sc(2, j), a_j = sc(0, j), m_j = sc(1, j);
            return k.gradient(rel) * Tensor(m_j * (a_i / (rho_i * rho_i) + a_j / (rho_j * rho_j)));
        });
        return sum * Tensor(rho_i);
    }
    if (op == "sph_L0") {
        double a_i = sc(0, i);
        Tensor zero = Tensor(0.0);
        return interact(ps, i, zero, [&](const Tensor& rel, int j, const Tensor&, const Tensor&) {
            double dd = rel.mat().norm();
            if (dd > radius || dd <= 0.0) return zero;
            double rho_j = sc(2, j), a_j = sc(0, j), m_j = sc(1, j);
            Tensor grad = k.gradient(rel);
            return Tensor(2.0 * (a_j - a_i) * dot(rel, grad).value() / (dd * dd) * m_j / rho_j);
        });
    }
    if (op == "sph_D00") {
        Tensor a_i = ops[0]->evaluate(i, 0);
        Tensor zero = Tensor(0.0);
        return interact(ps, i, zero, [&](const Tensor& rel, int j, const Tensor&, const Tensor& g) {
            double dd = rel.mat().norm();
            if (dd <= 0.0 || dd > radius) return zero;
            double rho_j = sc(2, j), m_j = sc(1, j);
            Tensor a_j = mirror(ops[0]->evaluate(j, 0), g);
            return dot(a_j - a_i, k.gradient(rel)) * Tensor(m_j / rho_j);
        });
    }
    if (op == "sph_A") {
        Tensor v_i = ops[0]->evaluate(i, 0);
        double rho_i = sc(2, i);
        Tensor zero = Tensor::zeros(d, 1);
        return interact(ps, i, zero, [&](const Tensor& rel, int j, const Tensor&, const Tensor& g) {
            double dd = rel.mat().norm();
            if (dd > radius || dd <= 0.0) return zero;
            Tensor v_j = mirror(ops[0]->evaluate(j, 0), g);
            double approach = dot(v_j - v_i, rel).value();
            if (approach >= 0.0) return zero;
            double m_j = sc(1, j);
            double pi_ij = approach / (rho_i * dd * dd);
            return k.gradient(rel) * Tensor(m_j * pi_ij);
        });
    }
    throw runtime_error("nref: unknown cubic op ", op);
}

// Linear spring-dashpot normal force + Coulomb sliding friction (BASELINE cfg3),
// structured exactly like dem_sum / hertz_contact_force (interactions.cpp:152-193,
// 288-316). Operands: v, R, kn, en, m, cf, search radius.
Tensor lsd_rule(Ref* h, const std::vector<sfl::ExpressionNode*>& ops, int i) {
    const ParticleSystem& ps = *h->cs->workspace.particle_system();
    auto sc = [&](int slot, int j) { return ops[slot]->evaluate(j, 0).value(); };
    double radius = sc(6, i);
    Tensor v_i = ops[0]->evaluate(i, 0);
    double Ri = sc(1, i), kn = sc(2, i), en = sc(3, i), mi = sc(4, i), cf = sc(5, i);
    const double pi = std::numbers::pi;
    double le = std::log(en);
    double zeta = -le / std::sqrt(pi * pi + le * le);  // damping ratio for restitution en
    const int d = ps.domain().dimension();
    Tensor zero = Tensor::zeros(d, 1);
    Tensor force = interact(ps, i, zero, [&](const Tensor& rel, int j, const Tensor&, const Tensor& g) {
        double dist = rel.mat().norm();
        if (dist > radius) return zero;
        if (dist <= 0.0) return zero;
        double Rj = sc(1, j), mj = sc(4, j);
        double overlap = Ri + Rj - dist;
        if (overlap <= 0.0) return zero;
        Tensor v_j = mirror(ops[0]->evaluate(j, 0), g);
        double m_eff = mi * mj / (mi + mj);
        double c_n = 2.0 * zeta * std::sqrt(m_eff * kn);
        Tensor n_ji = rel / Tensor(dist);
        double overlap_rate = -dot(v_j - v_i, n_ji).value();
        double normal = kn * overlap + c_n * overlap_rate;
        Tensor f = -(n_ji * Tensor(normal));
        if (cf != 0.0) {
            Tensor v_ij = v_i - v_j;
            Tensor v_t = -v_ij + n_ji * dot(v_ij, n_ji);
            double vt_norm = v_t.mat().norm();
            if (vt_norm > 1e-12) f = f + v_t * Tensor(cf * std::abs(normal) / vt_norm);
        }
        return f;
    });
    return force / Tensor(mi);
}

}  // namespace

extern "C" {

const char* nref_last_error() { return g_err.c_str(); }

// splitmix-based counter RNG of the reference (random_state.hpp:22-30):
// out[k*n + i] = draw k of particle i, k < ndraws.
void nref_uniform_draws(uint64_t seed, int n, int ndraws, double a, double b, double* out) {
    RandomState rs(seed);
    rs.resize(n);
    for (int i = 0; i < n; ++i)
        for (int k = 0; k < ndraws; ++k) out[static_cast<long>(k) * n + i] = rs.uniform(i, a, b);
}

void* nref_create(int dim, const int* min_cells, const int* max_cells, const double* cell_size,
                  const int* kinds, int n, const double* pos_soa, uint64_t seed) {
    try {
        auto h = std::make_unique<Ref>();
        std::array<int, 3> mn{0, 0, 0}, mx{1, 1, 1};
        std::array<double, 3> cs{1, 1, 1};
        std::array<BoundaryKind, 3> bk{BoundaryKind::Cutoff, BoundaryKind::Cutoff, BoundaryKind::Cutoff};
        for (int a = 0; a < dim; ++a) {
            mn[a] = min_cells[a];
            mx[a] = max_cells[a];
            cs[a] = cell_size[a];
            bk[a] = static_cast<BoundaryKind>(kinds[a]);
        }
        Domain dom(dim, mn, mx, cs, bk);
        std::vector<Tensor> pos;
        pos.reserve(n);
        for (int i = 0; i < n; ++i) {
            Tensor p = Tensor::zeros(dim, 1);
            for (int a = 0; a < dim; ++a) p(a) = pos_soa[static_cast<long>(a) * n + i];
            pos.push_back(std::move(p));
        }
        h->cs->random = RandomState(seed);
        auto r = h->cs->workspace.add_field("r", std::move(pos));
        auto ps = std::make_shared<ParticleSystem>(dom, r);
        h->cs->workspace.attach_particle_system(ps);
        h->cs->random.resize(ps->particle_count());
        ps->apply_boundary_shift();
        ps->build_cells();
        return h.release();
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void nref_destroy(void* p) { delete static_cast<Ref*>(p); }

int nref_add_constant(void* p, const char* name, int rows, int cols, const double* v) {
    try {
        static_cast<Ref*>(p)->cs->workspace.add_constant(name, tensor_from(rows, cols, v));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int nref_add_variable(void* p, const char* name, int rows, int cols, const double* v) {
    try {
        static_cast<Ref*>(p)->cs->workspace.add_variable(name, tensor_from(rows, cols, v));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// soa: component-major [(c*rows + r) * n + i] (column-major per particle).
int nref_add_field(void* p, const char* name, int rows, int cols, const double* soa) {
    try {
        Ref* h = static_cast<Ref*>(p);
        const int n = h->cs->workspace.particle_count();
        std::vector<Tensor> vals;
        vals.reserve(n);
        for (int i = 0; i < n; ++i) {
            Tensor t = Tensor::zeros(rows, cols);
            for (int c = 0; c < cols; ++c)
                for (int r = 0; r < rows; ++r) t(r, c) = soa[static_cast<long>(c * rows + r) * n + i];
            vals.push_back(std::move(t));
        }
        h->cs->workspace.add_field(name, std::move(vals));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// Returns rows*cols (and writes rows/cols) or -1.
int nref_get_field(void* p, const char* name, double* soa, int* rows, int* cols) {
    try {
        Ref* h = static_cast<Ref*>(p);
        auto f = h->cs->workspace.find_field(name);
        if (!f) throw runtime_error("nref: no field ", name);
        const int n = f->particle_count();
        if (n == 0) return 0;
        *rows = f->values[0].rows();
        *cols = f->values[0].cols();
        if (soa)
            for (int i = 0; i < n; ++i) put(soa, n, i, f->values[i]);
        return *rows * *cols;
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

int nref_add_equation(void* p, const char* name, const char* text) {
    try {
        Ref* h = static_cast<Ref*>(p);
        std::string t(text);
        size_t eq = t.find('=');
        Equation e;
        e.name = name;
        std::string lhs = t.substr(0, eq);
        if (Variable* v = h->cs->workspace.find_variable(lhs))
            e.lhs_variable = v;
        else
            e.lhs_field = h->cs->workspace.find_field(lhs);
        if (!e.lhs_variable && !e.lhs_field) throw runtime_error("nref: unknown LHS ", lhs);
        e.writes_positions = lhs == "r";
        e.rhs = parse(h, t.substr(eq + 1));
        e.rhs->collect(e.info);
        h->cs->equations.push_back(std::move(e));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// The reference's result frame writer (io/vtk.cpp:193-304): make_frame + write_vtk.
int nref_write_vtk(void* p, const char* path, int binary, int frame_index, double time,
                   double simulated_time) {
    try {
        Ref* h = static_cast<Ref*>(p);
        h->cs->parameters.simulated_time = simulated_time;
        write_vtk(make_frame(*h->cs, frame_index, time), path,
                  binary ? VtkFormat::Binary : VtkFormat::Ascii);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int nref_solve_step(void* p, int threads) {
    try {
        static_cast<Ref*>(p)->cs->solve_step(ThreadPool(threads));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// Evaluate `expr` at particles [i0, i0+count) over ThreadPool(threads), the
// reference's parallel path (case.cpp:31-49). out (may be null) is SoA with
// stride `count`. Inactive particles are skipped (left untouched).
int nref_eval(void* p, const char* expr, int i0, int count, int threads, double* out, int* ncomp) {
    try {
        Ref* h = static_cast<Ref*>(p);
        ParticleSystem& ps = *h->cs->workspace.particle_system();
        sfl::NodePtr node = parse(h, expr);
        sfl::TreeInfo info;
        node->collect(info);
        if (info.needs_cells && ps.dirty()) ps.build_cells();
        for (sfl::ReductionNode* r : info.reductions) r->refresh(0);
        std::atomic<int> comps{0};
        ThreadPool(threads).parallel_blocks(count, [&](int, int b, int e) {
            for (int k = b; k < e; ++k) {
                int i = i0 + k;
                if (!ps.is_active(i)) continue;
                Tensor v = node->evaluate(i, 0);
                comps.store(v.size());
                if (out) put(out, count, k, v);
            }
        });
        if (ncomp) *ncomp = comps.load();
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// Restated laws through interact(): op in {sph_S, sph_G11, sph_L0, sph_D00, sph_A}
// with the cubic spline of dimension kdim, operands "A,m,rho,radius"
// (the kernel keyword slot is dropped); or op == "dem_lsd" with operands
// "v,R,kn,en,m,cf,radius".
int nref_eval_law(void* p, const char* op, int kdim, const char* const* operands, int n_ops,
                  int i0, int count, int threads, double* out, int* ncomp) {
    try {
        Ref* h = static_cast<Ref*>(p);
        ParticleSystem& ps = *h->cs->workspace.particle_system();
        if (ps.dirty()) ps.build_cells();
        std::vector<sfl::NodePtr> owned;
        std::vector<sfl::ExpressionNode*> ops;
        for (int k = 0; k < n_ops; ++k) {
            owned.push_back(parse(h, operands[k]));
            ops.push_back(owned.back().get());
        }
        std::string name(op);
        std::atomic<int> comps{0};
        ThreadPool(threads).parallel_blocks(count, [&](int, int b, int e) {
            for (int k = b; k < e; ++k) {
                int i = i0 + k;
                if (!ps.is_active(i)) continue;
                Tensor v = name == "dem_lsd" ? lsd_rule(h, ops, i) : cubic_rule(h, name, kdim, ops, i);
                comps.store(v.size());
                if (out) put(out, count, k, v);
            }
        });
        if (ncomp) *ncomp = comps.load();
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int nref_boundary_shift(void* p) {
    try {
        ParticleSystem& ps = *static_cast<Ref*>(p)->cs->workspace.particle_system();
        ps.apply_boundary_shift();
        ps.mark_dirty();
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int nref_build_cells(void* p) {
    try {
        static_cast<Ref*>(p)->cs->workspace.particle_system()->build_cells();
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

long nref_rebuild_count(void* p) {
    return static_cast<Ref*>(p)->cs->workspace.particle_system()->rebuild_count();
}

long nref_warning_count(void* p) {
    return static_cast<Ref*>(p)->cs->workspace.particle_system()->warning_count();
}

int nref_active(void* p, uint8_t* out) {
    ParticleSystem& ps = *static_cast<Ref*>(p)->cs->workspace.particle_system();
    for (int i = 0; i < ps.particle_count(); ++i) out[i] = ps.is_active(i) ? 1 : 0;
    return ps.active_count();
}

// Cell tables as flat arrays: cell_of[i] = flat cell of particle i (-1 when
// inactive); cell_start/cell_count per flat cell; sorted = concatenation of
// cells_ (ascending i within a cell). Rebuilds first when dirty.
int nref_cell_tables(void* p, int* cell_of, int* cell_start, int* cell_count, int* sorted) {
    try {
        ParticleSystem& ps = *static_cast<Ref*>(p)->cs->workspace.particle_system();
        if (ps.dirty()) ps.build_cells();
        const Domain& dom = ps.domain();
        const int n = ps.particle_count();
        for (int i = 0; i < n; ++i) {
            if (!ps.is_active(i)) {
                cell_of[i] = -1;
                continue;
            }
            int flat = 0;
            for (int a = dom.dimension() - 1; a >= 0; --a) flat = flat * dom.cells(a) + ps.cell_of_[i][a];
            cell_of[i] = flat;
        }
        int pos = 0;
        for (size_t c = 0; c < ps.cells_.size(); ++c) {
            cell_start[c] = pos;
            cell_count[c] = static_cast<int>(ps.cells_[c].size());
            for (int j : ps.cells_[c]) sorted[pos++] = j;
        }
        return static_cast<int>(ps.cells_.size());
    } catch (const std::exception& e) { return -fail(e); }
}

// counts[i] = number of for_each_neighbor candidates with |rel| <= radius (self included).
int nref_neighbor_counts(void* p, double radius, int* counts) {
    try {
        ParticleSystem& ps = *static_cast<Ref*>(p)->cs->workspace.particle_system();
        if (ps.dirty()) ps.build_cells();
        for (int i = 0; i < ps.particle_count(); ++i) {
            int c = 0;
            ps.for_each_neighbor(i, [&](const Tensor& rel, int, const Tensor&, const Tensor&) {
                if (rel.mat().norm() <= radius) ++c;
            });
            counts[i] = c;
        }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}


// ---- whole decks: assemble_case (src/assemble.cpp) from a CaseDocument whose
// bindings the caller parsed from a deck file (the reference's YAML reader is the
// one source file left out: yaml-cpp is absent). sections[k] is one of
// "constant", "variable", "field", "equation" (name = binding name, expr = text),
// "domain" (name in cell_size / minimum / maximum / boundary), "grid" (gid / gpos /
// gsize / goffset / gip_dist), "param" (simulated_time / print_interval).
void* nref_assemble(const char* const* sections, const char* const* names,
                    const char* const* exprs, int count, uint64_t seed) {
    try {
        CaseDocument doc;
        for (int k = 0; k < count; ++k) {
            const std::string sec = sections[k], name = names[k], expr = exprs[k];
            if (sec == "constant") doc.constants.push_back({name, expr});
            else if (sec == "variable") doc.variables.push_back({name, expr});
            else if (sec == "field") doc.fields.push_back({name, expr});
            else if (sec == "equation") doc.equations.push_back({name, expr});
            else if (sec == "domain") {
                if (name == "cell_size") doc.cell_size = expr;
                else if (name == "minimum") doc.minimum = expr;
                else if (name == "maximum") doc.maximum = expr;
                else if (name == "boundary") doc.boundary = expr;
                else throw runtime_error("nref_assemble: domain key ", name);
            } else if (sec == "grid") {
                if (name == "gid") doc.grid_gid = expr;
                else if (name == "gpos") doc.gpos = expr;
                else if (name == "gsize") doc.gsize = expr;
                else if (name == "goffset") doc.goffset = expr;
                else if (name == "gip_dist") doc.gip_dist = expr;
                else throw runtime_error("nref_assemble: grid key ", name);
            } else if (sec == "param") {
                if (name == "simulated_time") doc.simulated_time = expr;
                else if (name == "print_interval") doc.print_interval = expr;
            } else {
                throw runtime_error("nref_assemble: section ", sec);
            }
        }
        AssembleOptions opts;
        opts.seed = seed;
        auto h = std::make_unique<Ref>();
        h->cs = assemble_case(doc, opts);
        return h.release();
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// The Case behind a handle (for the reference-side GPU binding's tests, integration/).
void* nref_case_ptr(void* p) { return static_cast<Ref*>(p)->cs.get(); }

// Domain of the assembled case: dim, min/max cells, cell sizes, kinds (3 each), N.
int nref_domain(void* p, int* dim, int* min_cells, int* max_cells, double* cell_size,
                int* kinds) {
    const ParticleSystem& ps = *static_cast<Ref*>(p)->cs->workspace.particle_system();
    const Domain& d = ps.domain();
    *dim = d.dimension();
    for (int a = 0; a < 3; ++a) {
        min_cells[a] = d.min_cells_[a];
        max_cells[a] = d.max_cells_[a];
        cell_size[a] = d.cell_size(a);
        kinds[a] = static_cast<int>(d.boundary(a));
    }
    return ps.particle_count();
}

// Symbols in definition order: kind 0 constants, 1 variables, 2 fields. Returns the
// count; for k < count writes the name (NUL-terminated, <= cap) and rows/cols, and
// for constants/variables the value (column-major, 9 doubles).
int nref_symbol(void* p, int kind, int k, char* name, int cap, int* rows, int* cols,
                double* value) {
    Workspace& ws = static_cast<Ref*>(p)->cs->workspace;
    auto out = [&](const std::string& nm, const Tensor& t) {
        std::snprintf(name, cap, "%s", nm.c_str());
        *rows = t.rows();
        *cols = t.cols();
        if (value)
            for (int c = 0; c < t.cols(); ++c)
                for (int r = 0; r < t.rows(); ++r) value[c * t.rows() + r] = t(r, c);
    };
    if (kind == 0) {
        const auto& v = ws.constants();
        if (k >= 0 && k < (int)v.size()) out(v[k]->name, v[k]->value);
        return (int)v.size();
    }
    if (kind == 1) {
        const auto& v = ws.variables();
        if (k >= 0 && k < (int)v.size()) out(v[k]->name, v[k]->value);
        return (int)v.size();
    }
    const auto& v = ws.fields();
    if (k >= 0 && k < (int)v.size())
        out(v[k]->name, v[k]->values.empty() ? Tensor(0.0) : v[k]->values[0]);
    return (int)v.size();
}

// Equation k as (name, "lhs=rhs" in the reference's canonical printed form).
int nref_equation(void* p, int k, char* name, int ncap, char* text, int tcap) {
    const auto& eqs = static_cast<Ref*>(p)->cs->equations;
    if (k >= 0 && k < (int)eqs.size()) {
        std::snprintf(name, ncap, "%s", eqs[k].name.c_str());
        std::snprintf(text, tcap, "%s=%s", eqs[k].lhs_name().c_str(), eqs[k].rhs->to_text().c_str());
    }
    return (int)eqs.size();
}

// The case's rand stream state (per-particle draw counters) and seed.
int nref_rand_counters(void* p, uint64_t* seed, uint64_t* counters) {
    Case& cs = *static_cast<Ref*>(p)->cs;
    *seed = cs.random.seed();
    const int n = cs.workspace.particle_count();
    const auto& cnt = cs.random.counters();
    for (int i = 0; i < n && counters; ++i) counters[i] = i < (int)cnt.size() ? cnt[i] : 0;
    return n;
}

// Variable value (column-major, <= 9) after solving; returns rows*cols or -1.
int nref_get_variable(void* p, const char* name, double* value, int* rows, int* cols) {
    try {
        Variable* v = static_cast<Ref*>(p)->cs->workspace.find_variable(name);
        if (!v) throw runtime_error("nref: no variable ", name);
        *rows = v->value.rows();
        *cols = v->value.cols();
        for (int c = 0; c < *cols; ++c)
            for (int r = 0; r < *rows; ++r) value[c * *rows + r] = v->value(r, c);
        return *rows * *cols;
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

// Wendland kernel of the reference (kernel.cpp:37-69) for KATs.
double nref_kernel_value(const char* keyword, double h, double d) {
    try {
        return Kernel(decode_kernel_keyword(keyword), h).value(d);
    } catch (const std::exception& e) {
        fail(e);
        return std::nan("");
    }
}

}  // extern "C"
