// integration/gpu_case.cpp — see gpu_case.hpp. Reference-side code: it uses only the
// reference's public API (Case, Workspace, ParticleSystem, Domain, Tensor, Error) and
// the C-ABI of include/nauticle_gpu.h.
#include "gpu_case.hpp"

#include <cmath>
#include <string>
#include <vector>

#include "nauticle/error.hpp"

namespace nauticle {

namespace {

// Field::values (AoS Tensors) <-> the C-ABI's SoA, component c = col * rows + row.
std::vector<double> to_soa(const Field& f) {
    const int n = f.particle_count();
    const int rows = n ? f.values[0].rows() : 1, cols = n ? f.values[0].cols() : 1;
    std::vector<double> soa(static_cast<size_t>(n) * rows * cols);
    for (int i = 0; i < n; ++i)
        for (int c = 0; c < cols; ++c)
            for (int r = 0; r < rows; ++r)
                soa[static_cast<size_t>(c * rows + r) * n + i] = f.values[i](r, c);
    return soa;
}

void from_soa(Field& f, const std::vector<double>& soa) {
    const int n = f.particle_count();
    for (int i = 0; i < n; ++i) {
        Tensor& t = f.values[i];
        for (int c = 0; c < t.cols(); ++c)
            for (int r = 0; r < t.rows(); ++r)
                t(r, c) = soa[static_cast<size_t>(c * t.rows() + r) * n + i];
    }
}

std::vector<double> col_major(const Tensor& t) {
    std::vector<double> v(9, 0.0);
    for (int c = 0; c < t.cols(); ++c)
        for (int r = 0; r < t.rows(); ++r) v[c * t.rows() + r] = t(r, c);
    return v;
}

ErrorKind kind_of(nau_status s) {
    if (s == NAU_ERR_NAN) return ErrorKind::Nan;
    if (s == NAU_ERR_ARG) return ErrorKind::Assembly;  // equations rejected when added
    return ErrorKind::Runtime;
}

}  // namespace

void GpuCase::check(nau_status s) const {
    if (s == NAU_OK) return;
    long bad = -1;
    const char* msg = nau_last_error(ctx_, &bad);  // the context's message, not the static one
    throw Error(kind_of(s), msg ? msg : "nau error");
}

void GpuCase::check_case(nau_status s) const {
    if (s == NAU_OK) return;
    long bad = -1;
    const char* msg = nau_case_last_error(exec_, &bad);  // "equation '<name>': ..."
    throw Error(kind_of(s), msg ? msg : "nau error");
}

GpuCase::GpuCase(Case& cs, int device, bool fast) : cs_(cs) {
    if (nau_create(device, &ctx_) != NAU_OK) throw Error(ErrorKind::Runtime, "nau_create failed");
    check(nau_set_mode(ctx_, fast ? NAU_MODE_FAST : NAU_MODE_EXACT));
    const ParticleSystem& ps = cs.particle_system();
    const Domain& d = ps.domain();
    int mn[3], mx[3], kind[3];
    double size[3];
    for (int a = 0; a < 3; ++a) {  // domain.hpp:26-33: lo = min_cells * cell_size
        mn[a] = static_cast<int>(std::lround(d.lo(a) / d.cell_size(a)));
        mx[a] = mn[a] + d.cells(a);
        size[a] = d.cell_size(a);
        kind[a] = static_cast<int>(d.boundary(a));  // Periodic 0, Symmetric 1, Cutoff 2
    }
    check(nau_set_domain(ctx_, d.dimension(), mn, mx, size, kind));
    const std::vector<double> pos = to_soa(ps.positions());
    check(nau_set_particles(ctx_, ps.particle_count(), pos.data()));
    for (const auto& f : cs.workspace.fields()) {
        if (f->name == "r") continue;
        const int rows = f->values.empty() ? 1 : f->values[0].rows();
        const int cols = f->values.empty() ? 1 : f->values[0].cols();
        int id = -1;
        check(nau_alloc_field(ctx_, rows, cols, &id));
        const std::vector<double> soa = to_soa(*f);
        check(nau_upload(ctx_, id, soa.data(), f->particle_count()));
        field_id_[f->name] = id;
    }
    // the case's rand stream: same seed and per-particle draw counters
    std::vector<unsigned long long> counters(ps.particle_count(), 0ULL);
    const auto& cnt = cs.random.counters();
    for (size_t i = 0; i < counters.size() && i < cnt.size(); ++i) counters[i] = cnt[i];
    check(nau_set_random_state(ctx_, cs.random.seed(), counters.data()));

    check(nau_case_create(ctx_, &exec_));
    for (const auto& kv : field_id_) check_case(nau_case_field(exec_, kv.first.c_str(), kv.second));
    for (const auto& c : cs.workspace.constants()) {
        const auto v = col_major(c->value);
        check_case(nau_case_constant(exec_, c->name.c_str(), c->value.rows(), c->value.cols(), v.data()));
    }
    for (const auto& var : cs.workspace.variables()) {
        const auto v = col_major(var->value);
        check_case(nau_case_variable(exec_, var->name.c_str(), var->value.rows(), var->value.cols(),
                                     v.data()));
    }
    for (const auto& eq : cs.equations) {  // equation.hpp: lhs=rhs in canonical printed form
        const std::string text = eq.lhs_name() + "=" + eq.rhs->to_text();
        check_case(nau_case_equation(exec_, eq.name.c_str(), text.c_str()));
    }
}

GpuCase::~GpuCase() {
    nau_case_destroy(exec_);
    nau_destroy(ctx_);
}

void GpuCase::solve_step() { check_case(nau_case_solve_step(exec_)); }

void GpuCase::download() {
    const int n = cs_.particle_system().particle_count();
    for (auto& f : cs_.workspace.fields()) {
        const int id = f->name == "r" ? 0 : field_id_.at(f->name);
        int rows = 1, cols = 1;
        check(nau_field_shape(ctx_, id, &rows, &cols));
        std::vector<double> soa(static_cast<size_t>(n) * rows * cols);
        check(nau_download(ctx_, id, soa.data(), n));
        from_soa(*f, soa);
    }
    for (auto& var : cs_.workspace.variables()) {
        double v[9];
        int rows = 1, cols = 1;
        check_case(nau_case_get_variable(exec_, var->name.c_str(), v, &rows, &cols));
        Tensor t = Tensor::zeros(rows, cols);
        for (int c = 0; c < cols; ++c)
            for (int r = 0; r < rows; ++r) t(r, c) = v[c * rows + r];
        var->value = t;
    }
}

}  // namespace nauticle

// ---- test glue: a C entry point per method, for tests/test_gpu_binding.py (ctypes) ----
extern "C" {

thread_local std::string g_gpucase_err;

const char* gpucase_last_error() { return g_gpucase_err.c_str(); }

void* gpucase_create(void* case_ptr, int device, int fast) {
    try {
        return new nauticle::GpuCase(*static_cast<nauticle::Case*>(case_ptr), device, fast != 0);
    } catch (const std::exception& e) {
        g_gpucase_err = e.what();
        return nullptr;
    }
}

int gpucase_solve_step(void* g) {
    try {
        static_cast<nauticle::GpuCase*>(g)->solve_step();
        return 0;
    } catch (const nauticle::Error& e) {
        g_gpucase_err = e.what();
        return 1 + static_cast<int>(e.kind());
    }
}

int gpucase_download(void* g) {
    try {
        static_cast<nauticle::GpuCase*>(g)->download();
        return 0;
    } catch (const std::exception& e) {
        g_gpucase_err = e.what();
        return 1;
    }
}

int gpucase_active(void* g, unsigned char* out) {
    return nau_get_active(static_cast<nauticle::GpuCase*>(g)->context(), out);
}

void gpucase_destroy(void* g) { delete static_cast<nauticle::GpuCase*>(g); }

}  // extern "C"
