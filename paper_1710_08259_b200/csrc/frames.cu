// frames.cu — result frames from device state and hot start:
// the legacy-VTK PolyData writer and reader of the reference (io/vtk.cpp:193-464,
// make_frame / write_vtk / read_vtk), byte for byte.
//
// Writer: every per-particle array leaves the GPU once, already in the file's
// layout — original particle order (the reference's index order), vectors padded
// to 3 components, matrices row-major, and for BINARY files big-endian doubles —
// produced by one gather kernel per array (k_frame_pack, HBM-bound byte work);
// the host only streams the bytes out (ASCII: shortest round-trip decimals,
// std::to_chars, as format.hpp:12-16). The case metadata the host owns (deck
// equations, variables, constants, parameters) comes in as the strings the
// reference would write; the domain string is rebuilt from the context
// (domain.cpp:68-83) and the rand counters come from the device RandomState.
//
// Reader: host-side parse of the reference's format (ASCII or BINARY) into a
// frame handle the host uses to hot-start a context (nau_set_particles /
// nau_alloc_field / nau_upload / nau_set_random_state), as assemble.cpp:227-271.
#include <charconv>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "nau_internal.cuh"

namespace nau {
namespace {

__device__ __forceinline__ double bswap_double(double v) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(v);
    const unsigned lo = (unsigned)u, hi = (unsigned)(u >> 32);
    const unsigned long long s = ((unsigned long long)__byte_perm(lo, 0, 0x0123) << 32) |
                                 __byte_perm(hi, 0, 0x0123);
    return __longlong_as_double((long long)s);
}

// One array of the frame: slot k (cell order) -> tuple orig[k] of `width`
// doubles; component q of the tuple is source component src_comp(q) (or 0.0
// past `rows` for a padded vector). Matrices: q = r * cols + c <- (c*rows + r).
__global__ void k_frame_pack(long n, int rows, int cols, int width, const double* src,
                             const int* orig, int big_endian, double* out) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const long o = orig[k];
    for (int q = 0; q < width; ++q) {
        double v = 0.0;
        if (q < rows * cols) {
            const int r = q / cols, c = q % cols;
            v = src[(long)(c * rows + r) * n + k];
        }
        out[o * width + q] = big_endian ? bswap_double(v) : v;
    }
}

std::string fmt(double v) {
    char buf[32];
    auto res = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, res.ptr);
}

double host_bswap(double v) {
    unsigned long long u;
    std::memcpy(&u, &v, 8);
    u = __builtin_bswap64(u);
    std::memcpy(&v, &u, 8);
    return v;
}

// VtkWriter::doubles / ints (vtk.cpp:31-63); `data` is already big-endian in binary mode.
void put_doubles(std::ostream& out, const double* data, size_t count, int per_line, bool binary) {
    if (binary) {
        out.write(reinterpret_cast<const char*>(data), (std::streamsize)(count * sizeof(double)));
        out << '\n';
        return;
    }
    std::string line;
    for (size_t k = 0; k < count; ++k) {
        line += fmt(data[k]);
        line += ((k + 1) % per_line == 0) ? '\n' : ' ';
        if (line.size() > (1 << 16)) {
            out << line;
            line.clear();
        }
    }
    if (count % per_line != 0) line += '\n';
    out << line;
}

void put_host_doubles(std::ostream& out, std::vector<double> v, int per_line, bool binary) {
    if (binary)
        for (double& x : v) x = host_bswap(x);
    put_doubles(out, v.data(), v.size(), per_line, binary);
}

void put_vertices(std::ostream& out, long n, bool binary) {
    if (binary) {
        std::vector<int32_t> cells(2 * n);
        for (long i = 0; i < n; ++i) {
            cells[2 * i] = (int32_t)__builtin_bswap32(1u);
            cells[2 * i + 1] = (int32_t)__builtin_bswap32((uint32_t)i);
        }
        out.write(reinterpret_cast<const char*>(cells.data()),
                  (std::streamsize)(cells.size() * sizeof(int32_t)));
        out << '\n';
        return;
    }
    std::string line;
    for (long i = 0; i < n; ++i) {
        line += "1 " + std::to_string(i) + '\n';
        if (line.size() > (1 << 16)) {
            out << line;
            line.clear();
        }
    }
    out << line;
}

void string_array(std::ostream& out, const char* name, const std::vector<std::string>& items) {
    out << name << " 1 " << items.size() << " string\n";
    for (const auto& s : items) out << s << '\n';
}

std::vector<std::string> strings_of(const char* const* v, int n) {
    std::vector<std::string> out;
    for (int k = 0; k < n; ++k) out.emplace_back(v[k]);
    return out;
}

}  // namespace
}  // namespace nau

// ---- reader ---------------------------------------------------------------
struct nau_vtk_frame {
    int dim = 1, frame_index = 0;
    double time = 0.0;
    long n = 0;
    std::vector<double> pos;  // dim x n
    struct Arr {
        std::string name;
        int rows = 1, cols = 1;
        std::vector<double> soa;  // (c*rows + r) * n + i
    };
    std::vector<Arr> arrays;
    std::vector<std::pair<std::string, std::vector<std::string>>> strings;
    std::vector<unsigned long long> rand_counters;
};

namespace {

struct Scanner {  // VtkScanner (vtk.cpp:100-181)
    std::string buf;
    size_t pos = 0;
    bool eof() {
        skip_ws();
        return pos >= buf.size();
    }
    void skip_ws() {
        while (pos < buf.size() && std::isspace((unsigned char)buf[pos])) ++pos;
    }
    std::string line() {
        size_t end = buf.find('\n', pos);
        std::string l = end == std::string::npos ? buf.substr(pos) : buf.substr(pos, end - pos);
        pos = end == std::string::npos ? buf.size() : end + 1;
        if (!l.empty() && l.back() == '\r') l.pop_back();
        return l;
    }
    std::string nonempty_line() {
        while (pos < buf.size()) {
            std::string l = line();
            if (!l.empty()) return l;
        }
        throw std::runtime_error("unexpected end of VTK file");
    }
    std::string word() {
        skip_ws();
        size_t s = pos;
        while (pos < buf.size() && !std::isspace((unsigned char)buf[pos])) ++pos;
        if (s == pos) throw std::runtime_error("unexpected end of VTK file");
        return buf.substr(s, pos - s);
    }
    std::vector<double> numbers(long count, bool binary) {
        std::vector<double> out(count);
        if (binary) {
            if (pos + count * sizeof(double) > buf.size())
                throw std::runtime_error("truncated binary block");
            for (long k = 0; k < count; ++k) {
                double v;
                std::memcpy(&v, buf.data() + pos, 8);
                out[k] = nau::host_bswap(v);
                pos += 8;
            }
            if (pos < buf.size() && buf[pos] == '\n') ++pos;
        } else {
            for (long k = 0; k < count; ++k) {
                std::string w = word();
                double v = 0.0;
                auto r = std::from_chars(w.data(), w.data() + w.size(), v);
                if (r.ec != std::errc() || r.ptr != w.data() + w.size())
                    throw std::runtime_error("expected a number, got '" + w + "'");
                out[k] = v;
            }
        }
        return out;
    }
    void skip_ints(long count, bool binary) {
        if (binary) {
            pos += count * sizeof(int32_t);
            if (pos > buf.size()) throw std::runtime_error("truncated binary block");
            if (pos < buf.size() && buf[pos] == '\n') ++pos;
        } else {
            for (long k = 0; k < count; ++k) word();
        }
    }
};

std::vector<std::string> words_of(const std::string& l) {
    std::istringstream ss(l);
    std::vector<std::string> w;
    std::string x;
    while (ss >> x) w.push_back(x);
    return w;
}

thread_local std::string g_vtk_err;

}  // namespace

extern "C" {

nau_status nau_write_vtk(nau_ctx* c, const char* path, int binary, const nau_frame_meta* m) {
    using namespace nau;
    if (!m || !path) return NAU_ERR_ARG;
    for (int k = 0; k < m->n_fields; ++k) {
        const int id = m->field_ids[k];
        if (id <= 0 || id >= (int)c->fields.size() || !c->fields[id].live) {
            c->last_error = "nau_write_vtk: bad field id";
            return NAU_ERR_ARG;
        }
    }
    std::ofstream out(path, std::ios::binary);
    if (!out) {
        c->last_error = std::string("cannot write result file '") + path + "'";
        return NAU_ERR_RUNTIME;
    }
    const bool bin = binary != 0;
    const long n = c->n;
    const int dim = c->dom.dim;
    // device staging for the largest array (n x 9 doubles), one D2H per array
    double* d_buf = nullptr;
    std::vector<double> h_buf((size_t)n * 9 + 1);
    if (n && cudaMalloc(&d_buf, sizeof(double) * n * 9) != cudaSuccess) {
        c->last_error = "nau_write_vtk: out of device memory";
        return NAU_ERR_CUDA;
    }
    auto fetch = [&](const double* src, int rows, int cols, int width) {
        if (n == 0) return;
        k_frame_pack<<<(int)((n + 255) / 256), 256, 0, c->stream>>>(n, rows, cols, width, src,
                                                                    c->d_orig, bin ? 1 : 0, d_buf);
        c->launches++;
        cudaMemcpyAsync(h_buf.data(), d_buf, sizeof(double) * n * width, cudaMemcpyDeviceToHost,
                        c->stream);
        cudaStreamSynchronize(c->stream);
    };

    out << "# vtk DataFile Version 3.0\n";
    out << "nauticle result frame\n";
    out << (bin ? "BINARY" : "ASCII") << '\n';
    out << "DATASET POLYDATA\n";
    std::vector<std::string> shapes;
    for (int k = 0; k < m->n_fields; ++k) {
        const FieldBuf& f = c->fields[m->field_ids[k]];
        if (n > 0 && f.comps() > 1)
            shapes.push_back(std::string(m->field_names[k]) + "=" + std::to_string(f.rows) + "x" +
                             std::to_string(f.cols));
    }
    // rand counters: written when any particle has drawn (vtk.cpp:208-213)
    std::vector<unsigned long long> counters;
    if (c->d_rng && c->rng_len >= n && n > 0) {
        counters.resize(n);
        cudaMemcpy(counters.data(), c->d_rng, sizeof(unsigned long long) * n,
                   cudaMemcpyDeviceToHost);
        bool any = false;
        for (auto v : counters) any |= v != 0;
        if (!any) counters.clear();
    }
    int arrays = 5;
    if (!shapes.empty()) ++arrays;
    if (m->n_variables) ++arrays;
    if (m->n_constants) ++arrays;
    if (m->n_equations) ++arrays;
    if (!counters.empty()) ++arrays;
    out << "FIELD CaseData " << arrays << '\n';
    out << "frame 1 1 double\n";
    put_host_doubles(out, {(double)m->frame_index}, 1, bin);
    out << "time 1 1 double\n";
    put_host_doubles(out, {m->time}, 1, bin);
    out << "dimension 1 1 double\n";
    put_host_doubles(out, {(double)dim}, 1, bin);
    std::string domain;
    if (m->domain_text) {
        domain = m->domain_text;
    } else {  // Domain::describe (domain.cpp:68-83)
        static const char* kind[3] = {"periodic", "symmetric", "cutoff"};
        auto join = [&](auto value_of) {
            std::string s;
            for (int a = 0; a < dim; ++a) s += (a ? "|" : "") + value_of(a);
            return s;
        };
        domain = "cell_size=" + join([&](int a) { return fmt(c->dom.cs[a]); });
        domain += ";minimum=" + join([&](int a) { return std::to_string(c->min_cells[a]); });
        domain += ";maximum=" + join([&](int a) { return std::to_string(c->max_cells[a]); });
        domain += ";boundary=" + join([&](int a) { return std::string(kind[c->dom.kind[a]]); });
    }
    string_array(out, "domain", {domain});
    string_array(out, "params", {m->params_text ? m->params_text : "simulated_time=0"});
    if (!shapes.empty()) string_array(out, "field_shapes", shapes);
    if (m->n_variables) string_array(out, "variables", strings_of(m->variables, m->n_variables));
    if (m->n_constants) string_array(out, "constants", strings_of(m->constants, m->n_constants));
    if (m->n_equations) string_array(out, "equations", strings_of(m->equations, m->n_equations));
    if (!counters.empty()) {
        out << "rand_counters 1 " << counters.size() << " double\n";
        std::vector<double> dc(counters.begin(), counters.end());
        put_host_doubles(out, std::move(dc), 1, bin);
    }
    out << "POINTS " << n << " double\n";
    fetch(c->fields[0].d, dim, 1, 3);
    put_doubles(out, h_buf.data(), (size_t)n * 3, 3, bin);
    out << "VERTICES " << n << ' ' << 2 * n << '\n';
    put_vertices(out, n, bin);
    out << "POINT_DATA " << n << '\n';
    std::vector<int> matrices;
    if (n > 0) {
        for (int k = 0; k < m->n_fields; ++k) {
            const FieldBuf& f = c->fields[m->field_ids[k]];
            if (f.comps() == 1) {
                out << "SCALARS " << m->field_names[k] << " double 1\n";
                out << "LOOKUP_TABLE default\n";
                fetch(f.d, 1, 1, 1);
                put_doubles(out, h_buf.data(), (size_t)n, 1, bin);
            } else if (f.cols == 1) {
                out << "VECTORS " << m->field_names[k] << " double\n";
                fetch(f.d, f.rows, 1, 3);
                put_doubles(out, h_buf.data(), (size_t)n * 3, 3, bin);
            } else {
                matrices.push_back(k);
            }
        }
    }
    if (!matrices.empty()) {
        out << "FIELD PerParticle " << matrices.size() << '\n';
        for (int k : matrices) {
            const FieldBuf& f = c->fields[m->field_ids[k]];
            out << m->field_names[k] << ' ' << f.comps() << ' ' << n << " double\n";
            fetch(f.d, f.rows, f.cols, f.comps());
            put_doubles(out, h_buf.data(), (size_t)n * f.comps(), f.comps(), bin);
        }
    }
    if (d_buf) cudaFree(d_buf);
    if (!out) {
        c->last_error = std::string("failed while writing result file '") + path + "'";
        return NAU_ERR_RUNTIME;
    }
    return NAU_OK;
}

nau_status nau_vtk_read(const char* path, nau_vtk_frame** out_frame) {
    *out_frame = nullptr;
    try {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw std::runtime_error(std::string("cannot open result file '") + path + "'");
        std::ostringstream ss;
        ss << in.rdbuf();
        Scanner sc{ss.str()};
        if (sc.line().rfind("# vtk DataFile", 0) != 0)
            throw std::runtime_error(std::string("'") + path + "' is not a legacy VTK file");
        sc.line();
        const std::string fmt_word = sc.nonempty_line();
        const bool binary = fmt_word == "BINARY";
        if (!binary && fmt_word != "ASCII")
            throw std::runtime_error("unknown VTK data format '" + fmt_word + "'");
        if (words_of(sc.nonempty_line()) != std::vector<std::string>{"DATASET", "POLYDATA"})
            throw std::runtime_error("expected DATASET POLYDATA");
        struct Raw {
            std::string name;
            int comps = 1;
            long tuples = 0;
            bool str = false;
            std::vector<double> data;
            std::vector<std::string> strings;
        };
        std::vector<Raw> case_data, point;
        std::vector<double> pts;
        long np = 0;
        bool in_point = false;
        auto field_block = [&](long count, std::vector<Raw>& into) {
            for (long k = 0; k < count; ++k) {
                auto h = words_of(sc.nonempty_line());
                if (h.size() != 4) throw std::runtime_error("malformed FIELD array header");
                Raw a;
                a.name = h[0];
                a.comps = std::stoi(h[1]);
                a.tuples = std::stol(h[2]);
                if (h[3] == "string") {
                    a.str = true;
                    for (long t = 0; t < a.tuples; ++t) a.strings.push_back(sc.line());
                } else {
                    a.data = sc.numbers(a.comps * a.tuples, binary);
                }
                into.push_back(std::move(a));
            }
        };
        while (!sc.eof()) {
            auto w = words_of(sc.nonempty_line());
            if (w.empty()) continue;
            if (w[0] == "FIELD") {
                field_block(std::stol(w[2]), in_point ? point : case_data);
            } else if (w[0] == "POINTS") {
                np = std::stol(w[1]);
                pts = sc.numbers(np * 3, binary);
            } else if (w[0] == "VERTICES") {
                sc.skip_ints(std::stol(w[2]), binary);
            } else if (w[0] == "POINT_DATA") {
                in_point = true;
                if (std::stol(w[1]) != np) throw std::runtime_error("POINT_DATA count mismatch");
            } else if (w[0] == "SCALARS") {
                if (sc.nonempty_line().rfind("LOOKUP_TABLE", 0) != 0)
                    throw std::runtime_error("SCALARS without LOOKUP_TABLE");
                Raw a;
                a.name = w[1];
                a.tuples = np;
                a.data = sc.numbers(np, binary);
                point.push_back(std::move(a));
            } else if (w[0] == "VECTORS") {
                Raw a;
                a.name = w[1];
                a.comps = 3;
                a.tuples = np;
                a.data = sc.numbers(np * 3, binary);
                point.push_back(std::move(a));
            } else {
                throw std::runtime_error("unsupported VTK section '" + w[0] + "'");
            }
        }
        auto find = [&](const char* name) -> const Raw* {
            for (const auto& a : case_data)
                if (a.name == name) return &a;
            return nullptr;
        };
        auto f = std::make_unique<nau_vtk_frame>();
        const Raw *dim = find("dimension"), *time = find("time"), *fidx = find("frame");
        if (!dim || !time || !fidx) throw std::runtime_error("no CaseData block of a result frame");
        f->dim = (int)dim->data.at(0);
        f->time = time->data.at(0);
        f->frame_index = (int)fidx->data.at(0);
        f->n = np;
        for (const auto& a : case_data)
            if (a.str) f->strings.emplace_back(a.name, a.strings);
        if (const Raw* rc = find("rand_counters"))
            for (double v : rc->data) f->rand_counters.push_back((unsigned long long)v);
        std::vector<std::pair<std::string, std::pair<int, int>>> shapes;
        if (const Raw* sh = find("field_shapes"))
            for (const auto& s : sh->strings) {
                size_t eq = s.find('='), x = s.find('x', eq);
                shapes.emplace_back(s.substr(0, eq),
                                    std::make_pair(std::stoi(s.substr(eq + 1, x - eq - 1)),
                                                   std::stoi(s.substr(x + 1))));
            }
        f->pos.assign((size_t)f->dim * np, 0.0);
        for (long i = 0; i < np; ++i)
            for (int a = 0; a < f->dim; ++a) f->pos[(size_t)a * np + i] = pts[i * 3 + a];
        for (const auto& a : point) {  // vtk.cpp:441-460
            nau_vtk_frame::Arr arr;
            arr.name = a.name;
            int rows = 1, cols = 1;
            if (a.comps != 1) {
                rows = std::min(3, f->dim);
                for (const auto& [nm, sh] : shapes)
                    if (nm == a.name) rows = sh.first, cols = sh.second;
                if (a.comps == 3 && rows * cols > 3) rows = 3, cols = 1;
            }
            arr.rows = rows;
            arr.cols = cols;
            arr.soa.assign((size_t)rows * cols * a.tuples, 0.0);
            for (long i = 0; i < a.tuples; ++i) {
                int k = 0;
                for (int r = 0; r < rows; ++r)
                    for (int cc = 0; cc < cols; ++cc)
                        arr.soa[(size_t)(cc * rows + r) * a.tuples + i] = a.data[i * a.comps + k++];
            }
            f->arrays.push_back(std::move(arr));
        }
        *out_frame = f.release();
        return NAU_OK;
    } catch (const std::exception& e) {
        g_vtk_err = e.what();
        return NAU_ERR_RUNTIME;
    }
}

void nau_vtk_free(nau_vtk_frame* f) { delete f; }

const char* nau_vtk_last_error(void) { return g_vtk_err.c_str(); }

long nau_vtk_points(const nau_vtk_frame* f, int* dim, int* frame_index, double* time,
                    const double** pos_soa) {
    if (dim) *dim = f->dim;
    if (frame_index) *frame_index = f->frame_index;
    if (time) *time = f->time;
    if (pos_soa) *pos_soa = f->pos.data();
    return f->n;
}

int nau_vtk_array_count(const nau_vtk_frame* f) { return (int)f->arrays.size(); }

const char* nau_vtk_array(const nau_vtk_frame* f, int k, int* rows, int* cols,
                          const double** soa) {
    if (k < 0 || k >= (int)f->arrays.size()) return nullptr;
    const auto& a = f->arrays[k];
    *rows = a.rows;
    *cols = a.cols;
    *soa = a.soa.data();
    return a.name.c_str();
}

int nau_vtk_strings(const nau_vtk_frame* f, const char* key, const char* const** items) {
    for (const auto& [name, v] : f->strings)
        if (name == key) {
            static thread_local std::vector<const char*> ptrs;
            ptrs.clear();
            for (const auto& s : v) ptrs.push_back(s.c_str());
            *items = ptrs.data();
            return (int)ptrs.size();
        }
    *items = nullptr;
    return 0;
}

long nau_vtk_rand_counters(const nau_vtk_frame* f, const unsigned long long** counters) {
    *counters = f->rand_counters.data();
    return (long)f->rand_counters.size();
}

}  // extern "C"
