// capi.cu — the C-ABI of include/nauticle_gpu.h: context, SoA arena, operand
// resolution, error surfacing, and the host-side mirror of the reference's
// operator registry (kOps[], src/interactions.cpp:259-269).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "nau_internal.cuh"
#include "sweep.cuh"

using nau::FieldBuf;

namespace {

thread_local std::string g_static_err;

#define NAU_CUDA(call)                                                             \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) return fail(c, NAU_ERR_CUDA, cudaGetErrorString(e_)); \
    } while (0)

nau_status fail(nau_ctx* c, nau_status s, const std::string& msg, long bad = -1) {
    if (c) {
        c->last_error = msg;
        c->last_bad = bad;
    } else {
        g_static_err = msg;
    }
    return s;
}

// ≙ kOps[] (src/interactions.cpp:259-269) + the new dem_lsd row.
const nau_op_info kOps[] = {
    {"sph_S", NAU_OP_SPH_S, 5, 5, 3, 4, 1},
    {"sph_D00", NAU_OP_SPH_D00, 5, 5, 3, 4, 1},
    {"sph_G11", NAU_OP_SPH_G11, 5, 5, 3, 4, 1},
    {"sph_L0", NAU_OP_SPH_L0, 5, 5, 3, 4, 1},
    {"sph_A", NAU_OP_SPH_A, 5, 5, 3, 4, 1},
    {"dem_l", NAU_OP_DEM_HERTZ, 7, 7, -1, 6, 1},
    {"dem_boundary_force", NAU_OP_DEM_BOUNDARY, 7, 7, -1, 6, 1},
    {"nbody_gravity", NAU_OP_GRAVITY, 2, 3, -1, -1, 0},
    {"dem_lsd", NAU_OP_DEM_LSD, 7, 7, -1, 6, 1},
    {"sfm", NAU_OP_SFM, 10, 10, -1, -1, 1},
};

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    return cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * count);
}

template <typename T>
void dfree(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

void free_particles(nau_ctx* c) {
    for (auto& f : c->fields) {
        dfree(f.d);
        dfree(f.alt);
    }
    c->fields.clear();
    dfree(c->d_orig);
    dfree(c->d_orig_s);
    dfree(c->d_key);
    dfree(c->d_key_s);
    dfree(c->d_active);
    dfree(c->d_active_s);
    dfree(c->d_perm);
    dfree(c->d_perm_tmp);
    dfree(c->d_okey);
    dfree(c->d_xl);
    dfree(c->d_aux);
    dfree(c->d_pk);
    dfree(c->d_p4);
    dfree(c->d_skey);
    dfree(c->d_skey_s);
    dfree(c->d_upd);
    c->cap = 0;
}

nau_status ensure_field_storage(nau_ctx* c, FieldBuf& f);

}  // namespace

extern "C" void nau_release_graphs(nau_ctx* c);  // the wcsph step graphs (below)

namespace nau {

// Per-particle arrays (not fields) with capacity `cap` (>= n).
nau_status alloc_particle_arrays(nau_ctx* c, long cap) {
    c->cap = cap;
    NAU_CUDA(dalloc(&c->d_orig, cap));
    NAU_CUDA(dalloc(&c->d_orig_s, cap));
    NAU_CUDA(dalloc(&c->d_key, cap));
    NAU_CUDA(dalloc(&c->d_key_s, cap));
    NAU_CUDA(dalloc(&c->d_active, cap));
    NAU_CUDA(dalloc(&c->d_active_s, cap));
    NAU_CUDA(dalloc(&c->d_perm, cap));
    NAU_CUDA(dalloc(&c->d_perm_tmp, cap));
    NAU_CUDA(dalloc(&c->d_okey, cap));
    NAU_CUDA(dalloc(&c->d_xl, cap));
    NAU_CUDA(dalloc(&c->d_aux, cap));
    NAU_CUDA(dalloc(&c->d_p4, cap));
    NAU_CUDA(dalloc(&c->d_skey, cap));
    NAU_CUDA(dalloc(&c->d_skey_s, cap));
    NAU_CUDA(dalloc(&c->d_upd, cap));
    return NAU_OK;
}

// Grow every per-particle array and field to hold `m` particles (contents dropped).
nau_status grow_capacity(nau_ctx* c, long m) {
    if (m <= c->cap) return NAU_OK;
    cudaStreamSynchronize(c->stream);
    const long cap = std::max(m, c->cap + c->cap / 4);
    std::vector<FieldBuf> fields = c->fields;  // shapes and liveness survive
    c->fields.clear();
    free_particles(c);  // per-particle arrays
    for (auto& f : fields) {  // old field storage
        dfree(f.d);
        dfree(f.alt);
    }
    nau_status s = alloc_particle_arrays(c, cap);
    if (s != NAU_OK) return s;
    for (auto& f : fields) {
        if (f.live) {
            s = ensure_field_storage(c, f);
            if (s != NAU_OK) return s;
        }
        c->fields.push_back(f);
    }
    return NAU_OK;
}

}  // namespace nau

namespace {

void free_cells(nau_ctx* c) {
    dfree(c->d_cell_start);
    dfree(c->d_cell_count);
    dfree(c->d_cursor);
    dfree(c->d_scan_tmp);
}

__global__ void k_iota(long n, int* a) {
    long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k < n) a[k] = (int)k;
}

__global__ void k_fill(long n, int comps, const double* v, double* f) {
    long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    for (int c = 0; c < comps; ++c) f[c * n + k] = v[c];
}

struct FillVal {
    double v[9];
};

__global__ void k_fill_val(long n, int comps, FillVal v, double* f) {
    long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    for (int c = 0; c < comps; ++c) f[c * n + k] = v.v[c];
}

bool field_ok(nau_ctx* c, int id) {
    return id >= 0 && id < (int)c->fields.size() && c->fields[id].live;
}

const char* msg_text(int msg) {
    switch (msg) {
        case nau::kMsgZeroDensity: return "zero density";
        case nau::kMsgRadius: return "influence radius must be positive";
        case nau::kMsgOutsideCutoff: return "particle outside the domain on a cut-off axis";
        case nau::kMsgCoincident: return "nbody_gravity: coincident particles with zero softening";
        case nau::kMsgDemParams: return "dem contact: nonpositive Young modulus or radius";
        case nau::kMsgRandBounds: return "rand: lower bound exceeds upper bound";
        case nau::kMsgSfmTau: return "sfm: relaxation time must be positive";
        case nau::kMsgSfmMass: return "sfm: mass must be positive";
        default: return "runtime error";
    }
}

void reset_err(nau_ctx* c) {
    nau::DevErr e{};
    e.first_bad = 0x7fffffffffffffffLL;
    e.nan_first = 0x7fffffffffffffffLL;
    cudaMemcpyAsync(c->d_err, &e, sizeof(e), cudaMemcpyHostToDevice, c->stream);
    cudaStreamSynchronize(c->stream);
}

// Fetch and clear the device error word; map it to a status.
nau_status collect(nau_ctx* c) {
    if (c->s_h2d) {  // asynchronous host I/O completes here too
        cudaStreamSynchronize(c->s_h2d);
        cudaStreamSynchronize(c->s_d2h);
    }
    cudaError_t ce = cudaStreamSynchronize(c->stream);
    if (ce != cudaSuccess) return fail(c, NAU_ERR_CUDA, cudaGetErrorString(ce));
    ce = cudaGetLastError();
    if (ce != cudaSuccess) return fail(c, NAU_ERR_CUDA, cudaGetErrorString(ce));
    cudaMemcpy(c->h_err, c->d_err, sizeof(nau::DevErr), cudaMemcpyDeviceToHost);
    nau::DevErr e = *c->h_err;
    c->warnings += e.warnings;
    if (e.warnings || e.code) reset_err(c);
    if (e.code & 5) {
        std::string m = msg_text(e.msg);
        m += " at particle " + std::to_string(e.first_bad);
        return fail(c, NAU_ERR_RUNTIME, m, (long)e.first_bad);
    }
    if (e.code & 2)
        return fail(c, NAU_ERR_NAN, "non-finite value at particle " + std::to_string(e.nan_first),
                    (long)e.nan_first);
    return NAU_OK;
}

nau_status ensure_field_storage(nau_ctx* c, FieldBuf& f) {
    long len = (long)f.comps() * c->cap;
    NAU_CUDA(dalloc(&f.d, len));
    NAU_CUDA(dalloc(&f.alt, len));
    NAU_CUDA(cudaMemsetAsync(f.d, 0, sizeof(double) * (len ? len : 1), c->stream));
    return NAU_OK;
}

}  // namespace

namespace nau {

Geo make_geo(nau_ctx* c) {
    Geo g;
    g.dom = c->dom;
    double ext_max = 0.0;
    for (int a = 0; a < c->dom.dim; ++a) ext_max = std::fmax(ext_max, c->dom.ext[a]);
    g.pre_abs = (float)(8.0 * ext_max * std::ldexp(1.0, -23));
    double cs_min = c->dom.cs[0];
    for (int a = 1; a < c->dom.dim; ++a) cs_min = std::fmin(cs_min, c->dom.cs[a]);
    g.min_cs = cs_min;
    for (int a = 0; a < 3; ++a) {
        g.img[a] = AxisImg{c->dom.ext[a], 2.0 * c->dom.lo[a], 2.0 * c->dom.hi[a], c->dom.cs[a]};
        g.lim[a] = a < c->dom.dim ? (float)(c->dom.cs[a] * 1.001) + g.pre_abs : 3.0e38f;
    }
    g.n = c->n;
    g.x = c->fields[0].d;
    g.key = c->d_key;
    g.orig = c->d_orig;
    g.active = c->d_active;
    g.cell_start = c->d_cell_start;
    g.cell_count = c->d_cell_count;
    g.nact = c->d_cell_start + c->dom.ncells;
    g.p4 = c->d_p4;
    g.upd = c->ghost_field >= 0 ? c->d_upd : nullptr;
    return g;
}

Opd make_opd(nau_ctx* c, const nau_operand& o) {
    Opd d;
    d.p = o.field_id >= 0 ? c->fields[o.field_id].d : nullptr;
    for (int k = 0; k < 9; ++k) d.v[k] = o.value[k];
    return d;
}

void prof_begin(nau_ctx* c, int cls) {
    if (!c->profile) return;
    if (c->ev_next + 2 > (int)c->ev_pool.size()) {
        for (int k = 0; k < 256; ++k) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            c->ev_pool.push_back(e);
        }
    }
    c->ev_pairs.push_back({cls, c->ev_next});
    cudaEventRecord(c->ev_pool[c->ev_next], c->stream);
    c->ev_next += 2;
}

void prof_end(nau_ctx* c, int cls) {
    (void)cls;
    if (!c->profile) return;
    cudaEventRecord(c->ev_pool[c->ev_pairs.back().second + 1], c->stream);
}

}  // namespace nau

extern "C" {

nau_status nau_find_interaction(const char* name, nau_op_info* out) {
    for (const auto& op : kOps)
        if (std::strcmp(op.name, name) == 0) {
            *out = op;
            return NAU_OK;
        }
    return fail(nullptr, NAU_ERR_ARG, std::string("unknown interaction '") + name + "'");
}

// kernel.cpp:20-35 (Wendland "Wp5D220") + the new cubic spline "Wc3D220".
nau_status nau_decode_kernel(const char* kw, int* family, int* dim) {
    std::string s(kw ? kw : "");
    if (s.size() == 7 && s[0] == 'W' && s.substr(4) == "220" && (s[3] >= '1' && s[3] <= '3')) {
        if (s[1] == 'p' && s[2] == '5') {
            *family = NAU_K_WENDLAND;
            *dim = s[3] - '0';
            return NAU_OK;
        }
        if (s[1] == 'c' && s[2] == '3') {
            *family = NAU_K_CUBIC;
            *dim = s[3] - '0';
            return NAU_OK;
        }
    }
    return fail(nullptr, NAU_ERR_ARG,
                "unknown kernel keyword '" + s +
                    "'; registered keywords: Wp51220, Wp52220, Wp53220, Wc31220, Wc32220, Wc33220");
}

nau_status nau_create(int device, nau_ctx** out) {
    *out = nullptr;
    nau_ctx* c = new nau_ctx();
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = dalloc(&c->d_err, 1);
    if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&c->h_err), sizeof(nau::DevErr));
    if (e == cudaSuccess) e = dalloc(&c->d_red, 296 * 9 + 2);
    if (e != cudaSuccess) {
        g_static_err = cudaGetErrorString(e);
        delete c;
        return NAU_ERR_CUDA;
    }
    c->own_stream = true;
    reset_err(c);
    *out = c;
    return NAU_OK;
}

static void io_release(nau_ctx* c);

void nau_destroy(nau_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->s_h2d) {
        cudaStreamSynchronize(c->s_h2d);
        cudaStreamSynchronize(c->s_d2h);
    }
    if (c->stream) cudaStreamSynchronize(c->stream);
    nau_release_graphs(c);
    nau_comm_destroy(c);
    io_release(c);
    free_particles(c);
    free_cells(c);
    dfree(c->d_err);
    dfree(c->d_red);
    dfree(c->d_sel);
    dfree(c->d_nlist);
    dfree(c->d_ncount);
    dfree(c->d_nover);
    dfree(c->d_work);
    dfree(c->d_nwork);
    if (c->h_nover) cudaFreeHost(c->h_nover);
    c->h_nover = c->h_nover_dev = nullptr;
    dfree(c->d_hq);
    dfree(c->d_pstart);
    dfree(c->d_pcount);
    dfree(c->d_hesc);
    if (c->d_vm) cudaFree(c->d_vm);
    c->d_vm = nullptr;
    dfree(c->d_rng);
    if (c->h_err) cudaFreeHost(c->h_err);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

nau_status nau_set_stream(nau_ctx* c, void* stream) {
    cudaStreamSynchronize(c->stream);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    if (stream) {
        c->stream = static_cast<cudaStream_t>(stream);
        c->own_stream = false;
    } else {
        NAU_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    return NAU_OK;
}

void* nau_get_stream(nau_ctx* c) { return c->stream; }

nau_status nau_set_domain(nau_ctx* c, int dim, const int* min_cells, const int* max_cells,
                          const double* cell_size, const int* kind) {
    if (dim < 1 || dim > 3) return fail(c, NAU_ERR_ARG, "domain dimension must be 1, 2 or 3");
    nau::DomainDev d{};
    d.dim = dim;
    long total = 1;
    for (int a = 0; a < 3; ++a) {
        int mn = 0, mx = 1, k = NAU_CUTOFF;
        double cs = 1.0;
        if (a < dim) {
            mn = min_cells[a];
            mx = max_cells[a];
            cs = cell_size[a];
            k = kind[a];
            if (mx <= mn)
                return fail(c, NAU_ERR_ARG, "domain axis " + std::to_string(a) +
                                                ": maximum cell count must exceed minimum");
            if (!(cs > 0.0))
                return fail(c, NAU_ERR_ARG,
                            "domain axis " + std::to_string(a) + ": cell size must be positive");
            if (k < 0 || k > 2) return fail(c, NAU_ERR_ARG, "unknown boundary kind");
        }
        d.cells[a] = mx - mn;
        c->min_cells[a] = mn;
        c->max_cells[a] = mx;
        d.cs[a] = cs;
        d.lo[a] = mn * cs;  // domain.hpp:28-30: products, not sums
        d.hi[a] = mx * cs;
        d.ext[a] = d.hi[a] - d.lo[a];
        d.kind[a] = k;
        if (a < dim) total *= d.cells[a];
    }
    if (total >= 0x7ffffff0L) return fail(c, NAU_ERR_ARG, "too many cells for int32 keys");
    d.ncells = (int)total;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    free_cells(c);
    NAU_CUDA(dalloc(&c->d_cell_start, total + 2));
    NAU_CUDA(dalloc(&c->d_cell_count, total + 1));
    NAU_CUDA(dalloc(&c->d_cursor, total + 1));
    c->scan_tmp_len = (total + 1 + 4095) / 4096 + 1;
    NAU_CUDA(dalloc(&c->d_scan_tmp, c->scan_tmp_len));
    NAU_CUDA(cudaMemsetAsync(c->d_cell_start, 0, sizeof(int) * (total + 2), c->stream));
    NAU_CUDA(cudaMemsetAsync(c->d_cell_count, 0, sizeof(int) * (total + 1), c->stream));
    c->dom = d;
    c->has_domain = true;
    c->dirty = true;
    return NAU_OK;
}

nau_status nau_set_particles(nau_ctx* c, long n, const double* pos_soa) {
    if (!c->has_domain) return fail(c, NAU_ERR_ARG, "nau_set_domain must precede nau_set_particles");
    if (n < 0 || n >= (1L << 25))  // sweep.cuh packs slot indices in 25 bits
        return fail(c, NAU_ERR_ARG,
                    "particle count must be below 2^25 per context (shard larger systems across GPUs)");
    cudaSetDevice(c->device);
    if (c->s_h2d) {
        cudaStreamSynchronize(c->s_h2d);
        cudaStreamSynchronize(c->s_d2h);
    }
    cudaStreamSynchronize(c->stream);
    free_particles(c);
    dfree(c->d_rng);  // a new particle set starts a fresh RandomState
    c->rng_len = 0;
    c->n = n;
    nau_status sa = nau::alloc_particle_arrays(c, n);
    if (sa != NAU_OK) return sa;
    if (n > 0) {
        k_iota<<<(int)((n + 255) / 256), 256, 0, c->stream>>>(n, c->d_orig);
        k_iota<<<(int)((n + 255) / 256), 256, 0, c->stream>>>(n, c->d_skey);
        c->launches += 2;
    }
    NAU_CUDA(cudaMemsetAsync(c->d_active, 1, n ? n : 1, c->stream));
    FieldBuf r;
    r.rows = c->dom.dim;
    r.cols = 1;
    r.live = true;
    nau_status s = ensure_field_storage(c, r);
    if (s != NAU_OK) return s;
    c->fields.push_back(r);
    if (n > 0 && pos_soa)
        NAU_CUDA(cudaMemcpyAsync(c->fields[0].d, pos_soa, sizeof(double) * n * c->dom.dim,
                                 cudaMemcpyHostToDevice, c->stream));
    c->dirty = true;
    c->built_once = false;
    c->rebuild_count = 0;
    c->nl_rev = -1;  // neighbour-list and fp16 caches belong to the old particle set
    c->hq_rev = -1;
    c->xl_rev = -1;
    c->warnings = 0;
    return collect(c);
}

long nau_particle_count(nau_ctx* c) { return c->n; }

nau_status nau_get_active(nau_ctx* c, uint8_t* active) {
    std::vector<uint8_t> a(c->n);
    std::vector<int> o(c->n);
    if (c->n) {
        NAU_CUDA(cudaMemcpyAsync(a.data(), c->d_active, c->n, cudaMemcpyDeviceToHost, c->stream));
        NAU_CUDA(cudaMemcpyAsync(o.data(), c->d_orig, sizeof(int) * c->n, cudaMemcpyDeviceToHost,
                                 c->stream));
    }
    NAU_CUDA(cudaStreamSynchronize(c->stream));
    for (long k = 0; k < c->n; ++k) active[o[k]] = a[k];
    return NAU_OK;
}

long nau_active_count(nau_ctx* c) {
    std::vector<uint8_t> a(c->n);
    if (c->n) cudaMemcpyAsync(a.data(), c->d_active, c->n, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    long s = 0;
    for (auto v : a) s += v;
    return s;
}

nau_status nau_alloc_field(nau_ctx* c, int rows, int cols, int* field_id) {
    if (rows < 1 || rows > 3 || cols < 1 || cols > 3)
        return fail(c, NAU_ERR_ARG, "tensor extent outside the supported 1..3 range");
    if (c->fields.empty()) return fail(c, NAU_ERR_ARG, "nau_set_particles must precede fields");
    FieldBuf f;
    f.rows = rows;
    f.cols = cols;
    f.live = true;
    cudaSetDevice(c->device);
    nau_status s = ensure_field_storage(c, f);
    if (s != NAU_OK) return s;
    for (size_t k = 1; k < c->fields.size(); ++k)
        if (!c->fields[k].live) {
            c->fields[k] = f;
            *field_id = (int)k;
            return NAU_OK;
        }
    if ((int)c->fields.size() >= nau::kMaxFields) return fail(c, NAU_ERR_ARG, "too many fields");
    c->fields.push_back(f);
    *field_id = (int)c->fields.size() - 1;
    return NAU_OK;
}

nau_status nau_field_shape(nau_ctx* c, int id, int* rows, int* cols) {
    if (!field_ok(c, id)) return fail(c, NAU_ERR_ARG, "bad field id");
    *rows = c->fields[id].rows;
    *cols = c->fields[id].cols;
    return NAU_OK;
}

nau_status nau_free_field(nau_ctx* c, int id) {
    if (id <= 0 || !field_ok(c, id)) return fail(c, NAU_ERR_ARG, "bad field id");
    cudaStreamSynchronize(c->stream);
    dfree(c->fields[id].d);
    dfree(c->fields[id].alt);
    c->fields[id].live = false;
    return NAU_OK;
}

nau_status nau_upload(nau_ctx* c, int id, const double* soa, long n) {
    if (!field_ok(c, id) || n != c->n) return fail(c, NAU_ERR_ARG, "bad field id or count");
    FieldBuf& f = c->fields[id];
    if (n == 0) return NAU_OK;
    NAU_CUDA(cudaMemcpyAsync(f.alt, soa, sizeof(double) * n * f.comps(), cudaMemcpyHostToDevice,
                             c->stream));
    nau::launch_sort_in(c, f.alt, f.d, f.comps());
    if (id == 0) c->dirty = true;
    return NAU_OK;
}

nau_status nau_download(nau_ctx* c, int id, double* soa, long n) {
    if (!field_ok(c, id) || n != c->n) return fail(c, NAU_ERR_ARG, "bad field id or count");
    FieldBuf& f = c->fields[id];
    if (n == 0) return NAU_OK;
    nau::launch_unsort(c, f.d, f.alt, f.comps());
    NAU_CUDA(cudaMemcpyAsync(soa, f.alt, sizeof(double) * n * f.comps(), cudaMemcpyDeviceToHost,
                             c->stream));
    return collect(c);
}

// ---- asynchronous host I/O -----------------------------------------------------
// Uploads: H2D into staging buffer b on s_h2d, then the context stream scatters it
// into cell order (k_sort_in). Downloads: the context stream gathers into staging
// buffer b (k_unsort), then D2H on s_d2h. Two buffers per field and direction, each
// guarded by events, so step k's copies overlap step k+-1's passes.
static nau_status io_prepare(nau_ctx* c, std::vector<nau_ctx::IoStage>& v, int id, size_t len) {
    if (!c->s_h2d) {
        NAU_CUDA(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
        NAU_CUDA(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    }
    if ((int)v.size() <= id) v.resize(id + 1);
    nau_ctx::IoStage& st = v[id];
    if (st.len < len) {
        cudaStreamSynchronize(c->s_h2d);
        cudaStreamSynchronize(c->s_d2h);
        cudaStreamSynchronize(c->stream);
        for (int b = 0; b < 2; ++b) {
            dfree(st.buf[b]);
            NAU_CUDA(dalloc(&st.buf[b], len));
            if (!st.ready[b]) NAU_CUDA(cudaEventCreateWithFlags(&st.ready[b], cudaEventDisableTiming));
            if (!st.consumed[b])
                NAU_CUDA(cudaEventCreateWithFlags(&st.consumed[b], cudaEventDisableTiming));
        }
        st.len = len;
    }
    return NAU_OK;
}

static void io_release(nau_ctx* c) {
    for (auto* v : {&c->io_up, &c->io_down})
        for (auto& st : *v)
            for (int b = 0; b < 2; ++b) {
                dfree(st.buf[b]);
                if (st.ready[b]) cudaEventDestroy(st.ready[b]);
                if (st.consumed[b]) cudaEventDestroy(st.consumed[b]);
            }
    c->io_up.clear();
    c->io_down.clear();
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    c->s_h2d = c->s_d2h = nullptr;
}

nau_status nau_upload_async(nau_ctx* c, int id, const double* soa, long n) {
    if (!field_ok(c, id) || n != c->n) return fail(c, NAU_ERR_ARG, "bad field id or count");
    if (n == 0) return NAU_OK;
    FieldBuf& f = c->fields[id];
    const size_t len = (size_t)n * f.comps();
    nau_status s = io_prepare(c, c->io_up, id, len);
    if (s != NAU_OK) return s;
    nau_ctx::IoStage& st = c->io_up[id];
    const int b = st.next;
    st.next ^= 1;
    NAU_CUDA(cudaStreamWaitEvent(c->s_h2d, st.consumed[b], 0));  // previous scatter read it
    NAU_CUDA(cudaMemcpyAsync(st.buf[b], soa, sizeof(double) * len, cudaMemcpyHostToDevice, c->s_h2d));
    NAU_CUDA(cudaEventRecord(st.ready[b], c->s_h2d));
    NAU_CUDA(cudaStreamWaitEvent(c->stream, st.ready[b], 0));
    nau::launch_sort_in(c, st.buf[b], f.d, f.comps());
    NAU_CUDA(cudaEventRecord(st.consumed[b], c->stream));
    if (id == 0) c->dirty = true;
    return NAU_OK;
}

nau_status nau_download_async(nau_ctx* c, int id, double* soa, long n) {
    if (!field_ok(c, id) || n != c->n) return fail(c, NAU_ERR_ARG, "bad field id or count");
    if (n == 0) return NAU_OK;
    FieldBuf& f = c->fields[id];
    const size_t len = (size_t)n * f.comps();
    nau_status s = io_prepare(c, c->io_down, id, len);
    if (s != NAU_OK) return s;
    nau_ctx::IoStage& st = c->io_down[id];
    const int b = st.next;
    st.next ^= 1;
    NAU_CUDA(cudaStreamWaitEvent(c->stream, st.consumed[b], 0));  // previous D2H read it
    nau::launch_unsort(c, f.d, st.buf[b], f.comps());
    NAU_CUDA(cudaEventRecord(st.ready[b], c->stream));
    NAU_CUDA(cudaStreamWaitEvent(c->s_d2h, st.ready[b], 0));
    NAU_CUDA(cudaMemcpyAsync(soa, st.buf[b], sizeof(double) * len, cudaMemcpyDeviceToHost, c->s_d2h));
    NAU_CUDA(cudaEventRecord(st.consumed[b], c->s_d2h));
    return NAU_OK;
}

nau_status nau_io_fence(nau_ctx* c) {
    if (!c->s_h2d) {
        NAU_CUDA(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
        NAU_CUDA(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    }
    cudaEvent_t e;
    NAU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEventRecord(e, c->stream);
    cudaStreamWaitEvent(c->s_h2d, e, 0);
    cudaStreamWaitEvent(c->s_d2h, e, 0);
    cudaEventDestroy(e);  // released once the waits are satisfied
    return NAU_OK;
}

nau_status nau_io_join(nau_ctx* c) {
    if (!c->s_h2d) return NAU_OK;
    for (cudaStream_t s : {c->s_h2d, c->s_d2h}) {
        cudaEvent_t e;
        NAU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        cudaEventRecord(e, s);
        cudaStreamWaitEvent(c->stream, e, 0);
        cudaEventDestroy(e);
    }
    return NAU_OK;
}

nau_status nau_fill(nau_ctx* c, int id, const double* value) {
    if (!field_ok(c, id)) return fail(c, NAU_ERR_ARG, "bad field id");
    FieldBuf& f = c->fields[id];
    FillVal v{};
    for (int k = 0; k < f.comps(); ++k) v.v[k] = value[k];
    if (c->n)
        k_fill_val<<<(int)((c->n + 255) / 256), 256, 0, c->stream>>>(c->n, f.comps(), v, f.d);
    c->launches++;
    if (id == 0) c->dirty = true;
    return NAU_OK;
}

nau_status nau_copy_field(nau_ctx* c, int dst, int src) {
    if (!field_ok(c, dst) || !field_ok(c, src) ||
        c->fields[dst].comps() != c->fields[src].comps())
        return fail(c, NAU_ERR_ARG, "bad field ids for copy");
    NAU_CUDA(cudaMemcpyAsync(c->fields[dst].d, c->fields[src].d,
                             sizeof(double) * c->n * c->fields[src].comps(),
                             cudaMemcpyDeviceToDevice, c->stream));
    if (dst == 0) c->dirty = true;
    return NAU_OK;
}

nau_status nau_field_device_ptr(nau_ctx* c, int id, double** ptr) {
    if (!field_ok(c, id)) return fail(c, NAU_ERR_ARG, "bad field id");
    *ptr = c->fields[id].d;
    return NAU_OK;
}

nau_status nau_boundary_shift(nau_ctx* c) {
    if (c->fields.empty()) return fail(c, NAU_ERR_ARG, "no particles");
    nau::launch_boundary_shift(c);
    c->dirty = true;  // case.cpp:59-62 marks dirty after the shift
    return NAU_OK;
}

nau_status nau_build_cells(nau_ctx* c) {
    if (c->fields.empty()) return fail(c, NAU_ERR_ARG, "no particles");
    nau::prof_begin(c, 300);
    nau::launch_build_cells(c);
    nau::prof_end(c, 300);
    c->dirty = false;
    c->built_once = true;
    ++c->rebuild_count;
    return NAU_OK;
}

int nau_cells_dirty(nau_ctx* c) { return c->dirty ? 1 : 0; }
long nau_rebuild_count(nau_ctx* c) { return c->rebuild_count; }
long nau_ncells(nau_ctx* c) { return c->dom.ncells; }

long nau_warning_count(nau_ctx* c) {
    collect(c);
    return (long)c->warnings;
}

nau_status nau_cell_tables(nau_ctx* c, int* cell_of, int* cell_start, int* cell_count,
                           int* sorted_ids) {
    if (c->dirty || !c->built_once) {
        nau_status s = nau_build_cells(c);
        if (s != NAU_OK) return s;
    }
    const long n = c->n;
    const int nc = c->dom.ncells;
    std::vector<int> key(n), orig(n);
    if (n) {
        NAU_CUDA(cudaMemcpyAsync(key.data(), c->d_key, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
        NAU_CUDA(cudaMemcpyAsync(orig.data(), c->d_orig, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    }
    NAU_CUDA(cudaMemcpyAsync(cell_start, c->d_cell_start, sizeof(int) * nc, cudaMemcpyDeviceToHost, c->stream));
    NAU_CUDA(cudaMemcpyAsync(cell_count, c->d_cell_count, sizeof(int) * nc, cudaMemcpyDeviceToHost, c->stream));
    nau_status s = collect(c);
    if (s != NAU_OK) return s;
    long nact = 0;
    for (long k = 0; k < n; ++k) {
        cell_of[orig[k]] = key[k] < nc ? key[k] : -1;
        if (key[k] < nc) sorted_ids[nact++] = orig[k];
    }
    return NAU_OK;
}

nau_status nau_neighbor_counts(nau_ctx* c, double radius, int* counts) {
    if (c->dirty || !c->built_once) {
        nau_status s = nau_build_cells(c);
        if (s != NAU_OK) return s;
    }
    int* d = nullptr;
    NAU_CUDA(dalloc(&d, c->n));
    nau::launch_neighbor_counts(c, radius, d);
    if (c->n) cudaMemcpyAsync(counts, d, sizeof(int) * c->n, cudaMemcpyDeviceToHost, c->stream);
    nau_status s = collect(c);
    cudaFree(d);
    return s;
}

nau_status nau_interact(nau_ctx* c, int op, int kf, int kdim, const nau_operand* ops, int nops,
                        int out_field) {
    if (op < 0 || op >= NAU_OP_COUNT) return fail(c, NAU_ERR_ARG, "unknown operator");
    const nau_op_info& info = kOps[op];
    const int arity = nops + (info.kernel_slot >= 0 ? 1 : 0);
    if (arity < info.arity_min || arity > info.arity_max)
        return fail(c, NAU_ERR_ARG, std::string("wrong number of operands for '") + info.name + "'");
    if (!field_ok(c, out_field) || out_field == 0)
        return fail(c, NAU_ERR_ARG, "bad output field (r is written by euler only)");
    const int dim = c->dom.dim;
    nau::Opd d_ops[10];
    for (int k = 0; k < nops; ++k) {
        if (ops[k].field_id >= 0 && !field_ok(c, ops[k].field_id))
            return fail(c, NAU_ERR_ARG, "bad operand field id");
        d_ops[k] = nau::make_opd(c, ops[k]);
    }
    auto shape = [&](int k, int& r, int& cc) {
        if (ops[k].field_id >= 0) {
            r = c->fields[ops[k].field_id].rows;
            cc = c->fields[ops[k].field_id].cols;
        } else {
            r = ops[k].rows;
            cc = ops[k].cols;
        }
    };
    int ar = 1, acl = 1;
    shape(0, ar, acl);
    int out_rows = 1, out_cols = 1;
    auto shape_str = [](int r, int cc) { return std::to_string(r) + "x" + std::to_string(cc); };
    if (op == NAU_OP_SFM) {
        // eval_social_force (interactions.cpp:216-257): r_d - x_i and (...) - v_i are
        // d-vector differences, every other operand goes through .value()
        out_rows = dim;
        int r = 1, cc = 1;
        for (int k : {1, 3, 4, 5, 6, 7, 8, 9}) {  // the scalar_operand calls, in order
            shape(k, r, cc);
            if (!(r == 1 && cc == 1))
                return fail(c, NAU_ERR_RUNTIME,
                            "expected a scalar, got a " + shape_str(r, cc) + " tensor");
        }
        shape(2, r, cc);
        if (!(r == dim && cc == 1))
            return fail(c, NAU_ERR_RUNTIME, "operator '-': incompatible shapes " +
                                                shape_str(r, cc) + " and " + shape_str(dim, 1));
        if (!(ar == dim && acl == 1))
            return fail(c, NAU_ERR_RUNTIME, "operator '-': incompatible shapes " +
                                                shape_str(dim, 1) + " and " + shape_str(ar, acl));
    } else if (op == NAU_OP_SPH_S) {
        out_rows = ar;
        out_cols = acl;
    } else if (op == NAU_OP_SPH_D00 || op == NAU_OP_SPH_L0) {
        if (op == NAU_OP_SPH_D00 && !(acl == 1 && ar == dim))
            return fail(c, NAU_ERR_RUNTIME, "sph_D00: operand must be a vector field");
        if (op == NAU_OP_SPH_L0 && !(ar == 1 && acl == 1))
            return fail(c, NAU_ERR_RUNTIME, "sph_L0: expected a scalar operand");
    } else {
        out_rows = dim;
        if ((op == NAU_OP_SPH_G11) && !(ar == 1 && acl == 1))
            return fail(c, NAU_ERR_RUNTIME, "sph_G11: expected a scalar operand");
        if ((op == NAU_OP_SPH_A || op >= NAU_OP_DEM_HERTZ) && op != NAU_OP_GRAVITY &&
            !(acl == 1 && ar == dim))
            return fail(c, NAU_ERR_RUNTIME, "velocity operand must be a d-vector");
    }
    FieldBuf& of = c->fields[out_field];
    if (of.rows != out_rows || of.cols != out_cols)
        return fail(c, NAU_ERR_RUNTIME, "LHS field shape does not match the operator result");
    if (info.finite_influence && (c->dirty || !c->built_once)) {
        nau_status s = nau_build_cells(c);  // case.cpp:11
        if (s != NAU_OK) return s;
        for (int k = 0; k < nops; ++k) d_ops[k] = nau::make_opd(c, ops[k]);
    }
    // Two-phase write (case.cpp:31-54): if the output aliases an operand,
    // evaluate into the twin buffer (pre-filled so inactive values persist).
    bool alias = false;
    for (int k = 0; k < nops; ++k) alias |= ops[k].field_id == out_field;
    double* out = of.d;
    if (alias) {
        NAU_CUDA(cudaMemcpyAsync(of.alt, of.d, sizeof(double) * c->n * of.comps(),
                                 cudaMemcpyDeviceToDevice, c->stream));
        out = of.alt;
    }
    const bool fast = c->mode == NAU_MODE_FAST && nau::fast_supports(op, ar, acl, dim);
    // SPH operators with a uniform radius share the cell build's neighbour list
    // (several operators per step walk the same candidates; same order either way)
    bool lists = false;
    if (op <= NAU_OP_SPH_A && ops[3].field_id < 0 && ops[3].value[0] > 0.0)
        lists = nau::nlist_for(c, ops[3].value[0], !fast);
    if (fast)
        nau::launch_interact_fast(c, op, kf, kdim, d_ops, out, ar, lists);
    else
        nau::launch_interact(c, op, kf, kdim, d_ops, nops, out, out_rows, out_cols, ar, acl,
                             nullptr, nullptr, lists);
    if (alias) std::swap(of.d, of.alt);
    return NAU_OK;
}

nau_status nau_interact_g11_l0(nau_ctx* c, int kf, int kdim, const nau_operand* ops, int nops,
                               int out_g, int out_l) {
    // Fused only where it is observably the same as the two calls in sequence: FAST
    // mode, valid shapes, and neither output aliasing an operand or the other output
    // (sph_L0 then reads exactly what sph_G11 read). Otherwise: the two calls, which
    // also produce the reference's error messages.
    const int dim = c->dom.dim;
    bool fuse = c->mode == NAU_MODE_FAST && nops == 4 && ops != nullptr && out_g != out_l &&
                field_ok(c, out_g) && field_ok(c, out_l) && out_g != 0 && out_l != 0;
    for (int k = 0; fuse && k < nops; ++k) {
        const int f = ops[k].field_id;
        fuse = f != out_g && f != out_l && (f < 0 || field_ok(c, f));
    }
    if (fuse) {
        const int f = ops[0].field_id;
        const int ar = f >= 0 ? c->fields[f].rows : ops[0].rows;
        const int acl = f >= 0 ? c->fields[f].cols : ops[0].cols;
        fuse = ar == 1 && acl == 1 && c->fields[out_g].rows == dim && c->fields[out_g].cols == 1 &&
               c->fields[out_l].rows == 1 && c->fields[out_l].cols == 1;
    }
    if (!fuse) {
        nau_status s = nau_interact(c, NAU_OP_SPH_G11, kf, kdim, ops, nops, out_g);
        if (s != NAU_OK) return s;
        return nau_interact(c, NAU_OP_SPH_L0, kf, kdim, ops, nops, out_l);
    }
    if (c->dirty || !c->built_once) {
        nau_status s = nau_build_cells(c);  // case.cpp:11
        if (s != NAU_OK) return s;
    }
    nau::Opd d_ops[4];
    for (int k = 0; k < 4; ++k) d_ops[k] = nau::make_opd(c, ops[k]);
    bool lists = false;
    if (ops[3].field_id < 0 && ops[3].value[0] > 0.0)
        lists = nau::nlist_for(c, ops[3].value[0], false);
    // sph_L0 goes to the twin buffer and is committed only if nothing failed: after a
    // sph_G11 error (or its NaN audit) the reference never evaluates the sph_L0 equation,
    // and after an sph_L0 NaN its staging is discarded (case.cpp:46-57) — L keeps its values.
    FieldBuf& fl = c->fields[out_l];
    nau::launch_g11_l0_fast(c, kf, kdim, d_ops, c->fields[out_g].d, fl.alt, lists);
    nau::launch_commit_if_ok(c, fl.alt, fl.d);
    return NAU_OK;
}

nau_status nau_euler(nau_ctx* c, int x, int xdot, double dt, int out_field) {
    if (!field_ok(c, x) || !field_ok(c, xdot) || !field_ok(c, out_field))
        return fail(c, NAU_ERR_ARG, "bad field id");
    FieldBuf& fx = c->fields[x];
    if (fx.comps() != c->fields[xdot].comps() || fx.comps() != c->fields[out_field].comps())
        return fail(c, NAU_ERR_RUNTIME, "euler: state and derivative shapes differ");
    FieldBuf& fo = c->fields[out_field];
    const bool alias = out_field == x || out_field == xdot;
    double* out = alias ? fo.alt : fo.d;
    nau::launch_euler(c, fx.d, c->fields[xdot].d, dt, out, fx.comps());
    if (alias) std::swap(fo.d, fo.alt);
    if (out_field == 0) {  // case.cpp:59-62
        nau::launch_boundary_shift(c);
        c->dirty = true;
    }
    return NAU_OK;
}

nau_status nau_symplectic_step(nau_ctx* c, int v, int vdot, int mask, double dt) {
    if (!field_ok(c, v) || !field_ok(c, vdot) || (mask >= 0 && !field_ok(c, mask)))
        return fail(c, NAU_ERR_ARG, "bad field id");
    nau::launch_symplectic(c, c->fields[v].d, c->fields[vdot].d,
                           mask >= 0 ? c->fields[mask].d : nullptr, dt);
    c->dirty = true;
    return NAU_OK;
}

// The deck's three passes (nau_wcsph_pass); nau_wcsph_step runs them in order.
nau_status nau_wcsph_pass(nau_ctx* c, const nau_wcsph_params* p, int pass) {
    int ids[5] = {p->f_rho, p->f_p, p->f_v, p->f_vdot, p->f_mask};
    for (int k = 0; k < 5; ++k)
        if (!(k == 4 && ids[k] < 0) && !field_ok(c, ids[k])) return fail(c, NAU_ERR_ARG, "bad field id");
    if (!(p->radius > 0.0)) return fail(c, NAU_ERR_RUNTIME, "influence radius must be positive");
    if (pass < 0 || pass > 2) return fail(c, NAU_ERR_ARG, "nau_wcsph_pass: pass is 0, 1 or 2");
    if (pass == 2) {  // v = euler(v, vdot*mask, dt); r = euler(r, v, dt); boundary shift
        nau::launch_symplectic(c, c->fields[p->f_v].d, c->fields[p->f_vdot].d,
                               p->f_mask >= 0 ? c->fields[p->f_mask].d : nullptr, p->dt);
        c->dirty = true;
        c->wcsph_rev = -1;
        return NAU_OK;
    }
    if (pass == 1) {  // the momentum pass reads what the density pass of this build wrote
        if (c->wcsph_rev != c->rebuild_count || c->dirty)
            return fail(c, NAU_ERR_ARG, "nau_wcsph_pass: the momentum pass needs the density pass first");
        if (c->mode == NAU_MODE_FAST)
            nau::launch_wcsph_fast(c, p, c->d_aux, c->wcsph_lists, 2);
        else
            nau::launch_wcsph(c, p, c->wcsph_lists != 0, 2);
        return NAU_OK;
    }
    if (c->dirty || !c->built_once) {
        // rho, p (density pass) and vdot (momentum pass) are written for every active
        // particle before anything reads them: the build moves their inactive slots only
        c->reorder_skip = (1ULL << p->f_rho) | (1ULL << p->f_p) | (1ULL << p->f_vdot);
        nau_status s = nau_build_cells(c);
        if (s != NAU_OK) return s;
    }
    // Both passes of the step share one neighbour list (same candidates, same order).
    // FAST + Wendland + radius within a cell (no per-axis test): paired lists
    double min_cs = c->dom.cs[0];
    for (int a = 1; a < c->dom.dim; ++a) min_cs = std::min(min_cs, c->dom.cs[a]);
    const bool pairs = c->mode == NAU_MODE_FAST && p->kernel_family == NAU_K_WENDLAND &&
                       p->radius <= min_cs;
    // no host synchronisation: an overflowing list is swept by the fallback pass
#ifndef NAU_ASYNC_LISTS
#define NAU_ASYNC_LISTS 1
#endif
    const int lists = nau::nlist_for(c, p->radius, c->mode == NAU_MODE_EXACT, pairs, NAU_ASYNC_LISTS);
    {
        int img = 0;
        for (int a = 0; a < c->dom.dim; ++a) img |= c->dom.kind[a] != NAU_CUTOFF;
        c->last_wcsph_path = (c->mode == NAU_MODE_FAST ? NAU_PATH_FAST : 0) | (lists << 2) |
                             (img ? NAU_PATH_IMAGES : 0);
    }
    if (c->mode == NAU_MODE_FAST)
        nau::launch_wcsph_fast(c, p, c->d_aux, lists, 1);
    else
        nau::launch_wcsph(c, p, lists != 0, 1);
    c->wcsph_lists = lists;
    c->wcsph_rev = c->rebuild_count;
    return NAU_OK;
}

// ---- CUDA graphs of the WCSPH step ----
// One nau_wcsph_step is ~15 launches and memsets with no host synchronisation (async
// neighbour lists). After two warm-up calls a step is captured into a graph together
// with the host state it started from (every buffer pointer the launches use, the
// pointer swaps of the cell build, cache keys relative to the rebuild counter, flags,
// the parameters) and the state it left. A later call that starts from the same state
// replays the graph and applies the recorded successor state on the host. Steps
// alternate between two buffer parities, so two graphs cover a run. Profiling, a
// capacity change or any mismatch runs the plain path (and may capture anew).
struct HostState {
    std::vector<uintptr_t> ptr;  // buffers / sizes that must match for a replay
    long n = 0, nl_rel = 0, hq_rel = 0, xl_rel = 0, wcsph_rel = 0;
    bool dirty = false, built_once = false, xl_used = false, hq_used = false, nl_async = false;
    unsigned long long reorder_skip = 0;
    double nl_radius = 0.0;
    bool nl_ordered = false, nl_pairs = false;
    int nl_cap = 0, wcsph_lists = 0, last_path = 0, mode = 0, ghost_field = -1;
    nau_wcsph_params prm{};
    std::vector<double*> fd, fa;  // field storage after the step (swapped by the build)
    int* orig = nullptr; int* orig_s = nullptr; int* skey = nullptr; int* skey_s = nullptr;
    int* key = nullptr; int* key_s = nullptr; uint8_t* act = nullptr; uint8_t* act_s = nullptr;
};

struct nau_ctx::StepGraph {
    cudaGraphExec_t exec = nullptr;
    HostState before, after;
    long d_rebuild = 0, kernels = 0;
};

static HostState capture_state(nau_ctx* c, const nau_wcsph_params* p) {
    HostState h;
    auto add = [&](const void* q) { h.ptr.push_back(reinterpret_cast<uintptr_t>(q)); };
    add(c->d_orig); add(c->d_orig_s); add(c->d_skey); add(c->d_skey_s); add(c->d_key);
    add(c->d_key_s); add(c->d_active); add(c->d_active_s); add(c->d_nlist); add(c->d_hq);
    add(c->d_pstart); add(c->d_work); add(c->d_xl); add(c->d_p4); add(c->d_aux); add(c->d_upd);
    add(reinterpret_cast<void*>(c->nl_len)); add(reinterpret_cast<void*>(c->hq_len));
    add(reinterpret_cast<void*>(c->pstart_len)); add(reinterpret_cast<void*>(c->cap));
    add(c->d_cell_start); add(c->d_cell_count); add(c->d_cursor); add(c->d_scan_tmp);
    add(c->d_perm); add(c->d_perm_tmp); add(c->d_okey); add(c->d_hesc); add(c->d_nover);
    add(c->d_ncount); add(c->d_nwork); add(c->d_pcount); add(c->d_err); add(c->h_nover_dev);
    add(reinterpret_cast<void*>((uintptr_t)c->dom.ncells));
    add(reinterpret_cast<void*>((uintptr_t)(c->use_nlist * 2 + c->use_pairs)));
    add(reinterpret_cast<void*>((uintptr_t)c->dom.dim));
    for (int a = 0; a < 3; ++a) {
        uint64_t bits;
        std::memcpy(&bits, &c->dom.cs[a], 8);
        add(reinterpret_cast<void*>(bits));
        std::memcpy(&bits, &c->dom.lo[a], 8);
        add(reinterpret_cast<void*>(bits));
        add(reinterpret_cast<void*>((uintptr_t)(c->dom.cells[a] * 4 + c->dom.kind[a])));
    }
    for (auto& f : c->fields) {
        add(f.d); add(f.alt); add(reinterpret_cast<void*>((uintptr_t)f.live));
        h.fd.push_back(f.d);
        h.fa.push_back(f.alt);
    }
    h.n = c->n;
    h.nl_rel = c->nl_rev - c->rebuild_count;
    h.hq_rel = c->hq_rev - c->rebuild_count;
    h.xl_rel = c->xl_rev - c->rebuild_count;
    h.wcsph_rel = c->wcsph_rev - c->rebuild_count;
    h.dirty = c->dirty; h.built_once = c->built_once; h.xl_used = c->xl_used;
    h.hq_used = c->hq_used; h.nl_async = c->nl_async; h.reorder_skip = c->reorder_skip;
    h.nl_radius = c->nl_radius; h.nl_ordered = c->nl_ordered; h.nl_pairs = c->nl_pairs;
    h.nl_cap = c->nl_cap; h.wcsph_lists = c->wcsph_lists; h.last_path = c->last_wcsph_path;
    h.mode = c->mode; h.ghost_field = c->ghost_field;
    h.prm = *p;
    h.orig = c->d_orig; h.orig_s = c->d_orig_s; h.skey = c->d_skey; h.skey_s = c->d_skey_s;
    h.key = c->d_key; h.key_s = c->d_key_s; h.act = c->d_active; h.act_s = c->d_active_s;
    return h;
}

static bool same_state(const HostState& a, const HostState& b) {
    return a.ptr == b.ptr && a.n == b.n && a.nl_rel == b.nl_rel && a.hq_rel == b.hq_rel &&
           a.xl_rel == b.xl_rel && a.wcsph_rel == b.wcsph_rel && a.dirty == b.dirty &&
           a.built_once == b.built_once && a.xl_used == b.xl_used && a.hq_used == b.hq_used &&
           a.nl_async == b.nl_async && a.reorder_skip == b.reorder_skip &&
           a.nl_radius == b.nl_radius && a.nl_ordered == b.nl_ordered &&
           a.nl_pairs == b.nl_pairs && a.nl_cap == b.nl_cap && a.wcsph_lists == b.wcsph_lists &&
           a.last_path == b.last_path && a.mode == b.mode && a.ghost_field == b.ghost_field &&
           std::memcmp(&a.prm, &b.prm, sizeof(a.prm)) == 0;
}

// The host side of a step: pointers and flags as `h`, counters advanced by d_rebuild.
static void apply_state(nau_ctx* c, const HostState& h, long d_rebuild) {
    c->rebuild_count += d_rebuild;
    for (size_t f = 0; f < c->fields.size() && f < h.fd.size(); ++f) {
        c->fields[f].d = h.fd[f];
        c->fields[f].alt = h.fa[f];
    }
    c->d_orig = h.orig; c->d_orig_s = h.orig_s; c->d_skey = h.skey; c->d_skey_s = h.skey_s;
    c->d_key = h.key; c->d_key_s = h.key_s; c->d_active = h.act; c->d_active_s = h.act_s;
    c->nl_rev = c->rebuild_count + h.nl_rel;
    c->hq_rev = c->rebuild_count + h.hq_rel;
    c->xl_rev = c->rebuild_count + h.xl_rel;
    c->wcsph_rev = c->rebuild_count + h.wcsph_rel;
    c->dirty = h.dirty; c->built_once = h.built_once; c->xl_used = h.xl_used;
    c->hq_used = h.hq_used; c->nl_async = h.nl_async; c->reorder_skip = h.reorder_skip;
    c->nl_radius = h.nl_radius; c->nl_ordered = h.nl_ordered; c->nl_pairs = h.nl_pairs;
    c->nl_cap = h.nl_cap; c->wcsph_lists = h.wcsph_lists; c->last_wcsph_path = h.last_path;
}

static void drop_graphs(nau_ctx* c) {
    for (auto* g : c->graphs) {
        if (g->exec) cudaGraphExecDestroy(g->exec);
        delete g;
    }
    c->graphs.clear();
    c->graph_warm = 0;
}

void nau_release_graphs(nau_ctx* c) { drop_graphs(c); }

static nau_status wcsph_step_plain(nau_ctx* c, const nau_wcsph_params* p) {
    for (int pass = 0; pass < 3; ++pass) {
        nau_status s = nau_wcsph_pass(c, p, pass);
        if (s != NAU_OK) return s;
    }
    return NAU_OK;
}

nau_status nau_wcsph_step(nau_ctx* c, const nau_wcsph_params* p) {
    static const bool env_off = std::getenv("NAU_GRAPHS") && std::atoi(std::getenv("NAU_GRAPHS")) == 0;
    if (!c->use_graphs || env_off || c->profile || c->n == 0) return wcsph_step_plain(c, p);
    // a list overflow published by an earlier step grows the capacity on the plain path
    if (c->h_nover && *(volatile int*)c->h_nover > c->nl_cap && c->nl_cap < 1024) {
        drop_graphs(c);
        return wcsph_step_plain(c, p);
    }
    const HostState before = capture_state(c, p);
    for (auto* g : c->graphs)
        if (same_state(g->before, before)) {
            if (cudaGraphLaunch(g->exec, c->stream) != cudaSuccess) {
                cudaGetLastError();
                drop_graphs(c);
                c->use_graphs = false;
                return wcsph_step_plain(c, p);
            }
            apply_state(c, g->after, g->d_rebuild);
            c->launches += g->kernels;
            return NAU_OK;
        }
    if (c->graph_warm < 2 || c->graphs.size() >= 4) {  // allocations settle first
        ++c->graph_warm;
        if (c->graphs.size() >= 4) drop_graphs(c);
        return wcsph_step_plain(c, p);
    }
    const long r0 = c->rebuild_count, l0 = c->launches;
    const std::string err0 = c->last_error;
    cudaGraph_t graph = nullptr;
    bool ok = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed) == cudaSuccess;
    nau_status st = ok ? wcsph_step_plain(c, p) : NAU_ERR_CUDA;
    if (ok) ok = cudaStreamEndCapture(c->stream, &graph) == cudaSuccess && st == NAU_OK;
    cudaGraphExec_t exec = nullptr;
    if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    if (!ok) {  // undo the host side of the captured step and run it for real
        cudaGetLastError();
        if (exec) cudaGraphExecDestroy(exec);
        apply_state(c, before, 0);
        c->rebuild_count = r0;
        c->launches = l0;
        c->last_error = err0;
        c->use_graphs = false;
        return wcsph_step_plain(c, p);
    }
    auto* g = new nau_ctx::StepGraph;
    g->exec = exec;
    g->before = before;
    g->after = capture_state(c, p);
    g->d_rebuild = c->rebuild_count - r0;
    g->kernels = c->launches - l0;
    c->graphs.push_back(g);
    if (cudaGraphLaunch(exec, c->stream) != cudaSuccess) return fail(c, NAU_ERR_CUDA, "graph launch failed");
    return NAU_OK;
}

nau_status nau_set_graphs(nau_ctx* c, int on) {
    drop_graphs(c);
    c->use_graphs = on != 0;
    return NAU_OK;
}

static void set_operand(nau_operand& o, int field_id, double uniform) {
    std::memset(&o, 0, sizeof(o));
    o.field_id = field_id;
    o.rows = 1;
    o.cols = 1;
    o.value[0] = uniform;
}

nau_status nau_dem_step(nau_ctx* c, const nau_dem_params* p) {
    if (p->law != NAU_OP_DEM_LSD && p->law != NAU_OP_DEM_HERTZ)
        return fail(c, NAU_ERR_ARG, "nau_dem_step: law must be dem_lsd or dem_l");
    if (!field_ok(c, p->f_v) || !field_ok(c, p->f_vdot) || (p->f_R >= 0 && !field_ok(c, p->f_R)) ||
        (p->f_m >= 0 && !field_ok(c, p->f_m)))
        return fail(c, NAU_ERR_ARG, "bad field id");
    if (c->dirty || !c->built_once) {
        c->reorder_skip = 1ULL << p->f_vdot;  // written by the contact sum before any read
        nau_status s = nau_build_cells(c);
        if (s != NAU_OK) return s;
    }
    nau_operand ops[7];
    set_operand(ops[0], p->f_v, 0.0);
    set_operand(ops[1], p->f_R, p->R);
    set_operand(ops[2], -1, p->P);
    set_operand(ops[3], -1, p->Q);
    set_operand(ops[4], p->f_m, p->m);
    set_operand(ops[5], -1, p->cf);
    set_operand(ops[6], -1, p->search_radius);
    nau::Opd d_ops[7];
    for (int k = 0; k < 7; ++k) d_ops[k] = nau::make_opd(c, ops[k]);
    const int dim = c->dom.dim;
    nau::launch_interact(c, p->law, 0, 0, d_ops, 7, c->fields[p->f_vdot].d, dim, 1, dim, 1, p->g);
    nau::launch_symplectic(c, c->fields[p->f_v].d, c->fields[p->f_vdot].d, nullptr, p->dt);
    c->dirty = true;
    return NAU_OK;
}

nau_status nau_leapfrog_step(nau_ctx* c, const nau_gravity_params* p) {
    if (!field_ok(c, p->f_v) || !field_ok(c, p->f_a) || (p->f_m >= 0 && !field_ok(c, p->f_m)))
        return fail(c, NAU_ERR_ARG, "bad field id");
    const double dth = 0.5 * p->dt;
    nau_status s = nau_euler(c, p->f_v, p->f_a, dth, p->f_v);  // v = euler(v, a, dt/2)
    if (s == NAU_OK) s = nau_euler(c, 0, p->f_v, p->dt, 0);     // r = euler(r, v, dt) + shift
    if (s != NAU_OK) return s;
    nau_operand ops[3];
    set_operand(ops[0], p->f_m, p->m);
    set_operand(ops[1], -1, p->G);
    set_operand(ops[2], -1, p->eps);
    s = nau_interact(c, NAU_OP_GRAVITY, 0, 0, ops, 3, p->f_a);  // a = nbody_gravity(m, G, eps)
    if (s == NAU_OK) s = nau_euler(c, p->f_v, p->f_a, dth, p->f_v);  // v = euler(v, a, dt/2)
    return s;
}

nau_status nau_set_mode(nau_ctx* c, int mode) {
    if (mode != NAU_MODE_EXACT && mode != NAU_MODE_FAST) return fail(c, NAU_ERR_ARG, "unknown mode");
    c->mode = mode;
    return NAU_OK;
}

int nau_get_mode(nau_ctx* c) { return c->mode; }

nau_status nau_set_neighbor_lists(nau_ctx* c, int on) {
    if (on < 0 || on > 2) return fail(c, NAU_ERR_ARG, "neighbour list mode must be 0, 1 or 2");
    c->use_nlist = on != 0;
    c->use_pairs = on == 1;
    c->nl_rev = -1;
    return NAU_OK;
}

nau_status nau_reduce(nau_ctx* c, int kind, int id, double* out) {
    if (!field_ok(c, id) || kind < 0 || kind > 3) return fail(c, NAU_ERR_ARG, "bad reduce args");
    if (nau_active_count(c) == 0)
        return fail(c, NAU_ERR_RUNTIME, "reduction over an empty particle system");
    nau::launch_reduce(c, kind, c->fields[id].d, c->fields[id].comps(), out);
    return collect(c);
}

nau_status nau_sync(nau_ctx* c) { return collect(c); }

const char* nau_last_error(nau_ctx* c, long* bad) {
    if (!c) {
        if (bad) *bad = -1;
        return g_static_err.c_str();
    }
    if (bad) *bad = c->last_bad;
    return c->last_error.c_str();
}

nau_status nau_profile_enable(nau_ctx* c, int on) {
    cudaStreamSynchronize(c->stream);
    c->profile = on != 0;
    c->ev_pairs.clear();
    c->ev_next = 0;
    return NAU_OK;
}

double nau_profile_ms(nau_ctx* c, int cls, long* launches) {
    cudaStreamSynchronize(c->stream);
    double total = 0.0;
    long cnt = 0;
    for (auto& pr : c->ev_pairs) {
        if (pr.first != cls) continue;
        float ms = 0.f;
        cudaError_t e = cudaEventElapsedTime(&ms, c->ev_pool[pr.second], c->ev_pool[pr.second + 1]);
        if (e == cudaSuccess) {
            total += ms;
            ++cnt;
        } else {
            c->last_error = std::string("profile: ") + cudaGetErrorString(e);
        }
    }
    if (launches) *launches = cnt;
    return total;
}

long nau_launch_count(nau_ctx* c) { return c->launches; }

int nau_wcsph_path(nau_ctx* c) { return c ? c->last_wcsph_path : -1; }

nau_status nau_list_stats(nau_ctx* c, double out[3]) {
    if (!c || !out) return NAU_ERR_ARG;
    if (c->nl_rev != c->rebuild_count || !c->d_ncount || c->n == 0)
        return fail(c, NAU_ERR_ARG, "no neighbour list is cached");
    const long threads = c->nl_pairs ? (c->n + 1) / 2 : c->n;
    std::vector<int> cnt((size_t)threads);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess ||
        cudaMemcpy(cnt.data(), c->d_ncount, sizeof(int) * (size_t)threads, cudaMemcpyDeviceToHost) != cudaSuccess)
        return fail(c, NAU_ERR_CUDA, "list statistics: copy failed");
    double walkers = 0, entries = 0, cost = 0;
    for (long w = 0; w < threads; w += 32) {
        int mx = 0;
        for (long t = w; t < std::min(threads, w + 32); ++t) {
            if (cnt[(size_t)t] <= 0) continue;  // ghosts / overflowed slots: not walked
            walkers += 1;
            entries += cnt[(size_t)t];
            mx = std::max(mx, cnt[(size_t)t]);
        }
        cost += 32.0 * mx;
    }
    out[0] = walkers;
    out[1] = entries;
    out[2] = cost;
    return NAU_OK;
}

}  // extern "C"
