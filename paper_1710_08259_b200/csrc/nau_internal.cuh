// nau_internal.cuh — shared device/host definitions of libnau_b200.so.
//
// Data layout in HBM (one context = one GPU):
//   * every field is an fp64 SoA array, component-major: f[c*n + k], c < rows*cols,
//     k = CELL-ORDER slot (particles sorted by (flat cell, original index));
//   * orig[k]   int32  original particle index of slot k;
//   * key[k]    int32  flat cell of slot k (== ncells for inactive particles,
//                      which therefore sort to the tail);
//   * active[k] uint8  ParticleSystem::active_ (particle_system.hpp:145);
//   * cell_start[c] / cell_count[c] int32 tables, c < ncells (+1 sentinel bin).
// A rebuild (build_cells) permutes every array with one gather pass, so the
// neighbour-sum kernels read each cell's particles as a contiguous range.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "nauticle_gpu.h"

namespace nau {

constexpr int kMaxFields = 64;
constexpr double kPi = 3.14159265358979323846;

struct DomainDev {
    int dim;
    int cells[3];
    int ncells;
    int kind[3];
    double lo[3], hi[3], ext[3], cs[3];
};

// Latched device error word (surfaced by nau_sync).
struct DevErr {
    unsigned long long warnings;  // ≙ ParticleSystem::warnings_ (atomic counter)
    long long first_bad;          // lowest original index of a runtime error
    long long nan_first;          // lowest original index of a non-finite result
    int code;                     // bit 1 runtime, bit 2 nan, bit 4 outside cutoff at build
    int msg;                      // message id of the runtime error (see capi.cu)
};

enum ErrMsg {
    kMsgNone = 0,
    kMsgZeroDensity = 1,
    kMsgRadius = 2,
    kMsgOutsideCutoff = 3,
    kMsgCoincident = 4,
    kMsgDemParams = 5,
    kMsgNan = 6,
    kMsgRandBounds = 7,
    kMsgSfmTau = 8,
    kMsgSfmMass = 9,
};

// Operand as seen by a kernel: field pointer (cell order) or uniform value.
struct Opd {
    const double* p;
    double v[9];
    __device__ __forceinline__ double at(int c, int k, long n) const {
        return p ? p[(long)c * n + k] : v[c];
    }
};

// Per-axis image constants (particle_system.hpp:113-119): 2*lo and 2*hi are
// exact scalings, so precomputing them keeps the reference's rounding.
struct AxisImg {
    double ext, twolo, twohi, cs;
};

// Geometry bundle handed to every neighbour kernel.
struct Geo {
    DomainDev dom;
    AxisImg img[3];
    const double4* p4;  // positions packed (x, y, z, 0) per slot, for gathers
    float lim[3];    // fp32 pre-filter per-axis limit: cell size * (1 + 1e-3) + pre_abs
    float pre_abs;   // absolute fp32 error bound of u = x - lo differences (8 ulp of extent)
    double min_cs;   // smallest cell size
    long n;
    const double* x;  // pos component 0..dim-1 (x + a*n)
    const int* key;
    const int* orig;
    const uint8_t* active;
    const int* cell_start;
    const int* cell_count;
    const int* nact;  // == cell_start[ncells]
    const uint8_t* upd;  // per slot: 0 = ghost (a neighbour only, never updated); null: all
};

// Ghost test of a slot (slab runs, nau_set_ghost_field): ghosts take part in the sums
// as neighbours but are not evaluated or integrated.
__device__ __forceinline__ bool is_ghost(const Geo& g, long k) { return g.upd && !g.upd[k]; }

// The slots one thread block of a per-particle pass evaluates. WORK = false: slot
// = global thread index, valid below the active count, not a ghost, and (LIST) with a
// complete neighbour list — a list that overflowed its capacity carries count -1 and
// its slot is handed to the fallback pass. WORK = true (the fallback pass): the
// overflow worklist, grid-strided in block-uniform chunks (the sweeps are
// warp-synchronous, so every lane runs every chunk).
template <bool LIST, bool WORK, class Body>
__device__ __forceinline__ void for_slots(const Geo& g, const int* lcount, const int* work,
                                          const int* nwork, Body&& body) {
    if constexpr (WORK) {
        const int nw = *nwork;
        for (int base = blockIdx.x * blockDim.x; base < nw; base += gridDim.x * blockDim.x) {
            const int t = base + threadIdx.x;
            const bool in = t < nw;
            body(in ? work[t] : 0, in);
        }
    } else {
        const int k = blockIdx.x * blockDim.x + threadIdx.x;
        bool valid = k < *g.nact && !is_ghost(g, k);
        if (LIST && valid && lcount[k] < 0) valid = false;  // overflowed: the fallback pass
        body(k, valid);
    }
}

struct FieldBuf {
    int rows = 0, cols = 0;
    double* d = nullptr;    // current storage (cell order)
    double* alt = nullptr;  // reorder / two-phase twin, swapped with d
    bool live = false;
    int comps() const { return rows * cols; }
};

// 32-byte gather in ONE load instruction (sm_100: LDG.E.ENL2.256). The pair
// gathers of the neighbour sums are bound by L1 wavefronts; a double4 read as
// two 128-bit loads costs two (profiles/r1_nl_*: L1/TEX throughput ~85%).
#ifndef NAU_LD256
#define NAU_LD256 1  // non-coherent path: every ld256 source is read-only in the kernel that gathers it
#endif
__device__ __forceinline__ double4 ld256(const double4* p) {
    double4 v;
#if NAU_LD256 == 1
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
#elif NAU_LD256 == 2
    asm("ld.global.L1::evict_last.v4.f64 {%0, %1, %2, %3}, [%4];"
#elif NAU_LD256 == 3
    asm("ld.global.nc.L1::evict_last.v4.f64 {%0, %1, %2, %3}, [%4];"
#elif NAU_LD256 == 4
    asm("ld.global.L2::256B.v4.f64 {%0, %1, %2, %3}, [%4];"
#else
    asm("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
#endif
        : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
        : "l"(p));
    return v;
}

__device__ __forceinline__ void latch_error(DevErr* e, int code, int msg, long long particle) {
    atomicOr(&e->code, code);
    if (code & 1) {
        atomicMin(&e->first_bad, particle);
        atomicCAS(&e->msg, 0, msg);
    } else if (code & 2) {
        atomicMin(&e->nan_first, particle);
    } else if (code & 4) {
        atomicMin(&e->first_bad, particle);
        atomicCAS(&e->msg, 0, msg);
    }
}

// particle_system.cpp:20-31 — IEEE division then floor, periodic modulo / clamp.
__device__ __forceinline__ int cell_index(const DomainDev& d, int a, double x) {
    int n = d.cells[a];
    int c = (int)floor((x - d.lo[a]) / d.cs[a]);
    if (d.kind[a] == NAU_PERIODIC) {
        c %= n;
        if (c < 0) c += n;
        return c;
    }
    return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

// ---- smoothing kernels: src/kernel.cpp:37-69 (Wendland), cubic spline (new) ----
// Operation order matches the reference's left-associative C++ expressions.
template <int KF>
__device__ __forceinline__ double kernel_alpha(int kdim, double h) {
    if (KF == NAU_K_WENDLAND) {
        if (kdim == 1) return 3.0 / (4.0 * h);
        if (kdim == 2) return 7.0 / (4.0 * kPi * h * h);
        return 21.0 / (16.0 * kPi * h * h * h);
    } else {
        if (kdim == 1) return 2.0 / (3.0 * h);
        if (kdim == 2) return 10.0 / (7.0 * kPi * h * h);
        return 1.0 / (kPi * h * h * h);
    }
}

template <int KF>
__device__ __forceinline__ double kernel_value(double alpha, double h, double dist) {
    double q = dist / h;
    if (q >= 2.0) return 0.0;
    if (KF == NAU_K_WENDLAND) {
        double t = 1.0 - 0.5 * q;
        double t2 = t * t;
        return alpha * t2 * t2 * (2.0 * q + 1.0);
    } else {
        if (q < 1.0) return alpha * (1.0 - 1.5 * q * q + 0.75 * q * q * q);
        double t = 2.0 - q;
        return alpha * (0.25 * t * t * t);
    }
}

template <int KF>
__device__ __forceinline__ double kernel_dq(double alpha, double q) {
    if (q >= 2.0) return 0.0;
    if (KF == NAU_K_WENDLAND) {
        double t = 1.0 - 0.5 * q;
        return -5.0 * alpha * q * t * t * t;
    } else {
        if (q < 1.0) return alpha * (-3.0 * q + 2.25 * q * q);
        double t = 2.0 - q;
        return alpha * (-0.75 * t * t);
    }
}

// Kernel::gradient scale (kernel.cpp:62-69): grad = rel * scale; 0 beyond support.
template <int KF>
__device__ __forceinline__ double kernel_grad_scale(double alpha, double h, double dist) {
    double q = dist / h;
    if (q >= 2.0) return 0.0;
    return -kernel_dq<KF>(alpha, q) / (h * dist);
}

template <int DIM>
__device__ __forceinline__ double norm_rel(const double* r) {
    double s = r[0] * r[0];
    if (DIM > 1) s = s + r[1] * r[1];
    if (DIM > 2) s = s + r[2] * r[2];
    return sqrt(s);
}

// ---- neighbour enumeration: include/nauticle/particle_system.hpp:59-138 ----
// Per axis the options are the surviving direct offsets -1,0,+1 (periodic wrap
// carries a shift of -/+extent), then mirror-low (cell 0 of a symmetric axis),
// then mirror-high (cell n-1); axes combine as an odometer, axis 0 fastest.
struct AxisOpts {
    int lo_off;  // first direct offset
    int ndir;    // number of direct options
    int cnt;     // total options
};

__device__ __forceinline__ AxisOpts axis_opts(const DomainDev& d, int a, int ci) {
    AxisOpts o;
    const int n = d.cells[a];
    if (d.kind[a] == NAU_PERIODIC) {
        o.lo_off = -1;
        o.ndir = 3;
        o.cnt = 3;
        return o;
    }
    o.lo_off = ci == 0 ? 0 : -1;
    int hi_off = ci == n - 1 ? 0 : 1;
    o.ndir = hi_off - o.lo_off + 1;
    o.cnt = o.ndir;
    if (d.kind[a] == NAU_SYMMETRIC) {
        if (ci == 0) o.cnt++;
        if (ci == n - 1) o.cnt++;
    }
    return o;
}

// Option `o` of axis a: cell, additive shift, reflect (0 direct, -1 low, +1 high).
__device__ __forceinline__ void axis_opt(const DomainDev& d, int a, int ci, const AxisOpts& ao,
                                         int o, int& cell, double& shift, int& refl) {
    const int n = d.cells[a];
    if (o < ao.ndir) {
        int c = ci + ao.lo_off + o;
        shift = 0.0;
        if (c < 0) {
            c += n;
            shift = -d.ext[a];
        } else if (c >= n) {
            c -= n;
            shift = d.ext[a];
        }
        cell = c;
        refl = 0;
    } else if (o == ao.ndir && ci == 0) {
        cell = 0;
        shift = 0.0;
        refl = -1;
    } else {
        cell = n - 1;
        shift = 0.0;
        refl = 1;
    }
}

__device__ __forceinline__ double image_coord(const DomainDev& d, int a, double xj, double shift,
                                              int refl) {
    if (refl == 0) return xj + shift;
    if (refl < 0) return 2.0 * d.lo[a] - xj;
    return 2.0 * d.hi[a] - xj;
}

// Calls fn(j, rel[3], mirror_mask) for every candidate of slot k in reference
// order; mirror_mask bit a set <=> guide(a) = -1.
template <int DIM, class Fn>
__device__ __forceinline__ void for_each_candidate(const Geo& g, int k, const double* xi, Fn&& fn) {
    const DomainDev& d = g.dom;
    const int key = g.key[k];
    int ci[3];
    ci[0] = key % d.cells[0];
    ci[1] = DIM > 1 ? (key / d.cells[0]) % d.cells[1] : 0;
    ci[2] = DIM > 2 ? key / (d.cells[0] * d.cells[1]) : 0;
    AxisOpts ao[3];
#pragma unroll
    for (int a = 0; a < DIM; ++a) ao[a] = axis_opts(d, a, ci[a]);
    const int c2n = DIM > 2 ? ao[2].cnt : 1;
    const int c1n = DIM > 1 ? ao[1].cnt : 1;
    for (int o2 = 0; o2 < c2n; ++o2) {
        int cell2 = 0, refl2 = 0;
        double sh2 = 0.0;
        if (DIM > 2) axis_opt(d, 2, ci[2], ao[2], o2, cell2, sh2, refl2);
        for (int o1 = 0; o1 < c1n; ++o1) {
            int cell1 = 0, refl1 = 0;
            double sh1 = 0.0;
            if (DIM > 1) axis_opt(d, 1, ci[1], ao[1], o1, cell1, sh1, refl1);
            for (int o0 = 0; o0 < ao[0].cnt; ++o0) {
                int cell0, refl0;
                double sh0;
                axis_opt(d, 0, ci[0], ao[0], o0, cell0, sh0, refl0);
                int flat = cell0;
                if (DIM > 1) flat += d.cells[0] * cell1;
                if (DIM > 2) flat += d.cells[0] * d.cells[1] * cell2;
                const int mask = (refl0 ? 1 : 0) | (refl1 ? 2 : 0) | (refl2 ? 4 : 0);
                const int s = g.cell_start[flat];
                const int e = s + g.cell_count[flat];
                for (int j = s; j < e; ++j) {
                    double rel[3] = {0.0, 0.0, 0.0};
                    rel[0] = image_coord(d, 0, g.x[j], sh0, refl0) - xi[0];
                    if (fabs(rel[0]) > d.cs[0]) continue;
                    if (DIM > 1) {
                        rel[1] = image_coord(d, 1, g.x[g.n + j], sh1, refl1) - xi[1];
                        if (fabs(rel[1]) > d.cs[1]) continue;
                    }
                    if (DIM > 2) {
                        rel[2] = image_coord(d, 2, g.x[2 * g.n + j], sh2, refl2) - xi[2];
                        if (fabs(rel[2]) > d.cs[2]) continue;
                    }
                    fn(j, rel, mask);
                }
            }
        }
    }
}

// mirror() (tensor.cpp:115-126) of component c (column-major, rows x cols).
__device__ __forceinline__ double mirror_comp(double v, int c, int rows, int cols, int mask,
                                              int dim) {
    if (rows == 1 && cols == 1) return v;
    int r = c % rows, col = c / rows;
    double srow = (r < dim && ((mask >> r) & 1)) ? -1.0 : 1.0;
    double scol = (cols == 1 || col >= dim) ? 1.0 : (((mask >> col) & 1) ? -1.0 : 1.0);
    return v * srow * scol;
}

}  // namespace nau

// Host-side context (capi.cu owns it; kernels*.cu receive plain arguments).
namespace nau {
struct SlabComm;  // comm.cu: native NCCL slab exchange
}

struct nau_ctx {
    int device = 0;
    nau::SlabComm* slab = nullptr;  // nau_comm_init (comm.cu)
    int min_cells[3] = {0, 0, 0}, max_cells[3] = {1, 1, 1};  // as given (frames.cu describe)
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool has_domain = false;
    nau::DomainDev dom{};
    long n = 0;
    long cap = 0;  // allocated particle capacity (>= n); SoA strides use n
    std::vector<nau::FieldBuf> fields;
    int* d_orig = nullptr;
    int* d_orig_s = nullptr;
    int* d_key = nullptr;
    int* d_key_s = nullptr;
    uint8_t* d_active = nullptr;
    uint8_t* d_active_s = nullptr;
    int* d_perm = nullptr;
    int* d_perm_tmp = nullptr;
    int* d_okey = nullptr;
    int* d_skey = nullptr;    // within-cell sort key (original index, or a global id in slabs)
    int* d_skey_s = nullptr;
    float4* d_xl = nullptr;  // fp32 global-origin coordinates (sweep pre-filters)
    double4* d_aux = nullptr;  // per-particle scratch (fast WCSPH: v and p / rho^2 packed)
    double4* d_pk = nullptr;   // (A, m, 1/rho, rho) of the scalar-A SPH rules (fast.cu), lazily
    double4* d_p4 = nullptr;  // packed positions (written by the reorder pass)
    int* d_sel = nullptr;     // nau_select block-count scratch
    long sel_len = 0;
    // per-step neighbour lists of the WCSPH deck (k_nlist): cap entries per slot,
    // grown on overflow; lists off => every pass sweeps the cells itself
    bool use_nlist = true;
    uint32_t* d_nlist = nullptr;
    size_t nl_len = 0;   // entries allocated
    int* d_ncount = nullptr;
    long nc_len = 0;
    int* d_nover = nullptr;  // max list length seen when > cap (0 = fits)
    int* h_nover = nullptr;  // its host copy: mapped pinned memory written by a kernel (no copy engine)
    int* h_nover_dev = nullptr;
    int nl_cap = 0;
    long nl_rev = -1;        // list cache key: cell build, radius, option order
    double nl_radius = 0.0;
    bool nl_ordered = false;
    bool nl_pairs = false;   // paired layout (sweep.cuh consume_pairs)
    bool use_pairs = true;
    // fp16 cell-relative coordinates in a cell-padded layout (sweep.cuh HalfGrid),
    // rebuilt lazily after each cell build
    __half* d_hq = nullptr;  // 3 x hq_len
    long hq_len = 0;
    int* d_pstart = nullptr;  // ncells + 1
    int* d_pcount = nullptr;  // ncells + 1 (rounded-up counts, scan input)
    long pstart_len = 0;
    int* d_hesc = nullptr;    // escape flag (device)
    long hq_rev = -1;         // rebuild_count the fp16 copy belongs to
    bool hq_used = false;     // the fp16 grid was used since the last build: k_reorder writes it
    long xl_rev = -1;         // rebuild_count d_xl belongs to (ensure_xl)
    bool xl_used = true;      // a sweep read d_xl since the last build: k_reorder writes it
    unsigned long long reorder_skip = 0;  // fields the next build moves for inactive slots only
    int ghost_field = -1;     // nau_set_ghost_field: scalar field, != 0 marks a ghost
    uint8_t* d_upd = nullptr; // per slot (written by the reorder): 1 = updated, 0 = ghost
    // asynchronous host I/O (nau_upload_async / nau_download_async): one copy
    // stream per direction, per-field double-buffered staging in original order
    struct IoStage {
        double* buf[2] = {nullptr, nullptr};
        size_t len = 0;                        // doubles per buffer
        cudaEvent_t ready[2] = {nullptr, nullptr};     // data in buf[b] is complete
        cudaEvent_t consumed[2] = {nullptr, nullptr};  // buf[b] may be overwritten
        int next = 0;
    };
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    void* d_vm = nullptr;  // nau_eval program (vm.cu)
    size_t vm_len = 0;
    unsigned long long* d_rng = nullptr;  // RandomState counters, original order (vm.cu)
    long rng_len = 0;
    unsigned long long rng_seed = 0;
    std::vector<IoStage> io_up, io_down;  // indexed by field id
    int mode = NAU_MODE_EXACT;
    int last_wcsph_path = -1;  // nau_wcsph_path: which kernels the last nau_wcsph_step ran
    int wcsph_lists = -1;      // neighbour source of the density pass, reused by the momentum pass
    int* d_work = nullptr;     // slots whose list overflowed (async list builds) + count
    int* d_nwork = nullptr;
    long work_len = 0;
    bool nl_async = false;     // the cached list may hold overflowed (count -1) entries
    long wcsph_rev = -1;       // ... for this cell build
    int* d_cell_start = nullptr;  // ncells + 2
    int* d_cell_count = nullptr;  // ncells + 1
    int* d_cursor = nullptr;      // ncells + 1
    int* d_scan_tmp = nullptr;
    long scan_tmp_len = 0;
    double* d_red = nullptr;  // reduction scratch
    nau::DevErr* d_err = nullptr;
    nau::DevErr* h_err = nullptr;
    bool dirty = true;
    bool built_once = false;
    long rebuild_count = 0;
    unsigned long long warnings = 0;
    std::string last_error;
    long last_bad = -1;
    long launches = 0;
    // CUDA graphs of nau_wcsph_step (capi.cu): captured steps keyed by the host state
    // they start from (pointers, flags, cache keys, parameters), replayed with that
    // state's successor applied on the host
    struct StepGraph;
    std::vector<StepGraph*> graphs;
    bool use_graphs = true;
    int graph_warm = 0;  // uncaptured calls since the last invalidation (allocations settle)
    bool profile = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, int>> ev_pairs;  // (class, start event index)
    int ev_next = 0;
};

// Launch helpers shared by the .cu files (implemented in capi.cu).
namespace nau {
nau_status alloc_particle_arrays(nau_ctx* c, long cap);
nau_status grow_capacity(nau_ctx* c, long m);
Geo make_geo(nau_ctx* c);
Opd make_opd(nau_ctx* c, const nau_operand& o);
void prof_begin(nau_ctx* c, int cls);
void prof_end(nau_ctx* c, int cls);

// cells.cu
void launch_boundary_shift(nau_ctx* c);
void launch_build_cells(nau_ctx* c);
// d_xl (fp32 pre-filter coordinates) valid for the current cell build; every launch
// that may sweep calls this (the paired fp16 list path does not read d_xl).
void ensure_xl(nau_ctx* c);
void launch_neighbor_counts(nau_ctx* c, double radius, int* d_out_orig);
// async: no host synchronisation — an overflowing slot gets count -1 and joins the
// worklist for the fallback pass (nau_wcsph_pass); capacity grows from the overflow
// the previous build published.
bool build_nlist(nau_ctx* c, double radius, bool ordered, bool pairs = false,
                 bool async = false);  // false: unusable
// The current cell build's list for (radius, order, layout), built on first use
// and shared by every neighbour pass until the cells are rebuilt. Returns 0 (no
// list: sweep), 1 (per-slot lists) or 2 (paired lists, when `pairs`).
int nlist_for(nau_ctx* c, double radius, bool ordered, bool pairs = false, bool async = false);
void launch_unsort(nau_ctx* c, const double* d_src, double* d_dst, int comps);
void launch_sort_in(nau_ctx* c, const double* d_src_orig, double* d_dst, int comps);
// interact.cu
struct GravSources {  // all-gathered (x, y, z, m) rows for sharded n-body
    const double4* src;
    long nsrc, self_off;
    int accumulate = 0;  // continue the sums already in the output (source chunks in order)
};
void launch_interact(nau_ctx* c, int op, int kf, int kdim, const Opd* ops, int nops,
                     double* out, int out_rows, int out_cols, int a_rows, int a_cols,
                     const double* gadd = nullptr, const GravSources* gsrc = nullptr,
                     bool lists = false);
// integrate.cu
void launch_commit_if_ok(nau_ctx* c, const double* src, double* dst);
void launch_euler(nau_ctx* c, const double* x, const double* xdot, double dt, double* out,
                  int comps);
void launch_symplectic(nau_ctx* c, double* v, const double* vdot, const double* mask, double dt);
// passes: 1 density/EOS, 2 momentum (the symplectic update is launch_symplectic)
void launch_wcsph(nau_ctx* c, const nau_wcsph_params* p, bool lists, int passes);
void launch_reduce(nau_ctx* c, int kind, const double* f, int comps, double* h_out);
// fast.cu
bool fast_supports(int op, int a_rows, int a_cols, int dim);
void launch_g11_l0_fast(nau_ctx* c, int kf, int kdim, const Opd* ops, double* out_g,
                        double* out_l, bool lists);
void launch_interact_fast(nau_ctx* c, int op, int kf, int kdim, const Opd* ops, double* out,
                          int a_rows, bool lists = false);
void launch_wcsph_fast(nau_ctx* c, const nau_wcsph_params* p, double4* vp, int lists, int passes);
}  // namespace nau
