// slab.cu — device primitives of the multi-GPU slab decomposition.
//
// A rank owns the particles whose x lies in its slab of whole cell planes and keeps
// copies (ghosts) of its neighbours' particles within two cell planes of its
// faces. Each step it selects leavers / ghost sources (nau_select), packs them
// into particle-major rows (nau_pack_rows), exchanges rows with its neighbours
// over NCCL (the Python driver, paper_1710_08259_b200/slab.py), and reloads its
// particle set (nau_load_rows). The row's global-id column becomes the
// within-cell sort key, so cell lists keep ascending GLOBAL index order and every
// neighbour sum runs in the single-GPU (= reference) order.
#include "nau_internal.cuh"

namespace nau {

namespace {

constexpr int kSelBlock = 1024;

struct RowTable {
    int nf;
    int comps[kMaxFields];
    double* f[kMaxFields];
};

// Selection is by CELL index along `axis` (the build's own cell_index, so slab
// membership agrees with the cell a particle is listed in), in [lo, hi).
// by_x: [lo, hi) is a coordinate range instead (x-threshold slabs, nau_select_x).
__device__ __forceinline__ bool selected(const DomainDev& d, const double* pos,
                                         const uint8_t* active, long n, long k, int axis,
                                         double lo, double hi, const double* flag, double flo,
                                         double fhi, int by_x) {
    if (!active[k]) return false;
    if (by_x) {
        const double x = pos[axis * n + k];
        if (!(x >= lo && x < hi)) return false;
    } else {
        const int cidx = cell_index(d, axis, pos[axis * n + k]);
        if (!(cidx >= lo && cidx < hi)) return false;
    }
    if (flag) {
        const double v = flag[k];
        if (!(v >= flo && v <= fhi)) return false;
    }
    return true;
}

__device__ __forceinline__ int block_excl(int v, int* total) {
    __shared__ int ws[kSelBlock / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < kSelBlock / 32 ? ws[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < kSelBlock / 32) ws[lane] = s;
    }
    __syncthreads();
    const int before = w > 0 ? ws[w - 1] : 0;
    *total = ws[kSelBlock / 32 - 1];
    __syncthreads();
    return before + x - v;
}

__global__ void k_sel_count(DomainDev d, const double* pos, const uint8_t* active, long n, int axis, double lo,
                            double hi, const double* flag, double flo, double fhi, int* bcount,
                            int by_x) {
    const long k = blockIdx.x * (long)kSelBlock + threadIdx.x;
    const int v = k < n && selected(d, pos, active, n, k, axis, lo, hi, flag, flo, fhi, by_x);
    int total;
    block_excl(v, &total);
    if (threadIdx.x == 0) bcount[blockIdx.x] = total;
}

__global__ void k_sel_scan(int* bcount, int nb, int* total_out) {
    int carry = 0;
    for (int base = 0; base < nb; base += kSelBlock) {
        const int i = base + threadIdx.x;
        const int v = i < nb ? bcount[i] : 0;
        int total;
        const int ex = block_excl(v, &total);
        if (i < nb) bcount[i] = carry + ex;
        carry += total;
    }
    if (threadIdx.x == 0) *total_out = carry;
}

__global__ void k_sel_write(DomainDev d, const double* pos, const uint8_t* active, long n, int axis, double lo,
                            double hi, const double* flag, double flo, double fhi,
                            const int* boff, int* out, int by_x) {
    const long k = blockIdx.x * (long)kSelBlock + threadIdx.x;
    const int v = k < n && selected(d, pos, active, n, k, axis, lo, hi, flag, flo, fhi, by_x);
    int total;
    const int ex = block_excl(v, &total);
    if (v) out[boff[blockIdx.x] + ex] = (int)k;
}

__global__ void k_pack(long n, const int* slots, long m, int width, RowTable t, double* rows) {
    const long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const long s = slots[r];
    double* out = rows + r * width;
    int off = 0;
    for (int f = 0; f < t.nf; ++f)
        for (int c = 0; c < t.comps[f]; ++c) out[off++] = t.f[f][c * n + s];
}

__global__ void k_unpack(long m, int width, const double* rows, RowTable t, int gid_col,
                         int* orig, int* skey, uint8_t* active) {
    const long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const double* in = rows + r * width;
    int off = 0;
    for (int f = 0; f < t.nf; ++f)
        for (int c = 0; c < t.comps[f]; ++c) t.f[f][c * m + r] = in[off++];
    orig[r] = (int)r;
    skey[r] = gid_col >= 0 ? (int)in[gid_col] : (int)r;
    active[r] = 1;
}

__global__ void k_pack_sources(long n, int dim, const double* pos, const uint8_t* active,
                               const double* mf, double m, double4* out) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    double x[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < dim; ++a) x[a] = pos[a * n + k];
    const double mk = active[k] ? (mf ? mf[k] : m) : 0.0;
    out[k] = make_double4(x[0], x[1], x[2], mk);
}

// nau_rebuild_rows: kept slots (in the given order) into the twin buffers at stride m
__global__ void k_keep(long n, long m, const int* keep, long mk, RowTable src, RowTable dst,
                       const int* skey, const uint8_t* active, int* orig_s, int* skey_s,
                       uint8_t* active_s) {
    const long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (r >= mk) return;
    const long s = keep[r];
    for (int f = 0; f < src.nf; ++f)
        for (int c = 0; c < src.comps[f]; ++c) dst.f[f][c * m + r] = src.f[f][c * n + s];
    orig_s[r] = (int)r;
    skey_s[r] = skey[s];
    active_s[r] = active[s];
}

// ... and new rows after them (rows particle-major, the nau_row_width layout)
__global__ void k_append(long m, long off, long mn, int width, const double* rows, RowTable dst,
                         int gid_col, int* orig_s, int* skey_s, uint8_t* active_s) {
    const long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (r >= mn) return;
    const double* in = rows + r * width;
    const long k = off + r;
    int o = 0;
    for (int f = 0; f < dst.nf; ++f)
        for (int c = 0; c < dst.comps[f]; ++c) dst.f[f][c * m + k] = in[o++];
    orig_s[k] = (int)k;
    skey_s[k] = gid_col >= 0 ? (int)in[gid_col] : (int)k;
    active_s[k] = 1;
}

__global__ void k_hist_x(long n, const double* x, const uint8_t* active, const double* flag,
                         double flo, double fhi, double x0, double inv_w, int nbins,
                         unsigned long long* counts) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n || !active[k]) return;
    if (flag && !(flag[k] >= flo && flag[k] <= fhi)) return;
    long b = (long)floor((x[k] - x0) * inv_w);
    b = b < 0 ? 0 : (b >= nbins ? nbins - 1 : b);
    atomicAdd(&counts[b], 1ULL);
}

// Halo values of the WCSPH deck: rho, p of ghost slots from their owners, and the
// momentum pass's per-slot payload (v, p / (rho * rho)) as the density pass writes it.
__global__ void k_ghost_rho_p(long n, int dim, const int* slots, long m, const double* rows,
                              double* rho, double* p, const double* v, double4* vp) {
    const long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const long s = slots[r];
    const double ro = rows[2 * r], pr = rows[2 * r + 1];
    rho[s] = ro;
    p[s] = pr;
    double vv[3] = {0.0, 0.0, 0.0};
    for (int d = 0; d < dim; ++d) vv[d] = v[d * n + s];
    vp[s] = make_double4(vv[0], vv[1], vv[2], pr / (ro * ro));
}

__global__ void k_pack_rho_p(const int* slots, long m, const double* rho, const double* p,
                             double* rows) {
    const long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const long s = slots[r];
    rows[2 * r] = rho[s];
    rows[2 * r + 1] = p[s];
}

__global__ void k_pack_sel(const int* slots, long m, long n, int width, RowTable t, double* rows) {
    const long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const long s = slots[r];
    int o = 0;
    for (int f = 0; f < t.nf; ++f)
        for (int c = 0; c < t.comps[f]; ++c) rows[r * width + o++] = t.f[f][c * n + s];
}

__global__ void k_unpack_sel(const int* slots, long m, long n, int width, RowTable t,
                             const double* rows) {
    const long r = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (r >= m) return;
    const long s = slots[r];
    int o = 0;
    for (int f = 0; f < t.nf; ++f)
        for (int c = 0; c < t.comps[f]; ++c) t.f[f][c * n + s] = rows[r * width + o++];
}

// The momentum payload (v, p / (rho * rho)) of every ghost slot, from its fields.
__global__ void k_ghost_payload(long n, int dim, const uint8_t* upd, const uint8_t* active,
                                const double* rho, const double* p, const double* v, double4* vp) {
    const long s = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (s >= n || upd[s] || !active[s]) return;
    double vv[3] = {0.0, 0.0, 0.0};
    for (int d = 0; d < dim; ++d) vv[d] = v[d * n + s];
    const double ro = rho[s];
    vp[s] = make_double4(vv[0], vv[1], vv[2], p[s] / (ro * ro));
}

RowTable row_table(nau_ctx* c, int* width, int gid_field, int* gid_col) {
    RowTable t{};
    int off = 0;
    if (gid_col) *gid_col = -1;
    for (size_t f = 0; f < c->fields.size(); ++f) {
        FieldBuf& fb = c->fields[f];
        if (!fb.live) continue;
        if (gid_col && (int)f == gid_field) *gid_col = off;
        t.comps[t.nf] = fb.comps();
        t.f[t.nf] = fb.d;
        ++t.nf;
        off += fb.comps();
    }
    *width = off;
    return t;
}

}  // namespace

}  // namespace nau

using nau::FieldBuf;

extern "C" {

int nau_row_width(nau_ctx* c) {
    int w = 0;
    nau::row_table(c, &w, -1, nullptr);
    return w;
}

static nau_status select_impl(nau_ctx* c, int axis, double lo, double hi, int flag_field,
                              double flag_lo, double flag_hi, int* dev_slots, long* count,
                              int by_x);

nau_status nau_select(nau_ctx* c, int axis, double lo, double hi, int flag_field, double flag_lo,
                      double flag_hi, int* dev_slots, long* count) {
    return select_impl(c, axis, lo, hi, flag_field, flag_lo, flag_hi, dev_slots, count, 0);
}

nau_status nau_select_x(nau_ctx* c, int axis, double xlo, double xhi, int flag_field,
                        double flag_lo, double flag_hi, int* dev_slots, long* count) {
    return select_impl(c, axis, xlo, xhi, flag_field, flag_lo, flag_hi, dev_slots, count, 1);
}

static nau_status select_impl(nau_ctx* c, int axis, double lo, double hi, int flag_field,
                              double flag_lo, double flag_hi, int* dev_slots, long* count,
                              int by_x) {
    *count = 0;
    if (axis < 0 || axis >= c->dom.dim || c->fields.empty()) return NAU_ERR_ARG;
    if (flag_field >= 0 && (flag_field >= (int)c->fields.size() || !c->fields[flag_field].live ||
                            c->fields[flag_field].comps() != 1))
        return NAU_ERR_ARG;
    const long n = c->n;
    if (n == 0) return NAU_OK;
    const int nb = (int)((n + nau::kSelBlock - 1) / nau::kSelBlock);
    if (c->sel_len < nb + 1) {  // context-owned scratch: no per-call malloc/free (cudaFree syncs)
        if (c->d_sel) cudaFree(c->d_sel);
        c->sel_len = 2L * (nb + 1);
        if (cudaMalloc(&c->d_sel, sizeof(int) * c->sel_len) != cudaSuccess) return NAU_ERR_CUDA;
    }
    int* scratch = c->d_sel;
    const double* flag = flag_field >= 0 ? c->fields[flag_field].d : nullptr;
    const double* pos = c->fields[0].d;
    nau::k_sel_count<<<nb, nau::kSelBlock, 0, c->stream>>>(c->dom, pos, c->d_active, n, axis, lo, hi, flag,
                                                           flag_lo, flag_hi, scratch, by_x);
    nau::k_sel_scan<<<1, nau::kSelBlock, 0, c->stream>>>(scratch, nb, scratch + nb);
    nau::k_sel_write<<<nb, nau::kSelBlock, 0, c->stream>>>(c->dom, pos, c->d_active, n, axis, lo, hi, flag,
                                                           flag_lo, flag_hi, scratch, dev_slots, by_x);
    c->launches += 3;
    int total = 0;
    cudaMemcpyAsync(&total, scratch + nb, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return NAU_ERR_CUDA;
    *count = total;
    return NAU_OK;
}

nau_status nau_pack_rows(nau_ctx* c, const int* dev_slots, long m, double* dev_rows) {
    if (m == 0) return NAU_OK;
    int w = 0;
    nau::RowTable t = nau::row_table(c, &w, -1, nullptr);
    nau::k_pack<<<(int)((m + 255) / 256), 256, 0, c->stream>>>(c->n, dev_slots, m, w, t, dev_rows);
    c->launches++;
    return NAU_OK;
}

nau_status nau_pack_sources(nau_ctx* c, int f_m, double m, double* dev_rows) {
    if (c->fields.empty() || (f_m >= 0 && (f_m >= (int)c->fields.size() || !c->fields[f_m].live)))
        return NAU_ERR_ARG;
    if (c->n == 0) return NAU_OK;
    nau::k_pack_sources<<<(int)((c->n + 255) / 256), 256, 0, c->stream>>>(
        c->n, c->dom.dim, c->fields[0].d, c->d_active, f_m >= 0 ? c->fields[f_m].d : nullptr, m,
        reinterpret_cast<double4*>(dev_rows));
    c->launches++;
    return NAU_OK;
}

nau_status nau_gravity_sources(nau_ctx* c, const double* dev_src, long nsrc, long self_off,
                               double G, double eps, int out_field) {
    return nau_gravity_sources_part(c, dev_src, nsrc, self_off, G, eps, out_field, 0);
}

nau_status nau_gravity_sources_part(nau_ctx* c, const double* dev_src, long nsrc, long self_off,
                                    double G, double eps, int out_field, int accumulate) {
    if (c->fields.empty() || out_field <= 0 || out_field >= (int)c->fields.size() ||
        !c->fields[out_field].live || c->fields[out_field].comps() != c->dom.dim)
        return NAU_ERR_ARG;
    nau::Opd ops[3];
    for (int k = 0; k < 3; ++k) {
        ops[k].p = nullptr;
        for (int q = 0; q < 9; ++q) ops[k].v[q] = 0.0;
    }
    ops[1].v[0] = G;
    ops[2].v[0] = eps;
    nau::GravSources gs{reinterpret_cast<const double4*>(dev_src), nsrc, self_off, accumulate};
    const int dim = c->dom.dim;
    nau::launch_interact(c, NAU_OP_GRAVITY, 0, 0, ops, 3, c->fields[out_field].d, dim, 1, 1, 1,
                         nullptr, &gs);
    return NAU_OK;
}

nau_status nau_load_rows(nau_ctx* c, const double* dev_rows, long m, int gid_field) {
    if (c->fields.empty()) return NAU_ERR_ARG;
    if (m < 0 || m >= (1L << 25)) return NAU_ERR_ARG;
    nau_status s = nau::grow_capacity(c, m);
    if (s != NAU_OK) return s;
    c->n = m;
    int w = 0, gid_col = -1;
    nau::RowTable t = nau::row_table(c, &w, gid_field, &gid_col);
    if (m > 0) {
        nau::k_unpack<<<(int)((m + 255) / 256), 256, 0, c->stream>>>(m, w, dev_rows, t, gid_col,
                                                                    c->d_orig, c->d_skey,
                                                                    c->d_active);
        c->launches++;
    }
    c->dirty = true;
    c->built_once = false;
    c->nl_rev = -1;
    c->hq_rev = -1;
    c->xl_rev = -1;
    return NAU_OK;
}

nau_status nau_reserve(nau_ctx* c, long cap) {
    if (c->fields.empty()) return NAU_ERR_ARG;
    if (cap >= (1L << 25)) return NAU_ERR_ARG;
    if (cap <= c->cap) return NAU_OK;
    const long n = c->n;
    nau_status s = nau::grow_capacity(c, cap);  // contents dropped: call before loading
    c->n = n;
    c->dirty = true;
    c->built_once = false;
    return s;
}

nau_status nau_rebuild_rows(nau_ctx* c, const int* dev_keep, long m_keep, const double* dev_rows,
                            long m_new, int gid_field) {
    if (c->fields.empty() || m_keep < 0 || m_new < 0) return NAU_ERR_ARG;
    const long m = m_keep + m_new;
    if (m > c->cap) {
        c->last_error = "nau_rebuild_rows: capacity exceeded (nau_reserve more)";
        return NAU_ERR_ARG;
    }
    int w = 0, gid_col = -1;
    nau::RowTable src = nau::row_table(c, &w, gid_field, &gid_col);
    nau::RowTable dst = src;
    for (int f = 0, q = 0; f < (int)c->fields.size(); ++f)
        if (c->fields[f].live) dst.f[q++] = c->fields[f].alt;
    if (m_keep)
        nau::k_keep<<<(int)((m_keep + 255) / 256), 256, 0, c->stream>>>(
            c->n, m, dev_keep, m_keep, src, dst, c->d_skey, c->d_active, c->d_orig_s,
            c->d_skey_s, c->d_active_s);
    if (m_new)
        nau::k_append<<<(int)((m_new + 255) / 256), 256, 0, c->stream>>>(
            m, m_keep, m_new, w, dev_rows, dst, gid_col, c->d_orig_s, c->d_skey_s, c->d_active_s);
    c->launches += (m_keep > 0) + (m_new > 0);
    for (auto& f : c->fields)
        if (f.live) std::swap(f.d, f.alt);
    std::swap(c->d_orig, c->d_orig_s);
    std::swap(c->d_skey, c->d_skey_s);
    std::swap(c->d_active, c->d_active_s);
    c->n = m;
    c->dirty = true;
    c->built_once = false;
    c->nl_rev = -1;
    c->hq_rev = -1;
    c->xl_rev = -1;
    c->wcsph_rev = -1;
    return NAU_OK;
}

nau_status nau_histogram_x(nau_ctx* c, int axis, double x0, double x1, int nbins, int flag_field,
                           double flag_lo, double flag_hi, unsigned long long* dev_counts) {
    if (axis < 0 || axis >= c->dom.dim || nbins <= 0 || !(x1 > x0)) return NAU_ERR_ARG;
    if (flag_field >= 0 && (flag_field >= (int)c->fields.size() || !c->fields[flag_field].live))
        return NAU_ERR_ARG;
    cudaMemsetAsync(dev_counts, 0, sizeof(unsigned long long) * nbins, c->stream);
    if (c->n == 0) return NAU_OK;
    nau::k_hist_x<<<(int)((c->n + 255) / 256), 256, 0, c->stream>>>(
        c->n, c->fields[0].d + (long)axis * c->n, c->d_active,
        flag_field >= 0 ? c->fields[flag_field].d : nullptr, flag_lo, flag_hi, x0,
        nbins / (x1 - x0), nbins, dev_counts);
    c->launches++;
    return NAU_OK;
}

static bool field_table(nau_ctx* c, const int* ids, int nf, nau::RowTable& t, int* width) {
    t = nau::RowTable{};
    *width = 0;
    for (int k = 0; k < nf; ++k) {
        const int f = ids[k];
        if (f < 0 || f >= (int)c->fields.size() || !c->fields[f].live) return false;
        t.comps[t.nf] = c->fields[f].comps();
        t.f[t.nf] = c->fields[f].d;
        ++t.nf;
        *width += c->fields[f].comps();
    }
    return true;
}

nau_status nau_pack_fields(nau_ctx* c, const int* dev_slots, long m, const int* field_ids,
                           int nfields, double* dev_rows) {
    nau::RowTable t;
    int w = 0;
    if (!field_table(c, field_ids, nfields, t, &w)) return NAU_ERR_ARG;
    if (m == 0) return NAU_OK;
    nau::k_pack_sel<<<(int)((m + 255) / 256), 256, 0, c->stream>>>(dev_slots, m, c->n, w, t, dev_rows);
    c->launches++;
    return NAU_OK;
}

nau_status nau_unpack_fields(nau_ctx* c, const int* dev_slots, long m, const int* field_ids,
                             int nfields, const double* dev_rows) {
    nau::RowTable t;
    int w = 0;
    if (!field_table(c, field_ids, nfields, t, &w)) return NAU_ERR_ARG;
    if (m == 0) return NAU_OK;
    nau::k_unpack_sel<<<(int)((m + 255) / 256), 256, 0, c->stream>>>(dev_slots, m, c->n, w, t, dev_rows);
    c->launches++;
    return NAU_OK;
}

nau_status nau_wcsph_ghost_payload(nau_ctx* c, const nau_wcsph_params* p) {
    if (c->ghost_field < 0 || c->n == 0) return NAU_OK;
    nau::k_ghost_payload<<<(int)((c->n + 255) / 256), 256, 0, c->stream>>>(
        c->n, c->dom.dim, c->d_upd, c->d_active, c->fields[p->f_rho].d, c->fields[p->f_p].d,
        c->fields[p->f_v].d, c->d_aux);
    c->launches++;
    return NAU_OK;
}

nau_status nau_set_ghost_field(nau_ctx* c, int field_id) {
    if (field_id >= 0 && (field_id >= (int)c->fields.size() || !c->fields[field_id].live ||
                          c->fields[field_id].comps() != 1))
        return NAU_ERR_ARG;
    c->ghost_field = field_id;
    c->dirty = true;  // the next build writes the per-slot update mask
    return NAU_OK;
}

nau_status nau_wcsph_pack_rho_p(nau_ctx* c, const nau_wcsph_params* p, const int* dev_slots, long m,
                                double* dev_rows) {
    if (m == 0) return NAU_OK;
    nau::k_pack_rho_p<<<(int)((m + 255) / 256), 256, 0, c->stream>>>(
        dev_slots, m, c->fields[p->f_rho].d, c->fields[p->f_p].d, dev_rows);
    c->launches++;
    return NAU_OK;
}

nau_status nau_wcsph_ghost_update(nau_ctx* c, const nau_wcsph_params* p, const int* dev_slots,
                                  long m, const double* dev_rows) {
    if (m == 0) return NAU_OK;
    nau::k_ghost_rho_p<<<(int)((m + 255) / 256), 256, 0, c->stream>>>(
        c->n, c->dom.dim, dev_slots, m, dev_rows, c->fields[p->f_rho].d, c->fields[p->f_p].d,
        c->fields[p->f_v].d, c->d_aux);
    c->launches++;
    return NAU_OK;
}

}  // extern "C"
