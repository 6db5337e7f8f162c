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
__device__ __forceinline__ bool selected(const DomainDev& d, const double* pos,
                                         const uint8_t* active, long n, long k, int axis,
                                         double lo, double hi, const double* flag, double flo,
                                         double fhi) {
    if (!active[k]) return false;
    const int cidx = cell_index(d, axis, pos[axis * n + k]);
    if (!(cidx >= lo && cidx < hi)) return false;
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
                            double hi, const double* flag, double flo, double fhi, int* bcount) {
    const long k = blockIdx.x * (long)kSelBlock + threadIdx.x;
    const int v = k < n && selected(d, pos, active, n, k, axis, lo, hi, flag, flo, fhi);
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
                            const int* boff, int* out) {
    const long k = blockIdx.x * (long)kSelBlock + threadIdx.x;
    const int v = k < n && selected(d, pos, active, n, k, axis, lo, hi, flag, flo, fhi);
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

nau_status nau_select(nau_ctx* c, int axis, double lo, double hi, int flag_field, double flag_lo,
                      double flag_hi, int* dev_slots, long* count) {
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
                                                           flag_lo, flag_hi, scratch);
    nau::k_sel_scan<<<1, nau::kSelBlock, 0, c->stream>>>(scratch, nb, scratch + nb);
    nau::k_sel_write<<<nb, nau::kSelBlock, 0, c->stream>>>(c->dom, pos, c->d_active, n, axis, lo, hi, flag,
                                                           flag_lo, flag_hi, scratch, dev_slots);
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
    nau::GravSources gs{reinterpret_cast<const double4*>(dev_src), nsrc, self_off};
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

}  // extern "C"
