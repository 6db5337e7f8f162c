// comm.cu — native multi-GPU slab exchange over NCCL (SURVEY.md §8(b) nau_comm_init /
// nau_halo_exchange / nau_migrate; §8(e)). The reference has no domain
// decomposition; this is new.
//
// The C++ form of slab.py's SlabRank, so a C++ host (the reference's Case loop)
// drives the multi-GPU path without Python. Rank r owns the particles whose
// coordinate along `axis` lies in [X_r, X_{r+1}) and holds ghosts: its neighbours'
// particles within the interaction radius R of its faces (flag 1 from the left, 2
// from the right), which take part in the sums but are never evaluated or integrated
// (nau_set_ghost_field). Per WCSPH step (§8(e)):
//   density pass; nau_halo_exchange(rho, p) + nau_wcsph_ghost_payload; momentum pass;
//   integrator; nau_migrate (migration and the new halo in one exchange round, the
//   local set rebuilt in place by nau_rebuild_rows); every K steps nau_slab_rebalance
//   (all-reduced x-histogram, new bounds, multi-hop migration, new halo).
// Every exchange is one ncclGroupStart; ncclSend / ncclRecv to left and right;
// ncclGroupEnd on the context's stream (counts first, then the rows). Rows carry the
// global id, which nau_rebuild_rows uses as the within-cell sort key, so every
// neighbour sum keeps the single-GPU order (tests/test_slab_gloo.py proves the Python
// driver of the same steps bitwise equal to one rank).
//
// NCCL is bound at run time (dlopen "libnccl.so.2": the copy torch already
// loaded, else the system one): the library has no link-time NCCL dependency
// and fails with NAU_ERR_COMM when NCCL is absent.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "nau_internal.cuh"

namespace nau {
namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("NCCL not found: ") + dlerror();
            return a;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p) a.why = std::string("NCCL symbol missing: ") + name;
            return p;
        };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
        a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
        a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        a.ok = a.why.empty();
        return a;
    }();
    return api;
}

// Grow-only device buffer.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t len = 0;
    cudaError_t reserve(size_t n) {
        if (n <= len) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        len = 0;
        n = n + n / 4 + 64;
        cudaError_t e = cudaMalloc(&p, sizeof(T) * n);
        if (e == cudaSuccess) len = n;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        len = 0;
    }
};

__global__ void k_set_col(double* rows, long m, int width, int col, double v) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k < m) rows[k * width + col] = v;
}

}  // namespace

struct SlabComm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    bool configured = false;
    int axis = 0, periodic = 0, gid_field = -1, flag_field = -1;
    std::vector<double> bounds;  // nranks + 1 coordinates, bounds[0] = lo, bounds[W] = hi
    double R = 0.0;              // interaction radius: the ghost halo width
    int left = -1, right = -1;
    DevBuf<int> slots;
    DevBuf<double> send_l, send_r, recv_l, recv_r, all, keep;
    DevBuf<long long> counts;  // 4: send left/right, recv right/left
    DevBuf<double> red;        // nau_allreduce staging
};

}  // namespace nau

using nau::SlabComm;

namespace {

nau_status comm_fail(nau_ctx* c, nau_status s, const std::string& msg) {
    c->last_error = msg;
    c->last_bad = -1;
    return s;
}

nau_status nccl_check(nau_ctx* c, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return NAU_OK;
    const char* m = nau::nccl().GetErrorString ? nau::nccl().GetErrorString(r) : "?";
    return comm_fail(c, NAU_ERR_COMM, std::string(what) + ": " + m);
}

// Slot lists of one exchange: kept + left + right selections, each at most n
// (reserved up front: a reallocation would drop the earlier selections).
nau_status reserve_slots(nau_ctx* c, SlabComm& s) {
    if (s.slots.reserve(3 * (size_t)c->n + 3) != cudaSuccess)
        return comm_fail(c, NAU_ERR_CUDA, "slab: out of device memory");
    return NAU_OK;
}

// Rows of the selected slots [0, m) into buf.
nau_status pack(nau_ctx* c, SlabComm& s, long from, long m, nau::DevBuf<double>& buf, int w) {
    if (buf.reserve((size_t)(m + 1) * w) != cudaSuccess)
        return comm_fail(c, NAU_ERR_CUDA, "slab: out of device memory");
    return m ? nau_pack_rows(c, s.slots.p + from, m, buf.p) : NAU_OK;
}

}  // namespace

extern "C" {

nau_status nau_comm_unique_id(unsigned char* id_out) {
    const nau::NcclApi& api = nau::nccl();
    if (!api.ok) return NAU_ERR_COMM;
    ncclUniqueId id;
    if (api.GetUniqueId(&id) != ncclSuccess) return NAU_ERR_COMM;
    static_assert(sizeof(ncclUniqueId) == NAU_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id_out, &id, sizeof(id));
    return NAU_OK;
}

nau_status nau_comm_init(nau_ctx* c, const unsigned char* id, int nranks, int rank) {
    const nau::NcclApi& api = nau::nccl();
    if (!api.ok) return comm_fail(c, NAU_ERR_COMM, api.why);
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return comm_fail(c, NAU_ERR_ARG, "nau_comm_init: bad rank / size");
    nau_comm_destroy(c);
    cudaSetDevice(c->device);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto* s = new SlabComm;
    s->nranks = nranks;
    s->rank = rank;
    nau_status st = nccl_check(c, api.CommInitRank(&s->comm, nranks, uid, rank), "ncclCommInitRank");
    if (st != NAU_OK) {
        delete s;
        return st;
    }
    c->slab = s;
    return NAU_OK;
}

void nau_comm_destroy(nau_ctx* c) {
    if (!c || !c->slab) return;
    SlabComm* s = c->slab;
    if (s->comm) nau::nccl().CommDestroy(s->comm);
    s->slots.release();
    s->send_l.release();
    s->send_r.release();
    s->recv_l.release();
    s->recv_r.release();
    s->all.release();
    s->keep.release();
    s->counts.release();
    s->red.release();
    delete s;
    c->slab = nullptr;
}

// Variable-size row swap with the neighbours (slab.py Exchanger.swap): sends are
// posted [to_left, to_right] and receives [from_right, from_left] — P2P messages
// between one pair of ranks match in posting order, and on a 2-rank ring (or a
// 1-rank ring: self) the left and right neighbour are the same rank.
nau_status nau_comm_swap(nau_ctx* c, const double* to_left, long n_left, const double* to_right,
                         long n_right, int width, const double** from_left, long* nf_left,
                         const double** from_right, long* nf_right) {
    SlabComm* s = c->slab;
    *nf_left = *nf_right = 0;
    *from_left = *from_right = nullptr;
    if (!s || !s->configured) return comm_fail(c, NAU_ERR_COMM, "slab exchange not configured");
    const nau::NcclApi& api = nau::nccl();
    if (s->counts.reserve(4) != cudaSuccess) return comm_fail(c, NAU_ERR_CUDA, "slab: no memory");
    long long h[4] = {s->left >= 0 ? n_left : 0, s->right >= 0 ? n_right : 0, 0, 0};
    cudaMemcpyAsync(s->counts.p, h, sizeof(h), cudaMemcpyHostToDevice, c->stream);
    nau_status st = nccl_check(c, api.GroupStart(), "ncclGroupStart");
    if (s->left >= 0) api.Send(s->counts.p + 0, 1, ncclInt64, s->left, s->comm, c->stream);
    if (s->right >= 0) {
        api.Send(s->counts.p + 1, 1, ncclInt64, s->right, s->comm, c->stream);
        api.Recv(s->counts.p + 2, 1, ncclInt64, s->right, s->comm, c->stream);
    }
    if (s->left >= 0) api.Recv(s->counts.p + 3, 1, ncclInt64, s->left, s->comm, c->stream);
    if (st == NAU_OK) st = nccl_check(c, api.GroupEnd(), "ncclGroupEnd");
    if (st != NAU_OK) return st;
    cudaMemcpyAsync(h, s->counts.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream);
    if (cudaStreamSynchronize(c->stream) != cudaSuccess)
        return comm_fail(c, NAU_ERR_CUDA, "slab: count exchange failed");
    const long rr = (long)h[2], rl = (long)h[3];
    if (s->recv_r.reserve((size_t)(rr + 1) * width) != cudaSuccess ||
        s->recv_l.reserve((size_t)(rl + 1) * width) != cudaSuccess)
        return comm_fail(c, NAU_ERR_CUDA, "slab: out of device memory");
    st = nccl_check(c, api.GroupStart(), "ncclGroupStart");
    if (s->left >= 0 && n_left)
        api.Send(to_left, (size_t)n_left * width, ncclFloat64, s->left, s->comm, c->stream);
    if (s->right >= 0 && n_right)
        api.Send(to_right, (size_t)n_right * width, ncclFloat64, s->right, s->comm, c->stream);
    if (s->right >= 0 && rr)
        api.Recv(s->recv_r.p, (size_t)rr * width, ncclFloat64, s->right, s->comm, c->stream);
    if (s->left >= 0 && rl)
        api.Recv(s->recv_l.p, (size_t)rl * width, ncclFloat64, s->left, s->comm, c->stream);
    if (st == NAU_OK) st = nccl_check(c, api.GroupEnd(), "ncclGroupEnd");
    if (st != NAU_OK) return st;
    *from_left = s->recv_l.p;
    *nf_left = rl;
    *from_right = s->recv_r.p;
    *nf_right = rr;
    return NAU_OK;
}

nau_status nau_allreduce(nau_ctx* c, double* values, int count, int op) {
    if (!c || count < 0 || op < 0 || op > 2) return NAU_ERR_ARG;
    SlabComm* s = c->slab;
    if (!s || count == 0) return NAU_OK;  // no communicator: the local value
    if (!nau::nccl().AllReduce) return comm_fail(c, NAU_ERR_COMM, "NCCL has no ncclAllReduce");
    if (s->red.reserve((size_t)count) != cudaSuccess)
        return comm_fail(c, NAU_ERR_CUDA, "allreduce: out of device memory");
    const ncclRedOp_t rop = op == 0 ? ncclSum : (op == 1 ? ncclMax : ncclMin);
    cudaMemcpyAsync(s->red.p, values, sizeof(double) * count, cudaMemcpyHostToDevice, c->stream);
    nau_status st = nccl_check(c, nau::nccl().AllReduce(s->red.p, s->red.p, (size_t)count,
                                                         ncclFloat64, rop, s->comm, c->stream),
                               "ncclAllReduce");
    cudaMemcpyAsync(values, s->red.p, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream);
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (st == NAU_OK && e != cudaSuccess) return comm_fail(c, NAU_ERR_CUDA, cudaGetErrorString(e));
    return st;
}

int nau_comm_size(nau_ctx* c) { return c && c->slab ? c->slab->nranks : 1; }

nau_status nau_slab_config(nau_ctx* c, int axis, const double* bounds, int periodic,
                           double radius, int gid_field, int flag_field) {
    SlabComm* s = c->slab;
    if (!s) return comm_fail(c, NAU_ERR_COMM, "nau_slab_config: call nau_comm_init first");
    if (axis < 0 || axis >= c->dom.dim || !(radius > 0.0))
        return comm_fail(c, NAU_ERR_ARG, "nau_slab_config: bad axis / radius");
    auto scalar_field = [&](int f) {
        return f >= 0 && f < (int)c->fields.size() && c->fields[f].live &&
               c->fields[f].comps() == 1;
    };
    if (!scalar_field(gid_field) || !scalar_field(flag_field))
        return comm_fail(c, NAU_ERR_ARG, "nau_slab_config: gid / flag must be scalar fields");
    const int W = s->nranks;
    for (int r = 0; r < W; ++r)
        if (!(bounds[r + 1] - bounds[r] >= (W > 1 ? 2.0 * radius : 0.0)))
            return comm_fail(c, NAU_ERR_ARG,
                             "nau_slab_config: bounds must rise, every slab at least 2 R wide");
    s->axis = axis;
    s->periodic = periodic != 0;
    s->R = radius;
    s->gid_field = gid_field;
    s->flag_field = flag_field;
    s->bounds.assign(bounds, bounds + W + 1);
    s->left = (s->periodic || s->rank > 0) ? (s->rank - 1 + W) % W : -1;
    s->right = (s->periodic || s->rank < W - 1) ? (s->rank + 1) % W : -1;
    s->configured = true;
    return nau_set_ghost_field(c, flag_field);
}

nau_status nau_slab_bounds(nau_ctx* c, double* out) {
    SlabComm* s = c->slab;
    if (!s || !s->configured) return comm_fail(c, NAU_ERR_COMM, "slab exchange not configured");
    for (size_t k = 0; k < s->bounds.size(); ++k) out[k] = s->bounds[k];
    return NAU_OK;
}

}  // extern "C"

namespace {

constexpr double kOwned = 0.0, kLeft = 1.0, kRight = 2.0;

// Column of the flag field in the nau_row_width layout (live fields in id order).
int flag_col(nau_ctx* c, int flag_field) {
    int col = 0;
    for (int f = 0; f < flag_field; ++f)
        if (c->fields[f].live) col += c->fields[f].comps();
    return col;
}

// The slab's selections: slots of active particles with x in [x0, x1) and the flag
// in [f0, f1], appended to `out` (host copy of the slots when `host` is given).
struct Sel {
    nau::DevBuf<int> d;
    long m = 0;
};

nau_status select(nau_ctx* c, SlabComm& s, double x0, double x1, double f0, double f1, Sel& out) {
    if (out.d.reserve((size_t)c->n + 1) != cudaSuccess)
        return comm_fail(c, NAU_ERR_CUDA, "slab: out of device memory");
    out.m = 0;
    return nau_select_x(c, s.axis, x0, x1, s.flag_field, f0, f1, out.d.p, &out.m);
}

// Rows of `sel` into buf at row offset `at`, flag column set to `flag` (< 0: kept).
nau_status pack_at(nau_ctx* c, const int* slots, long m, nau::DevBuf<double>& buf, long at,
                   int w, int fcol, double flag) {
    if (m == 0) return NAU_OK;
    nau_status st = nau_pack_rows(c, slots, m, buf.p + at * w);
    if (st == NAU_OK && flag >= 0.0)
        nau::k_set_col<<<(int)((m + 255) / 256), 256, 0, c->stream>>>(buf.p + at * w, m, w, fcol, flag);
    return st;
}

// x of the selected particles on the host (a small, synchronous read).
std::vector<double> host_x(nau_ctx* c, SlabComm& s, const Sel& sel, nau::DevBuf<double>& tmp, int w) {
    std::vector<double> x((size_t)sel.m);
    if (sel.m == 0) return x;
    if (tmp.reserve((size_t)sel.m * w) != cudaSuccess) return {};
    nau_pack_rows(c, sel.d.p, sel.m, tmp.p);
    const int col = s.axis;  // r is field 0: its components lead the row
    cudaMemcpy2DAsync(x.data(), sizeof(double), tmp.p + col, sizeof(double) * w, sizeof(double),
                      (size_t)sel.m, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    return x;
}

// Slot subsets (host lists) back on the device.
nau_status upload_slots(nau_ctx* c, const std::vector<int>& h, nau::DevBuf<int>& d) {
    if (d.reserve(h.size() + 1) != cudaSuccess) return comm_fail(c, NAU_ERR_CUDA, "slab: no memory");
    if (!h.empty())
        cudaMemcpyAsync(d.p, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice, c->stream);
    return NAU_OK;
}

std::vector<int> host_slots(nau_ctx* c, const Sel& sel) {
    std::vector<int> h((size_t)sel.m);
    if (sel.m) {
        cudaMemcpyAsync(h.data(), sel.d.p, sizeof(int) * sel.m, cudaMemcpyDeviceToHost, c->stream);
        cudaStreamSynchronize(c->stream);
    }
    return h;
}

// Misplaced owned particles (x outside [X0, X1)), split into the ones going left and
// right: by the nearer face (migration, dist < R enforced) or toward the new owner
// (rebalance, `owner_dir`).
nau_status split_outside(nau_ctx* c, SlabComm& s, bool rebalance, std::vector<int>& go_l,
                         std::vector<int>& go_r, nau::DevBuf<double>& tmp, int w) {
    const double lo = s.bounds.front(), hi = s.bounds.back(), ext = hi - lo;
    const double X0 = s.bounds[s.rank], X1 = s.bounds[s.rank + 1];
    const int W = s.nranks;
    go_l.clear();
    go_r.clear();
    for (int part = 0; part < 2; ++part) {
        Sel sel;
        nau_status st = part == 0 ? select(c, s, lo, X0, kOwned, kOwned, sel)
                                  : select(c, s, X1, hi, kOwned, kOwned, sel);
        if (st != NAU_OK) return st;
        const std::vector<double> x = host_x(c, s, sel, tmp, w);
        const std::vector<int> slot = host_slots(c, sel);
        for (long q = 0; q < sel.m; ++q) {
            bool left;
            if (rebalance) {
                const int own = (int)(std::upper_bound(s.bounds.begin(), s.bounds.end(), x[q]) -
                                      s.bounds.begin()) - 1;
                const int o = std::min(std::max(own, 0), W - 1);
                left = s.periodic ? ((o - s.rank + W) % W) > W / 2 : o < s.rank;
            } else {
                double dl = x[q] < X0 ? X0 - x[q] : INFINITY, dr = x[q] >= X1 ? x[q] - X1 : INFINITY;
                if (s.periodic) {
                    dl = std::fmod(std::fmod(X0 - x[q], ext) + ext, ext);
                    dr = std::fmod(std::fmod(x[q] - X1, ext) + ext, ext);
                }
                left = dl <= dr;
                if (std::min(dl, dr) >= s.R)
                    return comm_fail(c, NAU_ERR_COMM,
                                     "slab migration: a particle moved more than the interaction "
                                     "radius past the slab face in one step");
            }
            if ((left && s.left < 0) || (!left && s.right < 0))
                return comm_fail(c, NAU_ERR_COMM, "slab migration: a particle left the outermost slab");
            (left ? go_l : go_r).push_back(slot[q]);
        }
    }
    return NAU_OK;
}

long long allreduce_count(nau_ctx* c, long long v, nau_status* st) {
    double d = (double)v;
    *st = nau_allreduce(c, &d, 1, 0);
    return (long long)d;
}

// New slab bounds at histogram bin edges (slab.py bounds_from_xhist).
std::vector<double> bounds_from_hist(const std::vector<double>& hist, double x0, double x1, int W,
                                     double min_width) {
    const int nb = (int)hist.size();
    std::vector<double> cum(nb + 1, 0.0);
    for (int b = 0; b < nb; ++b) cum[b + 1] = cum[b] + hist[b];
    const double total = cum[nb];
    std::vector<double> out{x0};
    for (int r = 1; r < W; ++r) {
        const int i = (int)(std::lower_bound(cum.begin(), cum.end(), total * r / W) - cum.begin());
        const double b = x0 + (x1 - x0) * std::min(std::max(i, 0), nb) / nb;
        out.push_back(std::min(std::max(b, out.back() + min_width), x1 - (W - r) * min_width));
    }
    out.push_back(x1);
    return out;
}

}  // namespace

extern "C" {

// Halo values (§8(e) exchange 2): the listed fields of every owned particle within R of
// a face go to that neighbour, whose ghosts of that face receive them in slot order —
// the same global (cell, global id) order on both sides, so no ids travel.
nau_status nau_halo_exchange(nau_ctx* c, const int* field_ids, int nfields) {
    SlabComm* s = c->slab;
    if (!s || !s->configured) return comm_fail(c, NAU_ERR_COMM, "slab exchange not configured");
    if (s->nranks == 1) return NAU_OK;  // no neighbours: no ghosts
    int w = 0;
    for (int k = 0; k < nfields; ++k) {
        const int f = field_ids[k];
        if (f <= 0 || f >= (int)c->fields.size() || !c->fields[f].live)
            return comm_fail(c, NAU_ERR_ARG, "nau_halo_exchange: bad field id");
        w += c->fields[f].comps();
    }
    const double X0 = s->bounds[s->rank], X1 = s->bounds[s->rank + 1];
    Sel bl, br, gl, gr;
    nau_status st = select(c, *s, X0, X0 + s->R, kOwned, kOwned, bl);
    if (st == NAU_OK) st = select(c, *s, X1 - s->R, X1, kOwned, kOwned, br);
    if (st == NAU_OK) st = select(c, *s, -INFINITY, INFINITY, kLeft, kLeft, gl);
    if (st == NAU_OK) st = select(c, *s, -INFINITY, INFINITY, kRight, kRight, gr);
    if (st != NAU_OK) return st;
    if (s->send_l.reserve((size_t)(bl.m + 1) * w) != cudaSuccess ||
        s->send_r.reserve((size_t)(br.m + 1) * w) != cudaSuccess)
        return comm_fail(c, NAU_ERR_CUDA, "slab: out of device memory");
    st = nau_pack_fields(c, bl.d.p, bl.m, field_ids, nfields, s->send_l.p);
    if (st == NAU_OK) st = nau_pack_fields(c, br.d.p, br.m, field_ids, nfields, s->send_r.p);
    const double *fl = nullptr, *fr = nullptr;
    long nfl = 0, nfr = 0;
    if (st == NAU_OK)
        st = nau_comm_swap(c, s->send_l.p, bl.m, s->send_r.p, br.m, w, &fl, &nfl, &fr, &nfr);
    if (st != NAU_OK) return st;
    if (nfl != gl.m || nfr != gr.m)
        return comm_fail(c, NAU_ERR_COMM, "nau_halo_exchange: ghost count differs from the owner's");
    st = nau_unpack_fields(c, gl.d.p, gl.m, field_ids, nfields, fl);
    if (st == NAU_OK) st = nau_unpack_fields(c, gr.d.p, gr.m, field_ids, nfields, fr);
    cudaStreamSynchronize(c->stream);  // the receive buffers are reused by the next swap
    return st;
}

// Migration + halo (§8(e) exchange 3, after the integrator), one exchange round: owned
// particles that left the slab go to the neighbour (less than R past the face), owned
// particles within R of a face go to that neighbour as ghosts, and the emigrants stay
// here as ghosts of their new owner. The local set is rebuilt in place.
nau_status nau_migrate(nau_ctx* c) {
    SlabComm* s = c->slab;
    if (!s || !s->configured) return comm_fail(c, NAU_ERR_COMM, "slab exchange not configured");
    if (s->nranks == 1) return NAU_OK;  // one rank owns everything
    const int w = nau_row_width(c), fcol = flag_col(c, s->flag_field);
    const double X0 = s->bounds[s->rank], X1 = s->bounds[s->rank + 1];
    std::vector<int> el, er;
    nau_status st = split_outside(c, *s, false, el, er, s->keep, w);
    if (st != NAU_OK) return st;
    nau::DevBuf<int> del, der;
    st = upload_slots(c, el, del);
    if (st == NAU_OK) st = upload_slots(c, er, der);
    Sel keep, bl, br;
    if (st == NAU_OK) st = select(c, *s, X0, X1, kOwned, kOwned, keep);
    if (st == NAU_OK) st = select(c, *s, X0, X0 + s->R, kOwned, kOwned, bl);
    if (st == NAU_OK) st = select(c, *s, X1 - s->R, X1, kOwned, kOwned, br);
    if (st != NAU_OK) return st;
    const long ml = (long)el.size() + bl.m, mr = (long)er.size() + br.m;
    if (s->send_l.reserve((size_t)(ml + 1) * w) != cudaSuccess ||
        s->send_r.reserve((size_t)(mr + 1) * w) != cudaSuccess)
        return comm_fail(c, NAU_ERR_CUDA, "slab: out of device memory");
    st = pack_at(c, del.p, (long)el.size(), s->send_l, 0, w, fcol, -1.0);
    if (st == NAU_OK) st = pack_at(c, bl.d.p, bl.m, s->send_l, (long)el.size(), w, fcol, kRight);
    if (st == NAU_OK) st = pack_at(c, der.p, (long)er.size(), s->send_r, 0, w, fcol, -1.0);
    if (st == NAU_OK) st = pack_at(c, br.d.p, br.m, s->send_r, (long)er.size(), w, fcol, kLeft);
    const double *fl = nullptr, *fr = nullptr;
    long nfl = 0, nfr = 0;
    if (st == NAU_OK) st = nau_comm_swap(c, s->send_l.p, ml, s->send_r.p, mr, w, &fl, &nfl, &fr, &nfr);
    if (st != NAU_OK) return st;
    // arrivals + own emigrants as ghosts of their new owner
    const long ne = (long)el.size() + (long)er.size(), tot = nfl + nfr + ne;
    if (s->all.reserve((size_t)(tot + 1) * w) != cudaSuccess)
        return comm_fail(c, NAU_ERR_CUDA, "slab: out of device memory");
    if (nfl) cudaMemcpyAsync(s->all.p, fl, sizeof(double) * nfl * w, cudaMemcpyDeviceToDevice, c->stream);
    if (nfr)
        cudaMemcpyAsync(s->all.p + nfl * w, fr, sizeof(double) * nfr * w, cudaMemcpyDeviceToDevice,
                        c->stream);
    st = pack_at(c, del.p, (long)el.size(), s->all, nfl + nfr, w, fcol, kLeft);
    if (st == NAU_OK) st = pack_at(c, der.p, (long)er.size(), s->all, nfl + nfr + (long)el.size(), w, fcol, kRight);
    if (st == NAU_OK) st = nau_rebuild_rows(c, keep.d.p, keep.m, s->all.p, tot, s->gid_field);
    cudaStreamSynchronize(c->stream);
    return st;
}

// Re-balancing (§8(e): every ~100 steps): new bounds from the all-reduced x-histogram
// of owned particles, owned particles hop rank by rank toward their new owner (nearer
// direction on a ring) until none is misplaced, owned count checked, then a new halo.
nau_status nau_slab_rebalance(nau_ctx* c, int nbins) {
    SlabComm* s = c->slab;
    if (!s || !s->configured) return comm_fail(c, NAU_ERR_COMM, "slab exchange not configured");
    if (s->nranks == 1 || nbins < 1) return NAU_OK;
    const int w = nau_row_width(c), fcol = flag_col(c, s->flag_field);
    const double lo = s->bounds.front(), hi = s->bounds.back();
    Sel own;
    nau_status st = select(c, *s, lo, hi, kOwned, kOwned, own);  // drop the ghosts
    if (st == NAU_OK) st = nau_rebuild_rows(c, own.d.p, own.m, nullptr, 0, s->gid_field);
    nau::DevBuf<unsigned long long> dh;
    if (st == NAU_OK && dh.reserve((size_t)nbins) != cudaSuccess) st = NAU_ERR_CUDA;
    if (st == NAU_OK)
        st = nau_histogram_x(c, s->axis, lo, hi, nbins, s->flag_field, kOwned, kOwned, dh.p);
    if (st != NAU_OK) return st;
    std::vector<unsigned long long> hh((size_t)nbins);
    cudaMemcpyAsync(hh.data(), dh.p, sizeof(unsigned long long) * nbins, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
    std::vector<double> hist(hh.begin(), hh.end());
    st = nau_allreduce(c, hist.data(), nbins, 0);
    if (st != NAU_OK) return st;
    double total = 0.0;
    for (double v : hist) total += v;
    s->bounds = bounds_from_hist(hist, lo, hi, s->nranks, 2.0 * s->R);
    const double X0 = s->bounds[s->rank], X1 = s->bounds[s->rank + 1];
    for (int hop = 0;; ++hop) {
        if (hop > s->nranks) return comm_fail(c, NAU_ERR_COMM, "slab rebalance: particles still misplaced");
        std::vector<int> gl, gr;
        st = split_outside(c, *s, true, gl, gr, s->keep, w);
        if (st != NAU_OK) return st;
        if (allreduce_count(c, (long long)(gl.size() + gr.size()), &st) == 0 || st != NAU_OK) break;
        nau::DevBuf<int> dl, dr;
        Sel keep;
        st = upload_slots(c, gl, dl);
        if (st == NAU_OK) st = upload_slots(c, gr, dr);
        if (st == NAU_OK) st = select(c, *s, X0, X1, kOwned, kOwned, keep);
        if (st == NAU_OK && (s->send_l.reserve((gl.size() + 1) * w) != cudaSuccess ||
                             s->send_r.reserve((gr.size() + 1) * w) != cudaSuccess))
            st = NAU_ERR_CUDA;
        if (st == NAU_OK) st = pack_at(c, dl.p, (long)gl.size(), s->send_l, 0, w, fcol, -1.0);
        if (st == NAU_OK) st = pack_at(c, dr.p, (long)gr.size(), s->send_r, 0, w, fcol, -1.0);
        const double *fl = nullptr, *fr = nullptr;
        long nfl = 0, nfr = 0;
        if (st == NAU_OK)
            st = nau_comm_swap(c, s->send_l.p, (long)gl.size(), s->send_r.p, (long)gr.size(), w, &fl,
                               &nfl, &fr, &nfr);
        if (st == NAU_OK && s->all.reserve((size_t)(nfl + nfr + 1) * w) != cudaSuccess) st = NAU_ERR_CUDA;
        if (st != NAU_OK) return st;
        if (nfl) cudaMemcpyAsync(s->all.p, fl, sizeof(double) * nfl * w, cudaMemcpyDeviceToDevice, c->stream);
        if (nfr)
            cudaMemcpyAsync(s->all.p + nfl * w, fr, sizeof(double) * nfr * w, cudaMemcpyDeviceToDevice,
                            c->stream);
        st = nau_rebuild_rows(c, keep.d.p, keep.m, s->all.p, nfl + nfr, s->gid_field);
        cudaStreamSynchronize(c->stream);
        if (st != NAU_OK) return st;
    }
    Sel all;
    st = select(c, *s, lo, hi, kOwned, kOwned, all);
    if (st == NAU_OK && (double)allreduce_count(c, all.m, &st) != total && st == NAU_OK)
        return comm_fail(c, NAU_ERR_COMM, "slab rebalance: owned count changed in transit");
    // the halo for the new faces
    Sel keep, bl, br;
    if (st == NAU_OK) st = select(c, *s, X0, X1, kOwned, kOwned, keep);
    if (st == NAU_OK) st = select(c, *s, X0, X0 + s->R, kOwned, kOwned, bl);
    if (st == NAU_OK) st = select(c, *s, X1 - s->R, X1, kOwned, kOwned, br);
    if (st == NAU_OK && (s->send_l.reserve((size_t)(bl.m + 1) * w) != cudaSuccess ||
                         s->send_r.reserve((size_t)(br.m + 1) * w) != cudaSuccess))
        st = NAU_ERR_CUDA;
    if (st == NAU_OK) st = pack_at(c, bl.d.p, bl.m, s->send_l, 0, w, fcol, kRight);
    if (st == NAU_OK) st = pack_at(c, br.d.p, br.m, s->send_r, 0, w, fcol, kLeft);
    const double *fl = nullptr, *fr = nullptr;
    long nfl = 0, nfr = 0;
    if (st == NAU_OK) st = nau_comm_swap(c, s->send_l.p, bl.m, s->send_r.p, br.m, w, &fl, &nfl, &fr, &nfr);
    if (st == NAU_OK && s->all.reserve((size_t)(nfl + nfr + 1) * w) != cudaSuccess) st = NAU_ERR_CUDA;
    if (st != NAU_OK) return st;
    if (nfl) cudaMemcpyAsync(s->all.p, fl, sizeof(double) * nfl * w, cudaMemcpyDeviceToDevice, c->stream);
    if (nfr)
        cudaMemcpyAsync(s->all.p + nfl * w, fr, sizeof(double) * nfr * w, cudaMemcpyDeviceToDevice,
                        c->stream);
    st = nau_rebuild_rows(c, keep.d.p, keep.m, s->all.p, nfl + nfr, s->gid_field);
    cudaStreamSynchronize(c->stream);
    return st;
}

}  // extern "C"
