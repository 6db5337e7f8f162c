// comm.cu — native multi-GPU slab exchange over NCCL (SURVEY.md §8(b) nau_comm_init /
// nau_halo_exchange / nau_migrate; §8(e)). The reference has no domain
// decomposition; this is new.
//
// The C++ form of slab.py's SlabRank, so a C++ host (the reference's Case loop)
// drives the multi-GPU path without Python: rank r owns the particles whose cell
// along `axis` lies in [b_r, b_{r+1}) and keeps ghost copies of the `ghost_planes`
// cell planes beyond each face. After a physics step:
//   nau_migrate        owned particles whose cell left the slab go to the
//                      neighbour that owns it (they move < 1 cell per step);
//                      the context is reloaded with its owned particles only;
//   nau_halo_exchange  the first / last ghost_planes owned planes go to the
//                      neighbours, arrive flagged as ghosts; the context is
//                      reloaded with owned + ghosts.
// Every exchange is one ncclGroupStart; ncclSend / ncclRecv to left and right;
// ncclGroupEnd on the context's stream (counts first, then the rows). Rows carry
// the global id, which nau_load_rows uses as the within-cell sort key, so every
// neighbour sum keeps the single-GPU order (tests/test_slab_gloo.py proves the
// Python driver of the same steps bitwise equal to one rank).
//
// NCCL is bound at run time (dlopen "libnccl.so.2": the copy torch already
// loaded, else the system one): the library has no link-time NCCL dependency
// and fails with NAU_ERR_COMM when NCCL is absent.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
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
    int axis = 0, periodic = 0, ghost_planes = 2, gid_field = -1, ghost_field = -1;
    int lo_c = 0, hi_c = 0, ncx = 0;
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

// Slots (appended at *off) of active particles with axis-cell in [c0, c1) and
// ghost flag == ghost, wrapping on a periodic axis (slab.py SlabRank._sel).
nau_status select_range(nau_ctx* c, SlabComm& s, int c0, int c1, double ghost, long* off) {
    auto one = [&](int a, int b) -> nau_status {
        if (b <= a) return NAU_OK;
        long cnt = 0;
        nau_status st = nau_select(c, s.axis, (double)a, (double)b, s.ghost_field, ghost, ghost,
                                   s.slots.p + *off, &cnt);
        *off += cnt;
        return st;
    };
    if (!s.periodic) return one(std::max(c0, 0), std::min(c1, s.ncx));
    if (c1 <= c0) return NAU_OK;
    if (c1 - c0 >= s.ncx) return one(0, s.ncx);
    // shift into the ring (0 <= c0 < ncx), then split at the seam
    const int k = (c0 >= 0 ? c0 : c0 - s.ncx + 1) / s.ncx;
    c0 -= k * s.ncx;
    c1 -= k * s.ncx;
    nau_status st = one(c0, std::min(c1, s.ncx));
    if (st == NAU_OK && c1 > s.ncx) st = one(0, c1 - s.ncx);
    return st;
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

nau_status nau_slab_config(nau_ctx* c, int axis, const int* bounds, int periodic,
                           int ghost_planes, int gid_field, int ghost_field) {
    SlabComm* s = c->slab;
    if (!s) return comm_fail(c, NAU_ERR_COMM, "nau_slab_config: call nau_comm_init first");
    if (axis < 0 || axis >= c->dom.dim || ghost_planes < 1)
        return comm_fail(c, NAU_ERR_ARG, "nau_slab_config: bad axis / ghost planes");
    auto scalar_field = [&](int f) {
        return f >= 0 && f < (int)c->fields.size() && c->fields[f].live &&
               c->fields[f].comps() == 1;
    };
    if (!scalar_field(gid_field) || !scalar_field(ghost_field))
        return comm_fail(c, NAU_ERR_ARG, "nau_slab_config: gid / ghost must be scalar fields");
    const int ncx = c->dom.cells[axis];
    for (int r = 0; r < s->nranks; ++r)
        if (!(bounds[r] < bounds[r + 1]) || bounds[0] != 0 || bounds[s->nranks] != ncx)
            return comm_fail(c, NAU_ERR_ARG, "nau_slab_config: bounds must rise from 0 to the cell count");
    s->axis = axis;
    s->periodic = periodic != 0;
    s->ghost_planes = ghost_planes;
    s->gid_field = gid_field;
    s->ghost_field = ghost_field;
    s->ncx = ncx;
    s->lo_c = bounds[s->rank];
    s->hi_c = bounds[s->rank + 1];
    const int W = s->nranks;
    s->left = (s->periodic || s->rank > 0) ? (s->rank - 1 + W) % W : -1;
    s->right = (s->periodic || s->rank < W - 1) ? (s->rank + 1) % W : -1;
    s->configured = true;
    return NAU_OK;
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

// Concatenate row blocks into s->all and load them (owned particles first).
static nau_status load_blocks(nau_ctx* c, SlabComm* s, const double* const* blk, const long* m,
                              int nblk, int width) {
    long tot = 0;
    for (int b = 0; b < nblk; ++b) tot += m[b];
    if (s->all.reserve((size_t)(tot + 1) * width) != cudaSuccess)
        return comm_fail(c, NAU_ERR_CUDA, "slab: out of device memory");
    long off = 0;
    for (int b = 0; b < nblk; ++b) {
        if (m[b])
            cudaMemcpyAsync(s->all.p + off * width, blk[b], sizeof(double) * m[b] * width,
                            cudaMemcpyDeviceToDevice, c->stream);
        off += m[b];
    }
    return nau_load_rows(c, s->all.p, tot, s->gid_field);
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

nau_status nau_migrate(nau_ctx* c) {
    SlabComm* s = c->slab;
    if (!s || !s->configured) return comm_fail(c, NAU_ERR_COMM, "slab exchange not configured");
    // a 1-rank ring: the rank owns every plane (its own neighbour: nothing to send)
    if (s->nranks == 1 && s->periodic) return NAU_OK;
    const int w = nau_row_width(c), g = s->ghost_planes;
    long nk = 0, nl = 0, nr = 0;
    nau_status st = reserve_slots(c, *s);
    if (st == NAU_OK) st = select_range(c, *s, s->lo_c, s->hi_c, 0.0, &nk);
    if (st == NAU_OK) st = pack(c, *s, 0, nk, s->keep, w);
    long off = nk;
    if (st == NAU_OK) st = select_range(c, *s, s->lo_c - g, s->lo_c, 0.0, &off);
    nl = off - nk;
    if (st == NAU_OK) st = pack(c, *s, nk, nl, s->send_l, w);
    const long o2 = off;
    if (st == NAU_OK) st = select_range(c, *s, s->hi_c, s->hi_c + g, 0.0, &off);
    nr = off - o2;
    if (st == NAU_OK) st = pack(c, *s, o2, nr, s->send_r, w);
    if (st != NAU_OK) return st;
    const double *fl = nullptr, *fr = nullptr;
    long nfl = 0, nfr = 0;
    st = nau_comm_swap(c, s->send_l.p, nl, s->send_r.p, nr, w, &fl, &nfl, &fr, &nfr);
    if (st != NAU_OK) return st;
    const double* blk[3] = {s->keep.p, fl, fr};
    const long m[3] = {nk, nfl, nfr};
    st = load_blocks(c, s, blk, m, 3, w);
    cudaStreamSynchronize(c->stream);
    return st;
}

nau_status nau_halo_exchange(nau_ctx* c) {
    SlabComm* s = c->slab;
    if (!s || !s->configured) return comm_fail(c, NAU_ERR_COMM, "slab exchange not configured");
    if (s->nranks == 1 && s->periodic) return NAU_OK;  // ghosts of itself: none kept
    const int w = nau_row_width(c), g = s->ghost_planes;
    // owned rows (ghost flag 0 inside the slab), then the boundary planes
    long nk = 0;
    nau_status st = reserve_slots(c, *s);
    if (st == NAU_OK) st = select_range(c, *s, s->lo_c, s->hi_c, 0.0, &nk);
    long off = nk;
    if (st == NAU_OK) st = select_range(c, *s, s->lo_c, s->lo_c + g, 0.0, &off);
    const long nl = off - nk, o2 = off;
    if (st == NAU_OK) st = select_range(c, *s, s->hi_c - g, s->hi_c, 0.0, &off);
    const long nr = off - o2;
    if (st == NAU_OK) st = pack(c, *s, 0, nk, s->keep, w);
    if (st == NAU_OK) st = pack(c, *s, nk, nl, s->send_l, w);
    if (st == NAU_OK) st = pack(c, *s, o2, nr, s->send_r, w);
    const double *fl = nullptr, *fr = nullptr;
    long nfl = 0, nfr = 0;
    if (st == NAU_OK)
        st = nau_comm_swap(c, s->send_l.p, nl, s->send_r.p, nr, w, &fl, &nfl, &fr, &nfr);
    if (st == NAU_OK) {
        int gcol = 0;  // the ghost flag's column: live fields in id order (nau_row_width)
        for (int f = 0; f < s->ghost_field; ++f)
            if (c->fields[f].live) gcol += c->fields[f].comps();
        for (int b = 0; b < 2; ++b) {
            const long m = b ? nfr : nfl;
            double* p = const_cast<double*>(b ? fr : fl);
            if (m)
                nau::k_set_col<<<(int)((m + 255) / 256), 256, 0, c->stream>>>(p, m, w, gcol, 1.0);
        }
        const double* blk[3] = {s->keep.p, fl, fr};
        const long m[3] = {nk, nfl, nfr};
        st = load_blocks(c, s, blk, m, 3, w);
    }
    cudaStreamSynchronize(c->stream);
    return st;
}

}  // extern "C"
