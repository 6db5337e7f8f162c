// cells.cu — neighbour-search pipeline of ParticleSystem on the device.
//
//   boundary shift  ≙ ParticleSystem::apply_boundary_shift (particle_system.cpp:56-90)
//   build cells     ≙ ParticleSystem::build_cells          (particle_system.cpp:33-54)
//     1. k_hash      cell key per slot (cell_index, particle_system.cpp:20-31) + histogram
//     2. scan        exclusive prefix sum of the histogram -> cell_start
//     3. k_scatter   slot = cell_start[key] + atomic cursor (unordered within a cell)
//     4. k_rank      within each cell, rank by original index -> the reference order
//                    (cells_[c] holds ascending i, particle_system.cpp:37-51)
//     5. k_reorder   one gather pass permuting every SoA field + orig/key/active
// All passes are streaming (HBM-bound); see DESIGN.md for the per-particle bytes.
#include <cstdio>
#include <cstdlib>

#include "nau_internal.cuh"
#include "sweep.cuh"

namespace nau {

namespace {

constexpr int kBlock = 256;

inline int blocks_for(long n, int b = kBlock) { return (int)((n + b - 1) / b); }

__global__ void k_boundary_shift(DomainDev d, long n, double* pos, uint8_t* active, DevErr* err) {
    long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n || !active[k]) return;
    unsigned long long warn = 0;
    for (int a = 0; a < d.dim; ++a) {
        double* xp = pos + a * n + k;
        double x = *xp;
        const double lo = d.lo[a], hi = d.hi[a];
        if (d.kind[a] == NAU_PERIODIC) {
            if (x < lo || x >= hi) {
                double w = fmod(x - lo, d.ext[a]);
                if (w < 0.0) w += d.ext[a];
                x = lo + w;
                if (x >= hi) x = lo;  // seam guard
                *xp = x;
            }
        } else if (d.kind[a] == NAU_SYMMETRIC) {
            if (x < lo || x > hi) ++warn;
        } else if (x < lo || x > hi) {
            active[k] = 0;
            break;
        }
    }
    if (warn) atomicAdd(&err->warnings, warn);
}

// AGG: one atomic per distinct cell per warp (__match_any_sync) — consecutive
// slots mostly share a cell, so per-particle atomics serialise on one address
// (cfg2, 64 per cell: hash + scatter 0.27 -> 0.17 ms); at a few particles per
// cell the match costs more than it saves (cfg3: +5%), see build_cells.
// KH slots per thread, strided by the block size (each stride is one run of
// consecutive slots, so the warp aggregation still sees neighbours): all loads of
// a thread are issued before the first dependent use.
constexpr int kHashIlp = 4;

template <bool AGG>
__global__ void k_hash(DomainDev d, long n, const double* pos, const uint8_t* active,
                       const int* orig, int* key, int* count, int* arrival, DevErr* err) {
    const long base = (long)blockIdx.x * blockDim.x * kHashIlp + threadIdx.x;
    double x[kHashIlp][3];
    bool act[kHashIlp];
#pragma unroll
    for (int u = 0; u < kHashIlp; ++u) {
        const long k = base + (long)u * blockDim.x;
        const bool valid = k < n;
        act[u] = valid && active[k];
#pragma unroll
        for (int a = 0; a < 3; ++a) x[u][a] = (valid && a < d.dim) ? pos[a * n + k] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kHashIlp; ++u) {
        const long k = base + (long)u * blockDim.x;
        const bool valid = k < n;
        int flat = d.ncells;
        if (act[u]) {
            flat = 0;
#pragma unroll
            for (int a = 2; a >= 0; --a) {
                if (a >= d.dim) continue;
                const double xa = x[u][a];
                if (d.kind[a] == NAU_CUTOFF && (xa < d.lo[a] || xa > d.hi[a]))
                    latch_error(err, 4, kMsgOutsideCutoff, orig[k]);
                flat = flat * d.cells[a] + cell_index(d, a, xa);
            }
        }
        // arrival[k] = this particle's place among its cell's arrivals (the counter's old
        // value): the scatter needs no second round of atomics
        if (!AGG) {
            if (valid) {
                key[k] = flat;
                arrival[k] = atomicAdd(&count[flat], 1);
            }
            continue;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, valid ? flat : -1);
        const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
        int base = 0;
        if (valid && lane == leader) base = atomicAdd(&count[flat], __popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (!valid) continue;
        key[k] = flat;
        arrival[k] = base + __popc(peers & ((1u << lane) - 1u));
    }
}

// ---- exclusive scan of int32 (three-phase: tile scan, tile-sum scan, add) ----
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_exclusive_scan(int v, int* total) {
    __shared__ int warp_sums[kScanThreads / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int s = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < kScanThreads / 32) warp_sums[lane] = s;
    }
    __syncthreads();
    int before = wid > 0 ? warp_sums[wid - 1] : 0;
    *total = warp_sums[kScanThreads / 32 - 1];
    __syncthreads();
    return before + x - v;
}

__global__ void k_scan_tiles(const int* in, int* out, long n, int* tile_sums) {
    long base = (long)blockIdx.x * kScanTile + (long)threadIdx.x * kScanItems;
    int v[kScanItems];
    int s = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = base + i < n ? in[base + i] : 0;
        s += v[i];
    }
    int total;
    int run = block_exclusive_scan(s, &total);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// Single block: exclusive scan of the tile sums in place (any count).
__global__ void k_scan_sums(int* sums, int m) {
    int carry = 0;
    for (int base = 0; base < m; base += kScanThreads) {
        int i = base + threadIdx.x;
        int v = i < m ? sums[i] : 0;
        int total;
        int ex = block_exclusive_scan(v, &total);
        if (i < m) sums[i] = carry + ex;
        carry += total;
        __syncthreads();
    }
}

__global__ void k_scan_add(int* out, long n, const int* tile_sums) {
    long base = (long)blockIdx.x * kScanTile;
    int add = tile_sums[blockIdx.x];
    for (int i = threadIdx.x; i < kScanTile; i += kScanThreads)
        if (base + i < n) out[base + i] += add;
}

// Slot = the cell's start + the arrival place k_hash took (the within-cell order is
// fixed by k_rank afterwards).
__global__ void k_scatter(long n, const int* key, const int* orig, const int* start,
                          const int* arrival, int* perm_tmp, int* okey) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int slot = start[key[k]] + arrival[k];
    perm_tmp[slot] = (int)k;
    okey[slot] = orig[k];
}

// Rank each slot inside its cell by original index (distinct keys, so the
// ranks form a permutation of the cell's slots). The inactive tail bin keeps
// scatter order: inactive particles take part in no sum.
__global__ void k_rank(long n, int ncells, const int* key, const int* start, const int* count,
                       const int* perm_tmp, const int* okey, int* perm) {
    long s = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (s >= n) return;
    int k = perm_tmp[s];
    int c = key[k];
    if (c == ncells) {
        perm[s] = k;
        return;
    }
    int st = start[c], cnt = count[c];
    int my = okey[s];
    int rank = 0;
    for (int t = st; t < st + cnt; ++t) rank += okey[t] < my;
    perm[st + rank] = k;
}

// fp16 layout length: cells padded to 32-slot blocks (only non-empty cells pad) + slack
static long half_len(long n, long nc) { return ((n + 32L * std::min<long>(nc, n) + 64) + 7) & ~7L; }

struct HalfOut {  // fp16 cell-relative coordinates of the padded layout (sweep.cuh HalfGrid)
    __half* h;
    long hlen;
    const int* pstart;
    int* escaped;
};

// Slot k (active, cell c, position x) into the padded fp16 layout; the cell's last
// slot also writes the cell's +inf pads.
template <int DIM>
__device__ __forceinline__ void write_half(const DomainDev& d, const HalfOut& o, long k, int c,
                                          const double* x, const int* cell_start,
                                          const int* cell_count) {
    const long rank = k - cell_start[c];
    // 32-slot blocks, halves interleaved (sweep.cuh HalfGrid): rank -> word rank % 16
    auto at = [&](long r) { return o.pstart[c] + (r & ~31L) + 2 * (r & 15) + ((r >> 4) & 1); };
    const long p = at(rank);
    int rem = c;
    bool esc = false;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        const int ca = rem % d.cells[a];
        rem /= d.cells[a];
        const double q = (x[a] - d.lo[a]) / d.cs[a] - (double)ca;
        // in its cell (floor == cell index) q lies in [0, 1): the fp16 bound of
        // sweep.cuh HalfGrid assumes |h| <= 1; anything else disables the fp16 path
        esc |= !(q >= 0.0 && q <= 1.0);
        o.h[a * o.hlen + p] = __double2half(q);  // round to nearest
    }
    if (esc) atomicOr(o.escaped, 1);
    if (rank == cell_count[c] - 1) {
        const __half inf = __ushort_as_half((unsigned short)0x7c00);
        const long re = (cell_count[c] + 31) & ~31;
        for (long r = rank + 1; r < re; ++r)
#pragma unroll
            for (int a = 0; a < DIM; ++a) o.h[a * o.hlen + at(r)] = inf;
    }
}

struct ReorderTable {
    int nf;
    unsigned long long skip;  // bit f: field f is written before it is read this step:
                              // only inactive slots (whose values stay frozen) are moved
    int comps[kMaxFields];
    const double* src[kMaxFields];
    double* dst[kMaxFields];
};

// One gather pass per build: orig/key/active/skey, every field (minus `skip` for
// active slots), the packed positions p4 (one 256-bit gather per pair in the
// consumers), and when requested the fp32 pre-filter copy xl and the fp16
// cell-relative coordinates of the list builder (no separate pass over r).
template <int DIM>
__global__ void __launch_bounds__(kBlock, 6) k_reorder(DomainDev d, long n, const int* perm, const int* orig, const int* key,
                          const uint8_t* active, int* orig_s, int* key_s, uint8_t* active_s,
                          float4* xl, double4* p4, const int* skey, int* skey_s,
                          ReorderTable t, HalfOut ho, const int* cell_start,
                          const int* cell_count, const double* ghost, uint8_t* upd) {
    long s = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (s >= n) return;
    int k = perm[s];
    const int kk = key[k];
    orig_s[s] = orig[k];
    skey_s[s] = skey[k];
    key_s[s] = kk;
    active_s[s] = active[k];
    const bool act = kk < d.ncells;
    // positions first (field 0), then the other fields with each field's component
    // loads issued together before its stores (non-coherent loads: the compiler
    // cannot prove src and dst distinct, and a load -> store chain per component
    // leaves one gather in flight per thread)
    double x[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < DIM; ++a) x[a] = __ldg(t.src[0] + a * n + k);
    if (!(act && (t.skip & 1ULL))) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) t.dst[0][a * n + s] = x[a];
        for (int c = DIM; c < t.comps[0]; ++c) t.dst[0][c * n + s] = __ldg(t.src[0] + c * n + k);
    }
    for (int f = 1; f < t.nf; ++f) {
        if (act && ((t.skip >> f) & 1ULL)) continue;
        const double* src = t.src[f];
        double* dst = t.dst[f];
        const int nc = t.comps[f];
        for (int c0 = 0; c0 < nc; c0 += 4) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (c0 + u < nc) v[u] = __ldg(src + (c0 + u) * n + k);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (c0 + u < nc) dst[(c0 + u) * n + s] = v[u];
        }
    }
    if (xl) {
        float4 p = make_float4(__int_as_float(0x7fc00000), 0.f, 0.f, 0.f);
        if (act) {
            float v[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int a = 0; a < DIM; ++a) v[a] = (float)(x[a] - d.lo[a]);
            p = make_float4(v[0], v[1], v[2], 0.f);
        }
        xl[s] = p;
    }
    p4[s] = make_double4(x[0], x[1], x[2], 0.0);
    if (ghost) upd[s] = ghost[k] == 0.0;
    if (ho.h && act) write_half<DIM>(d, ho, s, kk, x, cell_start, cell_count);
}

template <int DIM>
__global__ void __launch_bounds__(kSweepThreads) k_neighbor_counts(Geo g, const float4* xl,
                                                                   double radius, int* out) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = k < *g.nact;
    const int kk = valid ? k : 0;
    double xi[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < DIM; ++a) xi[a] = g.x[a * g.n + kk];
    int cnt = 0;
    sweep<DIM, false, true>(g, xl, k, valid, xi, radius,  // order-free count: rows
               [&](int, const double* rel, int) {
        if (norm_rel<DIM>(rel) <= radius) ++cnt;
    });
    if (valid) out[g.orig[k]] = cnt;
}

// Neighbour lists: the sweep's scan phase alone, survivors written to the
// lane-interleaved list (sweep.cuh build_list). Per-lane loop, no warp votes.
template <int DIM, bool ORDERED>
__global__ void __launch_bounds__(kSweepThreads) k_nlist(const __grid_constant__ Geo g,
                                                         const float4* xl, double radius,
                                                         uint32_t* list, int* count, int cap,
                                                         int* over, const __grid_constant__ HalfGrid hg,
                                                         int* work, int* nwork) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= *g.nact) return;
    if (is_ghost(g, k)) {  // a ghost is never evaluated: no list
        count[k] = 0;
        return;
    }
    uint2* lst = reinterpret_cast<uint2*>(list) + nlist_base(k, cap);
    const float pre_r = (float)radius;
    int cnt = 0, nrec = 0;
    auto emit = [&](uint32_t v, uint32_t m) { emit_rec(lst, cap, nrec, cnt, v, m); };
    if (hg.on && *hg.escaped == 0)
        build_list_half<DIM, ORDERED>(g, hg, k, emit);
    else if (axis_mode(g, radius) < 2)
        build_list<DIM, ORDERED, false>(g, xl, k, pre_r, emit);
    else
        build_list<DIM, ORDERED, true>(g, xl, k, pre_r, emit);
    count[k] = cnt;
    if (nrec > cap) {
        atomicMax(over, nrec);
        if (work) {  // async build: this slot goes to the fallback pass
            count[k] = -1;
            work[atomicAdd(nwork, 1)] = k;
        }
    }
}

// Paired lists (sweep.cuh consume_pairs): thread t = slots 2t, 2t+1; count[t] =
// entries of the union masks, split[t] = first record of the second particle (-1:
// shared records).
template <int DIM>
__global__ void __launch_bounds__(kSweepThreads) k_nlist_pair(const __grid_constant__ Geo g,
                                                              const float4* xl, double radius,
                                                              uint32_t* list, int* count,
                                                              int* split, int cap, int* over,
                                                              const __grid_constant__ HalfGrid hg,
                                                              int* work, int* nwork) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int nact = *g.nact;
    const int k0 = 2 * t;
    if (k0 >= nact) return;
    if (is_ghost(g, k0) && (k0 + 1 >= nact || is_ghost(g, k0 + 1))) {  // ghosts only: no list
        count[t] = 0;
        return;
    }
    uint2* lst = reinterpret_cast<uint2*>(list) + nlist_base(t, cap);
    int cnt = 0, nrec = 0, sp = -1;
    const int room = cap - kPairTail;  // the terminator records need two rows
    build_pair_list<DIM>(g, xl, hg, radius, k0, k0 + 1 < nact,
                         [&](uint32_t v, uint32_t m) { emit_rec(lst, room, nrec, cnt, v, m); },
                         [&]() { sp = nrec; });
    if (nrec <= room) {
        st_rec(lst, (unsigned)nrec, (uint32_t)k0, 1u);
        st_rec(lst, (unsigned)nrec + 1u, (uint32_t)k0, 1u);
        count[t] = cnt;
        split[t] = sp;
        return;
    }
    count[t] = cnt;
    atomicMax(over, nrec + kPairTail);
    if (work) {  // async build: both slots go to the fallback pass
        count[t] = -1;
        const bool has1 = k0 + 1 < nact;
        const int w = atomicAdd(nwork, has1 ? 2 : 1);
        work[w] = k0;
        if (has1) work[w + 1] = k0 + 1;
    }
}

// fp16 cell-relative coordinates (sweep.cuh HalfGrid): padded cell sizes, then one
// scatter per slot; the last slot of each cell writes its cell's +inf pads.
__global__ void k_pcount(int nc, const int* count, int* pcount) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c <= nc) pcount[c] = c < nc ? (count[c] + 31) & ~31 : 0;
}

__global__ void k_half_coords(DomainDev d, long n, const double* pos, const int* key,
                              const int* cell_start, const int* cell_count, HalfOut o) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int c = key[k];
    if (c >= d.ncells) return;  // inactive tail
    double x[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < d.dim; ++a) x[a] = pos[a * n + k];
    if (d.dim == 3) write_half<3>(d, o, k, c, x, cell_start, cell_count);
    else if (d.dim == 2) write_half<2>(d, o, k, c, x, cell_start, cell_count);
    else write_half<1>(d, o, k, c, x, cell_start, cell_count);
}

// fp32 pre-filter coordinates xl[s] = (float)(x - lo) (NaN when inactive): the sweeps'
// conservative pre-filter input. Grid-strided. cond0 / cond1 (device words, may be
// null): a no-op unless one of them is non-zero — the list builds' fallbacks (a
// particle escaped its cell box for the fp16 pre-filter; a list overflowed, so the
// fallback pass sweeps).
__global__ void k_xl(DomainDev d, long n, const double* pos, const int* key, float4* xl,
                     const int* cond0, const int* cond1) {
    if ((cond0 || cond1) && !((cond0 && *cond0) || (cond1 && *cond1))) return;
    for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n;
         k += (long)gridDim.x * blockDim.x) {
        float4 p = make_float4(__int_as_float(0x7fc00000), 0.f, 0.f, 0.f);
        if (key[k] < d.ncells) {
            float v[3] = {0.f, 0.f, 0.f};
            for (int a = 0; a < d.dim; ++a) v[a] = (float)(pos[a * n + k] - d.lo[a]);
            p = make_float4(v[0], v[1], v[2], 0.f);
        }
        xl[k] = p;
    }
}

constexpr int kXlBlocks = 148 * 8;

__global__ void k_unsort(long n, int comps, const int* orig, const double* src, double* dst) {
    long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    long o = orig[k];
    for (int c = 0; c < comps; ++c) dst[c * n + o] = src[c * n + k];
}

__global__ void k_sort_in(long n, int comps, const int* orig, const double* src, double* dst) {
    long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    long o = orig[k];
    for (int c = 0; c < comps; ++c) dst[c * n + k] = src[c * n + o];
}

void scan_exclusive(nau_ctx* c, const int* in, int* out, long n) {
    int tiles = (int)((n + kScanTile - 1) / kScanTile);
    k_scan_tiles<<<tiles, kScanThreads, 0, c->stream>>>(in, out, n, c->d_scan_tmp);
    k_scan_sums<<<1, kScanThreads, 0, c->stream>>>(c->d_scan_tmp, tiles);
    k_scan_add<<<tiles, kScanThreads, 0, c->stream>>>(out, n, c->d_scan_tmp);
    c->launches += 3;
}

}  // namespace

void launch_boundary_shift(nau_ctx* c) {
    if (c->n == 0) return;
    k_boundary_shift<<<blocks_for(c->n), kBlock, 0, c->stream>>>(c->dom, c->n, c->fields[0].d,
                                                                 c->d_active, c->d_err);
    c->launches++;
}

void launch_build_cells(nau_ctx* c) {
    const long n = c->n;
    const int nc = c->dom.ncells;
    cudaMemsetAsync(c->d_cell_count, 0, sizeof(int) * (nc + 1), c->stream);
    const bool agg = n >= 8L * nc;  // >= 8 particles per cell on average
    if (n > 0) {
        // d_perm doubles as the arrival places until k_rank writes the permutation
        if (agg)
            k_hash<true><<<blocks_for(n, kBlock * kHashIlp), kBlock, 0, c->stream>>>(c->dom, n, c->fields[0].d, c->d_active,
                                                                  c->d_orig, c->d_key, c->d_cell_count,
                                                                  c->d_perm, c->d_err);
        else
            k_hash<false><<<blocks_for(n, kBlock * kHashIlp), kBlock, 0, c->stream>>>(c->dom, n, c->fields[0].d, c->d_active,
                                                                   c->d_orig, c->d_key, c->d_cell_count,
                                                                   c->d_perm, c->d_err);
        c->launches++;
    }
    // cell_start[ncells] (start of the inactive tail bin) = number of active particles.
    scan_exclusive(c, c->d_cell_count, c->d_cell_start, nc + 1);
    if (n == 0) return;
    k_scatter<<<blocks_for(n), kBlock, 0, c->stream>>>(n, c->d_key, c->d_skey, c->d_cell_start,
                                                       c->d_perm, c->d_perm_tmp, c->d_okey);
    // (okey = the within-cell sort key: original index, or a slab's global id)
    k_rank<<<blocks_for(n), kBlock, 0, c->stream>>>(n, nc, c->d_key, c->d_cell_start,
                                                    c->d_cell_count, c->d_perm_tmp, c->d_okey,
                                                    c->d_perm);
    ReorderTable t{};
    for (size_t f = 0; f < c->fields.size(); ++f) {
        FieldBuf& fb = c->fields[f];
        if (!fb.live) continue;
        if ((c->reorder_skip >> f) & 1ULL) t.skip |= 1ULL << t.nf;
        t.comps[t.nf] = fb.comps();
        t.src[t.nf] = fb.d;
        t.dst[t.nf] = fb.alt;
        ++t.nf;
    }
    c->reorder_skip = 0;  // a hint for this build only
    // the fp32 copy and the fp16 grid only when the last step read them
    const bool want_xl = c->xl_used;
    c->xl_used = false;
    HalfOut ho{};
    if (c->hq_used && c->d_hq && c->d_hesc && c->hq_len >= half_len(n, nc) &&
        c->pstart_len >= nc + 1) {
        k_pcount<<<blocks_for(nc + 1), kBlock, 0, c->stream>>>(nc, c->d_cell_count, c->d_pcount);
        scan_exclusive(c, c->d_pcount, c->d_pstart, nc + 1);
        cudaMemsetAsync(c->d_hesc, 0, sizeof(int), c->stream);
        ho = HalfOut{c->d_hq, c->hq_len, c->d_pstart, c->d_hesc};
        c->launches++;
    }
    c->hq_used = false;
    auto reorder = [&](auto kern) {
        kern<<<blocks_for(n), kBlock, 0, c->stream>>>(c->dom, n, c->d_perm, c->d_orig, c->d_key,
                                                      c->d_active, c->d_orig_s, c->d_key_s,
                                                      c->d_active_s, want_xl ? c->d_xl : nullptr,
                                                      c->d_p4, c->d_skey, c->d_skey_s, t, ho,
                                                      c->d_cell_start, c->d_cell_count,
                                                      c->ghost_field >= 0 ? c->fields[c->ghost_field].d
                                                                          : nullptr,
                                                      c->d_upd);
    };
    if (c->dom.dim == 3) reorder(k_reorder<3>);
    else if (c->dom.dim == 2) reorder(k_reorder<2>);
    else reorder(k_reorder<1>);
    c->launches += 3;
    // nau_build_cells increments rebuild_count after this: the copies belong to the next value
    c->xl_rev = want_xl ? c->rebuild_count + 1 : -1;
    c->hq_rev = ho.h ? c->rebuild_count + 1 : -1;
    std::swap(c->d_orig, c->d_orig_s);
    std::swap(c->d_skey, c->d_skey_s);
    std::swap(c->d_key, c->d_key_s);
    std::swap(c->d_active, c->d_active_s);
    for (auto& fb : c->fields)
        if (fb.live) std::swap(fb.d, fb.alt);
}

void ensure_xl(nau_ctx* c) {
    c->xl_used = true;  // the next build writes it in its reorder pass
    if (c->xl_rev == c->rebuild_count || c->n == 0) return;
    k_xl<<<std::min(kXlBlocks, blocks_for(c->n)), kBlock, 0, c->stream>>>(
        c->dom, c->n, c->fields[0].d, c->d_key, c->d_xl, nullptr, nullptr);
    c->launches++;
    c->xl_rev = c->rebuild_count;
}

void launch_neighbor_counts(nau_ctx* c, double radius, int* d_out_orig) {
    cudaMemsetAsync(d_out_orig, 0, sizeof(int) * c->n, c->stream);
    if (c->n == 0) return;
    ensure_xl(c);
    Geo g = make_geo(c);
    const int T = kSweepThreads;
    int b = blocks_for(c->n, T);
    switch (c->dom.dim) {
        case 1: k_neighbor_counts<1><<<b, T, 0, c->stream>>>(g, c->d_xl, radius, d_out_orig); break;
        case 2: k_neighbor_counts<2><<<b, T, 0, c->stream>>>(g, c->d_xl, radius, d_out_orig); break;
        default: k_neighbor_counts<3><<<b, T, 0, c->stream>>>(g, c->d_xl, radius, d_out_orig); break;
    }
    c->launches++;
}

// fp16 pre-filter data for the list build (sweep.cuh HalfGrid), rebuilt once per
// cell build. Off (fp32 pre-filter) for anisotropic cells or radius > 1.5 cells.
#ifndef NAU_HALF
#define NAU_HALF 1
#endif
static HalfGrid half_grid(nau_ctx* c, double radius) {
    HalfGrid hg{};
    const DomainDev& d = c->dom;
    const int nc = d.ncells;
    bool iso = true;
    for (int a = 1; a < d.dim; ++a) iso &= d.cs[a] == d.cs[0];
    const double rho = radius / d.cs[0];
    if (!NAU_HALF || !iso || !(rho <= 1.5) || c->n == 0) return hg;
    const long hlen = half_len(c->n, nc);
    if (c->hq_len < hlen) {
        if (c->d_hq) cudaFree(c->d_hq);
        c->d_hq = nullptr;
        c->hq_len = 0;
        if (cudaMalloc(&c->d_hq, sizeof(__half) * 3 * hlen) != cudaSuccess) {
            cudaGetLastError();
            return hg;
        }
        c->hq_len = hlen;
        c->hq_rev = -1;
    }
    if (c->pstart_len < nc + 1) {
        if (c->d_pstart) cudaFree(c->d_pstart);
        if (c->d_pcount) cudaFree(c->d_pcount);
        c->d_pstart = c->d_pcount = nullptr;
        c->pstart_len = 0;
        if (cudaMalloc(&c->d_pstart, sizeof(int) * (nc + 1)) != cudaSuccess ||
            cudaMalloc(&c->d_pcount, sizeof(int) * (nc + 1)) != cudaSuccess) {
            cudaGetLastError();
            return hg;
        }
        c->pstart_len = nc + 1;
        c->hq_rev = -1;
    }
    if (!c->d_hesc && cudaMalloc(&c->d_hesc, sizeof(int)) != cudaSuccess) return hg;
    if (c->hq_rev != c->rebuild_count) {
        k_pcount<<<blocks_for(nc + 1), kBlock, 0, c->stream>>>(nc, c->d_cell_count, c->d_pcount);
        scan_exclusive(c, c->d_pcount, c->d_pstart, nc + 1);
        cudaMemsetAsync(c->d_hesc, 0, sizeof(int), c->stream);
        k_half_coords<<<blocks_for(c->n), kBlock, 0, c->stream>>>(
            d, c->n, c->fields[0].d, c->d_key, c->d_cell_start, c->d_cell_count,
            HalfOut{c->d_hq, c->hq_len, c->d_pstart, c->d_hesc});
        c->launches += 2;
        c->hq_rev = c->rebuild_count;
    }
    c->hq_used = true;  // the next build writes the fp16 grid in its reorder pass
    for (int a = 0; a < 3; ++a) hg.h[a] = c->d_hq + a * c->hq_len;
    hg.pstart = c->d_pstart;
    hg.escaped = c->d_hesc;
    hg.rho = (float)rho;
    hg.on = 1;
    return hg;
}

static __global__ void k_publish(const int* src, int* dst) { *(volatile int*)dst = *src; }

bool build_nlist(nau_ctx* c, double radius, bool ordered, bool pairs, bool async) {
    const long n = c->n;
    if (n == 0 || !c->use_nlist) return false;
    constexpr int kMaxCap = 1024;  // records per slot; beyond this sweeping is cheaper
    const size_t slots = (size_t)((n + 31) / 32) * 32;
    if (c->nl_cap == 0) c->nl_cap = 64;
    if (!c->d_nover && cudaMalloc(&c->d_nover, sizeof(int)) != cudaSuccess) return false;
    if (!c->h_nover) {
        if (cudaHostAlloc(&c->h_nover, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
            cudaHostGetDevicePointer(&c->h_nover_dev, c->h_nover, 0) != cudaSuccess) {
            cudaGetLastError();
            if (c->h_nover) cudaFreeHost(c->h_nover);
            c->h_nover = c->h_nover_dev = nullptr;
            return false;
        }
    }
    if (c->nc_len < n) {
        if (c->d_ncount) cudaFree(c->d_ncount);
        c->d_ncount = nullptr;
        c->nc_len = 0;
        if (cudaMalloc(&c->d_ncount, sizeof(int) * slots) != cudaSuccess) return false;
        c->nc_len = (long)slots;
    }
    if (async && c->work_len < (long)slots) {
        if (c->d_work) cudaFree(c->d_work);
        c->d_work = nullptr;
        c->work_len = 0;
        if (cudaMalloc(&c->d_work, sizeof(int) * slots) != cudaSuccess) return false;
        c->work_len = (long)slots;
    }
    if (async && !c->d_nwork && cudaMalloc(&c->d_nwork, sizeof(int)) != cudaSuccess) return false;
    if (async) {
        // capacity from the overflow the last build published (mapped memory, no sync):
        // this build's overflowing slots go to the fallback pass
        const int seen = *(volatile int*)c->h_nover;
        if (seen > c->nl_cap) {
            c->nl_cap = std::min(kMaxCap, ((seen + seen / 4 + 31) / 32) * 32);
            *(volatile int*)c->h_nover = 0;
        }
    }
    int* wk = async ? c->d_work : nullptr;
    int* nwk = async ? c->d_nwork : nullptr;
    Geo g = make_geo(c);
    const int T = kSweepThreads;
    const int b = blocks_for(n, T);
    const HalfGrid hg = half_grid(c, radius);
    if (!hg.on) {
        ensure_xl(c);
    } else if (c->xl_rev != c->rebuild_count) {
        // the fp16 builder falls back to the fp32 pre-filter when some particle escaped
        // its cell box (a device flag): d_xl filled on the device in that case only
        k_xl<<<std::min(kXlBlocks, blocks_for(n)), kBlock, 0, c->stream>>>(
            c->dom, n, c->fields[0].d, c->d_key, c->d_xl, c->d_hesc, nullptr);
        c->launches++;
    }
    for (int attempt = 0; attempt < 3; ++attempt) {
        // uint2 records + two slack rows (consume_list reads two records ahead);
        // paired: uint2 union records per thread pair, same slack
        const size_t need = pairs ? ((size_t)(n + 63) / 64 * 32) * c->nl_cap * 2 + 64 * (kPairSlackRows + 1)
                                  : slots * (size_t)c->nl_cap * 2 + 64 * (2 + NAU_LIST_PF);
        if (c->nl_len < need) {
            if (c->d_nlist) cudaFree(c->d_nlist);
            c->d_nlist = nullptr;
            c->nl_len = 0;
            if (cudaMalloc(&c->d_nlist, sizeof(uint32_t) * need) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            c->nl_len = need;
        }
        cudaMemsetAsync(c->d_nover, 0, sizeof(int), c->stream);
        if (async) cudaMemsetAsync(c->d_nwork, 0, sizeof(int), c->stream);
        const double r = radius;
        prof_begin(c, 302);
        if (pairs) {
            const int pb = (int)(((n + 1) / 2 + T - 1) / T);
            switch (c->dom.dim) {
                case 1: k_nlist_pair<1><<<pb, T, 0, c->stream>>>(g, c->d_xl, r, c->d_nlist, c->d_ncount, c->d_ncount + (slots >> 1), c->nl_cap, c->d_nover, hg, wk, nwk); break;
                case 2: k_nlist_pair<2><<<pb, T, 0, c->stream>>>(g, c->d_xl, r, c->d_nlist, c->d_ncount, c->d_ncount + (slots >> 1), c->nl_cap, c->d_nover, hg, wk, nwk); break;
                default: k_nlist_pair<3><<<pb, T, 0, c->stream>>>(g, c->d_xl, r, c->d_nlist, c->d_ncount, c->d_ncount + (slots >> 1), c->nl_cap, c->d_nover, hg, wk, nwk); break;
            }
        } else if (ordered) {
            switch (c->dom.dim) {
                case 1: k_nlist<1, true><<<b, T, 0, c->stream>>>(g, c->d_xl, r, c->d_nlist, c->d_ncount, c->nl_cap, c->d_nover, hg, wk, nwk); break;
                case 2: k_nlist<2, true><<<b, T, 0, c->stream>>>(g, c->d_xl, r, c->d_nlist, c->d_ncount, c->nl_cap, c->d_nover, hg, wk, nwk); break;
                default: k_nlist<3, true><<<b, T, 0, c->stream>>>(g, c->d_xl, r, c->d_nlist, c->d_ncount, c->nl_cap, c->d_nover, hg, wk, nwk); break;
            }
        } else {
            switch (c->dom.dim) {
                case 1: k_nlist<1, false><<<b, T, 0, c->stream>>>(g, c->d_xl, r, c->d_nlist, c->d_ncount, c->nl_cap, c->d_nover, hg, wk, nwk); break;
                case 2: k_nlist<2, false><<<b, T, 0, c->stream>>>(g, c->d_xl, r, c->d_nlist, c->d_ncount, c->nl_cap, c->d_nover, hg, wk, nwk); break;
                default: k_nlist<3, false><<<b, T, 0, c->stream>>>(g, c->d_xl, r, c->d_nlist, c->d_ncount, c->nl_cap, c->d_nover, hg, wk, nwk); break;
            }
        }
        prof_end(c, 302);
        c->launches++;
        // The overflow word reaches the host through mapped memory written by a
        // one-thread kernel: a cudaMemcpy would queue on the D2H copy engine behind
        // the previous step's result downloads and stall the step until they finish.
        k_publish<<<1, 1, 0, c->stream>>>(c->d_nover, c->h_nover_dev);
        c->launches++;
        if (async && hg.on && c->xl_rev != c->rebuild_count) {
            // the fallback pass sweeps the overflowed slots' candidates with d_xl
            k_xl<<<std::min(kXlBlocks, blocks_for(n)), kBlock, 0, c->stream>>>(
                c->dom, n, c->fields[0].d, c->d_key, c->d_xl, c->d_nwork, nullptr);
            c->launches++;
        }
        if (async) return true;  // overflowed slots: count -1, in the worklist
        if (cudaStreamSynchronize(c->stream) != cudaSuccess) return false;
        const int over = *(volatile int*)c->h_nover;
        if (over == 0) return true;
        if (over > kMaxCap) return false;
        c->nl_cap = std::min(kMaxCap, ((over + over / 4 + 31) / 32) * 32);
    }
    return false;
}

int nlist_for(nau_ctx* c, double radius, bool ordered, bool pairs, bool async) {
    if (!c->use_nlist || c->n == 0) return 0;
    pairs = pairs && c->use_pairs && !ordered;
    // an async list may hold overflowed slots: only its own (fallback-aware) consumers reuse it
    if (c->nl_rev == c->rebuild_count && c->nl_radius == radius && c->nl_ordered == ordered &&
        c->nl_pairs == pairs && (async || !c->nl_async))
        return pairs ? 2 : 1;
    c->nl_rev = -1;
    if (!build_nlist(c, radius, ordered, pairs, async)) {
        if (!pairs || !build_nlist(c, radius, ordered, false, async)) return 0;
        pairs = false;
    }
    c->nl_rev = c->rebuild_count;
    c->nl_radius = radius;
    c->nl_ordered = ordered;
    c->nl_pairs = pairs;
    c->nl_async = async;
    return pairs ? 2 : 1;
}

void launch_unsort(nau_ctx* c, const double* d_src, double* d_dst, int comps) {
    if (c->n == 0) return;
    k_unsort<<<blocks_for(c->n), kBlock, 0, c->stream>>>(c->n, comps, c->d_orig, d_src, d_dst);
    c->launches++;
}

void launch_sort_in(nau_ctx* c, const double* d_src_orig, double* d_dst, int comps) {
    if (c->n == 0) return;
    k_sort_in<<<blocks_for(c->n), kBlock, 0, c->stream>>>(c->n, comps, c->d_orig, d_src_orig,
                                                          d_dst);
    c->launches++;
}

}  // namespace nau
