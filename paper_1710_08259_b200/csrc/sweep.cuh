// sweep.cuh — warp-cooperative neighbour sweep with a deferred pair queue.
//
// Same candidate set as the reference's ParticleSystem::for_each_neighbor
// (particle_system.hpp:59-138), restructured for SIMT efficiency
// (profiles/r1_v0_ncu_full_cfg2.md: the one-pass version ran 18 of 32 lanes per
// instruction and the pair arithmetic of an accepted pair at ~15% lane
// occupancy, because only ~1 in 6 candidates lies inside the support):
//
//   phase A (scan)   each lane (= one particle) walks ITS candidate sequence —
//                    stencil options, each option's cell range in slot order —
//                    testing candidates with a conservative fp32 pre-filter on the
//                    global-origin coordinates u = x - lo (float4 xl[], written by
//                    the reorder pass). Survivors go to the lane's FIFO in shared
//                    memory as (slot j | image code << 25).
//   phase B (drain)  when a FIFO could overflow on the next chunk, or all lanes
//                    are done, the warp drains the FIFOs in lockstep: lane L takes
//                    its q-th entry, recomputes image and rel in fp64 exactly as the
//                    reference (per-axis |rel_a| > cell_size rejection included) and
//                    calls fn(j, rel, mirror_mask) — the operator's pair rule.
//
// Option order. ORDERED = true walks the options in the reference's odometer
// order (axis 0 fastest): with FIFO order == candidate order every accumulator
// sums exactly as interact() does (bitwise EXACT mode). ORDERED = false (FAST
// mode, and the order-free neighbour count) visits option i and its point
// reflection N-1-i back to back: which cells a particle accepts from depends on
// where it sits in its cell, so in odometer order the lanes' FIFOs fill at very
// different rates mid-sweep and a drain runs at mean/max fill occupancy (53% on
// cfg2, profiles/r1_v3_*); opposite cells compensate each other.
// The pre-filter only ever passes a superset of the exact test (margin 1e-3 R
// plus 8 ulp of the extent; NaN passes).
#pragma once

#include "nau_internal.cuh"

namespace nau {

#ifndef NAU_ROWS
#define NAU_ROWS 1
#endif
constexpr int kQueue = 64;          // FIFO depth per lane (8 KB of shared memory per warp)
constexpr int kChunk = 16;          // max candidates scanned between warp votes
constexpr int kSweepThreads = 128;  // 4 warps, 32 KB shared memory per CTA
constexpr int kSlotBits = 25;       // FIFO entry = slot | image code << 25 (n < 2^25 per context)

struct SweepSmem {
    uint32_t e[kQueue * 32];
};

// Per-axis image code: 0 direct, 1 direct + extent, 2 direct - extent,
// 3 mirror across the low wall, 4 mirror across the high wall. Branch-free:
// img = (+/-xj) + off reproduces xj + shift and 2*lo - xj / 2*hi - xj exactly.
__device__ __forceinline__ double image_of(const AxisImg& ax, double xj, int c) {
    const double off = c == 0 ? 0.0 : (c == 1 ? ax.ext : (c == 2 ? -ax.ext : (c == 3 ? ax.twolo : ax.twohi)));
    const double xs = c >= 3 ? -xj : xj;
    return xs + off;
}

template <int DIM>
__device__ __forceinline__ void decode_cell(const DomainDev& d, int key, int* ci) {
    ci[0] = key % d.cells[0];
    ci[1] = DIM > 1 ? (key / d.cells[0]) % d.cells[1] : 0;
    ci[2] = DIM > 2 ? key / (d.cells[0] * d.cells[1]) : 0;
}

// Option `o` of axis a -> cell, image code, pre-filter transform in global-origin
// coordinates u = x - lo: u_img = sg * u_j + bs.
__device__ __forceinline__ void option_of(const DomainDev& d, int a, int ci, const AxisOpts& ao,
                                          int o, int& cell, int& icode, float& sg, float& bs) {
    const int n = d.cells[a];
    const float ext = (float)d.ext[a];
    if (o < ao.ndir) {
        int c = ci + ao.lo_off + o;
        icode = 0;
        bs = 0.0f;
        if (c < 0) {
            c += n;
            icode = 2;  // shift = -extent
            bs = -ext;
        } else if (c >= n) {
            c -= n;
            icode = 1;  // shift = +extent
            bs = ext;
        }
        cell = c;
        sg = 1.0f;
    } else if (o == ao.ndir && ci == 0) {
        cell = 0;
        icode = 3;  // 2 lo - x  ->  -u
        sg = -1.0f;
        bs = 0.0f;
    } else {
        cell = n - 1;
        icode = 4;  // 2 hi - x  ->  2 ext - u
        sg = -1.0f;
        bs = 2.0f * ext;
    }
}

// Per-axis cell test (|rel_a| > cell size rejects, particle_system.hpp:120-126).
// AX = 0: implied by the radius test for accepted pairs (radius < every cell
//         size with an fp64 rounding margin), skipped;
// AX = 1: exact fp64 test on the pre-filter survivors only (radius ~ cell size:
//         the fp32 sphere pre-filter already bounds every axis);
// AX = 2: also in the fp32 pre-filter (radius clearly above a cell size).
// The pre-filter is a superset filter either way; only the fp64 test decides.
__device__ __forceinline__ int axis_mode(const Geo& g, double radius) {
    if (radius * (1.0 + 0x1p-40) < g.min_cs) return 0;
    return radius <= 1.01 * g.min_cs ? 1 : 2;
}

// The sweep. Must be called by all 32 lanes of a warp (valid = false for lanes
// without a particle). `pre_r` is the pre-filter radius (>= the operator's
// acceptance radius).
template <int DIM, bool ORDERED, int AX, bool ROWS, class Fn>
__device__ __forceinline__ void sweep_impl(const Geo& g, const float4* __restrict__ xl4, int k,
                                           bool valid, const double* xi, float pre_r,
                                           SweepSmem& sm, Fn& fn) {
    const DomainDev& d = g.dom;
    const int lane = threadIdx.x & 31;
    uint32_t* qe = sm.e + lane;
    int ci[3] = {0, 0, 0};
    AxisOpts ao[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) ao[a] = AxisOpts{0, 1, 1};
    float xli[3] = {0.f, 0.f, 0.f};
    bool done = !valid;
    if (valid) {
        decode_cell<DIM>(d, g.key[k], ci);
#pragma unroll
        for (int a = 0; a < DIM; ++a) ao[a] = axis_opts(d, a, ci[a]);
        const float4 p = xl4[k];
        xli[0] = p.x;
        xli[1] = p.y;
        xli[2] = p.z;
    }
    const float rl = pre_r * 1.001f + g.pre_abs;
    const float r2lim = rl * rl;
    // ROWS: the direct axis-0 options of one (o1, o2) are consecutive flat cells, so
    // their candidates form ONE contiguous slot range (slots are ordered by flat
    // cell) unless a periodic wrap splits them: one super-option per row instead of
    // up to three, mirror options after it as before. The odometer order (axis 0
    // fastest, direct cells then mirrors) is unchanged, so ORDERED sums stay
    // bitwise; at ~3 particles per cell (cfg3) the per-option setup and its two
    // dependent table loads were most of the sweep.
    const bool row = NAU_ROWS && ROWS && valid &&
                     (d.kind[0] != NAU_PERIODIC || (ci[0] >= 1 && ci[0] + 1 < d.cells[0]));
    const int cnt0 = row ? 1 + ao[0].cnt - ao[0].ndir : ao[0].cnt;
    const int n01 = cnt0 * (DIM > 1 ? ao[1].cnt : 1);
    const int ncombo = n01 * (DIM > 2 ? ao[2].cnt : 1);
    int idx = -1;  // position in the option sequence
    int t = 0, e = 0;
    uint32_t icode = 0;  // (c0 + 5 c1 + 25 c2) << kSlotBits
    float sg[3] = {1.f, 1.f, 1.f}, bq[3] = {0.f, 0.f, 0.f};  // rel_f = sg * u_j + bq
    int fill = 0;

    auto advance = [&]() {
        while (t >= e) {
            if (++idx == ncombo) {
                done = true;
                return;
            }
            const int combo = ORDERED ? idx : ((idx & 1) ? ncombo - 1 - (idx >> 1) : (idx >> 1));
            const int o0 = combo % cnt0;
            const int o1 = DIM > 1 ? (combo / cnt0) % ao[1].cnt : 0;
            const int o2 = DIM > 2 ? combo / n01 : 0;
            int cell, ic;
            float bs;
            int row_last = 0;  // cells merged after `cell` along axis 0
            if (row && o0 == 0) {
                cell = ci[0] + ao[0].lo_off;
                ic = 0;
                sg[0] = 1.0f;
                bs = 0.0f;
                row_last = ao[0].ndir - 1;
            } else {
                option_of(d, 0, ci[0], ao[0], row ? ao[0].ndir + o0 - 1 : o0, cell, ic, sg[0], bs);
            }
            int flat = cell;
            int code = ic;
            bq[0] = bs - xli[0];
            if (DIM > 1) {
                option_of(d, 1, ci[1], ao[1], o1, cell, ic, sg[1], bs);
                flat += d.cells[0] * cell;
                code += 5 * ic;
                bq[1] = bs - xli[1];
            }
            if (DIM > 2) {
                option_of(d, 2, ci[2], ao[2], o2, cell, ic, sg[2], bs);
                flat += d.cells[0] * d.cells[1] * cell;
                code += 25 * ic;
                bq[2] = bs - xli[2];
            }
            icode = (uint32_t)code << kSlotBits;
            t = g.cell_start[flat];
            e = row_last ? g.cell_start[flat + row_last] + g.cell_count[flat + row_last]
                         : t + g.cell_count[flat];
        }
    };
    if (!done) advance();

    // per-axis tests: see axis_mode (AX chosen warp-uniformly by sweep() below)
    constexpr bool axis_implied = AX == 0;
    auto test = [&](const float4 p) {
        const float r0 = fmaf(sg[0], p.x, bq[0]);
        bool rej = AX == 2 && fabsf(r0) > g.lim[0];
        float r2 = r0 * r0;
        if (DIM > 1) {
            const float r1 = fmaf(sg[1], p.y, bq[1]);
            rej |= AX == 2 && fabsf(r1) > g.lim[1];
            r2 = fmaf(r1, r1, r2);
        }
        if (DIM > 2) {
            const float r3 = fmaf(sg[2], p.z, bq[2]);
            rej |= AX == 2 && fabsf(r3) > g.lim[2];
            r2 = fmaf(r3, r3, r2);
        }
        return !(rej || r2 > r2lim);
    };

    // Ring FIFO per lane: entries [head, head + fill) (mod kQueue), oldest first.
    int head = 0;
    auto push = [&](uint32_t ent) {
        qe[((head + fill) & (kQueue - 1)) * 32] = ent;
        ++fill;
    };
    // Process the `steps` oldest entries of every lane (fewer if a lane has fewer).
    auto drain = [&](int steps) {
        __syncwarp();
        const int took = min(fill, steps);
        // software pipeline: the next entry's position gather is in flight while
        // the current pair is evaluated (profiles/r1_v5: the gather's latency was the
        // top stall of the drain)
        uint32_t ent_n = took > 0 ? qe[(head & (kQueue - 1)) * 32] : 0u;
        double4 pj_n = took > 0 ? ld256(g.p4 + (ent_n & ((1u << kSlotBits) - 1))) : make_double4(0, 0, 0, 0);
        for (int s = 0; s < steps; ++s) {
            const uint32_t ent = ent_n;
            const double4 pj = pj_n;  // one 32-byte sector per pair
            if (s + 1 < took) {
                ent_n = qe[((head + s + 1) & (kQueue - 1)) * 32];
                pj_n = ld256(g.p4 + (ent_n & ((1u << kSlotBits) - 1)));
            }
            if (s < fill) {
                const int j = (int)(ent & ((1u << kSlotBits) - 1));
                const int c = (int)(ent >> kSlotBits);
                const double xj[3] = {pj.x, pj.y, pj.z};
                double rel[3] = {0.0, 0.0, 0.0};
                bool ok = true;
                int mask = 0;
                if (c == 0) {  // direct image in every axis: img = xj + 0.0
#pragma unroll
                    for (int a = 0; a < DIM; ++a) {
                        rel[a] = (xj[a] + 0.0) - xi[a];
                        ok &= axis_implied || !(fabs(rel[a]) > g.img[a].cs);
                    }
                } else {
                    const int cc[3] = {c % 5, (c / 5) % 5, c / 25};
#pragma unroll
                    for (int a = 0; a < DIM; ++a) {
                        const int ca = cc[a];
                        const double r = image_of(g.img[a], xj[a], ca) - xi[a];
                        ok &= axis_implied || !(fabs(r) > g.img[a].cs);
                        rel[a] = r;
                        mask |= (ca >= 3) << a;
                    }
                }
                if (ok) fn(j, rel, mask);
            }
        }
        head = (head + took) & (kQueue - 1);
        fill -= took;
        __syncwarp();
    };

    while (true) {
        if (!done) {
            const int stop = min(e, t + kChunk);
            // eight / four independent loads in flight per lane
            for (; t + 8 <= stop; t += 8) {
                float4 p[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) p[u] = xl4[t + u];
                bool acc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[u] = test(p[u]);
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (acc[u]) push((uint32_t)(t + u) | icode);
            }
            for (; t + 4 <= stop; t += 4) {
                const float4 p0 = xl4[t], p1 = xl4[t + 1], p2 = xl4[t + 2], p3 = xl4[t + 3];
                const bool a0 = test(p0), a1 = test(p1), a2 = test(p2), a3 = test(p3);
                if (a0) push((uint32_t)t | icode);
                if (a1) push((uint32_t)(t + 1) | icode);
                if (a2) push((uint32_t)(t + 2) | icode);
                if (a3) push((uint32_t)(t + 3) | icode);
            }
            for (; t < stop; ++t)
                if (test(xl4[t])) push((uint32_t)t | icode);
            if (t >= e) advance();
        }
        // Partial drains of the oldest kChunk entries keep every drain step busy for
        // all lanes holding >= kChunk entries (mean/max-fill occupancy otherwise).
        if (__any_sync(0xffffffffu, fill > kQueue - kChunk)) drain(kChunk);
        if (!__any_sync(0xffffffffu, !done)) {
            drain(__reduce_max_sync(0xffffffffu, fill));
            break;
        }
    }
}

// ---- per-step neighbour lists (used by the two-pass WCSPH deck) --------------
// The density and momentum passes of a step walk the same candidates, so the
// scan phase runs once (k_nlist) and stores the pre-filter survivors, in
// candidate order, as CHUNK RECORDS: one (base, mask) pair of u32 per block of
// 32 consecutive candidate slots with at least one survivor — base = first slot
// | image code << kSlotBits, bit b of mask = slot base + b survives. Record r of
// slot k lives at rec[((k/32)*cap + r)*32 + k%32] (coalesced 256 B per warp).
// The consumers expand the masks on the fly (consume_list), so they visit the
// same candidates in the same order as the sweep => same sums. A record costs
// one 8-byte store per block instead of one store sequence per survivor (~6
// per block at the BASELINE decks), and the list is ~half the bytes.
// AXIS = the fp32 pre-filter's per-axis test (axis_mode == 2).
//
// Record store: address = lane base + r * 256 B in one wide multiply-add (the
// compiler otherwise rebuilds the 64-bit address from the kernel parameter).
__device__ __forceinline__ void st_rec(uint2* base, unsigned r, uint32_t v, uint32_t m) {
    asm volatile(
        "{\n\t.reg .u64 a;\n\t"
        "mad.wide.u32 a, %1, 256, %0;\n\t"
        "st.global.v2.u32 [a], {%2, %3};\n\t}"
        :
        : "l"(base), "r"(r), "r"(v), "r"(m)
        : "memory");
}

// Emit one 32-candidate block's survivors (m != 0) as a record.
__device__ __forceinline__ void emit_rec(uint2* rec, int cap, int& nrec, int& cnt, uint32_t v,
                                         uint32_t m) {
    if (m) {
        if (nrec < cap) st_rec(rec, (unsigned)nrec, v, m);
        ++nrec;
        cnt += __popc(m);
    }
}

// emit(v, m) receives every 32-candidate block in candidate order: v = first
// slot | image code << kSlotBits, m = survivor mask (possibly 0).
template <int DIM, bool ORDERED, bool AXIS, class Emit>
__device__ __forceinline__ void build_list(const Geo& g, const float4* __restrict__ xl4, int k,
                                           float pre_r, Emit&& emit) {
    const DomainDev& d = g.dom;
    int ci[3] = {0, 0, 0};
    decode_cell<DIM>(d, g.key[k], ci);
    AxisOpts ao[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) ao[a] = AxisOpts{0, 1, 1};
#pragma unroll
    for (int a = 0; a < DIM; ++a) ao[a] = axis_opts(d, a, ci[a]);
    const float4 pi = xl4[k];
    const float xli[3] = {pi.x, pi.y, pi.z};
    const float rl = pre_r * 1.001f + g.pre_abs;
    const float r2lim = rl * rl;
    const int n01 = ao[0].cnt * (DIM > 1 ? ao[1].cnt : 1);
    const int ncombo = n01 * (DIM > 2 ? ao[2].cnt : 1);
    
    for (int idx = 0; idx < ncombo; ++idx) {
        const int combo = ORDERED ? idx : ((idx & 1) ? ncombo - 1 - (idx >> 1) : (idx >> 1));
        const int o0 = combo % ao[0].cnt;
        const int o1 = DIM > 1 ? (combo / ao[0].cnt) % ao[1].cnt : 0;
        const int o2 = DIM > 2 ? combo / n01 : 0;
        int cell, ic, flat, code;
        float sg[3] = {1.f, 1.f, 1.f}, bq[3] = {0.f, 0.f, 0.f}, bs;
        option_of(d, 0, ci[0], ao[0], o0, cell, ic, sg[0], bs);
        flat = cell;
        code = ic;
        bq[0] = bs - xli[0];
        if (DIM > 1) {
            option_of(d, 1, ci[1], ao[1], o1, cell, ic, sg[1], bs);
            flat += d.cells[0] * cell;
            code += 5 * ic;
            bq[1] = bs - xli[1];
        }
        if (DIM > 2) {
            option_of(d, 2, ci[2], ao[2], o2, cell, ic, sg[2], bs);
            flat += d.cells[0] * d.cells[1] * cell;
            code += 25 * ic;
            bq[2] = bs - xli[2];
        }
        const uint32_t icode = (uint32_t)code << kSlotBits;
        const int s = g.cell_start[flat], e = s + g.cell_count[flat];
        auto test = [&](const float4 p) {
            const float r0 = fmaf(sg[0], p.x, bq[0]);
            bool rej = AXIS && fabsf(r0) > g.lim[0];
            float r2 = r0 * r0;
            if (DIM > 1) {
                const float r1 = fmaf(sg[1], p.y, bq[1]);
                rej |= AXIS && fabsf(r1) > g.lim[1];
                r2 = fmaf(r1, r1, r2);
            }
            if (DIM > 2) {
                const float r3 = fmaf(sg[2], p.z, bq[2]);
                rej |= AXIS && fabsf(r3) > g.lim[2];
                r2 = fmaf(r3, r3, r2);
            }
            return !(rej || r2 > r2lim);
        };
        // Blocks of 32 candidates: the tests set a bit mask (eight loads in flight,
        // tail loads clamped and masked off), stored as one record.
        for (int t = s; t < e; t += 32) {
            const int nb = min(32, e - t);
            uint32_t m = 0;
#pragma unroll
            for (int u0 = 0; u0 < 32; u0 += 8) {
                if (u0 + 8 <= nb) {
                    const float4* q = xl4 + t + u0;
                    float4 p[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) p[u] = q[u];
#pragma unroll
                    for (int u = 0; u < 8; ++u) m |= (uint32_t)test(p[u]) << (u0 + u);
                } else if (u0 < nb) {  // tail: clamped loads, masked below
                    float4 p[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) p[u] = xl4[min(t + u0 + u, e - 1)];
#pragma unroll
                    for (int u = 0; u < 8; ++u) m |= (uint32_t)test(p[u]) << (u0 + u);
                }
            }
            if (nb < 32) m &= (1u << nb) - 1u;
            emit((uint32_t)t | icode, m);
        }
    }
}

// Evaluate fn(j, rel, mask, payload) over a slot's list, payload = load(j) (the
// pair's per-neighbour operands). Lane-private loop, software-pipelined: the
// position / payload gathers run 2 pairs ahead of the arithmetic and the list
// entries (expanded from the chunk records, loaded two records ahead) 4-5 pairs ahead, in buffers with fixed roles (loop unrolled: no
// register rotation; profiles/r1_nl_*: the rotating version spent ~30 moves
// per pair and the one-ahead version stalled on long_scoreboard).
// AXIS = the exact fp64 per-axis test. FAST drops the reference's "+ 0.0" of the
// direct image (it only normalises -0.0; FAST mode does not promise bitwise).
// NAU_GEN_SELECT: record switch by selects + a predicated load instead of a
// divergent branch (measured: cfg1 -3%, cfg2 even)
#ifndef NAU_GEN_SELECT
#define NAU_GEN_SELECT 1
#endif
#ifndef NAU_LIST_PF
#define NAU_LIST_PF 4
#endif
template <int DIM, bool AXIS, bool FAST, int NB, bool IMG = true, class Load, class Fn>
__device__ __forceinline__ void consume_list(const Geo& g, const uint2* __restrict__ rec, int cnt,
                                             const double* xi, Load&& load, Fn&& fn) {
    constexpr uint32_t kM = (1u << kSlotBits) - 1;
    using P = decltype(load(0));
    struct Buf {
        uint32_t ent;
        double4 p;
        P pl;
    };
    // entry generator: entries are requested in increasing order, once each
    // (records loaded two ahead: sparse records switch every 1-2 entries)
    uint2 cur = rec[0], n1 = rec[32], n2 = rec[64];
    int r = 0;
    auto gen = [&]() -> uint32_t {
#if NAU_GEN_SELECT
        const bool sw = cur.y == 0;
        cur.x = sw ? n1.x : cur.x;
        cur.y = sw ? n1.y : cur.y;
        n1.x = sw ? n2.x : n1.x;
        n1.y = sw ? n2.y : n1.y;
        r += sw;
        if (sw) {
            n2 = rec[(r + 2) * 32];
#if NAU_LIST_PF
            // sparse records switch every 1-2 entries and stream from DRAM: pull the
            // row NAU_LIST_PF switches ahead toward L1 (slack rows cover the overrun)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(rec + (r + 2 + NAU_LIST_PF) * 32));
#endif
        }
#else
        if (cur.y == 0) {
            cur = n1;
            n1 = n2;
            ++r;
            n2 = rec[(r + 2) * 32];  // at most record `count` + 1: the slack rows
        }
#endif
        const uint32_t b = (uint32_t)(__ffs(cur.y) - 1);
        cur.y &= cur.y - 1;
        return cur.x + b;
    };
    auto nx = [&](int s) { return s < cnt ? gen() : 0u; };
    auto fetch = [&](Buf& b, uint32_t ent) {
        b.ent = ent;
        b.p = ld256(g.p4 + (ent & kM));
        b.pl = load((int)(ent & kM));
    };
    auto process = [&](const Buf& b) {
        const int j = (int)(b.ent & kM);
        const int c = (int)(b.ent >> kSlotBits);
        const double xj[3] = {b.p.x, b.p.y, b.p.z};
        double rel[3] = {0.0, 0.0, 0.0};
        bool ok = true;
        int mask = 0;
        if (!IMG || c == 0) {  // !IMG: no periodic / symmetric axis, every code is 0
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                rel[a] = FAST ? xj[a] - xi[a] : (xj[a] + 0.0) - xi[a];
                ok &= !AXIS || !(fabs(rel[a]) > g.img[a].cs);
            }
        } else {
            const int cc[3] = {c % 5, (c / 5) % 5, c / 25};
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                const double r = image_of(g.img[a], xj[a], cc[a]) - xi[a];
                ok &= !AXIS || !(fabs(r) > g.img[a].cs);
                rel[a] = r;
                mask |= (cc[a] >= 3) << a;
            }
        }
        if (ok) fn(j, rel, mask, b.pl);
    };
    if constexpr (NB == 3) {
        Buf A, B, C;
        const uint32_t e0 = nx(0), e1 = nx(1);
        uint32_t eC = nx(2), eA = nx(3), eB = nx(4);
        fetch(A, e0);
        fetch(B, e1);
        for (int s = 0; s < cnt; s += 3) {
            fetch(C, eC);  // pair s + 2
            eC = nx(s + 5);
            process(A);  // pair s
            fetch(A, eA);  // pair s + 3
            eA = nx(s + 6);
            if (s + 1 < cnt) process(B);
            fetch(B, eB);  // pair s + 4
            eB = nx(s + 7);
            if (s + 2 < cnt) process(C);
        }
    } else {  // two buffers: gathers one pair ahead (register-lean)
        Buf A, B;
        const uint32_t e0 = nx(0);
        uint32_t eB = nx(1), eA = nx(2);
        fetch(A, e0);
        for (int s = 0; s < cnt; s += 2) {
            fetch(B, eB);  // pair s + 1
            eB = nx(s + 3);
            process(A);  // pair s
            fetch(A, eA);  // pair s + 2
            eA = nx(s + 4);
            if (s + 1 < cnt) process(B);
        }
    }
}

struct NoPayload {};
struct NoLoad {
    __device__ __forceinline__ NoPayload operator()(int) const { return NoPayload{}; }
};
// Per-neighbour 32-byte payload (e.g. the WCSPH momentum pass's (v, p/rho^2)).
struct Ld256 {
    const double4* p;
    __device__ __forceinline__ double4 operator()(int j) const { return ld256(p + j); }
};

// Entry point: `radius` is the lane's acceptance radius (fp64); the per-axis
// mode is the warp's maximum of axis_mode (BASELINE decks: radius = cell size,
// mode 1).
// ROWS (default: ORDERED, where it keeps the order) merges each stencil row's direct
// cells into one slot range; unordered callers opt in only where the summation
// order is free (FAST SPH sweeps must match the lists' order).
template <int DIM, bool ORDERED, bool ROWS = ORDERED, class Fn>
__device__ __forceinline__ void sweep(const Geo& g, const float4* __restrict__ xl4, int k,
                                      bool valid, const double* xi, double radius, Fn&& fn) {
    __shared__ SweepSmem smem[kSweepThreads / 32];
    SweepSmem& sm = smem[threadIdx.x >> 5];
    const float pre_r = (float)radius;
    const int ax = __reduce_max_sync(0xffffffffu, valid ? axis_mode(g, radius) : 0);
    if (ax == 0)
        sweep_impl<DIM, ORDERED, 0, ROWS>(g, xl4, k, valid, xi, pre_r, sm, fn);
    else if (ax == 1)
        sweep_impl<DIM, ORDERED, 1, ROWS>(g, xl4, k, valid, xi, pre_r, sm, fn);
    else
        sweep_impl<DIM, ORDERED, 2, ROWS>(g, xl4, k, valid, xi, pre_r, sm, fn);
}

// ---- half-precision pre-filter for the list build ------------------------------
// Isotropic cells, radius <= 1.5 cell sizes, every particle inside its cell's
// box (else the fp32 build_list runs). Each particle's coordinates relative to
// its cell origin, in cell units, are stored as fp16 in a cell-padded layout
// (every cell's range starts at a multiple of 32, pads = +inf), so four 128-bit
// loads bring a 32-candidate block per axis and HFMA2 tests two candidates per
// instruction: rel_a = sg * h_j + (off_a - h_i), off_a = the option's cell offset
// (-1, 0, 1; mirror-low 0 with sg = -1; mirror-high 2 with sg = -1).
// Within a block the halves are INTERLEAVED: half2 word k holds candidates k and
// k + 16, so d = r2 - lim has its two sign bits at 15 and 31 and
// (d & 0x80008000) >> (15 - k) drops them on mask bits k and k + 16 — two integer
// instructions per word instead of a compare-and-pack sequence.
// Error bound (cell units): |h| < 1 rounds to 2^-12, off - h_i (|.| <= 2) to
// 2^-11, the HFMA2 result (|rel| <= 2 near the threshold) to 2^-11: |rel error|
// <= 1.25 * 2^-10; |rel| <= rho => sqrt(r2) <= rho + 0.0022 before the three
// roundings of d = ((rx^2 - lim) + ry^2) + rz^2 (|d| < 4: <= 2^-10 each):
// lim = (rho + 0.0022)^2 + 0.003, rounded up to fp16, makes d < 0 for every
// candidate within rho. A superset filter again; the fp64 test decides. Pads
// (+inf) give d = +inf: never set.
struct HalfGrid {
    const __half* h[3];  // padded per-axis coordinates
    const int* pstart;   // padded start of each cell (multiple of 8)
    const int* escaped;  // set by the build when some particle lies outside its cell box
    float rho;           // radius / cell size
    int on;              // host-side eligibility (isotropic, rho <= 1.5)
};

__device__ __forceinline__ float half_offset(const AxisOpts& ao, int ci, int o, float& sg,
                                             int& icode, int& cell, int n, int kind) {
    if (o < ao.ndir) {
        const int off = ao.lo_off + o;
        int c = ci + off;
        icode = 0;
        if (c < 0) {
            c += n;
            icode = 2;
        } else if (c >= n) {
            c -= n;
            icode = 1;
        }
        cell = c;
        sg = 1.0f;
        return (float)off;
    }
    sg = -1.0f;
    if (o == ao.ndir && ci == 0) {
        cell = 0;
        icode = 3;
        return 0.0f;
    }
    cell = n - 1;
    icode = 4;
    return 2.0f;
}

// NP (1 or 2) particles of ONE cell share the option sequence and every
// coordinate load; each gets its own mask: emit(v, m) with m[NP]. UNI (NP = 2):
// only m[0] = the union of both masks is formed — min(d0, d1) < 0 is one sign
// test per candidate instead of two.
template <int DIM, bool ORDERED, int NP, bool UNI = false, class Emit>
__device__ __forceinline__ void half_scan(const Geo& g, const HalfGrid& hg, const int* ks,
                                          Emit&& emit) {
    const DomainDev& d = g.dom;
    const int flat_i = g.key[ks[0]];
    int ci[3] = {0, 0, 0};
    decode_cell<DIM>(d, flat_i, ci);
    AxisOpts ao[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) ao[a] = AxisOpts{0, 1, 1};
#pragma unroll
    for (int a = 0; a < DIM; ++a) ao[a] = axis_opts(d, a, ci[a]);
    float hi[NP][3];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        const int rk = ks[p] - g.cell_start[flat_i];  // rank in the cell -> interleaved position
        const int pk = hg.pstart[flat_i] + (rk & ~31) + 2 * (rk & 15) + ((rk >> 4) & 1);
#pragma unroll
        for (int a = 0; a < 3; ++a) hi[p][a] = a < DIM ? __half2float(hg.h[a][pk]) : 0.f;
    }
    const float rl = hg.rho + 0.0022f;
    const __half2 nlim2 = __hneg2(__half2half2(__float2half_ru(fmaf(rl, rl, 0.003f))));
    const int n01 = ao[0].cnt * (DIM > 1 ? ao[1].cnt : 1);
    const int ncombo = n01 * (DIM > 2 ? ao[2].cnt : 1);
    // option setup; the next option's cell-table reads are issued one option
    // ahead (a lane's 27 options are otherwise a chain of dependent latencies)
    struct Opt {
        __half2 sg2[3], bq2[NP][3];
        uint32_t icode;
        int s, ns, ps;
    };
    // option digits without integer divisions: an odometer counting up from the first
    // option and (balanced order) one counting down from the last, used alternately —
    // setup(idx) is called for idx = 0, 1, 2, ... exactly once each
    int up[3] = {0, 0, 0};
    int dn[3] = {ao[0].cnt - 1, DIM > 1 ? ao[1].cnt - 1 : 0, DIM > 2 ? ao[2].cnt - 1 : 0};
    auto setup = [&](int idx, Opt& o) {
        int oo[3];
        if (ORDERED || !(idx & 1)) {
#pragma unroll
            for (int a = 0; a < 3; ++a) oo[a] = up[a];
            if (++up[0] == ao[0].cnt) {
                up[0] = 0;
                if (DIM > 1 && ++up[1] == ao[1].cnt) {
                    up[1] = 0;
                    ++up[2];
                }
            }
        } else {
#pragma unroll
            for (int a = 0; a < 3; ++a) oo[a] = dn[a];
            if (--dn[0] < 0) {
                dn[0] = ao[0].cnt - 1;
                if (DIM > 1 && --dn[1] < 0) {
                    dn[1] = ao[1].cnt - 1;
                    --dn[2];
                }
            }
        }
        int flat = 0, code = 0, stride = 1, scode = 1;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            float sg;
            int ic, cell;
            const float off = half_offset(ao[a], ci[a], oo[a], sg, ic, cell, d.cells[a], d.kind[a]);
            o.sg2[a] = __float2half2_rn(sg);
#pragma unroll
            for (int p = 0; p < NP; ++p) o.bq2[p][a] = __float2half2_rn(off - hi[p][a]);
            flat += stride * cell;
            code += scode * ic;
            stride *= d.cells[a];
            scode *= 5;
        }
        o.icode = (uint32_t)code << kSlotBits;
        o.s = g.cell_start[flat];
        o.ns = g.cell_count[flat];
        o.ps = hg.pstart[flat];
    };
    Opt nxt;
    setup(0, nxt);
    for (int idx = 0; idx < ncombo; ++idx) {
        const Opt o = nxt;
        if (idx + 1 < ncombo) setup(idx + 1, nxt);
        for (int q0 = 0; q0 < o.ns; q0 += 32) {
            // the whole 32-slot block of each axis up front (cells are padded
            // to 32 slots with +inf)
            uint4 hv[4][3];
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int a = 0; a < DIM; ++a)
                    hv[u][a] = *reinterpret_cast<const uint4*>(hg.h[a] + o.ps + q0 + 8 * u);
            uint32_t m[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) m[p] = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t* w[3] = {&hv[u][0].x, &hv[u][1].x, &hv[u][2].x};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int kw = 4 * u + q;  // word kw: candidates kw, kw + 16
                    __half2 dp[NP];
#pragma unroll
                    for (int p = 0; p < NP; ++p) {
                        __half2 dd = nlim2;
#pragma unroll
                        for (int a = 0; a < DIM; ++a) {
                            const __half2 x2 = *reinterpret_cast<const __half2*>(w[a] + q);
                            const __half2 r = __hfma2(o.sg2[a], x2, o.bq2[p][a]);
                            dd = __hfma2(r, r, dd);
                        }
                        dp[p] = dd;
                    }
                    // the two sign bits enter at bits 15 / 31 and every later word rotates
                    // them one place down: word kw ends at bits kw, kw + 16 (a rotate and
                    // one bit-select per word instead of mask, shift, add)
                    auto push = [](uint32_t m, const __half2& dd) {
                        m = __funnelshift_r(m, m, 1);
                        uint32_t r;  // (m & ~K) | (bits & K), K = the sign bits: one LOP3
                        asm("lop3.b32 %0, %1, %2, 0x80008000, 0xD8;"
                            : "=r"(r)
                            : "r"(m), "r"(*reinterpret_cast<const uint32_t*>(&dd)));
                        return r;
                    };
                    if constexpr (UNI && NP == 2) {
                        m[0] = push(m[0], __hmin2(dp[0], dp[1]));
                    } else {
#pragma unroll
                        for (int p = 0; p < NP; ++p) m[p] = push(m[p], dp[p]);
                    }
                }
            }
            if (q0 == 0 && idx + 1 < ncombo) {
                // pull the next option's coordinate lines into L1 while this option
                // is expanded (an L1 miss on a block's loads stalls the whole block)
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    const __half* pp = hg.h[a] + nxt.ps;
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(pp));
                    if (nxt.ns > 56) asm volatile("prefetch.global.L1 [%0];" ::"l"(pp + 64));
                }
            }
            if (o.ns - q0 < 32)
#pragma unroll
                for (int p = 0; p < (UNI ? 1 : NP); ++p) m[p] &= (1u << (o.ns - q0)) - 1u;
            emit((uint32_t)(o.s + q0) | o.icode, m);
        }
    }
}

template <int DIM, bool ORDERED, class Emit>
__device__ __forceinline__ void build_list_half(const Geo& g, const HalfGrid& hg, int k,
                                                Emit&& emit) {
    half_scan<DIM, ORDERED, 1>(g, hg, &k, [&](uint32_t v, const uint32_t* m) { emit(v, m[0]); });
}

struct NList {  // per-step neighbour lists (k_nlist in cells.cu): chunk records
    const uint32_t* e;  // uint2 records (see st_rec), viewed as u32
    const int* count;   // pairs (expanded entries) per slot
    int cap;            // records per slot
    const int* split = nullptr;  // paired lists: first record of the second particle, or -1
};

// Record 0 of slot k, in uint2 units (record r is 32 r further).
__device__ __forceinline__ size_t nlist_base(int k, int cap) {
    return (size_t)(k >> 5) * cap * 32 + (k & 31);
}

// fn(j, rel, mask, load(j)) over k's neighbour candidates: from the step's list
// (LIST) or a fresh sweep. Both visit the same candidates in the same order.
// FAST (the FAST-mode kernels, whose smoothing kernels vanish at the support
// radius): the per-axis test is skipped whenever radius <= every cell size —
// a pair it would reject has |rel| > cell size >= radius up to one rounding,
// i.e. q = 2 where W and dW/dq are zero.
// IMG = false: the domain has no periodic or symmetric axis (host-checked), so
// every list entry is a direct image and the image branch compiles away.
template <int DIM, bool ORDERED, bool LIST, bool FAST = false, int NB = 3, bool IMG = true,
          class Load, class Fn>
__device__ __forceinline__ void for_neighbors(const Geo& g, const float4* __restrict__ xl4,
                                              const NList& nl, int k, bool valid,
                                              const double* xi, double radius, Load&& load,
                                              Fn&& fn) {
    if constexpr (LIST) {
        if (!valid) return;
        const uint2* lst = reinterpret_cast<const uint2*>(nl.e) + nlist_base(k, nl.cap);
        const int cnt = nl.count[k];
        const bool axis = FAST ? !(radius <= g.min_cs) : axis_mode(g, radius) != 0;
        if (!axis)
            consume_list<DIM, false, FAST, NB, IMG>(g, lst, cnt, xi, load, fn);
        else
            consume_list<DIM, true, FAST, NB, IMG>(g, lst, cnt, xi, load, fn);
    } else {
        sweep<DIM, ORDERED>(g, xl4, k, valid, xi, radius,
                            [&](int j, const double* rel, int mask) { fn(j, rel, mask, load(j)); });
    }
}

// ---- paired lists (FAST WCSPH deck) -------------------------------------------

// Thread t owns slots 2t and 2t+1. When both sit in one cell (all but ~1 in 64
// pairs at the BASELINE decks) they share the option sequence, and one 8-byte
// record per 32-candidate block carries the UNION of their survivor masks. The
// consumer evaluates every gathered neighbour (position + payload) for both
// particles as two independent chains: the masks are superset pre-filters, so a
// candidate only the other particle kept lies beyond the support radius and its
// contribution is clamped to zero like any other false survivor's. The gathers,
// which bound the per-slot consumers in L1, are shared, and no per-particle bit
// is stored or decoded. Pairs that straddle a cell boundary (or a thread whose
// second slot does not exist) store the first particle's records, then the
// second's; `split` = the first record of the second particle (-1: shared
// records), and a particle skips the records it does not own. Each particle
// still visits its own candidates in the sweep's order: the same sums as the
// per-slot lists. Two terminator records (own slot, one bit) follow a thread's
// last record so the consumer's gathers may run two entries past the end.
constexpr int kPairTail = 2;
#ifndef NAU_REC_PF
#define NAU_REC_PF 4  // record prefetch distance of the momentum consumer
#endif
constexpr int kPairSlackRows = 1 + NAU_REC_PF;  // rows a consumer may touch past a group's last

// Records of a thread pair: emit(v, union mask) per block as in build_list;
// mark() runs between the first particle's records and the second's when they
// are not shared.
template <int DIM, class Emit, class Mark>
__device__ __forceinline__ void build_pair_list(const Geo& g, const float4* __restrict__ xl4,
                                                const HalfGrid& hg, double radius, int k0,
                                                bool has1, Emit&& emit, Mark&& mark) {
    const int k1 = k0 + 1;
    if (hg.on && *hg.escaped == 0) {
        // one pass of the same code for every lane: a particle without a partner in its
        // cell is scanned as the pair (k0, k0), so a warp with a straddling pair pays that
        // pair's second scan only (once a flow has dissolved the lattice about every
        // second warp holds one)
        const bool shared = has1 && g.key[k0] == g.key[k1];
        const int ks[2] = {k0, shared ? k1 : k0};
        half_scan<DIM, false, 2, true>(g, hg, ks,
                                       [&](uint32_t v, const uint32_t* m) { emit(v, m[0]); });
        if (!shared) {
            mark();
            if (has1) build_list_half<DIM, false>(g, hg, k1, emit);
        }
        return;
    }
    const float pre_r = (float)radius;
    auto one = [&](int k) {
        if (axis_mode(g, radius) < 2)
            build_list<DIM, false, false>(g, xl4, k, pre_r, emit);
        else
            build_list<DIM, false, true>(g, xl4, k, pre_r, emit);
    };
    one(k0);
    mark();
    if (has1) one(k1);
}

// fn(j, xj_image, image_mask, dead0, dead1, payload) over the thread's entries;
// dead_p = ~0 when particle p does not own the entry's record (else 0): the
// caller ORs it into the word that zeroes the contribution. IMG = false: no
// periodic / symmetric axis. Entries two past the end are gathered (terminator
// records) but not evaluated.
// PF > 0: each record switch also pulls the row PF switches ahead toward L1 (the
// records stream from DRAM once; measured at cfg2: momentum -2.4%, density +2.7%).
template <int DIM, bool IMG, int PF = 0, class Load, class Fn>
__device__ __forceinline__ void consume_pairs(const Geo& g, const uint2* __restrict__ rec,
                                              int cnt, int split, Load&& load, Fn&& fn) {
    constexpr uint32_t kM = (1u << kSlotBits) - 1;
    using P = decltype(load(0));
    struct Buf {
        uint32_t ent;
        int o0, o1;  // record index relative to the particles' ownership bounds
        double4 p;
        P pl;
    };
    uint2 cur = rec[0], n1 = rec[32];
    const uint2* nx = rec + 64;
    // particle 0 owns records r < split (o0 < 0), particle 1 records r >= split
    // (o1 >= 0); shared records: both always
    int o0 = split < 0 ? -(1 << 30) : -split, o1 = split < 0 ? 0 : -split;
    auto fetch = [&](Buf& b) {
        const bool sw = cur.y == 0;
        cur.x = sw ? n1.x : cur.x;
        cur.y = sw ? n1.y : cur.y;
        o0 += sw;
        o1 += sw;
        if (sw) {
            n1 = *nx;  // at most two records past the terminators: inside the slack row
            if constexpr (PF > 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(nx + 32 * PF));
            nx += 32;
        }
        const uint32_t bit = (uint32_t)(__ffs(cur.y) - 1);
        cur.y &= cur.y - 1;
        b.ent = cur.x + bit;
        b.o0 = o0;
        b.o1 = o1;
        // !IMG: every image code is 0, the entry is the slot
#ifdef NAU_PROBE_L1HIT  // timing probe only (wrong results): every gather hits L1
        const uint32_t slot = b.ent & 1023u;
#else
        const uint32_t slot = IMG ? (b.ent & kM) : b.ent;
#endif
        b.p = ld256(g.p4 + slot);
        b.pl = load((int)slot);
    };
    auto process = [&](const Buf& b) {
        const int j = (int)(IMG ? (b.ent & kM) : b.ent);
        double xj[3] = {b.p.x, b.p.y, b.p.z};
        int mask = 0;
        if constexpr (IMG) {
            const int c = (int)(b.ent >> kSlotBits);
            if (c != 0) {
                const int cc[3] = {c % 5, (c / 5) % 5, c / 25};
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    xj[a] = image_of(g.img[a], xj[a], cc[a]);
                    mask |= (cc[a] >= 3) << a;
                }
            }
        }
        fn(j, xj, mask, ~(unsigned)(b.o0 >> 31), (unsigned)(b.o1 >> 31), b.pl);
    };
    Buf A, B;
    fetch(A);
    fetch(B);
    int s = 0;
    for (; s + 2 <= cnt; s += 2) {
        process(A);
        fetch(A);
        process(B);
        fetch(B);
    }
    if (s < cnt) process(A);
}

}  // namespace nau
