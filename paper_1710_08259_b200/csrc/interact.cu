// interact.cu — the interaction-operator evaluators of kOps[] (src/interactions.cpp:259-269)
// as whole-field sm_100a kernels.
//
// One thread owns one particle slot k (cell order) and walks the 3^d stencil
// in the reference's candidate order (particle_system.hpp:59-138), so every
// accumulator sums in the same order as interact() (interactions.hpp:29-36).
// Consecutive threads are consecutive particles of the same / adjacent cells,
// so a warp's candidate loads hit the same few cache lines (L1 broadcast).
// This TU is compiled with -fmad=false: with IEEE div/sqrt the results are
// bitwise identical to the reference wherever no libm transcendental (pow/log)
// enters (Hertz DEM, gravity, Tait EOS are tolerance-checked).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "nau_internal.cuh"
#include "sweep.cuh"

namespace nau {

namespace {

constexpr int kThreads = kSweepThreads;

struct SphArgs {
    Geo g;
    const float4* xl;
    Opd A, m, rho, R;
    double* out;
    int arows, acols;
    int kdim;
    DevErr* err;
    NList nl;  // the cell build's neighbour list (uniform radius), or e == nullptr
};

template <int DIM, int OP, int KF, int AC, bool LIST>
__global__ void __launch_bounds__(kThreads) k_sph(const __grid_constant__ SphArgs a) {
    const Geo& g = a.g;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    bool valid = k < *g.nact;
    const long n = g.n;
    const int kk = valid ? k : 0;
    double xi[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int d = 0; d < DIM; ++d) xi[d] = g.x[d * n + kk];
    // sph_context (interactions.cpp:22-27)
    const double radius = a.R.at(0, kk, n);
    if (valid && !(radius > 0.0)) {
        latch_error(a.err, 1, kMsgRadius, g.orig[k]);
        valid = false;
    }
    const double h = 0.5 * radius;
    const double alpha = kernel_alpha<KF>(a.kdim, h);
    // components of A held per particle: S any shape, D00/A a d-vector, G11/L0 scalar
    const int ac = OP == NAU_OP_SPH_S ? (AC == 1 ? 1 : a.arows * a.acols)
                                      : ((OP == NAU_OP_SPH_D00 || OP == NAU_OP_SPH_A) ? DIM : 1);
    double a_i[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) a_i[c] = (c < ac) ? a.A.at(c, kk, n) : 0.0;
    double rho_i = 1.0;
    if (OP == NAU_OP_SPH_G11 || OP == NAU_OP_SPH_A) {
        rho_i = a.rho.at(0, kk, n);
        if (valid && rho_i == 0.0) {
            latch_error(a.err, 1, kMsgZeroDensity, g.orig[k]);
            valid = false;
        }
    }
    double acc[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) acc[c] = 0.0;
    const int my_orig = g.orig[kk];

    for_neighbors<DIM, true, LIST>(g, a.xl, a.nl, k, valid, xi, radius, NoLoad{},
               [&](int j, const double* rel, int mask, NoPayload) {
        const double dist = norm_rel<DIM>(rel);
        if (OP == NAU_OP_SPH_S) {  // interactions.cpp:40-58
            if (dist > radius) return;
            const double w = kernel_value<KF>(alpha, h, dist);
            if (w == 0.0) return;
            const double rho_j = a.rho.at(0, j, n);
            if (rho_j == 0.0) {
                latch_error(a.err, 1, kMsgZeroDensity, g.orig[j]);
                return;
            }
            const double m_j = a.m.at(0, j, n);
            const double s = m_j / rho_j * w;
#pragma unroll
            for (int c = 0; c < (AC == 1 ? 1 : 9); ++c)
                if (c < ac)
                    acc[c] = acc[c] + mirror_comp(a.A.at(c, j, n), c, a.arows, a.acols, mask, DIM) * s;
        } else if (OP == NAU_OP_SPH_D00) {  // interactions.cpp:60-79
            if (dist <= 0.0 || dist > radius) return;
            const double rho_j = a.rho.at(0, j, n);
            if (rho_j == 0.0) {
                latch_error(a.err, 1, kMsgZeroDensity, g.orig[j]);
                return;
            }
            const double m_j = a.m.at(0, j, n);
            const double sc = kernel_grad_scale<KF>(alpha, h, dist);
            double dt = (mirror_comp(a.A.at(0, j, n), 0, DIM, 1, mask, DIM) - a_i[0]) * (rel[0] * sc);
#pragma unroll
            for (int d = 1; d < DIM; ++d)
                dt = dt + (mirror_comp(a.A.at(d, j, n), d, DIM, 1, mask, DIM) - a_i[d]) * (rel[d] * sc);
            acc[0] = acc[0] + dt * (m_j / rho_j);
        } else if (OP == NAU_OP_SPH_G11) {  // interactions.cpp:81-102
            if (dist <= 0.0 || dist > radius) return;
            const double rho_j = a.rho.at(0, j, n);
            if (rho_j == 0.0) {
                latch_error(a.err, 1, kMsgZeroDensity, g.orig[j]);
                return;
            }
            const double a_j = a.A.at(0, j, n);
            const double m_j = a.m.at(0, j, n);
            const double sc = kernel_grad_scale<KF>(alpha, h, dist);
            const double s = m_j * (a_i[0] / (rho_i * rho_i) + a_j / (rho_j * rho_j));
#pragma unroll
            for (int d = 0; d < DIM; ++d) acc[d] = acc[d] + (rel[d] * sc) * s;
        } else if (OP == NAU_OP_SPH_L0) {  // interactions.cpp:104-126
            if (dist > radius) return;
            if (dist <= 0.0) {  // warn_coincident (interactions.cpp:32-38)
                if (g.orig[j] != my_orig && mask == 0) atomicAdd(&a.err->warnings, 1ull);
                return;
            }
            const double rho_j = a.rho.at(0, j, n);
            if (rho_j == 0.0) {
                latch_error(a.err, 1, kMsgZeroDensity, g.orig[j]);
                return;
            }
            const double a_j = a.A.at(0, j, n);
            const double m_j = a.m.at(0, j, n);
            const double sc = kernel_grad_scale<KF>(alpha, h, dist);
            double rg = rel[0] * (rel[0] * sc);
#pragma unroll
            for (int d = 1; d < DIM; ++d) rg = rg + rel[d] * (rel[d] * sc);
            acc[0] = acc[0] + 2.0 * (a_j - a_i[0]) * rg / (dist * dist) * m_j / rho_j;
        } else {  // NAU_OP_SPH_A, interactions.cpp:128-150
            if (dist > radius) return;
            if (dist <= 0.0) {
                if (g.orig[j] != my_orig && mask == 0) atomicAdd(&a.err->warnings, 1ull);
                return;
            }
            double ap = (mirror_comp(a.A.at(0, j, n), 0, DIM, 1, mask, DIM) - a_i[0]) * rel[0];
#pragma unroll
            for (int d = 1; d < DIM; ++d)
                ap = ap + (mirror_comp(a.A.at(d, j, n), d, DIM, 1, mask, DIM) - a_i[d]) * rel[d];
            if (ap >= 0.0) return;
            const double m_j = a.m.at(0, j, n);
            const double pi_ij = ap / (rho_i * dist * dist);
            const double sc = kernel_grad_scale<KF>(alpha, h, dist);
            const double s = m_j * pi_ij;
#pragma unroll
            for (int d = 0; d < DIM; ++d) acc[d] = acc[d] + (rel[d] * sc) * s;
        }
    });

    int oc = 1;
    if (OP == NAU_OP_SPH_S) oc = ac;
    if (OP == NAU_OP_SPH_G11 || OP == NAU_OP_SPH_A) oc = DIM;
    if (OP == NAU_OP_SPH_G11) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) acc[d] = rho_i * acc[d];
    }
    if (!valid) return;
#pragma unroll
    for (int c = 0; c < 9; ++c) {
        if (c < oc) {
            if (!isfinite(acc[c])) latch_error(a.err, 2, kMsgNan, my_orig);
            a.out[c * n + k] = acc[c];
        }
    }
}

// ---- DEM contact sums: dem_sum (interactions.cpp:152-193) ----
struct DemArgs {
    Geo g;
    const float4* xl;
    Opd v, R, P, Q, m, cf, Rs;  // P = E (Hertz) | kn (LSD); Q = nu (Hertz) | en (LSD)
    double zeta_uniform;        // LSD damping ratio from a uniform en (host libm), else NaN
    double gadd[3];             // body acceleration added to the result (DEM deck: + g)
    int has_g;
    double* out;
    DevErr* err;
};

template <int DIM, int OP>
#ifndef NAU_DEM_MINB
#define NAU_DEM_MINB 4  // <= 128 registers: 4 blocks/SM (136 regs: 3 blocks, +28%; 96 with spills: +18%)
#endif
__global__ void __launch_bounds__(kThreads, NAU_DEM_MINB) k_dem(const __grid_constant__ DemArgs a) {
    const Geo& g = a.g;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = k < *g.nact && !is_ghost(g, k);
    const int kk = valid ? k : 0;
    const long n = g.n;
    constexpr bool kImagesOnly = OP == NAU_OP_DEM_BOUNDARY;
    constexpr bool kLsd = OP == NAU_OP_DEM_LSD;
    double xi[3] = {0.0, 0.0, 0.0}, v_i[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
        xi[d] = g.x[d * n + kk];
        v_i[d] = a.v.at(d, kk, n);
    }
    const double radius = a.Rs.at(0, kk, n);
    const double Ri = a.R.at(0, kk, n), Pi = a.P.at(0, kk, n), Qi = a.Q.at(0, kk, n);
    const double mi = a.m.at(0, kk, n), fr = a.cf.at(0, kk, n);
    double zeta = 0.0;
    if (kLsd) {
        if (a.zeta_uniform == a.zeta_uniform) {
            zeta = a.zeta_uniform;
        } else {
            double le = log(Qi);
            zeta = -le / sqrt(kPi * kPi + le * le);
        }
    }
    const int my_orig = g.orig[kk];
    double acc[3] = {0.0, 0.0, 0.0};
    sweep<DIM, true>(g, a.xl, k, valid, xi, radius,
               [&](int j, const double* rel, int mask) {
        const double dist = norm_rel<DIM>(rel);
        if (dist > radius) return;
        if (kImagesOnly && mask == 0) return;
        if (dist <= 0.0) {
            if (!kLsd && g.orig[j] != my_orig && mask == 0) atomicAdd(&a.err->warnings, 1ull);
            return;
        }
        const double Rj = a.R.at(0, j, n), Pj = a.P.at(0, j, n), Qj = a.Q.at(0, j, n);
        const double mj = a.m.at(0, j, n);
        if (Rj + Ri - dist <= 0.0) return;
        double v_j[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int d = 0; d < DIM; ++d) v_j[d] = mirror_comp(a.v.at(d, j, n), d, DIM, 1, mask, DIM);
        // hertz_contact_force (interactions.cpp:288-316) / linear spring-dashpot
        const double overlap = Ri + Rj - dist;
        double n_ji[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int d = 0; d < DIM; ++d) n_ji[d] = rel[d] / dist;
        double dd = (v_j[0] - v_i[0]) * n_ji[0];
#pragma unroll
        for (int d = 1; d < DIM; ++d) dd = dd + (v_j[d] - v_i[d]) * n_ji[d];
        const double overlap_rate = -dd;
        double normal;
        if (kLsd) {
            const double kn = Pi;
            const double m_eff = mi * mj / (mi + mj);
            const double c_n = 2.0 * zeta * sqrt(m_eff * kn);
            normal = kn * overlap + c_n * overlap_rate;
        } else {
            if (Pi <= 0.0 || Pj <= 0.0 || Ri <= 0.0 || Rj <= 0.0) {
                latch_error(a.err, 1, kMsgDemParams, my_orig);
                return;
            }
            const double r_eff = Ri * Rj / (Ri + Rj);
            const double m_eff = mi * mj / (mi + mj);
            const double e_eff = Pi * Pj / (Pj * (1.0 - Qi * Qi) + Pi * (1.0 - Qj * Qj));
            const double k_hz = 4.0 / 3.0 * sqrt(r_eff) * e_eff;
            const double c_hz = sqrt(m_eff * k_hz) / 8.0 * 1.0;
            normal = k_hz * pow(overlap, 1.5) + c_hz * pow(overlap, 0.25) * overlap_rate;
        }
        double f[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int d = 0; d < DIM; ++d) f[d] = -(n_ji[d] * normal);
        if (fr != 0.0) {
            double v_ij[3], v_t[3];
#pragma unroll
            for (int d = 0; d < DIM; ++d) v_ij[d] = v_i[d] - v_j[d];
            double dn = v_ij[0] * n_ji[0];
#pragma unroll
            for (int d = 1; d < DIM; ++d) dn = dn + v_ij[d] * n_ji[d];
#pragma unroll
            for (int d = 0; d < DIM; ++d) v_t[d] = -v_ij[d] + n_ji[d] * dn;
            const double vt_norm = norm_rel<DIM>(v_t);
            if (vt_norm > 1e-12) {
                const double s = fr * fabs(normal) / vt_norm;
#pragma unroll
                for (int d = 0; d < DIM; ++d) f[d] = f[d] + v_t[d] * s;
            }
        }
#pragma unroll
        for (int d = 0; d < DIM; ++d) acc[d] = acc[d] + f[d];
    });
    if (!valid) return;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
        double r = kImagesOnly ? acc[d] : acc[d] / mi;
        if (a.has_g) r = r + a.gadd[d];  // vdot = dem_...(...) + g (BinaryNode Add)
        if (!isfinite(r)) latch_error(a.err, 2, kMsgNan, my_orig);
        a.out[d * n + k] = r;
    }
}

// ---- social force model: eval_social_force (interactions.cpp:216-257) ----
// Agents i: driving term (e0 * (v0/|e0|) - v_i) / tau toward r_d, minus the sum
// over candidates 0 < d < min cell size of n_ji * (A exp((r_ij - d)/B) + body
// - c_ij), divided by m_i. Operands 3 (radius) and 7 (c) are read at j; the
// pair rule ignores mirror guides (the reference passes none to it).
struct SfmArgs {
    Geo g;
    const float4* xl;
    Opd v, v0, rd, rad, A, B, K, cc, m, tau;
    double cs_min;
    double* out;
    DevErr* err;
};

template <int DIM>
__global__ void __launch_bounds__(kThreads) k_sfm(const __grid_constant__ SfmArgs a) {
    const Geo& g = a.g;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    bool valid = k < *g.nact;
    const int kk = valid ? k : 0;
    const long n = g.n;
    double xi[3] = {0.0, 0.0, 0.0}, v_i[3] = {0.0, 0.0, 0.0}, e0[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
        xi[d] = g.x[d * n + kk];
        v_i[d] = a.v.at(d, kk, n);
    }
    const double v0 = a.v0.at(0, kk, n), radius_i = a.rad.at(0, kk, n);
    const double rep_a = a.A.at(0, kk, n), rep_b = a.B.at(0, kk, n), body_k = a.K.at(0, kk, n);
    const double c_i = a.cc.at(0, kk, n), m_i = a.m.at(0, kk, n), tau = a.tau.at(0, kk, n);
    const int my_orig = g.orig[kk];
    if (valid && !(tau > 0.0)) {
        latch_error(a.err, 1, kMsgSfmTau, my_orig);
        valid = false;
    } else if (valid && !(m_i > 0.0)) {
        latch_error(a.err, 1, kMsgSfmMass, my_orig);
        valid = false;
    }
#pragma unroll
    for (int d = 0; d < DIM; ++d) e0[d] = a.rd.at(d, kk, n) - xi[d];
    const double e0n = norm_rel<DIM>(e0);
    double drv[3] = {0.0, 0.0, 0.0};
    if (e0n > 0.0) {
        const double s = v0 / e0n;
#pragma unroll
        for (int d = 0; d < DIM; ++d) drv[d] = (e0[d] * s - v_i[d]) / tau;
    } else if (valid) {
        atomicAdd(&a.err->warnings, 1ull);  // agent already at its desired position
    }
    const double cs_min = a.cs_min;
    double acc[3] = {0.0, 0.0, 0.0};
    sweep<DIM, true>(g, a.xl, k, valid, xi, cs_min, [&](int j, const double* rel, int) {
        const double d_ji = norm_rel<DIM>(rel);
        if (!(d_ji > 0.0 && d_ji < cs_min)) return;
        const double r_ij = radius_i + a.rad.at(0, j, n);
        const double c_ij = 0.5 * (c_i + a.cc.at(0, j, n));
        const double body = r_ij - d_ji > 0.0 ? body_k * (r_ij - d_ji) : 0.0;
        const double s = rep_a * exp((r_ij - d_ji) / rep_b) + body - c_ij;
#pragma unroll
        for (int d = 0; d < DIM; ++d) acc[d] = acc[d] + (rel[d] / d_ji) * s;
    });
    if (!valid) return;
    bool bad = false;
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
        const double r = drv[d] - acc[d] / m_i;
        bad |= !isfinite(r);
        a.out[d * n + k] = r;
    }
    if (bad) latch_error(a.err, 2, kMsgNan, my_orig);
}

// ---- all-pairs softened gravity: eval_gravity (interactions.cpp:195-214) ----
// j-tiles of positions/masses staged in shared memory; each thread sums its
// body's acceleration over j in storage order (the reference order when no
// cell build has permuted the bodies).
constexpr int kGravTile = 256;

struct GravArgs {
    long n;
    const double* x;
    const uint8_t* active;
    const int* orig;
    Opd m, G, eps;
    int has_eps;
    double* out;
    DevErr* err;
    // external sources (multi-GPU all-gather): (x, y, z, m) rows in global order,
    // local body k is source self_off + k; m = 0 marks an inactive source
    const double4* src;
    long nsrc, self_off;
    int accumulate;  // start from the sums in `out` (a later chunk of the sources)
};

// FAST: s = G m_j rsqrt(r2)^3 with FMA (≈1e-15 relative per pair); exact: G m_j / (r2 sqrt r2).
template <int DIM, bool FAST>
__global__ void __launch_bounds__(kGravTile) k_gravity(const __grid_constant__ GravArgs a) {
    __shared__ double sx[3][kGravTile];
    __shared__ double sm[kGravTile];
    __shared__ unsigned char sa[kGravTile];
    const long n = a.n;
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    const bool mine = k < n && a.active[k];
    double xi[3] = {0.0, 0.0, 0.0};
    double G = 0.0, eps = 0.0;
    if (mine) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) xi[d] = a.x[d * n + k];
        G = a.G.at(0, k, n);
        eps = a.has_eps ? a.eps.at(0, k, n) : 0.0;
    }
    const double eps2 = eps * eps;
    double acc[3] = {0.0, 0.0, 0.0};
    if (mine && a.accumulate)
#pragma unroll
        for (int d = 0; d < DIM; ++d) acc[d] = a.out[d * n + k];
    bool coincident = false;
    const long ns = a.src ? a.nsrc : n;
    const long self = a.self_off + k;
    for (long base = 0; base < ns; base += kGravTile) {
        const long j = base + threadIdx.x;
        if (j < ns && a.src) {
            const double4 s4 = a.src[j];
            sx[0][threadIdx.x] = s4.x;
            if (DIM > 1) sx[1][threadIdx.x] = s4.y;
            if (DIM > 2) sx[2][threadIdx.x] = s4.z;
            sm[threadIdx.x] = s4.w;
            sa[threadIdx.x] = s4.w != 0.0;
        } else if (j < ns) {
#pragma unroll
            for (int d = 0; d < DIM; ++d) sx[d][threadIdx.x] = a.x[d * n + j];
            sm[threadIdx.x] = a.m.at(0, (int)j, n);
            sa[threadIdx.x] = a.active[j];
        } else {
            sa[threadIdx.x] = 0;
        }
        __syncthreads();
        if (mine && FAST) {
            // branch-free pair loop (FMA via explicit fma(); this TU is -fmad=false):
            // self / inactive pairs are masked, not skipped, so the loop unrolls.
            const int lim = (int)min((long)kGravTile, ns - base);
#pragma unroll 4
            for (int t = 0; t < lim; ++t) {
                double rel[3] = {0.0, 0.0, 0.0};
#pragma unroll
                for (int d = 0; d < DIM; ++d) rel[d] = sx[d][t] - xi[d];
                double r2 = eps2;
#pragma unroll
                for (int d = DIM - 1; d >= 0; --d) r2 = fma(rel[d], rel[d], r2);
                const bool ok = (base + t != self) && sa[t];
                coincident |= ok && r2 == 0.0;
                const double inv = rsqrt(ok && r2 > 0.0 ? r2 : 1.0);
                const double s = ok && r2 > 0.0 ? G * sm[t] * (inv * inv * inv) : 0.0;
#pragma unroll
                for (int d = 0; d < DIM; ++d) acc[d] = fma(rel[d], s, acc[d]);
            }
        } else if (mine) {
            const int lim = (int)min((long)kGravTile, ns - base);
            for (int t = 0; t < lim; ++t) {
                if (base + t == self || !sa[t]) continue;
                double rel[3] = {0.0, 0.0, 0.0};
#pragma unroll
                for (int d = 0; d < DIM; ++d) rel[d] = sx[d][t] - xi[d];
                double r2 = rel[0] * rel[0];
#pragma unroll
                for (int d = 1; d < DIM; ++d) r2 = r2 + rel[d] * rel[d];
                r2 = r2 + eps2;
                if (r2 == 0.0) {
                    coincident = true;
                    continue;
                }
                double s;
                if (FAST) {
                    const double inv = rsqrt(r2);
                    s = G * sm[t] * (inv * inv * inv);
                } else {
                    s = G * sm[t] / (r2 * sqrt(r2));
                }
#pragma unroll
                for (int d = 0; d < DIM; ++d) acc[d] = acc[d] + rel[d] * s;
            }
        }
        __syncthreads();
    }
    if (!mine) return;
    if (coincident) latch_error(a.err, 1, kMsgCoincident, a.orig[k]);
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
        if (!isfinite(acc[d])) latch_error(a.err, 2, kMsgNan, a.orig[k]);
        a.out[d * n + k] = acc[d];
    }
}

// FAST, uniform G, uniform eps > 0 (the BASELINE cfg4 deck): every thread sums
// kGravBodies bodies against each staged source, the source tile holds
// (x, y, z, G m_j) with G m_j = 0 for inactive sources, and the self pair needs no
// test: rel = 0 there, so it adds exactly zero (r2 = eps^2 > 0 keeps it finite).
// Per pair: 3 DADD + 3 DFMA + rsqrt + 3 DMUL + 3 DFMA and a quarter of a shared
// load — profiles/r1b: the one-body loop issued 45 instructions per pair.
#ifndef NAU_GRAV_BODIES
#define NAU_GRAV_BODIES 2
#endif
constexpr int kGravBodies = NAU_GRAV_BODIES;
constexpr int kGravThreads = 128;

template <int DIM>
__global__ void __launch_bounds__(kGravThreads) k_gravity_fast(const __grid_constant__ GravArgs a,
                                                               double G, double eps2) {
    __shared__ double4 s4[kGravTile];
    const long n = a.n;
    const long k0 = (long)blockIdx.x * (kGravThreads * kGravBodies) + threadIdx.x;
    double xi[kGravBodies][3], acc[kGravBodies][3];
#pragma unroll
    for (int b = 0; b < kGravBodies; ++b) {
        const long k = k0 + b * kGravThreads;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            xi[b][d] = (d < DIM && k < n) ? a.x[d * n + k] : 0.0;
            acc[b][d] = (a.accumulate && d < DIM && k < n) ? a.out[d * n + k] : 0.0;
        }
    }
    const long ns = a.src ? a.nsrc : n;
    for (long base = 0; base < ns; base += kGravTile) {
        for (int t = threadIdx.x; t < kGravTile; t += kGravThreads) {
            const long j = base + t;
            double4 v = make_double4(0.0, 0.0, 0.0, 0.0);
            if (j < ns) {
                if (a.src) {
                    v = a.src[j];
                    v.w = G * v.w;  // m = 0 marks an inactive source
                } else {
                    double xs[3] = {0.0, 0.0, 0.0};
#pragma unroll
                    for (int d = 0; d < DIM; ++d) xs[d] = a.x[d * n + j];
                    v = make_double4(xs[0], xs[1], xs[2], a.active[j] ? G * a.m.at(0, (int)j, n) : 0.0);
                }
            }
            s4[t] = v;
        }
        __syncthreads();
        const int lim = (int)min((long)kGravTile, ns - base);
#pragma unroll 2
        for (int t = 0; t < lim; ++t) {
            const double4 sj = s4[t];
            const double xj[3] = {sj.x, sj.y, sj.z};
#pragma unroll
            for (int b = 0; b < kGravBodies; ++b) {
                double rel[3] = {0.0, 0.0, 0.0};
                double r2 = eps2;
#pragma unroll
                for (int d = DIM - 1; d >= 0; --d) {
                    rel[d] = xj[d] - xi[b][d];
                    r2 = fma(rel[d], rel[d], r2);
                }
                // m / r^3 from the MUFU estimate y ~ 1/sqrt(r2) (r2 >= eps2 > 0, normal):
                // with e = 1 - r2 y^2, r2^(-3/2) = y^3 (1 - e)^(-3/2)
                //   = y^3 (1 + 3e/2 + 15e^2/8 + O(e^3)),  |e| < 2^-19 (tools/mufu_acc.cu),
                // no special-value branch (CUDA's rsqrt) and one FP64 op fewer than
                // rsqrt + two products
                double y;
                asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
                const double y2 = y * y;
                const double e = fma(-r2, y2, 1.0);
                const double s = ((sj.w * y) * y2) * fma(e, fma(1.875, e, 1.5), 1.0);
#pragma unroll
                for (int d = 0; d < DIM; ++d) acc[b][d] = fma(rel[d], s, acc[b][d]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int b = 0; b < kGravBodies; ++b) {
        const long k = k0 + b * kGravThreads;
        if (k >= n || !a.active[k]) continue;  // inactive bodies keep their value
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
            if (!isfinite(acc[b][d])) latch_error(a.err, 2, kMsgNan, a.orig[k]);
            a.out[d * n + k] = acc[b][d];
        }
    }
}

template <int DIM, int OP, int KF>
void sph_launch(nau_ctx* c, const SphArgs& a, int ac) {
    const int blocks = (int)((c->n + kThreads - 1) / kThreads);
    if (OP == NAU_OP_SPH_S && ac > 1)
        k_sph<DIM, OP, KF, 9, false><<<blocks, kThreads, 0, c->stream>>>(a);
    else if (a.nl.e)
        k_sph<DIM, OP, KF, 1, true><<<blocks, kThreads, 0, c->stream>>>(a);
    else
        k_sph<DIM, OP, KF, 1, false><<<blocks, kThreads, 0, c->stream>>>(a);
}

template <int DIM, int OP>
void sph_launch_kf(nau_ctx* c, const SphArgs& a, int kf, int ac) {
    if (kf == NAU_K_CUBIC)
        sph_launch<DIM, OP, NAU_K_CUBIC>(c, a, ac);
    else
        sph_launch<DIM, OP, NAU_K_WENDLAND>(c, a, ac);
}

template <int DIM>
void sph_dispatch(nau_ctx* c, int op, const SphArgs& a, int kf, int ac) {
    switch (op) {
        case NAU_OP_SPH_S: sph_launch_kf<DIM, NAU_OP_SPH_S>(c, a, kf, ac); break;
        case NAU_OP_SPH_D00: sph_launch_kf<DIM, NAU_OP_SPH_D00>(c, a, kf, ac); break;
        case NAU_OP_SPH_G11: sph_launch_kf<DIM, NAU_OP_SPH_G11>(c, a, kf, ac); break;
        case NAU_OP_SPH_L0: sph_launch_kf<DIM, NAU_OP_SPH_L0>(c, a, kf, ac); break;
        default: sph_launch_kf<DIM, NAU_OP_SPH_A>(c, a, kf, ac); break;
    }
}

template <int DIM>
void dem_dispatch(nau_ctx* c, int op, const DemArgs& a) {
    const int blocks = (int)((c->n + kThreads - 1) / kThreads);
    if (op == NAU_OP_DEM_LSD)
        k_dem<DIM, NAU_OP_DEM_LSD><<<blocks, kThreads, 0, c->stream>>>(a);
    else if (op == NAU_OP_DEM_BOUNDARY)
        k_dem<DIM, NAU_OP_DEM_BOUNDARY><<<blocks, kThreads, 0, c->stream>>>(a);
    else
        k_dem<DIM, NAU_OP_DEM_HERTZ><<<blocks, kThreads, 0, c->stream>>>(a);
}

}  // namespace

void launch_interact(nau_ctx* c, int op, int kf, int kdim, const Opd* ops, int nops, double* out,
                     int out_rows, int out_cols, int a_rows, int a_cols, const double* gadd,
                     const GravSources* gsrc, bool lists) {
    (void)out_rows;
    (void)out_cols;
    if (c->n == 0) return;
    const int dim = c->dom.dim;
    // every path that sweeps reads the fp32 pre-filter copy (sph_launch: a tensor-valued
    // sph_S operand sweeps even when a list exists)
    const bool list_path = op <= NAU_OP_SPH_A && lists && !(op == NAU_OP_SPH_S && a_rows * a_cols > 1);
    if (op != NAU_OP_GRAVITY && !list_path) ensure_xl(c);
    if (op <= NAU_OP_SPH_A) {
        SphArgs a;
        a.g = make_geo(c);
        a.xl = c->d_xl;
        a.A = ops[0];
        a.m = ops[1];
        a.rho = ops[2];
        a.R = ops[3];
        a.out = out;
        a.arows = a_rows;
        a.acols = a_cols;
        a.kdim = kdim;
        a.err = c->d_err;
        a.nl = NList{lists ? c->d_nlist : nullptr, c->d_ncount, c->nl_cap};
        const int ac = a_rows * a_cols;
        prof_begin(c, 100 + op);
        if (dim == 1) sph_dispatch<1>(c, op, a, kf, ac);
        else if (dim == 2) sph_dispatch<2>(c, op, a, kf, ac);
        else sph_dispatch<3>(c, op, a, kf, ac);
        prof_end(c, 100 + op);
    } else if (op == NAU_OP_GRAVITY) {
        GravArgs a;
        a.n = c->n;
        a.x = c->fields[0].d;
        a.active = c->d_active;
        a.orig = c->d_orig;
        a.m = ops[0];
        a.G = ops[1];
        a.has_eps = nops > 2;
        if (nops > 2) a.eps = ops[2];
        else a.eps = ops[1];
        a.out = out;
        a.err = c->d_err;
        a.src = gsrc ? gsrc->src : nullptr;
        a.nsrc = gsrc ? gsrc->nsrc : 0;
        a.self_off = gsrc ? gsrc->self_off : 0;
        a.accumulate = gsrc ? gsrc->accumulate : 0;
        const int blocks = (int)((c->n + kGravTile - 1) / kGravTile);
        prof_begin(c, 100 + op);
        const bool fast = c->mode == NAU_MODE_FAST;
        const bool uniform_soft = a.G.p == nullptr && a.has_eps && a.eps.p == nullptr &&
                                  a.eps.v[0] * a.eps.v[0] >= 1e-300;  // normal: MUFU is ftz
        if (fast && uniform_soft) {
            const int nb = (int)((c->n + kGravThreads * kGravBodies - 1) / (kGravThreads * kGravBodies));
            const double G = a.G.v[0], eps2 = a.eps.v[0] * a.eps.v[0];
            if (dim == 1) k_gravity_fast<1><<<nb, kGravThreads, 0, c->stream>>>(a, G, eps2);
            else if (dim == 2) k_gravity_fast<2><<<nb, kGravThreads, 0, c->stream>>>(a, G, eps2);
            else k_gravity_fast<3><<<nb, kGravThreads, 0, c->stream>>>(a, G, eps2);
        } else if (dim == 1) {
            if (fast) k_gravity<1, true><<<blocks, kGravTile, 0, c->stream>>>(a);
            else k_gravity<1, false><<<blocks, kGravTile, 0, c->stream>>>(a);
        } else if (dim == 2) {
            if (fast) k_gravity<2, true><<<blocks, kGravTile, 0, c->stream>>>(a);
            else k_gravity<2, false><<<blocks, kGravTile, 0, c->stream>>>(a);
        } else {
            if (fast) k_gravity<3, true><<<blocks, kGravTile, 0, c->stream>>>(a);
            else k_gravity<3, false><<<blocks, kGravTile, 0, c->stream>>>(a);
        }
        prof_end(c, 100 + op);
    } else if (op == NAU_OP_SFM) {
        SfmArgs a;
        a.g = make_geo(c);
        a.xl = c->d_xl;
        a.v = ops[0];
        a.v0 = ops[1];
        a.rd = ops[2];
        a.rad = ops[3];
        a.A = ops[4];
        a.B = ops[5];
        a.K = ops[6];
        a.cc = ops[7];
        a.m = ops[8];
        a.tau = ops[9];
        double cs_min = c->dom.cs[0];  // interactions.cpp:239-240
        for (int d = 1; d < dim; ++d) cs_min = std::min(cs_min, c->dom.cs[d]);
        a.cs_min = cs_min;
        a.out = out;
        a.err = c->d_err;
        const int blocks = (int)((c->n + kThreads - 1) / kThreads);
        prof_begin(c, 100 + op);
        if (dim == 1) k_sfm<1><<<blocks, kThreads, 0, c->stream>>>(a);
        else if (dim == 2) k_sfm<2><<<blocks, kThreads, 0, c->stream>>>(a);
        else k_sfm<3><<<blocks, kThreads, 0, c->stream>>>(a);
        prof_end(c, 100 + op);
    } else {
        DemArgs a;
        a.g = make_geo(c);
        a.xl = c->d_xl;
        a.v = ops[0];
        a.R = ops[1];
        a.P = ops[2];
        a.Q = ops[3];
        a.m = ops[4];
        a.cf = ops[5];
        a.Rs = ops[6];
        a.zeta_uniform = __builtin_nan("");
        a.has_g = gadd != nullptr;
        for (int d = 0; d < 3; ++d) a.gadd[d] = gadd ? gadd[d] : 0.0;
        if (op == NAU_OP_DEM_LSD && ops[3].p == nullptr) {
            double le = std::log(ops[3].v[0]);
            a.zeta_uniform = -le / std::sqrt(kPi * kPi + le * le);
        }
        a.out = out;
        a.err = c->d_err;
        prof_begin(c, 100 + op);
        if (dim == 1) dem_dispatch<1>(c, op, a);
        else if (dim == 2) dem_dispatch<2>(c, op, a);
        else dem_dispatch<3>(c, op, a);
        prof_end(c, 100 + op);
    }
    c->launches++;
}

}  // namespace nau
