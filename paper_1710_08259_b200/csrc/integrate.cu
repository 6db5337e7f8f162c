// integrate.cu — elementwise update kernels and the fused weakly-compressible
// SPH deck of BASELINE cfg0/cfg2.
//
//   k_euler       ≙ EulerNode::evaluate (src/sfl/ast.cpp:180-191), active particles only
//                   (inactive keep their value, src/case.cpp:36-40)
//   k_symplectic  ≙ v = euler(v, vdot*mask, dt); r = euler(r, v, dt); apply_boundary_shift
//                   (deck order dam_break_2d.yaml:37-38; case.cpp:59-62; particle_system.cpp:56-90)
//   k_wcsph_*     the BASELINE dam-break equations as two neighbour passes (see
//                 nauticle_gpu.h nau_wcsph_step) with per-operator accumulators
//                 combined in the RHS expression's evaluation order (ast.cpp:71-94).
// Compiled with -fmad=false like interact.cu.
#include <cmath>
#include <cstring>

#include "nau_internal.cuh"
#include "sweep.cuh"

namespace nau {

namespace {

constexpr int kBlock = 256;
constexpr int kThreads = kSweepThreads;
inline int blocks_for(long n, int b = kBlock) { return (int)((n + b - 1) / b); }

// dst = src on active particles unless an error is latched (the fused sph_G11 + sph_L0
// pass: the reference would not have evaluated the sph_L0 equation after a failure).
__global__ void k_commit_if_ok(long n, const uint8_t* active, const double* src, double* dst,
                               const DevErr* err) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n || err->code != 0 || !active[k]) return;
    dst[k] = src[k];
}

__global__ void k_euler(long n, int comps, const uint8_t* active, const int* orig, const double* x,
                        const double* xdot, double dt, double* out, DevErr* err) {
    long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const bool act = active[k];
    for (int c = 0; c < comps; ++c) {
        double v = x[c * n + k];
        if (act) {
            v = v + dt * xdot[c * n + k];
            if (!isfinite(v)) latch_error(err, 2, kMsgNan, orig[k]);
        }
        out[c * n + k] = v;
    }
}

// One thread per particle: the two euler equations then the boundary shift of r.
__global__ void k_symplectic(DomainDev d, long n, double* pos, double* v, const double* vdot,
                             const double* mask, double dt, uint8_t* active, const int* orig,
                             DevErr* err, const uint8_t* upd) {
    long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n || !active[k] || (upd && !upd[k])) return;  // ghosts: owned elsewhere
    // every load first (the compiler cannot move a load above a store through these
    // pointers): ten independent requests in flight per thread instead of a chain
    const double mk = mask ? __ldg(mask + k) : 1.0;
    double xd[3] = {0.0, 0.0, 0.0}, vo[3] = {0.0, 0.0, 0.0}, xo[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int a = 0; a < 3; ++a)
        if (a < d.dim) {
            xd[a] = __ldg(vdot + a * n + k);
            vo[a] = v[a * n + k];
            xo[a] = pos[a * n + k];
        }
    double vn[3];
    bool bad = false;
#pragma unroll
    for (int a = 0; a < 3; ++a)
        if (a < d.dim) {
            // euler(v, vdot*mask, dt): vdot*mask is mask * vdot (scalar broadcast, tensor.cpp:55-57)
            const double x1 = mask ? mk * xd[a] : xd[a];
            vn[a] = vo[a] + dt * x1;
            bad |= !isfinite(vn[a]);
            v[a * n + k] = vn[a];
        }
    if (bad) latch_error(err, 2, kMsgNan, orig[k]);
    bad = false;
    unsigned long long warn = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
        if (a < d.dim) {
            const double x = xo[a] + dt * vn[a];
            bad |= !isfinite(x);
            pos[a * n + k] = x;
        }
    if (bad) latch_error(err, 2, kMsgNan, orig[k]);
    // apply_boundary_shift (particle_system.cpp:56-90)
    for (int a = 0; a < d.dim; ++a) {
        double x = pos[a * n + k];
        const double lo = d.lo[a], hi = d.hi[a];
        if (d.kind[a] == NAU_PERIODIC) {
            if (x < lo || x >= hi) {
                double w = fmod(x - lo, d.ext[a]);
                if (w < 0.0) w += d.ext[a];
                x = lo + w;
                if (x >= hi) x = lo;
                pos[a * n + k] = x;
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

struct WcsphArgs {
    Geo g;
    const float4* xl;
    double mass, radius, rho0, B, gamma, visc, g_acc[3];
    int kdim;
    double* rho;
    double* p;
    const double* v;
    double* vdot;
    DevErr* err;
    NList nl;
    double4* vp;  // (vx, vy, vz, p / (rho * rho)) per slot, written by the density pass
    const int* work = nullptr;   // the fallback pass: slots whose list overflowed
    const int* nwork = nullptr;
};

// Pass 1: rho = sph_S(one, m, one, K, R) (interactions.cpp:40-58 with A = rho = 1),
//         p = B*((rho/rho0)^gamma - 1).
template <int DIM, int KF, bool LIST, bool WORK = false>
__global__ void __launch_bounds__(kThreads) k_wcsph_density(const __grid_constant__ WcsphArgs a) {
    const Geo& g = a.g;
    for_slots<LIST, WORK>(g, a.nl.count, a.work, a.nwork, [&](const int k, bool valid) {
        const int kk = valid ? k : 0;
        const long n = g.n;
        double xi[3] = {0.0, 0.0, 0.0};
    #pragma unroll
        for (int d = 0; d < DIM; ++d) xi[d] = g.x[d * n + kk];
        const double radius = a.radius;
        const double h = 0.5 * radius;
        const double alpha = kernel_alpha<KF>(a.kdim, h);
        const double s_unit = a.mass / 1.0;  // m_j / rho_j with the uniform operand rho = 1
        double acc = 0.0;
        for_neighbors<DIM, true, LIST>(g, a.xl, a.nl, k, valid, xi, radius, NoLoad{},
                   [&](int, const double* rel, int, NoPayload) {
            const double dist = norm_rel<DIM>(rel);
            if (dist > radius) return;
            const double w = kernel_value<KF>(alpha, h, dist);
            if (w == 0.0) return;
            acc = acc + 1.0 * (s_unit * w);
        });
        if (!valid) return;
        const double p = a.B * (pow(acc / a.rho0, a.gamma) - 1.0);
        if (!isfinite(acc) || !isfinite(p)) latch_error(a.err, 2, kMsgNan, g.orig[k]);
        a.rho[k] = acc;
        a.p[k] = p;
        // the momentum pass's per-neighbour operands in one 32-byte record; p/(rho*rho)
        // is the reference's per-pair subexpression (interactions.cpp:97), same value
        double vv[3] = {0.0, 0.0, 0.0};
    #pragma unroll
        for (int d = 0; d < DIM; ++d) vv[d] = a.v[d * n + k];
        a.vp[k] = make_double4(vv[0], vv[1], vv[2], p / (acc * acc));
    });
}

// Pass 2: vdot = -1/rho*sph_G11(p,m,rho,K,R) + visc*sph_A(v,m,rho,K,R) + g, one
// neighbour walk with the two operators' accumulators kept apart.
template <int DIM, int KF, bool LIST, bool WORK = false>
__global__ void __launch_bounds__(kThreads) k_wcsph_momentum(const __grid_constant__ WcsphArgs a) {
    const Geo& g = a.g;
    for_slots<LIST, WORK>(g, a.nl.count, a.work, a.nwork, [&](const int k, bool valid) {
        const int kk = valid ? k : 0;
        const long n = g.n;
        double xi[3] = {0.0, 0.0, 0.0}, v_i[3] = {0.0, 0.0, 0.0};
    #pragma unroll
        for (int d = 0; d < DIM; ++d) {
            xi[d] = g.x[d * n + kk];
            v_i[d] = a.v[d * n + kk];
        }
        const double radius = a.radius;
        const double h = 0.5 * radius;
        const double alpha = kernel_alpha<KF>(a.kdim, h);
        const double m = a.mass;
        const double rho_i = a.rho[kk];
        const double p_i = a.p[kk];
        const int my_orig = g.orig[kk];
        if (valid && rho_i == 0.0) {
            latch_error(a.err, 1, kMsgZeroDensity, my_orig);
            valid = false;
        }
        const double pr_i = p_i / (rho_i * rho_i);
        double G[3] = {0.0, 0.0, 0.0}, A[3] = {0.0, 0.0, 0.0};
        // per-neighbour operands (v_j, p_j / rho_j^2), gathered ahead of the pair arithmetic
        const Ld256 load{a.vp};
        for_neighbors<DIM, true, LIST, false, 2>(g, a.xl, a.nl, k, valid, xi, radius, load,
                   [&](int j, const double* rel, int mask, const double4& pj) {
            const double dist = norm_rel<DIM>(rel);
            if (dist > radius) return;
            if (dist <= 0.0) {  // G11 skips silently; sph_A warns (interactions.cpp:32-38)
                if (g.orig[j] != my_orig && mask == 0) atomicAdd(&a.err->warnings, 1ull);
                return;
            }
            const double sc = kernel_grad_scale<KF>(alpha, h, dist);
            const double pr_j = pj.w;  // non-finite only if rho_j == 0 or p_j overflowed
            if (!isfinite(pr_j) && a.rho[j] == 0.0) {
                latch_error(a.err, 1, kMsgZeroDensity, g.orig[j]);
                return;
            }
            const double s = m * (pr_i + pr_j);
    #pragma unroll
            for (int d = 0; d < DIM; ++d) G[d] = G[d] + (rel[d] * sc) * s;
            const double vj[3] = {pj.x, pj.y, pj.z};
            double ap = (mirror_comp(vj[0], 0, DIM, 1, mask, DIM) - v_i[0]) * rel[0];
    #pragma unroll
            for (int d = 1; d < DIM; ++d)
                ap = ap + (mirror_comp(vj[d], d, DIM, 1, mask, DIM) - v_i[d]) * rel[d];
            if (ap >= 0.0) return;
            const double pi_ij = ap / (rho_i * dist * dist);
            const double sa = m * pi_ij;
    #pragma unroll
            for (int d = 0; d < DIM; ++d) A[d] = A[d] + (rel[d] * sc) * sa;
        });
        if (!valid) return;
        const double s1 = -1.0 / rho_i;
        bool bad = false;
    #pragma unroll
        for (int d = 0; d < DIM; ++d) {
            const double gd = rho_i * G[d];
            const double r = (s1 * gd + a.visc * A[d]) + a.g_acc[d];
            bad |= !isfinite(r);
            a.vdot[d * n + k] = r;
        }
        if (bad) latch_error(a.err, 2, kMsgNan, my_orig);
    });
}

// ---- reductions (fmax/fmin/fsum/fmean), ast.cpp:237-274 ----
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 296;  // 2 x 148 SMs

__global__ void k_reduce_partial(long n, int comps, int kind, const uint8_t* active,
                                 const double* f, double* part, unsigned long long* cnt) {
    __shared__ double sh[kRedThreads][9];
    double acc[9];
    for (int c = 0; c < 9; ++c) acc[c] = kind == 0 ? -INFINITY : (kind == 1 ? INFINITY : 0.0);
    unsigned long long my = 0;
    for (long k = blockIdx.x * (long)blockDim.x + threadIdx.x; k < n; k += (long)gridDim.x * blockDim.x) {
        if (!active[k]) continue;
        ++my;
        if (kind >= 2) {
            for (int c = 0; c < comps; ++c) acc[c] += f[c * n + k];
        } else {
            double s;
            if (comps == 1) {
                s = f[k];
            } else {
                s = f[k] * f[k];
                for (int c = 1; c < comps; ++c) s = s + f[c * n + k] * f[c * n + k];
                s = sqrt(s);
            }
            acc[0] = kind == 0 ? fmax(acc[0], s) : fmin(acc[0], s);
        }
    }
    for (int c = 0; c < 9; ++c) sh[threadIdx.x][c] = acc[c];
    atomicAdd(cnt, my);
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            for (int c = 0; c < 9; ++c) {
                double o = sh[threadIdx.x + s][c];
                double& t = sh[threadIdx.x][c];
                t = kind == 0 ? fmax(t, o) : (kind == 1 ? fmin(t, o) : t + o);
            }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int c = 0; c < 9; ++c) part[blockIdx.x * 9 + c] = sh[0][c];
}

template <int DIM, bool LIST>
void wcsph_launch(nau_ctx* c, const WcsphArgs& a, int kf, int passes) {
    const int blocks = (int)((c->n + kThreads - 1) / kThreads);
    if (passes & 1) {
        prof_begin(c, 200);
        if (kf == NAU_K_CUBIC) {
            k_wcsph_density<DIM, NAU_K_CUBIC, LIST><<<blocks, kThreads, 0, c->stream>>>(a);
        } else {
            k_wcsph_density<DIM, NAU_K_WENDLAND, LIST><<<blocks, kThreads, 0, c->stream>>>(a);
        }
        prof_end(c, 200);
        c->launches++;
    }
    if (passes & 2) {
        prof_begin(c, 201);
        if (kf == NAU_K_CUBIC) {
            k_wcsph_momentum<DIM, NAU_K_CUBIC, LIST><<<blocks, kThreads, 0, c->stream>>>(a);
        } else {
            k_wcsph_momentum<DIM, NAU_K_WENDLAND, LIST><<<blocks, kThreads, 0, c->stream>>>(a);
        }
        prof_end(c, 201);
        c->launches++;
    }
}

template <int DIM>
void wcsph_launch_dim(nau_ctx* c, const WcsphArgs& a, int kf, int passes) {
    if (a.nl.e)
        wcsph_launch<DIM, true>(c, a, kf, passes);
    else
        wcsph_launch<DIM, false>(c, a, kf, passes);
}

// The fallback pass of an async list build: the overflowed slots swept per particle
// (the same candidates in the same order as the list).
template <int DIM>
void wcsph_fallback(nau_ctx* c, const WcsphArgs& a, int kf, int passes) {
    constexpr int kBlocks = 148 * 4;
    if (passes & 1) {
        if (kf == NAU_K_CUBIC) k_wcsph_density<DIM, NAU_K_CUBIC, false, true><<<kBlocks, kThreads, 0, c->stream>>>(a);
        else k_wcsph_density<DIM, NAU_K_WENDLAND, false, true><<<kBlocks, kThreads, 0, c->stream>>>(a);
    }
    if (passes & 2) {
        if (kf == NAU_K_CUBIC) k_wcsph_momentum<DIM, NAU_K_CUBIC, false, true><<<kBlocks, kThreads, 0, c->stream>>>(a);
        else k_wcsph_momentum<DIM, NAU_K_WENDLAND, false, true><<<kBlocks, kThreads, 0, c->stream>>>(a);
    }
    c->launches++;
}

}  // namespace

void launch_commit_if_ok(nau_ctx* c, const double* src, double* dst) {
    if (c->n == 0) return;
    k_commit_if_ok<<<blocks_for(c->n), kBlock, 0, c->stream>>>(c->n, c->d_active, src, dst, c->d_err);
    c->launches++;
}

void launch_euler(nau_ctx* c, const double* x, const double* xdot, double dt, double* out,
                  int comps) {
    if (c->n == 0) return;
    k_euler<<<blocks_for(c->n), kBlock, 0, c->stream>>>(c->n, comps, c->d_active, c->d_orig, x,
                                                         xdot, dt, out, c->d_err);
    c->launches++;
}

void launch_symplectic(nau_ctx* c, double* v, const double* vdot, const double* mask, double dt) {
    if (c->n == 0) return;
    prof_begin(c, 301);
    k_symplectic<<<blocks_for(c->n), kBlock, 0, c->stream>>>(c->dom, c->n, c->fields[0].d, v, vdot,
                                                              mask, dt, c->d_active, c->d_orig,
                                                              c->d_err,
                                                              c->ghost_field >= 0 ? c->d_upd : nullptr);
    prof_end(c, 301);
    c->launches++;
}

void launch_wcsph(nau_ctx* c, const nau_wcsph_params* p, bool lists, int passes) {
    if (c->n == 0) return;
    WcsphArgs a;
    a.nl = NList{lists ? c->d_nlist : nullptr, c->d_ncount, c->nl_cap};
    a.vp = c->d_aux;
    a.g = make_geo(c);
    if (!lists) ensure_xl(c);
    a.xl = c->d_xl;
    a.mass = p->mass;
    a.radius = p->radius;
    a.rho0 = p->rho0;
    a.B = p->B;
    a.gamma = p->gamma;
    a.visc = p->visc;
    for (int d = 0; d < 3; ++d) a.g_acc[d] = p->g[d];
    a.kdim = p->kernel_dim;
    a.rho = c->fields[p->f_rho].d;
    a.p = c->fields[p->f_p].d;
    a.v = c->fields[p->f_v].d;
    a.vdot = c->fields[p->f_vdot].d;
    a.err = c->d_err;
    switch (c->dom.dim) {
        case 1: wcsph_launch_dim<1>(c, a, p->kernel_family, passes); break;
        case 2: wcsph_launch_dim<2>(c, a, p->kernel_family, passes); break;
        default: wcsph_launch_dim<3>(c, a, p->kernel_family, passes); break;
    }
    if (lists && c->nl_async) {  // slots whose list overflowed: swept per particle
        WcsphArgs f = a;
        f.nl.e = nullptr;
        f.work = c->d_work;
        f.nwork = c->d_nwork;
        ensure_xl(c);
        switch (c->dom.dim) {
            case 1: wcsph_fallback<1>(c, f, p->kernel_family, passes); break;
            case 2: wcsph_fallback<2>(c, f, p->kernel_family, passes); break;
            default: wcsph_fallback<3>(c, f, p->kernel_family, passes); break;
        }
    }
}

void launch_reduce(nau_ctx* c, int kind, const double* f, int comps, double* h_out) {
    double* part = c->d_red;
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(c->d_red + kRedBlocks * 9);
    cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), c->stream);
    k_reduce_partial<<<kRedBlocks, kRedThreads, 0, c->stream>>>(c->n, comps, kind, c->d_active, f,
                                                                 part, cnt);
    c->launches++;
    std::vector<double> h(kRedBlocks * 9 + 1);
    cudaMemcpyAsync(h.data(), part, sizeof(double) * (kRedBlocks * 9 + 1), cudaMemcpyDeviceToHost,
                    c->stream);
    cudaStreamSynchronize(c->stream);
    unsigned long long count = 0;
    std::memcpy(&count, &h[kRedBlocks * 9], sizeof(count));
    const int oc = kind >= 2 ? comps : 1;
    for (int q = 0; q < oc; ++q) {
        double acc = kind == 0 ? -INFINITY : (kind == 1 ? INFINITY : 0.0);
        for (int b = 0; b < kRedBlocks; ++b) {
            double v = h[b * 9 + q];
            acc = kind == 0 ? std::fmax(acc, v) : (kind == 1 ? std::fmin(acc, v) : acc + v);
        }
        if (kind == 3) acc = acc / (double)count;
        h_out[q] = acc;
    }
}

}  // namespace nau
