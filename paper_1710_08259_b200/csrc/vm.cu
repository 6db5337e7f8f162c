// vm.cu — device evaluator for SFL particle-wise arithmetic.
//
// nau_eval runs a register program (include/nauticle_gpu.h nau_vm_instr) for
// every active particle: one thread per particle, the program in constant-like
// global memory read warp-uniformly, registers of up to 3 x 3 doubles. Shapes are
// fixed by the program, so the host validates them once with the reference's rules
// (tensor.cpp:11-93) and messages before the launch. Arithmetic follows the
// reference's evaluation order and the shim Eigen's storage-order reductions;
// compiled with -fmad=false like interact.cu, so every program without a libm
// transcendental is bitwise equal to the reference (tests/test_gpu_parity.py).
#include <cmath>
#include <string>
#include <vector>

#include "nau_internal.cuh"

namespace nau {

struct VmShape {
    int rows = 0, cols = 0;
    bool scalar() const { return rows == 1 && cols == 1; }
    int size() const { return rows * cols; }
};

struct VmIns {  // device copy (shape-annotated)
    int op, dst, a, b, field;
    int rows, cols;      // dst shape
    int ar, ac, br, bc;  // operand shapes
    double imm[9];
};

namespace {

constexpr int kVmThreads = 128;

struct VmFields {
    const double* p[kMaxFields];
};

__device__ __forceinline__ double vm_unary(int op, double x) {
    switch (op) {
        case NAU_VM_EXP: return exp(x);
        case NAU_VM_LOG: return log(x);
        case NAU_VM_SIN: return sin(x);
        case NAU_VM_COS: return cos(x);
        case NAU_VM_TAN: return tan(x);
        case NAU_VM_SQRT: return sqrt(x);
        case NAU_VM_ABS: return fabs(x);
        case NAU_VM_FLOOR: return floor(x);
        case NAU_VM_SGN: return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0);
        default: return -x;  // NAU_VM_NEG
    }
}

__device__ __forceinline__ double vm_binary(int op, double x, double y) {
    switch (op) {
        case NAU_VM_POW: return pow(x, y);
        case NAU_VM_MIN: return fmin(x, y);
        default: return fmax(x, y);  // NAU_VM_MAX
    }
}

// RandomState::uniform (sfl/random_state.hpp): splitmix64-style mixing of (seed,
// particle, per-particle counter), 53 random bits.
__device__ __forceinline__ unsigned long long rng_mix(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

__global__ void __launch_bounds__(kVmThreads) k_vm(const VmIns* __restrict__ prog, int nins,
                                                   int result, long n, VmFields f,
                                                   const uint8_t* active, const int* orig,
                                                   double* out, DevErr* err,
                                                   unsigned long long* rng, long rng_len,
                                                   unsigned long long seed) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= n || !active[k]) return;  // inactive particles keep their value (case.cpp:36-40)
    double R[NAU_VM_MAX_REGS][9];
    for (int pc = 0; pc < nins; ++pc) {
        const VmIns I = prog[pc];
        double* d = R[I.dst];
        const double* a = R[I.a];
        const double* b = R[I.b];
        const int sz = I.rows * I.cols;
        switch (I.op) {
            case NAU_VM_LOAD_FIELD:
                for (int c = 0; c < sz; ++c) d[c] = f.p[I.field][c * n + k];
                break;
            case NAU_VM_LOAD_CONST:
                for (int c = 0; c < sz; ++c) d[c] = I.imm[c];
                break;
            case NAU_VM_ADD:
                for (int c = 0; c < sz; ++c) d[c] = a[c] + b[c];
                break;
            case NAU_VM_SUB:
                for (int c = 0; c < sz; ++c) d[c] = a[c] - b[c];
                break;
            case NAU_VM_MUL: {
                if (I.ar == 1 && I.ac == 1) {  // a(0,0) * b.mat()
                    const double s = a[0];
                    for (int c = 0; c < sz; ++c) d[c] = s * b[c];
                } else if (I.br == 1 && I.bc == 1) {  // b(0,0) * a.mat()
                    const double s = b[0];
                    for (int c = 0; c < sz; ++c) d[c] = s * a[c];
                } else {  // matrix product, inner index summed in order
                    double t[9];
                    for (int r = 0; r < I.ar; ++r)
                        for (int cc = 0; cc < I.bc; ++cc) {
                            double s = a[r] * b[cc * I.br];
                            for (int q = 1; q < I.ac; ++q) s = s + a[q * I.ar + r] * b[cc * I.br + q];
                            t[cc * I.ar + r] = s;
                        }
                    for (int c = 0; c < sz; ++c) d[c] = t[c];
                }
                break;
            }
            case NAU_VM_DIV:
                if (I.br == 1 && I.bc == 1) {
                    const double s = b[0];
                    for (int c = 0; c < sz; ++c) d[c] = a[c] / s;
                } else {
                    for (int c = 0; c < sz; ++c) d[c] = a[c] / b[c];
                }
                break;
            case NAU_VM_POW:
            case NAU_VM_MIN:
            case NAU_VM_MAX: {  // elementwise_binary: scalar broadcast on either side
                const bool as = I.ar == 1 && I.ac == 1, bs = I.br == 1 && I.bc == 1;
                const double a0 = a[0], b0 = b[0];  // dst may alias an operand
                for (int c = 0; c < sz; ++c) {
                    const double x = (as && !bs) ? a0 : a[c];
                    const double y = (bs && !as) ? b0 : b[c];
                    d[c] = vm_binary(I.op, x, y);
                }
                break;
            }
            case NAU_VM_LT: d[0] = a[0] < b[0] ? 1.0 : 0.0; break;
            case NAU_VM_GT: d[0] = a[0] > b[0] ? 1.0 : 0.0; break;
            case NAU_VM_LE: d[0] = a[0] <= b[0] ? 1.0 : 0.0; break;
            case NAU_VM_GE: d[0] = a[0] >= b[0] ? 1.0 : 0.0; break;
            case NAU_VM_EQ: d[0] = a[0] == b[0] ? 1.0 : 0.0; break;
            case NAU_VM_NE: d[0] = a[0] != b[0] ? 1.0 : 0.0; break;
            case NAU_VM_JOIN: {
                const double tail = b[0];
                for (int c = 0; c < I.ar; ++c) d[c] = a[c];
                d[I.ar] = tail;
                break;
            }
            case NAU_VM_RAND: {  // RandNode (sfl/ast.cpp:212-217)
                const double lo = a[0], hi = b[0];
                if (lo > hi) {
                    latch_error(err, 1, kMsgRandBounds, orig[k]);
                    d[0] = 0.0;
                    break;
                }
                const long i = orig[k];
                const long slot = i < rng_len ? i : 0;
                const unsigned long long cnt = rng[slot]++;  // one thread per particle
                const unsigned long long x =
                    rng_mix(rng_mix(seed ^ 0x6e61757469636c65ULL) ^
                            rng_mix((unsigned long long)slot + 0x9e3779b9ULL) ^ cnt);
                const double u = (double)(x >> 11) * 0x1.0p-53;
                d[0] = lo + u * (hi - lo);
                break;
            }
            case NAU_VM_NORM: {  // sqrt(squaredNorm()), storage order
                const int m = I.ar * I.ac;
                double s = a[0] * a[0];
                for (int c = 1; c < m; ++c) s = s + a[c] * a[c];
                d[0] = sqrt(s);
                break;
            }
            case NAU_VM_DOT: {  // cwiseProduct(...).sum(), storage order
                const int m = I.ar * I.ac;
                double s = a[0] * b[0];
                for (int c = 1; c < m; ++c) s = s + a[c] * b[c];
                d[0] = s;
                break;
            }
            default:  // elementwise unary (incl. NEG)
                for (int c = 0; c < sz; ++c) d[c] = vm_unary(I.op, a[c]);
                break;
        }
    }
    const double* v = R[result];
    bool bad = false;
    // output shape = the register's shape, recorded by the host in the trailing record
    const int sz = prog[nins].rows * prog[nins].cols;
    for (int c = 0; c < sz; ++c) {
        bad |= !isfinite(v[c]);
        out[c * n + k] = v[c];
    }
    if (bad) latch_error(err, 2, kMsgNan, orig[k]);
}

std::string shape_str(const VmShape& s) { return std::to_string(s.rows) + "x" + std::to_string(s.cols); }

const char* op_symbol(int op) {
    switch (op) {
        case NAU_VM_ADD: return "+";
        case NAU_VM_SUB: return "-";
        case NAU_VM_MUL: return "*";
        case NAU_VM_DIV: return "/";
        case NAU_VM_POW: return "^";
        case NAU_VM_MIN: return "min";
        case NAU_VM_MAX: return "max";
        case NAU_VM_DOT: return "dot";
        default: return "comparison";
    }
}

}  // namespace

// Shape inference + validation with the reference's rules; on error returns the
// reference's message. `prog` receives the shape-annotated program plus one
// trailing record holding the result shape.
static bool vm_compile(nau_ctx* c, const nau_vm_instr* code, int n, int result, std::vector<VmIns>& prog,
                VmShape& out_shape, std::string& err) {
    std::vector<VmShape> reg(NAU_VM_MAX_REGS);
    std::vector<bool> def(NAU_VM_MAX_REGS, false);
    prog.clear();
    auto bad_reg = [&](int r) { return r < 0 || r >= NAU_VM_MAX_REGS; };
    for (int pc = 0; pc < n; ++pc) {
        const nau_vm_instr& in = code[pc];
        VmIns I{};
        I.op = in.op;
        I.dst = in.dst;
        I.a = in.a;
        I.b = in.b;
        I.field = in.field;
        for (int q = 0; q < 9; ++q) I.imm[q] = in.imm[q];
        if (in.op < 0 || in.op >= NAU_VM_OP_COUNT || bad_reg(in.dst)) {
            err = "nau_eval: bad instruction " + std::to_string(pc);
            return false;
        }
        const bool unary = in.op == NAU_VM_NEG || (in.op >= NAU_VM_EXP && in.op <= NAU_VM_NORM);
        // (NAU_VM_RAND is binary: the two bounds)
        const bool loads = in.op == NAU_VM_LOAD_FIELD || in.op == NAU_VM_LOAD_CONST;
        if (!loads && (bad_reg(in.a) || !def[in.a] || (!unary && (bad_reg(in.b) || !def[in.b])))) {
            err = "nau_eval: instruction " + std::to_string(pc) + " reads an undefined register";
            return false;
        }
        VmShape A = loads ? VmShape{} : reg[in.a];
        VmShape B = (loads || unary) ? VmShape{} : reg[in.b];
        I.ar = A.rows;
        I.ac = A.cols;
        I.br = B.rows;
        I.bc = B.cols;
        VmShape D;
        auto mismatch = [&](const char* sym) {
            err = std::string("operator '") + sym + "': incompatible shapes " + shape_str(A) +
                  " and " + shape_str(B);
            return false;
        };
        switch (in.op) {
            case NAU_VM_LOAD_FIELD:
                if (in.field < 0 || in.field >= (int)c->fields.size() || !c->fields[in.field].live) {
                    err = "nau_eval: bad field id";
                    return false;
                }
                D = {c->fields[in.field].rows, c->fields[in.field].cols};
                break;
            case NAU_VM_LOAD_CONST:
                if (in.rows < 1 || in.rows > 3 || in.cols < 1 || in.cols > 3) {
                    err = "nau_eval: constant shape must be within 3x3";
                    return false;
                }
                D = {in.rows, in.cols};
                break;
            case NAU_VM_ADD:
            case NAU_VM_SUB:  // tensor.cpp:43-51
                if (A.rows != B.rows || A.cols != B.cols) return mismatch(op_symbol(in.op));
                D = A;
                break;
            case NAU_VM_MUL:  // tensor.cpp:55-60
                if (A.scalar()) D = B;
                else if (B.scalar()) D = A;
                else if (A.cols == B.rows) D = {A.rows, B.cols};
                else return mismatch("*");
                break;
            case NAU_VM_DIV:  // tensor.cpp:62-66
                if (B.scalar()) D = A;
                else if (A.rows == B.rows && A.cols == B.cols) D = A;
                else return mismatch("/");
                break;
            case NAU_VM_POW:
            case NAU_VM_MIN:
            case NAU_VM_MAX:  // elementwise_binary, tensor.cpp:25-37
                if (A.scalar() && !B.scalar()) D = B;
                else if (B.scalar() && !A.scalar()) D = A;
                else if (A.rows == B.rows && A.cols == B.cols) D = A;
                else return mismatch(op_symbol(in.op));
                break;
            case NAU_VM_LT:
            case NAU_VM_GT:
            case NAU_VM_LE:
            case NAU_VM_GE:
            case NAU_VM_EQ:
            case NAU_VM_NE:  // tensor.cpp:72-86
                if (!A.scalar() || !B.scalar()) return mismatch("comparison");
                D = {1, 1};
                break;
            case NAU_VM_JOIN:  // ast.cpp:111-120
                if (A.cols != 1 || !B.scalar() || A.rows >= 3) {
                    err = "operator '|': cannot append a " + shape_str(B) + " component to a " +
                          shape_str(A) + " value";
                    return false;
                }
                D = {A.rows + 1, 1};
                break;
            case NAU_VM_NORM:
                D = {1, 1};
                break;
            case NAU_VM_RAND:  // Tensor::value() on both bounds (tensor.hpp:50-53)
                if (!A.scalar() || !B.scalar()) {
                    err = "expected a scalar, got a " + shape_str(A.scalar() ? B : A) + " tensor";
                    return false;
                }
                D = {1, 1};
                break;
            case NAU_VM_DOT:  // tensor.cpp:107-110
                if (A.rows != B.rows || A.cols != B.cols) return mismatch("dot");
                D = {1, 1};
                break;
            default:  // elementwise unary
                D = A;
                break;
        }
        I.rows = D.rows;
        I.cols = D.cols;
        reg[in.dst] = D;
        def[in.dst] = true;
        prog.push_back(I);
    }
    if (bad_reg(result) || !def[result]) {
        err = "nau_eval: result register undefined";
        return false;
    }
    out_shape = reg[result];
    VmIns tail{};
    tail.rows = out_shape.rows;
    tail.cols = out_shape.cols;
    prog.push_back(tail);
    return true;
}

static void launch_vm(nau_ctx* c, const VmIns* d_prog, int nins, int result, double* out) {
    if (c->n == 0) return;
    VmFields f{};
    for (size_t q = 0; q < c->fields.size() && q < (size_t)kMaxFields; ++q) f.p[q] = c->fields[q].d;
    const int blocks = (int)((c->n + kVmThreads - 1) / kVmThreads);
    k_vm<<<blocks, kVmThreads, 0, c->stream>>>(d_prog, nins, result, c->n, f, c->d_active,
                                               c->d_orig, out, c->d_err, c->d_rng, c->rng_len,
                                               c->rng_seed);
    c->launches++;
}

}  // namespace nau

extern "C" nau_status nau_eval(nau_ctx* c, const nau_vm_instr* code, int n_instr, int result,
                               int out_field) {
    if (!c || !code || n_instr <= 0 || n_instr > NAU_VM_MAX_INSTR) {
        if (c) c->last_error = "nau_eval: empty or oversized program";
        return NAU_ERR_ARG;
    }
    if (out_field < 0 || out_field >= (int)c->fields.size() || !c->fields[out_field].live) {
        c->last_error = "nau_eval: bad output field";
        return NAU_ERR_ARG;
    }
    std::vector<nau::VmIns> prog;
    nau::VmShape shape;
    std::string err;
    if (!nau::vm_compile(c, code, n_instr, result, prog, shape, err)) {
        c->last_error = err;
        c->last_bad = -1;
        return NAU_ERR_RUNTIME;
    }
    nau::FieldBuf& of = c->fields[out_field];
    if (shape.rows != of.rows || shape.cols != of.cols) {  // case.cpp:41-44
        c->last_error = "LHS field is " + std::to_string(of.rows) + "x" + std::to_string(of.cols) +
                        " but RHS produced " + std::to_string(shape.rows) + "x" +
                        std::to_string(shape.cols);
        c->last_bad = -1;
        return NAU_ERR_RUNTIME;
    }
    const size_t bytes = prog.size() * sizeof(nau::VmIns);
    if (c->vm_len < bytes) {
        if (c->d_vm) cudaFree(c->d_vm);
        c->d_vm = nullptr;
        c->vm_len = 0;
        if (cudaMalloc(&c->d_vm, bytes) != cudaSuccess) {
            c->last_error = "nau_eval: device allocation failed";
            return NAU_ERR_CUDA;
        }
        c->vm_len = bytes;
    }
    // the host vector is pageable: the copy is staged before cudaMemcpyAsync returns
    if (cudaMemcpyAsync(c->d_vm, prog.data(), bytes, cudaMemcpyHostToDevice, c->stream) != cudaSuccess) {
        c->last_error = "nau_eval: program upload failed";
        return NAU_ERR_CUDA;
    }
    bool alias = false;  // two-phase write (case.cpp:31-54)
    for (int pc = 0; pc < n_instr; ++pc)
        alias |= code[pc].op == NAU_VM_LOAD_FIELD && code[pc].field == out_field;
    double* out = of.d;
    if (alias) {
        cudaMemcpyAsync(of.alt, of.d, sizeof(double) * c->n * of.comps(), cudaMemcpyDeviceToDevice,
                        c->stream);
        out = of.alt;
    }
    bool uses_rand = false;
    for (int pc = 0; pc < n_instr; ++pc) uses_rand |= code[pc].op == NAU_VM_RAND;
    if (uses_rand && c->rng_len < c->n) {  // a fresh RandomState: zero counters
        nau_status s = nau_set_random_state(c, c->rng_seed, nullptr);
        if (s != NAU_OK) return s;
    }
    nau::launch_vm(c, static_cast<const nau::VmIns*>(c->d_vm), n_instr, result, out);
    if (alias) std::swap(of.d, of.alt);
    if (out_field == 0) {  // r written: apply_boundary_shift + dirty (case.cpp:59-62)
        nau::launch_boundary_shift(c);
        c->dirty = true;
    }
    return NAU_OK;
}

extern "C" nau_status nau_set_random_state(nau_ctx* c, unsigned long long seed,
                                           const unsigned long long* counters) {
    c->rng_seed = seed;
    if (c->rng_len < c->n) {
        if (c->d_rng) cudaFree(c->d_rng);
        c->d_rng = nullptr;
        c->rng_len = 0;
        if (c->n > 0 && cudaMalloc(&c->d_rng, sizeof(unsigned long long) * c->n) != cudaSuccess) {
            c->last_error = "nau_set_random_state: device allocation failed";
            return NAU_ERR_CUDA;
        }
        c->rng_len = c->n;
    }
    if (c->n == 0) return NAU_OK;
    const size_t bytes = sizeof(unsigned long long) * c->n;
    cudaError_t e = counters ? cudaMemcpyAsync(c->d_rng, counters, bytes, cudaMemcpyHostToDevice, c->stream)
                             : cudaMemsetAsync(c->d_rng, 0, bytes, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        c->last_error = cudaGetErrorString(e);
        return NAU_ERR_CUDA;
    }
    return NAU_OK;
}

extern "C" nau_status nau_get_random_counters(nau_ctx* c, unsigned long long* counters) {
    if (c->n == 0) return NAU_OK;
    if (c->rng_len < c->n) {  // never drawn: zeros
        for (long i = 0; i < c->n; ++i) counters[i] = 0;
        return NAU_OK;
    }
    cudaError_t e = cudaMemcpyAsync(counters, c->d_rng, sizeof(unsigned long long) * c->n,
                                    cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        c->last_error = cudaGetErrorString(e);
        return NAU_ERR_CUDA;
    }
    return NAU_OK;
}
