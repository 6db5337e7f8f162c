// Accuracy probe for the FP64 reciprocal-square-root estimate (MUFU.RSQ64H via
// rsqrt.approx.ftz.f64) and the one-step Newton forms built on it in fast.cu.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_acc.cu -o build/mufu_acc
#include <cstdio>
#include <cmath>
#include <cstring>
#include <cuda_runtime.h>

__global__ void probe(double lo, double hi, long n, unsigned long long* out) {
    const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    double emax = 0.0, q2max = 0.0, q3max = 0.0;
    for (long k = i; k < n; k += (long)gridDim.x * blockDim.x) {
        // log-uniform x in [lo, hi) with scrambled low mantissa bits
        const double f = (double)k / (double)n;
        double x = lo * pow(hi / lo, f);
        unsigned long long b = __double_as_longlong(x) ^ ((k * 0x9E3779B97F4A7C15ull) >> 40);
        x = __longlong_as_double(b);
        double y;
        asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
        const double e = fma(-x * y, y, 1.0);
        const double ref = 1.0 / sqrt(x);  // IEEE sqrt and division: correctly rounded pieces
        const double q2 = fma(0.5 * y, e, y);
        const double q3 = fma(fma(0.375, e, 0.5), y * e, y);
        emax = fmax(emax, fabs(e));
        q2max = fmax(q2max, fabs(q2 - ref) / ref);
        q3max = fmax(q3max, fabs(q3 - ref) / ref);
    }
    atomicMax(out + 0, (unsigned long long)__double_as_longlong(emax));
    atomicMax(out + 1, (unsigned long long)__double_as_longlong(q2max));
    atomicMax(out + 2, (unsigned long long)__double_as_longlong(q3max));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 3 * sizeof(unsigned long long));
    const double ranges[][2] = {{1e-12, 1e-3}, {0.5, 2.0}, {1e-300, 1e300}};
    for (auto& r : ranges) {
        cudaMemset(d, 0, 3 * sizeof(unsigned long long));
        probe<<<592, 256>>>(r[0], r[1], 1L << 28, d);
        unsigned long long h[3];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double v[3];
        for (int k = 0; k < 3; ++k) memcpy(&v[k], &h[k], 8);
        printf("x in [%g, %g): max|e| = %.3e (2^%.2f)  quadratic rel err %.3e  cubic rel err %.3e\n",
               r[0], r[1], v[0], log2(v[0]), v[1], v[2]);
    }
    return 0;
}
