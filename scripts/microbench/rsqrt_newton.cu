// Accuracy of MUFU-based fp64 rsqrt / rcp with 0, 1, 2 Newton steps (max relative error vs fp64 division/sqrt).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

template <int IT> __device__ double rsq(double x) {
    double r; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    for (int i = 0; i < IT; ++i) { const double e = fma(-x * r, r, 1.0); r = fma(0.5 * r, e, r); }
    return r;
}
template <int IT> __device__ double rcp(double x) {
    double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    for (int i = 0; i < IT; ++i) { const double e = fma(-x, r, 1.0); r = fma(r, e, r); }
    return r;
}
__global__ void k(double* out, int n) {
    double m[6] = {0, 0, 0, 0, 0, 0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double x = ldexp(1.0 + (i % 1000003) * 1e-6, (i % 61) - 30);  // spans 2^-30 .. 2^31
        const double rs = 1.0 / sqrt(x), rc = 1.0 / x;
        m[0] = fmax(m[0], fabs(rsq<0>(x) - rs) / rs); m[1] = fmax(m[1], fabs(rsq<1>(x) - rs) / rs);
        m[2] = fmax(m[2], fabs(rsq<2>(x) - rs) / rs); m[3] = fmax(m[3], fabs(rcp<0>(x) - rc) / rc);
        m[4] = fmax(m[4], fabs(rcp<1>(x) - rc) / rc); m[5] = fmax(m[5], fabs(rcp<2>(x) - rc) / rc);
    }
    for (int j = 0; j < 6; ++j) {
        unsigned long long* p = reinterpret_cast<unsigned long long*>(out + j);
        atomicMax(p, __double_as_longlong(m[j]));  // positive doubles order like their bits
    }
}
int main() {
    double* d; cudaMalloc(&d, 6 * sizeof(double)); cudaMemset(d, 0, 6 * sizeof(double));
    k<<<1184, 256>>>(d, 1 << 26);
    double h[6]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("rsqrt rel err: 0 steps %.3e  1 step %.3e  2 steps %.3e\n", h[0], h[1], h[2]);
    printf("rcp   rel err: 0 steps %.3e  1 step %.3e  2 steps %.3e\n", h[3], h[4], h[5]);
    return 0;
}
