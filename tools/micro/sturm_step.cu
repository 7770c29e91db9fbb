// Latency of one Sturm-count step q <- (d - x) - e2 / q on sm_100a, for
// several reciprocal implementations (single dependent chain, 1 warp).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_mufu_nr1(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    return r * fma(-q, r, 2.0);
}
__device__ __forceinline__ double rcp_mufu(double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    return r;
}
__device__ __forceinline__ double rcp_f32_nr2(double q) {
    double r = static_cast<double>(__frcp_rn(static_cast<float>(q)));
    r = r * fma(-q, r, 2.0);
    return r * fma(-q, r, 2.0);
}
template <int M>
__global__ void chain(double* out, double d, double e2, double x, int n, long long* cyc) {
    double q = out[threadIdx.x] + 1.0;
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        double r;
        if constexpr (M == 0) r = e2 / q;
        else if constexpr (M == 1) r = e2 * rcp_mufu_nr1(q);
        else if constexpr (M == 2) r = e2 * rcp_mufu(q);
        else r = e2 * rcp_f32_nr2(q);
        q = (d - x) - r;
        if (fabs(q) < 1e-300) q = -1e-300;
    }
    const long long t1 = clock64();
    out[threadIdx.x] = q;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double* out;
    long long *cyc, h;
    cudaMalloc(&out, 8 * 32);
    cudaMemset(out, 0, 8 * 32);
    cudaMalloc(&cyc, 8);
    const int n = 10000;
    const char* names[] = {"IEEE division", "rcp.approx + 1 Newton", "rcp.approx only", "f32 rcp + 2 Newton"};
    for (int m = 0; m < 4; ++m) {
        for (int rep = 0; rep < 2; ++rep) {
            if (m == 0) chain<0><<<1, 32>>>(out, 3.0, 0.5, 0.1, n, cyc);
            if (m == 1) chain<1><<<1, 32>>>(out, 3.0, 0.5, 0.1, n, cyc);
            if (m == 2) chain<2><<<1, 32>>>(out, 3.0, 0.5, 0.1, n, cyc);
            if (m == 3) chain<3><<<1, 32>>>(out, 3.0, 0.5, 0.1, n, cyc);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("%-24s %.1f cycles per step\n", names[m], double(h) / n);
    }
    return 0;
}
