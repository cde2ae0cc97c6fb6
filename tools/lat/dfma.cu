// FP64 vs FP32 FMA throughput per SM: one CTA per SM, W warps, 8 independent
// chains per thread.  Reports lane-FMAs per clock per SM.
#include <cstdio>
template <typename F>
__global__ void k(F *out, long long *cyc, int iters) {
    F a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (F)(threadIdx.x + i);
    const F m = (F)1.0000001, c = (F)0.5;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = a[i] * m + c;
    __syncthreads();
    long long t1 = clock64();
    F s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double *od; float *of; long long *cyc, h;
    cudaMalloc(&od, 148 * 1024 * 8); cudaMalloc(&of, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    for (int w : {1, 2, 4, 8, 16}) {
        k<double><<<148, 32 * w>>>(od, cyc, iters); cudaDeviceSynchronize();
        k<double><<<148, 32 * w>>>(od, cyc, iters); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        double fp64 = (double)iters * 8 * 32 * w / h;
        k<float><<<148, 32 * w>>>(of, cyc, iters); cudaDeviceSynchronize();
        k<float><<<148, 32 * w>>>(of, cyc, iters); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        double fp32 = (double)iters * 8 * 32 * w / h;
        printf("warps/SM %2d: FP64 %.2f  FP32 %.2f lane-FMA/clk/SM\n", w, fp64, fp32);
    }
    return 0;
}
