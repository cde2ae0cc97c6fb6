// float->double conversion (F2F.F64.F32) and LDS->F2F->DFMA chain costs per warp.
#include <cstdio>
__global__ void conv(double *out, long long *cyc, int iters) {
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 0.25f + i;
    double acc = 0.0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { acc += (double)f[i]; f[i] += 1.0f; }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void conv_only(double *out, long long *cyc, int iters) {
    float f[8];
    double d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { f[i] = threadIdx.x * 0.25f + i; d[i] = 0; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { d[i] = (double)f[i]; f[i] = __int_as_float(__float_as_int(f[i]) ^ (int)(d[i] != 0.0)); }
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += d[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double *o; long long *c, h; cudaMalloc(&o, 148 * 1024 * 8); cudaMalloc(&c, 148 * 8);
    const int iters = 2048;
    for (int w : {1, 4, 16}) {
        conv_only<<<148, 32 * w>>>(o, c, iters); cudaDeviceSynchronize();
        conv_only<<<148, 32 * w>>>(o, c, iters); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("warps/SM %2d: F2F.F64 %.2f lane-conv/clk/SM (%.1f cycles per warp-conversion per warp)\n", w,
               (double)iters * 8 * 32 * w / h, (double)h / (iters * 8));
    }
    return 0;
}
