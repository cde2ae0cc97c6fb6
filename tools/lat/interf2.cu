// Why does a 10-step fp64 shuffle chain take ~490 cycles per step inside
// decode_ll.cu?  Same chain, kernel attributes added one at a time.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__global__ void __launch_bounds__(384, 1) k(long long *out, double *sink, int worker) {
    extern __shared__ double sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128; i += blockDim.x) sm[i] = i * 0.5;
    __syncthreads();
    if (warp != worker) return;
    double s = 0, g = 0;
    long long c0 = clock64();
    for (int r = 0; r < 10; ++r) {
        s = wsum(sm[lane] + sm[lane + 32] + 0.0 * s);
        g = wmax(fmax(sm[lane + 64], sm[lane + 96]) + 0.0 * g);
    }
    long long c1 = clock64() + (s + g == 1.2345 ? 1 : 0);
    if (lane == 0) { out[blockIdx.x] = c1 - c0; sink[blockIdx.x] = s + g; }
}
int main() {
    long long *out; double *sink;
    cudaMalloc(&out, 8 * 148); cudaMalloc(&sink, 8 * 148);
    for (int cfg = 0; cfg < 4; ++cfg) {
        size_t smem = (cfg & 1) ? 200 * 1024 : 1024;
        bool pdl = cfg & 2;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        for (int rep = 0; rep < 3; ++rep) {
            cudaLaunchConfig_t c = {};
            c.gridDim = dim3(148); c.blockDim = dim3(384); c.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            c.attrs = at; c.numAttrs = pdl ? 1 : 0;
            cudaLaunchKernelEx(&c, k, out, sink, 10);
            cudaDeviceSynchronize();
        }
        long long h[148];
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
        printf("smem %6zu pdl %d: %.0f cycles per (sum + max) butterfly pair\n", smem, (int)pdl, s / 148 / 10);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
