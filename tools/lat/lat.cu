// Latency microbenchmarks (debug tool): dependent-chain costs of the memory
// operations the fused kernels' critical paths are made of.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void chase(const int *__restrict__ next, int n, int iters, long long *out, int mode) {
    int i = 0;
    long long c0 = clock64();
    unsigned long long g0 = gt();
    for (int k = 0; k < iters; ++k) {
        if (mode == 0) i = __ldcg(next + i);
        else if (mode == 1) i = __ldg(next + i);
        else if (mode == 2) { i = *(volatile const int *)(next + i); }
        else if (mode == 3) { __threadfence(); i = __ldcg(next + i); }
        else if (mode == 4) { i = atomicAdd((int *)next + i, 0); }
    }
    long long c1 = clock64();
    unsigned long long g1 = gt();
    if (threadIdx.x == 0) { out[0] = (c1 - c0) / iters; out[1] = (long long)(g1 - g0) / iters; out[2] = i; }
}

__global__ void fence_cost(int *buf, int iters, long long *out) {
    long long c0 = clock64();
    unsigned long long g0 = gt();
    for (int k = 0; k < iters; ++k) { buf[threadIdx.x] = k; __threadfence(); }
    long long c1 = clock64();
    unsigned long long g1 = gt();
    if (threadIdx.x == 0) { out[0] = (c1 - c0) / iters; out[1] = (long long)(g1 - g0) / iters; }
}

int main1() {
    int n = 1 << 20;
    int *d; long long *o; cudaMalloc(&d, n * 4); cudaMalloc(&o, 64);
    int *h = new int[n];
    for (int i = 0; i < n; ++i) h[i] = (int)(((long long)i * 7919 + 4099) % n);  // pseudo-random permutation-ish chain
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    const char *names[] = {"ldcg", "ldg", "volatile", "fence+ldcg", "atomicAdd"};
    for (int mode = 0; mode < 5; ++mode) {
        chase<<<1, 1>>>(d, n, 2000, o, mode);  // warm (L2 resident: 4 MB)
        chase<<<1, 1>>>(d, n, 2000, o, mode);
        long long r[3]; cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost);
        printf("%-12s %lld cycles  %lld ns per dependent op\n", names[mode], r[0], r[1]);
    }
    for (int t : {1, 32, 128}) {
        fence_cost<<<1, t>>>(d, 2000, o);
        long long r[2]; cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
        printf("store+threadfence x%d threads: %lld cycles %lld ns\n", t, r[0], r[1]);
    }
    int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    printf("clock rate attr %d kHz\n", clk);
    return 0;
}
// (appended) globaltimer granularity and loaded-latency tests
__global__ void gt_res(long long *out) {
    unsigned long long t[64];
    for (int i = 0; i < 64; ++i) t[i] = gt();
    for (int i = 0; i < 63; ++i) out[i] = (long long)(t[i + 1] - t[i]);
}
__global__ void loaded(const int *next, int iters, long long *out, const float4 *big, size_t nbig, float *sink) {
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0) {
            int i = 0;
            // let the streamers ramp up
            long long w = clock64(); while (clock64() - w < 20000) {}
            long long c0 = clock64();
            for (int k = 0; k < iters; ++k) i = __ldcg(next + i);
            long long c1 = clock64();
            out[0] = (c1 - c0) / iters; out[2] = i;
        }
        return;
    }
    float4 acc = make_float4(0, 0, 0, 0);
    for (size_t j = (size_t)(blockIdx.x - 1) * blockDim.x + threadIdx.x; j < nbig; j += (size_t)(gridDim.x - 1) * blockDim.x) {
        float4 v = __ldcs(big + j); acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (acc.x == 1234.5f) sink[0] = acc.y + acc.z + acc.w;
}
int main2() {
    long long *o; cudaMalloc(&o, 64 * 8);
    gt_res<<<1, 1>>>(o);
    long long r[63]; cudaMemcpy(r, o, 63 * 8, cudaMemcpyDeviceToHost);
    printf("globaltimer deltas:"); for (int i = 0; i < 20; ++i) printf(" %lld", r[i]); printf("\n");
    int n = 1 << 20; int *d; cudaMalloc(&d, n * 4);
    int *h = new int[n]; for (int i = 0; i < n; ++i) h[i] = (int)(((long long)i * 7919 + 4099) % n);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    size_t nbig = (size_t)2 << 30 >> 4; float4 *big; cudaMalloc(&big, nbig * 16); cudaMemset(big, 0, nbig * 16);
    float *sink; cudaMalloc(&sink, 4);
    for (int grid : {2, 148, 296}) {
        loaded<<<grid, 512>>>(d, 3000, o, big, nbig, sink);
        loaded<<<grid, 512>>>(d, 3000, o, big, nbig, sink);
        long long q[3]; cudaMemcpy(q, o, 24, cudaMemcpyDeviceToHost);
        printf("ldcg chase under %d streaming CTAs: %lld cycles\n", grid - 1, q[0]);
    }
    return 0;
}
int main() { main1(); return main2(); }
