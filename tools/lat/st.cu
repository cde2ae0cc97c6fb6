// Store-throughput microbenchmark: the block kernel's dense epilogue pattern
// (128 threads = 128 rows m; per column: one fp32 store y[col*M + m] and one
// bf16 store xb[row[col]*M + m]) timed with clock64.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__global__ void epi(float *y, uint16_t *xb, const int *rowmap, int M, int ncol, int mode, long long *cyc) {
    __shared__ int mi[256];
    const int et = threadIdx.x, m = blockIdx.x % (M / 128) * 128 + et;
    for (int c = et; c < ncol; c += 128) mi[c] = rowmap[c];
    __syncthreads();
    float v[16];
    for (int j = 0; j < 16; ++j) v[j] = et * 0.5f + j;
    long long t0 = clock64();
    for (int c0 = 0; c0 < ncol; c0 += 16) {
        int row[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) row[j] = mi[c0 + j];
        float *o = y + (size_t)c0 * M + m;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (mode == 0) __stcg(o + (size_t)j * M, v[j]);
            else o[(size_t)j * M] = v[j];
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint16_t b = __bfloat16_as_ushort(__float2bfloat16_rn(v[j]));
            if (mode == 0) __stcg(xb + (size_t)row[j] * M + m, b);
            else xb[(size_t)row[j] * M + m] = b;
        }
    }
    long long t1 = clock64();
    if (et == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    const int M = 768, T = 256;
    float *y; uint16_t *xb; int *rm; long long *cyc;
    cudaMalloc(&y, (size_t)T * M * 4); cudaMalloc(&xb, (size_t)T * M * 2); cudaMalloc(&rm, T * 4); cudaMalloc(&cyc, 1024 * 8);
    int h[T]; for (int i = 0; i < T; ++i) h[i] = (i * 37) % T;
    cudaMemcpy(rm, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 2; ++mode)
        for (int grid : {1, 24, 148}) {
            for (int ncol : {16, 64}) {
                epi<<<grid, 128>>>(y, xb, rm, M, ncol, mode, cyc);
                epi<<<grid, 128>>>(y, xb, rm, M, ncol, mode, cyc);
                long long c[148]; cudaMemcpy(c, cyc, grid * 8, cudaMemcpyDeviceToHost);
                long long mx = 0; for (int i = 0; i < grid; ++i) mx = c[i] > mx ? c[i] : mx;
                printf("mode %d grid %3d ncol %2d: %lld cycles (cta0 %lld)\n", mode, grid, ncol, mx, c[0]);
            }
        }
    return 0;
}
