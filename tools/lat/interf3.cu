// fp64 shuffle-reduction chain on CTA 0 while the other CTAs run (0) nothing,
// (1) DFMA loops, (2) SHFL loops, (3) bulk async copies global->shared,
// (4) mma.sync loops.  Cycles per (sum + max) butterfly pair.
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
__global__ void __launch_bounds__(384, 1) k(int mode, volatile int *stop, const char *src, long long *out, double *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (blockIdx.x == 0) {
        if (warp != 0) return;
        long long w0 = clock64();
        if (mode == 5) { for (int i = 0; i < 200; ++i) __nanosleep(200); }
        else if (mode == 6) { for (int i = 0; i < 200; ++i) { unsigned long long v; asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"((const unsigned long long *)src + lane) : "memory"); if (v == 77) sink[2] = 1; __nanosleep(200); } }
        else if (mode == 7) { for (int i = 0; i < 200; ++i) { unsigned long long v; asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"((const unsigned long long *)src + lane) : "memory"); if (v == 77) sink[2] = 1; } }
        else while (clock64() - w0 < 100000) {}
        double s = lane, g = lane * 0.5;
        long long c0 = clock64();
        for (int r = 0; r < 10; ++r) {
            s = wsum(s * 0.5);
            g = wmax(g * 0.5);
        }
        long long c1 = clock64() + (s + g == 1.2345 ? 1 : 0);
        if (lane == 0) { out[0] = c1 - c0; sink[0] = s + g; *stop = 1; }
        return;
    }
    if (mode == 0 || mode >= 5) return;
    if (mode == 1) {
        double a = threadIdx.x, b = 1.0001;
        while (!*stop) for (int i = 0; i < 64; ++i) a = fma(a, b, 0.5);
        if (a == 1.2345) sink[1] = a;
    } else if (mode == 2) {
        int v = threadIdx.x;
        while (!*stop) for (int i = 0; i < 64; ++i) v += __shfl_xor_sync(0xffffffffu, v, i & 31);
        if (v == 12345) sink[1] = v;
    } else if (mode == 3) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(1));
            unsigned ph = 0;
            size_t off = (size_t)blockIdx.x * 65536;
            while (!*stop) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(65536) : "memory");
                for (int i = 0; i < 16; ++i)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"((unsigned)__cvta_generic_to_shared(sm + i * 4096)), "l"(src + (off + i * 4096) % (1ull << 30)), "r"(4096), "r"((unsigned)__cvta_generic_to_shared(&bar)) : "memory");
                asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(ph) : "memory");
                ph ^= 1;
                off += 148 * 65536;
            }
        }
    } else if (mode == 4) {
        float c[4] = {0, 0, 0, 0};
        unsigned a = threadIdx.x, b = 3;
        while (!*stop)
            for (int i = 0; i < 64; ++i)
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
                             : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a), "r"(b));
        if (c[0] == 1.2345f) sink[1] = c[0];
    }
}
int main() {
    int *stop; char *src; long long *out; double *sink;
    cudaMalloc(&stop, 4); cudaMalloc(&src, 1ull << 30); cudaMalloc(&out, 8); cudaMalloc(&sink, 64);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
    const char *names[] = {"others idle", "others DFMA loops", "others SHFL loops", "others bulk async copies (HBM)", "others mma.sync loops", "worker nanosleeps first", "worker polls + nanosleeps first", "worker polls first"};
    for (int mode = 0; mode < 8; ++mode) {
        long long h, best = -1;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(stop, 0, 4);
            k<<<148, 384, 70 * 1024>>>(mode, stop, src, out, sink);
            cudaDeviceSynchronize();
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            best = best < 0 || h < best ? h : best;
        }
        printf("%-34s %lld cycles per (sum + max) pair\n", names[mode], best / 10);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
