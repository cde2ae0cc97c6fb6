// HBM -> shared-memory streaming with cp.async.bulk on every SM: aggregate GB/s
// as a function of the copy size (bytes per cp.async.bulk instruction) and of
// the ring (slots x slot bytes) each CTA keeps in flight.  One producer warp
// per CTA (lane-parallel issue, like decode_ll.cu's producer), one consumer
// warp that waits for each slot and releases it at once.  Each CTA streams its
// own disjoint 4 MiB region (evict-first).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(sa(b)), "r"(ph)
        : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            sa(dst)),
        "l"(src), "r"(bytes), "r"(sa(bar)), "l"(pol)
        : "memory");
}

__global__ void __launch_bounds__(64, 1) k(const unsigned char *src, size_t per_cta, int slots, int slot_bytes,
                                           int copy_bytes, long long *out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ uint64_t full[16], empty[16];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < slots; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned char *base = src + (size_t)blockIdx.x * per_cta;
    const int pieces = (int)(per_cta / slot_bytes), ncopy = slot_bytes / copy_bytes;
    long long t0 = clock64();
    if (warp == 0) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        for (int pc = 0; pc < pieces; ++pc) {
            const int s = pc % slots;
            if (pc >= slots) mbar_wait(&empty[s], ((pc / slots) - 1) & 1);
            if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)(ncopy * copy_bytes));
            __syncwarp();
            for (int i = lane; i < ncopy; i += 32)
                bulk(sm + (size_t)s * slot_bytes + (size_t)i * copy_bytes,
                     base + (size_t)pc * slot_bytes + (size_t)i * copy_bytes, copy_bytes, &full[s], pol);
            __syncwarp();
        }
    } else {
        for (int pc = 0; pc < pieces; ++pc) {
            const int s = pc % slots;
            mbar_wait(&full[s], (pc / slots) & 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
    const size_t per_cta = 4u << 20;
    const int G = 148;
    unsigned char *src;
    long long *out;
    cudaMalloc(&src, per_cta * G);
    cudaMemset(src, 1, per_cta * G);
    cudaMalloc(&out, G * sizeof(long long));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int ring[][2] = {{2, 65536}, {3, 65536}, {2, 49152}, {4, 32768}, {6, 32768}, {8, 16384}, {12, 16384}};
    const int copies[] = {512, 1024, 2048, 4096, 8192, 16384, 32768, 65536};
    for (auto &r : ring)
        for (int cb : copies) {
            if (cb > r[1]) continue;
            const int smem = r[0] * r[1];
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k<<<G, 64, smem>>>(src, per_cta, r[0], r[1], cb, out);
            cudaEventRecord(a);
            k<<<G, 64, smem>>>(src, per_cta, r[0], r[1], cb, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            printf("ring %2d x %5d  copy %5d B: %7.1f GB/s  (%s)\n", r[0], r[1], cb, per_cta * G / (ms * 1e6),
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
