// Cycles per ring piece of the LL decoder's GEMV (decode_ll.cu piece_gemv),
// shared-memory operands only (no HBM, no LL polls): 148 CTAs x 8 compute
// warps, each loops over the same piece.  Modes: 0 = full piece (mma K-split
// + cross-warp reduction + 2 barriers), 1 = mma loop only, 2 = mma loop with
// ldmatrix A fragments.  Shapes: up piece (32 rows, K=768), down piece (10
// rows, K=3072).
#include <cstdio>
#include <cstdint>
constexpr int kCWarps = 8, kCThreads = 256;
__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"r"(kCThreads) : "memory"); }

// MODE 3: every warp covers all m-tiles (rows <= 32) over K / 8 with
// ldmatrix A fragments; two independent accumulator chains per warp (one per
// m-tile, or even / odd k-steps when there is one m-tile); B loaded once per
// k-step.  Full reduction + barriers as mode 0.
__device__ __forceinline__ float piece3(const unsigned char *A, int apitch, int nrows, const unsigned char *B,
                                        int bpitch, int K, float *red, int ct) {
    const int w = ct >> 5, lane = ct & 31, g = lane >> 2, t4 = lane & 3;
    const int mt = nrows > 16 ? 2 : 1;
    const int KS = K / 16, k0 = KS * w / kCWarps, k1 = KS * (w + 1) / kCWarps;
    const int lr0 = min(lane & 15, nrows - 1), lr1 = min(16 + (lane & 15), nrows - 1);
    const uint32_t ab0 = (uint32_t)__cvta_generic_to_shared(A + (size_t)lr0 * apitch + (lane >> 4) * 16);
    const uint32_t ab1 = (uint32_t)__cvta_generic_to_shared(A + (size_t)lr1 * apitch + (lane >> 4) * 16);
    const unsigned char *bp = B + (size_t)g * bpitch + t4 * 4;
    float c[4] = {0.f, 0.f, 0.f, 0.f}, d[4] = {0.f, 0.f, 0.f, 0.f};
    if (mt == 2) {
#pragma unroll 2
        for (int ks = k0; ks < k1; ++ks) {
            uint32_t a0, a1, a2, a3, e0, e1, e2, e3;
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                         : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(ab0 + ks * 32));
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                         : "=r"(e0), "=r"(e1), "=r"(e2), "=r"(e3) : "r"(ab1 + ks * 32));
            const uint32_t b0 = *reinterpret_cast<const uint32_t *>(bp + ks * 32);
            const uint32_t b1 = *reinterpret_cast<const uint32_t *>(bp + ks * 32 + 16);
            mma_bf16(c, a0, a1, a2, a3, b0, b1);
            mma_bf16(d, e0, e1, e2, e3, b0, b1);
        }
    } else {
        int ks = k0;
#pragma unroll 2
        for (; ks + 1 < k1; ks += 2) {
            uint32_t a0, a1, a2, a3, e0, e1, e2, e3;
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                         : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(ab0 + ks * 32));
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                         : "=r"(e0), "=r"(e1), "=r"(e2), "=r"(e3) : "r"(ab0 + ks * 32 + 32));
            const uint32_t b0 = *reinterpret_cast<const uint32_t *>(bp + ks * 32);
            const uint32_t b1 = *reinterpret_cast<const uint32_t *>(bp + ks * 32 + 16);
            const uint32_t b2 = *reinterpret_cast<const uint32_t *>(bp + ks * 32 + 32);
            const uint32_t b3 = *reinterpret_cast<const uint32_t *>(bp + ks * 32 + 48);
            mma_bf16(c, a0, a1, a2, a3, b0, b1);
            mma_bf16(d, e0, e1, e2, e3, b2, b3);
        }
        if (ks < k1) {
            uint32_t a0, a1, a2, a3;
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                         : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(ab0 + ks * 32));
            mma_bf16(c, a0, a1, a2, a3, *reinterpret_cast<const uint32_t *>(bp + ks * 32),
                     *reinterpret_cast<const uint32_t *>(bp + ks * 32 + 16));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) { c[i] += d[i]; d[i] = 0.f; }
    }
    float *rw = red + w * 256;
    rw[g * 8 + 2 * t4] = c[0];
    rw[g * 8 + 2 * t4 + 1] = c[1];
    rw[(g + 8) * 8 + 2 * t4] = c[2];
    rw[(g + 8) * 8 + 2 * t4 + 1] = c[3];
    if (mt == 2) {
        rw[128 + g * 8 + 2 * t4] = d[0];
        rw[128 + g * 8 + 2 * t4 + 1] = d[1];
        rw[128 + (g + 8) * 8 + 2 * t4] = d[2];
        rw[128 + (g + 8) * 8 + 2 * t4 + 1] = d[3];
    }
    csync();
    float v = 0.f;
    if (ct < mt * 128) {
#pragma unroll
        for (int z = 0; z < kCWarps; ++z) v += red[z * 256 + ct];
    }
    csync();
    return v;
}

template <int MODE>
__device__ __forceinline__ float piece(const unsigned char *A, int apitch, int nrows, const unsigned char *B, int bpitch,
                                       int K, float *red, int ct) {
    const int w = ct >> 5, lane = ct & 31, g = lane >> 2, t4 = lane & 3;
    const int mt = nrows > 16 ? 2 : 1, S = kCWarps / mt;
    const int m = w / S, s = w - m * S;
    const int KS = K / 16, k0 = KS * s / S, k1 = KS * (s + 1) / S;
    const int r0 = min(m * 16 + g, nrows - 1), r1 = min(m * 16 + g + 8, nrows - 1);
    const unsigned char *a0p = A + (size_t)r0 * apitch + t4 * 4;
    const unsigned char *a1p = A + (size_t)r1 * apitch + t4 * 4;
    const unsigned char *bp = B + (size_t)g * bpitch + t4 * 4;
    float c[4] = {0.f, 0.f, 0.f, 0.f};
    if (MODE == 4) {  // mma issue rate: register operands, 4 independent chains
        float d[4] = {0.f, 0.f, 0.f, 0.f}, e[4] = {0.f, 0.f, 0.f, 0.f}, f[4] = {0.f, 0.f, 0.f, 0.f};
        const uint32_t x = 0x3f803f80u + lane;
        for (int ks = k0; ks < k1; ks += 4) {
            mma_bf16(c, x, x, x, x, x, x);
            mma_bf16(d, x, x, x, x, x, x);
            mma_bf16(e, x, x, x, x, x, x);
            mma_bf16(f, x, x, x, x, x, x);
        }
        return c[0] + d[1] + e[2] + f[3];
    }
    if (MODE == 5) {  // the shared-memory loads of mode 1 without the mma
        uint32_t acc = 0;
#pragma unroll 4
        for (int ks = k0; ks < k1; ++ks) {
            const int o = ks * 32;
            acc += *reinterpret_cast<const volatile uint32_t *>(a0p + o) ^ *reinterpret_cast<const volatile uint32_t *>(a1p + o) ^
                   *reinterpret_cast<const volatile uint32_t *>(a0p + o + 16) ^ *reinterpret_cast<const volatile uint32_t *>(a1p + o + 16) ^
                   *reinterpret_cast<const volatile uint32_t *>(bp + o) ^ *reinterpret_cast<const volatile uint32_t *>(bp + o + 16);
        }
        return (float)acc;
    }
    if (MODE == 2) {
        // ldmatrix.x4: lanes 0-15 rows 0-15 at k, lanes 16-31 rows 0-15 at k+8
        const int lr = min(m * 16 + (lane & 15), nrows - 1);
        const uint32_t abase = (uint32_t)__cvta_generic_to_shared(A + (size_t)lr * apitch + (lane >> 4) * 16);
#pragma unroll 4
        for (int ks = k0; ks < k1; ++ks) {
            uint32_t a0, a1, a2, a3;
            asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                         : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "r"(abase + ks * 32));
            const uint32_t b0 = *reinterpret_cast<const uint32_t *>(bp + ks * 32);
            const uint32_t b1 = *reinterpret_cast<const uint32_t *>(bp + ks * 32 + 16);
            mma_bf16(c, a0, a1, a2, a3, b0, b1);
        }
    } else {
#pragma unroll 4
        for (int ks = k0; ks < k1; ++ks) {
            const int o = ks * 32;
            const uint32_t a0 = *reinterpret_cast<const uint32_t *>(a0p + o);
            const uint32_t a1 = *reinterpret_cast<const uint32_t *>(a1p + o);
            const uint32_t a2 = *reinterpret_cast<const uint32_t *>(a0p + o + 16);
            const uint32_t a3 = *reinterpret_cast<const uint32_t *>(a1p + o + 16);
            const uint32_t b0 = *reinterpret_cast<const uint32_t *>(bp + o);
            const uint32_t b1 = *reinterpret_cast<const uint32_t *>(bp + o + 16);
            mma_bf16(c, a0, a1, a2, a3, b0, b1);
        }
    }
    if (MODE != 0) return c[0] + c[1] + c[2] + c[3];
    float *rw = red + w * 128;
    rw[g * 8 + 2 * t4] = c[0];
    rw[g * 8 + 2 * t4 + 1] = c[1];
    rw[(g + 8) * 8 + 2 * t4] = c[2];
    rw[(g + 8) * 8 + 2 * t4 + 1] = c[3];
    csync();
    float v = 0.f;
    if (ct < mt * 128) {
        const int mm = ct >> 7, q = ct & 127;
        for (int z = 0; z < S; ++z) v += red[(mm * S + z) * 128 + q];
    }
    csync();
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(int K, int nrows, int iters, long long *out, float *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int ct = threadIdx.x, pitch = K * 2 + 16;
    const int ar = K > 1024 ? 16 : 32;
    unsigned char *A = sm, *B = sm + ar * pitch;
    float *red = reinterpret_cast<float *>(B + 8 * pitch);
    for (int i = ct; i < ((ar + 8) * pitch) / 4; i += 256) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u ^ (i & 7);
    __syncthreads();
    float acc = 0.f;
    long long c0 = clock64();
    for (int it = 0; it < iters; ++it) acc += MODE == 3 ? piece3(A, pitch, nrows, B, pitch, K, red, ct) : piece<MODE>(A, pitch, nrows, B, pitch, K, red, ct);
    __syncthreads();
    long long c1 = clock64();
    if (ct == 0) out[blockIdx.x] = c1 - c0;
    if (acc == 1.2345f) sink[0] = acc;
}

int main() {
    long long *out, h[148];
    float *sink;
    cudaMalloc(&out, sizeof(h));
    cudaMalloc(&sink, 4);
    const int shapes[2][2] = {{768, 32}, {3072, 10}};
    for (int s = 0; s < 2; ++s)
        for (int mode = 0; mode < 6; ++mode) {
            const int K = shapes[s][0], nrows = shapes[s][1], iters = 200;
            const size_t smem = ((K > 1024 ? 16 : 32) + 8) * (K * 2 + 16) + 8 * 256 * 4 + 256;
            auto fn = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : mode == 4 ? k<4> : k<5>;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            fn<<<148, 256, smem>>>(K, nrows, iters, out, sink);
            fn<<<148, 256, smem>>>(K, nrows, iters, out, sink);
            cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0, sum = 0;
            for (int i = 0; i < 148; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
            printf("K=%d rows=%d mode=%d cycles/piece avg %.0f max %.0f err=%s\n", K, nrows, mode,
                   (double)sum / 148 / iters, (double)mx / iters, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
