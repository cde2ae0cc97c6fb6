// Straight-line code (cold i-cache) executed by one warp of CTA 0 while the
// other 147 CTAs (a) idle, (b) poll global words with ld.relaxed.gpu,
// (c) poll with nanosleep(128), (d) stream a large buffer.  If instruction
// fetch shares the congested L2 path, (b)-(d) slow the straight-line code.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/lat/icache_load.cu -o tools/lat/icache_load
#include <cstdio>
#include <cstdint>
#define F4(i) a0 = fmaf(a0, 1.0001f, (float)(i)); a1 = fmaf(a1, 0.9999f, (float)(i)); a2 = fmaf(a2, 1.0002f, (float)(i)); a3 = fmaf(a3, 0.9998f, (float)(i));
#define F16(i) F4(i) F4(i + 1) F4(i + 2) F4(i + 3)
#define F64(i) F16(i) F16(i + 4) F16(i + 8) F16(i + 12)
#define F256(i) F64(i) F64(i + 16) F64(i + 32) F64(i + 48)
#define F1024(i) F256(i) F256(i + 64) F256(i + 128) F256(i + 192)

__global__ void __launch_bounds__(384, 1) k(int mode, volatile int *stop, const unsigned long long *buf, size_t nbuf,
                                            long long *out, float *sink) {
    if (blockIdx.x == 0) {
        if (threadIdx.x >= 32) return;
        // wait a bit so the others are running
        long long w0 = clock64();
        while (clock64() - w0 < 200000) {}
        float a0 = sink[2] + threadIdx.x, a1 = sink[3], a2 = sink[4], a3 = sink[5];
        long long c0;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0) : "f"(a0), "f"(a1), "f"(a2), "f"(a3) : "memory");
        F1024(0) F1024(1) F1024(2) F1024(3)
        long long c1;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1) : "f"(a0), "f"(a1), "f"(a2), "f"(a3) : "memory");
        if (threadIdx.x == 0) { out[0] = c1 - c0; sink[0] = a0 + a1 + a2 + a3; *stop = 1; }
        return;
    }
    if (mode == 0) return;
    unsigned long long acc = 0;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    while (!*stop) {
        unsigned long long v;
        if (mode == 3) {
            for (int r = 0; r < 16; ++r) {
                asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(v) : "l"(buf + (i % nbuf)) : "memory");
                acc += v;
                i += 148 * 384;
            }
        } else {
            asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(buf + (i % 8192)) : "memory");
            acc += v;
            if (mode == 2) __nanosleep(128);
        }
    }
    if (acc == 12345) sink[1] = 1.f;
}

int main() {
    int *stop; unsigned long long *buf; long long *out; float *sink;
    const size_t nbuf = (size_t)1 << 27;  // 1 GiB
    cudaMalloc(&stop, 4); cudaMalloc(&buf, nbuf * 8); cudaMalloc(&out, 8); cudaMalloc(&sink, 64); cudaMemset(sink, 0, 64);
    cudaMemset(buf, 0, nbuf * 8);
    const char *names[] = {"others idle", "others poll (ld.relaxed.gpu, 8K words)", "others poll + nanosleep(128)", "others stream 1 GiB (HBM)"};
    for (int mode = 0; mode < 4; ++mode) {
        long long best = 0, h;
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemset(stop, 0, 4);
            k<<<148, 384>>>(mode, stop, buf, nbuf, out, sink);
            cudaDeviceSynchronize();
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            best = rep == 0 ? h : (h < best ? h : best);
        }
        printf("%-42s 4096 straight-line FMAs (cold i-cache): %lld cycles\n", names[mode], best);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
