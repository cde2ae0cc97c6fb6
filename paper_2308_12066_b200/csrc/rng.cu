// rng.cu — the reference's synthetic weights, generated on the device.
//
// Bit-exact restatement of rng.py:15-93 (SplitMix64-seeded xoshiro256**,
// fill = lo + span*((r>>11)*2^-53) with every fp64 op rounded, no FMA) and of
// core.py:200-211 (one substream per matrix: derive_seed(seed, tag, block,
// expert)).  Values are rounded fp64 -> fp32 (RNE) and, for bf16 storage,
// fp32 -> bf16 (RNE).  xoshiro is sequential within a matrix, so one thread
// owns one matrix; thousands of matrices run in parallel.
#include "common.cuh"
#include "rng.h"

namespace pgmoe {

__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t derive_seed(uint64_t base, const int64_t *tags, int ntags) {
    const uint64_t golden = 0x9E3779B97F4A7C15ULL;
    uint64_t x = base;
    for (int i = 0; i < ntags; ++i) {
        x = mix64(x + golden);
        x = mix64(x ^ static_cast<uint64_t>(tags[i]));
    }
    return x;
}

uint64_t matrix_seed(uint64_t seed, int tag, int block, int expert) {
    const int64_t tags[3] = {tag, block, expert};
    return derive_seed(seed, tags, 3);
}

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

template <int DT>
__global__ void gen_kernel(const GenJob *jobs, int njobs) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= njobs) return;
    const GenJob job = jobs[j];
    const uint64_t golden = 0x9E3779B97F4A7C15ULL;
    uint64_t s0, s1, s2, s3, sm = job.seed;
    sm += golden; s0 = mix64(sm);
    sm += golden; s1 = mix64(sm);
    sm += golden; s2 = mix64(sm);
    sm += golden; s3 = mix64(sm);
    const double span = 0.2;  // 0.1 - (-0.1), exact in fp64
    const double lo = -0.1;
    auto next = [&]() -> float {
        const uint64_t r = rotl64(s1 * 5, 7) * 9;
        const uint64_t t = s1 << 17;
        s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t;
        s3 = rotl64(s3, 45);
        const double uu = __dmul_rn((double)(r >> 11), 0x1p-53);
        const double v = __dadd_rn(lo, __dmul_rn(span, uu));
        return __double2float_rn(v);
    };
    const int64_t n = job.n;
    const bool vec = (n % 8 == 0) && ((reinterpret_cast<uintptr_t>(job.out) & 15) == 0);
    if (DT == PGMOE_BF16) {
        uint16_t *o = static_cast<uint16_t *>(job.out);
        if (vec) {
            for (int64_t i = 0; i < n; i += 8) {
                uint32_t w[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t a = __bfloat16_as_ushort(__float2bfloat16_rn(next()));
                    const uint32_t b = __bfloat16_as_ushort(__float2bfloat16_rn(next()));
                    w[q] = a | (b << 16);
                }
                *reinterpret_cast<uint4 *>(o + i) = make_uint4(w[0], w[1], w[2], w[3]);
            }
        } else {
            for (int64_t i = 0; i < n; ++i) o[i] = __bfloat16_as_ushort(__float2bfloat16_rn(next()));
        }
    } else {
        float *o = static_cast<float *>(job.out);
        if (vec) {
            for (int64_t i = 0; i < n; i += 8) {
                float v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = next();
                reinterpret_cast<float4 *>(o + i)[0] = make_float4(v[0], v[1], v[2], v[3]);
                reinterpret_cast<float4 *>(o + i)[1] = make_float4(v[4], v[5], v[6], v[7]);
            }
        } else {
            for (int64_t i = 0; i < n; ++i) o[i] = next();
        }
    }
}

int gen_matrices(const GenJob *jobs_dev, int njobs, int wdtype, cudaStream_t s) {
    if (njobs == 0) return PGMOE_OK;
    const int threads = 32;  // one matrix per thread: spread matrices over SMs
    const int grid = (njobs + threads - 1) / threads;
    if (wdtype == PGMOE_BF16) gen_kernel<PGMOE_BF16><<<grid, threads, 0, s>>>(jobs_dev, njobs);
    else gen_kernel<PGMOE_F32><<<grid, threads, 0, s>>>(jobs_dev, njobs);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}

}  // namespace pgmoe

using namespace pgmoe;

extern "C" int pgmoe_fill_weights(void *out, int32_t wdtype, uint64_t seed, int32_t tag, int32_t block,
                                  int32_t expert, int64_t rows, int64_t cols, pgmoe_stream_t stream) {
    PG_REQUIRE(wdtype == PGMOE_F32 || wdtype == PGMOE_BF16, PGMOE_E_CONFIG, "bad dtype %d", wdtype);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    GenJob job{out, matrix_seed(seed, tag, block, expert), rows * cols};
    GenJob *dj = nullptr;
    PG_CUDA(cudaMallocAsync(&dj, sizeof(GenJob), s));
    PG_CUDA(cudaMemcpyAsync(dj, &job, sizeof(GenJob), cudaMemcpyHostToDevice, s));
    int st = gen_matrices(dj, 1, wdtype, s);
    PG_CUDA(cudaFreeAsync(dj, s));
    PG_CUDA(cudaStreamSynchronize(s));
    return st;
}
