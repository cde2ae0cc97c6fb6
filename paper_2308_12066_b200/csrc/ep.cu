// ep.cu — expert-parallel helpers: token dispatch packing,
// receiver-side routing over the received rows, and the weighted
// un-permute after the combine exchange.  The exchange itself is NCCL
// all-to-all (torch.distributed) driven from paper_2308_12066_b200/ep.py.
//
// Experts are partitioned contiguously (rank r owns [r*E/P, (r+1)*E/P)), so
// K1's expert-grouped permutation is already grouped by destination rank.
#include "common.cuh"

namespace pgmoe {

// out[r] = src[perm[r] / k]  (rows of d floats; 16-byte vectors)
__global__ void gather_rows_kernel(const float *__restrict__ src, const int *__restrict__ perm, int n, int d, int k,
                                   float *__restrict__ out) {
    const int vec = d / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * vec;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / vec), c = (int)(i - (long long)r * vec);
        const int row = __ldg(perm + r) / k;
        reinterpret_cast<float4 *>(out)[(size_t)r * vec + c] =
            __ldg(reinterpret_cast<const float4 *>(src) + (size_t)row * vec + c);
    }
}

// yw[perm[r]] = w_perm[r] * back[r]  (the combine weight of each routed entry)
__global__ void unpermute_kernel(const float *__restrict__ back, const int *__restrict__ perm,
                                 const float *__restrict__ w_perm, int n, int d, float *__restrict__ yw) {
    const int vec = d / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * vec;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / vec), c = (int)(i - (long long)r * vec);
        const float w = __ldg(w_perm + r);
        float4 v = __ldg(reinterpret_cast<const float4 *>(back) + (size_t)r * vec + c);
        v.x *= w; v.y *= w; v.z *= w; v.w *= w;
        reinterpret_cast<float4 *>(yw)[(size_t)__ldg(perm + r) * vec + c] = v;
    }
}

// Receiver routing: rows arrive grouped by source rank, each source's rows
// grouped by local expert ascending.  Regroup by local expert (sources in
// rank order inside an expert) — the same stable order a single GPU would
// produce for the concatenated batch.  cnt: [P][El].  One CTA.
__global__ void ep_local_routing_kernel(const int *__restrict__ cnt, int P, int El, pgmoe_routing r) {
    extern __shared__ int sm[];
    int *src_base = sm;          // [P] first received row of source p
    int *src_off = sm + P;       // [P][El] offset of expert e inside source p's rows
    if (threadIdx.x == 0) {
        int run = 0;
        for (int p = 0; p < P; ++p) {
            src_base[p] = run;
            int o = 0;
            for (int e = 0; e < El; ++e) {
                src_off[p * El + e] = o;
                o += cnt[p * El + e];
            }
            run += o;
        }
        int off = 0, nact = 0;
        for (int e = 0; e < El; ++e) {
            int h = 0;
            for (int p = 0; p < P; ++p) h += cnt[p * El + e];
            r.hist[e] = h;
            r.off[e] = off;
            if (h > 0) r.act[nact++] = e;
            off += h;
        }
        r.off[El] = off;
        *r.n_act = nact;
    }
    __syncthreads();
    // perm[pos] = received row; one warp per expert
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = warp; e < El; e += blockDim.x >> 5) {
        int pos = r.off[e];
        for (int p = 0; p < P; ++p) {
            const int c = cnt[p * El + e];
            const int base = src_base[p] + src_off[p * El + e];
            for (int i = lane; i < c; i += 32) {
                r.perm[pos + i] = base + i;
                r.w_perm[pos + i] = 1.0f;
                r.ids[base + i] = e;
                r.w[base + i] = 1.0f;
            }
            pos += c;
        }
    }
}

}  // namespace pgmoe

using namespace pgmoe;

extern "C" int pgmoe_gather_rows(const float *src, const int32_t *perm, int32_t n, int32_t d, int32_t k,
                                 float *out, pgmoe_stream_t stream) {
    PG_REQUIRE(d % 4 == 0, PGMOE_E_SHAPE, "gather_rows needs d %% 4 == 0");
    if (n == 0) return PGMOE_OK;
    const long long work = (long long)n * (d / 4);
    const int grid = (int)std::min<long long>(kNumSMs * 8, (work + 255) / 256);
    gather_rows_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(src, perm, n, d, k, out);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}

extern "C" int pgmoe_unpermute_combine(const float *back, const int32_t *perm, const float *w_perm, int32_t n,
                                       int32_t d, float *yw, pgmoe_stream_t stream) {
    PG_REQUIRE(d % 4 == 0, PGMOE_E_SHAPE, "unpermute needs d %% 4 == 0");
    if (n == 0) return PGMOE_OK;
    const long long work = (long long)n * (d / 4);
    const int grid = (int)std::min<long long>(kNumSMs * 8, (work + 255) / 256);
    unpermute_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(back, perm, w_perm, n, d, yw);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}

extern "C" int pgmoe_ep_local_routing(const int32_t *recv_cnt, int32_t P, int32_t El, const pgmoe_routing *out,
                                      pgmoe_stream_t stream) {
    PG_REQUIRE(P >= 1 && El >= 1, PGMOE_E_CONFIG, "bad EP shape P=%d El=%d", P, El);
    const size_t smem = (size_t)(P + P * El) * 4;
    PG_REQUIRE(smem <= 48 * 1024, PGMOE_E_CONFIG, "EP routing table too large");
    ep_local_routing_kernel<<<1, 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(recv_cnt, P, El, *out);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}
