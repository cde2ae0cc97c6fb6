// ffn_simt.cu — K2/K3 on CUDA cores: grouped GEMV-style expert FFN with the
// combine fused into the down-projection epilogue, and the dense layer.
//
// This is the fp32-weight path (fp32 accumulate, rel. error ~1e-6 vs the
// fp64 reference) and the reference path the tcgen05 kernels are checked
// against.  Persistent grid (multiple of the SM count); each warp owns RW
// weight rows of one active expert and streams them once with 16-byte
// loads while NT routed token rows are broadcast from L1/L2.
#include "common.cuh"

namespace pgmoe {

enum GemvMode { kUp = 0, kDown = 1, kDense = 2 };

struct GemvParams {
    const unsigned char *W;  // weight base
    size_t expert_stride;    // bytes between expert records (0 for dense)
    size_t w_offset;         // byte offset of this matrix inside a record
    int M, K;                // rows (outputs), reduction length
    int indexed_by_act;      // 0: record e at e*stride; 1: at i*stride (slot)
    const int *act, *n_act, *off, *hist, *perm;
    const float *w_perm;
    const float *src;        // kUp: x [T][K]; kDown: h [T*k][K]; kDense: yw [T*k][K]
    float *dst;              // kUp: h [T*k][M]; kDown: yw [T*k][M]; kDense: y [T][M]
    int T, k;
    int mode;                // GemvMode
};

constexpr int RW = 4;  // weight rows per warp
constexpr int NT = 4;  // tokens per pass

template <typename WT>
__device__ __forceinline__ void load8(const WT *p, float (&o)[8]);
template <>
__device__ __forceinline__ void load8<uint16_t>(const uint16_t *p, float (&o)[8]) {
    uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        o[2 * i] = __uint_as_float(w[i] << 16);
        o[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}
template <>
__device__ __forceinline__ void load8<float>(const float *p, float (&o)[8]) {
    float4 a = __ldg(reinterpret_cast<const float4 *>(p));
    float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
    o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}

// Source row of B column n (token slot) for the three modes, as an fp32
// pointer list: kDense sums k slot rows in routing order (linalg.py:45-51).
template <typename WT, bool VEC>
__global__ void __launch_bounds__(256)
gemv_grouped_kernel(GemvParams p) {
    const int lane = threadIdx.x & 31;
    const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int groups = (p.mode == kDense) ? 1 : *p.n_act;
    const int rblocks = (p.M + RW - 1) / RW;
    const long units = (long)groups * rblocks;
    for (long u = gwarp; u < units; u += nwarps) {
        const int g = (int)(u / rblocks);
        const int m0 = (int)(u - (long)g * rblocks) * RW;
        int e = 0, tok0 = 0, ntok = p.T;
        const unsigned char *rec = p.W + p.w_offset;
        if (p.mode != kDense) {
            e = p.act[g];
            tok0 = p.off[e];
            ntok = p.hist[e];
            rec += (size_t)(p.indexed_by_act ? g : e) * p.expert_stride;
        }
        const WT *Wm = reinterpret_cast<const WT *>(rec);
        for (int n0 = 0; n0 < ntok; n0 += NT) {
            const float *srow[NT][8];
            int nrows[NT];
#pragma unroll
            for (int n = 0; n < NT; ++n) {
                nrows[n] = 0;
                const int col = n0 + n;
                if (col < ntok) {
                    if (p.mode == kUp) {
                        srow[n][0] = p.src + (size_t)(p.perm[tok0 + col] / p.k) * p.K;
                        nrows[n] = 1;
                    } else if (p.mode == kDown) {
                        srow[n][0] = p.src + (size_t)(tok0 + col) * p.K;
                        nrows[n] = 1;
                    } else {
                        for (int s = 0; s < p.k && s < 8; ++s)
                            srow[n][s] = p.src + ((size_t)col * p.k + s) * p.K;
                        nrows[n] = p.k;
                    }
                }
            }
            float acc[RW][NT];
#pragma unroll
            for (int r = 0; r < RW; ++r)
#pragma unroll
                for (int n = 0; n < NT; ++n) acc[r][n] = 0.f;
            if (VEC) {
                for (int kk = lane * 8; kk < p.K; kk += 256) {
                    float xv[NT][8];
#pragma unroll
                    for (int n = 0; n < NT; ++n) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) xv[n][q] = 0.f;
                        for (int s = 0; s < nrows[n]; ++s) {
                            const float4 a = __ldg(reinterpret_cast<const float4 *>(srow[n][s] + kk));
                            const float4 b = __ldg(reinterpret_cast<const float4 *>(srow[n][s] + kk) + 1);
                            xv[n][0] += a.x; xv[n][1] += a.y; xv[n][2] += a.z; xv[n][3] += a.w;
                            xv[n][4] += b.x; xv[n][5] += b.y; xv[n][6] += b.z; xv[n][7] += b.w;
                        }
                    }
#pragma unroll
                    for (int r = 0; r < RW; ++r) {
                        if (m0 + r < p.M) {
                            float wv[8];
                            load8<WT>(Wm + (size_t)(m0 + r) * p.K + kk, wv);
#pragma unroll
                            for (int n = 0; n < NT; ++n)
#pragma unroll
                                for (int q = 0; q < 8; ++q) acc[r][n] = fmaf(wv[q], xv[n][q], acc[r][n]);
                        }
                    }
                }
            } else {
                for (int kk = lane; kk < p.K; kk += 32) {
                    float xv[NT];
#pragma unroll
                    for (int n = 0; n < NT; ++n) {
                        xv[n] = 0.f;
                        for (int s = 0; s < nrows[n]; ++s) xv[n] += srow[n][s][kk];
                    }
#pragma unroll
                    for (int r = 0; r < RW; ++r) {
                        if (m0 + r < p.M) {
                            const float wv = WTraits<WT>::f32(Wm[(size_t)(m0 + r) * p.K + kk]);
#pragma unroll
                            for (int n = 0; n < NT; ++n) acc[r][n] = fmaf(wv, xv[n], acc[r][n]);
                        }
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < RW; ++r)
#pragma unroll
                for (int n = 0; n < NT; ++n) acc[r][n] = warp_sum(acc[r][n]);
            // lane (r*NT + n) stores element (m0+r, col n0+n)
            float v = 0.f;
#pragma unroll
            for (int r = 0; r < RW; ++r)
#pragma unroll
                for (int n = 0; n < NT; ++n)
                    if (lane == r * NT + n) v = acc[r][n];
            if (lane < RW * NT) {
                const int r = lane / NT, n = lane % NT;
                const int m = m0 + r, col = n0 + n;
                if (m < p.M && col < ntok) {
                    if (p.mode == kUp) {
                        p.dst[(size_t)(tok0 + col) * p.M + m] = v > 0.f ? v : 0.f;  // relu, linalg.py:41-42
                    } else if (p.mode == kDown) {
                        const int rr = tok0 + col;
                        p.dst[(size_t)p.perm[rr] * p.M + m] = p.w_perm[rr] * v;  // combine weight
                    } else {
                        p.dst[(size_t)col * p.M + m] = v;
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Tiled grouped GEMM for many tokens per expert (fp32 weights, T*k >= 64):
// the GEMV above re-reads every weight row once per 4 tokens; here a 64-row
// x 32-token output tile stages 64 x 32 weight and 32 x 32 token elements
// per k-step in shared memory (transposed, so a thread's 4 rows and 2
// tokens are vector loads) and each thread accumulates a 4 x 2 register
// tile in K order (fp32, like the GEMV).  Units (expert, row tile, token
// tile) are spread over a persistent grid; token tiles of an expert follow
// its routing order (off/hist), so the epilogues (ReLU, combine weight +
// un-permute, dense slot sum) are the GEMV's.
constexpr int TBN = 32, TBK = 32;

// BM = 64 or 32 weight rows per tile (32 when 64-row tiles would leave SMs
// idle: the down projection has only d / 64 row tiles per expert).  The next
// k-step's tiles are loaded into registers while the current one is
// multiplied (one global round trip per k-step hidden behind 32 FMA rounds).
template <typename WT, int BM>
__global__ void __launch_bounds__(256) sgemm_grouped_kernel(GemvParams p) {
    constexpr int RM = BM / 16;            // rows per thread (16 thread rows)
    constexpr int WL = BM * TBK / 4 / 256;  // weight float4 loads per thread per k-step (2 or 1)
    __shared__ __align__(16) float As[TBK][BM + 4];
    __shared__ __align__(16) float Bs[TBK][TBN + 4];
    __shared__ int tile0[1025];  // prefix of tiles per expert group
    __shared__ int wtot[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int groups = (p.mode == kDense) ? 1 : *p.n_act;
    const int mtiles = (p.M + BM - 1) / BM;
    {   // tiles per group (4 groups per thread, loaded in parallel), exclusive scan
        int cnt[4], run = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int g = 4 * tid + q;
            const int ntok = g < groups ? (p.mode == kDense ? p.T : __ldg(p.hist + __ldg(p.act + g))) : 0;
            cnt[q] = mtiles * ((ntok + TBN - 1) / TBN);
            run += cnt[q];
        }
        int incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wtot[warp] = incl;
        __syncthreads();
        int base = 0;
        for (int w = 0; w < warp; ++w) base += wtot[w];
        int acc = base + incl - run;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int g = 4 * tid + q;
            if (g <= groups) tile0[g] = acc;
            acc += cnt[q];
        }
    }
    __syncthreads();
    const int total = tile0[groups];
    const int tx = tid % 16, ty = tid / 16;  // thread tile: rows RM ty .. +RM-1, tokens 2 tx .. +1
    for (int u = blockIdx.x; u < total; u += gridDim.x) {
        int lo = 0, hi = groups - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (tile0[mid] <= u) lo = mid;
            else hi = mid - 1;
        }
        const int g = lo, l = u - tile0[g];
        const int nt = l / mtiles, mt = l - nt * mtiles;
        int e = 0, tok0 = 0, ntok = p.T;
        const unsigned char *rec = p.W + p.w_offset;
        if (p.mode != kDense) {
            e = p.act[g];
            tok0 = p.off[e];
            ntok = p.hist[e];
            rec += (size_t)(p.indexed_by_act ? g : e) * p.expert_stride;
        }
        const WT *Wm = reinterpret_cast<const WT *>(rec);
        const int m0 = mt * BM, n0 = nt * TBN;
        float acc[RM][2];
#pragma unroll
        for (int r = 0; r < RM; ++r) acc[r][0] = acc[r][1] = 0.f;
        // loaders: weights BM rows x 32 k (WL float4 per thread), tokens 32 x 32 (1 float4)
        const int bn = tid / 8, bk = (tid % 8) * 4;
        const int col = n0 + bn;
        const float *srow[8];
        int ns = 0;
        if (col < ntok) {
            if (p.mode == kUp) {
                srow[0] = p.src + (size_t)(p.perm[tok0 + col] / p.k) * p.K;
                ns = 1;
            } else if (p.mode == kDown) {
                srow[0] = p.src + (size_t)(tok0 + col) * p.K;
                ns = 1;
            } else {
                for (int q = 0; q < p.k && q < 8; ++q) srow[q] = p.src + ((size_t)col * p.k + q) * p.K;
                ns = p.k < 8 ? p.k : 8;
            }
        }
        float4 wv[WL], xv;
        auto fetch = [&](int k0) {
#pragma unroll
            for (int h = 0; h < WL; ++h) {
                const int idx = tid + h * 256, wr = idx / 8, wk = (idx % 8) * 4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (m0 + wr < p.M) {
                    if constexpr (sizeof(WT) == 4) {
                        v = __ldg(reinterpret_cast<const float4 *>(Wm + (size_t)(m0 + wr) * p.K + k0 + wk));
                    } else {
                        const uint2 b2 = __ldg(reinterpret_cast<const uint2 *>(Wm + (size_t)(m0 + wr) * p.K + k0 + wk));
                        v = make_float4(__uint_as_float(b2.x << 16), __uint_as_float(b2.x & 0xffff0000u),
                                        __uint_as_float(b2.y << 16), __uint_as_float(b2.y & 0xffff0000u));
                    }
                }
                wv[h] = v;
            }
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int q = 0; q < ns; ++q) {  // kDense: the k slot rows summed in routing order
                const float4 a4 = __ldg(reinterpret_cast<const float4 *>(srow[q] + k0 + bk));
                v.x += a4.x; v.y += a4.y; v.z += a4.z; v.w += a4.w;
            }
            xv = v;
        };
        fetch(0);
        for (int k0 = 0; k0 < p.K; k0 += TBK) {
#pragma unroll
            for (int h = 0; h < WL; ++h) {
                const int idx = tid + h * 256, wr = idx / 8, wk = (idx % 8) * 4;
                As[wk][wr] = wv[h].x;
                As[wk + 1][wr] = wv[h].y;
                As[wk + 2][wr] = wv[h].z;
                As[wk + 3][wr] = wv[h].w;
            }
            Bs[bk][bn] = xv.x;
            Bs[bk + 1][bn] = xv.y;
            Bs[bk + 2][bn] = xv.z;
            Bs[bk + 3][bn] = xv.w;
            __syncthreads();
            if (k0 + TBK < p.K) fetch(k0 + TBK);  // in flight while this step multiplies
#pragma unroll 8
            for (int kk = 0; kk < TBK; ++kk) {
                float av[RM];
                if constexpr (RM == 4) {
                    const float4 a4 = *reinterpret_cast<const float4 *>(&As[kk][4 * ty]);
                    av[0] = a4.x; av[1] = a4.y; av[2] = a4.z; av[3] = a4.w;
                } else {
                    const float2 a2 = *reinterpret_cast<const float2 *>(&As[kk][RM * ty]);
                    av[0] = a2.x; av[1] = a2.y;
                }
                const float2 b = *reinterpret_cast<const float2 *>(&Bs[kk][2 * tx]);
#pragma unroll
                for (int r = 0; r < RM; ++r) {
                    acc[r][0] = fmaf(av[r], b.x, acc[r][0]);
                    acc[r][1] = fmaf(av[r], b.y, acc[r][1]);
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int r = 0; r < RM; ++r)
#pragma unroll
            for (int c2 = 0; c2 < 2; ++c2) {
                const int m = m0 + RM * ty + r, cc = n0 + 2 * tx + c2;
                if (m >= p.M || cc >= ntok) continue;
                const float v = acc[r][c2];
                if (p.mode == kUp) {
                    p.dst[(size_t)(tok0 + cc) * p.M + m] = v > 0.f ? v : 0.f;  // relu, linalg.py:41-42
                } else if (p.mode == kDown) {
                    const int rr = tok0 + cc;
                    p.dst[(size_t)p.perm[rr] * p.M + m] = p.w_perm[rr] * v;  // combine weight
                } else {
                    p.dst[(size_t)cc * p.M + m] = v;
                }
            }
    }
}

template <typename WT>
static int launch_gemv(const GemvParams &p, cudaStream_t s) {
    const bool vec = (p.K % 8 == 0) && (p.w_offset % 16 == 0) && (p.expert_stride % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(p.W) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(p.src) % 16 == 0);
    const int grid = kNumSMs * 4;
    // many tokens per launch: the tiled kernel reads each weight tile once per
    // 32 tokens instead of once per 4 (fp32: 236 GB/s -> see DESIGN §5)
    const bool tiled = vec && p.K % TBK == 0 && (long long)p.T * (p.mode == kDense ? 1 : p.k) >= 64 &&
                       (p.mode == kDense || p.expert_stride % 16 == 0);
    // 32-row tiles when 64-row tiles would not give every SM two units (estimate: T*k tokens spread
    // over min(T*k, E) groups is unknown here; the row count decides)
    if (tiled && p.M / 64 * 8 < 2 * kNumSMs) sgemm_grouped_kernel<WT, 32><<<grid, 256, 0, s>>>(p);
    else if (tiled) sgemm_grouped_kernel<WT, 64><<<grid, 256, 0, s>>>(p);
    else if (vec) gemv_grouped_kernel<WT, true><<<grid, 256, 0, s>>>(p);
    else gemv_grouped_kernel<WT, false><<<grid, 256, 0, s>>>(p);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}

int gemv_dispatch(const GemvParams &p, int wdtype, cudaStream_t s) {
    if (wdtype == PGMOE_BF16) return launch_gemv<uint16_t>(p, s);
    if (wdtype == PGMOE_F32) return launch_gemv<float>(p, s);
    set_error("unknown weight dtype %d", wdtype);
    return PGMOE_E_CONFIG;
}

int expert_ffn_simt(const float *x, int T, int d, int f, int k, const void *experts,
                    size_t stride, int wdtype, int indexed_by_act, const pgmoe_routing *r,
                    float *h, float *yw, cudaStream_t s) {
    GemvParams up{};
    up.W = static_cast<const unsigned char *>(experts);
    up.expert_stride = stride;
    up.w_offset = 0;
    up.M = f;
    up.K = d;
    up.indexed_by_act = indexed_by_act;
    up.act = r->act; up.n_act = r->n_act; up.off = r->off; up.hist = r->hist; up.perm = r->perm;
    up.w_perm = r->w_perm;
    up.src = x;
    up.dst = h;
    up.T = T;
    up.k = k;
    up.mode = kUp;
    PG_TRY(gemv_dispatch(up, wdtype, s));
    GemvParams dn = up;
    dn.w_offset = (size_t)f * d * dtype_bytes(wdtype);
    dn.M = d;
    dn.K = f;
    dn.src = h;
    dn.dst = yw;
    dn.mode = kDown;
    return gemv_dispatch(dn, wdtype, s);
}

int dense_simt(const float *yw, int T, int d, int k, const void *dense_w, int wdtype, float *y,
               cudaStream_t s) {
    GemvParams p{};
    p.W = static_cast<const unsigned char *>(dense_w);
    p.M = d;
    p.K = d;
    p.src = yw;
    p.dst = y;
    p.T = T;
    p.k = k;
    p.mode = kDense;
    return gemv_dispatch(p, wdtype, s);
}

}  // namespace pgmoe
