// ep.cu — expert-parallel helpers: token dispatch packing,
// receiver-side routing over the received rows, and the weighted
// un-permute after the combine exchange.  The exchange itself is NCCL
// all-to-all (torch.distributed) driven from paper_2308_12066_b200/ep.py.
//
// Experts are partitioned contiguously (rank r owns [r*E/P, (r+1)*E/P)), so
// K1's expert-grouped permutation is already grouped by destination rank.
#include <algorithm>

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

// Exclusive scan of v[0, n) in place by the whole CTA (256 threads, n <= 256 * 16);
// returns the total.  Each thread scans a contiguous chunk, chunk totals go
// through a warp scan and a scan of the 8 warp totals.
__device__ int block_exclusive_scan(int *v, int n, int *warp_tot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n + 255) / 256, i0 = min(n, tid * per), i1 = min(n, i0 + per);
    int run = 0;
    for (int i = i0; i < i1; ++i) run += v[i];
    int incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    int base = 0, total = 0;
    for (int w = 0; w < 8; ++w) {
        if (w < warp) base += warp_tot[w];
        total += warp_tot[w];
    }
    int acc = base + incl - run;
    for (int i = i0; i < i1; ++i) {
        const int x = v[i];
        v[i] = acc;
        acc += x;
    }
    __syncthreads();
    return total;
}

// Receiver-side routing of expert-parallel dispatch: rows arrive grouped by
// source rank p (ascending), inside a source grouped by local expert e (the
// sender's K1 permutation is expert-grouped), so local expert e's rows are
// [source 0's e rows, source 1's e rows, ...] — in (source, sender position)
// = global token order within an expert, i.e. the permutation a single GPU
// would build for the concatenated batch.  cnt: [P][El].  One CTA of 256
// threads; counts, offsets and the active list are parallel scans (the
// per-source offset tables of a serial version cost ~20 us per block).
// src_stride > 0: source p's rows start at row p * src_stride (fixed-size,
// padded exchange) instead of right after source p-1's.
// cnt_stride: ints between sources' count rows (El when contiguous).
__global__ void __launch_bounds__(256) ep_local_routing_kernel(const int *__restrict__ cnt, int cnt_stride, int P,
                                                               int El, int src_stride, pgmoe_routing r) {
    extern __shared__ int sm[];
    int *src_base = sm;               // [P]     first received row of source p
    int *src_off = sm + P;            // [P][El] offset of expert e inside source p's rows (scan of cnt)
    int *hist = src_off + P * El;     // [El]    -> exclusive scan: off
    int *actf = hist + El;            // [El]    active flags -> exclusive scan: position in act
    int *wt = actf + El;              // [8]     scan scratch
    const int tid = threadIdx.x;
    for (int i = tid; i < P * El; i += blockDim.x) src_off[i] = __ldg(cnt + (size_t)(i / El) * cnt_stride + i % El);
    __syncthreads();
    for (int e = tid; e < El; e += blockDim.x) {
        int h = 0;
        for (int p = 0; p < P; ++p) h += src_off[p * El + e];
        hist[e] = h;
        actf[e] = h > 0;
        r.hist[e] = h;
    }
    __syncthreads();
    int run = 0;
    for (int p = 0; p < P; ++p) {  // per-source exclusive scans over the experts
        const int tot = block_exclusive_scan(src_off + p * El, El, wt);
        if (tid == 0) src_base[p] = src_stride > 0 ? p * src_stride : run;
        run += tot;
    }
    const int total = block_exclusive_scan(hist, El, wt);
    const int nact = block_exclusive_scan(actf, El, wt);
    for (int e = tid; e < El; e += blockDim.x) {
        r.off[e] = hist[e];
        if ((e + 1 < El ? hist[e + 1] : total) > hist[e]) r.act[actf[e]] = e;  // active: a non-empty range
    }
    if (tid == 0) {
        r.off[El] = total;
        *r.n_act = nact;
    }
    __syncthreads();
    // perm[pos] = received row; one warp per expert
    const int warp = tid >> 5, lane = tid & 31;
    for (int e = warp; e < El; e += blockDim.x >> 5) {
        int pos = hist[e];
        for (int p = 0; p < P; ++p) {
            const int c = __ldg(cnt + (size_t)p * cnt_stride + e);
            const int base = src_base[p] + src_off[p * El + e];
            for (int i = lane; i < c; i += 32) {
                r.perm[pos + i] = base + i;
                r.w_perm[pos + i] = 1.0f;
                if (r.ids) r.ids[base + i] = e;
                if (r.w) r.w[base + i] = 1.0f;
            }
            pos += c;
        }
    }
}

// Received row of local routing position pos: expert e = the last with
// off[e] <= pos (a non-empty range), then the sources in order (counts cnt[p][e],
// rows of e inside source p's slot at src_off[p][e]).
__device__ __forceinline__ int ep_row_of(int pos, const int *off, const int *cnt, const int *src_off, int P, int El,
                                         int slot) {
    int lo = 0, hi = El - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= pos) lo = mid;
        else hi = mid - 1;
    }
    int j = pos - off[lo];
    for (int p = 0; p < P; ++p) {
        const int c = cnt[p * El + lo];
        if (j < c) return p * slot + src_off[p * El + lo] + j;
        j -= c;
    }
    return 0;  // unreachable for pos < total
}

// The receiver side of the fixed-size exchange in one launch: every CTA builds
// the local routing tables from the counts headers in shared memory (E =
// P*El ints); CTA 0 publishes them (the pgmoe_routing a single GPU would build
// for the concatenated batch, as ep_local_routing_kernel) and all CTAs pack the
// received bf16 rows into local-expert order (xb, the FFN's operand).
__global__ void __launch_bounds__(256) ep_recv_route_pack_kernel(const uint16_t *__restrict__ recv,
                                                                 const int *__restrict__ cnt_g, int cnt_stride, int P,
                                                                 int El, int slot, int d, int n_max, pgmoe_routing r,
                                                                 uint16_t *__restrict__ xb) {
    extern __shared__ int sm[];
    int *cnt = sm;                   // [P][El] counts
    int *src_off = cnt + P * El;     // [P][El] -> offsets of expert e inside source p's rows
    int *hist = src_off + P * El;    // [El]    -> exclusive scan: off
    int *actf = hist + El;           // [El]    -> exclusive scan: position in act
    int *wt = actf + El;             // [8]
    const int tid = threadIdx.x;
    const bool pub = blockIdx.x == 0;
    for (int i = tid; i < P * El; i += blockDim.x) {
        const int v = __ldg(cnt_g + (size_t)(i / El) * cnt_stride + i % El);
        cnt[i] = v;
        src_off[i] = v;
    }
    __syncthreads();
    for (int e = tid; e < El; e += blockDim.x) {
        int h = 0;
        for (int p = 0; p < P; ++p) h += cnt[p * El + e];
        hist[e] = h;
        actf[e] = h > 0;
        if (pub) r.hist[e] = h;
    }
    __syncthreads();
    for (int p = 0; p < P; ++p) block_exclusive_scan(src_off + p * El, El, wt);
    const int total = block_exclusive_scan(hist, El, wt);
    const int nact = block_exclusive_scan(actf, El, wt);
    if (pub) {
        for (int e = tid; e < El; e += blockDim.x) {
            r.off[e] = hist[e];
            if ((e + 1 < El ? hist[e + 1] : total) > hist[e]) r.act[actf[e]] = e;
        }
        if (tid == 0) {
            r.off[El] = total;
            *r.n_act = nact;
        }
        for (int pos = tid; pos < total; pos += blockDim.x) {
            const int row = ep_row_of(pos, hist, cnt, src_off, P, El, slot);
            r.perm[pos] = row;
            r.w_perm[pos] = 1.0f;
            if (r.ids || r.w) {
                int lo = 0, hi = El - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (hist[mid] <= pos) lo = mid;
                    else hi = mid - 1;
                }
                if (r.ids) r.ids[row] = lo;
                if (r.w) r.w[row] = 1.0f;
            }
        }
    }
    const int vec = d / 8, n = min(n_max, total);
    for (long long i = blockIdx.x * (long long)blockDim.x + tid; i < (long long)n * vec;
         i += (long long)gridDim.x * blockDim.x) {
        const int pos = (int)(i / vec), c = (int)(i - (long long)pos * vec);
        const int row = ep_row_of(pos, hist, cnt, src_off, P, El, slot);
        reinterpret_cast<uint4 *>(xb)[(size_t)pos * vec + c] =
            __ldg(reinterpret_cast<const uint4 *>(recv) + (size_t)row * vec + c);
    }
}

// ---- fixed-size (padded) exchange: no host round trip for split sizes ----
// Rank p owns experts [p*El, (p+1)*El), so K1's expert-grouped permutation
// sends a contiguous run of routing positions to each peer: positions
// [off[p*El], off[(p+1)*El]).  Each peer gets a fixed slot of `cap` rows.

__device__ __forceinline__ int owner_of(const int *off, int El, int P, int r) {
    int p = 0;
    while (p + 1 < P && __ldg(off + (p + 1) * El) <= r) ++p;
    return p;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a)) |
           ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b)) << 16);
}

// Each peer's slot is `slot` rows: cap routed rows, then header rows whose
// bytes carry this rank's per-expert counts for that peer (int32 [El]), so
// the counts travel in the same all-to-all as the rows.
__host__ __device__ inline int ep_header_rows(int El, int d) { return (El * 4 + 2 * d - 1) / (2 * d); }

// send[p][i] = bf16(x[perm[r] / k]) for r = off[p*El] + i (the rows the
// FFN consumes in bf16 anyway, so the exchange is exact and half the bytes);
// send[p][cap..] = hist[p*El .. (p+1)*El) as int32
__global__ void ep_pack_send_kernel(const float *__restrict__ x, const int *__restrict__ perm,
                                    const int *__restrict__ off, const int *__restrict__ hist, int n, int d, int k,
                                    int P, int El, int cap, int slot, uint16_t *__restrict__ send) {
    const int vec = d / 8;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P * El; i += gridDim.x * blockDim.x) {
        const int p = i / El, e = i - p * El;
        reinterpret_cast<int *>(send + ((size_t)p * slot + cap) * d)[e] = __ldg(hist + i);
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * vec;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / vec), c = (int)(i - (long long)r * vec);
        const int p = owner_of(off, El, P, r);
        const int row = r - __ldg(off + p * El);
        const float4 *src = reinterpret_cast<const float4 *>(x + (size_t)(__ldg(perm + r) / k) * d) + 2 * c;
        const float4 a = __ldg(src), b = __ldg(src + 1);
        uint4 o;
        o.x = pack_bf16x2(a.x, a.y);
        o.y = pack_bf16x2(a.z, a.w);
        o.z = pack_bf16x2(b.x, b.y);
        o.w = pack_bf16x2(b.z, b.w);
        reinterpret_cast<uint4 *>(send)[((size_t)p * slot + row) * vec + c] = o;
    }
}

// xb[pos] = recv[perm[pos]] for pos < off[El] (device count): the received
// bf16 rows in local-expert order, the tcgen05 FFN's packed operand
__global__ void ep_pack_recv_kernel(const uint16_t *__restrict__ recv, const int *__restrict__ perm,
                                    const int *__restrict__ off_end, int n_max, int d, uint16_t *__restrict__ xb) {
    const int vec = d / 8;
    const int n = min(n_max, __ldg(off_end));
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * vec;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / vec), c = (int)(i - (long long)r * vec);
        reinterpret_cast<uint4 *>(xb)[(size_t)r * vec + c] =
            __ldg(reinterpret_cast<const uint4 *>(recv) + (size_t)__ldg(perm + r) * vec + c);
    }
}

// yw[perm[r]] = w_perm[r] * back[p][r - off[p*El]] (the combine weight)
__global__ void ep_unpermute_padded_kernel(const float *__restrict__ back, const int *__restrict__ perm,
                                           const float *__restrict__ w_perm, const int *__restrict__ off, int n,
                                           int d, int P, int El, int slot, float *__restrict__ yw) {
    const int vec = d / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * vec;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / vec), c = (int)(i - (long long)r * vec);
        const int p = owner_of(off, El, P, r);
        const size_t row = (size_t)p * slot + (r - __ldg(off + p * El));
        const float w = __ldg(w_perm + r);
        float4 v = __ldg(reinterpret_cast<const float4 *>(back) + row * vec + c);
        v.x *= w; v.y *= w; v.z *= w; v.w *= w;
        reinterpret_cast<float4 *>(yw)[(size_t)__ldg(perm + r) * vec + c] = v;
    }
}

// Top-1 combine straight into the dense layer's bf16 operand: mixb[t] =
// bf16(w * y) — the same product and rounding the fused single-GPU down
// epilogue writes (so EP == one GPU bitwise), one launch fewer per block.
__global__ void ep_unpermute_padded_bf16_kernel(const float *__restrict__ back, const int *__restrict__ perm,
                                                const float *__restrict__ w_perm, const int *__restrict__ off, int n,
                                                int d, int P, int El, int slot, uint16_t *__restrict__ mixb) {
    const int vec = d / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * vec;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / vec), c = (int)(i - (long long)r * vec);
        const int p = owner_of(off, El, P, r);
        const size_t row = (size_t)p * slot + (r - __ldg(off + p * El));
        const float w = __ldg(w_perm + r);
        const float4 v = __ldg(reinterpret_cast<const float4 *>(back) + row * vec + c);
        uint2 o;
        o.x = pack_bf16x2(w * v.x, w * v.y);
        o.y = pack_bf16x2(w * v.z, w * v.w);
        reinterpret_cast<uint2 *>(mixb)[(size_t)__ldg(perm + r) * vec + c] = o;
    }
}

static int grid_for(long long work) { return (int)std::min<long long>(kNumSMs * 8, std::max(1LL, (work + 255) / 256)); }

}  // namespace pgmoe

using namespace pgmoe;

extern "C" int pgmoe_ep_pack_send(const float *x, const pgmoe_routing *r, int32_t T, int32_t d, int32_t k, int32_t P,
                                  int32_t El, int32_t cap, uint16_t *send, pgmoe_stream_t stream) {
    PG_REQUIRE(d % 8 == 0, PGMOE_E_SHAPE, "ep_pack_send needs d %% 8 == 0");
    PG_REQUIRE(cap >= T * k, PGMOE_E_CONFIG, "ep slot of %d rows cannot hold %d routed entries", cap, T * k);
    const int n = T * k;  // n == 0 still sends the (zero) counts
    ep_pack_send_kernel<<<grid_for(std::max((long long)n * d / 8, (long long)P * El)), 256, 0,
                          reinterpret_cast<cudaStream_t>(stream)>>>(x, r->perm, r->off, r->hist, n, d, k, P, El, cap,
                                                                    cap + ep_header_rows(El, d), send);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}

extern "C" int pgmoe_ep_pack_recv(const uint16_t *recv, const pgmoe_routing *local, int32_t El, int32_t n_max,
                                  int32_t d, uint16_t *xb, pgmoe_stream_t stream) {
    PG_REQUIRE(d % 8 == 0, PGMOE_E_SHAPE, "ep_pack_recv needs d %% 8 == 0");
    if (n_max == 0) return PGMOE_OK;
    ep_pack_recv_kernel<<<grid_for((long long)n_max * d / 8), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        recv, local->perm, local->off + El, n_max, d, xb);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}

extern "C" int pgmoe_ep_unpermute_padded(const float *back, const pgmoe_routing *r, int32_t T, int32_t d, int32_t k,
                                         int32_t P, int32_t El, int32_t cap, float *yw, pgmoe_stream_t stream) {
    PG_REQUIRE(d % 4 == 0, PGMOE_E_SHAPE, "ep_unpermute needs d %% 4 == 0");
    const int n = T * k;
    if (n == 0) return PGMOE_OK;
    ep_unpermute_padded_kernel<<<grid_for((long long)n * d / 4), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        back, r->perm, r->w_perm, r->off, n, d, P, El, cap + ep_header_rows(El, d), yw);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}

extern "C" int pgmoe_ep_unpermute_padded_bf16(const float *back, const pgmoe_routing *r, int32_t T, int32_t d,
                                              int32_t P, int32_t El, int32_t cap, uint16_t *mixb,
                                              pgmoe_stream_t stream) {
    PG_REQUIRE(d % 4 == 0, PGMOE_E_SHAPE, "ep_unpermute needs d %% 4 == 0");
    if (T == 0) return PGMOE_OK;
    ep_unpermute_padded_bf16_kernel<<<grid_for((long long)T * d / 4), 256, 0,
                                      reinterpret_cast<cudaStream_t>(stream)>>>(
        back, r->perm, r->w_perm, r->off, T, d, P, El, cap + ep_header_rows(El, d), mixb);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}

extern "C" int32_t pgmoe_ep_slot_rows(int32_t cap, int32_t El, int32_t d) { return cap + ep_header_rows(El, d); }

extern "C" int pgmoe_ep_local_routing_padded(const uint16_t *recv, int32_t P, int32_t El, int32_t cap, int32_t d,
                                             const pgmoe_routing *out, pgmoe_stream_t stream) {
    PG_REQUIRE(P >= 1 && El >= 1 && cap >= 1 && d >= 1, PGMOE_E_CONFIG, "bad EP shape P=%d El=%d cap=%d", P, El, cap);
    const size_t smem = (size_t)(P + P * El + 2 * El + 8) * 4;
    PG_REQUIRE(smem <= 48 * 1024 && El <= 256 * 16, PGMOE_E_CONFIG, "EP routing table too large");
    const int slot = cap + ep_header_rows(El, d);
    // counts of source p: the header of its slot (slot * d bf16 = slot * d / 2 ints apart)
    const int *cnt = reinterpret_cast<const int *>(recv + (size_t)cap * d);
    PG_REQUIRE(d % 2 == 0, PGMOE_E_SHAPE, "ep header needs an even d");
    ep_local_routing_kernel<<<1, 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(cnt, slot * d / 2, P, El, slot,
                                                                                      *out);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}

extern "C" int pgmoe_ep_recv_route_pack(const uint16_t *recv, int32_t P, int32_t El, int32_t cap, int32_t d,
                                        const pgmoe_routing *out, uint16_t *xb, pgmoe_stream_t stream) {
    PG_REQUIRE(P >= 1 && El >= 1 && cap >= 1 && d >= 1, PGMOE_E_CONFIG, "bad EP shape P=%d El=%d cap=%d", P, El, cap);
    PG_REQUIRE(d % 8 == 0, PGMOE_E_SHAPE, "ep_recv_route_pack needs d %% 8 == 0");
    const size_t smem = (size_t)(2 * P * El + 2 * El + 8) * 4;
    PG_REQUIRE(smem <= 48 * 1024, PGMOE_E_CONFIG, "EP routing table too large");
    const int slot = cap + ep_header_rows(El, d);
    const int *cnt = reinterpret_cast<const int *>(recv + (size_t)cap * d);  // source p's header: slot * d / 2 ints apart
    const int n_max = P * cap;
    ep_recv_route_pack_kernel<<<grid_for((long long)n_max * d / 8), 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
        recv, cnt, slot * d / 2, P, El, slot, d, n_max, *out, xb);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}

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
    const size_t smem = (size_t)(P + P * El + 2 * El + 8) * 4;
    PG_REQUIRE(smem <= 48 * 1024 && El <= 256 * 16, PGMOE_E_CONFIG, "EP routing table too large");
    ep_local_routing_kernel<<<1, 256, smem, reinterpret_cast<cudaStream_t>(stream)>>>(recv_cnt, El, P, El, 0, *out);
    PG_CUDA(cudaGetLastError());
    count_launch();
    return PGMOE_OK;
}
