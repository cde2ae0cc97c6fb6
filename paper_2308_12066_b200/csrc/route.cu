// route.cu — K1: pre-gate / route, fused with histogram, scan and a stable
// permutation.  Replaces gate_forward (core.py:284-305) for T tokens.
//
// Routing must equal the reference bit-for-bit.  The reference's logits are
// fp64 sums accumulated serially over i ascending with every product
// rounded (linalg.py:25-38).  Inputs here are fp32 activations and fp32/bf16
// weights, so every product x_i*G_ij is EXACT in fp64; only the summation
// order differs.  Any summation order of n terms has |error| <=
// gamma_{n-1} * sum|p_i| (gamma_n = n*u/(1-n*u)), so both our fast
// parallel sum f_j and the reference's serial sum s_j lie within
// b_j = 2*gamma_{d}*sum_i |p_i| of each other.  If the top-k intervals
// [f-b, f+b] are strictly separated from everything ranked below, the
// reference order is certified; otherwise the candidates that could reach
// the top-k are recomputed in exactly the reference order (serial
// __dadd_rn/__dmul_rn) and ranked with the reference key (-logit, id).
// The fallback count is reported: ids equal the serial-fp64 ranking by
// construction (flips against the reference are measured by the tests and
// bench.py on the same inputs, not assumed).
//
// One kernel, grid (token tiles x K splits):
//   1. every CTA accumulates fp64 partial logits of TOK tokens over its K
//      slice (V adjacent experts per thread, exact products -> one rounding
//      per DFMA) and the slice's column max |G|;
//   2. the last CTA of a token tile (atomic ticket) sums the split partials
//      in split order, bounds the error by sum|x| * max|G|, certifies or
//      recomputes, softmaxes and writes ids & weights (one warp per token);
//   3. the last token tile builds the histogram, exclusive scan, stable
//      permutation and active-expert list.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "common.cuh"
#include "route_common.cuh"

namespace pgmoe {

constexpr int kLogitThreads = 256;
constexpr int kSelectWarps = 8;  // one warp per token of a tile (TOK <= 8)
constexpr int kSelectThreads = kLogitThreads;
constexpr int kMaxTiles = 8192;
constexpr int kMaxSplits = 64;

struct RouteParams {
    const void *x;  // [T][d] fp32, or fp64 (the drop-in's reference-precision inputs)
    const void *G;
    int T, d, E, k;
    int tok;      // tokens per logits CTA
    int splits;   // K splits
    pgmoe_routing out;
    int *counter;      // workspace: token tiles finished (reset by the last one)
    int *tile_counter; // workspace: [tiles] K splits finished per token tile
    double *plogit;    // workspace: [splits][T][E]
    float *pcmax;      // workspace: [tiles][splits][E] column max |G| of each K slice
    double *pxsum;     // workspace: [splits][T] sum |x_i| of each K slice
    unsigned long long *probe;  // debug stamps [tiles*splits][kProbeSlots] or null
};

template <typename GT, typename XT>
__device__ void select_tokens(const RouteParams &p, int tok0, int ntok, unsigned char *base, int *m_ids = nullptr,
                              float *m_w = nullptr);

// fp32/bf16 operands: products exact, d - 1 roundings on either side;
// fp64 operands: one more (the product), gamma_{d+1}
template <typename GT, typename XT>
__device__ __forceinline__ void bound_constants(int d, double *gam, double *bscale) {
    const double u = 1.1102230246251565e-16;  // 2^-53
    const double nd = (double)d + (std::is_same<GT, double>::value || std::is_same<XT, double>::value ? 1.0 : 0.0);
    *gam = nd * u / (1.0 - nd * u);
    *bscale = 2.0 * *gam / (1.0 - *gam) * 1.001;
}

// Phase 2: tokens [tok0, tok0+ntok) of tile `tile`, all splits present.
template <typename GT, typename XT>
__device__ void select_tile(const RouteParams &p, int tile, int tok0, int ntok, unsigned char *smem_raw) {
    const int E = p.E;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ double s_xsum[kSelectWarps];
    double gam, bscale;
    bound_constants<GT, XT>(p.d, &gam, &bscale);
    const double bpad = 1e-300;  // products are exact in fp64: no underflow below ~1e-90
    // sum_i |x_i G_ij| <= (sum_i |x_i|) * max_i |G_ij|; the split CTAs
    // wrote sum |x_i| of their slices.  All split partials are loaded in one
    // batch (16 in flight per thread), then summed in split order.
    if (warp < ntok) {
        double xs = 0.0;
        for (int z = lane; z < p.splits; z += 32) xs += __ldcg(p.pxsum + (size_t)z * p.T + tok0 + warp);
        xs = warp_sumd(xs);
        if (lane == 0) s_xsum[warp] = xs * (1.0 + 2.0 * gam);  // rounding of the fp64 |x| sums
    }
    for (int q = tid; q < ntok * E; q += kSelectThreads) {
        const int t = q / E, j = q - t * E;
        double sum = 0.0;
        float cm = 0.f;
        for (int z0 = 0; z0 < p.splits; z0 += 16) {
            double pl[16];
            float pc[16];
#pragma unroll
            for (int z = 0; z < 16; ++z) {
                pl[z] = (z0 + z < p.splits) ? __ldcg(p.plogit + ((size_t)(z0 + z) * p.T + tok0 + t) * E + j) : 0.0;
                pc[z] = (z0 + z < p.splits) ? __ldcg(p.pcmax + ((size_t)tile * p.splits + z0 + z) * E + j) : 0.f;
            }
#pragma unroll
            for (int z = 0; z < 16; ++z) {  // fixed order: deterministic
                if (z0 + z < p.splits) {
                    sum += pl[z];
                    cm = fmaxf(cm, pc[z]);
                }
            }
        }
        double *lgt = reinterpret_cast<double *>(smem_raw) + (size_t)t * 2 * E;
        lgt[j] = sum;
        lgt[E + j] = (double)cm;
    }
    __syncthreads();
    for (int q = tid; q < ntok * E; q += kSelectThreads) {
        const int t = q / E, j = q - t * E;
        double *lgt = reinterpret_cast<double *>(smem_raw) + (size_t)t * 2 * E;
        lgt[E + j] = bscale * s_xsum[t] * lgt[E + j] + bpad;
    }
    __syncthreads();
    if (tid == 0) probe(p.probe, blockIdx.y * gridDim.x + blockIdx.x, 7);  // partials reduced
    select_tokens<GT, XT>(p, tok0, ntok, smem_raw);
}

// Certified selection + softmax of tokens [tok0, tok0 + ntok), one warp per
// token, from shared memory: token w's fp64 logits at base + w * 2E and
// their error bounds right after them (E doubles each).
template <typename GT, typename XT>
__device__ void select_tokens(const RouteParams &p, int tok0, int ntok, unsigned char *base, int *m_ids,
                              float *m_w) {
    const int d = p.d, E = p.E, k = p.k;
    const GT *G = static_cast<const GT *>(p.G);
    const XT *X = static_cast<const XT *>(p.x);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // The softmax normaliser of the fast logits does not depend on the
    // ranking: when there are idle warps, warp ntok + t computes token t's
    // (max, sum exp) while warp t ranks; a token whose ranking needs the
    // serial recompute (its logits change) redoes it itself.
    __shared__ double s_mz[kSelectWarps][2];
    const bool helpers = 2 * ntok <= kSelectWarps;
    auto normaliser = [&](const double *lg, double &m, double &z) {  // softmax over all E (linalg.py:54-59)
        m = -INFINITY;
        for (int j = lane; j < E; j += 32) m = fmax(m, lg[j]);
        m = warp_max(m);
        z = 0.0;
        for (int j = lane; j < E; j += 32) z += exp(lg[j] - m);
        z = warp_sumd(z);
    };
    if (helpers && warp >= ntok && warp < 2 * ntok) {
        double m, z;
        normaliser(reinterpret_cast<const double *>(base) + (size_t)(warp - ntok) * 2 * E, m, z);
        if (lane == 0) {
            s_mz[warp - ntok][0] = m;
            s_mz[warp - ntok][1] = z;
        }
    }
    const int tok = tok0 + warp;
    double *lg = reinterpret_cast<double *>(base) + (size_t)warp * 2 * E;
    double *bd = lg + E;
    bool finite = true, certified = true;
    int sel[8];
    double minlow = INFINITY;
    if (warp < ntok) {  // tok < p.T follows
        // finite check (core.py:297)
        for (int j = lane; j < E; j += 32) finite &= (bool)isfinite(lg[j]);
        finite = __all_sync(0xffffffffu, finite);
        if (finite) {
            uint32_t taken = 0;  // bit q: expert lane + 32*q taken
            for (int s = 0; s < k; ++s) {
                double bf = -INFINITY;
                int bi = -1;
                for (int j = lane, q = 0; j < E; j += 32, ++q)
                    if (!(taken >> q & 1u) && (bi < 0 || better(lg[j], j, bf, bi))) {
                        bf = lg[j];
                        bi = j;
                    }
                warp_argmax(bf, bi);
                sel[s] = bi;
                if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
                const double low = bf - bd[bi];
                minlow = fmin(minlow, low);
                double up = -INFINITY;
                for (int j = lane, q = 0; j < E; j += 32, ++q)
                    if (!(taken >> q & 1u)) up = fmax(up, lg[j] + bd[j]);
                up = warp_max(up);
                certified &= (low > up);
            }
        }
    }
    if (helpers) __syncthreads();  // normalisers in shared memory; lg no longer read by helpers
    if (warp < ntok) {
        if (!finite) {
            if (lane == 0) atomicCAS(p.out.status, 0, (int)PGMOE_E_GATE_OVERFLOW);
            for (int s = lane; s < k; s += 32) {
                p.out.ids[(size_t)tok * k + s] = 0;
                p.out.w[(size_t)tok * k + s] = 0.f;
                if (m_ids) {
                    m_ids[(size_t)tok * k + s] = 0;
                    m_w[(size_t)tok * k + s] = 0.f;
                }
            }
        } else {
            if (!certified) {
                // Candidates that could be in the reference top-k: recompute
                // them in the reference's serial order.
                uint32_t cand = 0;
                for (int j = lane, q = 0; j < E; j += 32, ++q)
                    if (lg[j] + bd[j] >= minlow) cand |= 1u << q;
                __syncwarp();
                for (int j = lane, q = 0; j < E; j += 32, ++q)
                    if (cand >> q & 1u) lg[j] = serial_logit<GT, XT>(X + (size_t)tok * d, G, d, E, j);
                __syncwarp();
                for (int s = 0; s < k; ++s) {
                    double bf = -INFINITY;
                    int bi = -1;
                    for (int j = lane, q = 0; j < E; j += 32, ++q)
                        if ((cand >> q & 1u) && (bi < 0 || better(lg[j], j, bf, bi))) {
                            bf = lg[j];
                            bi = j;
                        }
                    warp_argmax(bf, bi);
                    sel[s] = bi;
                    if ((bi & 31) == lane) cand &= ~(1u << (bi >> 5));
                }
                if (lane == 0) atomicAdd(p.out.status + 1, 1);
            }
            if (lane == 0 && warp == 0) probe(p.probe, blockIdx.y * gridDim.x + blockIdx.x, 8);  // ranked
            double m, z;
            if (helpers && certified) {
                m = s_mz[warp][0];
                z = s_mz[warp][1];
            } else {
                normaliser(lg, m, z);
            }
            for (int s = 0; s < k; ++s) {
                const double pr = exp(lg[sel[s]] - m) / z;
                if (lane == 0) {
                    if (!(pr > 0.0)) atomicCAS(p.out.status, 0, (int)PGMOE_E_GATE_UNDERFLOW);
                    p.out.ids[(size_t)tok * k + s] = sel[s];
                    p.out.w[(size_t)tok * k + s] = __double2float_rn(pr);
                    if (m_ids) {  // shared-memory copy (the caller permutes from it)
                        m_ids[(size_t)tok * k + s] = sel[s];
                        m_w[(size_t)tok * k + s] = __double2float_rn(pr);
                    }
                }
            }
        }
    }
}

// Permutation of N = T*k <= 32 routed rows by one warp, straight from the
// ids in registers (no shared-memory histogram, no block barriers): row r
// goes to #{rows with a smaller expert} + #{earlier rows, same expert}, the
// same stable order permute_all builds.
__device__ void permute_warp(const RouteParams &p, const int *s_ids = nullptr, const float *s_w = nullptr) {
    const int E = p.E, N = p.T * p.k, lane = threadIdx.x & 31;
    const bool v = lane < N;
    const int e = v ? (s_ids ? s_ids[lane] : __ldcg(p.out.ids + lane)) : 0x7fffffff;
    const float w = v ? (s_w ? s_w[lane] : __ldcg(p.out.w + lane)) : 0.f;
    int ev[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) ev[l] = __shfl_sync(0xffffffffu, e, l);
    int less = 0, before = 0;
#pragma unroll
    for (int l = 0; l < 32; ++l) {
        less += ev[l] < e;
        before += (ev[l] == e) & (l < lane);
    }
    if (v) {
        const int pos = less + before;
        p.out.perm[pos] = lane;
        if (p.out.inv) p.out.inv[lane] = pos;
        p.out.w_perm[pos] = w;
    }
    int nact = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
        const int ex = e0 + lane;
        int h = 0, lt = 0;
#pragma unroll
        for (int l = 0; l < 32; ++l) {  // padding lanes hold INT_MAX: never counted
            h += ev[l] == ex;
            lt += ev[l] < ex;
        }
        const unsigned am = __ballot_sync(0xffffffffu, ex < E && h > 0);
        if (ex < E) {
            p.out.hist[ex] = h;
            p.out.off[ex] = lt;
            if (h > 0) p.out.act[nact + __popc(am & ((1u << lane) - 1u))] = ex;
        }
        nact += __popc(am);
    }
    if (lane == 0) {
        p.out.off[E] = N;
        *p.out.n_act = nact;
    }
}

// permute_warp with the histogram in shared memory (`scratch`: E ints; ids
// and weights from `s_ids` / `s_w` or, when null, from the outputs): N
// smem atomics, one warp scan over E / 32 expert blocks, and the rank of a
// row among its expert's rows by __match_any_sync — no 32-way compare loop
// per expert block.  Same outputs as permute_warp.
__device__ void permute_warp_smem(const RouteParams &p, const int *s_ids, const float *s_w, int *scratch) {
    const int E = p.E, N = p.T * p.k, lane = threadIdx.x & 31;
    const bool v = lane < N;
    const int e = v ? (s_ids ? s_ids[lane] : __ldcg(p.out.ids + lane)) : -1;
    const float w = v ? (s_w ? s_w[lane] : __ldcg(p.out.w + lane)) : 0.f;
    for (int ex = lane; ex < E; ex += 32) scratch[ex] = 0;
    __syncwarp();
    if (v) atomicAdd(&scratch[e], 1);
    __syncwarp();
    const int epl = (E + 31) / 32, b0 = min(E, lane * epl), b1 = min(E, b0 + epl);
    int cnt = 0, na = 0;
    for (int ex = b0; ex < b1; ++ex) {
        const int h = scratch[ex];
        cnt += h;
        na += h > 0;
    }
    int ic = cnt, ia = na;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int c2 = __shfl_up_sync(0xffffffffu, ic, o), a2 = __shfl_up_sync(0xffffffffu, ia, o);
        if (lane >= o) {
            ic += c2;
            ia += a2;
        }
    }
    const int nact = __shfl_sync(0xffffffffu, ia, 31);
    int run = ic - cnt, arun = ia - na;
    __syncwarp();  // every lane has read its counts
    for (int ex = b0; ex < b1; ++ex) {
        const int h = scratch[ex];
        p.out.hist[ex] = h;
        p.out.off[ex] = run;
        if (h > 0) p.out.act[arun++] = ex;
        scratch[ex] = run;  // offset, for the rows below
        run += h;
    }
    const unsigned same = __match_any_sync(0xffffffffu, e);
    __syncwarp();
    if (v) {
        const int pos = scratch[e] + __popc(same & ((1u << lane) - 1u));
        p.out.perm[pos] = lane;
        if (p.out.inv) p.out.inv[lane] = pos;
        p.out.w_perm[pos] = w;
    }
    if (lane == 0) {
        p.out.off[E] = N;
        *p.out.n_act = nact;
    }
}

// Phase 3: histogram, exclusive scan, stable permutation, active list.
__device__ void permute_all(const RouteParams &p, unsigned char *smem_raw) {
    const int E = p.E, k = p.k;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = p.T * k;
    int *whist = reinterpret_cast<int *>(smem_raw);  // [kSelectWarps][E] -> cursors
    int *tot = whist + (size_t)kSelectWarps * E;     // [E]
    for (int i = tid; i < kSelectWarps * E; i += kSelectThreads) whist[i] = 0;
    __syncthreads();
    const int seg = (N + kSelectWarps - 1) / kSelectWarps;
    const int r0 = warp * seg, r1 = min(N, r0 + seg);
    for (int r = r0 + lane; r < r1; r += 32) atomicAdd(&whist[warp * E + __ldcg(p.out.ids + r)], 1);
    __syncthreads();
    for (int e = tid; e < E; e += kSelectThreads) {
        int s = 0;
        for (int w = 0; w < kSelectWarps; ++w) s += whist[w * E + e];
        tot[e] = s;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of tot over E, active list
        int run = 0, nact = 0;
        for (int e0 = 0; e0 < E; e0 += 32) {
            const int e = e0 + lane;
            const int h = e < E ? tot[e] : 0;
            int incl = h;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const unsigned am = __ballot_sync(0xffffffffu, h > 0);
            if (e < E) {
                const int ex = run + incl - h;
                p.out.hist[e] = h;
                p.out.off[e] = ex;
                tot[e] = ex;  // reuse as exclusive offset
                if (h > 0) p.out.act[nact + __popc(am & ((1u << lane) - 1u))] = e;
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
            nact += __popc(am);
        }
        if (lane == 0) {
            p.out.off[E] = run;
            *p.out.n_act = nact;
        }
    }
    __syncthreads();
    if (tid == 0) probe(p.probe, blockIdx.y * gridDim.x + blockIdx.x, 11);  // histogram + scan
    for (int e = tid; e < E; e += kSelectThreads) {
        int base = tot[e];
        for (int w = 0; w < kSelectWarps; ++w) {
            const int c = whist[w * E + e];
            whist[w * E + e] = base;
            base += c;
        }
    }
    __syncthreads();
    const unsigned ltmask = (1u << lane) - 1u;
    for (int c0 = r0; c0 < r1; c0 += 32) {
        const int r = c0 + lane;
        const bool valid = r < r1;
        const unsigned vm = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const int e = __ldcg(p.out.ids + r);
            const unsigned grp = __match_any_sync(vm, e);
            const int rank = __popc(grp & ltmask);
            const int pos = whist[warp * E + e] + rank;
            p.out.perm[pos] = r;
            if (p.out.inv) p.out.inv[r] = pos;
            p.out.w_perm[pos] = __ldcg(p.out.w + r);
            __syncwarp(vm);
            if (rank == __popc(grp) - 1) whist[warp * E + e] += __popc(grp);
        }
        __syncwarp();
    }
}

// Tokens per logits CTA: more tokens re-read each gate row fewer times;
// K splits (up to d/32) keep the grid >= ~2 CTAs per SM at small T.

// Partial logits of TOK tokens over the CTA's K range (phase 1), then the
// tile / global last-arriver phases.  Products of fp32 activations and
// fp32/bf16 gate values are exact in fp64, so every DFMA rounds once, like
// one step of the reference's serial sum.
template <typename GT, typename XT, int TOK, bool VECLOAD>
__global__ void __launch_bounds__(kLogitThreads)
route_kernel(const RouteParams p_in) {
    constexpr int V = Vec<GT>::N;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // parameters copied to shared memory once: the select / permute tails
    // re-read them often, and LDS beats indexed constant-bank reads
    __shared__ RouteParams p_sh;
    static_assert(sizeof(RouteParams) % 4 == 0 && sizeof(RouteParams) / 4 <= kLogitThreads, "params copy");
    if (threadIdx.x < sizeof(RouteParams) / 4)
        reinterpret_cast<int *>(&p_sh)[threadIdx.x] = reinterpret_cast<const int *>(&p_in)[threadIdx.x];
    __syncthreads();
    const RouteParams &p = p_sh;
    const int d = p.d, E = p.E;
    const GT *G = static_cast<const GT *>(p.G);
    const int tile = blockIdx.x;
    const int t0 = tile * TOK;
    const int ntok = min(TOK, p.T - t0);
    const int split = blockIdx.y;
    const int k0 = (int)((long)d * split / p.splits), k1 = (int)((long)d * (split + 1) / p.splits);
    const int kn = k1 - k0;
    const int CG = (E + V - 1) / V;                // column groups
    const int RG = max(1, kLogitThreads / CG);     // row groups
    const int tid = threadIdx.x;
    const int cg = tid % CG, rg = tid / CG;

    double *xd = reinterpret_cast<double *>(smem_raw);                    // [TOK][kn]
    double *red = reinterpret_cast<double *>(smem_raw);                   // reuse: [RG][TOK][E]
    float *redm = reinterpret_cast<float *>(red + (size_t)RG * TOK * E);  // [RG][E]

    const int cta = split * gridDim.x + tile;
    if (tid == 0) probe(p.probe, cta, 0);
    pdl_wait();  // x is produced by the previous kernel in the stream
    // No early trigger: the next launch (a block launch) reads this routing in
    // its prologue, so dependents start only when every CTA has exited or —
    // the permuting CTA — triggered after its last write.
    if (tid == 0) probe(p.probe, cta, 1);
    for (int i = tid; i < TOK * kn; i += kLogitThreads) {
        const int t = i / kn;
        xd[i] = (t < ntok) ? (double)__ldg(static_cast<const XT *>(p.x) + (size_t)(t0 + t) * d + k0 + (i - t * kn))
                           : 0.0;
    }
    __syncthreads();
    {   // sum |x_i| over this K slice, one warp per token (bounds the logit error)
        const int warp = tid >> 5, lane = tid & 31;
        if (warp < ntok) {
            double xs = 0.0;
            for (int i = lane; i < kn; i += 32) xs += fabs(xd[warp * kn + i]);
            xs = warp_sumd(xs);
            if (lane == 0) p.pxsum[(size_t)split * p.T + t0 + warp] = xs;
        }
    }

    double acc[TOK][V];
    float cmax[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        cmax[v] = 0.f;
#pragma unroll
        for (int t = 0; t < TOK; ++t) acc[t][v] = 0.0;
    }
    const int j0 = cg * V;
    constexpr int U = 4;  // gate rows in flight per thread
    if (rg < RG && cg < CG) {
        // U rows per batch with no per-row guard (a guard per row makes each
        // row its own basic block and serialises the load -> convert -> FMA
        // chains); the tail rows one at a time, in the same order
        auto rows = [&](auto nu, int i) {
            constexpr int NU = decltype(nu)::value;
            double gd[NU][V];
            float ga[NU][V];
#pragma unroll
            for (int u = 0; u < NU; ++u) {
                const GT *row = G + (size_t)(k0 + i + u * RG) * E;
                if (VECLOAD) {
                    Vec<GT>::load(row + j0, gd[u], ga[u]);
                } else {
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        gd[u][v] = (j0 + v < E) ? gval(row, j0 + v) : 0.0;
                        ga[u][v] = (j0 + v < E) ? gabs_up(row, j0 + v) : 0.f;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < NU; ++u) {
                const int ii = i + u * RG;
#pragma unroll
                for (int v = 0; v < V; ++v) cmax[v] = fmaxf(cmax[v], ga[u][v]);
#pragma unroll
                for (int t = 0; t < TOK; ++t) {
                    const double xv = xd[t * kn + ii];
#pragma unroll
                    for (int v = 0; v < V; ++v) acc[t][v] = fma(xv, gd[u][v], acc[t][v]);
                }
            }
        };
        int i = rg;
        for (; i + (U - 1) * RG < kn; i += RG * U) rows(std::integral_constant<int, U>{}, i);
        for (; i < kn; i += RG) rows(std::integral_constant<int, 1>{}, i);
    }
    __syncthreads();  // x tile no longer needed: reuse smem for the reduction
    if (rg < RG && cg < CG) {
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (j0 + v < E) {
#pragma unroll
                for (int t = 0; t < TOK; ++t) red[((size_t)rg * TOK + t) * E + j0 + v] = acc[t][v];
                redm[(size_t)rg * E + j0 + v] = cmax[v];
            }
    }
    __syncthreads();
    for (int q = tid; q < ntok * E; q += kLogitThreads) {
        const int t = q / E, j = q - t * E;
        double s = 0.0;
        for (int r = 0; r < RG; ++r) s += red[((size_t)r * TOK + t) * E + j];  // fixed order
        p.plogit[((size_t)split * p.T + t0 + t) * E + j] = s;
    }
    for (int j = tid; j < E; j += kLogitThreads) {
        float m = 0.f;
        for (int r = 0; r < RG; ++r) m = fmaxf(m, redm[(size_t)r * E + j]);
        p.pcmax[((size_t)tile * p.splits + split) * E + j] = m;
    }

    // ---- phase 2: the last split of this token tile selects ---------------
    __shared__ int s_last;
    __syncthreads();
    if (tid == 0) {
        probe(p.probe, cta, 2);  // partial logits written
        __threadfence();
        s_last = (atomicAdd(p.tile_counter + tile, 1) == p.splits - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (tid == 0) probe(p.probe, cta, 3);  // select start
    select_tile<GT, XT>(p, tile, t0, ntok, smem_raw);

    // ---- phase 3: the last token tile permutes ----------------------------
    __syncthreads();
    if (tid == 0) {
        probe(p.probe, cta, 4);  // select done
        p.tile_counter[tile] = 0;
        __threadfence();
        s_last = (atomicAdd(p.counter, 1) == (int)gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (tid == 0) probe(p.probe, cta, 5);  // permute start
    if (p.T * p.k <= 32) {
        if (threadIdx.x < 32) permute_warp(p);
    } else {
        permute_all(p, smem_raw);
    }
    if (tid == 0) {
        *p.counter = 0;
        probe(p.probe, cta, 6);  // permute done
    }
    __threadfence();
    __syncthreads();
    pdl_trigger();
}

// ---------------------------------------------------------------------------
// K1, cluster form (E <= 256, fp32 / bf16 gates).  A token tile of TOK
// tokens is one thread-block cluster of S CTAs; CTA `rank` owns gate rows
// [rank*kn, (rank+1)*kn).  Its gate slice is static weight data, so it is
// staged into shared memory BEFORE the programmatic-dependent-launch wait
// (the load overlaps the previous kernel's tail).  Partial logits, column
// maxima and sum|x| stay in each CTA's shared memory; rank 0 sums them over
// the cluster through distributed shared memory in rank order
// (deterministic), bounds, certifies / recomputes and selects.  No global
// partials, no per-tile atomic ticket: the only global round trip left is
// the permutation's ticket when the batch spans several tiles (a single
// tile permutes straight from shared memory).
// Same arithmetic contract as route_kernel: exact fp64 products, any
// summation order within the certified bound, serial reference fallback.
constexpr int kClusterMaxS = 16;

constexpr size_t kClusterGBytes = 64 * 1024;  // gate slice per CTA

struct ClusterLayout {
    size_t r0, x, part, cm, xs, ext, rp, rc, rs, total;  // byte offsets in dynamic shared memory
};
// register blocking of the partial-logit loop: a thread owns 2 experts x TB tokens
__host__ __device__ constexpr int cl_tb(int tok) { return tok < 4 ? tok : 4; }
__host__ __device__ inline int cl_row_slices(int tok, int E) {
    const int units = (E / 2) * (tok / cl_tb(tok));
    return units >= kLogitThreads ? 1 : kLogitThreads / units;
}
__host__ __device__ inline ClusterLayout cluster_layout(int tok, int kn, int E, size_t gbytes, int S) {
    auto up = [](size_t v) { return (v + 15) & ~(size_t)15; };
    ClusterLayout l;
    size_t r0 = gbytes;                                         // gate slice
    r0 = r0 > (size_t)tok * 2 * E * 8 ? r0 : (size_t)tok * 2 * E * 8;        // rank 0: logits + bounds
    r0 = r0 > (size_t)(kSelectWarps + 1) * E * 4 ? r0 : (size_t)(kSelectWarps + 1) * E * 4;  // permutation
    l.r0 = 0;
    l.x = up(r0);
    l.part = l.x + up((size_t)tok * kn * 8);
    l.cm = l.part + up((size_t)tok * E * 8);
    l.xs = l.cm + up((size_t)E * 4);
    l.ext = l.xs + up((size_t)tok * 8);  // row slices > 0: partial logits + column maxima
    const int rs = cl_row_slices(tok, E);
    // receive buffers of an owning rank (tiles of <= 2 tokens, whose ranks
    // push): every rank's partials of the owned tokens [S][c][E], column
    // maxima [S][E] and slice sums [S][c]
    const int c = tok <= 2 ? (tok + S - 1) / S : 0;
    l.rp = l.ext + up((size_t)(rs - 1) * tok * E * 8) + up((size_t)rs * E * 4);
    l.rc = l.rp + up((size_t)S * c * E * 8);
    l.rs = l.rc + up((size_t)S * E * 4);
    l.total = l.rs + up((size_t)S * c * 8) + 16;
    return l;
}

template <typename GT, int TOK>
__global__ void __launch_bounds__(kLogitThreads) route_cluster_kernel(const RouteParams p_in) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ RouteParams p_sh;
    if (threadIdx.x < sizeof(RouteParams) / 4)
        reinterpret_cast<int *>(&p_sh)[threadIdx.x] = reinterpret_cast<const int *>(&p_in)[threadIdx.x];
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int S = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    __syncthreads();
    const RouteParams &p = p_sh;
    const int d = p.d, E = p.E, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tile = blockIdx.x / S;
    const int t0 = tile * TOK, ntok = min(TOK, p.T - t0);
    const int kn = d / S, k0 = rank * kn;
    const ClusterLayout L = cluster_layout(TOK, kn, E, (size_t)kn * E * sizeof(GT), S);
    GT *sG = reinterpret_cast<GT *>(smem_raw + L.r0);
    double *sx = reinterpret_cast<double *>(smem_raw + L.x);
    double *part = reinterpret_cast<double *>(smem_raw + L.part);
    float *scm = reinterpret_cast<float *>(smem_raw + L.cm);
    double *sxs = reinterpret_cast<double *>(smem_raw + L.xs);
    const int cta = blockIdx.x;
    if (tid == 0) {
        probe(p.probe, cta, 0);
        if (p.probe) p.probe[(size_t)cta * kProbeSlots + 12] = clock64();
    }

    // 1. gate rows [k0, k0 + kn): contiguous, 16-byte vectors, 8 in flight per thread
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(static_cast<const GT *>(p.G) + (size_t)k0 * E);
        uint4 *dst = reinterpret_cast<uint4 *>(sG);
        const int nv = (int)((size_t)kn * E * sizeof(GT) / 16);
        for (int i0 = tid; i0 < nv; i0 += 8 * kLogitThreads) {
            uint4 v[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int i = i0 + b * kLogitThreads;
                if (i < nv) v[b] = __ldg(src + i);
            }
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const int i = i0 + b * kLogitThreads;
                if (i < nv) dst[i] = v[b];
            }
        }
    }
    pdl_wait();  // x is produced by the previous kernel in the stream
    if (tid == 0) probe(p.probe, cta, 1);
    // 2. x slice (fp32 -> fp64, exact), row-major [i][TOK]: a row's tokens are adjacent
    const float *X = static_cast<const float *>(p.x);
    for (int q = tid; q < TOK * kn; q += kLogitThreads) {
        const int t = q / kn, i = q - t * kn;
        sx[i * TOK + t] = t < ntok ? (double)__ldg(X + (size_t)(t0 + t) * d + k0 + i) : 0.0;
    }
    __syncthreads();
    if (warp < TOK) {  // sum |x_i| over the slice (bounds the logit error)
        double v = 0.0;
        for (int i = lane; i < kn; i += 32) v += fabs(sx[i * TOK + warp]);
        v = warp_sumd(v);
        if (lane == 0) sxs[warp] = v;
    }
    if (tid == 0) probe(p.probe, cta, 10);  // x slice in shared memory
    // 3. partial logits, register-blocked: thread (row slice rs, token group tg,
    //    expert pair jp) owns experts 2jp, 2jp+1 for tokens [TB tg, TB tg + TB) over
    //    its rows; per row one gate-pair load and TB/2 16-byte (broadcast) x loads
    //    feed 2 TB independent DFMA chains (the per-DFMA shared-memory load of the
    //    one-expert form kept the loop MIO-bound).  Row slices are added in slice
    //    order: deterministic, and any order is inside the certified bound.
    {
        constexpr int TB = cl_tb(TOK), NTG = TOK / TB;
        const int NP = E / 2, units = NP * NTG, RS = cl_row_slices(TOK, E);
        const int u = tid % units, rs = tid / units;
        const int jp = u % NP, tg = u / NP;
        double *ext = reinterpret_cast<double *>(smem_raw + L.ext);
        float *cmx = reinterpret_cast<float *>(smem_raw + L.ext + (((size_t)(RS - 1) * TOK * E * 8 + 15) & ~(size_t)15));
        if (rs < RS) {
            double acc[TB][2];
#pragma unroll
            for (int tt = 0; tt < TB; ++tt) acc[tt][0] = acc[tt][1] = 0.0;
            float cm0 = 0.f, cm1 = 0.f;
            const int i0 = kn * rs / RS, i1 = kn * (rs + 1) / RS;
            const GT *gp = sG + 2 * jp;
            const double *xp = sx + TB * tg;
            auto row = [&](int i) {
                GT g2[2];
                if constexpr (sizeof(GT) == 2) {
                    const uint32_t w = *reinterpret_cast<const uint32_t *>(gp + (size_t)i * E);
                    g2[0] = (GT)(w & 0xffffu);
                    g2[1] = (GT)(w >> 16);
                } else {
                    const float2 w = *reinterpret_cast<const float2 *>(gp + (size_t)i * E);
                    g2[0] = reinterpret_cast<const GT &>(w.x);
                    g2[1] = reinterpret_cast<const GT &>(w.y);
                }
                const float f0 = WTraits<GT>::f32(g2[0]), f1 = WTraits<GT>::f32(g2[1]);
                cm0 = fmaxf(cm0, fabsf(f0));
                cm1 = fmaxf(cm1, fabsf(f1));
                const double d0 = f0, d1 = f1;
                double xv[TB];
                if constexpr (TB == 4) {
                    const double2 a = *reinterpret_cast<const double2 *>(xp + (size_t)i * TOK);
                    const double2 b = *reinterpret_cast<const double2 *>(xp + (size_t)i * TOK + 2);
                    xv[0] = a.x; xv[1] = a.y; xv[2] = b.x; xv[3] = b.y;
                } else {
#pragma unroll
                    for (int tt = 0; tt < TB; ++tt) xv[tt] = xp[(size_t)i * TOK + tt];
                }
#pragma unroll
                for (int tt = 0; tt < TB; ++tt) {
                    acc[tt][0] = fma(xv[tt], d0, acc[tt][0]);  // exact product, one rounding
                    acc[tt][1] = fma(xv[tt], d1, acc[tt][1]);
                }
            };
            int i = i0;
            for (; i + 4 <= i1; i += 4) {
#pragma unroll
                for (int b = 0; b < 4; ++b) row(i + b);
            }
            for (; i < i1; ++i) row(i);
            double *dst = rs == 0 ? part : ext + (size_t)(rs - 1) * TOK * E;
#pragma unroll
            for (int tt = 0; tt < TB; ++tt) {
                dst[(TB * tg + tt) * E + 2 * jp] = acc[tt][0];
                dst[(TB * tg + tt) * E + 2 * jp + 1] = acc[tt][1];
            }
            if (tg == 0) {
                cmx[rs * E + 2 * jp] = cm0;
                cmx[rs * E + 2 * jp + 1] = cm1;
            }
        }
        __syncthreads();
        if (RS > 1)
            for (int q = tid; q < TOK * E; q += kLogitThreads) {
                double v = part[q];
                for (int z = 1; z < RS; ++z) v += ext[(size_t)(z - 1) * TOK * E + q];
                part[q] = v;
            }
        for (int j = tid; j < E; j += kLogitThreads) {
            float m = cmx[j];
            for (int z = 1; z < RS; ++z) m = fmaxf(m, cmx[z * E + j]);
            scm[j] = m;
        }
    }
    if (tid == 0) probe(p.probe, cta, 2);  // partial logits in shared memory
    // 4a. tiles of <= 2 tokens: push this rank's partials, column maxima and
    //     slice sums to the ranks that own the tokens (remote stores ahead of
    //     the barrier: the owner sums from its own shared memory, no DSMEM
    //     round trip after it; measured -0.4 us at T=1, slower at T >= 8)
    constexpr bool kPush = TOK <= 2;
    const int c = (TOK + S - 1) / S;
    __shared__ int s_sel_ids[TOK * 8];  // one-token tiles: the selection, for the permutation (k <= 8)
    __shared__ float s_sel_w[TOK * 8];
    if constexpr (kPush) {
        __syncthreads();  // part / scm / sxs complete
        double *rp = reinterpret_cast<double *>(smem_raw + L.rp);
        float *rc = reinterpret_cast<float *>(smem_raw + L.rc);
        double *rsx = reinterpret_cast<double *>(smem_raw + L.rs);
        for (int q = tid; q < ntok * E; q += kLogitThreads) {
            const int tl = q / E, j = q - tl * E, o = tl / c;
            cl.map_shared_rank(rp, o)[((size_t)rank * c + (tl - o * c)) * E + j] = part[q];
        }
        const int owners = (ntok + c - 1) / c;
        for (int q = tid; q < owners * E; q += kLogitThreads) {
            const int o = q / E, j = q - o * E;
            cl.map_shared_rank(rc, o)[rank * E + j] = scm[j];
        }
        if (tid < ntok) {
            const int o = tid / c;
            cl.map_shared_rank(rsx, o)[rank * c + (tid - o * c)] = sxs[tid];
        }
    }
    cl.sync();  // every rank's pushes (or partials) visible cluster-wide
    // 4. rank r owns the tile's tokens [r*c, (r+1)*c): sums over the cluster
    //    in rank order, bounds -> [t][logit E | bound E] at r0
    const int own0 = rank * c, nown = max(0, min(c, ntok - own0));
    if (nown > 0) {
        double gam, bscale;
        bound_constants<GT, float>(d, &gam, &bscale);
        double *lgs = reinterpret_cast<double *>(smem_raw + L.r0);
        if constexpr (kPush) {  // from the pushed copies in this CTA
            const double *rp = reinterpret_cast<const double *>(smem_raw + L.rp);
            const float *rc = reinterpret_cast<const float *>(smem_raw + L.rc);
            const double *rsx = reinterpret_cast<const double *>(smem_raw + L.rs);
            for (int q = tid; q < nown * E; q += kLogitThreads) {
                const int tl = q / E, j = q - tl * E;
                double sum = 0.0, sx = 0.0;
                float cm = 0.f;
                for (int z = 0; z < S; ++z) {  // fixed order: deterministic
                    sum += rp[((size_t)z * c + tl) * E + j];
                    cm = fmaxf(cm, rc[z * E + j]);
                    sx += rsx[z * c + tl];
                }
                lgs[tl * 2 * E + j] = sum;
                lgs[tl * 2 * E + E + j] = bscale * (sx * (1.0 + 2.0 * gam)) * (double)cm + 1e-300;
            }
        } else {  // one round of DSMEM loads per (token, expert)
            // the owned tokens' slice sums |x| over the cluster, once per token (rank order)
            __shared__ double s_sx[kSelectWarps];
            if (tid < nown) {
                double xv[kClusterMaxS];
#pragma unroll
                for (int z = 0; z < kClusterMaxS; ++z) xv[z] = z < S ? cl.map_shared_rank(sxs, z)[own0 + tid] : 0.0;
                double sx = 0.0;
#pragma unroll
                for (int z = 0; z < kClusterMaxS; ++z)
                    if (z < S) sx += xv[z];
                s_sx[tid] = sx;
            }
            __syncthreads();  // every thread is past its partial loop: r0 is free; s_sx written
            for (int q = tid; q < nown * E; q += kLogitThreads) {
                const int tl = q / E, j = q - tl * E;
                // one round of DSMEM loads: the S partials and column maxima
                double pv[kClusterMaxS];
                float cv[kClusterMaxS];
#pragma unroll
                for (int z = 0; z < kClusterMaxS; ++z) {
                    pv[z] = z < S ? cl.map_shared_rank(part, z)[(own0 + tl) * E + j] : 0.0;
                    cv[z] = z < S ? cl.map_shared_rank(scm, z)[j] : 0.f;
                }
                double sum = 0.0;
                float cm = 0.f;
#pragma unroll
                for (int z = 0; z < kClusterMaxS; ++z)  // fixed order: deterministic
                    if (z < S) {
                        sum += pv[z];
                        cm = fmaxf(cm, cv[z]);
                    }
                const double sx = s_sx[tl];
                lgs[tl * 2 * E + j] = sum;
                lgs[tl * 2 * E + E + j] = bscale * (sx * (1.0 + 2.0 * gam)) * (double)cm + 1e-300;
            }
        }
        __syncthreads();
        if (tid == 0) probe(p.probe, cta, 3);  // cluster sums done
        // 5. certified selection + softmax (one warp per token)
        if (kPush && ntok <= c)  // one-token tile: rank 0 permutes from its own copy
            select_tokens<GT, float>(p, t0 + own0, nown, smem_raw + L.r0, s_sel_ids, s_sel_w);
        else
            select_tokens<GT, float>(p, t0 + own0, nown, smem_raw + L.r0);
        if (p.T > TOK) __threadfence();  // ids / weights visible GPU-wide before rank 0's ticket
    }
    // every token of the tile owned by rank 0 (a one-token tile): the pushes
    // are complete and nobody reads remote shared memory any more, so the
    // other ranks are done and rank 0 needs no second barrier
    if (!(kPush && ntok <= c)) cl.sync();  // the tile's ids / weights written by their owners
    if (rank != 0) return;
    if (tid == 0) probe(p.probe, cta, 4);  // tile selected
    // 6. permutation: one tile -> straight away; several -> the last tile
    //    through a global ticket
    __shared__ int s_last;
    if (p.T > TOK) {
        if (tid == 0) s_last = (atomicAdd(p.counter, 1) == (int)(gridDim.x / S) - 1);
        __syncthreads();
        if (!s_last) return;
        __threadfence();
    }
    if (tid == 0) probe(p.probe, cta, 5);
    if (p.T * p.k <= 32) {
        if (warp == 0) {
            const bool own = kPush && ntok <= c && p.T <= TOK;  // rank 0 selected every row
            __syncwarp();
            permute_warp_smem(p, own ? s_sel_ids : nullptr, own ? s_sel_w : nullptr,
                              reinterpret_cast<int *>(smem_raw + L.r0));
        }
    } else {
        permute_all(p, smem_raw + L.r0);
    }
    if (tid == 0) {
        if (p.T > TOK) *p.counter = 0;
        probe(p.probe, cta, 6);  // permutation written
        if (p.probe) p.probe[(size_t)cta * kProbeSlots + 13] = clock64();
    }
    __threadfence();
    __syncthreads();
    pdl_trigger();
}

// Cluster size for T tokens: the smallest power of two that puts >= one CTA
// on every SM (at most 16), with the gate slice <= 64 KB and d % S == 0.
static int pick_cluster(int T, int d, int E, size_t gsz, int tok) {
    const int tiles = (T + tok - 1) / tok;
    int S = 1;
    while (S < kClusterMaxS && (long long)tiles * S < kNumSMs) S <<= 1;
    while (S < kClusterMaxS && (size_t)(d / S) * E * gsz > kClusterGBytes) S <<= 1;
    while (S > 1 && d % S != 0) S >>= 1;
    if (d % S != 0 || (size_t)(d / S) * E * gsz > kClusterGBytes) return 0;
    return S;
}

template <typename GT, int TOK>
static int launch_route_cluster(const RouteParams &p, int S, cudaStream_t s) {
    auto kern = route_cluster_kernel<GT, TOK>;
    const int kn = p.d / S;
    const size_t smem = cluster_layout(TOK, kn, p.E, (size_t)kn * p.E * sizeof(GT), S).total;
    static unsigned long long attr_set[2] = {0, 0};  // per device: [0] smem + cluster attrs, [1] S = 16 usable
    const int dev = current_device();
    PG_REQUIRE(dev >= 0 && dev < 64, PGMOE_E_CONFIG, "device ordinal %d unsupported", dev);
    if (!(attr_set[0] & (1ull << dev))) {
        PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr_set[0] |= 1ull << dev;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(((p.T + TOK - 1) / TOK) * S));
    cfg.blockDim = dim3(kLogitThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = (unsigned)S;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (S == kClusterMaxS && !(attr_set[1] & (1ull << dev))) {  // 16-CTA clusters are opt-in: check once
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
            cudaGetLastError();
            return launch_route_cluster<GT, TOK>(p, kClusterMaxS / 2, s);
        }
        attr_set[1] |= 1ull << dev;
    }
    // one wave: a tile that has to wait for a free cluster costs a whole
    // launch (measured: Large-128 T=128, 32 tiles of 8 CTAs, 12 us later);
    // halve the cluster (each CTA then owns twice the gate rows) until every
    // tile is co-resident
    if (S > 1) {
        static int max_clusters[64][kClusterMaxS + 1] = {};  // per device, per S (0: not queried)
        int &mc = max_clusters[dev][S];
        if (mc == 0) {
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
                cudaGetLastError();
                n = 1 << 30;  // unknown: keep the form
            }
            mc = std::max(n, 1);
        }
        const int tiles = (p.T + TOK - 1) / TOK;
        const size_t half_g = (size_t)(p.d / (S / 2)) * p.E * sizeof(GT);
        if (tiles > mc && p.d % (S / 2) == 0 && half_g <= kClusterGBytes) return launch_route_cluster<GT, TOK>(p, S / 2, s);
    }
    PG_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
    count_launch();
    return PGMOE_OK;
}

template <typename GT>
static int route_cluster_dispatch(const RouteParams &p, int tok, int S, cudaStream_t s) {
    if (tok == 1) return launch_route_cluster<GT, 1>(p, S, s);
    if (tok == 2) return launch_route_cluster<GT, 2>(p, S, s);
    if (tok == 4) return launch_route_cluster<GT, 4>(p, S, s);
    return launch_route_cluster<GT, 8>(p, S, s);
}

static int pick_tok(int T) {
    if (T < 64) return 1;
    if (T < 128) return 2;
    if (T < 256) return 4;
    return 8;
}

static int pick_splits(int T, int d, int tok) {
    const int tiles = (T + tok - 1) / tok;
    int s = std::max(1, (2 * kNumSMs) / std::max(1, tiles));
    s = std::min(s, std::max(1, d / 64));  // at least 64 gate rows per CTA
    s = std::min(s, 16);                   // keeps the select kernel's split reduction short
    s = std::max(s, (int)(((size_t)d * tok * 8 + 131071) / 131072));  // x tile fits in shared memory
    return std::min(s, kMaxSplits);
}

template <typename GT>
static size_t route_smem(int tok, int d, int splits, int E) {
    constexpr int V = Vec<GT>::N;
    const int kn = (d + splits - 1) / splits;
    const int CG = (E + V - 1) / V, RG = std::max(1, kLogitThreads / CG);
    const size_t a = (size_t)tok * kn * 8;                              // x tile
    const size_t b = (size_t)RG * tok * E * 8 + (size_t)RG * E * 4;    // split reduction
    const size_t c = (size_t)kSelectWarps * E * 16;                     // select: logit + bound
    const size_t e = (size_t)(kSelectWarps + 1) * E * 4;                // permutation
    return std::max(std::max(a, b), std::max(c, e));
}

template <typename GT, typename XT, int TOK>
static int launch_route(const RouteParams &p, cudaStream_t s) {
    constexpr int V = Vec<GT>::N;
    const size_t smem = route_smem<GT>(TOK, p.d, p.splits, p.E);
    PG_REQUIRE(smem <= 200 * 1024, PGMOE_E_CONFIG, "route: d=%d E=%d exceeds shared memory", p.d, p.E);
    const bool vec = (p.E % V == 0) && (reinterpret_cast<uintptr_t>(p.G) % 16 == 0);
    auto kern = vec ? route_kernel<GT, XT, TOK, true> : route_kernel<GT, XT, TOK, false>;
    static size_t attr[64][2] = {};  // per device
    const int dev = current_device();
    PG_REQUIRE(dev >= 0 && dev < 64, PGMOE_E_CONFIG, "device ordinal %d unsupported", dev);
    if (smem > attr[dev][vec]) {
        const size_t want = std::max<size_t>(smem, 64 * 1024);
        PG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want));
        attr[dev][vec] = want;
    }
    const dim3 grid((p.T + TOK - 1) / TOK, p.splits);
    PG_CUDA(launch_pdl(kern, grid, dim3(kLogitThreads), smem, s, p));
    count_launch();
    return PGMOE_OK;
}

template <typename GT, typename XT = float>
static int route_dispatch(RouteParams p, cudaStream_t s) {
    PG_REQUIRE((p.T + p.tok - 1) / p.tok <= kMaxTiles, PGMOE_E_CONFIG, "route: T=%d too large", p.T);
    if (p.tok == 1) return launch_route<GT, XT, 1>(p, s);
    if (p.tok == 2) return launch_route<GT, XT, 2>(p, s);
    if (p.tok == 4) return launch_route<GT, XT, 4>(p, s);
    return launch_route<GT, XT, 8>(p, s);
}

}  // namespace pgmoe

using namespace pgmoe;

// workspace: [counter | tile counters [kMaxTiles] | plogit f64 [S][T][E] | pcmax f32 [tiles][S][E]]
static size_t ws_head() { return 256 + (size_t)kMaxTiles * 4; }

extern "C" size_t pgmoe_route_workspace_bytes(int32_t T, int32_t E) {
    // the split count depends on the call's T (and d); size for the worst T' <= T
    size_t worst = 0;
    for (int t = 1; t <= std::max(T, 1); ++t) {
        const int tok = pick_tok(t), sp = pick_splits(t, 1 << 20, tok);
        const size_t tiles = (t + tok - 1) / tok;
        worst = std::max(worst, ((size_t)sp * t * 8 + tiles * sp * 4) * std::max(E, 1) + 256 + (size_t)sp * t * 8);
    }
    return ws_head() + worst + 256;
}

static int gate_forward_any(const void *x, bool x64, int32_t T, int32_t d, const void *gate_w, int32_t wdtype,
                            int32_t E, int32_t k, const pgmoe_routing *out, void *workspace, pgmoe_stream_t stream) {
    PG_REQUIRE(out != nullptr && workspace != nullptr, PGMOE_E_CONFIG, "gate_forward: null buffers");
    PG_REQUIRE(gate_w != nullptr && (x != nullptr || T == 0), PGMOE_E_CONFIG, "gate_forward: null inputs");
    PG_REQUIRE(k <= E, PGMOE_E_CONFIG, "k=%d exceeds expert count %d", k, E);
    PG_REQUIRE(k >= 1 && k <= 8, PGMOE_E_CONFIG, "top_k=%d unsupported (1..8)", k);
    PG_REQUIRE(E >= 1 && E <= 1024, PGMOE_E_CONFIG, "num_experts=%d unsupported (1..1024)", E);
    PG_REQUIRE(d >= 1, PGMOE_E_SHAPE, "gate expects input of width %d", d);
    PG_REQUIRE(T >= 0, PGMOE_E_SHAPE, "negative token count");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (T == 0) {
        PG_CUDA(cudaMemsetAsync(out->hist, 0, sizeof(int32_t) * E, s));
        PG_CUDA(cudaMemsetAsync(out->off, 0, sizeof(int32_t) * (E + 1), s));
        PG_CUDA(cudaMemsetAsync(out->n_act, 0, sizeof(int32_t), s));
        return PGMOE_OK;
    }
    char *ws = static_cast<char *>(workspace);
    RouteParams p{};
    p.x = x;
    p.G = gate_w;
    p.T = T;
    p.d = d;
    p.E = E;
    p.k = k;
    p.out = *out;
    p.tok = pick_tok(T);
    p.splits = pick_splits(T, d, p.tok);
    p.counter = reinterpret_cast<int *>(ws);
    p.tile_counter = reinterpret_cast<int *>(ws + 256);
    const size_t n = (size_t)p.splits * T * E;
    p.plogit = reinterpret_cast<double *>(ws + ws_head());
    p.pcmax = reinterpret_cast<float *>(ws + ws_head() + n * 8);
    const size_t ncm = (size_t)((T + p.tok - 1) / p.tok) * p.splits * E;
    p.pxsum = reinterpret_cast<double *>(ws + ws_head() + ((n * 8 + ncm * 4 + 255) & ~(size_t)255));
    p.probe = probe_buffer(0, ((T + p.tok - 1) / p.tok) * p.splits);
    if (x64) {
        PG_REQUIRE(wdtype == PGMOE_F64, PGMOE_E_CONFIG, "fp64 inputs route with fp64 gate weights");
        return route_dispatch<double, double>(p, s);
    }
    // cluster form unless the shape needs the split-partials kernel (E > 256,
    // misaligned gate rows) or PGMOE_ROUTE_KERNEL=split forces it (A/B tests)
    const char *force = getenv("PGMOE_ROUTE_KERNEL");
    const size_t gsz = wdtype == PGMOE_BF16 ? 2 : 4;
    if ((wdtype == PGMOE_BF16 || wdtype == PGMOE_F32) && E <= 256 && ((size_t)E * gsz) % 16 == 0 &&
        (reinterpret_cast<uintptr_t>(gate_w) & 15) == 0 && !(force && strcmp(force, "split") == 0)) {
        // measured (tools/route_bench.py): the cluster form wins at T <= 4 and
        // T >= 128, the split form at 8..64 tokens (more CTAs select in parallel)
        const bool want = (force && strcmp(force, "cluster") == 0) || T <= 4 || T >= 128;
        const int tok = T <= 1 ? 1 : T <= 2 ? 2 : T <= 4 ? 4 : 8;
        const int S = want ? pick_cluster(T, d, E, gsz, tok) : 0;
        if (S > 0 && (T + tok - 1) / tok * S <= (1 << 20)) {
            p.probe = probe_buffer(0, (T + tok - 1) / tok * S);
            return wdtype == PGMOE_BF16 ? route_cluster_dispatch<uint16_t>(p, tok, S, s)
                                        : route_cluster_dispatch<float>(p, tok, S, s);
        }
    }
    if (wdtype == PGMOE_BF16) return route_dispatch<uint16_t>(p, s);
    if (wdtype == PGMOE_F32) return route_dispatch<float>(p, s);
    set_error("unknown weight dtype %d", wdtype);
    return PGMOE_E_CONFIG;
}

extern "C" int pgmoe_gate_forward(const float *x, int32_t T, int32_t d, const void *gate_w, int32_t wdtype,
                                  int32_t E, int32_t k, const pgmoe_routing *out, void *workspace,
                                  pgmoe_stream_t stream) {
    PG_REQUIRE(wdtype == PGMOE_F32 || wdtype == PGMOE_BF16, PGMOE_E_CONFIG,
               "fp32 activations route with fp32 / bf16 gate weights (fp64: pgmoe_gate_forward_f64)");
    return gate_forward_any(x, false, T, d, gate_w, wdtype, E, k, out, workspace, stream);
}

extern "C" int pgmoe_gate_forward_f64(const double *x, int32_t T, int32_t d, const double *gate_w, int32_t E,
                                      int32_t k, const pgmoe_routing *out, void *workspace,
                                      pgmoe_stream_t stream) {
    PG_REQUIRE((reinterpret_cast<uintptr_t>(gate_w) & 15) == 0 || E % 2 != 0, PGMOE_E_CONFIG,
               "fp64 gate weights must be 16-byte aligned");
    return gate_forward_any(x, true, T, d, gate_w, PGMOE_F64, E, k, out, workspace, stream);
}

extern "C" int pgmoe_check_routing(const pgmoe_routing *r, int32_t *fallbacks) {
    int32_t st[4];
    PG_CUDA(cudaMemcpy(st, r->status, sizeof(st), cudaMemcpyDeviceToHost));
    if (fallbacks) *fallbacks = st[1];
    if (st[0] == PGMOE_E_GATE_OVERFLOW) {
        set_error("numerical overflow in gate");
        return PGMOE_E_GATE_OVERFLOW;
    }
    if (st[0] == PGMOE_E_GATE_UNDERFLOW) {
        set_error("gate routing weight underflowed to zero");
        return PGMOE_E_GATE_UNDERFLOW;
    }
    if (st[0] == PGMOE_E_ROUTING) {
        set_error("supplied routing decision invalid (expert id out of range, duplicate id, or combine weight "
                  "outside (0, 1])");
        return PGMOE_E_ROUTING;
    }
    return st[0];
}

// Supplied decisions (core.py:342-364 `supplied_decisions`, synthetic traces
// core.py:436-479): ids/w [T][k] given, gate math bypassed.  One CTA copies
// them into the routing buffer while checking RoutingDecision's invariants
// (core.py:110-140: ids distinct and in [0, E), weights in (0, 1]), then
// builds the same histogram / scan / stable permutation K1 builds.
__global__ void __launch_bounds__(kSelectThreads) route_from_decisions_kernel(const int32_t *__restrict__ ids,
                                                                              const float *__restrict__ w,
                                                                              const RouteParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    const int N = p.T * p.k;
    bool bad = false;
    for (int r = threadIdx.x; r < N; r += kSelectThreads) {
        const int e = __ldg(ids + r);
        const float wv = __ldg(w + r);
        bad |= (e < 0 || e >= p.E || !(wv > 0.f && wv <= 1.f));
        const int t = r / p.k;
        for (int s = t * p.k; s < r; ++s) bad |= (__ldg(ids + s) == e);
        p.out.ids[r] = (e < 0 || e >= p.E) ? 0 : e;  // keep the permutation in range
        p.out.w[r] = wv;
    }
    if (__syncthreads_or(bad)) {
        if (threadIdx.x == 0) atomicCAS(p.out.status, 0, (int)PGMOE_E_ROUTING);
    }
    __threadfence_block();
    __syncthreads();
    permute_all(p, smem_raw);
    __threadfence();
    __syncthreads();
    pdl_trigger();
}

extern "C" int pgmoe_route_from_decisions(const int32_t *ids, const float *w, int32_t T, int32_t E, int32_t k,
                                          const pgmoe_routing *out, pgmoe_stream_t stream) {
    PG_REQUIRE(out != nullptr, PGMOE_E_CONFIG, "route_from_decisions: null routing buffers");
    PG_REQUIRE(k >= 1 && k <= 8 && k <= E, PGMOE_E_CONFIG, "top_k=%d unsupported for E=%d", k, E);
    PG_REQUIRE(E >= 1 && E <= 1024, PGMOE_E_CONFIG, "num_experts=%d unsupported (1..1024)", E);
    PG_REQUIRE(T >= 0, PGMOE_E_SHAPE, "negative token count");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (T == 0) {
        PG_CUDA(cudaMemsetAsync(out->hist, 0, sizeof(int32_t) * E, s));
        PG_CUDA(cudaMemsetAsync(out->off, 0, sizeof(int32_t) * (E + 1), s));
        PG_CUDA(cudaMemsetAsync(out->n_act, 0, sizeof(int32_t), s));
        return PGMOE_OK;
    }
    RouteParams p{};
    p.T = T;
    p.E = E;
    p.k = k;
    p.out = *out;
    const size_t smem = (size_t)(kSelectWarps + 1) * E * 4;
    static bool attr = false;
    if (!attr && smem > 48 * 1024) {
        PG_CUDA(cudaFuncSetAttribute(route_from_decisions_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(smem, 64 * 1024)));
        attr = true;
    }
    PG_CUDA(launch_pdl(route_from_decisions_kernel, dim3(1), dim3(kSelectThreads), smem, s, ids, w, p));
    count_launch();
    return PGMOE_OK;
}
