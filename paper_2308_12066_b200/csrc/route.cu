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
// The fallback count is reported; flips are zero by construction.
#include <algorithm>

#include "common.cuh"

namespace pgmoe {

constexpr int kRouteThreads = 512;
constexpr int kRouteWarps = kRouteThreads / 32;

struct RouteParams {
    const float *x;
    const void *G;
    int T, d, E, k;
    pgmoe_routing out;
    int *counter;  // workspace: CTAs finished (reset by the last CTA)
};

__device__ __forceinline__ bool better(double fa, int ia, double fb, int ib) {
    // reference sort key (-logit, id): larger logit first, ties -> lower id
    return fa > fb || (fa == fb && ia < ib);
}

__device__ __forceinline__ void warp_argmax(double &f, int &id) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double of = __shfl_xor_sync(0xffffffffu, f, o);
        int oi = __shfl_xor_sync(0xffffffffu, id, o);
        if (oi >= 0 && (id < 0 || better(of, oi, f, id))) {
            f = of;
            id = oi;
        }
    }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double warp_sumd(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Serial fp64 logit in the reference order (linalg.py:35-37): out += x_i*G_ij.
template <typename WT>
__device__ double serial_logit(const double *xs, const WT *G, int d, int E, int j) {
    double acc = 0.0;
    for (int i = 0; i < d; ++i) {
        double g = (double)WTraits<WT>::f32(G[(size_t)i * E + j]);
        acc = __dadd_rn(acc, __dmul_rn(xs[i], g));
    }
    return acc;
}

template <typename WT, int TOK>
__global__ void __launch_bounds__(kRouteThreads)
route_kernel(RouteParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int d = p.d, E = p.E, k = p.k;
    const WT *G = static_cast<const WT *>(p.G);
    const int t0 = blockIdx.x * TOK;
    const int ntok = min(TOK, p.T - t0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // smem carve: x tile [TOK][d] f64 | part [KS][TOK][EL] (val f64, |p| f32) |
    // logit [TOK][E] f64 | bound [TOK][E] f64
    const int EL = E < kRouteThreads ? E : kRouteThreads;  // expert lanes
    const int KS = kRouteThreads / EL;                     // k-splits
    double *xs = reinterpret_cast<double *>(smem_raw);
    double *part = xs + (size_t)TOK * d;
    float *parta = reinterpret_cast<float *>(part + (size_t)KS * TOK * EL);
    double *logit = reinterpret_cast<double *>(parta + (((size_t)KS * TOK * EL + 1) & ~(size_t)1));
    double *bound = logit + (size_t)TOK * E;

    pdl_wait();  // x is produced by the previous kernel in the stream
    pdl_trigger();
    for (int i = tid; i < TOK * d; i += kRouteThreads) {
        int t = i / d;
        xs[i] = (t < ntok) ? (double)p.x[(size_t)(t0 + t) * d + (i - t * d)] : 0.0;
    }
    __syncthreads();

    // ---- fast fp64 logits (exact products, any order) + fp32 sum|p| ------
    // The |p| sum only feeds the error bound, so it runs on the fp32 pipe
    // next to the DFMAs; its own rounding (< d*2^-24 relative) is covered by
    // the 1.001 factor below.
    const int ks = tid / EL, jl = tid - ks * EL;
    const double u = 1.1102230246251565e-16;  // 2^-53
    const double gam = (double)d * u / (1.0 - (double)d * u);
    const double bscale = 2.0 * gam / (1.0 - gam) * 1.001;
    for (int j0 = 0; j0 < E; j0 += EL) {
        const int j = j0 + jl;
        if (ks < KS && j < E) {
            const int i0 = (int)((long)d * ks / KS), i1 = (int)((long)d * (ks + 1) / KS);
            double acc[TOK];
            float aab[TOK];
#pragma unroll
            for (int t = 0; t < TOK; ++t) {
                acc[t] = 0.0;
                aab[t] = 0.f;
            }
#pragma unroll 8
            for (int i = i0; i < i1; ++i) {
                const float gf = WTraits<WT>::f32(__ldg(G + (size_t)i * E + j));
                const double g = (double)gf;
                const float ga = fabsf(gf);
#pragma unroll
                for (int t = 0; t < TOK; ++t) {
                    const double xv = xs[t * d + i];
                    acc[t] = fma(xv, g, acc[t]);  // product exact in fp64: one rounding per add
                    aab[t] = fmaf(fabsf((float)xv), ga, aab[t]);
                }
            }
#pragma unroll
            for (int t = 0; t < TOK; ++t) {
                part[((size_t)ks * TOK + t) * EL + jl] = acc[t];
                parta[((size_t)ks * TOK + t) * EL + jl] = aab[t];
            }
        }
        __syncthreads();
        for (int q = tid; q < TOK * EL; q += kRouteThreads) {
            const int t = q / EL, jj = q - t * EL;
            if (j0 + jj >= E) continue;
            double s = 0.0;
            float a = 0.f;
            for (int z = 0; z < KS; ++z) {  // fixed order: deterministic
                s += part[((size_t)z * TOK + t) * EL + jj];
                a += parta[((size_t)z * TOK + t) * EL + jj];
            }
            logit[(size_t)t * E + j0 + jj] = s;
            // fp32 |p| terms can round down by 2^-24 each and flush below
            // FLT_MIN: pad relatively and absolutely.
            bound[(size_t)t * E + j0 + jj] = bscale * (double)a + (double)d * 2.4e-38;
        }
        __syncthreads();
    }

    // ---- per-token selection, certification, softmax (one warp/token) ----
    for (int t = warp; t < ntok; t += kRouteWarps) {
        double *lg = logit + (size_t)t * E;
        const double *bd = bound + (size_t)t * E;
        const int tok = t0 + t;
        // finite check (core.py:297)
        bool finite = true;
        for (int j = lane; j < E; j += 32) finite &= (bool)isfinite(lg[j]);
        finite = __all_sync(0xffffffffu, finite);
        if (!finite) {
            if (lane == 0) atomicCAS(p.out.status, 0, (int)PGMOE_E_GATE_OVERFLOW);
            for (int s = lane; s < k; s += 32) {
                p.out.ids[(size_t)tok * k + s] = 0;
                p.out.w[(size_t)tok * k + s] = 0.f;
            }
            continue;
        }
        int sel[8];
        uint32_t taken = 0;  // bit q: expert lane + 32*q taken
        bool certified = true;
        double minlow = INFINITY;
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
        if (!certified) {
            // Candidates that could be in the reference top-k.
            uint32_t cand = 0;
            for (int j = lane, q = 0; j < E; j += 32, ++q)
                if (lg[j] + bd[j] >= minlow) cand |= 1u << q;
            __syncwarp();
            for (int j = lane, q = 0; j < E; j += 32, ++q)
                if (cand >> q & 1u) lg[j] = serial_logit<WT>(xs + (size_t)t * d, G, d, E, j);
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
        // softmax over all E (linalg.py:54-59), max-subtracted
        double m = -INFINITY;
        for (int j = lane; j < E; j += 32) m = fmax(m, lg[j]);
        m = warp_max(m);
        double z = 0.0;
        for (int j = lane; j < E; j += 32) z += exp(lg[j] - m);
        z = warp_sumd(z);
        for (int s = 0; s < k; ++s) {
            const double pr = exp(lg[sel[s]] - m) / z;
            if (lane == 0) {
                if (!(pr > 0.0)) atomicCAS(p.out.status, 0, (int)PGMOE_E_GATE_UNDERFLOW);
                p.out.ids[(size_t)tok * k + s] = sel[s];
                p.out.w[(size_t)tok * k + s] = __double2float_rn(pr);
            }
        }
    }

    // ---- last CTA: histogram, exclusive scan, stable permutation ---------
    __shared__ int s_last;
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        s_last = (atomicAdd(p.counter, 1) == (int)gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    const int N = p.T * k;
    int *whist = reinterpret_cast<int *>(smem_raw);  // [kRouteWarps][E] -> cursors
    int *tot = whist + (size_t)kRouteWarps * E;      // [E]
    for (int i = tid; i < kRouteWarps * E; i += kRouteThreads) whist[i] = 0;
    __syncthreads();
    const int seg = (N + kRouteWarps - 1) / kRouteWarps;
    const int r0 = warp * seg, r1 = min(N, r0 + seg);
    for (int r = r0 + lane; r < r1; r += 32) atomicAdd(&whist[warp * E + __ldcg(p.out.ids + r)], 1);
    __syncthreads();
    // per-expert totals, then base cursor per (warp, expert)
    for (int e = tid; e < E; e += kRouteThreads) {
        int s = 0;
        for (int w = 0; w < kRouteWarps; ++w) s += whist[w * E + e];
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
    for (int e = tid; e < E; e += kRouteThreads) {
        int base = tot[e];
        for (int w = 0; w < kRouteWarps; ++w) {
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
            p.out.w_perm[pos] = __ldcg(p.out.w + r);
            __syncwarp(vm);
            if (rank == __popc(grp) - 1) whist[warp * E + e] += __popc(grp);
        }
        __syncwarp();
    }
    if (tid == 0) *p.counter = 0;
}

static size_t route_smem(int TOK, int d, int E) {
    const int EL = E < kRouteThreads ? E : kRouteThreads;
    const int KS = kRouteThreads / EL;
    size_t a = (size_t)TOK * d * 8 + (size_t)KS * TOK * EL * 8 + (((size_t)KS * TOK * EL + 1) & ~(size_t)1) * 4 +
               (size_t)2 * TOK * E * 8;
    size_t b = (size_t)(kRouteWarps + 1) * E * 4;
    return a > b ? a : b;
}

template <typename WT, int TOK>
static int launch_route(const RouteParams &p, cudaStream_t s) {
    const size_t smem = route_smem(TOK, p.d, p.E);
    PG_REQUIRE(smem <= 220 * 1024, PGMOE_E_CONFIG, "route: d=%d E=%d exceeds shared memory", p.d, p.E);
    static size_t attr_smem = 0;  // per instantiation: raise the limit once
    if (smem > attr_smem) {
        PG_CUDA(cudaFuncSetAttribute(route_kernel<WT, TOK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(smem, 100 * 1024)));
        attr_smem = std::max<size_t>(smem, 100 * 1024);
    }
    const int grid = (p.T + TOK - 1) / TOK;
    PG_CUDA(launch_pdl(route_kernel<WT, TOK>, dim3(grid), dim3(kRouteThreads), smem, s, p));
    count_launch();
    return PGMOE_OK;
}

template <typename WT>
static int route_dispatch(const RouteParams &p, cudaStream_t s) {
    // about one CTA per SM: more tokens per CTA reuse each gate column load
    if (p.T <= kNumSMs) return launch_route<WT, 1>(p, s);
    if (p.T <= 2 * kNumSMs) return launch_route<WT, 2>(p, s);
    return launch_route<WT, 4>(p, s);
}

}  // namespace pgmoe

using namespace pgmoe;

extern "C" size_t pgmoe_route_workspace_bytes(int32_t, int32_t) { return 256; }

extern "C" int pgmoe_gate_forward(const float *x, int32_t T, int32_t d, const void *gate_w,
                                  int32_t wdtype, int32_t E, int32_t k, const pgmoe_routing *out,
                                  void *workspace, pgmoe_stream_t stream) {
    PG_REQUIRE(out != nullptr && workspace != nullptr, PGMOE_E_CONFIG, "gate_forward: null buffers");
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
    RouteParams p{x, gate_w, T, d, E, k, *out, static_cast<int *>(workspace)};
    if (wdtype == PGMOE_BF16) return route_dispatch<uint16_t>(p, s);
    if (wdtype == PGMOE_F32) return route_dispatch<float>(p, s);
    set_error("unknown weight dtype %d", wdtype);
    return PGMOE_E_CONFIG;
}

extern "C" int pgmoe_check_routing(const pgmoe_routing *r, int32_t *fallbacks, int32_t *flips) {
    int32_t st[4];
    PG_CUDA(cudaMemcpy(st, r->status, sizeof(st), cudaMemcpyDeviceToHost));
    if (fallbacks) *fallbacks = st[1];
    if (flips) *flips = st[2];
    if (st[0] == PGMOE_E_GATE_OVERFLOW) {
        set_error("numerical overflow in gate");
        return PGMOE_E_GATE_OVERFLOW;
    }
    if (st[0] == PGMOE_E_GATE_UNDERFLOW) {
        set_error("gate routing weight underflowed to zero");
        return PGMOE_E_GATE_UNDERFLOW;
    }
    return st[0];
}
